#!/bin/bash
# A/B of variants/lib_*.so on config 1 (bench stages) and config 2 (mapping stages), with parity.
mkdir -p gpurun_out
bash tools/ab_bench.sh ${1:-20} 2>&1
for f in variants/lib_*.so; do
  n=$(basename $f .so)
  echo "== $n config 2: $(SPLAT_B200_LIB=$PWD/$f timeout 300 python tools/map_stages.py 2>&1 | grep -E 'stages|x200' | tr '\n' ' ')"
  echo "   parity: $(SPLAT_B200_LIB=$PWD/$f timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1)"
done
