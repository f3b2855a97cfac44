#!/bin/bash
# A/B of variants/lib_*.so: config-1 bench stages and the config-3 registration render.
bash tools/ab_bench.sh ${1:-20} 2>&1
for f in variants/lib_*.so; do
  n=$(basename $f .so)
  echo "== $n config 3 render: $(SPLAT_B200_LIB=$PWD/$f timeout 300 python tools/anchor_probe.py 2>&1 | tr '\n' ' ')"
done
SPLAT_B200_LIB=$PWD/variants/lib_b_1024.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
