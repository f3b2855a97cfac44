#!/bin/bash
# A/B of variants/lib_*.so plus a GPU parity run of each variant's blend kernels.
mkdir -p gpurun_out
bash tools/ab_bench.sh ${1:-20} 2>&1 | tee gpurun_out/ab.txt
for f in variants/lib_*.so; do
  n=$(basename $f .so)
  SPLAT_B200_LIB=$PWD/$f timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/par_$n.log 2>&1
  echo "$n parity rc=$? $(tail -1 gpurun_out/par_$n.log)" | tee -a gpurun_out/ab.txt
done
