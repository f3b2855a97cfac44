#!/bin/bash
# Config-2 (mapping) A/B of variants/lib_*.so: eager stage times + graph refine ms/iter, plus
# the render parity tests of each variant.
mkdir -p gpurun_out
for f in variants/lib_*.so; do
  n=$(basename $f .so)
  echo "== $n" 
  SPLAT_B200_LIB=$PWD/$f timeout 300 python tools/map_stages.py 2>&1 | grep -v "^records"
  SPLAT_B200_LIB=$PWD/$f timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mapping.py -x -q 2>&1 | tail -1
done
