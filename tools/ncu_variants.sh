#!/bin/bash
# Full ncu capture of one kernel (regex $1) for each variants/lib_*.so in the config-1 step loop.
mkdir -p gpurun_out
K=${1:-k_backward}
for f in variants/lib_*.so; do
  n=$(basename $f .so)
  SPLAT_B200_LIB=$PWD/$f timeout 300 ncu --set full --clock-control none --import-source on -k regex:$K -s ${3:-1} -c ${2:-1} \
    -o gpurun_out/var_${n}_$K python tools/prof_step.py 1 > gpurun_out/ncu_$n.log 2>&1
  echo "$n rc=$? $(tail -1 gpurun_out/ncu_$n.log)"
done
