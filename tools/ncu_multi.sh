#!/bin/bash
# Full ncu capture of several kernels (regex $1) of the config-1 step loop (one launch each).
mkdir -p gpurun_out
K=${1:-k_forward}
TAG=${2:-multi}
python tools/prof_step.py 1 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$K" -s ${4:-12} -c ${3:-6} -o gpurun_out/prof_$TAG python tools/prof_step.py 1 > gpurun_out/ncu_full.log 2>&1
rc=$?
tail -3 gpurun_out/ncu_full.log
exit $rc
