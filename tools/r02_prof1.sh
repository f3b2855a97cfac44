#!/bin/bash
# ncu --set full of one kernel (regex $1) in a config-1 step; report under gpurun_out/$2
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$1" -s ${3:-2} -c 1 -o gpurun_out/$2 python tools/step_once.py 3 > gpurun_out/ncu_$2.log 2>&1; echo "ncu rc=$?"; tail -1 gpurun_out/ncu_$2.log
