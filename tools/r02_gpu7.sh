#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none --cache-control none -k regex:"k_preprocess" -s 1 -c 1 -o gpurun_out/preprof python tools/fwd_once.py 2 > gpurun_out/ncu_pre.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ncu_pre.log
