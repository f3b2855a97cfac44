#!/bin/bash
mkdir -p gpurun_out
SS_BINNING=legacy timeout 300 python tools/ab_binning.py > gpurun_out/ab_legacy.json 2>&1; echo "legacy rc=$?"; cat gpurun_out/ab_legacy.json
SS_BINNING=legacy timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/bin_launches_legacy.csv python tools/fwd_once.py 3 > gpurun_out/ncu_bin.log 2>&1; echo "ncu rc=$?"
python tools/launch_table.py gpurun_out/bin_launches_legacy.csv 16
