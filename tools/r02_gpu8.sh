#!/bin/bash
mkdir -p gpurun_out
SS_BINNING=legacy timeout 300 python tools/ab_binning.py > gpurun_out/ab_pre5.json 2>&1; echo "minb5: $(head -c 330 gpurun_out/ab_pre5.json)"
SS_BINNING=legacy SPLAT_B200_LIB=variants/libsplat_pre4.so timeout 300 python tools/ab_binning.py > gpurun_out/ab_pre4.json 2>&1; echo "minb4: $(head -c 330 gpurun_out/ab_pre4.json)"
timeout 900 python -m pytest tests -q -x -m gpu -p no:cacheprovider -k "parity or golden or densify or keyframe or spec or capi or registration" > gpurun_out/pytest_gpu2.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu2.log
