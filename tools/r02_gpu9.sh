#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_registration.py -q -x -p no:cacheprovider -k batch > gpurun_out/pytest_reg.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_reg.log
timeout 300 python tools/reg_batch_probe.py > gpurun_out/reg_batch.json 2> gpurun_out/reg_batch.err; echo "probe rc=$?"; cat gpurun_out/reg_batch.json; tail -3 gpurun_out/reg_batch.err
