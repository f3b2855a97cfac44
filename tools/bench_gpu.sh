#!/bin/bash
mkdir -p gpurun_out
timeout 600 python bench.py ${@} > gpurun_out/bench.log 2>&1
rc=$?
tail -20 gpurun_out/bench.log
exit $rc
