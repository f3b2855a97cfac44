#!/bin/bash
# Run the GPU test suite on the box, logging to gpurun_out/.
mkdir -p gpurun_out
timeout ${1:-900} python -m pytest tests -x -q -m gpu -s ${2:-} > gpurun_out/pytest_gpu.log 2>&1
rc=$?
tail -60 gpurun_out/pytest_gpu.log
exit $rc
