#!/bin/bash
# Round-2 checkpoint: GPU tests, smoke, then the profile evidence (tools/round_profile.sh).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
bash tools/round_profile.sh
tail -1 gpurun_out/bench.log | cut -c1-400
