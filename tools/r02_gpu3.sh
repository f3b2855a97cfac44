#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/ab_binning.py > gpurun_out/ab_new.json 2> gpurun_out/ab_new.err; echo "new rc=$?"; cat gpurun_out/ab_new.json; tail -3 gpurun_out/ab_new.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/bin_launches.csv python tools/fwd_once.py 3 > gpurun_out/ncu_bin.log 2>&1; echo "ncu rc=$?"
python tools/launch_table.py gpurun_out/bin_launches.csv 20
timeout 900 python -m pytest tests -q -x -m gpu -p no:cacheprovider -k "parity or golden or densify or keyframe or spec or capi" --deselect tests/test_gpu_parity.py::test_long_lists_and_tie_runs_bit_exact > gpurun_out/pytest_gpu2.log 2>&1
echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu2.log
timeout 300 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "long_lists" > gpurun_out/sanitizer.log 2>&1; echo "sanitizer rc=$?"; grep -m5 -A12 "Invalid\|ERROR" gpurun_out/sanitizer.log | head -40
