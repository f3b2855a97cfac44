#!/bin/bash
# Launch list + full capture of one kernel (regex $1) for the config-1 step loop.
mkdir -p gpurun_out
K=${1:-k_backward}
python tools/prof_step.py 2 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/prof_step.py 2 > gpurun_out/ncu_list.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o gpurun_out/prof_$K python tools/prof_step.py 1 > gpurun_out/ncu_full.log 2>&1
rc=$?
tail -3 gpurun_out/ncu_full.log
exit $rc
