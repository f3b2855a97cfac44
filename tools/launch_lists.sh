#!/bin/bash
# ncu launch lists (gpu__time_duration) of the config-1 and config-2 step loops (tools/prof_step.py).
mkdir -p gpurun_out
for c in 1 2; do
  python tools/prof_step.py 2 $c > gpurun_out/plain_c$c.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c$c.csv \
    python tools/prof_step.py 2 $c > gpurun_out/ncu_list_c$c.log 2>&1
  echo "config $c rc=$?"
done
