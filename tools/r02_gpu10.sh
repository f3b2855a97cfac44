#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"^k_forward$|^k_backward$" -s 2 -c 2 \
  --metrics smsp__thread_inst_executed_per_inst_executed.ratio,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active \
  -o gpurun_out/blendprof python tools/step_once.py 3 > gpurun_out/ncu_blend.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ncu_blend.log
