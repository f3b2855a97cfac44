#!/bin/bash
# Evidence for profiles/: plain bench, ncu launch list of the bench command, full capture of the blend kernels.
mkdir -p gpurun_out
timeout 600 python bench.py --steps 20 > gpurun_out/bench.log 2>&1 || exit 1
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_list.log 2>&1
python tools/prof_step.py 1 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_forward|k_backward|k_tile_sort|k_preprocess" -s 8 -c 4 \
    -o gpurun_out/prof_round python tools/prof_step.py 1 > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
# config 2 (mapping: block-per-tile forward, segment backward) and config-3 registration kernels
python tools/map_step.py 4 > gpurun_out/plain_map.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_forward|k_backward|k_tile_sort" -s 8 -c 4 \
    -o gpurun_out/prof_map python tools/map_step.py 4 > gpurun_out/ncu_map.log 2>&1
python tools/geo_probe.py > gpurun_out/plain_reg.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_reg_solve|k_leaf_top" -c 2 \
    -o gpurun_out/prof_reg python tools/geo_probe.py > gpurun_out/ncu_reg.log 2>&1
tail -n 1 gpurun_out/ncu_map.log; tail -n 1 gpurun_out/ncu_reg.log
