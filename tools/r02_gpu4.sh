#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none --cache-control none -k regex:"k_bucket_count|k_emit_chunk|k_bucket_scan|k_tile_place" -s 4 -c 4 -o gpurun_out/sortprof5 python tools/fwd_once.py 3 > gpurun_out/ncu_sort.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ncu_sort.log
