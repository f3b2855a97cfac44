#!/bin/bash
# Per-stage split of the 8 concurrent loops of register_batch (block 0 of each loop; -DSS_RS_PROF)
set -e
mkdir -p variants gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -shared -DSS_RS_PROF \
  -o variants/prof_rs.so paper_2503_17491_b200/csrc/capi.cu
SPLAT_B200_LIB=$PWD/variants/prof_rs.so SS_BATCH_TIMING=1 python tools/reg_batch_phases.py 2>&1 | tail -12
