#!/bin/bash
# Per-stage time split of the device registration loop (block 0's view):
# builds a -DSS_RS_PROF variant library and runs reg_probe.py against it.
set -e
mkdir -p variants gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -shared -DSS_RS_PROF \
  -o variants/prof_rs.so paper_2503_17491_b200/csrc/capi.cu
SPLAT_B200_LIB=$PWD/variants/prof_rs.so python tools/reg_probe.py
