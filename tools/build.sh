#!/bin/bash
# Build libsplatb200.so (sm_100a) and the oracle; non-zero exit on any failure.
set -e
cd "$(dirname "$0")/.."
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xptxas -v -shared \
  -Xcompiler -fPIC -o paper_2503_17491_b200/libsplatb200.so paper_2503_17491_b200/csrc/capi.cu 2> /tmp/ptxas.log || { grep -E "error" /tmp/ptxas.log; exit 1; }
grep -E "k_(forward|backward)ILi8" -A2 /tmp/ptxas.log | grep -E "registers" | sed 's/ptxas info    : //'
make -s -C oracle
