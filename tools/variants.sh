#!/bin/bash
# Build kernel variants (-D flags) into gpurun_out-free dir variants/ for A/B timing on the box.
# usage: tools/variants.sh NAME "FLAGS" [NAME "FLAGS" ...]
set -e
cd "$(dirname "$0")/.."
mkdir -p variants
while [ $# -gt 0 ]; do
  name=$1; flags=$2; shift 2
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xptxas -v -shared \
    -Xcompiler -fPIC $flags -o variants/lib_$name.so paper_2503_17491_b200/csrc/capi.cu 2> /tmp/ptx_$name.log || { grep error /tmp/ptx_$name.log; exit 1; }
  echo "$name: $(grep -E 'k_(forward|backward)ILi8' -A2 /tmp/ptx_$name.log | grep -oE 'Used [0-9]+ registers|[0-9]+ bytes spill stores' | tr '\n' ' ')"
done
