#!/bin/bash
# Probe the GPU box: host CPU, GPU, clocks, and FP32 FFMA peak.
mkdir -p gpurun_out
{
echo "nproc=$(nproc)"; lscpu | grep -E "Model name|Socket|Core|Thread|NUMA node\(s\)"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/probe_clocks.csv &
CP=$!
./tools/ffma_peak
./tools/ffma_peak
kill $CP
python -c "import numpy, scipy; print('numpy', numpy.__version__, 'scipy', scipy.__version__)"
} > gpurun_out/probe_box.txt 2>&1
cat gpurun_out/probe_box.txt
