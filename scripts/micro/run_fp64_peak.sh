#!/bin/bash
# builds and runs the fp64 pipe microbenchmark, sampling SM clocks while it runs
set -e
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/fp64_peak scripts/micro/fp64_peak.cu
nvidia-smi --query-gpu=clocks.sm,clocks_throttle_reasons.active --format=csv,noheader -lms 100 > gpurun_out/fp64_clk.txt &
P=$!
/tmp/fp64_peak > gpurun_out/fp64_peak.json
/tmp/fp64_peak >> gpurun_out/fp64_peak.json
kill $P
cat gpurun_out/fp64_peak.json
sort gpurun_out/fp64_clk.txt | uniq -c | sort -rn | head -5
