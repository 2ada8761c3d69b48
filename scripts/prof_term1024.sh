#!/bin/bash
# ncu --set full of one term_tma_kernel launch at 1024^2 (cfg5 shape, 256 paths)
set -e
CMD="python bench.py --config cfg5 --paths 256 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --euler-steps 0"
$CMD > gpurun_out/plain_t1024.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:term_tma -s 40 -c 1 -o gpurun_out/prof_t1024 $CMD > gpurun_out/ncu_t1024.log 2>&1
