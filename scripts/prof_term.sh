#!/bin/bash
# ncu capture of the dominant kernel (term_tma_kernel) on a reduced path count.
set -e
CMD="python bench.py --paths 2048 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --euler-steps 0"
$CMD > gpurun_out/plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:term_tma -s 40 -c 1 -o gpurun_out/prof_term $CMD > gpurun_out/ncu_full.log 2>&1
