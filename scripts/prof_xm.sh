#!/bin/bash
set -e
CMD="python bench.py --paths 288 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --euler-steps 0"
$CMD > gpurun_out/plain_xm.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:cluster_xm -s 1 -c 1 -o gpurun_out/prof_xm $CMD > gpurun_out/ncu_xm.log 2>&1
