#!/bin/bash
set -e
CMD="python bench.py --d 512 --dt 0.005 --paths 112 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --euler-steps 0"
$CMD > gpurun_out/plain_xmi.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:cluster_xmi -s 1 -c 1 -o gpurun_out/prof_xmi $CMD > gpurun_out/ncu_xmi.log 2>&1
