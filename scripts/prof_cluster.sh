#!/bin/bash
set -e
CMD="python bench.py --paths 288 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --euler-steps 0"
S2B_ENGINE=cluster $CMD > gpurun_out/plain_cl.log 2>&1
S2B_ENGINE=cluster ncu --set full --clock-control none --import-source on -k regex:cluster_magnus -s 1 -c 1 -o gpurun_out/prof_cluster $CMD > gpurun_out/ncu_cl.log 2>&1
