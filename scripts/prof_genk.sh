#!/bin/bash
set -e
CMD="python bench.py --family langevin-variable --order 2 --paths 512 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --euler-steps 0"
$CMD > gpurun_out/plain_genk.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:term_var -s 20 -c 1 -o gpurun_out/prof_genk $CMD > gpurun_out/ncu_genk.log 2>&1
