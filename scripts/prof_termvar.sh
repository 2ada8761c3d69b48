#!/bin/bash
# ncu --set full of one term_var_kernel launch (cfg3 order 3 at 256^2, 512 paths)
set -e
CMD="python bench.py --config cfg3 --order ${ORDER:-3} --paths 512 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --euler-steps 0"
$CMD > gpurun_out/plain_termvar.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:term_var -s 20 -c 1 -o gpurun_out/prof_termvar $CMD > gpurun_out/ncu_termvar.log 2>&1
