#!/bin/bash
# ncu --set full of one em_rows_kernel launch at 1024^2 (4096 paths)
set -e
CMD="python scripts/em_probe.py --d 1024 --paths 4096 --steps 10 20"
$CMD > gpurun_out/plain_emrows.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:em_rows -s 5 -c 1 -o gpurun_out/prof_emrows $CMD > gpurun_out/ncu_emrows.log 2>&1
