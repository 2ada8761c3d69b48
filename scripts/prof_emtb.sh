#!/bin/bash
# ncu --set full of one em_tb_kernel launch (two E-M steps) at 1024^2, 4096 paths
set -e
CMD="python scripts/em_probe.py --d 1024 --paths 4096 --steps 10 20"
$CMD > gpurun_out/plain_emtb.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:em_tb -s 3 -c 1 -o gpurun_out/prof_emtb $CMD > gpurun_out/ncu_emtb.log 2>&1
