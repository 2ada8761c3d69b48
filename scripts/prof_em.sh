#!/bin/bash
# ncu captures of the cluster E-M kernels (256^2 double-buffered, 512^2 in place)
set -e
C256="python bench.py --paths 240 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --euler-steps 100"
C512="python bench.py --d 512 --dt 0.005 --paths 112 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --euler-steps 100"
ncu --set full --clock-control none -k regex:em_cluster_kernel -s 1 -c 1 -o gpurun_out/prof_em256 $C256 > gpurun_out/ncu_em256.log 2>&1
ncu --set full --clock-control none -k regex:em_cluster_ip -s 1 -c 1 -o gpurun_out/prof_em512 $C512 > gpurun_out/ncu_em512.log 2>&1
ncu --set full --clock-control none -k regex:term_generic_k -s 20 -c 1 -o gpurun_out/prof_genk3 python bench.py --family langevin-variable --order 3 --paths 512 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --euler-steps 0 > gpurun_out/ncu_genk3.log 2>&1
