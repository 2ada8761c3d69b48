#!/bin/bash
# ncu --set full captures of the dominant kernels bench.py launches today (one per config),
# each after the same command exited 0 without ncu.  Reports: gpurun_out/prof_<name>.ncu-rep;
# summarise here with scripts/ncu_r02.py.  Usage: bash scripts/prof_r02.sh [name ...]
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --euler-steps 0 --no-north-star"
declare -A CMD KERN SKIP
CMD[xm_cfg2]="$B --paths 288";                                  KERN[xm_cfg2]="cluster_xm_kernel"; SKIP[xm_cfg2]=1
CMD[xm_cfg1]="$B --config cfg1 --paths 296";                   KERN[xm_cfg1]="cluster_xm_kernel"; SKIP[xm_cfg1]=1
# the hybrid slice is only split off from 64 paths up: 600 paths -> 72 streaming paths at 256^2
CMD[xs_hybrid256]="$B --paths 600";                             KERN[xs_hybrid256]="term_xs_kernel"; SKIP[xs_hybrid256]=40
CMD[xs_hybrid512]="$B --config cfg4 --paths 448 --T 0.01";      KERN[xs_hybrid512]="term_xs_kernel"; SKIP[xs_hybrid512]=40
CMD[tma_hybrid256]="env S2B_XS_SLICE=0 $B --paths 600";                            KERN[tma_hybrid256]="term_tma_kernel"; SKIP[tma_hybrid256]=40
CMD[xmi_cfg4]="$B --config cfg4 --paths 112 --T 0.01";          KERN[xmi_cfg4]="cluster_xmi_kernel"; SKIP[xmi_cfg4]=1
CMD[tma_hybrid512]="env S2B_XS_SLICE=0 $B --config cfg4 --paths 560 --T 0.01";     KERN[tma_hybrid512]="term_tma_kernel"; SKIP[tma_hybrid512]=40
CMD[var_cfg3]="$B --config cfg3 --paths 1184 --T 0.02";         KERN[var_cfg3]="term_var_kernel"; SKIP[var_cfg3]=40
CMD[varx_cfg3k]="$B --config cfg3k --paths 1184 --T 0.02";      KERN[varx_cfg3k]="term_varx_kernel"; SKIP[varx_cfg3k]=40
CMD[tma_cfg5]="env S2B_XS=0 $B --config cfg5 --paths 296 --T 0.001";         KERN[tma_cfg5]="term_tma_kernel"; SKIP[tma_cfg5]=40
CMD[xs_cfg5]="env S2B_XS2=0 $B --config cfg5 --paths 296 --T 0.001";          KERN[xs_cfg5]="term_xs_kernel"; SKIP[xs_cfg5]=40
CMD[xs2_cfg5]="$B --config cfg5 --paths 296 --T 0.001"; KERN[xs2_cfg5]="term_xs2_kernel"; SKIP[xs2_cfg5]=20
CMD[varx_cfg5var]="$B --config cfg5 --family langevin-variable --paths 296 --T 0.001"; KERN[varx_cfg5var]="term_varx_kernel"; SKIP[varx_cfg5var]=40
# E-M: the timed solve_euler of the bench's E-M leg (the warm-up solve is launch 0)
CMD[em_cfg2]="$B --paths 288 --euler-steps 40";                 KERN[em_cfg2]="em_cluster_ip_kernel"; SKIP[em_cfg2]=1
CMD[em_cfg5]="$B --config cfg5 --paths 296 --T 0.001 --euler-steps 20"; KERN[em_cfg5]="em_tb_kernel"; SKIP[em_cfg5]=6
NAMES=${@:-xm_cfg2 xm_cfg1 xs_hybrid256 xmi_cfg4 xs_hybrid512 var_cfg3 varx_cfg3k xs2_cfg5 varx_cfg5var em_cfg2 em_cfg5}
for nm in $NAMES; do
  ${CMD[$nm]} > gpurun_out/plain_$nm.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:${KERN[$nm]} -s ${SKIP[$nm]} -c 1 \
      -o gpurun_out/prof_$nm -f ${CMD[$nm]} > gpurun_out/ncu_$nm.log 2>&1
  echo "$nm rc=$?"
  python scripts/ncu_r02.py $nm && rm -f gpurun_out/prof_$nm.ncu-rep
done
