#!/bin/bash
# streaming E-M: row-marching kernel (rows in flight S2B_EM_D) vs the one-thread-per-point kernel
timeout 900 python -m pytest tests/test_gpu_1024.py tests/test_gpu_parity.py -q -x -k "euler" 2>&1 | tail -3
for cfg in ${CFGS:-"S2B_EMROWS=0" "S2B_EM_D=2" "S2B_EM_D=4" "S2B_EM_D=6"}; do
  echo "== $cfg"
  for rep in 1 2; do
  env $cfg timeout 300 python scripts/em_probe.py --d 1024 --paths 4096 --steps 20 420
  env $cfg timeout 300 python scripts/em_probe.py --d 256 --paths 16384 --family langevin-variable --dt-leb 1e-4 --steps 50 650
  env $cfg S2B_EMXM=0 timeout 300 python scripts/em_probe.py --d 512 --paths 4096 --dt-leb 1e-4 --steps 50 650
  done
done
