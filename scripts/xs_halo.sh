#!/bin/bash
# x-march two-term kernel: parity of every x-march variant, then 28-row vs 32-row items (S2B_XS2H) at cfg5
cd "${GRAFT_REPO_ROOT:-.}"
timeout 1500 python -m pytest tests/test_gpu_xs.py tests/test_gpu_stress.py -q -x -k "xs" > gpurun_out/xs_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/xs_tests.log
bash scripts/xs_ab.sh "S2B_XS2H=0" "S2B_XS2H=1"
