#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
timeout 1500 python -m pytest tests/test_gpu_xs.py -q -x > gpurun_out/xs_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/xs_tests.log
bash scripts/xs_ab.sh "S2B_XS2=0" "S2B_XS2=1"
bash scripts/prof_r02.sh xs2_cfg5
