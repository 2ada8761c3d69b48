#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
timeout 900 python -m pytest tests/test_gpu_xs.py -x -q > gpurun_out/xs_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/xs_tests.log
bash scripts/prof_r02.sh xs_cfg5
