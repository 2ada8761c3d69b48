#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
timeout 1500 python -m pytest tests/test_gpu_xs.py tests/test_gpu_engines.py tests/test_gpu_1024.py tests/test_gpu_stress.py tests/test_gpu_adaptive.py -q > gpurun_out/xs_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/xs_tests.log
bash scripts/prof_r02.sh xs_cfg5
timeout 900 python bench.py --config cfg5 > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; echo "bench rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/bench_cfg5.json').read().strip().splitlines()[-1]); print(d['value'], d['roofline'], d.get('clocks'), d.get('e2e'))"
