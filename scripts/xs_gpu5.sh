#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
timeout 900 python -m pytest tests/test_gpu_xs.py tests/test_gpu_1024.py -q -k "xs or magnus" > gpurun_out/xs_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/xs_tests.log
B="python bench.py --config cfg5 --no-cpu-baseline --euler-steps 0 --no-e2e --no-north-star --no-tte --steps 3 --warmup 3"
pr() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$1 value %.4g frac %.3f ms/step %.1f clocks %s' % (d['value'], r['frac'], d['ms_per_step'], d.get('clocks')))"; }
for i in 1 2; do timeout 600 $B 2>/dev/null | pr xs; done
bash scripts/prof_r02.sh xs_cfg5
