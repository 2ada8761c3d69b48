#!/bin/bash
# streaming x-march engine: parity tests, then cfg5 / cfg4-stream A/B against term_tma (S2B_XS=0)
cd "${GRAFT_REPO_ROOT:-.}"
timeout 1500 python -m pytest tests/test_gpu_xs.py tests/test_gpu_engines.py tests/test_gpu_1024.py tests/test_gpu_stress.py -x -q "$@" > gpurun_out/xs_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/xs_tests.log
B="python bench.py --config cfg5 --no-cpu-baseline --euler-steps 0 --no-e2e --no-north-star --no-tte --steps 3 --warmup 3"
pr() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$1 value %.4g frac %.3f ms/step %.1f clocks %s' % (d['value'], r['frac'], d['ms_per_step'], d.get('clocks')))"; }
for i in 1 2; do
S2B_XS=0 timeout 600 $B 2> gpurun_out/xs_b_tma.err | tee gpurun_out/xs_b_tma_$i.json | pr tma
timeout 600 $B 2> gpurun_out/xs_b_xs.err | tee gpurun_out/xs_b_xs_$i.json | pr xs
done
