#!/bin/bash
# hybrid slice on the x-march engine: parity, then slice-fraction A/B at cfg2 and cfg4
cd "${GRAFT_REPO_ROOT:-.}"
timeout 900 python -m pytest tests/test_gpu_engines.py -q -k "hybrid" > gpurun_out/xs_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/xs_tests.log
pr() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('%-44s value %.4g frac %.3f ms/step %.1f clocks %s' % ('$1', d['value'], r['frac'], d['ms_per_step'], d.get('clocks',{}).get('sm_mhz')))"; }
B="python bench.py --no-cpu-baseline --euler-steps 0 --no-e2e --no-north-star --no-tte --steps 4 --warmup 3"
for e in "S2B_XS_SLICE=0" "S2B_HYBRID=0.12" "S2B_HYBRID=0.16" "S2B_HYBRID=0.20" "S2B_HYBRID=0.24"; do env $e timeout 600 $B 2>>gpurun_out/hyb.err | pr "cfg2 $e"; done
B="python bench.py --config cfg4 --no-cpu-baseline --euler-steps 0 --no-e2e --no-north-star --no-tte --steps 4 --warmup 3"
for e in "S2B_XS_SLICE=0" "S2B_HYBRID=0.20" "S2B_HYBRID=0.25" "S2B_HYBRID=0.30" "S2B_HYBRID=0.35"; do env $e timeout 600 $B 2>>gpurun_out/hyb.err | pr "cfg4 $e"; done
