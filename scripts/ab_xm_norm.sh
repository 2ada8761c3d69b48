#!/bin/bash
# cluster_xm high-word maxima: parity (default bounds + forced exact pass), then cfg2 / cfg1 bench
timeout 1500 python -m pytest tests/test_gpu_engines.py tests/test_gpu_sweep.py tests/test_gpu_adaptive.py -q -x 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_stress.py -q -x -k "cluster_xm" 2>&1 | tail -2
B="python bench.py --no-cpu-baseline --no-e2e --euler-steps 0 --no-north-star --steps 3 --warmup 3"
show() { tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('value %.4g  GB/s %.0f  frac %.3f  ms/step %.1f  %s' % (d['value'], r['achieved'], r['frac'], d['ms_per_step'], r.get('kernel')))"; }
run() { local envs="$1"; shift; echo -n "[$envs] $*: "; env $envs timeout 900 $B "$@" 2>&1 | show; }
run "S2B_XM_EXACT=0" --config cfg2
run "S2B_XM_EXACT=1" --config cfg2
run "S2B_XM_EXACT=0" --config cfg1
run "S2B_VAR_ROWS=256" --config cfg3k
run "S2B_VAR_ROWS=128" --config cfg3k
