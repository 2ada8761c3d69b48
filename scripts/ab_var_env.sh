#!/bin/bash
# term_var / term_varx launch-shape A/B through the env knobs (bench only; parity is shape-independent
# and covered by tests/test_gpu_stress.py)
B="python bench.py --no-cpu-baseline --no-e2e --euler-steps 0 --no-north-star --steps 3 --warmup 3"
show() { tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('value %.4g  GB/s %.0f  frac %.3f  ms/step %.1f  %s' % (d['value'], r['achieved'], r['frac'], d['ms_per_step'], r.get('kernel')))"; }
run() { local envs="$1"; shift; echo -n "[$envs] $*: "; env $envs timeout 900 $B "$@" 2>&1 | show; }
run "S2B_VAR_G=1" --config cfg3
run "S2B_VAR_G=2" --config cfg3
run "S2B_VAR_ROWS=64" --config cfg3
run "S2B_VAR_ROWS=256" --config cfg3
run "S2B_VARX=1" --config cfg3
run "S2B_VARX=1 S2B_VARX_G=2" --config cfg3
run "S2B_VARX_G=1" --config cfg3k
run "S2B_VARX_G=2" --config cfg3k
run "S2B_VARX_G=2" --config cfg5 --family langevin-variable
