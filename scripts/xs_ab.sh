#!/bin/bash
# same-run A/B of term_xs knobs at cfg5: xs_ab.sh "ENV=.. ENV2=.." "ENV=.." ...
cd "${GRAFT_REPO_ROOT:-.}"
B="python bench.py --config cfg5 --no-cpu-baseline --euler-steps 0 --no-e2e --no-north-star --no-tte --steps 3 --warmup 3"
pr() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('%-28s value %.4g frac %.3f ms/step %.1f clocks %s' % ('$1', d['value'], r['frac'], d['ms_per_step'], d.get('clocks',{}).get('sm_mhz')))"; }
for i in 1 2; do for cfg in "$@"; do env $cfg timeout 600 $B 2>/dev/null | pr "$cfg"; done; done
