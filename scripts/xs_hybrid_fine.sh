#!/bin/bash
# fine sweep of the hybrid slice fraction around the defaults (cfg2 0.16, cfg4 0.25)
cd "${GRAFT_REPO_ROOT:-.}"
pr() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('%-28s value %.4g frac %.3f ms/step %.1f clocks %s' % ('$1', d['value'], r['frac'], d['ms_per_step'], d.get('clocks',{}).get('sm_mhz')))"; }
B="python bench.py --no-cpu-baseline --euler-steps 0 --no-e2e --no-north-star --no-tte --steps 4 --warmup 3"
for i in 1 2; do for e in 0.14 0.16 0.18; do S2B_HYBRID=$e timeout 600 $B 2>/dev/null | pr "cfg2 $e"; done; done
B="python bench.py --config cfg4 --no-cpu-baseline --euler-steps 0 --no-e2e --no-north-star --no-tte --steps 4 --warmup 3"
for i in 1 2; do for e in 0.23 0.25 0.27; do S2B_HYBRID=$e timeout 600 $B 2>/dev/null | pr "cfg4 $e"; done; done
