#!/bin/bash
# streaming engines alone at 256^2 / 512^2: term_xs2 vs term_xs vs term_tma (same run)
cd "${GRAFT_REPO_ROOT:-.}"
pr() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('%-40s value %.4g frac %.3f ms/step %.1f clocks %s' % ('$1', d['value'], r['frac'], d['ms_per_step'], d.get('clocks',{}).get('sm_mhz')))"; }
for cfg in "--paths 4096 --T 0.08" "--config cfg4 --paths 2048 --T 0.04"; do
B="python bench.py --no-cpu-baseline --euler-steps 0 --no-e2e --no-north-star --no-tte --steps 3 --warmup 3 $cfg"
for e in "S2B_ENGINE=stream" "S2B_ENGINE=stream S2B_XS2=0" "S2B_ENGINE=stream S2B_XS=0"; do env $e timeout 600 $B 2>>gpurun_out/ab256.err | pr "$cfg $e"; done
done
