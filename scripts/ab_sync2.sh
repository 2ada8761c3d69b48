#!/bin/bash
# term_tma_kernel: one CTA barrier per G ring steps (S2B_TMA_SYNC=1/2/4)
for g in 4 2; do
S2B_TMA_SYNC=$g timeout 1500 python -m pytest tests/test_gpu_1024.py tests/test_gpu_engines.py tests/test_gpu_stress.py -q -x 2>&1 | tail -1
done
B="python bench.py --no-cpu-baseline --no-e2e --euler-steps 0 --no-north-star --steps 3 --warmup 3"
show() { tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('value %.4g  GB/s %.0f  frac %.3f  ms/step %.1f  %s mhz %s %s' % (d['value'], r['achieved'], r['frac'], d['ms_per_step'], r.get('kernel'), d['clocks']['sm_mhz'], d['clocks']['reasons']))"; }
run() { local envs="$1"; shift; echo -n "[$envs] $*: "; env $envs timeout 900 $B "$@" 2>&1 | show; }
for g in 4 2 1 4; do run "S2B_TMA_SYNC=$g" --config cfg5; done
for g in 4 2; do run "S2B_TMA_SYNC=$g" --config cfg4; done
for g in 4 2; do run "S2B_TMA_SYNC=$g" --config cfg2; done
