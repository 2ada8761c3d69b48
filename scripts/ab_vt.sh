#!/bin/bash
# term_tma_kernel at 1024^2: two virtual threads per thread (256 threads) vs 512 threads
S2B_TMA_VT=2 timeout 1500 python -m pytest tests/test_gpu_1024.py -q -x 2>&1 | tail -1
S2B_TMA_VT=2 timeout 900 python -m pytest tests/test_gpu_stress.py -q -x -k "term" 2>&1 | tail -1
B="python bench.py --no-cpu-baseline --no-e2e --euler-steps 0 --no-north-star --steps 3 --warmup 3"
show() { tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('value %.4g  GB/s %.0f  frac %.3f  ms/step %.1f  %s mhz %s %s' % (d['value'], r['achieved'], r['frac'], d['ms_per_step'], r.get('kernel_mangled')[-40:], d['clocks']['sm_mhz'], d['clocks']['reasons']))"; }
run() { local envs="$1"; shift; echo -n "[$envs] $*: "; env $envs timeout 900 $B "$@" 2>&1 | show; }
for v in 2 1 2 1; do run "S2B_TMA_VT=$v" --config cfg5; done
