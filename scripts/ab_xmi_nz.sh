#!/bin/bash
# cluster_xmi: accumulator starting at the first product (NZ) vs 0.0 + it; parity then cfg4
timeout 1500 python -m pytest tests/test_gpu_engines.py -q -x -k "512 or bit_patterns" 2>&1 | tail -1
S2B_XMI_NZ=0 timeout 1500 python -m pytest tests/test_gpu_engines.py -q -x -k "512 or bit_patterns" 2>&1 | tail -1
B="python bench.py --no-cpu-baseline --no-e2e --euler-steps 0 --no-north-star --steps 3 --warmup 3"
show() { tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('value %.4g  GB/s %.0f  frac %.3f  ms/step %.1f  %s mhz %s %s' % (d['value'], r['achieved'], r['frac'], d['ms_per_step'], r.get('kernel'), d['clocks']['sm_mhz'], d['clocks']['reasons']))"; }
run() { local envs="$1"; shift; echo -n "[$envs] $*: "; env $envs timeout 900 $B "$@" 2>&1 | show; }
for v in 1 0 1 0; do run "S2B_XMI_NZ=$v" --config cfg4; done
