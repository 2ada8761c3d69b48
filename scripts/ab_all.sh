#!/bin/bash
# full GPU parity suite, then one bench line per preset (Magnus only, short)
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
B="python bench.py --no-cpu-baseline --no-e2e --euler-steps 0 --no-north-star --steps 3 --warmup 3"
show() { tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('value %.4g  GB/s %.0f  frac %.3f  ms/step %.1f  %s mhz %s %s' % (d['value'], r['achieved'], r['frac'], d['ms_per_step'], r.get('kernel'), d['clocks']['sm_mhz'], d['clocks']['reasons']))"; }
run() { local envs="$1"; shift; echo -n "[$envs] $*: "; env $envs timeout 900 $B "$@" 2>&1 | show; }
for c in "$@"; do run "" --config $c; done
