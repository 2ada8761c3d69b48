#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_engines.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2
for cfg in "64 1000 2 0.1" "128 4096 3 0.05"; do set -- $cfg
  for xm in 1 0; do
    echo -n "d=$1 S2B_XM=$xm: "
    S2B_XM=$xm timeout 600 python bench.py --d $1 --paths $2 --order $3 --dt $4 --no-cpu-baseline --euler-steps 0 --no-e2e --steps 3 --warmup 2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('value %.4g frac %.3f %s' % (d['value'], r['frac'], r['engine']))"
  done
done
