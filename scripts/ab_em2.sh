#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_engines.py -q -x -k euler 2>&1 | tail -2
for v in 1 0; do
  echo -n "S2B_EM2=$v: "
  S2B_EM2=$v timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 1 --warmup 3 --euler-steps 400 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read())['euler_maruyama']; print('E-M %.4g path*pt*steps/s frac %.3f ms %.1f blown %d' % (d['value'], d['roofline']['frac'], d['ms'], d['blown']))"
done
