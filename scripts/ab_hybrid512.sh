#!/bin/bash
for h in 0 0.1 0.15 0.2 0.25; do
  echo -n "512 S2B_HYBRID=$h: "
  S2B_HYBRID=$h timeout 600 python bench.py --d 512 --paths 4096 --dt 0.005 --no-cpu-baseline --euler-steps 0 --no-e2e --steps 3 --warmup 2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value %.4g frac %.3f ms/step %.1f' % (d['value'], d['roofline']['frac'], d['ms_per_step']))"
done
for h in 0.11 0.13; do
  echo -n "256 S2B_HYBRID=$h: "
  S2B_HYBRID=$h timeout 600 python bench.py --no-cpu-baseline --euler-steps 0 --no-e2e --steps 3 --warmup 2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value %.4g frac %.3f ms/step %.1f' % (d['value'], d['roofline']['frac'], d['ms_per_step']))"
done
