#!/bin/bash
# term_tma_kernel strip height (S2B_STRIP output rows per work item) at cfg5 (1024^2)
for st in 128 256 512 128; do
  echo -n "S2B_STRIP=$st cfg5: "
  S2B_STRIP=$st timeout 300 python bench.py --config cfg5 --no-cpu-baseline --euler-steps 0 --no-e2e --steps 3 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('value %.4g frac %.3f ms/step %.1f clocks %s' % (d['value'], r['frac'], d['ms_per_step'], d['clocks']))"
done
