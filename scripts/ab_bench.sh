#!/bin/bash
# A/B: one-row (S2B_TERM_ROWS=1) vs two-row term kernel on 256^2 and 512^2
for rows in 1 2; do
  for cfg in "--d 256 --paths 16384 --dt 0.01" "--d 512 --paths 4096 --dt 0.005"; do
    echo -n "rows=$rows $cfg: "
    S2B_TERM_ROWS=$rows python bench.py --no-cpu-baseline --euler-steps 0 --no-e2e --steps 3 --warmup 2 $cfg 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('value %.4g GB/s %.0f frac %.3f ms/step %.1f terms/win %.2f' % (d['value'], r['achieved'], r['frac'], d['ms_per_step'], d['path_terms_per_window']))"
  done
done
