#!/bin/bash
# 512^2 engine parity, then in-place cluster vs streaming at 512^2
timeout 1200 python -m pytest tests/test_gpu_engines.py -q -x -k 512 2>&1 | tail -3
for eng in cluster stream; do
  echo -n "engine=$eng: "
  S2B_ENGINE=$eng timeout 900 python bench.py --d 512 --paths 4096 --dt 0.005 --no-cpu-baseline --euler-steps 0 --no-e2e --steps 3 --warmup 2 "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; c=d['compute_roofline']; print('value %.4g GB/s(alg) %.0f frac %.3f fp64 %.2f ms/step %.1f terms/win %.3f %s' % (d['value'], r['achieved'], r['frac'], c['frac'], d['ms_per_step'], d['path_terms_per_window'], r['engine']))"
done
