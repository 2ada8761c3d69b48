#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_engines.py -q -x -k hybrid 2>&1 | tail -2
for h in 0 0.06 0.1 0.14 0.18; do
  echo -n "S2B_HYBRID=$h: "
  S2B_HYBRID=$h timeout 600 python bench.py --no-cpu-baseline --euler-steps 0 --no-e2e --steps 3 --warmup 2 "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value %.4g ms/step %.1f terms/win %.3f' % (d['value'], d['ms_per_step'], d['path_terms_per_window']))"
done
