#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
for k in 1 0; do for o in 2 3; do
  echo -n "GENK=$k order $o: "
  S2B_GENK=$k timeout 600 python bench.py --family langevin-variable --order $o --paths 2048 --no-cpu-baseline --euler-steps 0 --no-e2e --steps 2 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('value %.4g frac %.3f terms/win %.1f ms/step %.1f' % (d['value'], r['frac'], d['path_terms_per_window'], d['ms_per_step']))"
done; done
