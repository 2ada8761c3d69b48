#!/bin/bash
python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -2
for cl in 16 8; do
  echo -n "cluster=$cl: "
  S2B_CLUSTER=$cl python bench.py --no-cpu-baseline --euler-steps 0 --no-e2e --steps 3 --warmup 2 "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('value %.4g GB/s(alg) %.0f frac %.3f ms/step %.1f terms/win %.3f' % (d['value'], r['achieved'], r['frac'], d['ms_per_step'], d['path_terms_per_window']))"
done
