#!/bin/bash
# engine parity at 256^2, then x-march vs row-band cluster kernels on cfg2
timeout 900 python -m pytest tests/test_gpu_engines.py -q -x 2>&1 | tail -5
for xm in 1 0; do
  echo -n "S2B_XM=$xm: "
  S2B_XM=$xm timeout 600 python bench.py --no-cpu-baseline --euler-steps 0 --no-e2e --steps 3 --warmup 2 "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('value %.4g GB/s(alg) %.0f frac %.3f ms/step %.1f terms/win %.3f' % (d['value'], r['achieved'], r['frac'], d['ms_per_step'], d['path_terms_per_window']))"
done
