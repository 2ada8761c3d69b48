#!/bin/bash
# term_varx_kernel (x-split, 2 CTAs/SM) vs term_var_kernel (S2B_VARX=0), parity first
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_1024.py tests/test_gpu_adaptive.py -q -x 2>&1 | tail -2
for vx in 1 0; do
  for order in 3 2; do
  echo -n "S2B_VARX=$vx cfg3 order $order: "
  S2B_VARX=$vx timeout 600 python bench.py --config cfg3 --order $order --no-cpu-baseline --no-e2e --euler-steps 0 --steps 2 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('value %.4g  terms/s %.4g  frac %.3f  ms/step %.1f' % (d['value'], d['path_gridpoint_terms_per_s'], r['frac'], d['ms_per_step']))"
  done
  echo -n "S2B_VARX=$vx cfg5 var: "
  S2B_VARX=$vx timeout 600 python bench.py --config cfg5 --family langevin-variable --no-cpu-baseline --no-e2e --euler-steps 0 --steps 2 --warmup 2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('value %.4g  terms/s %.4g  frac %.3f' % (d['value'], d['path_gridpoint_terms_per_s'], r['frac']))"
done
