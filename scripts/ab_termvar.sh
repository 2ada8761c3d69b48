#!/bin/bash
# x-dependent coefficients (cfg3): term_var_kernel vs term_generic_k_kernel (parity first)
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_1024.py tests/test_gpu_adaptive.py -q -x 2>&1 | tail -3
for tv in 1 0; do
  for order in 3 2; do
  echo -n "S2B_TERMVAR=$tv order $order: "
  S2B_TERMVAR=$tv timeout 600 python bench.py --config cfg3 --order $order --no-cpu-baseline --no-e2e --euler-steps 0 --steps 2 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('value %.4g  terms/s %.4g  GB/s %.0f  frac %.3f  ms/step %.1f terms/window %.1f' % (d['value'], d['path_gridpoint_terms_per_s'], r['achieved'], r['frac'], d['ms_per_step'], d['path_terms_per_window']))"
  done
done
