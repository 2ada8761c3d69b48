#!/bin/bash
# term_var / term_varx after a fold change: parity first, then the variable-coefficient presets
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_1024.py tests/test_gpu_adaptive.py tests/test_gpu_stress.py -q -x 2>&1 | tail -3
B="python bench.py --no-cpu-baseline --no-e2e --euler-steps 0 --no-north-star --steps 3 --warmup 3"
show() { tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('value %.4g  GB/s %.0f  frac %.3f  ms/step %.1f  %s' % (d['value'], r['achieved'], r['frac'], d['ms_per_step'], r.get('kernel')))"; }
for args in "--config cfg3" "--config cfg3 --order 2" "--config cfg3k" "--config cfg3k --order 2" "--config cfg5 --family langevin-variable"; do
  echo -n "$args $EXTRA: "; timeout 900 $B $args 2>&1 | show
done
