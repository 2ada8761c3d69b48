#!/bin/bash
# parity tests + a short default-config bench line (development loop)
python -m pytest tests -q -m gpu -x 2>&1 | tail -2
python bench.py --no-cpu-baseline --euler-steps 0 --no-e2e "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('value %.4g  GB/s %.0f  frac %.3f  ms/step %.1f terms/window %.1f' % (d['value'], r['achieved'], r['frac'], d['ms_per_step'], d['path_terms_per_window']))"
