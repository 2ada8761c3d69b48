#!/bin/bash
# Round-end validation on one B200: GPU tests, smoke, every bench preset, launch list of the default bench
mkdir -p gpurun_out
python -m pytest tests -q -m gpu 2>&1 | tail -4 > gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python bench.py > gpurun_out/bench_default.log 2>&1
for c in cfg1 cfg3 cfg3k cfg4 cfg5; do python bench.py --config $c > gpurun_out/bench_$c.log 2>&1; done
python bench.py --config cfg5 --family langevin-variable --no-cpu-baseline > gpurun_out/bench_cfg5var.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launches.log 2>&1
cat gpurun_out/pytest_gpu.log; tail -1 gpurun_out/smoke.log
for f in default cfg1 cfg3 cfg3k cfg4 cfg5 cfg5var; do echo "$f: $(tail -1 gpurun_out/bench_$f.log | cut -c1-120)"; done
