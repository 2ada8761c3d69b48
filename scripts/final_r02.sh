#!/bin/bash
# Round-end evidence on one B200 (round 2): GPU tests, smoke, every bench preset, the launch
# list of the default bench, and ncu --set full captures of every dominant kernel
# (summarised on the box by scripts/ncu_r02.py; install here with scripts/install_profiles.py
# and scripts/summarize_r02.py).
mkdir -p gpurun_out
python -m pytest tests -q -m gpu 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python bench.py > gpurun_out/bench_default.log 2>&1
for c in cfg1 cfg3 cfg3k cfg4 cfg5; do python bench.py --config $c > gpurun_out/bench_$c.log 2>&1; done
python bench.py --config cfg5 --family langevin-variable --no-cpu-baseline > gpurun_out/bench_cfg5var.log 2>&1
python bench.py --config cfg3 --order 2 --no-cpu-baseline > gpurun_out/bench_cfg3o2.log 2>&1
python bench.py --config cfg3k --order 2 --no-cpu-baseline > gpurun_out/bench_cfg3ko2.log 2>&1
python bench.py --impl reference > gpurun_out/bench_reference.log 2>&1
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-north-star"
$B > gpurun_out/plain_launches.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $B \
    > gpurun_out/ncu_launches.log 2>&1
bash scripts/prof_r02.sh > gpurun_out/prof_r02.log 2>&1
cat gpurun_out/pytest_gpu.log; tail -1 gpurun_out/smoke.log; cat gpurun_out/prof_r02.log
for f in default cfg1 cfg3 cfg3k cfg4 cfg5 cfg5var cfg3o2 cfg3ko2 reference; do echo "$f: $(tail -1 gpurun_out/bench_$f.log | cut -c1-150)"; done
