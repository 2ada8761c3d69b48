#!/bin/bash
# compute-sanitizer racecheck / synccheck / memcheck over the synchronisation-heavy kernels
# (scripts/sanitize_cases.py); one log per (tool, case) and a summary in gpurun_out/sanitize/.
# Usage (on the GPU box): bash scripts/sanitize.sh [case ...]
mkdir -p gpurun_out/sanitize
CASES=${@:-xm64 xm128 xm256 xmi512 band256 tma256 var256 varx256 emip64 emip256 emip512 emtb96 expmv}
for c in $CASES; do
  for tool in racecheck synccheck memcheck; do
    extra=""
    [ $tool = racecheck ] && extra="--racecheck-report hazard"
    timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool $extra --print-limit 20 \
        python scripts/sanitize_cases.py $c > gpurun_out/sanitize/${tool}_${c}.log 2>&1
    rc=$?
    summ=$(grep -E "ERROR SUMMARY|RACECHECK SUMMARY" gpurun_out/sanitize/${tool}_${c}.log | tail -1)
    echo "$c $tool rc=$rc $summ" | tee -a gpurun_out/sanitize/summary.txt
  done
done
