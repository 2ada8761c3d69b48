#!/bin/bash
# em_rows_kernel per-launch durations under ncu (accurate kernel time; 1024^2, 4096 paths, 16 B/pt/step)
for cfg in ${CFGS:-"S2B_EMTB=1" "S2B_EMTB=0" "S2B_EMROWS=0"}; do
  env $cfg ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:em_ -s 4 -c 8 --csv \
    python scripts/em_probe.py --d 1024 --paths 4096 --steps 10 20 --family ${FAM:-langevin-constant} 2>/dev/null > gpurun_out/emncu.csv
  python - "$cfg" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open("gpurun_out/emncu.csv")) if len(r) > 10]
h = rows[0]; i_n = h.index("Metric Name"); i_v = h.index("Metric Value")
t = [float(r[i_v].replace(",", "")) for r in rows[1:] if r[i_n] == "gpu__time_duration.sum"]
b = [float(r[i_v].replace(",", "")) for r in rows[1:] if r[i_n].startswith("dram__bytes")]
alg = 4096 * 1024 * 1024 * 16
ms = sum(t) / len(t) / 1e3  # ncu reports usecond
print(sys.argv[1], "launches", len(t), "avg %.3f ms" % ms, "alg GB/s %.0f" % (alg / (ms / 1e3) / 1e9), "dram/alg %.3f" % (sum(b) / len(t) / alg if t else 0))
PY
done
