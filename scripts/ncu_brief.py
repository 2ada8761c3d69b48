"""Brief of an ncu report: key metrics, stall reasons, opcode mix.  usage: ncu_brief.py REP"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
d = {a: (b, c) for a, b, c in zip(r[0], r[2], r[1])}
for k in ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
          "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
          "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
          "smsp__inst_executed.sum", "sm__cycles_elapsed.avg", "smsp__cycles_active.avg",
          "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]:
    print(k, d.get(k))
st = {k[34:-23]: float(x[0]) for k, x in d.items()
      if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")}
print("stalls:", {k: round(v, 2) for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:10]})
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
ia, isamp, isrc = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
ti = sum(float(x[ia] or 0) for x in rows[2:])
ts = sum(float(x[isamp] or 0) for x in rows[2:])
c, cs = Counter(), Counter()
for x in rows[2:]:
    toks = x[isrc].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    op = op.split(".")[0]
    c[op] += float(x[ia] or 0)
    cs[op] += float(x[isamp] or 0)
print("opcode mix (inst %, stall-sample %):")
for op, v in c.most_common(18):
    print(f"  {op:10s} {v / ti * 100:6.2f} {cs[op] / ts * 100:6.2f}")
if len(sys.argv) > 2:
    with open(sys.argv[2], "w") as f:
        for i, x in enumerate(rows[2:]):
            f.write(f"{i:5d} {float(x[ia] or 0) / 1e6:9.3f} {float(x[isamp] or 0):7.0f}  {x[isrc]}\n")
