"""Key metrics of one ncu capture as JSON (for profiles/).  usage: ncu_summary.py REP OUT NOTE"""
import csv
import io
import json
import subprocess
import sys
from collections import Counter

rep, out, note = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
d = {a: (b, c) for a, b, c in zip(r[0], r[2], r[1])}


def f(k):
    try:
        return float(d[k][0])
    except Exception:
        return None


keys = {
    "duration": "gpu__time_duration.sum", "dram_read": "dram__bytes_read.sum", "dram_write": "dram__bytes_write.sum",
    "fp64_pipe_pct_of_active": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "registers_per_thread": "launch__registers_per_thread", "instructions": "smsp__inst_executed.sum",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "clusters_resident": "launch__cluster_max_active", "grid_ctas": "launch__grid_size",
    "smem_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smem_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
}
summary = {"kernel": d.get("Kernel Name", ("?",))[0], "capture": note}
for name, k in keys.items():
    if k in d:
        summary[name] = {"value": f(k), "unit": d[k][1]}
try:
    summary["sm_active_over_elapsed"] = f("sm__cycles_active.avg") / f("sm__cycles_elapsed.avg")
except Exception:
    pass
st = {k[34:-23]: float(v[0]) for k, v in d.items()
      if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")}
summary["top_stalls_cycles_per_issue"] = dict(sorted(st.items(), key=lambda kv: -kv[1])[:8])
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
if len(rows) > 2:
    h = rows[1]
    ia, isrc = h.index("Instructions Executed"), h.index("Source")
    mix = Counter()
    for x in rows[2:]:
        toks = x[isrc].split()
        if toks:
            mix[(toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]] += float(x[ia] or 0)
    tot = sum(mix.values())
    summary["opcode_mix_pct"] = {k: round(v / tot * 100, 2) for k, v in mix.most_common(12)}
with open(out, "w") as fh:
    json.dump(summary, fh, indent=1)
print(json.dumps({k: summary[k] for k in ("kernel", "fp64_pipe_pct_of_active") if k in summary}))
