"""Summarize an ncu capture of a cluster-resident Magnus kernel into profiles/.

usage: python scripts/summarize_cluster_ncu.py ROUND NAME REP BENCH_LOG
  REP        the .ncu-rep of ONE launch of `bench.py --paths P --steps 1` (one window per path)
  BENCH_LOG  the same command's plain (un-profiled) JSON line, for P, the grid and S*K
writes profiles/<ROUND>_<NAME>_kernel_ncu.json and profiles/<NAME>_kernel_ncu.json (the file
bench.py reads for roofline.traffic of that engine).
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import Counter

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    rnd, name, rep, log = sys.argv[1:5]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    d = {a: (b, c) for a, b, c in zip(r[0], r[2], r[1])}

    def f(k):
        try:
            return float(d[k][0])
        except Exception:
            return None

    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
    rd = f("dram__bytes_read.sum") * scale.get(d["dram__bytes_read.sum"][1], 1.0)
    wr = f("dram__bytes_write.sum") * scale.get(d["dram__bytes_write.sum"][1], 1.0)
    dur = f("gpu__time_duration.sum") * {"msecond": 1e-3, "ms": 1e-3, "usecond": 1e-6, "us": 1e-6, "nsecond": 1e-9, "ns": 1e-9}[d["gpu__time_duration.sum"][1]]
    with open(log) as fh:
        line = json.loads([x for x in fh if x.startswith("{")][-1])
    paths = line["config"]["paths_per_gpu"]
    n = line["config"]["grid"] ** 2
    spk = line["path_terms_per_window"]
    alg = 32.0 * n * spk * paths  # streaming-equivalent bytes (k=1 counted at 32 B: upper bound)
    stalls = {k[34:-23]: float(v[0]) for k, v in d.items()
              if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")}
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    h = rows[1]
    ia, isrc = h.index("Instructions Executed"), h.index("Source")
    mix = Counter()
    for x in rows[2:]:
        toks = x[isrc].split()
        if toks:
            op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
            mix[op] += float(x[ia] or 0)
    tot = sum(mix.values())
    summary = {
        "kernel": d["Kernel Name"][0],
        "capture": f"ncu --set full --clock-control none, one launch of bench.py --paths {paths} --steps 1 "
                   f"({line['config']['grid']}^2, order {line['config']['order']}, 1 window per path)",
        "duration_ms": dur * 1e3,
        "dram_bytes_read": rd,
        "dram_bytes_write": wr,
        "dram_bytes_total": rd + wr,
        "dram_bytes_per_path_window": (rd + wr) / paths,
        "path_terms_per_window": spk,
        "algorithmic_bytes_streaming_model": alg,
        "traffic_over_algorithmic": (rd + wr) / alg,
        "achieved_algorithmic_GBps": alg / dur / 1e9,
        "fp64_pipe_pct_of_active": f("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        "fp64_pipe_pct_of_elapsed": f("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed"),
        "issue_active_pct": f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "sm_active_over_elapsed": f("sm__cycles_active.avg") / f("sm__cycles_elapsed.avg"),
        "clusters_resident": f("launch__cluster_max_active"),
        "grid_ctas": f("launch__grid_size"),
        "registers_per_thread": f("launch__registers_per_thread"),
        "instructions": f("smsp__inst_executed.sum"),
        "top_stalls_cycles_per_issue": dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:8]),
        "opcode_mix_pct": {k: round(v / tot * 100, 2) for k, v in mix.most_common(12)},
    }
    out = os.path.join(ROOT, "profiles")
    os.makedirs(out, exist_ok=True)
    for p in (os.path.join(out, f"{rnd}_{name}_kernel_ncu.json"), os.path.join(out, f"{name}_kernel_ncu.json")):
        with open(p, "w") as fh:
            json.dump(summary, fh, indent=1)
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
