"""Summarize an ncu capture of the term kernel + the launch list into profiles/.

usage: python scripts/summarize_ncu.py ROUND  (reads gpurun_out/prof_term.ncu-rep and
gpurun_out/launches.csv, writes profiles/<ROUND>_term_kernel_ncu.{json,md} and
profiles/term_kernel_ncu.json, the file bench.py reads for roofline.traffic)
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles")


def ncu_raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(txt)))
    hdr, units, vals = r[0], r[1], r[2]
    return {h: (v, u) for h, v, u in zip(hdr, vals, units)}


def f(d, k):
    try:
        return float(d[k][0])
    except Exception:
        return None


def launches(path):
    if not os.path.exists(path):
        return None
    rows = []
    with open(path) as fh:
        lines = [l for l in fh if l.startswith('"')]
    r = csv.DictReader(io.StringIO("".join(lines)))
    for x in r:
        if x.get("Metric Name") == "gpu__time_duration.sum":
            rows.append((x["Kernel Name"], float(x["Metric Value"]), x.get("Metric Unit", "")))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for k, v, u in rows:
        scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(u, 1.0)
        name = k.split("(")[0].split("<")[0].replace("void ", "").strip()
        tot[name] += v * scale
        cnt[name] += 1
    all_us = sum(tot.values())
    return {name: {"launches": cnt[name], "total_us": tot[name], "share": tot[name] / all_us}
            for name in sorted(tot, key=lambda n: -tot[n])}


def main():
    rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
    rep = os.path.join(ROOT, "gpurun_out", "prof_term.ncu-rep")
    d = ncu_raw(rep)
    dur_ms = f(d, "gpu__time_duration.sum")
    rd = f(d, "dram__bytes_read.sum")
    wr = f(d, "dram__bytes_write.sum")
    unit = d["dram__bytes_read.sum"][1]
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}.get(unit, 1.0)
    traffic = (rd + wr) * scale
    # profiled launch: bench --paths 2048 on 256^2 (all paths live, k > 1: 32 B per point)
    paths, n = 2048, 256 * 256
    alg = 32.0 * paths * n
    stalls = {k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""):
              float(v[0]) for k, v in d.items()
              if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")}
    top = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:8])
    summary = {
        "kernel": d.get("Kernel Name", ("term_tma_kernel", ""))[0] if "Kernel Name" in d else "term_tma_kernel",
        "capture": "ncu --set full --clock-control none -k regex:term_tma -s 40 -c 1, "
                   "python bench.py --paths 2048 --steps 1 --warmup 1 (256x256, order 3)",
        "duration_ms": dur_ms,
        "dram_bytes_read": rd * scale,
        "dram_bytes_write": wr * scale,
        "dram_bytes_total": traffic,
        "algorithmic_bytes": alg,
        "traffic_over_algorithmic": traffic / alg,
        "dram_bytes_per_path_term": traffic / paths,
        "achieved_dram_GBps": traffic / (dur_ms * 1e-3) / 1e9,
        "registers_per_thread": f(d, "launch__registers_per_thread"),
        "warps_active_pct": f(d, "sm__warps_active.avg.pct_of_peak_sustained_active"),
        "issue_active_pct": f(d, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "instructions": f(d, "smsp__inst_executed.sum"),
        "top_stalls_cycles_per_issue": top,
        "launch_list_share_us": launches(os.path.join(ROOT, "gpurun_out", "launches.csv")),
    }
    os.makedirs(OUT, exist_ok=True)
    for path in (os.path.join(OUT, f"{rnd}_term_kernel_ncu.json"), os.path.join(OUT, "term_kernel_ncu.json")):
        with open(path, "w") as fh:
            json.dump(summary, fh, indent=1)
    print(json.dumps({k: v for k, v in summary.items() if k != "launch_list_share_us"}, indent=1))
    ll = summary["launch_list_share_us"] or {}
    for k, v in list(ll.items())[:8]:
        print(f"{v['share']*100:6.2f}%  {v['launches']:5d}  {k}")


if __name__ == "__main__":
    main()
