"""Install the round-end evidence of scripts/final_r02.sh into profiles/: every bench line as
profiles/r02_bench_<cfg>.json and the launch list as profiles/r02_launches_bench.{csv,json}."""
import csv
import io
import json
import os
import shutil
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
for f in sorted(os.listdir(G)):
    if f.startswith("bench_") and f.endswith(".log") and f[6:-4] in (
            "default", "cfg1", "cfg3", "cfg3k", "cfg4", "cfg5", "cfg5var", "cfg3o2", "cfg3ko2", "reference"):
        lines = [l for l in open(os.path.join(G, f)) if l.startswith("{")]
        if lines:
            d = json.loads(lines[-1])
            name = f[len("bench_"):-len(".log")]
            json.dump(d, open(os.path.join(P, f"r02_bench_{name}.json"), "w"), indent=1)
            print(name, d.get("value"), (d.get("roofline") or {}).get("frac"))
src = os.path.join(G, "launches.csv")
if os.path.exists(src):
    shutil.copy(src, os.path.join(P, "r02_launches_bench.csv"))
    rows = [l for l in open(src) if l.startswith('"')]
    tot, cnt = defaultdict(float), defaultdict(int)
    for x in csv.DictReader(io.StringIO("".join(rows))):
        if x.get("Metric Name") != "gpu__time_duration.sum":
            continue
        scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}.get(
            x.get("Metric Unit", ""), 1.0)
        name = x["Kernel Name"].replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
        name = name.split("(")[0].split("<")[0].replace("void ", "").split("::")[-1].strip()
        tot[name] += float(x["Metric Value"]) * scale
        cnt[name] += 1
    all_us = sum(tot.values())
    out = {"command": "ncu --metrics gpu__time_duration.sum --clock-control none -c 400 python bench.py --steps 2 "
                      "--warmup 3 --no-cpu-baseline --no-e2e --no-north-star (cfg2 default workload)",
           "launches": sum(cnt.values()), "total_us": all_us,
           "note": "serialised, cold-cache per-launch times: compare shares, not absolutes; the hybrid slice "
                   "(term_tma_kernel) runs concurrently with the cluster kernel outside ncu",
           "kernels": [{"kernel": k, "launches": cnt[k], "total_us": tot[k], "share": round(tot[k] / all_us, 4)}
                       for k in sorted(tot, key=lambda k: -tot[k])]}
    json.dump(out, open(os.path.join(P, "r02_launches_bench.json"), "w"), indent=1)
    print(out["kernels"][:4])
