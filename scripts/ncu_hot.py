"""Hot SASS lines of a source-page export (gpurun_out/src_<name>.csv.gz): the instructions
with the most stall samples, with their dominant stall reasons.  usage: ncu_hot.py name [N]"""
import csv
import gzip
import io
import sys

name = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
rows = list(csv.reader(io.StringIO(gzip.open(f"gpurun_out/src_{name}.csv.gz", "rt").read())))
h = rows[1]
isrc, isamp = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
data = []
tot = 0.0
for r in rows[2:]:
    try:
        s = float(r[isamp] or 0)
    except ValueError:
        continue
    tot += s
    st = sorted(((float(r[i] or 0), h[i][6:]) for i in stall_cols), reverse=True)[:3]
    data.append((s, r[0], r[isrc], st))
data.sort(reverse=True)
agg = {}
for s, a, src, st in data:
    op = src.split()[1] if src.split() and src.split()[0].startswith("@") else (src.split()[0] if src.split() else "")
    agg[op.split(".")[0]] = agg.get(op.split(".")[0], 0) + s
print("samples", tot)
print("by opcode:", sorted(((round(v / tot * 100, 1), k) for k, v in agg.items()), reverse=True)[:12])
for s, a, src, st in data[:N]:
    print(f"{s / tot * 100:5.1f}% {a} {src[:60]:60s} " + " ".join(f"{n}:{v:.0f}" for v, n in st if v))
