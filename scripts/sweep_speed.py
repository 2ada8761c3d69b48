"""Batched step-size sweep vs one solve per dt on shared paths (small M, where one solve
leaves clusters idle).  usage: python scripts/sweep_speed.py [--d 256] [--paths 64]"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2207_09776_b200 as s2b  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--d", type=int, default=256)
ap.add_argument("--paths", type=int, default=64)
ap.add_argument("--T", type=float, default=0.2)
ap.add_argument("--dts", default="0.05,0.04,0.02,0.01,0.005")
args = ap.parse_args()
g = s2b.GridSpec.square(args.d)
ctx = s2b.default_context()
op = s2b.Operator.from_family(g, "langevin-constant", order=3, ctx=ctx)
paths = s2b.BrownianPaths.philox(args.T, 1e-4, args.paths, seed=3, ctx=ctx)
phi = s2b.gaussian_datum(g)
cfgs = [s2b.MagnusConfig(order=3, dt=float(x)) for x in args.dts.split(",")]
s2b.solve_iterated_magnus(cfgs[0], op, phi, paths, args.T, g)  # warm-up
ctx.synchronize()
t0 = time.perf_counter()
for c in cfgs:
    s2b.solve_iterated_magnus(c, op, phi, paths, args.T, g)
ctx.synchronize()
seq = time.perf_counter() - t0
t0 = time.perf_counter()
s2b.solve_iterated_magnus_sweep(cfgs, op, phi, paths, args.T, g)
ctx.synchronize()
bat = time.perf_counter() - t0
print(json.dumps({"d": args.d, "paths": args.paths, "dts": args.dts, "sequential_s": seq, "batched_s": bat,
                  "speedup": seq / bat}))
