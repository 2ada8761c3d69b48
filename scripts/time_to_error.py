"""Time-to-accuracy: iterated Magnus (orders 2, 3) vs Euler-Maruyama on the GPU (cfg4).

The paper's claim (Section 5, BASELINE.json configs[3]): for the stochastic Langevin
equation the iterated Magnus scheme reaches a given accuracy 20-200x faster than
Euler-Maruyama.  This sweeps both schemes on ONE shared Brownian batch (Philox, dt_leb) at
d x d, measures Err = mean_m ||u_exact - u_app||_F / ||u_exact||_F at T against the closed
form (exact_reference, the reference's own error measure, analysis.cpp:99-127) and the wall
time of each solve call (synchronous; per path = total / M like the reference's
time_per_sim_s), then reads the speed-up off the log-log interpolated curves.

For the variable-coefficient family (cfg3, no closed form) the reference is the reference's
own choice (build_reference, experiment.cpp:379-397): a finest-dt E-M run on the same paths
(--ref-dt, default dt_leb), and Err is measured against it.

usage: python scripts/time_to_error.py [--d 512] [--paths 128] [--family langevin-variable]
                                       [--ref-dt 1e-5] [--out FILE]
"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2207_09776_b200 as s2b  # noqa: E402


def interp_time(curve, err):
    """log-log interpolation of time at a given error on a (err, time) curve; None outside."""
    pts = sorted((e, t) for e, t in curve if math.isfinite(e) and e > 0)
    for (e0, t0), (e1, t1) in zip(pts, pts[1:]):
        if e0 <= err <= e1:
            if e1 == e0:
                return t0
            w = (math.log(err) - math.log(e0)) / (math.log(e1) - math.log(e0))
            return math.exp(math.log(t0) + w * (math.log(t1) - math.log(t0)))
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--d", type=int, default=512)
    ap.add_argument("--paths", type=int, default=128)
    ap.add_argument("--T", type=float, default=1.0)
    ap.add_argument("--dt-leb", type=float, default=1e-5)
    ap.add_argument("--seed", type=int, default=424242)
    ap.add_argument("--magnus-dt", default="0.05,0.02,0.01,0.005,0.0025")
    ap.add_argument("--euler-dt", default="1e-4,5e-5,2e-5,1e-5")
    ap.add_argument("--family", default="langevin-constant",
                    choices=["langevin-constant", "langevin-variable", "kinetic-variable"])
    ap.add_argument("--ref-dt", type=float, default=None, help="E-M reference dt (variable family)")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "time_to_error.json"))
    args = ap.parse_args()
    fam = args.family

    a, sigma = 1.1, 1.0 / math.sqrt(10.0)
    g = s2b.GridSpec.square(args.d)
    ctx = s2b.default_context()
    t0 = time.perf_counter()
    paths = s2b.BrownianPaths.philox(args.T, args.dt_leb, args.paths, seed=args.seed, ctx=ctx)
    phi = s2b.gaussian_datum(g)
    if fam == "kinetic-variable":  # the general kinetic SPDE, x/v-dependent a, b, c, sigma, beta
        from bench import kinetic_fields
        kf = kinetic_fields(args.d)
        fields = s2b.Fields.from_arrays(g, kf, ctx=ctx)
        make_op = lambda order: s2b.Operator.from_family(g, "fields", order=order, fields=kf, ctx=ctx)  # noqa: E731
    else:
        fields = s2b.Fields.from_family(g, fam, a=a, sigma=sigma, ctx=ctx)
        make_op = lambda order: s2b.Operator.from_family(g, fam, a=a, sigma=sigma, order=order, ctx=ctx)  # noqa: E731
    if fam == "langevin-constant":
        ref = s2b.exact_reference(g, args.T, a, sigma, paths, ctx=ctx)
        ref_desc = "exact_reference (closed form)"
    else:
        rdt = args.ref_dt or args.dt_leb
        ref = s2b.solve_euler(s2b.EulerConfig(dt=rdt), fields, g, phi, paths, args.T)[-1]
        if ref.blowup_count():
            raise SystemExit("reference E-M run blew up (experiment.cpp:391-397)")
        ref_desc = f"finest-dt E-M run, dt={rdt} (build_reference, experiment.cpp:379-397)"
    setup_s = time.perf_counter() - t0
    rows = []

    def record(method, order, dt, fn):
        ctx.synchronize()
        t1 = time.perf_counter()
        ens = fn()
        ctx.synchronize()
        el = time.perf_counter() - t1
        e = s2b.mean_rel_error(ref, ens[-1], 4)
        row = {"method": method, "order": order, "dt": dt, "seconds": el,
               "seconds_per_path": el / args.paths, "err": e["err"], "blowups": int(e["blowups"])}
        rows.append(row)
        print(json.dumps(row), flush=True)

    for order in (2, 3):
        op = make_op(order)
        for dt in [float(x) for x in args.magnus_dt.split(",")]:
            record("magnus", order, dt, lambda: s2b.solve_iterated_magnus(
                s2b.MagnusConfig(order=order, dt=dt), op, phi, paths, args.T, g))
        del op
    for dt in [float(x) for x in args.euler_dt.split(",")]:
        record("euler", 0, dt, lambda: s2b.solve_euler(s2b.EulerConfig(dt=dt), fields, g, phi, paths, args.T))

    # speed-up at matched accuracy: every finite E-M error against each Magnus curve
    speedups = []
    em = [(r["err"], r["seconds"]) for r in rows if r["method"] == "euler"]
    for order in (2, 3):
        curve = [(r["err"], r["seconds"]) for r in rows if r["method"] == "magnus" and r["order"] == order]
        for e, t in em:
            if not math.isfinite(e):
                continue
            tm = interp_time(curve, e)
            if tm is not None:
                speedups.append({"order": order, "err": e, "euler_s": t, "magnus_s": tm, "speedup": t / tm})
        # Magnus points more accurate than every E-M run: lower bound against the best E-M
        fin = [x for x in em if math.isfinite(x[0])]
        if fin:
            best_e, best_t = min(fin)
            for e, t in curve:
                if math.isfinite(e) and e <= best_e:
                    speedups.append({"order": order, "err": e, "euler_s_at_worse_err": best_t,
                                     "euler_err": best_e, "magnus_s": t, "speedup_lower_bound": best_t / t})
    out = {"config": {"d": args.d, "paths": args.paths, "T": args.T, "dt_leb": args.dt_leb,
                      "seed": args.seed, "family": fam, "a": a, "sigma": sigma,
                      "error": f"mean_rel_error vs {ref_desc} at T (Frobenius, all paths)",
                      "timing": "wall time of each synchronous solve call on one B200"},
           "setup_s": setup_s, "runs": rows, "speedups": speedups,
           "gpu": os.popen("nvidia-smi --query-gpu=name,clocks.sm --format=csv,noheader").read().strip()}
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)
    for s in speedups:
        print(json.dumps(s))


if __name__ == "__main__":
    main()
