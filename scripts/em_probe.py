"""E-M streaming-engine probe: path*gridpoint*steps/s of solve_euler on one grid, from the
difference of two call lengths (removes allocation / state-init overhead).

  python scripts/em_probe.py --d 1024 --paths 4096 --family langevin-constant
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2207_09776_b200 as s2b  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--d", type=int, default=1024)
ap.add_argument("--paths", type=int, default=4096)
ap.add_argument("--family", default="langevin-constant")
ap.add_argument("--dt-leb", type=float, default=1e-5)
ap.add_argument("--steps", type=int, nargs=2, default=[20, 120])
a = ap.parse_args()

ctx = s2b.Context(0)
g = s2b.GridSpec.square(a.d)
f = s2b.Fields.from_family(g, a.family, ctx=ctx)
paths = s2b.BrownianPaths.philox(a.steps[1] * a.dt_leb, a.dt_leb, a.paths, seed=3, ctx=ctx)
phi = s2b.gaussian_datum(g)
cfg = s2b.EulerConfig(dt=a.dt_leb)
s2b.solve_euler(cfg, f, g, phi, paths, 5 * a.dt_leb)
ts = []
for k in a.steps:
    ctx.synchronize()
    t0 = time.perf_counter()
    ens = s2b.solve_euler(cfg, f, g, phi, paths, k * a.dt_leb)
    ctx.synchronize()
    ts.append(time.perf_counter() - t0)
    blown = ens[-1].blowup_count()
    del ens
rate = a.paths * a.d * a.d * (a.steps[1] - a.steps[0]) / (ts[1] - ts[0])
print(f"E-M {a.family} {a.d}^2 M={a.paths} S2B_EMROWS={os.environ.get('S2B_EMROWS', '1')}: "
      f"{rate:.4g} path*pt*steps/s = {16 * rate / 1e9:.0f} GB/s ({16 * rate / 6548.2e9:.3f} of HBM); "
      f"calls {ts[0]:.3f}/{ts[1]:.3f} s, blown {blown}")
