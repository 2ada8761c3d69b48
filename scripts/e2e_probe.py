import sys, time, numpy as np
sys.path.insert(0, '.')
import paper_2207_09776_b200 as s2b
import torch
d, M = 256, 16384
g = s2b.GridSpec.square(d); ctx = s2b.default_context()
op = s2b.Operator.from_family(g, "langevin-constant", order=3, ctx=ctx)
paths = s2b.BrownianPaths.philox(1.0, 1e-4, M, seed=1, ctx=ctx)
sess = s2b.MagnusSession(s2b.MagnusConfig(order=3, dt=0.01), op, s2b.gaussian_datum(g), paths, 1.0)
for _ in range(2): sess.advance(1)
host = torch.empty((M, paths.steps + 1), dtype=torch.float64).pin_memory(); hv = host.numpy(); hv[:] = paths.values()
mom = torch.empty(2 * d * d, dtype=torch.float64).pin_memory().numpy()
w = 2
for it in range(3):
    ctx.synchronize(); t0 = time.perf_counter()
    paths.upload(w * 100, (w + 1) * 100, hv); ctx.synchronize(); t1 = time.perf_counter()
    sess.advance(1); ctx.synchronize(); t2 = time.perf_counter()
    sess.moments(mom); ctx.synchronize(); t3 = time.perf_counter()
    print(f"upload {1e3*(t1-t0):.1f} ms  advance {1e3*(t2-t1):.1f} ms  moments {1e3*(t3-t2):.1f} ms")
    w += 1
