"""Quick GPU-vs-reference parity probe (development aid)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2207_09776_b200 as s2b
from oracle import ref

def run(family, d, order, dt, T=0.2, dt_leb=1e-3, M=4, seed=7, rec=()):
    ops = ref.Ops(family, d, order=order)
    vals, _ = ref.simulate_brownian(T, dt_leb, M, seed)
    rs, rst, _ = ops.solve_magnus(vals, dt_leb, T, dt, record_times=list(rec), seed=seed)
    g = s2b.GridSpec.square(d)
    op = s2b.Operator.from_family(g, family, order=order)
    op2 = s2b.Operator.from_csr(g, order, [ops.csr(s) for s in ref.SLOTS])
    paths = s2b.BrownianPaths.from_values(vals, dt_leb, seed=seed)
    stats = {}
    t0 = time.time()
    ens = s2b.solve_iterated_magnus(s2b.MagnusConfig(order=order, dt=dt, record_times=list(rec)), op, ops.datum(), paths, T, g, stats=stats)
    ens2 = s2b.solve_iterated_magnus(s2b.MagnusConfig(order=order, dt=dt, record_times=list(rec)), op2, ops.datum(), paths, T, g)
    t1 = time.time()
    for r, e in enumerate(ens):
        st = e.states(); st2 = ens2[r].states()
        same = np.array_equal(st, rs[r], equal_nan=True) and np.array_equal(e.status, rst[r])
        same2 = np.array_equal(st2, rs[r], equal_nan=True)
        rel = np.linalg.norm(np.nan_to_num(st - rs[r])) / np.linalg.norm(np.nan_to_num(rs[r]))
        print(f"{family} d={d} order={order} dt={dt} rec{r}: bitwise={same} csr_bitwise={same2} rel={rel:.3e} status={e.status} info={op.info()} {t1-t0:.2f}s", flush=True)
    print("stats", stats)
    # euler
    f = s2b.Fields.from_family(g, family)
    ee = s2b.solve_euler(s2b.EulerConfig(dt=dt_leb*10), f, g, ops.datum(), paths, T)
    es, est, _ = ops.solve_euler(vals, dt_leb, T, dt_leb*10)
    print("euler bitwise", np.array_equal(ee[-1].states(), es[-1], equal_nan=True), est[-1], ee[-1].status)
    ex = s2b.exact_reference(g, T, 1.1, 1/np.sqrt(10), paths).states()
    exr = ops.exact_reference(vals, dt_leb, T)
    print("exact maxrel", np.max(np.abs(ex-exr)/np.abs(exr)))

for fam in ["langevin-constant", "langevin-variable"]:
    for d, order in [(16, 3), (20, 2), (14, 1), (9, 3), (64, 3)]:
        try:
            run(fam, d, order, 0.1, rec=(0.1,))
        except Exception as ex:
            import traceback; traceback.print_exc()
