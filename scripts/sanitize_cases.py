"""Small instances of every synchronisation-heavy kernel for compute-sanitizer
(racecheck / synccheck / memcheck): scripts/sanitize.sh runs each case under each tool.
Each case is one tiny solve through the public API on cuda:0 (1-3 paths, one short window),
and prints the engine it ran so the log shows which kernel was checked."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2207_09776_b200 as s2b  # noqa: E402


def magnus(d, family="langevin-constant", order=3, M=2, dt=0.002, fields=None, env=None):
    for k, v in (env or {}).items():
        os.environ[k] = v
    ctx = s2b.Context(0)
    g = s2b.GridSpec.square(d)
    op = s2b.Operator.from_family(g, family, order=order, fields=fields, ctx=ctx)
    paths = s2b.BrownianPaths.philox(dt, 1e-4, M, seed=3, ctx=ctx)
    st = {}
    ens = s2b.solve_iterated_magnus(s2b.MagnusConfig(order=order, dt=dt), op, s2b.gaussian_datum(g), paths, dt, g,
                                    stats=st)
    assert ens[-1].blowup_count() == 0
    print(f"magnus d={d} {family} order={order}: engine {st['engine']}, kernels {ctx.kernel_names()}")


def euler(d, family="langevin-constant", M=3, steps=4, fields=None, env=None):
    for k, v in (env or {}).items():
        os.environ[k] = v
    ctx = s2b.Context(0)
    g = s2b.GridSpec.square(d)
    f = s2b.Fields.from_arrays(g, fields, ctx=ctx) if fields else s2b.Fields.from_family(g, family, ctx=ctx)
    paths = s2b.BrownianPaths.philox(steps * 1e-5, 1e-5, M, seed=3, ctx=ctx)
    ens = s2b.solve_euler(s2b.EulerConfig(dt=1e-5), f, g, s2b.gaussian_datum(g), paths, steps * 1e-5)
    assert ens[-1].blowup_count() == 0
    print(f"euler d={d} {family}: ok")


def expmv():
    ctx = s2b.Context(0)
    rng = np.random.default_rng(1)
    n = 600
    m = (rng.random((n, n)) < 0.01) * rng.normal(0.0, 2.0, (n, n))
    rp, ci, v = [0], [], []
    for r in range(n):
        nz = np.nonzero(m[r])[0]
        ci += list(nz)
        v += list(m[r, nz])
        rp.append(len(ci))
    y, rep = s2b.expmv_into((np.array(rp, np.uint64), np.array(ci, np.int32), np.array(v)), rng.normal(size=n), 1e-10,
                            ws=s2b.ExpmvWorkspace(ctx))
    print("expmv_into:", rep)


CASES = {
    "xm64": lambda: magnus(64),                        # cluster_xm, one CTA per path
    "xm128": lambda: magnus(128),                      # cluster_xm, 4-CTA clusters (DSMEM halos)
    "xm256": lambda: magnus(256, M=1),                 # cluster_xm, 8-CTA clusters
    "xmi512": lambda: magnus(512, M=1, dt=0.0005),     # cluster_xmi, 16-CTA clusters, in place
    "band256": lambda: magnus(256, M=1, order=2, env={"S2B_XM": "0"}),  # cluster_magnus row-band
    "tma256": lambda: magnus(256, M=2, env={"S2B_ENGINE": "stream"}),   # term_tma_kernel (TMA ring)
    "var256": lambda: magnus(256, "langevin-variable", M=4, dt=0.001),  # term_var_kernel (TMA rows)
    "varx256": lambda: magnus(256, "fields", M=4, dt=0.0005, fields=__import__("fieldsets").kinetic_fields(256)),
    "emip64": lambda: euler(64, M=6),                  # em_cluster_ip, 2-CTA clusters
    "emip256": lambda: euler(256),                     # em_cluster_ip, 8-CTA clusters
    "emip512": lambda: euler(512, M=1),                # em_cluster_ip, 16-CTA clusters
    "emtb96": lambda: euler(96, "langevin-variable", M=2, env={"S2B_EMXM": "0"}),  # em_tb_kernel (TMA ring)
    "expmv": expmv,                                    # expmv_coop_kernel (grid barrier)
}

if __name__ == "__main__":
    CASES[sys.argv[1]]()
