"""Step-size sweep on shared paths in batched launches (SURVEY 8(f) rank 3,
run_stepsize_sweep, experiment.cpp:486-551): every configuration of the sweep is pinned bit
for bit to the reference's own solve_iterated_magnus (magnus.cpp:239-304) on the same
increments, on the batched x-march engines (256^2, 512^2) and on the one-by-one fallback;
its counters equal the individual GPU solve's."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("d,order,dts", [(256, 3, [0.01, 0.02, 0.005]), (256, 2, [0.02, 0.01]),
                                         (512, 3, [0.01, 0.02]), (24, 3, [0.1, 0.05])])
def test_sweep_bitwise_vs_reference(ref, s2b, ctx, d, order, dts):
    T, dt_leb, M, seed = 0.04 if d >= 256 else 0.2, 1e-3, 3, 17
    g = s2b.GridSpec.square(d)
    ops = ref.Ops("langevin-constant", d, order=order)
    values, _ = ref.simulate_brownian(T, dt_leb, M, seed)
    op = s2b.Operator.from_family(g, "langevin-constant", order=order, ctx=ctx)
    paths = s2b.BrownianPaths.from_values(values, dt_leb, seed=seed, ctx=ctx)
    phi = s2b.gaussian_datum(g)
    recs = [[dts[0] * 2] if d >= 256 else [] for _ in dts]
    cfgs = [s2b.MagnusConfig(order=order, dt=dt, record_times=r) for dt, r in zip(dts, recs)]
    stats = []
    sweep = s2b.solve_iterated_magnus_sweep(cfgs, op, phi, paths, T, g, stats=stats)
    assert len(sweep) == len(cfgs) and len(stats) == len(cfgs)
    for cfg, rec, ens, st in zip(cfgs, recs, sweep, stats):
        want, wst, _ = ops.solve_magnus(values, dt_leb, T, cfg.dt, record_times=rec, seed=seed)
        assert len(ens) == len(want)
        for r, e in enumerate(ens):
            assert np.array_equal(e.status, wst[r])
            assert np.array_equal(e.states(), want[r], equal_nan=True)
        one_stats = {}
        s2b.solve_iterated_magnus(cfg, op, phi, paths, T, g, stats=one_stats)
        assert st["path_terms"] == one_stats["path_terms"] and st["engine"] == one_stats["engine"]
