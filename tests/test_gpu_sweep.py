"""Step-size sweep on shared paths in batched launches (SURVEY 8(f) rank 3,
run_stepsize_sweep, experiment.cpp:486-551): every configuration of the sweep equals its own
solve (which tests/test_gpu_parity.py and test_gpu_engines.py pin to the reference), bit for
bit, on the batched x-march engines (256^2, 512^2) and on the one-by-one fallback."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("d,order,dts", [(256, 3, [0.01, 0.02, 0.005]), (256, 2, [0.02, 0.01]),
                                         (512, 3, [0.01, 0.02]), (24, 3, [0.1, 0.05])])
def test_sweep_equals_individual_solves(s2b, ctx, d, order, dts):
    T, dt_leb, M = 0.04 if d >= 256 else 0.2, 1e-3, 3
    g = s2b.GridSpec.square(d)
    op = s2b.Operator.from_family(g, "langevin-constant", order=order, ctx=ctx)
    paths = s2b.BrownianPaths.philox(T, dt_leb, M, seed=17, ctx=ctx)
    phi = s2b.gaussian_datum(g)
    cfgs = [s2b.MagnusConfig(order=order, dt=dt, record_times=[dts[0] * 2] if d >= 256 else []) for dt in dts]
    stats = []
    sweep = s2b.solve_iterated_magnus_sweep(cfgs, op, phi, paths, T, g, stats=stats)
    assert len(sweep) == len(cfgs) and len(stats) == len(cfgs)
    for cfg, ens, st in zip(cfgs, sweep, stats):
        one_stats = {}
        one = s2b.solve_iterated_magnus(cfg, op, phi, paths, T, g, stats=one_stats)
        assert len(ens) == len(one)
        for e, o in zip(ens, one):
            assert np.array_equal(e.status, o.status)
            assert np.array_equal(e.states(), o.states(), equal_nan=True)
        assert st["path_terms"] == one_stats["path_terms"] and st["engine"] == one_stats["engine"]
