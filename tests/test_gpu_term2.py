"""The two-term streaming engine (term2_kernel.cuh, S2B_TERM2=1; opt-in because it measures
slower than one-term passes on B200): bitwise against the reference on the compressed
Langevin stencils, with records, the norm cap, the 55-term cap and the hybrid slice."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _term2(monkeypatch):
    monkeypatch.setenv("S2B_TERM2", "1")


@pytest.mark.parametrize("d,order,dt,engine", [(24, 3, 0.1, "stream"), (16, 2, 0.05, "stream"), (14, 1, 0.1, "stream"),
                                               (64, 3, 0.1, "stream"), (130, 3, 0.05, "stream"),
                                               (256, 3, 0.01, "cluster")])
def test_term2_bitwise_vs_reference(ref, s2b, ctx, monkeypatch, d, order, dt, engine):
    if engine == "stream":
        monkeypatch.setenv("S2B_ENGINE", "stream")
    else:
        monkeypatch.setenv("S2B_HYBRID", "0.5")  # half the paths on the streaming engine
    T, dt_leb, M, seed = (0.2, 1e-3, 4, 3 + d) if d < 256 else (0.02, 1e-3, 64, 5)
    ops = ref.Ops("langevin-constant", d, order=order)
    values, _ = ref.simulate_brownian(T, dt_leb, M, seed)
    rec = [dt]
    want, wst, _ = ops.solve_magnus(values, dt_leb, T, dt, record_times=rec, seed=seed)
    g = s2b.GridSpec.square(d)
    op = s2b.Operator.from_family(g, "langevin-constant", order=order, ctx=ctx)
    paths = s2b.BrownianPaths.from_values(values, dt_leb, seed=seed, ctx=ctx)
    stats = {}
    ens = s2b.solve_iterated_magnus(s2b.MagnusConfig(order=order, dt=dt, record_times=rec), op, ops.datum(), paths,
                                    T, g, stats=stats)
    for r, e in enumerate(ens):
        assert np.array_equal(e.status, wst[r])
        assert np.array_equal(e.states(), want[r], equal_nan=True)
    terms, _ = ens[-1].counters()
    assert stats["path_terms"] == terms.sum()


@pytest.mark.parametrize("d,dt,kw,rkw", [(16, 0.1, {"blowup_norm_cap": 0.5}, {"cap": 0.5}),
                                         (64, 0.2, {"expmv_theta": 1e3}, {"theta": 1e3})])
def test_term2_blowups(ref, s2b, ctx, monkeypatch, d, dt, kw, rkw):
    """Norm cap and ToleranceNotReached (one segment, 55 terms not enough) on the two-term passes."""
    monkeypatch.setenv("S2B_ENGINE", "stream")
    T, dt_leb = 0.2, 1e-3
    ops = ref.Ops("langevin-constant", d, order=3)
    values, _ = ref.simulate_brownian(T, dt_leb, 3, 8)
    want, wst, _ = ops.solve_magnus(values, dt_leb, T, dt, seed=8, **rkw)
    g = s2b.GridSpec.square(d)
    op = s2b.Operator.from_family(g, "langevin-constant", order=3, ctx=ctx)
    paths = s2b.BrownianPaths.from_values(values, dt_leb, seed=8, ctx=ctx)
    ens = s2b.solve_iterated_magnus(s2b.MagnusConfig(order=3, dt=dt, **kw), op, ops.datum(), paths, T, g)
    assert np.array_equal(ens[-1].status, wst[-1]) and ens[-1].blowup_count() == 3
    assert np.array_equal(ens[-1].states(), want[-1], equal_nan=True)
