"""The streaming x-march engine (term_xs.cu: lane = row, x-major term/accumulator tiles by TMA,
Y in registers; one Taylor term per pass, or two with S2B_XS2=1: term_xs2_kernel) against the reference CPU solver and against the row-marching streaming kernel
(term_tma_kernel, S2B_XS=0) on identical increments: bit patterns including zero signs, the
NZ (datum without -0.0) and literal folds, non-square grids, records, window-by-window session
advances (x-major <-> row-major relayout at every call), moments and snapshots between
advances, the adaptive driver, and the per-path Taylor-term counts."""
import numpy as np
import pytest

from test_gpu_parity import gpu_magnus

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["1", "2", "2h"], ids=["xs1", "xs2", "xs2h"])
def terms(request, monkeypatch):
    """terms per pass of the x-march engine (2h: 32-row items, t_k's halo rows by 2-point marches)"""
    monkeypatch.setenv("S2B_XS2", "0" if request.param == "1" else "1")
    monkeypatch.setenv("S2B_XS2H", "1" if request.param == "2h" else "0")
    return request.param


def _solve(s2b, ctx, g, order, phi, M, T, dt, seed, rec=(), **kw):
    op = s2b.Operator.from_family(g, "langevin-constant", order=order, ctx=ctx)
    paths = s2b.BrownianPaths.philox(T, 1e-4, M, seed=seed, ctx=ctx)
    stats = {}
    ens = s2b.solve_iterated_magnus(s2b.MagnusConfig(order=order, dt=dt, record_times=list(rec), **kw),
                                    op, phi, paths, T, g, stats=stats)
    return ens, stats, op


@pytest.mark.parametrize("negzero", [False, True])
@pytest.mark.parametrize("d,order", [(256, 3), (512, 3), (256, 2), (256, 1)])
def test_xs_bit_patterns_vs_reference(ref, s2b, ctx, monkeypatch, terms, negzero, d, order):
    monkeypatch.setenv("S2B_ENGINE", "stream")
    T, dt, dt_leb, M, seed = 0.02, 0.01, 1e-3, 2, 93 + d + order
    ops = ref.Ops("langevin-constant", d, order=order)
    phi = ops.datum().copy()
    phi[::5] = 0.0
    if negzero:
        phi[::13] = -0.0
    values, _ = ref.simulate_brownian(T, dt_leb, M, seed)
    want, wst, _ = ops.solve_magnus(values, dt_leb, T, dt, record_times=[0.01], seed=seed, phi=phi)
    ens, _, _, stats = gpu_magnus(s2b, ctx, "langevin-constant", d, order, values, dt_leb, T, dt,
                                  rec=[0.01], seed=seed, phi=phi)
    assert stats["engine"] == 0
    assert len(ens) == len(want)
    for r, e in enumerate(ens):
        assert np.array_equal(e.status, wst[r])
        assert np.array_equal(e.states().view(np.uint64), want[r].view(np.uint64))


@pytest.mark.parametrize("nx,nv,order", [(384, 96, 3), (256, 160, 2), (640, 64, 3), (256, 32, 1), (256, 56, 3)])
def test_xs_equals_row_march_non_square(s2b, ctx, monkeypatch, terms, nx, nv, order):
    """Non-square grids (several tiles, several row blocks, one row block): the x-march and the
    row-march streaming kernels give the same bits, records and Taylor-term counts."""
    monkeypatch.setenv("S2B_ENGINE", "stream")
    g = s2b.GridSpec(nx, nv, -4.0, 4.0, -3.0, 5.0)
    phi = s2b.gaussian_datum(g)
    T, dt, M = 0.006, 0.002, 5
    got, st_xs, _ = _solve(s2b, ctx, g, order, phi, M, T, dt, 41, rec=[0.002, 0.004])
    monkeypatch.setenv("S2B_XS", "0")
    monkeypatch.setenv("S2B_XS2", "0")
    monkeypatch.setenv("S2B_XS2H", "0")
    want, st_tma, _ = _solve(s2b, ctx, g, order, phi, M, T, dt, 41, rec=[0.002, 0.004])
    assert len(got) == len(want) == 3
    for w, e in zip(want, got):
        assert np.array_equal(w.status, e.status)
        assert np.array_equal(w.states().view(np.uint64), e.states().view(np.uint64))
    assert st_xs["path_terms"] == st_tma["path_terms"] > 0
    assert st_xs["path_segments"] == st_tma["path_segments"]


def test_xs_session_window_by_window(ref, s2b, ctx, monkeypatch, terms):
    """advance(1) at a time with moments and a snapshot between calls: the state is relaid out
    (row-major <-> x-major) around every pass loop; the result equals the reference's."""
    monkeypatch.setenv("S2B_ENGINE", "stream")
    d, T, dt, dt_leb, M, seed = 256, 0.04, 0.01, 1e-3, 3, 17
    ops = ref.Ops("langevin-constant", d, order=3)
    values, _ = ref.simulate_brownian(T, dt_leb, M, seed)
    want, wst, _ = ops.solve_magnus(values, dt_leb, T, dt, record_times=[0.02], seed=seed)
    g = s2b.GridSpec.square(d)
    op = s2b.Operator.from_family(g, "langevin-constant", order=3, ctx=ctx)
    paths = s2b.BrownianPaths.from_values(values, dt_leb, seed=seed, ctx=ctx)
    sess = s2b.MagnusSession(s2b.MagnusConfig(order=3, dt=dt, record_times=[0.02]), op, ops.datum(), paths, T)
    for w in range(4):
        sess.advance(1)
        s1, s2, live = sess.moments()
        assert live == M and np.isfinite(s1).all()
        if w == 1:  # t = 0.02: the record equals the snapshot taken now
            snap = sess.snapshot().states()
            assert np.array_equal(snap, want[0])
    ens = sess.finish()
    for r, e in enumerate(ens):
        assert np.array_equal(e.status, wst[r])
        assert np.array_equal(e.states(), want[r])


def test_xs_adaptive_vs_reference(ref, s2b, ctx, monkeypatch, terms):
    """solve_adaptive_magnus on the streaming x-march engine (one-window attempt sessions, two
    relayouts per attempt) against the reference's adaptive driver, bitwise."""
    monkeypatch.setenv("S2B_ENGINE", "stream")
    d, T, dt, dt_leb, M, seed = 256, 0.2, 0.1, 1e-3, 3, 267
    ops = ref.Ops("langevin-constant", d, order=3)
    values, _ = ref.simulate_brownian(T, dt_leb, M, seed)
    for tol in (1e-6, 1e-5, 1e-4, 1e-3):  # the tightest gate at which some path finishes Ok
        want, wst, _ = ops.solve_magnus(values, dt_leb, T, dt, order=3, record_times=[0.1], seed=seed,
                                        adaptive={"tolerance": tol, "shrink": 0.5})
        if (wst[-1] == 0).any():
            break
    g = s2b.GridSpec.square(d)
    op = s2b.Operator.from_family(g, "langevin-constant", order=3, ctx=ctx)
    paths = s2b.BrownianPaths.from_values(values, dt_leb, seed=seed, ctx=ctx)
    cfg = s2b.MagnusConfig(order=3, dt=dt, record_times=[0.1],
                           adaptive=s2b.AdaptiveConfig(enabled=True, tolerance=tol, shrink=0.5))
    ens = s2b.solve_adaptive_magnus(cfg, op, ops.datum(), paths, T, g)
    assert (wst[-1] == 0).any()  # not a degenerate all-blown case
    for r, e in enumerate(ens):
        assert np.array_equal(e.status, wst[r])
        assert np.array_equal(e.states(), want[r], equal_nan=True)


def test_xs_kernel_is_the_one_launched(s2b, ctx, monkeypatch):
    """At 1024^2 (cfg5's grid) the constant family runs on term_xs2_kernel by default, on
    term_xs_kernel with S2B_XS2=0 and on term_tma_kernel with S2B_XS=0 (the A/B switches)."""
    g = s2b.GridSpec.square(1024)
    phi = s2b.gaussian_datum(g)
    _solve(s2b, ctx, g, 3, phi, 2, 4e-4, 2e-4, 3)
    assert "term_xs2_kernel" in ctx.kernel_names().get("stream", "")  # two terms per pass: default
    monkeypatch.setenv("S2B_XS2", "0")
    _solve(s2b, ctx, g, 3, phi, 2, 4e-4, 2e-4, 3)
    assert "term_xs_kernel" in ctx.kernel_names().get("stream", "")
    monkeypatch.setenv("S2B_XS", "0")
    _solve(s2b, ctx, g, 3, phi, 2, 4e-4, 2e-4, 3)
    assert "term_tma_kernel" in ctx.kernel_names().get("stream", "")


@pytest.mark.parametrize("halo", ["0", "1"])
def test_xs2_kernel_is_the_one_launched_1024(ref, s2b, ctx, monkeypatch, halo):
    """cfg5's grid with two terms per pass (28-row items, or 32-row items with separate halo
    marches): term_xs2_kernel runs and the result is the reference's, bit for bit (records
    included)."""
    monkeypatch.setenv("S2B_XS2", "1")
    monkeypatch.setenv("S2B_XS2H", halo)
    d, T, dt, dt_leb, M, seed = 1024, 4e-4, 2e-4, 1e-5, 2, 1027
    ops = ref.Ops("langevin-constant", d, order=3)
    values, _ = ref.simulate_brownian(T, dt_leb, M, seed)
    want, wst, _ = ops.solve_magnus(values, dt_leb, T, dt, record_times=[dt], seed=seed)
    ens, _, _, stats = gpu_magnus(s2b, ctx, "langevin-constant", d, 3, values, dt_leb, T, dt, rec=[dt], seed=seed)
    assert "term_xs2_kernel" in ctx.kernel_names().get("stream", "")
    for r, e in enumerate(ens):
        assert np.array_equal(e.status, wst[r])
        assert np.array_equal(e.states().view(np.uint64), want[r].view(np.uint64))
