"""Engine coverage at the benchmark grid (256 x 256): every Magnus engine — the x-march
cluster kernel (default for constant Langevin), the row-band cluster kernel (S2B_XM=0) and
the streaming pass engines (S2B_ENGINE=stream: the x-march kernels with two terms per pass
and, S2B_XS2=0, one; S2B_XS=0: the row-march kernel) — against the reference CPU solver on
identical increments, bit for bit, including the blow-up exits (norm cap, non-finite
terms, exhausted Taylor budget) and record snapshots."""
import os

import numpy as np
import pytest

from test_gpu_parity import gpu_magnus

pytestmark = pytest.mark.gpu

ENGINES = {"xm": {}, "band": {"S2B_XM": "0"}, "stream": {"S2B_ENGINE": "stream"},
           "stream-xs1": {"S2B_ENGINE": "stream", "S2B_XS2": "0"},
           "stream-tma": {"S2B_ENGINE": "stream", "S2B_XS": "0"}}


@pytest.fixture
def engine(request, monkeypatch):
    for k, v in ENGINES[request.param].items():
        monkeypatch.setenv(k, v)
    return request.param


def _ref_run(ref, d, order, T, dt, dt_leb, M, seed, rec=(), **kw):
    ops = ref.Ops("langevin-constant", d, order=order)
    values, _ = ref.simulate_brownian(T, dt_leb, M, seed)
    want, wst, _ = ops.solve_magnus(values, dt_leb, T, dt, record_times=rec, seed=seed, **kw)
    return ops, values, want, wst


@pytest.mark.parametrize("engine", list(ENGINES), indirect=True)
@pytest.mark.parametrize("order", [1, 2, 3])
def test_engines_bitwise_256(ref, s2b, ctx, engine, order):
    d, T, dt, dt_leb, M, seed = 256, 0.02, 0.01, 1e-3, 3, 31 + order
    _, values, want, wst = _ref_run(ref, d, order, T, dt, dt_leb, M, seed, rec=[0.01])
    ens, _, _, stats = gpu_magnus(s2b, ctx, "langevin-constant", d, order, values, dt_leb, T, dt,
                                  rec=[0.01], seed=seed)
    assert len(ens) == len(want)
    for r, e in enumerate(ens):
        assert np.array_equal(e.status, wst[r])
        assert np.array_equal(e.states(), want[r], equal_nan=True)
    assert stats["path_terms"] > 0


@pytest.mark.parametrize("engine", ["xm"], indirect=True)
@pytest.mark.parametrize("d", [64, 128, 256])
@pytest.mark.parametrize("tol", [1e-4, 1e-8, 1e-13, 0.3])
def test_xm_stopping_rule_tolerances(ref, s2b, ctx, engine, d, tol):
    """The x-march kernel's stopping rule (path-wide maxima through DSMEM slots, one cluster
    barrier per term) against the reference's decisions at loose, default-like, tight and
    > 0.1 tolerances, bitwise."""
    T, dt, dt_leb, M, seed = 0.02, 0.01, 1e-3, 3, 71
    _, values, want, wst = _ref_run(ref, d, 3, T, dt, dt_leb, M, seed, rec=[0.01], tol=tol)
    ens, _, _, stats = gpu_magnus(s2b, ctx, "langevin-constant", d, 3, values, dt_leb, T, dt,
                                  rec=[0.01], seed=seed, expmv_tol=tol)
    for r, e in enumerate(ens):
        assert np.array_equal(e.status, wst[r])
        assert np.array_equal(e.states(), want[r], equal_nan=True)
    assert stats["engine"] == 2


@pytest.mark.parametrize("engine", ["xm", "band", "stream", "stream-xs1", "stream-tma"], indirect=True)
def test_engines_blowup_exits_256(ref, s2b, ctx, engine):
    d, T, dt, dt_leb, M = 256, 0.02, 0.01, 1e-3, 2
    # window norm cap
    _, values, want, wst = _ref_run(ref, d, 3, T, dt, dt_leb, M, 5, cap=1e-3)
    ens, _, _, _ = gpu_magnus(s2b, ctx, "langevin-constant", d, 3, values, dt_leb, T, dt, seed=5,
                              blowup_norm_cap=1e-3)
    assert np.array_equal(ens[-1].status, wst[-1]) and ens[-1].blowup_count() == M
    # exhausted Taylor budget (ToleranceNotReached)
    _, values, want, wst = _ref_run(ref, d, 2, T, dt, dt_leb, M, 6, tol=1e-300)
    ens, _, _, _ = gpu_magnus(s2b, ctx, "langevin-constant", d, 2, values, dt_leb, T, dt, seed=6,
                              expmv_tol=1e-300)
    assert np.array_equal(ens[-1].status, wst[-1]) and ens[-1].blowup_count() == M
    # non-finite terms (Overflow): a datum near DBL_MAX
    ops = ref.Ops("langevin-constant", d, order=3)
    phi = ops.datum() * 1e307
    values, _ = ref.simulate_brownian(T, dt_leb, M, 7)
    want, wst, _ = ops.solve_magnus(values, dt_leb, T, dt, seed=7, phi=phi)
    ens, _, _, _ = gpu_magnus(s2b, ctx, "langevin-constant", d, 3, values, dt_leb, T, dt, seed=7,
                              phi=phi)
    assert np.array_equal(ens[-1].status, wst[-1])
    assert np.array_equal(ens[-1].states(), want[-1], equal_nan=True)


EM_ENGINES = {"em-cluster": {}, "em-stream": {"S2B_EMXM": "0"}}


@pytest.fixture
def em_engine(request, monkeypatch):
    for k, v in EM_ENGINES[request.param].items():
        monkeypatch.setenv(k, v)
    return request.param


@pytest.mark.parametrize("em_engine", list(EM_ENGINES), indirect=True)
@pytest.mark.parametrize("d", [64, 128, 256, 512])
@pytest.mark.parametrize("family", ["langevin-constant", "langevin-variable"])
def test_euler_engines_bitwise_256(ref, s2b, ctx, em_engine, d, family):
    """solve_euler at 256^2 / 512^2 (Langevin: the cluster-resident kernels, in place; the
    variable family's a(x), sigma(x) from a column table) vs the reference, with a mid-run
    record."""
    T, dt_leb, dt, M, seed = 0.01, 1e-4, 1e-4, 4, 21
    ops = ref.Ops(family, d, order=1)
    values, _ = ref.simulate_brownian(T, dt_leb, M, seed)
    want, wst, _ = ops.solve_euler(values, dt_leb, T, dt, record_times=[0.005], seed=seed)
    g = s2b.GridSpec.square(d)
    f = s2b.Fields.from_family(g, family, ctx=ctx)
    paths = s2b.BrownianPaths.from_values(values, dt_leb, seed=seed, ctx=ctx)
    ens = s2b.solve_euler(s2b.EulerConfig(dt=dt, record_times=[0.005]), f, g, ops.datum(), paths, T)
    assert len(ens) == len(want)
    for r, e in enumerate(ens):
        assert np.array_equal(e.status, wst[r])
        assert np.array_equal(e.states(), want[r])


@pytest.mark.parametrize("em_engine", list(EM_ENGINES), indirect=True)
@pytest.mark.parametrize("d", [64, 256, 512])
def test_euler_engines_blowup_256(ref, s2b, ctx, em_engine, d):
    """dt far beyond the stability bound: Ok (finite, huge) at t = 20, blown by T = 200."""
    T, M, seed = 200.0, 2, 9
    values, _ = ref.simulate_brownian(T, 1.0, M, seed)
    ops = ref.Ops("langevin-constant", d, order=1)
    want, wst, _ = ops.solve_euler(values, 1.0, T, 1.0, record_times=[20.0], seed=seed)
    g = s2b.GridSpec.square(d)
    f = s2b.Fields.from_family(g, "langevin-constant", ctx=ctx)
    paths = s2b.BrownianPaths.from_values(values, 1.0, seed=seed, ctx=ctx)
    ens = s2b.solve_euler(s2b.EulerConfig(dt=1.0, record_times=[20.0]), f, g, ops.datum(), paths, T)
    assert np.array_equal(ens[0].status, wst[0]) and np.array_equal(ens[-1].status, wst[-1])
    assert ens[-1].blowup_count() == M
    assert np.array_equal(ens[0].states(), want[0])


ENGINES_512 = {"xmi": {}, "stream": {"S2B_ENGINE": "stream"},
               "stream-tma": {"S2B_ENGINE": "stream", "S2B_XS": "0"}}


@pytest.fixture
def engine512(request, monkeypatch):
    for k, v in ENGINES_512[request.param].items():
        monkeypatch.setenv(k, v)
    return request.param


@pytest.mark.parametrize("engine512", list(ENGINES_512), indirect=True)
@pytest.mark.parametrize("order", [2, 3])
def test_engines_bitwise_512(ref, s2b, ctx, engine512, order):
    """512^2: the in-place cluster engine (16-CTA clusters, accumulator in L2) and the
    streaming engine against the reference, with a record snapshot."""
    d, T, dt, dt_leb, M, seed = 512, 0.02, 0.01, 1e-3, 2, 51 + order
    _, values, want, wst = _ref_run(ref, d, order, T, dt, dt_leb, M, seed, rec=[0.01])
    ens, _, _, stats = gpu_magnus(s2b, ctx, "langevin-constant", d, order, values, dt_leb, T, dt,
                                  rec=[0.01], seed=seed)
    assert len(ens) == len(want)
    for r, e in enumerate(ens):
        assert np.array_equal(e.status, wst[r])
        assert np.array_equal(e.states(), want[r], equal_nan=True)
    assert stats["engine"] == (3 if engine512 == "xmi" else 0)


@pytest.mark.parametrize("engine512", ["xmi"], indirect=True)
def test_engines_blowup_exits_512(ref, s2b, ctx, engine512):
    d, T, dt, dt_leb, M = 512, 0.02, 0.01, 1e-3, 2
    _, values, want, wst = _ref_run(ref, d, 3, T, dt, dt_leb, M, 5, cap=1e-3)
    ens, _, _, _ = gpu_magnus(s2b, ctx, "langevin-constant", d, 3, values, dt_leb, T, dt, seed=5,
                              blowup_norm_cap=1e-3)
    assert np.array_equal(ens[-1].status, wst[-1]) and ens[-1].blowup_count() == M


@pytest.mark.parametrize("slice_engine", ["xs", "tma"])
@pytest.mark.parametrize("d", [256, 512])
def test_hybrid_split_bitwise(s2b, ctx, monkeypatch, d, slice_engine):
    """S2B_HYBRID: a slice of the paths runs on the streaming engine beside the cluster kernel
    (on the SMs the clusters leave idle); every path's result is unchanged."""
    T, dt, dt_leb, M = 0.02, 0.01, 1e-3, 96
    g = s2b.GridSpec.square(d)
    op = s2b.Operator.from_family(g, "langevin-constant", order=3, ctx=ctx)
    paths = s2b.BrownianPaths.philox(T, dt_leb, M, seed=23, ctx=ctx)
    phi = s2b.gaussian_datum(g)
    cfg = s2b.MagnusConfig(order=3, dt=dt, record_times=[0.01])
    monkeypatch.setenv("S2B_XS_SLICE", "1" if slice_engine == "xs" else "0")
    monkeypatch.setenv("S2B_HYBRID", "0")
    want = s2b.solve_iterated_magnus(cfg, op, phi, paths, T, g)
    monkeypatch.setenv("S2B_HYBRID", "0.3")
    got = s2b.solve_iterated_magnus(cfg, op, phi, paths, T, g)
    for w, e in zip(want, got):
        assert np.array_equal(w.status, e.status)
        assert np.array_equal(w.states(), e.states(), equal_nan=True)


@pytest.mark.parametrize("em_engine", ["em-cluster"], indirect=True)
@pytest.mark.parametrize("negzero", [False, True])
def test_euler_cluster_bit_patterns(ref, s2b, ctx, em_engine, negzero):
    """Bit patterns, not just values, including the sign of zeros: a datum without -0.0 takes
    the shortened drift / noise folds (em_cluster.cu, NZ), one with -0.0 the literal ones."""
    d, T, dt_leb, M, seed = 256, 0.005, 1e-4, 2, 77
    ops = ref.Ops("langevin-constant", d, order=1)
    phi = ops.datum().copy()
    phi[::7] = 0.0  # zero rows of points whose stencil sums vanish
    if negzero:
        phi[::11] = -0.0
    values, _ = ref.simulate_brownian(T, dt_leb, M, seed)
    want, wst, _ = ops.solve_euler(values, dt_leb, T, dt_leb, seed=seed, phi=phi)
    g = s2b.GridSpec.square(d)
    f = s2b.Fields.from_family(g, "langevin-constant", ctx=ctx)
    paths = s2b.BrownianPaths.from_values(values, dt_leb, seed=seed, ctx=ctx)
    got = s2b.solve_euler(s2b.EulerConfig(dt=dt_leb), f, g, phi, paths, T)[-1].states()
    assert np.array_equal(got.view(np.uint64), want[-1].view(np.uint64))


@pytest.mark.parametrize("negzero", [False, True])
@pytest.mark.parametrize("d", [256, 512])
def test_xm_bit_patterns(ref, s2b, ctx, negzero, d):
    """x-march Magnus (256^2 cluster_xm, 512^2 in-place cluster_xmi): bit patterns (incl. zero
    signs) equal the reference's, with the shortened stencil fold (datum without -0.0) and the
    literal one (datum with -0.0)."""
    T, dt, dt_leb, M, seed = 0.02, 0.01, 1e-3, 2, 91
    ops = ref.Ops("langevin-constant", d, order=3)
    phi = ops.datum().copy()
    phi[::5] = 0.0
    if negzero:
        phi[::13] = -0.0
    values, _ = ref.simulate_brownian(T, dt_leb, M, seed)
    want, wst, _ = ops.solve_magnus(values, dt_leb, T, dt, seed=seed, phi=phi)
    ens, _, _, stats = gpu_magnus(s2b, ctx, "langevin-constant", d, 3, values, dt_leb, T, dt, seed=seed, phi=phi)
    assert stats["engine"] == (2 if d == 256 else 3)
    assert np.array_equal(ens[-1].status, wst[-1])
    assert np.array_equal(ens[-1].states().view(np.uint64), want[-1].view(np.uint64))


@pytest.mark.parametrize("d,order", [(64, 2), (128, 3), (64, 3)])
def test_xm_small_grids_bitwise(ref, s2b, ctx, d, order):
    """x-march engine on 128^2 (4-CTA clusters) and 64^2 (one CTA per path) vs the reference."""
    T, dt, dt_leb, M, seed = 0.2, 0.1, 1e-3, 3, 61 + d
    _, values, want, wst = _ref_run(ref, d, order, T, dt, dt_leb, M, seed, rec=[0.1])
    ens, _, _, stats = gpu_magnus(s2b, ctx, "langevin-constant", d, order, values, dt_leb, T, dt,
                                  rec=[0.1], seed=seed)
    assert stats["engine"] == 2
    for r, e in enumerate(ens):
        assert np.array_equal(e.status, wst[r])
        assert np.array_equal(e.states(), want[r], equal_nan=True)


@pytest.mark.parametrize("em_engine", list(EM_ENGINES), indirect=True)
@pytest.mark.parametrize("d", [64, 128, 256, 512])
def test_euler_kinetic_fields_bitwise(ref, s2b, ctx, em_engine, d):
    """The paper's general kinetic SPDE (x/v-dependent a, b, c, sigma, beta): the in-place
    cluster E-M kernels read every field per point from a (0.5 g pre-applied) table; the
    streaming kernels as before; both bitwise against the reference with a mid-run record."""
    from fieldsets import kinetic_fields
    T, dt_leb, M, seed = 0.002, 1e-4, 4, 31
    fields = kinetic_fields(d)
    ops = ref.Ops("fields", d, order=1, fields=fields)
    values, _ = ref.simulate_brownian(T, dt_leb, M, seed)
    want, wst, _ = ops.solve_euler(values, dt_leb, T, dt_leb, record_times=[0.0007], seed=seed)
    g = s2b.GridSpec.square(d)
    f = s2b.Fields.from_arrays(g, fields, ctx=ctx)
    paths = s2b.BrownianPaths.from_values(values, dt_leb, seed=seed, ctx=ctx)
    ens = s2b.solve_euler(s2b.EulerConfig(dt=dt_leb, record_times=[0.0007]), f, g, ops.datum(), paths, T)
    for r, e in enumerate(ens):
        assert np.array_equal(e.status, wst[r])
        assert np.array_equal(e.states(), want[r])
