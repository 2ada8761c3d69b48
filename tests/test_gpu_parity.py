"""GPU parity tests: the sm_100a path through the C ABI vs the reference's CPU implementation
on identical increments.  The bar is bit-exactness (np.array_equal) for the solution fields
of both schemes, the statuses and the norms computed from identical ensembles; the closed
form differs only through exp() (CUDA vs glibc), so it is held to 1e-14 relative."""
import glob
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))
SIGMA = 1.0 / np.sqrt(10.0)


def gpu_magnus(s2b, ctx, family, d, order, values, dt_leb, T, dt, rec=(), seed=1, phi=None,
               ops_csr=None, **kw):
    g = s2b.GridSpec.square(d)
    if ops_csr is not None:
        op = s2b.Operator.from_csr(g, order, ops_csr, ctx=ctx)
    else:
        op = s2b.Operator.from_family(g, family, order=order, ctx=ctx)
    paths = s2b.BrownianPaths.from_values(values, dt_leb, seed=seed, ctx=ctx)
    phi = s2b.gaussian_datum(g) if phi is None else phi
    stats = {}
    ens = s2b.solve_iterated_magnus(s2b.MagnusConfig(order=order, dt=dt, record_times=list(rec), **kw),
                                    op, phi, paths, T, g, stats=stats)
    return ens, op, paths, stats


CASES = [
    ("langevin-constant", 16, 3, 0.1), ("langevin-constant", 24, 2, 0.05),
    ("langevin-constant", 14, 1, 0.1), ("langevin-constant", 9, 3, 0.1),
    ("langevin-constant", 64, 3, 0.1), ("langevin-constant", 6, 3, 0.1),
    ("langevin-variable", 16, 3, 0.1), ("langevin-variable", 20, 2, 0.05),
    ("langevin-variable", 33, 3, 0.1), ("langevin-constant", 130, 3, 0.05),
]


@pytest.mark.parametrize("family,d,order,dt", CASES)
def test_magnus_bitwise_vs_reference(ref, s2b, ctx, family, d, order, dt):
    T, dt_leb, M, seed = 0.2, 1e-3, 4, 7 + d
    ops = ref.Ops(family, d, order=order)
    values, _ = ref.simulate_brownian(T, dt_leb, M, seed)
    rec = [0.1]
    want, wst, _ = ops.solve_magnus(values, dt_leb, T, dt, record_times=rec, seed=seed)
    ens, op, _, _ = gpu_magnus(s2b, ctx, family, d, order, values, dt_leb, T, dt, rec, seed)
    assert len(ens) == len(want)
    for r, e in enumerate(ens):
        assert np.array_equal(e.status, wst[r])
        assert np.array_equal(e.states(), want[r], equal_nan=True)
    # the reference's own CSR CommutatorSet through s2b_operator_create gives the same bits
    ens2, _, _, _ = gpu_magnus(s2b, ctx, family, d, order, values, dt_leb, T, dt, rec, seed,
                               ops_csr=[ops.csr(s) for s in ref.SLOTS])
    assert np.array_equal(ens2[-1].states(), want[-1], equal_nan=True)


def test_magnus_term_counts_match_oracle(ref, rs, s2b, ctx):
    """Per-path Taylor-term and window counts equal the reference rule's (S*K)."""
    d, order, T, dt_leb, dt, M = 20, 3, 0.3, 1e-3, 0.1, 3
    ops = ref.Ops("langevin-constant", d, order=order)
    values, _ = ref.simulate_brownian(T, dt_leb, M, 3)
    ens, _, _, stats = gpu_magnus(s2b, ctx, "langevin-constant", d, order, values, dt_leb, T, dt)
    terms, windows = ens[-1].counters()
    srcs = [ops.csr(s) for s in ref.SLOTS]
    for m in range(M):
        _, _, wt, _ = rs.magnus_path(d * d, order, srcs, ops.datum(), values[m], dt_leb, 100, 300, [300])
        assert terms[m] == wt.sum() and windows[m] == 3
    assert stats["path_terms"] == terms.sum()


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p) for p in GOLDEN])
def test_magnus_and_euler_reproduce_golden(s2b, ctx, path):
    """Runs without /root/reference: the committed fixtures made by the reference itself."""
    g = dict(np.load(path))
    d, order, M = int(g["d"]), int(g["order"]), int(g["M"])
    dt_leb, dt, T = float(g["dt_leb"]), float(g["dt"]), float(g["T"])
    srcs = []
    for slot in ("B", "A", "A2", "BA", "BAA", "BAB"):
        k = f"csr_{slot}_rp"
        srcs.append((g[k], g[f"csr_{slot}_ci"], g[f"csr_{slot}_v"]) if k in g else None)
    grid = s2b.GridSpec.square(d)
    op = s2b.Operator.from_csr(grid, order, srcs, ctx=ctx)
    paths = s2b.BrownianPaths.from_values(g["values"], dt_leb, seed=int(g["seed"]), ctx=ctx)
    rec = list(g["record_times"])
    ens = s2b.solve_iterated_magnus(s2b.MagnusConfig(order=order, dt=dt, record_times=rec), op,
                                    g["phi"], paths, T, grid)
    for r, e in enumerate(ens):
        assert np.array_equal(e.status, g["magnus_status"][r])
        assert np.array_equal(e.states(), g["magnus"][r], equal_nan=True)
    fields = {n: g[f"field_{n}"] for n in ("h", "fx", "fv", "gxx", "gxv", "gvv", "sig", "sigx", "sigv")
              if f"field_{n}" in g}
    f = s2b.Fields.from_arrays(grid, fields, ctx=ctx)
    em = s2b.solve_euler(s2b.EulerConfig(dt=float(g["em_dt"]), record_times=rec), f, grid, g["phi"],
                         paths, T)
    for r, e in enumerate(em):
        assert np.array_equal(e.status, g["euler_status"][r])
        assert np.array_equal(e.states(), g["euler"][r], equal_nan=True)
    if "exact" in g:
        ex = s2b.exact_reference(grid, T, 1.1, SIGMA, paths)
        got = ex.states()
        assert np.max(np.abs(got - g["exact"]) / np.abs(g["exact"])) <= 1e-14
        for kappa in (0, 2):
            st = s2b.exact_errors(ens[-1], 1.1, SIGMA, paths, kappa)
            want = g[f"err_k{kappa}"]
            assert abs(st["err"] - want[0]) <= 1e-12 * abs(want[0])
            assert abs(st["ame"] - want[1]) <= 1e-12 * abs(want[1])


def test_magnus_custom_nine_fields(ref, s2b, ctx):
    """General kinetic SPDE with all nine coefficient fields: 45-point order-3 stencil
    (radius 3), non-compressed weights -> generic kernel; still bitwise."""
    from fieldsets import custom_fields
    d, order, T, dt_leb, dt = 14, 3, 0.1, 1e-3, 0.05
    fields = custom_fields(d)
    ops = ref.Ops("fields", d, order=order, fields=fields)
    values, _ = ref.simulate_brownian(T, dt_leb, 2, 5)
    want, wst, _ = ops.solve_magnus(values, dt_leb, T, dt, seed=5)
    g = s2b.GridSpec.square(d)
    op = s2b.Operator.from_family(g, "fields", order=order, fields=fields, ctx=ctx)
    info = op.info()
    assert info["stencil_points"] == 45 and info["rx"] == 3 and info["rv"] == 3
    paths = s2b.BrownianPaths.from_values(values, dt_leb, seed=5, ctx=ctx)
    ens = s2b.solve_iterated_magnus(s2b.MagnusConfig(order=order, dt=dt), op, ops.datum(), paths, T, g)
    assert np.array_equal(ens[-1].states(), want[-1], equal_nan=True)


@pytest.mark.parametrize("d,order", [(16, 2), (20, 3), (130, 3), (258, 2)])
def test_magnus_kinetic_variable_fields(ref, s2b, ctx, d, order):
    """The paper's general kinetic SPDE with x- and v-dependent a, b, c, sigma, beta (23-point
    order-3 union, 64 source pairs): term_var_kernel / term_varx_kernel (64-column parts,
    a last part 2 columns wide at 130 / 258), bitwise."""
    from fieldsets import kinetic_fields
    T, dt_leb, dt = 0.004, 1e-4, 0.002
    fields = kinetic_fields(d)
    ops = ref.Ops("fields", d, order=order, fields=fields)
    values, _ = ref.simulate_brownian(T, dt_leb, 5, d)
    want, wst, _ = ops.solve_magnus(values, dt_leb, T, dt, record_times=[dt], seed=d)
    g = s2b.GridSpec.square(d)
    op = s2b.Operator.from_family(g, "fields", order=order, fields=fields, ctx=ctx)
    info = op.info()
    assert info["stencil_points"] == (23 if order == 3 else 11)
    paths = s2b.BrownianPaths.from_values(values, dt_leb, seed=d, ctx=ctx)
    ens = s2b.solve_iterated_magnus(s2b.MagnusConfig(order=order, dt=dt, record_times=[dt]), op,
                                    ops.datum(), paths, T, g)
    for r, e in enumerate(ens):
        assert np.array_equal(e.status, wst[r])
        assert np.array_equal(e.states(), want[r], equal_nan=True)


def test_magnus_blowup_flagged(ref, s2b, ctx):
    """test_magnus.cpp:208-223: a tiny norm cap trips on the first window."""
    d, T, dt_leb = 10, 0.2, 1e-3
    values, _ = ref.simulate_brownian(T, dt_leb, 3, 8)
    ens, _, _, _ = gpu_magnus(s2b, ctx, "langevin-constant", d, 2, values, dt_leb, T, 0.1,
                              seed=8, blowup_norm_cap=1e-6)
    assert ens[-1].blowup_count() == 3
    assert np.all(np.isnan(ens[-1].states()))
    ops = ref.Ops("langevin-constant", d, order=2)
    _, wst, _ = ops.solve_magnus(values, dt_leb, T, 0.1, cap=1e-6, seed=8)
    assert np.array_equal(ens[-1].status, wst[-1])


def test_magnus_tolerance_budget_blowup(ref, s2b, ctx):
    """An unreachable tolerance exhausts the 55-term budget: ToleranceNotReached -> blown."""
    d, T, dt_leb = 12, 0.1, 1e-3
    values, _ = ref.simulate_brownian(T, dt_leb, 2, 4)
    ens, _, _, _ = gpu_magnus(s2b, ctx, "langevin-constant", d, 3, values, dt_leb, T, 0.1, seed=4,
                              expmv_tol=1e-300)
    ops = ref.Ops("langevin-constant", d, order=3)
    _, wst, _ = ops.solve_magnus(values, dt_leb, T, 0.1, tol=1e-300, seed=4)
    assert np.array_equal(ens[-1].status, wst[-1]) and ens[-1].blowup_count() == 2


def test_magnus_record_snapshot_equals_truncated_run(ref, s2b, ctx):
    """test_magnus.cpp:225-243: the first snapshot equals a run stopped there, bitwise."""
    d, dt_leb = 8, 1e-3
    values, _ = ref.simulate_brownian(0.4, dt_leb, 2, 5)
    ens, _, _, _ = gpu_magnus(s2b, ctx, "langevin-constant", d, 2, values, dt_leb, 0.4, 0.1,
                              rec=[0.2, 0.4], seed=5)
    assert len(ens) == 2 and abs(ens[0].t - 0.2) < 1e-12
    stop, _, _, _ = gpu_magnus(s2b, ctx, "langevin-constant", d, 2, values, dt_leb, 0.2, 0.1, seed=5)
    assert np.array_equal(ens[0].states(), stop[-1].states())


def test_magnus_deterministic_window_invariance(ref, s2b, ctx):
    """test_magnus.cpp:174-187: sigma = 0, order 1: one window of 0.5 == ten of 0.05 (1e-8)."""
    d = 20
    values, _ = ref.simulate_brownian(0.5, 1e-3, 2, 3)
    g = s2b.GridSpec.square(d)
    op = s2b.Operator.from_family(g, "langevin-constant", sigma=0.0, order=1, ctx=ctx)
    paths = s2b.BrownianPaths.from_values(values, 1e-3, seed=3, ctx=ctx)
    phi = s2b.gaussian_datum(g)
    one = s2b.solve_iterated_magnus(s2b.MagnusConfig(order=1, dt=0.5), op, phi, paths, 0.5, g)[-1].states()
    ten = s2b.solve_iterated_magnus(s2b.MagnusConfig(order=1, dt=0.05), op, phi, paths, 0.5, g)[-1].states()
    assert np.max(np.abs(one[0] - ten[0])) / np.max(np.abs(ten[0])) <= 1e-8


def test_session_windows_equal_full_solve(ref, s2b, ctx):
    """Advancing a resident session window by window equals the one-shot solve bitwise,
    and repeated runs are bit-identical (the reference's thread-count invariance)."""
    d, T, dt_leb, dt = 32, 0.3, 1e-3, 0.05
    g = s2b.GridSpec.square(d)
    op = s2b.Operator.from_family(g, "langevin-constant", order=3, ctx=ctx)
    paths = s2b.BrownianPaths.philox(T, dt_leb, 6, seed=11, ctx=ctx)
    phi = s2b.gaussian_datum(g)
    cfg = s2b.MagnusConfig(order=3, dt=dt)
    full = s2b.solve_iterated_magnus(cfg, op, phi, paths, T, g)[-1].states()
    again = s2b.solve_iterated_magnus(cfg, op, phi, paths, T, g)[-1].states()
    assert np.array_equal(full, again)
    sess = s2b.MagnusSession(cfg, op, phi, paths, T)
    for _ in range(6):
        sess.advance(1)
    snap = sess.snapshot().states()
    assert np.array_equal(snap, full)
    s1, s2, live = sess.moments()
    assert live == 6
    assert np.allclose(s1, full.sum(0), rtol=1e-14, atol=0)
    sess.reset()
    sess.advance(2)
    sess.advance(4)
    assert np.array_equal(sess.finish()[-1].states(), full)


def test_philox_paths_feed_the_reference(ref, s2b, ctx):
    """Philox mode: the device-generated prefix values, given to the reference, reproduce the
    GPU solution bitwise (so Philox runs are checkable path by path), and are N(0, dt_leb)."""
    d, T, dt_leb = 16, 0.2, 1e-3
    paths = s2b.BrownianPaths.philox(T, dt_leb, 4, seed=99, path_offset=1000, ctx=ctx)
    values = paths.values()
    assert np.all(values[:, 0] == 0.0)
    inc = np.diff(values, axis=1)
    assert abs(inc.std() / np.sqrt(dt_leb) - 1.0) < 0.05
    g = s2b.GridSpec.square(d)
    op = s2b.Operator.from_family(g, "langevin-constant", order=3, ctx=ctx)
    ens = s2b.solve_iterated_magnus(s2b.MagnusConfig(order=3, dt=0.1), op, s2b.gaussian_datum(g),
                                    paths, T, g)
    want, _, _ = ref.Ops("langevin-constant", d, order=3).solve_magnus(values, dt_leb, T, 0.1, seed=99)
    assert np.array_equal(ens[-1].states(), want[-1])
    # sharding invariance: path 1001 of offset 1000 == path 1 of a batch at offset 1000
    p2 = s2b.BrownianPaths.philox(T, dt_leb, 2, seed=99, path_offset=1001, ctx=ctx)
    assert np.array_equal(p2.values()[0], values[1])


@pytest.mark.parametrize("family", ["langevin-constant", "langevin-variable"])
def test_euler_bitwise_vs_reference(ref, s2b, ctx, family):
    d, T, dt_leb = 24, 0.05, 1e-4
    ops = ref.Ops(family, d, order=1)
    values, _ = ref.simulate_brownian(T, dt_leb, 3, 17)
    want, wst, _ = ops.solve_euler(values, dt_leb, T, 2e-4, record_times=[0.02], seed=17)
    g = s2b.GridSpec.square(d)
    f = s2b.Fields.from_family(g, family, ctx=ctx)
    paths = s2b.BrownianPaths.from_values(values, dt_leb, seed=17, ctx=ctx)
    ens = s2b.solve_euler(s2b.EulerConfig(dt=2e-4, record_times=[0.02]), f, g, ops.datum(), paths, T)
    for r, e in enumerate(ens):
        assert np.array_equal(e.status, wst[r])
        assert np.array_equal(e.states(), want[r])


def test_euler_stiff_blowup_flagged(ref, s2b, ctx):
    """test_euler.cpp:123-140: dt far beyond the stability bound blows up and is flagged."""
    d = 40
    values, _ = ref.simulate_brownian(200.0, 1.0, 2, 9)
    g = s2b.GridSpec.square(d)
    phi = np.array([1.0 if (i + j) % 2 == 0 else -1.0 for j in range(d) for i in range(d)])
    f = s2b.Fields.from_family(g, "langevin-constant", sigma=0.0, ctx=ctx)
    paths = s2b.BrownianPaths.from_values(values, 1.0, seed=9, ctx=ctx)
    ens = s2b.solve_euler(s2b.EulerConfig(dt=1.0), f, g, phi, paths, 200.0)
    ops = ref.Ops("langevin-constant", d, sigma=0.0, order=1)
    _, wst, _ = ops.solve_euler(values, 1.0, 200.0, 1.0, phi=phi, seed=9)
    assert np.array_equal(ens[-1].status, wst[-1]) and ens[-1].blowup_count() == 2


def test_euler_all_nine_fields_bitwise(ref, s2b, ctx):
    from fieldsets import custom_fields
    d, T, dt_leb = 12, 0.02, 1e-3
    fields = custom_fields(d)
    ops = ref.Ops("fields", d, order=1, fields=fields)
    values, _ = ref.simulate_brownian(T, dt_leb, 2, 2)
    want, wst, _ = ops.solve_euler(values, dt_leb, T, dt_leb, seed=2)
    g = s2b.GridSpec.square(d)
    f = s2b.Fields.from_arrays(g, fields, ctx=ctx)
    paths = s2b.BrownianPaths.from_values(values, dt_leb, seed=2, ctx=ctx)
    ens = s2b.solve_euler(s2b.EulerConfig(dt=dt_leb), f, g, ops.datum(), paths, T)
    assert np.array_equal(ens[-1].states(), want[-1])


def test_exact_reference_and_norms(ref, s2b, ctx):
    d, T, dt_leb, M = 32, 0.3, 1e-3, 5
    ops = ref.Ops("langevin-constant", d, order=3)
    values, _ = ref.simulate_brownian(T, dt_leb, M, 21)
    want = ops.exact_reference(values, dt_leb, T, seed=21)
    g = s2b.GridSpec.square(d)
    paths = s2b.BrownianPaths.from_values(values, dt_leb, seed=21, ctx=ctx)
    ex = s2b.exact_reference(g, T, 1.1, SIGMA, paths)
    assert np.max(np.abs(ex.states() - want) / np.abs(want)) <= 1e-14
    ens, _, _, _ = gpu_magnus(s2b, ctx, "langevin-constant", d, 3, values, dt_leb, T, 0.1, seed=21)
    app = ens[-1]
    for kappa in (0, 2, 4):
        # GPU norms on identical ensembles == reference norms, bitwise
        got = s2b.mean_rel_error(ex, app, kappa)
        me = s2b.mean_abs_error(ex, app, kappa)
        w = ops.errors(kappa, ex.states(), app.states(), app_status=app.status, seed=21)
        assert got["err"] == w["err"] and me["ame"] == w["ame"]
        assert np.array_equal(me["me"], w["me"])
        # fused exact norms (no reference ensemble) vs the reference's own exact_reference
        w2 = ops.errors(kappa, want, app.states(), app_status=app.status, seed=21)
        fz = s2b.exact_errors(app, 1.1, SIGMA, paths, kappa, moments=True)
        assert abs(fz["err"] - w2["err"]) <= 1e-12 * w2["err"]
        assert np.allclose(fz["me"], w2["me"], rtol=1e-10, atol=1e-17)
        assert np.allclose(fz["sum_u"], app.states().sum(0), rtol=1e-13)


def test_norms_blowup_semantics(ref, s2b, ctx):
    d, T, dt_leb = 10, 0.2, 1e-3
    values, _ = ref.simulate_brownian(T, dt_leb, 3, 8)
    g = s2b.GridSpec.square(d)
    paths = s2b.BrownianPaths.from_values(values, dt_leb, seed=8, ctx=ctx)
    ex = s2b.exact_reference(g, T, 1.1, SIGMA, paths)
    ens, _, _, _ = gpu_magnus(s2b, ctx, "langevin-constant", d, 2, values, dt_leb, T, 0.1, seed=8,
                              blowup_norm_cap=1e-6)
    r = s2b.mean_rel_error(ex, ens[-1], 0)
    assert r["err"] == np.inf and r["blowups"] == 3
    assert s2b.mean_abs_error(ex, ens[-1], 0)["excluded"] == 3
    with pytest.raises(s2b.ConfigError):
        s2b.mean_rel_error(ens[-1], ex, 0)  # blown reference -> ConfigError


def test_expmv_general_csr_bitwise(ref, s2b, ctx):
    rng = np.random.default_rng(27)
    for rep in range(6):
        n = 9
        dense = np.where(rng.random((n, n)) < 0.5, rng.uniform(-1, 1, (n, n)), 0.0)
        rp = np.zeros(n + 1, np.uint64)
        ci, v = [], []
        for r in range(n):
            nz = np.nonzero(dense[r])[0]
            ci += list(nz)
            v += list(dense[r, nz])
            rp[r + 1] = len(ci)
        ci = np.array(ci, np.int32)
        v = np.array(v)
        x = rng.normal(size=n)
        y, rep_g = s2b.expmv((rp, ci, v), x, 1e-10, ctx=ctx)
        yw, rep_w = ref.expmv(rp, ci, v, x, 1e-10)
        assert np.array_equal(y, yw)
        assert (rep_g["segments"], rep_g["max_terms"]) == (rep_w["segments"], rep_w["max_terms"])
    with pytest.raises(s2b.ExpmvError):
        s2b.expmv((np.arange(5, dtype=np.uint64), np.arange(4, dtype=np.int32), np.full(4, 2000.0)),
                  np.ones(4), 1e-10, ctx=ctx)
    z, rep = s2b.expmv((np.zeros(7, np.uint64), np.zeros(0, np.int32), np.zeros(0)), np.ones(6), 1e-12, ctx=ctx)
    assert np.array_equal(z, np.ones(6))


def test_config_errors_mirror_reference(s2b, ctx):
    g = s2b.GridSpec.square(8)
    op = s2b.Operator.from_family(g, "langevin-constant", order=2, ctx=ctx)
    paths = s2b.BrownianPaths.philox(0.2, 1e-3, 2, ctx=ctx)
    phi = s2b.gaussian_datum(g)
    with pytest.raises(s2b.ConfigError):  # order above the commutator set
        s2b.solve_iterated_magnus(s2b.MagnusConfig(order=3, dt=0.1), op, phi, paths, 0.2, g)
    with pytest.raises(s2b.ConfigError):  # T not a multiple of dt
        s2b.solve_iterated_magnus(s2b.MagnusConfig(order=2, dt=0.15), op, phi, paths, 0.2, g)
    with pytest.raises(s2b.ConfigError):  # record time off the window grid
        s2b.solve_iterated_magnus(s2b.MagnusConfig(order=2, dt=0.1, record_times=[0.05]), op, phi,
                                  paths, 0.2, g)
    with pytest.raises(s2b.ConfigError):  # non-finite datum
        bad = phi.copy()
        bad[3] = np.nan
        s2b.solve_iterated_magnus(s2b.MagnusConfig(order=2, dt=0.1), op, bad, paths, 0.2, g)
    with pytest.raises(s2b.DimensionError):
        s2b.solve_iterated_magnus(s2b.MagnusConfig(order=2, dt=0.1), op, phi[:-1], paths, 0.2, g)


def test_smoke_entry(s2b):
    import __graft_entry__
    __graft_entry__.smoke()


# BASELINE cfg3 at its exact grid (256^2, dt = 0.01, dt_leb = 1e-4): the engines bench.py
# --config cfg3 / cfg3k time (term_var_kernel with TMA weight rows and the largest ring;
# term_varx_kernel at the kinetic family's 64 source pairs), two windows plus a record.
@pytest.mark.parametrize("kind,order,pairs", [("langevin-variable", 2, 15), ("langevin-variable", 3, 39),
                                              ("kinetic", 2, 24), ("kinetic", 3, 64)])
def test_magnus_cfg3_grid_bitwise(ref, s2b, ctx, kind, order, pairs):
    from fieldsets import kinetic_fields
    d, T, dt_leb, dt, M, seed = 256, 0.02, 1e-4, 0.01, 4, 303 + order
    fields = kinetic_fields(d) if kind == "kinetic" else None
    family = "fields" if kind == "kinetic" else kind
    ops = ref.Ops(family, d, order=order, fields=fields)
    values, _ = ref.simulate_brownian(T, dt_leb, M, seed)
    want, wst, _ = ops.solve_magnus(values, dt_leb, T, dt, record_times=[dt], seed=seed)
    g = s2b.GridSpec.square(d)
    op = s2b.Operator.from_family(g, family, order=order, fields=fields, ctx=ctx)
    info = op.info()
    assert not info["compressed"] and info["pairs"] == pairs
    paths = s2b.BrownianPaths.from_values(values, dt_leb, seed=seed, ctx=ctx)
    stats = {}
    ens = s2b.solve_iterated_magnus(s2b.MagnusConfig(order=order, dt=dt, record_times=[dt]), op,
                                    ops.datum(), paths, T, g, stats=stats)
    assert stats["engine"] == 0  # the streaming pass engine (term_var / term_varx)
    for r, e in enumerate(ens):
        assert np.array_equal(e.status, wst[r])
        assert np.array_equal(e.states(), want[r], equal_nan=True)
