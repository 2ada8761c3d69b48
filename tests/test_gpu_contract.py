"""Session / API contract on the GPU: lifetimes, use-after-finish, the zero-norm window cap
rule of solve_iterated_magnus (magnus.cpp:277-286) and engine-independent adaptive counters."""
import gc

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _setup(s2b, ctx, d=16, M=3, T=0.2, dt_leb=1e-3, seed=3):
    g = s2b.GridSpec.square(d)
    values = s2b.simulate_brownian(T, dt_leb, M, seed)
    paths = s2b.BrownianPaths.from_values(values, dt_leb, seed=seed, ctx=ctx)
    return g, values, paths


def test_finish_twice_and_use_after_finish_are_refused(s2b, ctx):
    g, _, paths = _setup(s2b, ctx)
    op = s2b.Operator.from_family(g, "langevin-constant", order=3, ctx=ctx)
    sess = s2b.MagnusSession(s2b.MagnusConfig(order=3, dt=0.1), op, s2b.gaussian_datum(g), paths, 0.2)
    sess.advance(1)
    ens = sess.finish()
    want = ens[-1].states()
    for call in (sess.finish, sess.reset, lambda: sess.advance(1), sess.snapshot, sess.moments, sess.stats):
        with pytest.raises(s2b.ConfigError):
            call()
    # the context is not poisoned and the ensemble the first finish returned is intact
    assert np.array_equal(ens[-1].states(), want)
    again = s2b.solve_iterated_magnus(s2b.MagnusConfig(order=3, dt=0.1), op, s2b.gaussian_datum(g), paths, 0.2, g)
    assert np.array_equal(again[-1].states(), want)


def test_session_keeps_its_operator_alive(s2b, ctx):
    """MagnusSession(cfg, Operator.from_family(...), ...) with no other reference to the operator."""
    g, _, paths = _setup(s2b, ctx)
    phi = s2b.gaussian_datum(g)
    cfg = s2b.MagnusConfig(order=3, dt=0.1)
    sess = s2b.MagnusSession(cfg, s2b.Operator.from_family(g, "langevin-constant", order=3, ctx=ctx),
                             phi, paths, 0.2)
    gc.collect()
    sess.advance(2)
    got = sess.finish()[-1].states()
    op = s2b.Operator.from_family(g, "langevin-constant", order=3, ctx=ctx)
    want = s2b.solve_iterated_magnus(cfg, op, phi, paths, 0.2, g)[-1].states()
    assert np.array_equal(got, want)


@pytest.mark.parametrize("cap,phi_scale", [(100.0, 1e3), (1e4, 1e3), (0.5, 1.0)])
def test_zero_norm_windows_apply_the_cap_like_the_reference(ref, s2b, ctx, cap, phi_scale):
    """All-zero operator: every window has norm 0; the reference still blows up a path whose
    datum exceeds the cap after the first window (magnus.cpp:282-286)."""
    d, T, dt_leb, dt, M = 12, 0.2, 1e-3, 0.1, 3
    ops = ref.Ops("fields", d, order=3, fields={})
    values, _ = ref.simulate_brownian(T, dt_leb, M, 5)
    phi = ops.datum() * phi_scale
    want, wst, _ = ops.solve_magnus(values, dt_leb, T, dt, record_times=[0.1], cap=cap, phi=phi)
    g = s2b.GridSpec.square(d)
    op = s2b.Operator.from_csr(g, 3, [ops.csr(s) for s in ref.SLOTS], ctx=ctx)
    paths = s2b.BrownianPaths.from_values(values, dt_leb, seed=5, ctx=ctx)
    ens = s2b.solve_iterated_magnus(s2b.MagnusConfig(order=3, dt=dt, record_times=[0.1], blowup_norm_cap=cap),
                                    op, phi, paths, T, g)
    for r, e in enumerate(ens):
        assert np.array_equal(e.status, wst[r])
        ok = wst[r] == 0
        assert np.array_equal(e.states()[ok], want[r][ok])


def test_datum_above_cap_with_real_first_window(ref, s2b, ctx):
    """max|phi| > cap but window 0 has a non-zero Y: the cap is checked on the window's result."""
    d, T, dt_leb, dt, M = 16, 0.2, 1e-3, 0.1, 3
    ops = ref.Ops("langevin-constant", d, order=3)
    values, _ = ref.simulate_brownian(T, dt_leb, M, 9)
    phi = ops.datum() * 50.0
    want, wst, _ = ops.solve_magnus(values, dt_leb, T, dt, record_times=[0.1], cap=30.0, phi=phi)
    g = s2b.GridSpec.square(d)
    op = s2b.Operator.from_family(g, "langevin-constant", order=3, ctx=ctx)
    paths = s2b.BrownianPaths.from_values(values, dt_leb, seed=9, ctx=ctx)
    ens = s2b.solve_iterated_magnus(s2b.MagnusConfig(order=3, dt=dt, record_times=[0.1], blowup_norm_cap=30.0),
                                    op, phi, paths, T, g)
    for r, e in enumerate(ens):
        assert np.array_equal(e.status, wst[r])
        assert np.array_equal(e.states(), want[r], equal_nan=True)


def test_adaptive_counters_do_not_depend_on_the_engine(s2b, ctx, monkeypatch):
    """The streaming engine used to zero the counters every attempt round; now both engines
    accumulate the Taylor terms of every order-3 and order-2 attempt."""
    g, _, paths = _setup(s2b, ctx, d=64, M=4, T=0.2, seed=17)
    op = s2b.Operator.from_family(g, "langevin-constant", order=3, ctx=ctx)
    cfg = s2b.MagnusConfig(order=3, dt=0.1, adaptive=s2b.AdaptiveConfig(enabled=True, tolerance=1e-6))
    phi = s2b.gaussian_datum(g)
    st_cl, st_sm = {}, {}
    a = s2b.solve_adaptive_magnus(cfg, op, phi, paths, 0.2, g, stats=st_cl)[-1].states()
    monkeypatch.setenv("S2B_ENGINE", "stream")
    b = s2b.solve_adaptive_magnus(cfg, op, phi, paths, 0.2, g, stats=st_sm)[-1].states()
    assert np.array_equal(a, b, equal_nan=True)
    assert st_sm["engine"] == 0 and st_cl["engine"] != 0
    assert st_cl["path_terms"] == st_sm["path_terms"] > 0
    assert st_cl["path_segments"] == st_sm["path_segments"] > 0
