"""solve_adaptive_magnus on the GPU against the reference's (magnus.cpp:306-404) on identical
increments: bit-exact states and statuses, including shrink-and-retry, record boundaries,
the Lebesgue-grid floor (blow-up), and the reference's own adaptive test cases
(test_magnus.cpp:245-290)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run(ref, s2b, ctx, family, d, T, dt, dt_leb, M, seed, tol, shrink=0.5, rec=(), sigma=None, **kw):
    opts = {} if sigma is None else {"sigma": sigma}
    ops = ref.Ops(family, d, order=3, **opts)
    values, _ = ref.simulate_brownian(T, dt_leb, M, seed)
    want, wst, _ = ops.solve_magnus(values, dt_leb, T, dt, order=3, record_times=rec, seed=seed,
                                    adaptive={"tolerance": tol, "shrink": shrink}, **kw)
    g = s2b.GridSpec.square(d)
    op = s2b.Operator.from_family(g, family, order=3, ctx=ctx, **opts)
    paths = s2b.BrownianPaths.from_values(values, dt_leb, seed=seed, ctx=ctx)
    cfg = s2b.MagnusConfig(order=3, dt=dt, record_times=list(rec),
                           adaptive=s2b.AdaptiveConfig(enabled=True, tolerance=tol, shrink=shrink),
                           **{k.replace("cap", "blowup_norm_cap"): v for k, v in kw.items()})
    stats = {}
    ens = s2b.solve_adaptive_magnus(cfg, op, ops.datum(), paths, T, g, stats=stats)
    return ens, want, wst, stats, (op, ops, values, paths, g)


CASES = [
    ("langevin-constant", 16, 1e-6), ("langevin-constant", 24, 1e-9), ("langevin-variable", 20, 1e-7),
    ("langevin-constant", 64, 1e-8), ("langevin-constant", 256, 1e-9),
]


@pytest.mark.parametrize("family,d,tol", CASES)
def test_adaptive_bitwise_vs_reference(ref, s2b, ctx, family, d, tol):
    ens, want, wst, stats, _ = _run(ref, s2b, ctx, family, d, 0.2, 0.1, 1e-3, 3, 11 + d, tol, rec=[0.1])
    assert len(ens) == len(want)
    for r, e in enumerate(ens):
        assert np.array_equal(e.status, wst[r])
        assert np.array_equal(e.states(), want[r], equal_nan=True)


def test_adaptive_shrinks_and_differs_from_fixed_step(ref, s2b, ctx):
    """A tight gate makes the reference shrink windows; the GPU follows it bit for bit and the
    result is not the fixed-step one."""
    d, T, dt, dt_leb, M, seed = 16, 0.2, 0.1, 1e-3, 2, 5
    ens, want, wst, stats, (op, ops, values, paths, g) = _run(ref, s2b, ctx, "langevin-constant", d, T, dt,
                                                               dt_leb, M, seed, 1e-10, shrink=0.3)
    assert np.array_equal(ens[-1].states(), want[-1], equal_nan=True)
    fixed, _, _ = ops.solve_magnus(values, dt_leb, T, dt, order=3, seed=seed)
    assert not np.array_equal(fixed[-1], want[-1])


def test_adaptive_infinite_tolerance_is_fixed_order3(ref, s2b, ctx):
    """test_magnus.cpp:245-264: the gate never fires -> exactly the fixed-step order-3 solve."""
    d, T, dt, dt_leb, M, seed = 12, 0.3, 0.1, 1e-3, 3, 21
    ens, want, wst, _, (op, ops, values, paths, g) = _run(ref, s2b, ctx, "langevin-constant", d, T, dt,
                                                          dt_leb, M, seed, float("inf"))
    plain = s2b.solve_iterated_magnus(s2b.MagnusConfig(order=3, dt=dt), op, ops.datum(), paths, T, g)
    assert np.array_equal(ens[-1].states(), plain[-1].states())
    assert np.array_equal(ens[-1].states(), want[-1])


def test_adaptive_deterministic_never_shrinks(ref, s2b, ctx):
    """test_magnus.cpp:266-290: sigma = 0 (A = 0) -> orders 2 and 3 coincide; no shrinking."""
    d, T, dt, dt_leb, M, seed = 12, 0.2, 0.1, 1e-3, 2, 4
    ens, want, wst, _, (op, ops, values, paths, g) = _run(ref, s2b, ctx, "langevin-constant", d, T, dt,
                                                          dt_leb, M, seed, 1e-9, sigma=0.0)
    assert np.array_equal(ens[-1].states(), want[-1])
    assert np.array_equal(ens[-1].status, wst[-1]) and ens[-1].blowup_count() == 0


def test_adaptive_lebesgue_floor_blows_up(ref, s2b, ctx):
    """An unreachable gate shrinks below one Lebesgue step: BlownUp, like the reference."""
    ens, want, wst, _, _ = _run(ref, s2b, ctx, "langevin-constant", 10, 0.02, 0.01, 1e-3, 2, 8, 1e-300,
                                rec=[0.01])
    for r in range(len(ens)):
        assert np.array_equal(ens[r].status, wst[r])
    assert ens[-1].blowup_count() == 2


def test_adaptive_norm_cap(ref, s2b, ctx):
    ens, want, wst, _, _ = _run(ref, s2b, ctx, "langevin-constant", 10, 0.2, 0.1, 1e-3, 2, 8, 1e-6, cap=1e-6)
    assert np.array_equal(ens[-1].status, wst[-1]) and ens[-1].blowup_count() == 2


def test_adaptive_config_errors(s2b, ctx):
    d = 8
    g = s2b.GridSpec.square(d)
    op3 = s2b.Operator.from_family(g, order=3, ctx=ctx)
    op2 = s2b.Operator.from_family(g, order=2, ctx=ctx)
    paths = s2b.BrownianPaths.philox(0.2, 1e-3, 2, seed=1, ctx=ctx)
    phi = s2b.gaussian_datum(g)
    with pytest.raises(s2b.ConfigError, match="adaptive flag"):
        s2b.solve_adaptive_magnus(s2b.MagnusConfig(dt=0.1), op3, phi, paths, 0.2, g)
    with pytest.raises(s2b.ConfigError, match="shrink"):
        s2b.solve_adaptive_magnus(s2b.MagnusConfig(dt=0.1, adaptive=s2b.AdaptiveConfig(True, 1e-4, 1.0)),
                                  op3, phi, paths, 0.2, g)
    with pytest.raises(s2b.ConfigError, match="order-3"):
        s2b.solve_adaptive_magnus(s2b.MagnusConfig(order=2, dt=0.1, adaptive=s2b.AdaptiveConfig(True)),
                                  op2, phi, paths, 0.2, g)
