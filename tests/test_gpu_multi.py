"""Multi-GPU product API (s2b_multi_*) on the one B200 of the test box:
a one-device NCCL clique, and a device listed twice (two path shards on their own contexts
and host threads, host combine).  Either way the combined Err and the per-path errors are
bitwise the single-context values (Philox keyed by the global path id, Err summed in global
path order); moments agree to rounding (sums split across shards)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

A, SIGMA = 1.1, 1.0 / np.sqrt(10.0)


def single(s2b, ctx, scheme, d, M, T, dt_leb, dt, seed, kappa, order=3):
    g = s2b.GridSpec.square(d)
    phi = s2b.gaussian_datum(g)
    paths = s2b.BrownianPaths.philox(T, dt_leb, M, seed=seed, ctx=ctx)
    if scheme == "magnus":
        op = s2b.Operator.from_family(g, "langevin-constant", order=order, ctx=ctx)
        ens = s2b.solve_iterated_magnus(s2b.MagnusConfig(order=order, dt=dt), op, phi, paths, T, g)
    else:
        f = s2b.Fields.from_family(g, "langevin-constant", ctx=ctx)
        ens = s2b.solve_euler(s2b.EulerConfig(dt=dt), f, g, phi, paths, T)
    return g, phi, s2b.exact_errors(ens[-1], A, SIGMA, paths, kappa, moments=True, per_path=True)


@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 0, 0]])
@pytest.mark.parametrize("scheme", ["magnus", "euler"])
def test_multi_matches_single_context(s2b, ctx, devices, scheme):
    d, M, T, dt_leb, seed, kappa = 64, 11, 0.2, 1e-3, 23, 1
    dt = 0.1 if scheme == "magnus" else dt_leb
    g, phi, want = single(s2b, ctx, scheme, d, M, T, dt_leb, dt, seed, kappa)
    mg = s2b.MultiGPU(devices)
    assert mg.nccl == (len(set(devices)) == len(devices))
    if scheme == "magnus":
        got = mg.solve_magnus(s2b.MagnusConfig(order=3, dt=dt), g, phi, T, dt_leb, M, seed=seed, kappa=kappa,
                              a=A, sigma=SIGMA)
    else:
        got = mg.solve_euler(s2b.EulerConfig(dt=dt), g, phi, T, dt_leb, M, seed=seed, kappa=kappa, a=A, sigma=SIGMA)
    assert got["devices"] == len(devices) and got["M_total"] == M
    assert np.array_equal(got["per_path_rel"], want["per_path_rel"], equal_nan=True)
    assert got["err"] == want["err"] and got["blowups"] == want["blowups"] and got["used"] == want["used"]
    assert np.allclose(got["me"], want["me"], rtol=1e-13, atol=0)
    assert np.allclose(got["sum_u"], want["sum_u"], rtol=1e-13, atol=1e-300)
    assert np.allclose(got["sum_u2"], want["sum_u2"], rtol=1e-13, atol=1e-300)
    if len(devices) == 1:  # one shard: the moments are the device's own sums (ME is rescaled by used)
        assert np.array_equal(got["sum_u"], want["sum_u"]) and np.array_equal(got["sum_u2"], want["sum_u2"])
    assert got["max_solve_ms"] > 0


def test_multi_moments_only_and_counters(s2b, ctx):
    """kappa < 0 (any family): moments + counts; the Taylor-term counters add up over shards."""
    d, M, T, dt_leb, seed = 32, 5, 0.2, 1e-3, 3
    g = s2b.GridSpec.square(d)
    phi = s2b.gaussian_datum(g)
    paths = s2b.BrownianPaths.philox(T, dt_leb, M, seed=seed, ctx=ctx)
    op = s2b.Operator.from_family(g, "langevin-variable", order=2, ctx=ctx)
    stats = {}
    ens = s2b.solve_iterated_magnus(s2b.MagnusConfig(order=2, dt=0.1), op, phi, paths, T, g, stats=stats)
    s1, s2, live = ens[-1].moments()
    got = s2b.MultiGPU([0, 0]).solve_magnus(s2b.MagnusConfig(order=2, dt=0.1), g, phi, T, dt_leb, M, seed=seed,
                                            family="langevin-variable")
    assert got["path_terms"] == stats["path_terms"] and got["used"] == live
    assert np.allclose(got["sum_u"], s1, rtol=1e-13) and np.allclose(got["sum_u2"], s2, rtol=1e-13)
