"""Kernel-level drop-in: expmv_into with an ExpmvWorkspace (sparse.hpp:106-151)
and euler_step_into with EulerStencils (euler.hpp:19-40) on the GPU, bit for bit against the
reference's CPU functions on the same inputs -- the result vector, every ExpmvReport field
(status, residual, segments, max_terms) and the returned max-abs."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def random_csr(n, density, scale, rng, diag_shift=0.0):
    m = (rng.random((n, n)) < density) * rng.normal(0.0, scale, (n, n))
    m += np.eye(n) * diag_shift
    rp = [0]
    ci, v = [], []
    for r in range(n):
        nz = np.nonzero(m[r])[0]
        ci += list(nz)
        v += list(m[r, nz])
        rp.append(len(ci))
    return np.array(rp, np.uint64), np.array(ci, np.int32), np.array(v)


def check_same(ref, s2b, csr, x, tol=1e-10, theta=1.0, ws=None):
    want, wrep = ref.expmv(*csr, x, tol, theta)
    got, grep = s2b.expmv_into(csr, x, tol, theta, ws=ws)
    status = {0: "Ok", 1: "Overflow", 2: "ToleranceNotReached"}[wrep["status"]]
    assert grep["status"] == status
    assert grep["segments"] == wrep["segments"] and grep["max_terms"] == wrep["max_terms"]
    assert np.array_equal(np.float64(grep["residual"]), np.float64(wrep["residual"])), (grep, wrep)
    assert np.array_equal(got, want, equal_nan=True)
    return grep


@pytest.mark.parametrize("n,density,scale,theta", [(12, 0.3, 0.8, 1.0), (40, 0.2, 2.0, 1.0), (300, 0.02, 5.0, 0.5),
                                                   (1000, 0.005, 1.0, 2.0)])
def test_expmv_into_random_matrices(ref, s2b, ctx, n, density, scale, theta):
    rng = np.random.default_rng(n)
    csr = random_csr(n, density, scale, rng)
    rep = check_same(ref, s2b, csr, rng.normal(size=n), theta=theta)
    assert rep["status"] == "Ok" and rep["residual"] > 0.0


def test_expmv_into_statuses(ref, s2b, ctx):
    """Overflow (sparse_scale(I, 2000), test_sparse.cpp:212-223), ToleranceNotReached (one
    segment for a large norm: 55 terms are not enough; residual = the last ratio), a zero
    matrix (norm 0: y = x, residual 0) and an empty row pattern."""
    n = 4
    eye = (np.arange(n + 1, dtype=np.uint64), np.arange(n, dtype=np.int32), np.full(n, 2000.0))
    assert check_same(ref, s2b, eye, np.ones(n))["status"] == "Overflow"
    big = (np.arange(n + 1, dtype=np.uint64), np.arange(n, dtype=np.int32), np.full(n, -60.0))
    rep = check_same(ref, s2b, big, np.ones(n), theta=1e3)
    assert rep["status"] == "ToleranceNotReached" and rep["max_terms"] == 55
    zero = (np.zeros(n + 1, np.uint64), np.zeros(0, np.int32), np.zeros(0))
    rep = check_same(ref, s2b, zero, np.arange(n, dtype=float))
    assert rep["status"] == "Ok" and rep["residual"] == 0.0 and rep["segments"] == 1


@pytest.mark.parametrize("family,d,order", [("langevin-constant", 32, 3), ("langevin-variable", 24, 2),
                                            ("langevin-constant", 128, 3)])
def test_expmv_into_magnus_logs_share_one_workspace(ref, s2b, ctx, family, d, order):
    """The MagnusLogBuilder case: one union pattern, values refilled per window; the workspace
    keeps the pattern on the device and every window is still bitwise the reference's."""
    ops = ref.Ops(family, d, order=order)
    values, _ = ref.simulate_brownian(0.3, 1e-3, 1, d)
    ws = s2b.ExpmvWorkspace(ctx)
    x = ops.datum()
    for w in range(3):
        f = ref.functionals(values[0], 100 * w, 100 * (w + 1), 1e-3)
        rp, ci, v = ops.fill(order, f)
        x_next, _ = ref.expmv(rp, ci, v, x)
        check_same(ref, s2b, (rp, ci, v), x, ws=ws)
        x = x_next


@pytest.mark.parametrize("family,d", [("langevin-constant", 20), ("langevin-variable", 17), ("custom", 14)])
def test_euler_step_into_bitwise(ref, s2b, ctx, family, d):
    """euler_step_into (euler.cpp:28-86) incl. the g^xv mixed stencil of the nine-field case."""
    from fieldsets import custom_fields
    fields = custom_fields(d) if family == "custom" else None
    fam = "fields" if family == "custom" else family
    ops = ref.Ops(fam, d, order=1, fields=fields)
    g = s2b.GridSpec.square(d)
    f = (s2b.Fields.from_arrays(g, fields, ctx=ctx) if fields is not None
         else s2b.Fields.from_family(g, family, ctx=ctx))
    rng = np.random.default_rng(d)
    u = ops.datum() * (1.0 + 0.1 * rng.normal(size=d * d))
    for dW, dt in [(0.013, 1e-3), (-0.2, 1e-2)]:
        want, wmax = ops.euler_step(u, dW, dt)
        got, gmax = s2b.euler_step(f, u, dW, dt)
        assert np.array_equal(got, want)
        assert gmax == wmax
    # the caller's stencils, not the grid's (EulerStencils is an argument of the reference)
    st = s2b.EulerStencils.from_grid(g)
    st2 = s2b.EulerStencils(st.inv2dx * 2, st.invdx2, st.inv2dv, st.invdv2 * 0.5, st.inv4dxdv)
    a, _ = s2b.euler_step(f, u, 0.01, 1e-3, st2)
    b, _ = s2b.euler_step(f, u, 0.01, 1e-3, st)
    assert not np.array_equal(a, b)


def test_euler_step_maxabs_ignores_nan_like_std_max(ref, s2b, ctx):
    d = 10
    ops = ref.Ops("langevin-constant", d, order=1)
    g = s2b.GridSpec.square(d)
    f = s2b.Fields.from_family(g, "langevin-constant", ctx=ctx)
    u = ops.datum()
    u[37] = np.nan
    want, wmax = ops.euler_step(u, 0.01, 1e-3)
    got, gmax = s2b.euler_step(f, u, 0.01, 1e-3)
    assert np.array_equal(got, want, equal_nan=True)
    assert gmax == wmax and np.isfinite(gmax)
