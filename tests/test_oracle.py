"""Pin the CPU oracle (oracle/restate.c) before trusting it: bitwise against the compiled
reference (oracle/_ref) and against the committed golden fixtures (tests/golden/), plus the
known-answer tests the reference's own suite holds for this path."""
import glob
import os

import numpy as np
import pytest

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))


def load(path):
    z = np.load(path, allow_pickle=False)
    return {k: z[k] for k in z.files}


def csr_sources(g):
    out = []
    for slot in ("B", "A", "A2", "BA", "BAA", "BAB"):
        k = f"csr_{slot}_rp"
        out.append((g[k], g[f"csr_{slot}_ci"], g[f"csr_{slot}_v"]) if k in g else None)
    return out


def fields9(g, ref_like=None):
    names = ("h", "fx", "fv", "gxx", "gxv", "gvv", "sig", "sigx", "sigv")
    return [g.get(f"field_{n}") for n in names]


# ---------------------------------------------------------------- golden fixtures
@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p) for p in GOLDEN])
def test_restatement_reproduces_golden_magnus(rs, path):
    g = load(path)
    d, order, M = int(g["d"]), int(g["order"]), int(g["M"])
    dt_leb, dt, T = float(g["dt_leb"]), float(g["dt"]), float(g["T"])
    srcs = csr_sources(g)
    dt_steps = int(round(dt / dt_leb))
    total = int(round(T / dt_leb))
    rec = [int(round(t / dt_leb)) for t in g["record_times"]] + [total]
    rec = sorted(set(rec))
    for m in range(M):
        states, status, _, _ = rs.magnus_path(d * d, order, srcs, g["phi"], g["values"][m],
                                              dt_leb, dt_steps, total, rec)
        assert np.array_equal(status, g["magnus_status"][:, m])
        assert np.array_equal(states, g["magnus"][:, m], equal_nan=True)


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p) for p in GOLDEN])
def test_restatement_reproduces_golden_trace(rs, path):
    g = load(path)
    d, order = int(g["d"]), int(g["order"])
    dt_steps = int(round(float(g["dt"]) / float(g["dt_leb"])))
    f5 = rs.functionals(g["values"][0], 0, dt_steps, float(g["dt_leb"]))
    assert np.array_equal(f5, g["trace_f5"])
    c = rs.log_coefficients(order, f5)
    rp, ci, v = rs.union_fill(d * d, order, order, csr_sources(g), c)
    assert len(v) == int(g["trace_nnz"])
    assert rs.one_norm(rp, ci, v) == float(g["trace_norm"])
    y, rep = rs.expmv(rp, ci, v, g["phi"])
    assert np.array_equal(y, g["trace_y"])
    assert rep["segments"] == int(g["trace_segments"])
    assert rep["max_terms"] == int(g["trace_max_terms"])


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p) for p in GOLDEN])
def test_restatement_reproduces_golden_euler(rs, path):
    g = load(path)
    d, M = int(g["d"]), int(g["M"])
    dt_leb, T, em_dt = float(g["dt_leb"]), float(g["T"]), float(g["em_dt"])
    f9 = fields9(g)
    h = 8.0 / (d + 1)
    st = rs.stencils(h, h)
    step = int(round(em_dt / dt_leb))
    total = int(round(T / dt_leb))
    rec = sorted(set([int(round(t / dt_leb)) for t in g["record_times"]] + [total]))
    for m in range(M):
        states, status = rs.euler_path(d, d, f9, st, g["phi"], g["values"][m], step, total,
                                       em_dt, rec)
        assert np.array_equal(status, g["euler_status"][:, m])
        assert np.array_equal(states, g["euler"][:, m], equal_nan=True)


def test_restatement_reproduces_golden_exact_and_norms(rs):
    g = load(os.path.join(os.path.dirname(__file__), "golden", "cfg1_const64_o2.npz"))
    d, M, T, dt_leb = int(g["d"]), int(g["M"]), float(g["T"]), float(g["dt_leb"])
    h = 8.0 / (d + 1)
    nodes = np.array([-4.0 + float(i + 1) * h for i in range(d)])
    total = int(round(T / dt_leb))
    for m in range(M):
        f5 = rs.functionals(g["values"][m], 0, total, dt_leb)
        ex = rs.exact_field(nodes, nodes, T, 1.1, 0.31622776601683794, f5[1], f5[2])
        assert np.array_equal(ex, g["exact"][m])
    for kappa in (0, 2):
        e = rs.errors(d, kappa, g["exact"], g["magnus"][-1], app_status=g["magnus_status"][-1])
        want = g[f"err_k{kappa}"]
        assert e["err"] == want[0] and e["ame"] == want[1]
        assert np.array_equal(e["me"], g[f"me_k{kappa}"])


# ---------------------------------------------------------------- against oracle/_ref
@pytest.mark.parametrize("family,d,order", [("langevin-constant", 10, 3), ("langevin-variable", 12, 2),
                                            ("langevin-constant", 7, 1)])
def test_restatement_bitwise_vs_reference_magnus(ref, rs, family, d, order):
    ops = ref.Ops(family, d, order=order)
    values, _ = ref.simulate_brownian(0.3, 1e-3, 3, 11)
    states, status, _ = ops.solve_magnus(values, 1e-3, 0.3, 0.1, record_times=[0.1, 0.2], seed=11)
    srcs = [ops.csr(s) for s in ref.SLOTS]
    for m in range(3):
        got, st, _, _ = rs.magnus_path(d * d, order, srcs, ops.datum(), values[m], 1e-3, 100, 300,
                                       [100, 200, 300])
        assert np.array_equal(st, status[:, m])
        assert np.array_equal(got, states[:, m], equal_nan=True)


def test_restatement_bitwise_vs_reference_pieces(ref, rs):
    v1, i1 = ref.simulate_brownian(0.5, 1e-3, 5, 77)
    v2, i2 = rs.simulate_brownian(0.5, 1e-3, 5, 77)
    assert np.array_equal(v1, v2) and np.array_equal(i1, i2)
    assert np.array_equal(ref.functionals(v1[2], 100, 350, 1e-3), rs.functionals(v1[2], 100, 350, 1e-3))
    ops = ref.Ops("langevin-variable", 14, order=3)
    f5 = ref.functionals(v1[0], 0, 200, 1e-3)
    for order in (1, 2, 3):
        rp, ci, v = ops.fill(order, f5)
        rp2, ci2, v2_ = rs.union_fill(14 * 14, 3, order, [ops.csr(s) for s in ref.SLOTS],
                                      rs.log_coefficients(order, f5))
        assert np.array_equal(rp, rp2) and np.array_equal(ci, ci2) and np.array_equal(v, v2_)
        assert ref.one_norm(rp, ci, v) == rs.one_norm(rp, ci, v)
        y, rep = ref.expmv(rp, ci, v, ops.datum())
        y2, rep2 = rs.expmv(rp, ci, v, ops.datum())
        assert np.array_equal(y, y2)
        assert (rep["segments"], rep["max_terms"], rep["status"]) == (rep2["segments"], rep2["max_terms"], rep2["status"])


def test_restatement_bitwise_vs_reference_euler(ref, rs):
    for family in ("langevin-constant", "langevin-variable"):
        ops = ref.Ops(family, 11, order=1)
        values, _ = ref.simulate_brownian(0.05, 1e-3, 2, 3)
        states, status, _ = ops.solve_euler(values, 1e-3, 0.05, 1e-3, record_times=[0.02])
        f9 = [None if ops.field(n)[1] else ops.field(n)[0] for n in ref.FIELD_NAMES]
        h = 8.0 / 12
        for m in range(2):
            got, st = rs.euler_path(11, 11, f9, rs.stencils(h, h), ops.datum(), values[m], 1, 50,
                                    1e-3, [20, 50])
            assert np.array_equal(st, status[:, m])
            assert np.array_equal(got, states[:, m])


def test_restatement_exact_and_norms_vs_reference(ref, rs):
    ops = ref.Ops("langevin-constant", 18, order=1)
    values, _ = ref.simulate_brownian(0.4, 1e-3, 4, 44)
    ex = ops.exact_reference(values, 1e-3, 0.4, seed=44)
    nodes = ops.nodes(0)
    for m in range(4):
        f5 = rs.functionals(values[m], 0, 400, 1e-3)
        assert np.array_equal(rs.exact_field(nodes, nodes, 0.4, 1.1, 1 / np.sqrt(10.0), f5[1], f5[2]), ex[m])
    app = ex * (1.0 + 1e-3 * np.arange(4)[:, None])
    status = np.array([0, 1, 0, 0], np.uint8)
    for kappa in (0, 1, 3):
        a = ref.Ops("langevin-constant", 18, order=1).errors(kappa, ex, app, app_status=status, seed=44)
        b = rs.errors(18, kappa, ex, app, app_status=status)
        assert a["err"] == b["err"] == np.inf and a["blowups"] == b["blowups"] == 1
        assert a["ame"] == b["ame"] and np.array_equal(a["me"], b["me"])


# ---------------------------------------------------------------- reference known answers
def test_known_answer_ramp_functionals(rs):
    """test_stochastics.cpp:237-249: the injected ramp path."""
    dt, n = 1e-4, 10000
    ramp = np.arange(n + 1) * dt
    f = rs.functionals(ramp, 0, n, dt)
    assert abs(f[0] - 1.0) < 1e-12 and abs(f[1] - 1.0) < 1e-12
    assert abs(f[2] - 0.5) <= 1e-4 and abs(f[3] - 1 / 3) <= 1e-3 and abs(f[4] - 1 / 3) <= 1e-3


def test_known_answer_central_region(rs):
    """test_analysis.cpp:27-39."""
    assert rs.central_region(300, 4) == (139, 158)
    assert rs.central_region(4, 0) == (0, 3)
    with pytest.raises(ValueError):
        rs.central_region(2, 3)


def test_known_answer_diagonal_counts(ref):
    """Paper Figure 1 / test_operators.cpp:127-156: 2, 5, 5, 8, 10 diagonals for A, B, [B,A],
    [[B,A],A], [[B,A],B], independent of d."""
    for d in (10, 50):
        ops = ref.Ops("langevin-constant", d, order=3)
        assert [ops.diagonals(s) for s in ("A", "B", "BA", "BAA", "BAB")] == [2, 5, 5, 8, 10]


def test_known_answer_scalar_gbm(rs):
    """test_magnus.cpp:55-73: for 1x1 operators the logarithm is b h + a W - a^2 h / 2."""
    rng = np.random.default_rng(42)
    for rep in range(10):
        a, b = rng.uniform(-2, 2, 2)
        one = (np.array([0, 1], np.uint64), np.array([0], np.int32))
        srcs = [(*one, np.array([b])), (*one, np.array([a])), (*one, np.array([a * a])),
                None, None, None]
        values, _ = rs.simulate_brownian(1.0, 1e-2, 1, 900 + rep)
        f = rs.functionals(values[0], 0, 100, 1e-2)
        c = rs.log_coefficients(2, f)
        rp, ci, v = rs.union_fill(1, 2, 2, srcs, c)
        expected = b * f[0] + a * f[1] - 0.5 * a * a * f[0]
        assert abs(v[0] - expected) <= 1e-14 * max(1.0, abs(expected))


def test_known_answer_expmv_overflow(rs):
    """test_sparse.cpp:212-222: 2000*I overflows the segmented series."""
    rp = np.arange(5, dtype=np.uint64)
    ci = np.arange(4, dtype=np.int32)
    _, rep = rs.expmv(rp, ci, np.full(4, 2000.0), np.ones(4))
    assert rep["status"] == 1
