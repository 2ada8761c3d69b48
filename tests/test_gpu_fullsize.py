"""Cross-engine parity at the benchmark sizes.  The reference CPU solver needs hours for one
BASELINE-size run, so at full size the check is a size-independent property:
engines with different decompositions -- cluster-resident x-march (+ its streaming slice),
in-place cluster, streaming x-march with two Taylor terms per pass, row-march streaming -- each
pinned to the reference bit for bit at smaller sizes, must agree bit for bit with one another on
the same increments at the bench grids and path counts."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run(s2b, ctx, d, M, dt, dt_leb, windows, seed=2024):
    g = s2b.GridSpec.square(d)
    op = s2b.Operator.from_family(g, "langevin-constant", order=3, ctx=ctx)
    T = windows * dt
    paths = s2b.BrownianPaths.philox(T, dt_leb, M, seed=seed, ctx=ctx)
    stats = {}
    ens = s2b.solve_iterated_magnus(s2b.MagnusConfig(order=3, dt=dt, record_times=[dt]), op,
                                    s2b.gaussian_datum(g), paths, T, g, stats=stats)
    out = [(e.status.copy(), e.states().copy()) for e in ens]
    del ens, paths, op
    return out, stats


def _same(a, b):
    assert len(a) == len(b)
    for (sa, xa), (sb, xb) in zip(a, b):
        assert np.array_equal(sa, sb)
        assert np.array_equal(xa.view(np.uint64), xb.view(np.uint64))


def test_cfg5_grid_two_term_xmarch_equals_row_march(s2b, ctx, monkeypatch):
    """1024^2 (cfg5's grid and steps), 256 paths, 2 windows: term_xs2_kernel vs term_tma_kernel."""
    want, st0 = _run(s2b, ctx, 1024, 256, 5e-4, 1e-5, 2)
    monkeypatch.setenv("S2B_XS", "0")
    got, st1 = _run(s2b, ctx, 1024, 256, 5e-4, 1e-5, 2)
    _same(want, got)
    assert st0["path_terms"] == st1["path_terms"] > 0


def test_cfg2_grid_cluster_hybrid_equals_streaming(s2b, ctx, monkeypatch):
    """256^2 (cfg2's grid, dt, dt_leb), 4096 paths, 3 windows: the default cluster x-march with
    its x-march slice on the idle SMs vs the pure cluster engine vs the streaming x-march engine
    (two terms per pass)."""
    want, st = _run(s2b, ctx, 256, 4096, 0.01, 1e-4, 3)
    assert st["hybrid_paths"] > 0
    monkeypatch.setenv("S2B_HYBRID", "0")
    _same(want, _run(s2b, ctx, 256, 4096, 0.01, 1e-4, 3)[0])
    monkeypatch.delenv("S2B_HYBRID")
    monkeypatch.setenv("S2B_ENGINE", "stream")
    _same(want, _run(s2b, ctx, 256, 4096, 0.01, 1e-4, 3)[0])


def test_cfg4_grid_inplace_cluster_equals_streaming(s2b, ctx, monkeypatch):
    """512^2 (cfg4's grid, dt, dt_leb), 1024 paths, 2 windows: in-place cluster engine with its
    x-march slice vs the streaming x-march engine."""
    want, st = _run(s2b, ctx, 512, 1024, 0.005, 1e-4, 2)
    assert st["engine"] == 3 and st["hybrid_paths"] > 0
    monkeypatch.setenv("S2B_ENGINE", "stream")
    _same(want, _run(s2b, ctx, 512, 1024, 0.005, 1e-4, 2)[0])
