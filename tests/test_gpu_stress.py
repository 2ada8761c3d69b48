"""Race / synchronisation stress in place of compute-sanitizer (closed on this GPU pool, see
profiles/r02_sanitizer.txt): every synchronisation-heavy kernel -- DSMEM halo pushes and
cluster barriers (cluster_xm, cluster_xmi, cluster_magnus, em_cluster), TMA rings with
mbarrier phases (term_tma, term_xs, term_var, term_varx, em_tb) -- is run with its persistent grid capped
at 1, 2, 3 and 5 CTAs / clusters (S2B_GRID_CAP) and at full size, several times.  Different
grids change which work items share an SM, how long every CTA runs and how its mbarrier
phases wrap across items; a race or a missed wait shows up as a bit difference between runs.
Every run must be bitwise the full-grid run."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CAPS = ["1", "2", "3", "5", ""]


def _magnus(s2b, ctx, d, family="langevin-constant", order=3, M=3, dt=0.002, fields=None):
    g = s2b.GridSpec.square(d)
    op = s2b.Operator.from_family(g, family, order=order, fields=fields, ctx=ctx)
    paths = s2b.BrownianPaths.philox(2 * dt, 1e-4, M, seed=5, ctx=ctx)
    ens = s2b.solve_iterated_magnus(s2b.MagnusConfig(order=order, dt=dt, record_times=[dt]), op,
                                    s2b.gaussian_datum(g), paths, 2 * dt, g)
    return [e.states() for e in ens]


def _euler(s2b, ctx, d, family="langevin-constant", M=3, steps=6):
    g = s2b.GridSpec.square(d)
    f = s2b.Fields.from_family(g, family, ctx=ctx)
    paths = s2b.BrownianPaths.philox(steps * 1e-5, 1e-5, M, seed=5, ctx=ctx)
    ens = s2b.solve_euler(s2b.EulerConfig(dt=1e-5, record_times=[3e-5]), f, g, s2b.gaussian_datum(g), paths,
                          steps * 1e-5)
    return [e.states() for e in ens]


CASES = {
    "cluster_xm-64": (lambda s, c: _magnus(s, c, 64, M=7), {}),
    "cluster_xm-128": (lambda s, c: _magnus(s, c, 128, M=5), {}),
    "cluster_xm-256": (lambda s, c: _magnus(s, c, 256, M=3), {}),
    "cluster_xmi-512": (lambda s, c: _magnus(s, c, 512, M=2, dt=0.0005), {}),
    "cluster_band-256": (lambda s, c: _magnus(s, c, 256, M=3, order=2), {"S2B_XM": "0"}),
    "term_tma-256": (lambda s, c: _magnus(s, c, 256, M=3), {"S2B_ENGINE": "stream", "S2B_XS": "0"}),
    "term_xs-256": (lambda s, c: _magnus(s, c, 256, M=3), {"S2B_ENGINE": "stream", "S2B_XS2": "0"}),
    "term_xs-512": (lambda s, c: _magnus(s, c, 512, M=2), {"S2B_ENGINE": "stream", "S2B_XS2": "0"}),
    "term_tma-1024": (lambda s, c: _magnus(s, c, 1024, M=2, dt=0.0002), {"S2B_XS": "0"}),
    "term_xs-1024": (lambda s, c: _magnus(s, c, 1024, M=2, dt=0.0002), {"S2B_XS2": "0"}),
    "term_xs2-256": (lambda s, c: _magnus(s, c, 256, M=3), {"S2B_ENGINE": "stream", "S2B_XS2H": "0"}),
    "term_xs2-1024": (lambda s, c: _magnus(s, c, 1024, M=2, dt=0.0002), {"S2B_XS2H": "0"}),
    "term_xs2h-256": (lambda s, c: _magnus(s, c, 256, M=3), {"S2B_ENGINE": "stream"}),
    "term_xs2h-1024": (lambda s, c: _magnus(s, c, 1024, M=2, dt=0.0002), {}),
    "term2-256": (lambda s, c: _magnus(s, c, 256, M=3), {"S2B_ENGINE": "stream", "S2B_TERM2": "1"}),
    "term_var-256": (lambda s, c: _magnus(s, c, 256, "langevin-variable", M=5, dt=0.001), {}),
    "em_cluster_ip-64": (lambda s, c: _euler(s, c, 64, M=7), {}),
    "em_cluster_ip-256": (lambda s, c: _euler(s, c, 256, M=4), {}),
    "em_cluster_ip-512": (lambda s, c: _euler(s, c, 512, M=2), {}),
    "em_tb-96": (lambda s, c: _euler(s, c, 96, "langevin-variable", M=3), {}),
}


@pytest.mark.parametrize("case", sorted(CASES))
def test_grid_caps_do_not_change_a_bit(s2b, ctx, monkeypatch, case):
    run, env = CASES[case]
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    monkeypatch.delenv("S2B_GRID_CAP", raising=False)
    want = run(s2b, ctx)
    for cap in CAPS:
        if cap:
            monkeypatch.setenv("S2B_GRID_CAP", cap)
        else:
            monkeypatch.delenv("S2B_GRID_CAP", raising=False)
        got = run(s2b, ctx)
        for a, b in zip(got, want):
            assert np.array_equal(a.view(np.uint64), b.view(np.uint64)), f"{case}: grid cap {cap or 'none'}"


def test_kinetic_term_varx_grid_caps(s2b, ctx, monkeypatch):
    import sys, os
    sys.path.insert(0, os.path.dirname(__file__))
    from fieldsets import kinetic_fields
    f = kinetic_fields(256)
    want = _magnus(s2b, ctx, 256, "fields", M=5, dt=0.0005, fields=f)
    for cap in ("1", "3"):
        monkeypatch.setenv("S2B_GRID_CAP", cap)
        got = _magnus(s2b, ctx, 256, "fields", M=5, dt=0.0005, fields=f)
        for a, b in zip(got, want):
            assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
