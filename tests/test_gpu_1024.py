"""cfg5's grid (1024 x 1024): the streaming pass engine (a path's 8 MB term does not fit any
cluster) and the streaming E-M kernel against the reference CPU solver on identical
increments, bit for bit, for the constant and the variable-coefficient Langevin families.
Small windows keep the reference's CPU time to seconds (a full T = 1 is hours)."""
import numpy as np
import pytest

from test_gpu_parity import gpu_magnus

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("family,order,d", [("langevin-constant", 3, 1024), ("langevin-variable", 2, 1024),
                                            ("langevin-variable", 3, 512), ("langevin-variable", 3, 1024),
                                            ("langevin-variable", 2, 258)])
def test_magnus_bitwise_1024(ref, s2b, ctx, family, order, d):
    """Streaming engines at 512^2 / 1024^2: term_tma_kernel (constant), term_varx_kernel
    (variable coefficients, x-split; 258 columns leave a last part 2 columns wide)."""
    T, dt, dt_leb, M, seed = 4e-4, 2e-4, 1e-5, 3, d + order
    ops = ref.Ops(family, d, order=order)
    values, _ = ref.simulate_brownian(T, dt_leb, M, seed)
    want, wst, _ = ops.solve_magnus(values, dt_leb, T, dt, record_times=[dt], seed=seed)
    ens, _, _, stats = gpu_magnus(s2b, ctx, family, d, order, values, dt_leb, T, dt,
                                  rec=[dt], seed=seed)
    assert stats["engine"] == 0  # streaming passes
    assert len(ens) == len(want)
    for r, e in enumerate(ens):
        assert np.array_equal(e.status, wst[r])
        assert np.array_equal(e.states(), want[r], equal_nan=True)
    assert ens[-1].blowup_count() == 0


@pytest.mark.parametrize("family", ["langevin-constant", "langevin-variable"])
def test_euler_bitwise_1024(ref, s2b, ctx, family):
    d, T, dt_leb, M, seed = 1024, 6e-5, 1e-5, 2, 77
    ops = ref.Ops(family, d, order=1)
    values, _ = ref.simulate_brownian(T, dt_leb, M, seed)
    want, wst, _ = ops.solve_euler(values, dt_leb, T, dt_leb, record_times=[3e-5], seed=seed)
    g = s2b.GridSpec.square(d)
    f = s2b.Fields.from_family(g, family, ctx=ctx)
    paths = s2b.BrownianPaths.from_values(values, dt_leb, seed=seed, ctx=ctx)
    ens = s2b.solve_euler(s2b.EulerConfig(dt=dt_leb, record_times=[3e-5]), f, g, ops.datum(), paths, T)
    assert len(ens) == len(want)
    for r, e in enumerate(ens):
        assert np.array_equal(e.status, wst[r])
        assert np.array_equal(e.states(), want[r])


@pytest.mark.parametrize("d,nsteps,rec", [(34, 7, 3), (258, 9, 4), (130, 5, 2)])
def test_euler_streaming_two_step_bitwise(ref, s2b, ctx, monkeypatch, d, nsteps, rec):
    """Streaming E-M (S2B_EMXM=0): two-step passes (em_tb_kernel) between records, single steps
    (em_rows_kernel) where a record or an odd step count falls, both families."""
    monkeypatch.setenv("S2B_EMXM", "0")
    dt_leb = 1e-4
    T = nsteps * dt_leb
    for family in ("langevin-constant", "langevin-variable"):
        ops = ref.Ops(family, d, order=1)
        values, _ = ref.simulate_brownian(T, dt_leb, 3, d)
        want, wst, _ = ops.solve_euler(values, dt_leb, T, dt_leb, record_times=[rec * dt_leb], seed=d)
        g = s2b.GridSpec.square(d)
        f = s2b.Fields.from_family(g, family, ctx=ctx)
        paths = s2b.BrownianPaths.from_values(values, dt_leb, seed=d, ctx=ctx)
        ens = s2b.solve_euler(s2b.EulerConfig(dt=dt_leb, record_times=[rec * dt_leb]), f, g, ops.datum(), paths, T)
        for r, e in enumerate(ens):
            assert np.array_equal(e.status, wst[r])
            assert np.array_equal(e.states(), want[r])
