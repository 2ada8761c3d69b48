"""Engine coverage at the benchmark grid (256 x 256): every Magnus engine — the x-march
cluster kernel (default for constant Langevin), the row-band cluster kernel (S2B_XM=0) and
the streaming pass engine (S2B_ENGINE=stream) — against the reference CPU solver on
identical increments, bit for bit, including the blow-up exits (norm cap, non-finite
terms, exhausted Taylor budget) and record snapshots."""
import os

import numpy as np
import pytest

from test_gpu_parity import gpu_magnus

pytestmark = pytest.mark.gpu

ENGINES = {"xm": {}, "band": {"S2B_XM": "0"}, "stream": {"S2B_ENGINE": "stream"}}


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


@pytest.mark.parametrize("engine", ["xm", "band"], indirect=True)
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
