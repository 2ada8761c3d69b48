"""Device-side operator assembly: the CommutatorSet computed on the GPU
(assemble.cu) equals the host builder's CSR -- and through it the reference's -- byte for byte
(row_ptr, col_idx, values of B, A, A2, [B,A], [[B,A],A], [[B,A],B]), for the Langevin families,
the general kinetic fields and all nine fields; and a solve on the device-built operator is
bitwise the host-built one."""
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _same(a, b):
    if a is None or b is None:
        return a is None and b is None
    return all(np.array_equal(x.view(np.uint8), y.view(np.uint8)) for x, y in zip(a, b))


@pytest.mark.parametrize("family,d,nv,order", [("langevin-constant", 16, 16, 3), ("langevin-variable", 33, 33, 3),
                                               ("langevin-constant", 64, 40, 2), ("kinetic", 48, 48, 3),
                                               ("custom", 20, 26, 3), ("custom", 12, 12, 1),
                                               ("langevin-variable", 256, 256, 3)])
def test_device_commutators_equal_host_csr(s2b, ctx, family, d, nv, order):
    from fieldsets import custom_fields, kinetic_fields
    g = s2b.GridSpec(d, nv)
    fields = None
    fam = family
    if family in ("kinetic", "custom"):
        fam = "fields"
        f = kinetic_fields(max(d, nv)) if family == "kinetic" else custom_fields(max(d, nv))
        # resample on the (possibly rectangular) grid's nodes
        x, v = g.nodes(0), g.nodes(1)
        X, V = np.meshgrid(x, v, indexing="xy")
        fields = {k: np.ascontiguousarray((np.cos(0.3 * X * (q + 1)) + 0.2 * np.sin(V * (q + 2)) + 0.05 * q).reshape(-1))
                  for q, k in enumerate(f)}
        if family == "kinetic":
            fields["fx"] = np.ascontiguousarray(-V.reshape(-1))
    host = s2b.HostOps(g, fam, order=order, fields=fields)
    dev = s2b.HostOps(g, fam, order=order, fields=fields, device=ctx)
    for slot in s2b.SLOTS:
        assert _same(host.csr(slot), dev.csr(slot)), slot


def test_device_built_operator_solves_bitwise(s2b, ctx):
    d, T, dt_leb, M = 64, 0.2, 1e-3, 3
    g = s2b.GridSpec.square(d)
    phi = s2b.gaussian_datum(g)
    paths = s2b.BrownianPaths.philox(T, dt_leb, M, seed=9, ctx=ctx)
    cfg = s2b.MagnusConfig(order=3, dt=0.1)
    for family in ("langevin-constant", "langevin-variable"):
        a = s2b.solve_iterated_magnus(cfg, s2b.Operator.from_family(g, family, order=3, ctx=ctx), phi, paths, T, g)
        b = s2b.solve_iterated_magnus(cfg, s2b.Operator.from_family_device(g, family, order=3, ctx=ctx), phi, paths,
                                      T, g)
        assert np.array_equal(a[-1].states(), b[-1].states())


def test_device_assembly_time_1024(s2b, ctx):
    """The setup the device assembly removes from a 1024^2 run (host builder ~3 s)."""
    g = s2b.GridSpec.square(1024)
    s2b.HostOps(s2b.GridSpec.square(64), "langevin-variable", order=3, device=ctx)  # warm-up
    t0 = time.perf_counter()
    dev = s2b.HostOps(g, "langevin-variable", order=3, device=ctx)
    t_dev = time.perf_counter() - t0
    t0 = time.perf_counter()
    host = s2b.HostOps(g, "langevin-variable", order=3)
    t_host = time.perf_counter() - t0
    print(f"1024^2 order-3 CommutatorSet: device {t_dev:.3f} s, host {t_host:.3f} s")
    for slot in ("BAA", "BAB"):
        assert _same(host.csr(slot), dev.csr(slot))
