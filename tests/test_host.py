"""CPU tests of the host side: the C ABI library loads and exports every symbol the header
declares, and the host-kept C++ builder (grid, CSR operators, commutators, xoshiro Brownian
batch) is bitwise the reference's.  No GPU compute is called here."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "spde2d_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(s2b_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(s2b):
    from paper_2207_09776_b200 import _capi
    L = _capi.lib()
    decl = declared_symbols()
    assert len(decl) > 40
    missing = [s for s in decl if not hasattr(L, s)]
    assert not missing, missing
    # the Python binding covers the whole header too
    assert sorted(set(decl) - set(_capi.SIGNATURES)) == []


def test_library_has_no_oracle_dependency():
    """The product .so must not link or embed the oracle/reference code."""
    import subprocess
    lib = os.path.join(ROOT, "paper_2207_09776_b200", "lib", "libspde2d_b200.so")
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True).stdout
    assert "ref_" not in " ".join(l.split()[-1] for l in out.splitlines() if l.strip())
    assert "rs_" not in " ".join(l.split()[-1] for l in out.splitlines() if l.strip()).split("s2b")[0]
    deps = subprocess.run(["ldd", lib], capture_output=True, text=True).stdout
    assert "spde2d_ref" not in deps and "restate" not in deps


@pytest.mark.parametrize("family,d,order", [
    ("langevin-constant", 10, 3), ("langevin-constant", 50, 3), ("langevin-variable", 16, 3),
    ("langevin-variable", 9, 2), ("langevin-constant", 5, 1), ("langevin-constant", 3, 3)])
def test_host_builder_bitwise_vs_reference(ref, s2b, family, d, order):
    g = s2b.GridSpec.square(d)
    host = s2b.HostOps(g, family, order=order)
    ops = ref.Ops(family, d, order=order)
    for slot in ref.SLOTS:
        a, b = host.csr(slot), ops.csr(slot)
        if b is None:
            assert a is None
            continue
        for x, y in zip(a, b):
            assert np.array_equal(x, y), slot
    for name in ref.FIELD_NAMES:
        fa, za = host.field(name)
        fb, zb = ops.field(name)
        assert za == zb and np.array_equal(fa, fb)


def test_host_builder_custom_fields_bitwise(ref, s2b):
    d = 12
    g = s2b.GridSpec.square(d)
    x = g.nodes(0)
    X, V = np.meshgrid(x, x, indexing="xy")
    fields = {"h": (0.2 * np.cos(X)).ravel(), "fx": (-V).ravel(), "fv": (0.3 * np.sin(X)).ravel(),
              "gxx": (0.05 + 0 * X).ravel(), "gxv": (0.02 * np.sin(X + V)).ravel(),
              "gvv": (1.1 + 0.1 * np.cos(X)).ravel(), "sig": (0.1 * np.cos(V)).ravel(),
              "sigx": (0.05 * np.sin(X)).ravel(), "sigv": (0.3 + 0 * X).ravel()}
    host = s2b.HostOps(g, "fields", order=3, fields=fields)
    ops = ref.Ops("fields", d, order=3, fields=fields)
    for slot in ref.SLOTS:
        for x_, y_ in zip(host.csr(slot), ops.csr(slot)):
            assert np.array_equal(x_, y_), slot


def test_host_brownian_bitwise_vs_reference(ref, s2b):
    for seed in (1, 424242):
        a = s2b.simulate_brownian(0.3, 1e-3, 7, seed)
        b, _ = ref.simulate_brownian(0.3, 1e-3, 7, seed)
        assert np.array_equal(a, b)
    assert np.all(a[:, 0] == 0.0)


def test_host_errors_mirror_reference(s2b):
    g = s2b.GridSpec.square(8)
    with pytest.raises(s2b.ConfigError):
        s2b.HostOps(g, "langevin-constant", a=0.05, sigma=1.0)  # a - sigma^2 <= 0
    with pytest.raises(s2b.ConfigError):
        s2b.HostOps(g, "langevin-constant", order=4)
    with pytest.raises(s2b.ConfigError):
        s2b.simulate_brownian(1.0, 0.3, 4, 1)  # incommensurate
    with pytest.raises(s2b.ConfigError):
        s2b.simulate_brownian(1.0, 1e-3, 0, 1)
    with pytest.raises(s2b.ConfigError):
        s2b.HostOps(s2b.GridSpec(0, 4), "langevin-constant")


def test_central_region_mirror(s2b, rs):
    for d in (4, 20, 64, 256, 300):
        for kappa in range(0, 6):
            try:
                want = rs.central_region(d, kappa)
            except ValueError:
                with pytest.raises(s2b.ConfigError):
                    s2b.central_region(d, kappa)
                continue
            assert s2b.central_region(d, kappa) == want


def test_gaussian_datum_bitwise(ref, s2b):
    for d in (7, 16):
        assert np.array_equal(s2b.gaussian_datum(s2b.GridSpec.square(d)),
                              ref.Ops("langevin-constant", d, order=1).datum())


def test_bench_presets_parse(monkeypatch):
    """bench.py --config presets: every BASELINE workload shape parses; explicit flags win."""
    import importlib
    import sys as _sys
    bench = importlib.import_module("bench")
    for cfg, d in (("cfg1", 64), ("cfg2", 256), ("cfg3", 256), ("cfg4", 512), ("cfg5", 1024)):
        monkeypatch.setattr(_sys, "argv", ["bench.py", "--config", cfg])
        a = bench.parse()
        assert a.d == d and a.preset == cfg
        nwin = int(round(a.T / a.dt))
        assert a.warmup >= 3 and a.warmup + 2 * a.steps <= nwin  # timed + e2e windows fit T
    monkeypatch.setattr(_sys, "argv", ["bench.py", "--config", "cfg5", "--paths", "128"])
    assert bench.parse().paths == 128
    monkeypatch.setattr(_sys, "argv", ["bench.py"])
    a = bench.parse()
    assert (a.d, a.paths, a.order, a.preset) == (256, 16384, 3, "cfg2")


def _ref_built():
    return os.path.isdir(os.path.join(ROOT, "oracle", "_ref")) and any(
        f.endswith(".so") for f in os.listdir(os.path.join(ROOT, "oracle", "_ref")))


@pytest.mark.skipif(not _ref_built(), reason="oracle/_ref not built")
def test_bench_reference_arm_contract(tmp_path):
    """`bench.py --impl reference` (the driver's reference arm): rank 0 prints ONE JSON line
    with the arm's keys on a bounded cfg1 sample; any other rank exits 0 without output."""
    import json
    import subprocess
    import sys as _sys
    env = dict(os.environ, OMP_NUM_THREADS="2")
    cmd = [_sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "cfg1",
           "--steps", "1", "--warmup", "0"]
    out = subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=tmp_path, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["metric"] == "magnus path*gridpoint*windows/s"
    assert d["value"] > 0 and d["steps"] == 1 and d["warmup"] == 0 and d["higher_is_better"]
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["value"] == d["value"]
    assert d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    env.update(RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    out = subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=tmp_path, timeout=120)
    assert out.returncode == 0 and out.stdout.strip() == ""


def test_python_mirror_validates_host_buffers(s2b):
    """Shapes/dtypes are checked before any pointer reaches C (no silent reinterpretation)."""
    g = s2b.GridSpec.square(8)
    with pytest.raises(s2b.DimensionError):
        s2b.HostOps(g, "fields", fields={"h": np.ones(63)})
    with pytest.raises(s2b.ConfigError):
        s2b.HostOps(g, "fields", fields={"bogus": np.ones(64)})
    s2b.HostOps(g, "fields", fields={"h": np.ones(64), "sig": np.ones((8, 8))})
    p = object.__new__(s2b.BrownianPaths)
    p.h, p.M, p.steps = None, 2, 4
    with pytest.raises(s2b.DimensionError):
        p.upload(0, 4, np.zeros((2, 4)))
    with pytest.raises(s2b.DimensionError):
        p.upload(0, 4, np.zeros((2, 5), np.float32))
    with pytest.raises(s2b.DimensionError):
        p.upload(0, 4, np.zeros((5, 2)).T)
    with pytest.raises(s2b.DimensionError):
        s2b.BrownianPaths.from_values(np.zeros(5), 1e-3)


UNIT_REF = os.path.join(ROOT, "build", "dropin", "unit_ref")
UNIT_B200 = os.path.join(ROOT, "build", "dropin", "unit_b200")


@pytest.mark.skipif(not os.path.exists(UNIT_REF), reason="reference unit suite not built (needs /root/reference)")
def test_doctest_compat_harness_passes_the_reference_suite_on_the_reference():
    """tests/cpp/compat/doctest.h runs the reference's 83 unit test cases against the reference
    library itself with no failure (the harness check behind test_reference_unit_suite_on_b200)."""
    import subprocess
    r = subprocess.run([UNIT_REF], capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, OMP_NUM_THREADS=str(max(1, min(16, os.cpu_count() or 1)))))
    assert "test cases: 83 | 83 passed | 0 failed" in r.stdout, r.stdout[-500:] + r.stderr[-2000:]


@pytest.mark.skipif(not os.path.exists(UNIT_B200), reason="drop-in unit suite not built")
def test_reference_unit_suite_host_cases_on_cpu():
    """The host-kept half of the drop-in (grid, CSR algebra, operators, commutators, Brownian
    batch, MagnusLogBuilder, central region) passes the reference's own unit cases without a
    GPU; every case that reaches the GPU fails loudly on the missing device (no CPU fallback)."""
    import subprocess
    r = subprocess.run([UNIT_B200], capture_output=True, text=True, timeout=600)
    failed = [l for l in r.stderr.splitlines() if "FAILED:" in l]
    threw = [l for l in r.stderr.splitlines() if " threw: " in l]
    assert "test cases: 83 |" in r.stdout, r.stdout
    passed = int(r.stdout.split("test cases: 83 | ")[1].split(" passed")[0])
    assert passed >= 49, r.stdout + r.stderr[-2000:]
    assert len(threw) == len(failed) == 83 - passed, r.stderr[-2000:]
    assert all("CUDA" in l or "cuda" in l for l in threw), threw


LOGB = [os.path.join(ROOT, "build", "dropin", n) for n in ("logb_b200", "logb_ref")]


@pytest.mark.skipif(not all(os.path.exists(p) for p in LOGB), reason="MagnusLogBuilder drivers not built")
def test_magnus_log_builder_bytes_equal_the_reference(tmp_path):
    """MagnusLogBuilder (magnus.hpp:61-86): union pattern and fill() values of the drop-in equal
    the reference's byte for byte -- constant, variable and nine-field families, builder
    orders 1-3, every fill order, zero and non-zero functionals, square and rectangular grids."""
    import subprocess
    outs = []
    for exe in LOGB:
        out = tmp_path / os.path.basename(exe)
        subprocess.run([exe, str(out)], check=True, timeout=300)
        outs.append(out.read_bytes())
    assert len(outs[0]) > 1_000_000 and outs[0] == outs[1]


def test_bench_world_size_must_match_gpus(tmp_path):
    """A launcher world size that differs from --gpus is refused (exit 2), never reported as a
    mislabelled one-GPU number."""
    import subprocess
    import sys as _sys
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([_sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2"], capture_output=True,
                         text=True, env=env, cwd=tmp_path, timeout=300)
    assert out.returncode == 2 and "WORLD_SIZE=1" in out.stderr


@pytest.mark.skipif(not _ref_built(), reason="oracle/_ref not built")
def test_bench_self_spawns_ranks(tmp_path):
    """`bench.py --gpus 2` with no launcher re-executes itself under torch.distributed.run:
    two ranks, one JSON line (rank 0), labelled n_gpus 2."""
    import json
    import subprocess
    import sys as _sys
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["OMP_NUM_THREADS"] = "2"
    cmd = [_sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--impl", "reference", "--config",
           "cfg1", "--steps", "1", "--warmup", "0"]
    out = subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=tmp_path, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["impl"] == "reference"
    assert d["cpu_baseline"]["setup_s_per_call"] >= 0.0
