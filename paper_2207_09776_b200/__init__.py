"""B200-native iterated stochastic Magnus / Euler-Maruyama solver for the 2-D kinetic SPDE
of arXiv 2207.09776 (du = (a/2 d_vv + v d_x + b d_v + c) u dt + (sigma d_v + beta) u dW).

Python host mirror of the reference's solver API (/root/reference/proj/include/spde2d):
same names, argument meaning and error classes, backed by the sm_100a kernels through
the C ABI (include/spde2d_b200.h).  Data stays on the GPU between calls; ensembles are
device handles that download on demand.  There is no CPU fallback: the product path
raises if the CUDA library or a B200 is missing.

Reference interface mirrored (file:line under /root/reference/proj/include/spde2d):
  MagnusConfig            magnus.hpp:19-28         EulerConfig          euler.hpp:12-16
  solve_iterated_magnus   magnus.hpp:93-97         solve_euler          euler.hpp:46-49
  exact_reference         exact_langevin.hpp:44-46 gaussian_datum       exact_langevin.hpp:30
  central_region          analysis.hpp:26          mean_rel_error       analysis.hpp:48-50
  mean_abs_error          analysis.hpp:35-37       avg_mean_abs_error   analysis.hpp:40
  expmv                   sparse.hpp:153-155       CommutatorSet        operators.hpp:78-88
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _capi
from ._capi import lib

__all__ = [
    "ConfigError", "DimensionError", "ExpmvError", "Context", "GridSpec", "Operator", "Fields",
    "BrownianPaths", "MagnusConfig", "EulerConfig", "Ensemble", "MagnusSession",
    "solve_iterated_magnus", "solve_euler", "exact_reference", "central_region",
    "mean_rel_error", "mean_abs_error", "avg_mean_abs_error", "exact_errors", "gaussian_datum",
    "expmv", "default_context", "ExpmvWorkspace", "expmv_into", "EulerStencils", "euler_step",
    "MultiGPU", "shard",
]


class ConfigError(ValueError):
    """spde2d::ConfigError (errors.hpp:10-14)."""


class DimensionError(ValueError):
    """spde2d::DimensionError (errors.hpp:16-19)."""


class ExpmvError(RuntimeError):
    """spde2d::ExpmvError (sparse.hpp:132-142)."""

    def __init__(self, status, msg):
        super().__init__(msg)
        self.status = status


class CudaError(RuntimeError):
    pass


def _check(rc):
    if rc == _capi.OK:
        return
    msg = lib().s2b_last_error().decode()
    if rc == _capi.ERR_CONFIG:
        raise ConfigError(msg)
    if rc == _capi.ERR_DIMENSION:
        raise DimensionError(msg)
    if rc == _capi.ERR_CUDA:
        raise CudaError(msg)
    raise RuntimeError(msg)


def _dptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


# ---------------------------------------------------------------- context
class Context:
    """One GPU: a CUDA stream and launch counter (s2b_context)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        _check(lib().s2b_context_create(int(device), C.byref(h)))
        self.h = h
        self.device = device

    def synchronize(self):
        _check(lib().s2b_context_synchronize(self.h))

    @property
    def stream(self) -> int:
        return lib().s2b_context_stream(self.h) or 0

    @property
    def launches(self) -> int:
        return int(lib().s2b_context_launches(self.h))

    def kernel_names(self):
        """Mangled names of the dominant Magnus kernels and of the E-M step kernel this context
        launched last."""
        a, b = C.create_string_buffer(4096), C.create_string_buffer(4096)
        _check(lib().s2b_context_kernel_names(self.h, a, b, 4096))
        e = C.create_string_buffer(4096)
        _check(lib().s2b_context_em_kernel_name(self.h, e, 4096))
        return {"cluster": a.value.decode(), "stream": b.value.decode(), "em": e.value.decode()}

    def close(self):
        if getattr(self, "h", None):
            lib().s2b_context_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default = {}


def default_context(device: int = 0) -> Context:
    if device not in _default:
        _default[device] = Context(device)
    return _default[device]


# ---------------------------------------------------------------- grid / operators
@dataclass
class GridSpec:
    """GridSpec (grid.hpp:28-40): n interior nodes a + (i+1)(b-a)/(n+1) per axis."""
    nx: int
    nv: int
    ax: float = -4.0
    bx: float = 4.0
    av: float = -4.0
    bv: float = 4.0

    @staticmethod
    def square(d, a=-4.0, b=4.0):
        return GridSpec(int(d), int(d), a, b, a, b)

    def dim(self):
        return self.nx * self.nv

    def c(self):
        return _capi.Grid(self.ax, self.bx, self.nx, self.av, self.bv, self.nv)

    def nodes(self, axis):
        a, b, n = (self.ax, self.bx, self.nx) if axis == 0 else (self.av, self.bv, self.nv)
        delta = (b - a) / float(n + 1)
        return np.array([a + float(i + 1) * delta for i in range(n)])


FAMILIES = {"langevin-constant": 0, "langevin-variable": 1, "fields": 2}
FIELD_NAMES = ("h", "fx", "fv", "gxx", "gxv", "gvv", "sig", "sigx", "sigv")
SLOTS = ("B", "A", "A2", "BA", "BAA", "BAB")


def _fields_array(fields, grid):
    arr = (C.POINTER(C.c_double) * 9)()
    keep = []
    if fields:
        unknown = set(fields) - set(FIELD_NAMES)
        if unknown:
            raise ConfigError(f"coefficient fields: unknown names {sorted(unknown)}")
        for k, name in enumerate(FIELD_NAMES):
            f = fields.get(name)
            if f is not None:
                f = np.ascontiguousarray(f, dtype=np.float64).reshape(-1)
                if f.size != grid.dim():  # C copies exactly nx*nv doubles per field
                    raise DimensionError(f"coefficient field {name}: {f.size} values, grid has {grid.dim()}")
                keep.append(f)
                arr[k] = _dptr(f)
    return arr, keep


class Operator:
    """The CommutatorSet uploaded as 2-D stencil weights (s2b_operator)."""

    def __init__(self, h, ctx, grid, order):
        self.h, self.ctx, self.grid, self.order = h, ctx, grid, order

    @classmethod
    def from_family(cls, grid: GridSpec, family="langevin-constant", a=1.1,
                    sigma=1.0 / np.sqrt(10.0), order=3, fields=None, ctx: Context = None):
        """Host-kept builder (sample_coefficients -> assemble_* -> precompute_commutators)."""
        ctx = ctx or default_context()
        arr, keep = _fields_array(fields, grid)
        h = C.c_void_p()
        _check(lib().s2b_operator_build(ctx.h, C.byref(grid.c()), FAMILIES[family], a, sigma, arr,
                                        order, C.byref(h)))
        return cls(h, ctx, grid, order)

    @classmethod
    def from_family_device(cls, grid: GridSpec, family="langevin-constant", a=1.1,
                           sigma=1.0 / np.sqrt(10.0), order=3, fields=None, ctx: Context = None):
        """from_family with the CommutatorSet assembled on the GPU."""
        ctx = ctx or default_context()
        arr, keep = _fields_array(fields, grid)
        h = C.c_void_p()
        _check(lib().s2b_operator_build_device(ctx.h, C.byref(grid.c()), FAMILIES[family], a, sigma, arr,
                                               order, C.byref(h)))
        return cls(h, ctx, grid, order)

    @classmethod
    def from_csr(cls, grid: GridSpec, order, sources: Sequence, ctx: Context = None):
        """sources: six (row_ptr, col_idx, values) CSR triples in slot order B, A, A2, BA,
        BAA, BAB (None for absent), e.g. a reference CommutatorSet."""
        ctx = ctx or default_context()
        arr = (_capi.Csr * 6)()
        keep = []
        for s, src in enumerate(sources):
            if src is None:
                continue
            rp = np.ascontiguousarray(src[0], np.uint64)
            ci = np.ascontiguousarray(src[1], np.int32)
            v = np.ascontiguousarray(src[2], np.float64)
            keep += [rp, ci, v]
            arr[s] = _capi.Csr(len(rp) - 1, rp.ctypes.data_as(C.POINTER(C.c_size_t)),
                               ci.ctypes.data_as(C.POINTER(C.c_int32)), _dptr(v))
        h = C.c_void_p()
        _check(lib().s2b_operator_create(ctx.h, C.byref(grid.c()), int(order), arr, C.byref(h)))
        return cls(h, ctx, grid, order)

    def info(self):
        out = (C.c_int64 * 6)()
        _check(lib().s2b_operator_info(self.h, out))
        return {"stencil_points": out[0], "compressed": bool(out[1]), "rx": out[2], "rv": out[3],
                "pairs": out[4], "order": out[5]}

    def __del__(self):
        try:
            if self.h:
                lib().s2b_operator_destroy(self.h)
        except Exception:
            pass


class Fields:
    """CoefficientFields for Euler-Maruyama (s2b_fields)."""

    def __init__(self, h, ctx, grid):
        self.h, self.ctx, self.grid = h, ctx, grid

    @classmethod
    def from_family(cls, grid: GridSpec, family="langevin-constant", a=1.1,
                    sigma=1.0 / np.sqrt(10.0), ctx: Context = None):
        ctx = ctx or default_context()
        h = C.c_void_p()
        _check(lib().s2b_fields_build(ctx.h, C.byref(grid.c()), FAMILIES[family], a, sigma,
                                      C.byref(h)))
        return cls(h, ctx, grid)

    @classmethod
    def from_arrays(cls, grid: GridSpec, fields: dict, ctx: Context = None):
        ctx = ctx or default_context()
        arr, keep = _fields_array(fields, grid)
        h = C.c_void_p()
        _check(lib().s2b_fields_create(ctx.h, C.byref(grid.c()), arr, C.byref(h)))
        return cls(h, ctx, grid)

    def __del__(self):
        try:
            if self.h:
                lib().s2b_fields_destroy(self.h)
        except Exception:
            pass


class HostOps:
    """Host-kept CommutatorSet + CoefficientFields from the C++ builder (no GPU needed):
    the CSR the GPU operator is laid out from (operators.cpp:134-208 arithmetic)."""

    def __init__(self, grid: GridSpec, family="langevin-constant", a=1.1,
                 sigma=1.0 / np.sqrt(10.0), order=3, fields=None, device: Optional[Context] = None):
        """device: assemble the CommutatorSet on that context's GPU (s2b_host_ops_assemble_device)
        instead of the host builder; the CSR is the same, bit for bit."""
        arr, keep = _fields_array(fields, grid)
        h = C.c_void_p()
        if device is None:
            _check(lib().s2b_host_ops_build(C.byref(grid.c()), FAMILIES[family], a, sigma, arr, order,
                                            C.byref(h)))
        else:
            _check(lib().s2b_host_ops_assemble_device(device.h, C.byref(grid.c()), FAMILIES[family], a, sigma,
                                                      arr, order, C.byref(h)))
        self.h, self.grid, self.order = h, grid, order

    def csr(self, slot):
        s = SLOTS.index(slot) if isinstance(slot, str) else slot
        m = _capi.Csr()
        _check(lib().s2b_host_ops_csr(self.h, s, C.byref(m)))
        if m.rows == 0:
            return None
        rp = np.ctypeslib.as_array(m.row_ptr, (m.rows + 1,)).astype(np.uint64).copy()
        nnz = int(rp[-1])
        ci = np.ctypeslib.as_array(m.col_idx, (nnz,)).copy() if nnz else np.zeros(0, np.int32)
        v = np.ctypeslib.as_array(m.values, (nnz,)).copy() if nnz else np.zeros(0)
        return rp, ci, v

    def sources(self):
        return [self.csr(s) for s in range(6)]

    def field(self, name):
        d = C.POINTER(C.c_double)()
        z = C.c_int()
        _check(lib().s2b_host_ops_field(self.h, FIELD_NAMES.index(name), C.byref(d), C.byref(z)))
        return np.ctypeslib.as_array(d, (self.grid.dim(),)).copy(), bool(z.value)

    def __del__(self):
        try:
            if self.h:
                lib().s2b_host_ops_destroy(self.h)
        except Exception:
            pass


def simulate_brownian(T, dt_leb, M, seed) -> np.ndarray:
    """Host BrownianBatch::values [M][steps+1] (the reference's xoshiro256++ stream)."""
    steps = int(round(T / dt_leb))
    out = np.empty((M, steps + 1))
    _check(lib().s2b_host_simulate_brownian(T, dt_leb, M, seed, _dptr(out)))
    return out


def gaussian_datum(grid: GridSpec) -> np.ndarray:
    """phi = exp(-(x^2+v^2)/2) at the interior nodes, column-major (exact_langevin.cpp:29-39)."""
    out = np.empty(grid.dim())
    _check(lib().s2b_gaussian_datum(C.byref(grid.c()), _dptr(out)))
    return out


# ---------------------------------------------------------------- Brownian paths
class BrownianPaths:
    """Device BrownianBatch: prefix values [M][steps+1] (stochastics.hpp:32-43)."""

    def __init__(self, h, ctx, dt_leb, steps, M, seed):
        self.h, self.ctx, self.dt_leb, self.steps, self.M, self.seed = h, ctx, dt_leb, steps, M, seed

    @property
    def T(self):
        return self.steps * self.dt_leb

    @classmethod
    def from_values(cls, values, dt_leb, seed=1, ctx: Context = None):
        """Parity mode: the reference's own BrownianBatch::values."""
        v = np.ascontiguousarray(values, np.float64)
        if v.ndim != 2 or v.shape[1] < 2:
            raise DimensionError(f"BrownianPaths.from_values: need [M][steps+1] values, got {v.shape}")
        ctx = ctx or default_context()
        M, steps = v.shape[0], v.shape[1] - 1
        h = C.c_void_p()
        _check(lib().s2b_paths_create_host(ctx.h, dt_leb, steps, M, seed, _dptr(v), C.byref(h)))
        return cls(h, ctx, dt_leb, steps, M, seed)

    @classmethod
    def philox(cls, T, dt_leb, M, seed=1, path_offset=0, ctx: Context = None):
        ctx = ctx or default_context()
        steps = int(round(T / dt_leb))
        if steps < 1 or abs(T - steps * dt_leb) > 1e-12 * max(1.0, abs(T)):
            raise ConfigError("simulate_brownian: horizon is not an integer multiple of dt_leb")
        h = C.c_void_p()
        _check(lib().s2b_paths_create_philox(ctx.h, dt_leb, steps, M, seed, path_offset,
                                             C.byref(h)))
        return cls(h, ctx, dt_leb, steps, M, seed)

    def upload(self, k0, k1, values):
        """Overwrite Lebesgue columns [k0, k1] of every path from a host [M][steps+1] array
        (asynchronous on the context stream when `values` is pinned).  The array is handed to
        C as is (no copy, so a pinned buffer stays pinned): it must be float64, C-contiguous
        and exactly [M][steps+1]."""
        if not isinstance(values, np.ndarray) or values.dtype != np.float64 or not values.flags.c_contiguous:
            raise DimensionError("BrownianPaths.upload: values must be a C-contiguous float64 array")
        if values.shape != (self.M, self.steps + 1):
            raise DimensionError(f"BrownianPaths.upload: values shape {values.shape} != "
                                 f"{(self.M, self.steps + 1)}")
        _check(lib().s2b_paths_upload(self.h, k0, k1, _dptr(values)))

    def values(self):
        out = np.empty((self.M, self.steps + 1))
        _check(lib().s2b_paths_download(self.h, _dptr(out)))
        return out

    def __del__(self):
        try:
            if self.h:
                lib().s2b_paths_destroy(self.h)
        except Exception:
            pass


# ---------------------------------------------------------------- configs / ensembles
@dataclass
class AdaptiveConfig:
    """AdaptiveConfig (magnus.hpp:14-17)."""
    enabled: bool = False
    tolerance: float = 1e-4
    shrink: float = 0.5

    def c(self):
        return _capi.AdaptiveConfig(1 if self.enabled else 0, float(self.tolerance), float(self.shrink))


@dataclass
class MagnusConfig:
    """MagnusConfig (magnus.hpp:19-28); `threads` is accepted and ignored on the GPU."""
    order: int = 3
    dt: float = 0.1
    expmv_tol: float = 1e-10
    expmv_theta: float = 1.0
    blowup_norm_cap: float = 1e10
    threads: int = 0
    record_times: list = field(default_factory=list)
    adaptive: AdaptiveConfig = field(default_factory=AdaptiveConfig)

    def c(self, T):
        rec = np.ascontiguousarray(self.record_times, np.float64)
        cfg = _capi.MagnusConfig(int(self.order), float(self.dt), float(T), float(self.expmv_tol),
                                 float(self.expmv_theta), float(self.blowup_norm_cap),
                                 _dptr(rec) if len(rec) else None, len(rec))
        return cfg, rec


@dataclass
class EulerConfig:
    """EulerConfig (euler.hpp:12-16)."""
    dt: float = 1e-4
    threads: int = 0
    record_times: list = field(default_factory=list)

    def c(self, T):
        rec = np.ascontiguousarray(self.record_times, np.float64)
        cfg = _capi.EulerConfig(float(self.dt), float(T), _dptr(rec) if len(rec) else None,
                                len(rec))
        return cfg, rec


class _EnsembleHandle:
    def __init__(self, h):
        self.h = h

    def __del__(self):
        try:
            if self.h:
                lib().s2b_ensemble_destroy(self.h)
        except Exception:
            pass


class Ensemble:
    """One SolutionEnsemble (magnus.hpp:34-44) living on the GPU: record `record` of a
    device ensemble handle.  states() downloads [M][n] (NaN rows for blown paths)."""

    def __init__(self, handle: _EnsembleHandle, record: int, t: float, M: int, n: int,
                 grid: GridSpec, seed: int, ctx: Context):
        self._h, self.record, self.t, self.M, self.n = handle, record, t, M, n
        self.grid, self.seed, self.ctx = grid, seed, ctx
        self._status = None

    @property
    def status(self) -> np.ndarray:
        """0 Ok, 1 BlownUp per trajectory."""
        if self._status is None:
            st = np.empty(self.M, np.uint8)
            _check(lib().s2b_ensemble_download(self._h.h, self.record, None,
                                               st.ctypes.data_as(C.POINTER(C.c_uint8))))
            self._status = st
        return self._status

    def states(self) -> np.ndarray:
        out = np.empty((self.M, self.n))
        st = np.empty(self.M, np.uint8)
        _check(lib().s2b_ensemble_download(self._h.h, self.record, _dptr(out),
                                           st.ctypes.data_as(C.POINTER(C.c_uint8))))
        self._status = st
        return out

    def trajectories(self):
        return self.M

    def blowup_count(self):
        return int(self.status.sum())

    def moments(self):
        """(sum_m u_m, sum_m u_m^2) over the non-blown paths of this record, and the live count."""
        mom = np.empty(2 * self.n)
        live = C.c_size_t()
        _check(lib().s2b_ensemble_moments(self._h.h, self.record, _dptr(mom), C.byref(live)))
        return mom[:self.n], mom[self.n:], int(live.value)

    def counters(self):
        t = np.empty(self.M, np.int64)
        w = np.empty(self.M, np.int64)
        _check(lib().s2b_ensemble_counters(self._h.h, t.ctypes.data_as(C.POINTER(C.c_int64)),
                                           w.ctypes.data_as(C.POINTER(C.c_int64))))
        return t, w


def _ensembles(h, grid, seed, ctx):
    handle = _EnsembleHandle(h)
    info = (C.c_int64 * 5)()
    _check(lib().s2b_ensemble_info(h, info, None))
    times = (C.c_double * info[0])()
    _check(lib().s2b_ensemble_info(h, info, times))
    return [Ensemble(handle, r, times[r], info[1], info[2], grid, seed, ctx)
            for r in range(info[0])]


# ---------------------------------------------------------------- solvers
def solve_iterated_magnus(cfg: MagnusConfig, comms: Operator, phi, batch: BrownianPaths, T,
                          grid: GridSpec, stats: Optional[dict] = None):
    """solve_iterated_magnus (magnus.hpp:93-97): one Ensemble per record time."""
    if len(phi) != grid.dim() or comms.grid.dim() != grid.dim():
        raise DimensionError("solve_iterated_magnus: dimension mismatch")
    ccfg, keep = cfg.c(T)
    phi = np.ascontiguousarray(phi, np.float64)
    h = C.c_void_p()
    st = _capi.MagnusStats()
    _check(lib().s2b_solve_magnus(comms.ctx.h, comms.h, C.byref(ccfg), _dptr(phi), batch.h,
                                  C.byref(h), C.byref(st)))
    if stats is not None:
        stats.update({k: getattr(st, k) for k, _ in _capi.MagnusStats._fields_})
    return _ensembles(h, grid, batch.seed, comms.ctx)


def solve_iterated_magnus_sweep(cfgs: Sequence[MagnusConfig], comms: Operator, phi, batch: BrownianPaths, T,
                                grid: GridSpec, stats: Optional[list] = None):
    """Several MagnusConfigs (e.g. one order at several dt) on shared paths in batched launches
    (run_stepsize_sweep, experiment.cpp:486-551).  Returns one ensemble list per config."""
    if len(phi) != grid.dim() or comms.grid.dim() != grid.dim():
        raise DimensionError("solve_iterated_magnus_sweep: dimension mismatch")
    n = len(cfgs)
    made = [c.c(T) for c in cfgs]
    arr = (_capi.MagnusConfig * n)(*[m[0] for m in made])
    phi = np.ascontiguousarray(phi, np.float64)
    outs = (C.c_void_p * n)()
    st = (_capi.MagnusStats * n)()
    _check(lib().s2b_solve_magnus_sweep(comms.ctx.h, comms.h, arr, n, _dptr(phi), batch.h, outs, st))
    if stats is not None:
        stats.extend({k: getattr(x, k) for k, _ in _capi.MagnusStats._fields_} for x in st)
    return [_ensembles(C.c_void_p(h), grid, batch.seed, comms.ctx) for h in outs]


def solve_adaptive_magnus(cfg: MagnusConfig, comms: Operator, phi, batch: BrownianPaths, T,
                          grid: GridSpec, stats: Optional[dict] = None):
    """solve_adaptive_magnus (magnus.hpp:104-108): orders 2 and 3 per window, shrink-and-retry
    on a relative gap above cfg.adaptive.tolerance; needs an order-3 operator."""
    if len(phi) != grid.dim() or comms.grid.dim() != grid.dim():
        raise DimensionError("solve_adaptive_magnus: dimension mismatch")
    ccfg, keep = cfg.c(T)
    acfg = cfg.adaptive.c()
    phi = np.ascontiguousarray(phi, np.float64)
    h = C.c_void_p()
    st = _capi.MagnusStats()
    _check(lib().s2b_solve_adaptive_magnus(comms.ctx.h, comms.h, C.byref(ccfg), C.byref(acfg), _dptr(phi),
                                           batch.h, C.byref(h), C.byref(st)))
    if stats is not None:
        stats.update({k: getattr(st, k) for k, _ in _capi.MagnusStats._fields_})
    return _ensembles(h, grid, batch.seed, comms.ctx)


def solve_euler(cfg: EulerConfig, fields: Fields, grid: GridSpec, phi, batch: BrownianPaths, T):
    """solve_euler (euler.hpp:46-49): one Ensemble per record time."""
    if len(phi) != grid.dim():
        raise DimensionError("solve_euler: datum shape mismatch")
    ccfg, keep = cfg.c(T)
    phi = np.ascontiguousarray(phi, np.float64)
    h = C.c_void_p()
    _check(lib().s2b_solve_euler(fields.ctx.h, fields.h, C.byref(ccfg), _dptr(phi), batch.h,
                                 C.byref(h)))
    return _ensembles(h, grid, batch.seed, fields.ctx)


class MagnusSession:
    """Resident solver: state stays in HBM; advance(n) moves every path n windows."""

    def __init__(self, cfg: MagnusConfig, comms: Operator, phi, batch: BrownianPaths, T):
        ccfg, keep = cfg.c(T)
        phi = np.ascontiguousarray(phi, np.float64)
        h = C.c_void_p()
        _check(lib().s2b_magnus_session_create(comms.ctx.h, comms.h, C.byref(ccfg), _dptr(phi),
                                               batch.h, C.byref(h)))
        # the C session borrows the operator and the paths: keep both alive as long as it
        self.h, self.ctx, self.grid, self.batch, self.op = h, comms.ctx, comms.grid, batch, comms

    def advance(self, n_windows=1):
        _check(lib().s2b_magnus_session_advance(self.h, n_windows))

    def reset(self):
        _check(lib().s2b_magnus_session_reset(self.h))

    def set_timing(self, on=True):
        _check(lib().s2b_magnus_session_set_timing(self.h, 1 if on else 0))

    def stats(self):
        st = _capi.MagnusStats()
        _check(lib().s2b_magnus_session_stats(self.h, C.byref(st)))
        return {k: getattr(st, k) for k, _ in _capi.MagnusStats._fields_}

    def moments(self, out=None):
        """(sum_m u_m, sum_m u_m^2) over live paths at the current time, and the live count."""
        n = self.grid.dim()
        out = np.empty(2 * n) if out is None else out
        live = C.c_double()
        _check(lib().s2b_magnus_session_moments(self.h, _dptr(out), C.byref(live)))
        return out[:n], out[n:], int(live.value)

    def snapshot(self):
        h = C.c_void_p()
        _check(lib().s2b_magnus_session_ensemble(self.h, C.byref(h)))
        return _ensembles(h, self.grid, self.batch.seed, self.ctx)[0]

    def finish(self):
        h = C.c_void_p()
        _check(lib().s2b_magnus_session_finish(self.h, C.byref(h)))
        return _ensembles(h, self.grid, self.batch.seed, self.ctx)

    def __del__(self):
        try:
            if self.h:
                lib().s2b_magnus_session_destroy(self.h)
        except Exception:
            pass


# ---------------------------------------------------------------- exact solution + norms
def exact_reference(grid: GridSpec, t, a, sigma, batch: BrownianPaths, ctx: Context = None):
    """exact_reference (exact_langevin.hpp:44-46) for LangevinParams{a, sigma}."""
    ctx = ctx or batch.ctx
    h = C.c_void_p()
    _check(lib().s2b_exact_reference(ctx.h, C.byref(grid.c()), t, a, sigma, batch.h, C.byref(h)))
    return _ensembles(h, grid, batch.seed, ctx)[0]


def central_region(d, kappa):
    """central_region (analysis.cpp:9-31): 0-based inclusive (lo, hi)."""
    import math
    if d < 2:
        raise ConfigError("central_region: need d >= 2")
    if kappa < 0:
        raise ConfigError("central_region: kappa must be non-negative")
    if kappa >= 63 or (1 << kappa) > d:
        raise ConfigError("central_region: empty region, kappa too large")
    half = d / 2.0
    width = d / math.pow(2.0, kappa + 1)
    lo1, hi1 = math.floor(half - width), math.floor(half + width)
    lo, hi = max(lo1 - 1, 0), min(hi1 - 1, d - 1)
    if hi < lo:
        raise ConfigError("central_region: empty region")
    return lo, hi


def _errors(ref: Ensemble, app: Ensemble, kappa):
    st = _capi.ErrorStats()
    lo, hi = central_region(ref.grid.nx, kappa)
    w = hi - lo + 1
    me = np.empty(w * w)
    _check(lib().s2b_errors(app.ctx.h, ref._h.h, ref.record, app._h.h, app.record, kappa,
                            C.byref(st), _dptr(me)))
    return st, me.reshape(w, w)


def mean_rel_error(ref: Ensemble, app: Ensemble, kappa):
    """RelError (analysis.hpp:43-50): dict(err, blowups)."""
    st, _ = _errors(ref, app, kappa)
    return {"err": st.err, "blowups": st.blowups}


def mean_abs_error(ref: Ensemble, app: Ensemble, kappa):
    """MeanAbsError (analysis.hpp:28-37): dict(me [w][w] Field order, excluded)."""
    st, me = _errors(ref, app, kappa)
    return {"me": me, "excluded": st.excluded, "ame": st.ame}


def avg_mean_abs_error(me):
    s = 0.0
    for v in np.asarray(me).reshape(-1):
        s += float(v)
    return s / me.size if me.size else 0.0


def exact_errors(app: Ensemble, a, sigma, batch: BrownianPaths, kappa, moments=False,
                 per_path=False):
    """Fused exact-reference norms: no reference ensemble is materialised."""
    st = _capi.ErrorStats()
    lo, hi = central_region(app.grid.nx, kappa)
    w = hi - lo + 1
    me = np.empty(w * w)
    rel = np.empty(app.M) if per_path else None
    mom = np.empty(2 * app.n) if moments else None
    _check(lib().s2b_exact_errors(app.ctx.h, app._h.h, app.record, a, sigma, batch.h, kappa,
                                  C.byref(st), _dptr(me), _dptr(rel) if per_path else None,
                                  _dptr(mom) if moments else None))
    out = {k: getattr(st, k) for k, _ in _capi.ErrorStats._fields_}
    out["me"] = me.reshape(w, w)
    if per_path:
        out["per_path_rel"] = rel
    if moments:
        out["sum_u"], out["sum_u2"] = mom[:app.n], mom[app.n:]
    return out


def expmv(csr, x, tol, theta=1.0, ctx: Context = None, throw=True):
    """expmv (sparse.hpp:144-155) of a general CSR matrix (row_ptr, col_idx, values)."""
    ctx = ctx or default_context()
    rp = np.ascontiguousarray(csr[0], np.uint64)
    ci = np.ascontiguousarray(csr[1], np.int32)
    v = np.ascontiguousarray(csr[2], np.float64)
    x = np.ascontiguousarray(x, np.float64)
    m = _capi.Csr(len(rp) - 1, rp.ctypes.data_as(C.POINTER(C.c_size_t)),
                  ci.ctypes.data_as(C.POINTER(C.c_int32)), _dptr(v))
    y = np.empty(len(rp) - 1)
    rep = (C.c_int * 4)()
    _check(lib().s2b_expmv(ctx.h, C.byref(m), _dptr(x), tol, theta, _dptr(y), rep))
    report = {"status": rep[0], "segments": rep[1], "max_terms": rep[2], "terms": rep[3]}
    if throw and rep[0] != 0:
        raise ExpmvError(rep[0], "expmv: overflow" if rep[0] == 1 else
                         "expmv: tolerance not reached within term budget")
    return y, report


# ---------------------------------------------------------------- kernel level
def _csr_struct(csr):
    rp = np.ascontiguousarray(csr[0], np.uint64)
    ci = np.ascontiguousarray(csr[1], np.int32)
    v = np.ascontiguousarray(csr[2], np.float64)
    if rp.ndim != 1 or len(rp) < 1 or len(ci) != len(v) or int(rp[-1]) != len(v):
        raise DimensionError("expmv: malformed CSR (row_ptr, col_idx, values)")
    m = _capi.Csr(len(rp) - 1, rp.ctypes.data_as(C.POINTER(C.c_size_t)),
                  ci.ctypes.data_as(C.POINTER(C.c_int32)), _dptr(v))
    return m, (rp, ci, v)


_EXPMV_STATUS = {0: "Ok", 1: "Overflow", 2: "ToleranceNotReached"}


class ExpmvWorkspace:
    """ExpmvWorkspace (sparse.hpp:121-130): device scratch reused across expmv_into calls;
    caches the device copy of the last CSR pattern (a refill of the same pattern only moves
    the values)."""

    def __init__(self, ctx: Context = None):
        self.ctx = ctx or default_context()
        h = C.c_void_p()
        _check(lib().s2b_expmv_workspace_create(self.ctx.h, C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            if self.h:
                lib().s2b_expmv_workspace_destroy(self.h)
        except Exception:
            pass


def expmv_into(csr, x, tol, theta=1.0, ws: ExpmvWorkspace = None, y=None):
    """expmv_into (sparse.hpp:149-151): returns (y, report) with the reference's ExpmvReport
    fields (status, residual, segments, max_terms) plus the Taylor terms applied.  Never
    raises on numerical failure (the status says it), like the reference."""
    ws = ws or ExpmvWorkspace()
    m, keep = _csr_struct(csr)
    n = m.rows
    x = np.ascontiguousarray(x, np.float64)
    if x.shape != (n,):
        raise DimensionError("expmv: vector length mismatch")
    y = np.empty(n) if y is None else y
    if y.dtype != np.float64 or y.shape != (n,) or not y.flags.c_contiguous:
        raise DimensionError("expmv_into: y must be a contiguous float64 vector of length n")
    rep = _capi.ExpmvReport()
    _check(lib().s2b_expmv_into(ws.h, C.byref(m), _dptr(x), float(tol), float(theta), _dptr(y),
                                C.byref(rep)))
    return y, {"status": _EXPMV_STATUS[rep.status], "residual": rep.residual, "segments": rep.segments,
               "max_terms": rep.max_terms, "terms": rep.terms}


@dataclass
class EulerStencils:
    """EulerStencils (euler.hpp:19-28)."""
    inv2dx: float = 0.0
    invdx2: float = 0.0
    inv2dv: float = 0.0
    invdv2: float = 0.0
    inv4dxdv: float = 0.0

    @staticmethod
    def from_grid(grid: GridSpec):
        dx = (grid.bx - grid.ax) / float(grid.nx + 1)
        dv = (grid.bv - grid.av) / float(grid.nv + 1)
        return EulerStencils(1.0 / (2.0 * dx), 1.0 / (dx * dx), 1.0 / (2.0 * dv), 1.0 / (dv * dv),
                             1.0 / (4.0 * dx * dv))

    def c(self):
        return (C.c_double * 5)(self.inv2dx, self.invdx2, self.inv2dv, self.invdv2, self.inv4dxdv)


def euler_step(fields: Fields, u, dW, dt, stencils: EulerStencils = None):
    """euler_step_into (euler.hpp:36-40): (out, max|out|) for one field u (n doubles,
    column-major), on the GPU."""
    n = fields.grid.dim()
    u = np.ascontiguousarray(u, np.float64).reshape(-1)
    if u.size != n:
        raise DimensionError("euler_step: field shape mismatch")
    out = np.empty(n)
    mx = C.c_double()
    st = (stencils or EulerStencils.from_grid(fields.grid)).c()
    _check(lib().s2b_euler_step(fields.h, st, _dptr(u), _dptr(out), float(dW), float(dt), C.byref(mx)))
    return out, mx.value


# ---------------------------------------------------------------- multi-GPU (one node)
def shard(M_total, rank, world):
    """Contiguous path range (offset, count) of `rank` (s2b_shard)."""
    off, cnt = C.c_size_t(), C.c_size_t()
    rc = lib().s2b_shard(int(M_total), int(rank), int(world), C.byref(off), C.byref(cnt))
    if rc != _capi.OK:
        raise ConfigError("shard: need 0 <= rank < world")
    return off.value, cnt.value


class MultiGPU:
    """Path-sharded solves over several devices of one node from ONE process (s2b_multi):
    a context and a host thread per device, Philox paths keyed by the global path id, one
    NCCL all-reduce + all-gather of the statistics at the end.  A device listed twice
    combines on the host (the sharding path on a one-GPU box)."""

    def __init__(self, devices: Sequence[int]):
        arr = (C.c_int * len(devices))(*devices)
        h = C.c_void_p()
        _check(lib().s2b_multi_create(arr, len(devices), C.byref(h)))
        self.h, self.devices = h, list(devices)
        info = (C.c_int * 2)()
        _check(lib().s2b_multi_info(self.h, info))
        self.nccl = bool(info[1])

    def _run(self, fn, grid, family, cfgc, phi, dt_leb, steps, M_total, seed, kappa, a, sigma, order, fields):
        arr, keep = _fields_array(fields, grid)
        spec = _capi.OperatorSpec(FAMILIES[family], float(a), float(sigma),
                                  C.cast(arr, C.POINTER(C.POINTER(C.c_double))) if fields else None, int(order))
        phi = np.ascontiguousarray(phi, np.float64)
        if phi.size != grid.dim():
            raise DimensionError("multi solve: datum shape mismatch")
        st = _capi.MultiStats()
        n = grid.dim()
        w2 = 0
        if kappa >= 0:
            lo, hi = central_region(grid.nx, kappa)
            w2 = (hi - lo + 1) ** 2
        me = np.empty(max(w2, 1))
        mom = np.empty(2 * n)
        rel = np.empty(M_total) if kappa >= 0 else None
        _check(fn(self.h, C.byref(grid.c()), C.byref(spec), C.byref(cfgc), _dptr(phi), float(dt_leb), int(steps),
                  int(M_total), int(seed), int(kappa), C.byref(st), _dptr(me), _dptr(mom),
                  _dptr(rel) if rel is not None else None))
        out = {k: getattr(st, k) for k, _ in _capi.MultiStats._fields_ if k != "errors"}
        out.update({k: getattr(st.errors, k) for k, _ in _capi.ErrorStats._fields_})
        out["sum_u"], out["sum_u2"] = mom[:n], mom[n:]
        if kappa >= 0:
            w = int(round(np.sqrt(w2)))
            out["me"] = me[:w2].reshape(w, w)
            out["per_path_rel"] = rel
        return out

    def solve_magnus(self, cfg: MagnusConfig, grid: GridSpec, phi, T, dt_leb, M_total, seed=1, kappa=-1,
                     family="langevin-constant", a=1.1, sigma=1.0 / np.sqrt(10.0), fields=None):
        steps = int(round(T / dt_leb))
        cfgc, keep = cfg.c(T)
        return self._run(lib().s2b_multi_solve_magnus, grid, family, cfgc, phi, dt_leb, steps, M_total, seed,
                         kappa, a, sigma, cfg.order, fields)

    def solve_euler(self, cfg: EulerConfig, grid: GridSpec, phi, T, dt_leb, M_total, seed=1, kappa=-1,
                    family="langevin-constant", a=1.1, sigma=1.0 / np.sqrt(10.0), fields=None):
        steps = int(round(T / dt_leb))
        cfgc, keep = cfg.c(T)
        return self._run(lib().s2b_multi_solve_euler, grid, family, cfgc, phi, dt_leb, steps, M_total, seed,
                         kappa, a, sigma, 1, fields)

    def __del__(self):
        try:
            if self.h:
                lib().s2b_multi_destroy(self.h)
        except Exception:
            pass
