"""TEST INFRASTRUCTURE ONLY — ctypes access to the plain-C restatement (oracle/restate.c).

The restatement re-derives the reference hot path operation by operation; it is
pinned against the compiled reference (oracle/_ref) and the committed golden
fixtures in tests/test_oracle.py.  Only tests/, ``__graft_entry__.smoke()`` and
bench.py's cpu_baseline leg may use it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_build", "librestate.so")

_dp = C.POINTER(C.c_double)
_sz = C.c_size_t
_szp = C.POINTER(C.c_size_t)
_i32p = C.POINTER(C.c_int32)
_u8p = C.POINTER(C.c_uint8)
_ip = C.POINTER(C.c_int)

_lib = None


def build():
    if not os.path.exists(LIB_PATH):
        subprocess.check_call(["make", "-s", "-C", _HERE, "restate"])


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(LIB_PATH)
        _lib.rs_one_norm.restype = C.c_double
        _lib.rs_euler_step.restype = C.c_double
        _lib.rs_union_pattern.restype = C.c_size_t
    return _lib


def _d(a):
    return a.ctypes.data_as(_dp)


class _Csr(C.Structure):
    _fields_ = [("rp", _szp), ("ci", _i32p), ("v", _dp)]


def _csr_array(sources):
    """sources: list of 6 (rp, ci, v) or None -> (ctypes array, keepalive)."""
    arr = (_Csr * 6)()
    keep = []
    for s, src in enumerate(sources):
        if src is None:
            continue
        rp = np.ascontiguousarray(src[0], np.uint64)
        ci = np.ascontiguousarray(src[1], np.int32)
        v = np.ascontiguousarray(src[2], np.float64)
        keep += [rp, ci, v]
        arr[s] = _Csr(rp.ctypes.data_as(_szp), ci.ctypes.data_as(_i32p), _d(v))
    return arr, keep


def simulate_brownian(T, dt_leb, M, seed):
    steps = int(round(T / dt_leb))
    values = np.empty((M, steps + 1))
    inc = np.empty((M, steps))
    lib().rs_simulate_brownian(_sz(steps), C.c_double(dt_leb), _sz(M), C.c_uint64(seed),
                               _d(values), _d(inc))
    return values, inc


def functionals(path, k0, k1, dt_leb):
    p = np.ascontiguousarray(path, np.float64)
    out = np.empty(5)
    lib().rs_functionals(_d(p), _sz(k0), _sz(k1), C.c_double(dt_leb), _d(out))
    return out


def log_coefficients(order, f5):
    f = np.ascontiguousarray(f5, np.float64)
    c = np.empty(6)
    lib().rs_log_coefficients(C.c_int(order), _d(f), _d(c))
    return c


def union_fill(n, build_order, order, sources, c):
    arr, keep = _csr_array(sources)
    nnz = lib().rs_union_pattern(_sz(n), C.c_int(build_order), arr, None, None)
    rp = np.empty(n + 1, np.uint64)
    ci = np.empty(nnz, np.int32)
    lib().rs_union_pattern(_sz(n), C.c_int(build_order), arr, rp.ctypes.data_as(_szp),
                           ci.ctypes.data_as(_i32p))
    v = np.empty(nnz)
    cc = np.ascontiguousarray(c, np.float64)
    lib().rs_union_fill(_sz(n), C.c_int(build_order), C.c_int(order), arr, _d(cc),
                        rp.ctypes.data_as(_szp), ci.ctypes.data_as(_i32p), _d(v))
    return rp, ci, v


def one_norm(rp, ci, v):
    rp = np.ascontiguousarray(rp, np.uint64)
    ci = np.ascontiguousarray(ci, np.int32)
    v = np.ascontiguousarray(v, np.float64)
    return lib().rs_one_norm(_sz(len(rp) - 1), rp.ctypes.data_as(_szp), ci.ctypes.data_as(_i32p),
                             _d(v))


def expmv(rp, ci, v, x, tol=1e-10, theta=1.0, max_segments=4096):
    n = len(rp) - 1
    rp = np.ascontiguousarray(rp, np.uint64)
    ci = np.ascontiguousarray(ci, np.int32)
    v = np.ascontiguousarray(v, np.float64)
    x = np.ascontiguousarray(x, np.float64)
    y = np.empty(n)
    rep = np.zeros(4, np.int32)
    kseg = np.zeros(max_segments, np.int32)
    norm = C.c_double()
    lib().rs_expmv(_sz(n), rp.ctypes.data_as(_szp), ci.ctypes.data_as(_i32p), _d(v), _d(x),
                   C.c_double(tol), C.c_double(theta), _d(y), rep.ctypes.data_as(_ip),
                   kseg.ctypes.data_as(_ip), C.c_int(max_segments), C.byref(norm))
    return y, {"status": int(rep[0]), "segments": int(rep[1]), "max_terms": int(rep[2]),
               "terms": int(rep[3]), "norm": norm.value,
               "k_per_segment": kseg[:min(int(rep[1]), max_segments)].copy()}


def magnus_path(n, order, sources, phi, path, dt_leb, dt_steps, total_steps, record_steps,
                tol=1e-10, theta=1.0, cap=1e10):
    """One trajectory of solve_iterated_magnus; returns (states[R][n], status[R],
    terms per window, segments per window)."""
    arr, keep = _csr_array(sources)
    rec = np.ascontiguousarray(record_steps, np.uint64)
    R = len(rec)
    nwin = total_steps // dt_steps
    states = np.full((R, n), np.nan)
    status = np.ones(R, np.uint8)
    wt = np.zeros(nwin, np.int32)
    ws = np.zeros(nwin, np.int32)
    phi = np.ascontiguousarray(phi, np.float64)
    path = np.ascontiguousarray(path, np.float64)
    lib().rs_magnus_path(_sz(n), C.c_int(order), arr, _d(phi), _d(path), C.c_double(dt_leb),
                         _sz(dt_steps), _sz(total_steps), rec.ctypes.data_as(_szp), _sz(R),
                         C.c_double(tol), C.c_double(theta), C.c_double(cap), _d(states),
                         status.ctypes.data_as(_u8p), wt.ctypes.data_as(_ip),
                         ws.ctypes.data_as(_ip))
    return states, status, wt, ws


def _fields_array(fields9):
    arr = (_dp * 9)()
    keep = []
    for k, f in enumerate(fields9):
        if f is not None:
            f = np.ascontiguousarray(f, np.float64)
            keep.append(f)
            arr[k] = _d(f)
    return arr, keep


def stencils(dx, dv):
    """EulerStencils::from_grid (euler.cpp:18-26)."""
    return np.array([1.0 / (2.0 * dx), 1.0 / (dx * dx), 1.0 / (2.0 * dv), 1.0 / (dv * dv),
                     1.0 / (4.0 * dx * dv)])


def euler_step(nx, nv, fields9, st, u, dW, dt):
    arr, keep = _fields_array(fields9)
    st = np.ascontiguousarray(st, np.float64)
    u = np.ascontiguousarray(u, np.float64)
    out = np.empty(nx * nv)
    mx = lib().rs_euler_step(_sz(nx), _sz(nv), arr, _d(st), _d(u), _d(out), C.c_double(dW),
                             C.c_double(dt))
    return out, mx


def euler_path(nx, nv, fields9, st, phi, path, step_leb, total_steps, dt, record_steps):
    arr, keep = _fields_array(fields9)
    st = np.ascontiguousarray(st, np.float64)
    rec = np.ascontiguousarray(record_steps, np.uint64)
    R = len(rec)
    states = np.full((R, nx * nv), np.nan)
    status = np.ones(R, np.uint8)
    phi = np.ascontiguousarray(phi, np.float64)
    path = np.ascontiguousarray(path, np.float64)
    lib().rs_euler_path(_sz(nx), _sz(nv), arr, _d(st), _d(phi), _d(path), _sz(step_leb),
                        _sz(total_steps), C.c_double(dt), rec.ctypes.data_as(_szp), _sz(R),
                        _d(states), status.ctypes.data_as(_u8p))
    return states, status


def exact_field(xn, vn, t, a, sigma, W, IW):
    xn = np.ascontiguousarray(xn, np.float64)
    vn = np.ascontiguousarray(vn, np.float64)
    out = np.empty(len(xn) * len(vn))
    lib().rs_exact_field(_sz(len(xn)), _sz(len(vn)), _d(xn), _d(vn), C.c_double(t),
                         C.c_double(a), C.c_double(sigma), C.c_double(W), C.c_double(IW), _d(out))
    return out


def central_region(d, kappa):
    lo, hi = _sz(), _sz()
    rc = lib().rs_central_region(_sz(d), C.c_int(kappa), C.byref(lo), C.byref(hi))
    if rc:
        raise ValueError("empty central region")
    return lo.value, hi.value


def errors(nx, kappa, ref, app, app_status=None, ref_status=None):
    lo, hi = central_region(nx, kappa)
    w = hi - lo + 1
    ref = np.ascontiguousarray(ref, np.float64)
    app = np.ascontiguousarray(np.nan_to_num(app), np.float64)
    M = ref.shape[0]
    me = np.empty(w * w)
    err, ame = C.c_double(), C.c_double()
    bl, ex = _sz(), _sz()
    ast = None if app_status is None else np.ascontiguousarray(app_status, np.uint8)
    rst = None if ref_status is None else np.ascontiguousarray(ref_status, np.uint8)
    rc = lib().rs_errors(_sz(nx), _sz(lo), _sz(hi), _d(ref),
                         rst.ctypes.data_as(_u8p) if rst is not None else None, _d(app),
                         ast.ctypes.data_as(_u8p) if ast is not None else None, _sz(M),
                         C.byref(err), C.byref(bl), C.byref(ame), C.byref(ex), _d(me))
    if rc:
        raise ValueError("reference blew up or has zero norm")
    return {"err": err.value, "blowups": bl.value, "ame": ame.value, "excluded": ex.value,
            "me": me.reshape(w, w)}
