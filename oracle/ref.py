"""TEST INFRASTRUCTURE ONLY — ctypes access to the UNMODIFIED reference library.

``oracle/_ref/libspde2d_ref.so`` is compiled by ``oracle/Makefile`` from the
reference sources under /root/reference/proj/src (never copied into this repo)
plus ``oracle/ref_shim.cpp``.  Only tests/, ``__graft_entry__.smoke()`` and
bench.py's cpu_baseline / ``--impl reference`` legs may import this module.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libspde2d_ref.so")

_dp = C.POINTER(C.c_double)
_sz = C.c_size_t
_szp = C.POINTER(C.c_size_t)
_u8p = C.POINTER(C.c_uint8)
_i32p = C.POINTER(C.c_int32)

_lib = None


class RefError(RuntimeError):
    pass


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RefError(f"reference oracle not built: {LIB_PATH} (run make -C oracle)")
        _lib = C.CDLL(LIB_PATH)
        _lib.ref_last_error.restype = C.c_char_p
    return _lib


def _ck(rc):
    if rc != 0:
        raise RefError(f"reference error {rc}: {lib().ref_last_error().decode()}")


def _d(a):
    return a.ctypes.data_as(_dp)


def max_threads() -> int:
    return int(lib().ref_max_threads())


FIELD_NAMES = ("h", "fx", "fv", "gxx", "gxv", "gvv", "sig", "sigx", "sigv")
SLOTS = ("B", "A", "A2", "BA", "BAA", "BAB")


class Ops:
    """Reference grid + coefficient fields + CommutatorSet (operators.hpp:60-88)."""

    def __init__(self, family, d, a=1.1, sigma=1.0 / np.sqrt(10.0), order=3,
                 bounds=(-4.0, 4.0, -4.0, 4.0), nv=None, fields=None):
        fam = {"langevin-constant": 0, "langevin-variable": 1, "fields": 2}[family]
        self.nx = int(d)
        self.nv = int(nv if nv is not None else d)
        self.n = self.nx * self.nv
        self.order = order
        self.a, self.sigma = a, sigma
        arr = (_dp * 9)()
        keep = []
        if fields is not None:
            for k, name in enumerate(FIELD_NAMES):
                f = fields.get(name)
                if f is not None:
                    f = np.ascontiguousarray(f, dtype=np.float64).reshape(-1)
                    keep.append(f)
                    arr[k] = _d(f)
        h = C.c_void_p()
        _ck(lib().ref_ops_create(C.c_int(fam), C.c_double(a), C.c_double(sigma), _sz(self.nx),
                                 _sz(self.nv), C.c_double(bounds[0]), C.c_double(bounds[1]),
                                 C.c_double(bounds[2]), C.c_double(bounds[3]), C.c_int(order),
                                 arr, C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            if getattr(self, "h", None) is not None and _lib is not None:
                _lib.ref_ops_destroy(self.h)
        except Exception:
            pass

    def csr(self, slot):
        """(row_ptr uint64, col_idx int32, values float64) copies; slot name or index."""
        s = SLOTS.index(slot) if isinstance(slot, str) else slot
        rows, nnz = _sz(), _sz()
        rp, ci, v = _szp(), _i32p(), _dp()
        _ck(lib().ref_ops_csr(self.h, C.c_int(s), C.byref(rows), C.byref(nnz), C.byref(rp),
                              C.byref(ci), C.byref(v)))
        r, z = rows.value, nnz.value
        if r == 0:
            return None
        return (np.ctypeslib.as_array(rp, (r + 1,)).astype(np.uint64).copy(),
                np.ctypeslib.as_array(ci, (z,)).copy() if z else np.zeros(0, np.int32),
                np.ctypeslib.as_array(v, (z,)).copy() if z else np.zeros(0))

    def field(self, name):
        data, z = _dp(), C.c_int()
        _ck(lib().ref_ops_field(self.h, C.c_int(FIELD_NAMES.index(name)), C.byref(data),
                                C.byref(z)))
        return np.ctypeslib.as_array(data, (self.n,)).copy(), bool(z.value)

    def diagonals(self, slot):
        out = _sz()
        _ck(lib().ref_ops_diagonals(self.h, C.c_int(SLOTS.index(slot)), C.byref(out)))
        return out.value

    def datum(self):
        out = np.empty(self.n)
        _ck(lib().ref_gaussian_datum(self.h, _d(out)))
        return out

    def nodes(self, axis):
        n = self.nx if axis == 0 else self.nv
        out = np.empty(n)
        v = C.c_double()
        for i in range(n):
            _ck(lib().ref_node(self.h, C.c_int(axis), _sz(i), C.byref(v)))
            out[i] = v.value
        return out

    def fill(self, order, f5, build_order=None):
        """Union CSR of the order-`order` logarithm (MagnusLogBuilder::fill)."""
        bo = self.order if build_order is None else build_order
        f = np.asarray(f5, dtype=np.float64)
        nnz = _sz()
        _ck(lib().ref_magnus_fill(self.h, C.c_int(bo), C.c_int(order), _d(f), C.byref(nnz),
                                  None, None, None))
        rp = np.empty(self.n + 1, np.uint64)
        ci = np.empty(nnz.value, np.int32)
        v = np.empty(nnz.value)
        _ck(lib().ref_magnus_fill(self.h, C.c_int(bo), C.c_int(order), _d(f), C.byref(nnz),
                                  rp.ctypes.data_as(_szp), ci.ctypes.data_as(_i32p), _d(v)))
        return rp, ci, v

    # -- solvers -------------------------------------------------------------------
    def solve_magnus(self, values, dt_leb, T, dt, order=None, tol=1e-10, theta=1.0, cap=1e10,
                     threads=0, record_times=(), seed=1, phi=None, adaptive=None):
        values = np.ascontiguousarray(values, dtype=np.float64)
        M, steps = values.shape[0], values.shape[1] - 1
        phi = self.datum() if phi is None else np.ascontiguousarray(phi, dtype=np.float64)
        rec = np.asarray(record_times, dtype=np.float64)
        R = len(rec) + 1
        states = np.empty((R, M, self.n))
        status = np.empty((R, M), np.uint8)
        secs = np.empty(M)
        nrec = _sz()
        ad = adaptive or {}
        _ck(lib().ref_solve_magnus(
            self.h, C.c_int(order or self.order), C.c_double(dt), C.c_double(tol),
            C.c_double(theta), C.c_double(cap), C.c_int(threads), C.c_int(1 if adaptive else 0),
            C.c_double(ad.get("tolerance", 1e-4)), C.c_double(ad.get("shrink", 0.5)),
            _d(rec) if len(rec) else None, _sz(len(rec)), _d(phi), _d(values), _sz(M), _sz(steps),
            C.c_double(dt_leb), C.c_uint64(seed), C.c_double(T), C.byref(nrec), _d(states),
            status.ctypes.data_as(_u8p), _d(secs)))
        r = nrec.value
        return states[:r], status[:r], secs

    def solve_euler(self, values, dt_leb, T, dt, threads=0, record_times=(), seed=1, phi=None):
        values = np.ascontiguousarray(values, dtype=np.float64)
        M, steps = values.shape[0], values.shape[1] - 1
        phi = self.datum() if phi is None else np.ascontiguousarray(phi, dtype=np.float64)
        rec = np.asarray(record_times, dtype=np.float64)
        R = len(rec) + 1
        states = np.empty((R, M, self.n))
        status = np.empty((R, M), np.uint8)
        secs = np.empty(M)
        nrec = _sz()
        _ck(lib().ref_solve_euler(
            self.h, C.c_double(dt), C.c_int(threads), _d(rec) if len(rec) else None,
            _sz(len(rec)), _d(phi), _d(values), _sz(M), _sz(steps), C.c_double(dt_leb),
            C.c_uint64(seed), C.c_double(T), C.byref(nrec), _d(states),
            status.ctypes.data_as(_u8p), _d(secs)))
        r = nrec.value
        return states[:r], status[:r], secs

    def euler_step(self, u, dW, dt):
        u = np.ascontiguousarray(u, dtype=np.float64)
        out = np.empty(self.n)
        mx = C.c_double()
        _ck(lib().ref_euler_step(self.h, _d(u), C.c_double(dW), C.c_double(dt), _d(out),
                                 C.byref(mx)))
        return out, mx.value

    def exact_reference(self, values, dt_leb, t, seed=1):
        values = np.ascontiguousarray(values, dtype=np.float64)
        M, steps = values.shape[0], values.shape[1] - 1
        out = np.empty((M, self.n))
        _ck(lib().ref_exact_reference(self.h, C.c_double(t), C.c_double(self.a),
                                      C.c_double(self.sigma), _d(values), _sz(M), _sz(steps),
                                      C.c_double(dt_leb), C.c_uint64(seed), _d(out)))
        return out

    def exact_field(self, t, W, IW, a=None, sigma=None):
        out = np.empty(self.n)
        _ck(lib().ref_exact_field(self.h, C.c_double(t), C.c_double(self.a if a is None else a),
                                  C.c_double(self.sigma if sigma is None else sigma),
                                  C.c_double(W), C.c_double(IW), _d(out)))
        return out

    def errors(self, kappa, ref_states, app_states, app_status=None, ref_status=None, seed=1):
        ref_states = np.ascontiguousarray(ref_states, dtype=np.float64)
        app_states = np.ascontiguousarray(np.nan_to_num(app_states), dtype=np.float64)
        M = ref_states.shape[0]
        lo, hi = central_region(self.nx, kappa)
        w = hi - lo + 1
        me = np.empty(w * w)
        err, ame = C.c_double(), C.c_double()
        bl, ex = _sz(), _sz()
        ast = None if app_status is None else np.ascontiguousarray(app_status, np.uint8)
        rst = None if ref_status is None else np.ascontiguousarray(ref_status, np.uint8)
        _ck(lib().ref_errors(self.h, C.c_int(kappa), _d(ref_states),
                             rst.ctypes.data_as(_u8p) if rst is not None else None,
                             _d(app_states), ast.ctypes.data_as(_u8p) if ast is not None else None,
                             _sz(M), C.c_uint64(seed), C.byref(err), C.byref(bl), C.byref(ame),
                             C.byref(ex), _d(me)))
        return {"err": err.value, "blowups": bl.value, "ame": ame.value, "excluded": ex.value,
                "me": me.reshape(w, w)}


def simulate_brownian(T, dt_leb, M, seed):
    """Prefix values [M][steps+1] and increments [M][steps] (stochastics.cpp:76-101)."""
    steps = int(round(T / dt_leb))
    values = np.empty((M, steps + 1))
    inc = np.empty((M, steps))
    st = _sz()
    _ck(lib().ref_simulate_brownian(C.c_double(T), C.c_double(dt_leb), _sz(M), C.c_uint64(seed),
                                    C.byref(st), _d(values), _d(inc)))
    assert st.value == steps
    return values, inc


def functionals(path, k0, k1, dt_leb):
    p = np.ascontiguousarray(path, dtype=np.float64)
    out = np.empty(5)
    _ck(lib().ref_functionals(_d(p), _sz(len(p)), _sz(k0), _sz(k1), C.c_double(dt_leb), _d(out)))
    return out


def one_norm(rp, ci, v):
    n = len(rp) - 1
    out = C.c_double()
    rp = np.ascontiguousarray(rp, np.uint64)
    ci = np.ascontiguousarray(ci, np.int32)
    v = np.ascontiguousarray(v, np.float64)
    _ck(lib().ref_one_norm(_sz(n), rp.ctypes.data_as(_szp), ci.ctypes.data_as(_i32p), _d(v),
                           C.byref(out)))
    return out.value


def expmv(rp, ci, v, x, tol=1e-10, theta=1.0):
    n = len(rp) - 1
    rp = np.ascontiguousarray(rp, np.uint64)
    ci = np.ascontiguousarray(ci, np.int32)
    v = np.ascontiguousarray(v, np.float64)
    x = np.ascontiguousarray(x, np.float64)
    y = np.empty(n)
    st, seg, mt = C.c_int(), C.c_int(), C.c_int()
    res = C.c_double()
    _ck(lib().ref_expmv(_sz(n), rp.ctypes.data_as(_szp), ci.ctypes.data_as(_i32p), _d(v), _d(x),
                        C.c_double(tol), C.c_double(theta), _d(y), C.byref(st), C.byref(res),
                        C.byref(seg), C.byref(mt)))
    return y, {"status": st.value, "residual": res.value, "segments": seg.value,
               "max_terms": mt.value}


def central_region(d, kappa):
    lo, hi = _sz(), _sz()
    _ck(lib().ref_central_region(_sz(d), C.c_int(kappa), C.byref(lo), C.byref(hi)))
    return lo.value, hi.value
