"""ctypes binding of the C ABI in include/spde2d_b200.h.

Loads the in-tree ``paper_2207_09776_b200/lib/libspde2d_b200.so`` (built by
``__graft_entry__.build()`` / ``make -C paper_2207_09776_b200/csrc``).  There
is no fallback: if the library is missing or no B200 is visible, calls fail
loudly.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libspde2d_b200.so")

OK, ERR_CONFIG, ERR_DIMENSION, ERR_EXPMV, ERR_RUNTIME, ERR_CUDA = range(6)


class Grid(C.Structure):
    _fields_ = [("ax", C.c_double), ("bx", C.c_double), ("nx", C.c_size_t),
                ("av", C.c_double), ("bv", C.c_double), ("nv", C.c_size_t)]


class Csr(C.Structure):
    _fields_ = [("rows", C.c_size_t), ("row_ptr", C.POINTER(C.c_size_t)),
                ("col_idx", C.POINTER(C.c_int32)), ("values", C.POINTER(C.c_double))]


class MagnusConfig(C.Structure):
    _fields_ = [("order", C.c_int), ("dt", C.c_double), ("T", C.c_double),
                ("expmv_tol", C.c_double), ("expmv_theta", C.c_double),
                ("blowup_norm_cap", C.c_double), ("record_times", C.POINTER(C.c_double)),
                ("n_record", C.c_size_t)]


class AdaptiveConfig(C.Structure):
    _fields_ = [("enabled", C.c_int), ("tolerance", C.c_double), ("shrink", C.c_double)]


class EulerConfig(C.Structure):
    _fields_ = [("dt", C.c_double), ("T", C.c_double), ("record_times", C.POINTER(C.c_double)),
                ("n_record", C.c_size_t)]


class ErrorStats(C.Structure):
    _fields_ = [("err", C.c_double), ("blowups", C.c_size_t), ("ame", C.c_double),
                ("excluded", C.c_size_t), ("sum_rel", C.c_double), ("used", C.c_size_t),
                ("region_lo", C.c_size_t), ("region_hi", C.c_size_t)]


class MagnusStats(C.Structure):
    _fields_ = [("passes", C.c_int64), ("path_terms", C.c_int64), ("path_windows", C.c_int64),
                ("term_launches", C.c_int64), ("term_kernel_ms", C.c_double),
                ("gridpoints", C.c_double), ("path_segments", C.c_int64),
                ("engine", C.c_int32), ("hybrid_paths", C.c_int64)]


class ExpmvReport(C.Structure):
    _fields_ = [("status", C.c_int), ("residual", C.c_double), ("segments", C.c_int),
                ("max_terms", C.c_int), ("terms", C.c_int64)]


class OperatorSpec(C.Structure):
    _fields_ = [("family", C.c_int), ("a", C.c_double), ("sigma", C.c_double),
                ("fields9", C.POINTER(C.POINTER(C.c_double))), ("order", C.c_int)]


class MultiStats(C.Structure):
    _fields_ = [("errors", ErrorStats), ("path_terms", C.c_int64), ("path_windows", C.c_int64),
                ("max_solve_ms", C.c_double), ("M_total", C.c_size_t), ("devices", C.c_int),
                ("nccl", C.c_int)]


# Exported symbols with their ctypes signatures (restype int unless noted).
_VP = C.c_void_p
_P = C.POINTER
SIGNATURES = {
    "s2b_last_error": (C.c_char_p, []),
    "s2b_version": (C.c_char_p, []),
    "s2b_context_create": (C.c_int, [C.c_int, _P(_VP)]),
    "s2b_context_destroy": (C.c_int, [_VP]),
    "s2b_context_synchronize": (C.c_int, [_VP]),
    "s2b_context_stream": (_VP, [_VP]),
    "s2b_context_launches": (C.c_int64, [_VP]),
    "s2b_operator_create": (C.c_int, [_VP, _P(Grid), C.c_int, _P(Csr), _P(_VP)]),
    "s2b_operator_build": (C.c_int, [_VP, _P(Grid), C.c_int, C.c_double, C.c_double,
                                     _P(_P(C.c_double)), C.c_int, _P(_VP)]),
    "s2b_operator_info": (C.c_int, [_VP, _P(C.c_int64)]),
    "s2b_operator_destroy": (C.c_int, [_VP]),
    "s2b_fields_create": (C.c_int, [_VP, _P(Grid), _P(_P(C.c_double)), _P(_VP)]),
    "s2b_fields_build": (C.c_int, [_VP, _P(Grid), C.c_int, C.c_double, C.c_double, _P(_VP)]),
    "s2b_fields_destroy": (C.c_int, [_VP]),
    "s2b_gaussian_datum": (C.c_int, [_P(Grid), _P(C.c_double)]),
    "s2b_host_ops_build": (C.c_int, [_P(Grid), C.c_int, C.c_double, C.c_double,
                                     _P(_P(C.c_double)), C.c_int, _P(_VP)]),
    "s2b_host_ops_csr": (C.c_int, [_VP, C.c_int, _P(Csr)]),
    "s2b_host_ops_field": (C.c_int, [_VP, C.c_int, _P(_P(C.c_double)), _P(C.c_int)]),
    "s2b_host_ops_destroy": (C.c_int, [_VP]),
    "s2b_host_simulate_brownian": (C.c_int, [C.c_double, C.c_double, C.c_size_t, C.c_uint64,
                                             _P(C.c_double)]),
    "s2b_paths_create_host": (C.c_int, [_VP, C.c_double, C.c_size_t, C.c_size_t, C.c_uint64,
                                        _P(C.c_double), _P(_VP)]),
    "s2b_paths_create_philox": (C.c_int, [_VP, C.c_double, C.c_size_t, C.c_size_t, C.c_uint64,
                                          C.c_uint64, _P(_VP)]),
    "s2b_paths_download": (C.c_int, [_VP, _P(C.c_double)]),
    "s2b_paths_upload": (C.c_int, [_VP, C.c_size_t, C.c_size_t, _P(C.c_double)]),
    "s2b_paths_destroy": (C.c_int, [_VP]),
    "s2b_solve_magnus": (C.c_int, [_VP, _VP, _P(MagnusConfig), _P(C.c_double), _VP, _P(_VP),
                                   _P(MagnusStats)]),
    "s2b_solve_euler": (C.c_int, [_VP, _VP, _P(EulerConfig), _P(C.c_double), _VP, _P(_VP)]),
    "s2b_solve_magnus_sweep": (C.c_int, [_VP, _VP, _P(MagnusConfig), C.c_size_t, _P(C.c_double), _VP, _P(_VP),
                                         _P(MagnusStats)]),
    "s2b_solve_adaptive_magnus": (C.c_int, [_VP, _VP, _P(MagnusConfig), _P(AdaptiveConfig), _P(C.c_double),
                                            _VP, _P(_VP), _P(MagnusStats)]),
    "s2b_magnus_session_create": (C.c_int, [_VP, _VP, _P(MagnusConfig), _P(C.c_double), _VP,
                                            _P(_VP)]),
    "s2b_magnus_session_advance": (C.c_int, [_VP, C.c_size_t]),
    "s2b_magnus_session_reset": (C.c_int, [_VP]),
    "s2b_magnus_session_stats": (C.c_int, [_VP, _P(MagnusStats)]),
    "s2b_magnus_session_set_timing": (C.c_int, [_VP, C.c_int]),
    "s2b_magnus_session_ensemble": (C.c_int, [_VP, _P(_VP)]),
    "s2b_magnus_session_finish": (C.c_int, [_VP, _P(_VP)]),
    "s2b_magnus_session_moments": (C.c_int, [_VP, _P(C.c_double), _P(C.c_double)]),
    "s2b_magnus_session_destroy": (C.c_int, [_VP]),
    "s2b_ensemble_create_host": (C.c_int, [_VP, _P(Grid), C.c_double, C.c_uint64, C.c_size_t,
                                           _P(C.c_double), _P(C.c_uint8), _P(_VP)]),
    "s2b_ensemble_info": (C.c_int, [_VP, _P(C.c_int64), _P(C.c_double)]),
    "s2b_ensemble_download": (C.c_int, [_VP, C.c_size_t, _P(C.c_double), _P(C.c_uint8)]),
    "s2b_ensemble_counters": (C.c_int, [_VP, _P(C.c_int64), _P(C.c_int64)]),
    "s2b_ensemble_destroy": (C.c_int, [_VP]),
    "s2b_exact_reference": (C.c_int, [_VP, _P(Grid), C.c_double, C.c_double, C.c_double, _VP,
                                      _P(_VP)]),
    "s2b_exact_field": (C.c_int, [_VP, _P(Grid), C.c_double, C.c_double, C.c_double, C.c_double,
                                  C.c_double, _P(C.c_double)]),
    "s2b_errors": (C.c_int, [_VP, _VP, C.c_size_t, _VP, C.c_size_t, C.c_int, _P(ErrorStats),
                             _P(C.c_double)]),
    "s2b_exact_errors": (C.c_int, [_VP, _VP, C.c_size_t, C.c_double, C.c_double, _VP, C.c_int,
                                   _P(ErrorStats), _P(C.c_double), _P(C.c_double),
                                   _P(C.c_double)]),
    "s2b_expmv": (C.c_int, [_VP, _P(Csr), _P(C.c_double), C.c_double, C.c_double,
                            _P(C.c_double), _P(C.c_int)]),
    "s2b_context_kernel_names": (C.c_int, [_VP, C.c_char_p, C.c_char_p, C.c_size_t]),
    "s2b_context_em_kernel_name": (C.c_int, [_VP, C.c_char_p, C.c_size_t]),
    "s2b_host_ops_assemble_device": (C.c_int, [_VP, _P(Grid), C.c_int, C.c_double, C.c_double,
                                               _P(_P(C.c_double)), C.c_int, _P(_VP)]),
    "s2b_operator_build_device": (C.c_int, [_VP, _P(Grid), C.c_int, C.c_double, C.c_double,
                                            _P(_P(C.c_double)), C.c_int, _P(_VP)]),
    "s2b_ensemble_moments": (C.c_int, [_VP, C.c_size_t, _P(C.c_double), _P(C.c_size_t)]),
    "s2b_shard": (C.c_int, [C.c_size_t, C.c_int, C.c_int, _P(C.c_size_t), _P(C.c_size_t)]),
    "s2b_multi_create": (C.c_int, [_P(C.c_int), C.c_int, _P(_VP)]),
    "s2b_multi_destroy": (C.c_int, [_VP]),
    "s2b_multi_info": (C.c_int, [_VP, _P(C.c_int)]),
    "s2b_multi_solve_magnus": (C.c_int, [_VP, _P(Grid), _P(OperatorSpec), _P(MagnusConfig), _P(C.c_double),
                                         C.c_double, C.c_size_t, C.c_size_t, C.c_uint64, C.c_int,
                                         _P(MultiStats), _P(C.c_double), _P(C.c_double), _P(C.c_double)]),
    "s2b_multi_solve_euler": (C.c_int, [_VP, _P(Grid), _P(OperatorSpec), _P(EulerConfig), _P(C.c_double),
                                        C.c_double, C.c_size_t, C.c_size_t, C.c_uint64, C.c_int,
                                        _P(MultiStats), _P(C.c_double), _P(C.c_double), _P(C.c_double)]),
    "s2b_expmv_workspace_create": (C.c_int, [_VP, _P(_VP)]),
    "s2b_expmv_workspace_destroy": (C.c_int, [_VP]),
    "s2b_expmv_into": (C.c_int, [_VP, _P(Csr), _P(C.c_double), C.c_double, C.c_double,
                                 _P(C.c_double), _P(ExpmvReport)]),
    "s2b_expmv_into_device": (C.c_int, [_VP, _P(Csr), C.c_void_p, C.c_double, C.c_double,
                                        C.c_void_p, _P(ExpmvReport)]),
    "s2b_euler_step": (C.c_int, [_VP, _P(C.c_double), _P(C.c_double), _P(C.c_double), C.c_double,
                                 C.c_double, _P(C.c_double)]),
    "s2b_euler_step_device": (C.c_int, [_VP, _P(C.c_double), C.c_void_p, C.c_void_p, C.c_size_t,
                                        _P(C.c_double), C.c_double, _P(C.c_double)]),
}

_lib = None


class LibraryMissing(RuntimeError):
    pass


def lib():
    """The loaded C ABI.  Raises if the in-tree library was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise LibraryMissing(
                f"{LIB_PATH} not found: build it with __graft_entry__.build() "
                "(make -C paper_2207_09776_b200/csrc); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def exported_symbols():
    return list(SIGNATURES)
