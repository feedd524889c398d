"""ctypes binding of libinvaskit.so (declared in include/invaskit.h).

The library is built in-tree for sm_100a (`make`, or `__graft_entry__.build()`).
There is no CPU fallback: if the shared library is missing or fails to load,
importing the solver raises immediately.
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libinvaskit.so")

(KS_OK, KS_ERR_INVALID, KS_ERR_NOT_SPD, KS_ERR_SINGULAR, KS_ERR_ILL_COND, KS_ERR_CUDA, KS_ERR_UNSUPPORTED,
 KS_ERR_IO) = range(8)

_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)


class KsProblem(C.Structure):
    _fields_ = [
        ("n", C.c_int64),
        ("d", C.c_int64),
        ("coords", _f64p),
        ("perm", _i64p),
        ("n_nodes", C.c_int64),
        ("node_begin", _i64p),
        ("node_end", _i64p),
        ("node_left", _i64p),
        ("node_right", _i64p),
        ("rank", _i64p),
        ("skel_off", _i64p),
        ("skel", _i64p),
        ("coeff_off", _i64p),
        ("coeff", _f64p),
        ("bandwidth", C.c_double),
    ]


class KsDiag(C.Structure):
    _fields_ = [
        ("cholesky_fallbacks", C.c_int64),
        ("n_z_cond", C.c_int64),
        ("n_warnings", C.c_int64),
        ("error_node", C.c_int64),
        ("error_cond", C.c_double),
        ("max_z_cond", C.c_double),
    ]


# every entry point include/invaskit.h declares: name -> (restype, argtypes)
SIGNATURES = {
    "ks_create": (C.c_int, [C.POINTER(KsProblem), C.c_int, C.POINTER(C.c_void_p)]),
    "ks_factorize": (C.c_int, [C.c_void_p, C.c_double, C.c_void_p]),
    "ks_solve": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "ks_create_shard": (C.c_int, [C.POINTER(KsProblem), C.c_int, C.c_int64, C.POINTER(C.c_void_p)]),
    "ks_factorize_top": (C.c_int, [C.c_void_p, C.c_void_p]),
    "ks_solve_up": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "ks_solve_top": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p]),
    "ks_solve_down": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "ks_node_exchange": (C.c_int, [C.c_void_p, C.c_int, C.c_int64, C.c_void_p, C.c_int64, C.c_int, C.c_void_p]),
    "ks_shard_info": (C.c_int, [C.c_void_p, _i64p, C.c_int64]),
    "ks_matvec": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "ks_kernel_matvec": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int64, C.c_double, C.c_void_p,
                                   C.c_void_p, C.c_int, C.c_void_p]),
    "ks_save_problem": (C.c_int, [C.POINTER(KsProblem), C.c_char_p]),
    "ks_load_problem": (C.c_int, [C.c_char_p, C.POINTER(KsProblem), C.POINTER(C.c_void_p)]),
    "ks_free_problem": (C.c_int, [C.c_void_p]),
    "ks_save_factor": (C.c_int, [C.c_void_p, C.POINTER(KsProblem), C.c_char_p]),
    "ks_load_factor": (C.c_int, [C.c_char_p, C.POINTER(KsProblem), C.c_int, C.POINTER(C.c_void_p)]),
    "ks_get_diag": (C.c_int, [C.c_void_p, C.POINTER(KsDiag)]),
    "ks_get_lam": (C.c_int, [C.c_void_p, C.POINTER(C.c_double)]),
    "ks_get_z_cond": (C.c_int64, [C.c_void_p, _i64p, _f64p, C.c_int64]),
    "ks_get_fallback_nodes": (C.c_int64, [C.c_void_p, _i64p, C.c_int64]),
    "ks_get_node_h": (C.c_int, [C.c_void_p, C.c_int64, _f64p]),
    "ks_get_leaf_factor": (C.c_int, [C.c_void_p, C.c_int64, _f64p]),
    "ks_device_bytes": (C.c_int64, [C.c_void_p]),
    "ks_upload_bytes": (C.c_int64, [C.c_void_p]),
    "ks_set_profiling": (C.c_int, [C.c_void_p, C.c_int]),
    "ks_get_phase_ms": (C.c_int, [C.c_void_p, _f64p, C.c_int]),
    "ks_get_level_ms": (C.c_int, [C.c_void_p, _f64p, C.c_int]),
    "ks_pipelined_levels": (C.c_int, [C.c_void_p, C.POINTER(C.c_int)]),
    "ks_trace_report": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int64]),
    "ks_last_launches": (C.c_int64, [C.c_void_p, C.c_int]),
    "ks_debug_copy": (C.c_int, [C.c_void_p, C.c_int, C.c_int64, _f64p, C.c_int64]),
    "ks_debug_layout": (C.c_int, [C.c_void_p, _i64p]),
    "ks_debug_ptr": (C.c_int64, [C.c_void_p, C.c_int]),
    "ks_test_gemm": (C.c_int, [C.c_int] * 5 + [C.c_void_p] * 3 + [C.c_int64] * 6
                     + [C.c_double, C.c_double, C.c_int, C.c_int, C.c_void_p]),
    "ks_test_gemm_cidx": (C.c_int, [C.c_int] * 4 + [C.c_void_p] * 4 + [C.c_int64] * 6 + [C.c_int, C.c_int, C.c_void_p]),
    "ks_destroy": (None, [C.c_void_p]),
    "ks_trim_pool": (C.c_int, [C.c_int]),
    "ks_last_error": (C.c_int, [C.c_char_p, C.c_int64]),
    "ks_version": (C.c_char_p, []),
}

_lib = None


def load() -> C.CDLL:
    """Load libinvaskit.so (raises OSError if it is missing: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise OSError(f"{LIB_PATH} is missing; build it with `make` (sm_100a CUDA library, no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    lib = load()
    buf = C.create_string_buffer(1024)
    lib.ks_last_error(buf, len(buf))
    return buf.value.decode(errors="replace")
