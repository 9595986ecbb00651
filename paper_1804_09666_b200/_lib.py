"""ctypes binding of libbandix_b200.so (the C ABI in include/bandix_b200.h).

There is no CPU fallback: if the library is missing or CUDA is unavailable,
every solver raises.  Build with ``python -m paper_1804_09666_b200.build``.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import CudaError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BX_LIB") or os.path.join(_HERE, "libbandix_b200.so")  # BX_LIB: dev A/B

BX_OK = 0
LAYOUT_INTERLEAVED = 0
LAYOUT_SYSTEM_MAJOR = 1
ALGO_SEQUENTIAL = 0
ALGO_PARTITIONED = 1
SOLVER = {"ntdm": 0, "npdm": 1, "mnpdm": 2, "stdm": 3, "spdm": 4, "sip": 5, "hb": 6, "pd2td": 7}

_p = C.c_void_p
_i64 = C.c_int64
_i32 = C.c_int32
_sz = C.c_size_t

_SIGS = {
    "bx_version": ([], C.c_char_p),
    "bx_last_error": ([], C.c_char_p),
    "bx_workspace_bytes": ([_i32, _i64, _i64, _i32, _i32], _sz),
    "bx_sip_workspace_bytes": ([_i64, _i64, _i64], _sz),
    "bx_ntdm_f64": ([_p] * 7 + [_i64, _i64, _i64, _i32, _i32, _p, _sz, _p], C.c_int),
    "bx_npdm_f64": ([_p] * 9 + [_i64, _i64, _i64, _i32, _i32, _p, _sz, _p], C.c_int),
    "bx_mnpdm_f64": ([_p] * 10 + [_i64, _i64, _i64, _i32, _i32, _p, _sz, _p], C.c_int),
    "bx_residual_inf_f64": ([_i32] + [_p] * 8 + [_i64, _i64, _i64, _i32, _p], C.c_int),
    "bx_band_matvec_f64": ([_i32, _i64] + [_p] * 8 + [_i64, _i64, _i64, _i32, _p], C.c_int),
    "bx_lu_penta_f64": ([_p] * 12 + [_i64, _i64, _i64, _i32, _p], C.c_int),
    "bx_forward_sub_f64": ([_i64] + [_p] * 4 + [_i64, _i64, _i64, _i32, _p], C.c_int),
    "bx_backward_sub_f64": ([_i64] + [_p] * 7 + [_i64, _i64, _i64, _i32, _p], C.c_int),
    "bx_pd2td_f64": ([_p] * 13 + [_i64, _i64, _i64, _i64, _i32, _p], C.c_int),
    "bx_pd2td_ntdm_f64": ([_p] * 10 + [_i64, _i64, _i64, _i32, _p, _sz, _p], C.c_int),
    "bx_stdm_f64": ([_p] * 8 + [_i64, _i64, _i64, _i32, _p, _sz, _p], C.c_int),
    "bx_spdm_f64": ([_p] * 10 + [_i64, _i64, _i64, _i32, _p, _sz, _p], C.c_int),
    "bx_det_band_f64": ([_i32] + [_p] * 10 + [_i64, _i64, _i64, _i32, _p], C.c_int),
    "bx_hb_banded_workspace_bytes": ([_i64, _i64, _i64], _sz),
    "bx_hb_invert_banded_f64": ([_p] * 5 + [_i32, _i64, _p, _i64] + [_p] * 6
                                + [_i64, _i64, _i64, _i32, _p, _sz, _p], C.c_int),
    "bx_sip_hb_banded_f64": ([_p] * 15 + [_i64, _i64] + [_p] * 4
                             + [_i64, _i64, _i64, _i64, _i32, _i64, _i32, _p, _sz, _p], C.c_int),
    "bx_rcond_workspace_bytes": ([_i32, _i64, _i64], _sz),
    "bx_rcond_band_f64": ([_i32] + [_p] * 8 + [_i64, _i64, _i64, _i32, _p, _sz, _p], C.c_int),
    "bx_outer_compact_f64": ([_p] * 6 + [_i64, _i64, _i64, _i64, _i32, _p], C.c_int),
    "bx_mnpdm_sparse_f64": ([_p] * 3 + [_i64] + [_p] * 8 + [_i64, _i64, _i64, _i32, _p], C.c_int),
    "bx_transpose_f64": ([_p, _p] + [_i64] * 7 + [_p], C.c_int),
    "bx_hb_workspace_bytes": ([_i64, _i64], _sz),
    "bx_hb_invert_dense_workspace_bytes": ([_i64, _i64], _sz),
    "bx_hb_invert_dense_f64": ([_p, _i64, _i64, _i64, _i64, _p, _i64, _p, _i64, _i64] + [_p] * 6
                               + [_sz, _p], C.c_int),
    "bx_hb_invert_f64": ([_p] * 12 + [_i64, _i64, _i64, C.c_double, _i64, _i64, _i32, _p, _sz, _p],
                         C.c_int),
    "bx_sip_hb_f64": ([_p] * 17 + [_i64, _i64, _i64, C.c_double, _i64, _i64, _i32, _i64, _i32, _p,
                                   _sz, _p], C.c_int),
    "bx_ilu0_f64": ([_p] * 19 + [_i64, _i64, _i64, C.c_double, _i64, _i32, _p, _sz, _p], C.c_int),
    "bx_sip_f64": ([_p] * 15 + [_i64, _i64, _i64, C.c_double, _i64, _i32, _i64, _i32, _i32, _p,
                                _sz, _p], C.c_int),
}

_lib = None


def lib():
    """Load (once) and return the CDLL; raises if it is not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise CudaError(f"{LIB_PATH} is missing: build it with "
                            "`python -m paper_1804_09666_b200.build` (no CPU fallback exists)")
        h = C.CDLL(LIB_PATH)
        for name, (args, res) in _SIGS.items():
            fn = getattr(h, name, None)
            if fn is None:
                continue
            fn.argtypes = args
            fn.restype = res
        _lib = h
    return _lib


def exported_symbols():
    return list(_SIGS)


def check(rc, what):
    if rc != BX_OK:
        msg = lib().bx_last_error().decode(errors="replace")
        raise CudaError(f"{what} failed (rc={rc}): {msg}")


def call(name, *args):
    check(getattr(lib(), name)(*args), name)
