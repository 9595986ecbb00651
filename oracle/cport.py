"""ctypes binding of the C restatement (oracle/c/bx_oracle.c).

TEST INFRASTRUCTURE / CPU BASELINE ONLY (see oracle/__init__.py).  Arrays are
row-aligned, system-major (B, n) float64, C-contiguous.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
SRC = os.path.join(HERE, "c", "bx_oracle.c")
_lib = None


def build():
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.run(["make", "-s", "-C", HERE, "liboracle.so"], check=True)
    return LIB


def set_threads(n):
    """OpenMP threads of the C restatement's timed sections."""
    lib().ox_set_threads(int(n))


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(LIB)
        p = C.c_void_p
        i64 = C.c_int64
        _lib.ox_threads.restype = C.c_int
        _lib.ox_set_threads.argtypes = [C.c_int]
        _lib.ox_ntdm.argtypes = [p] * 7 + [i64] * 3
        _lib.ox_penta.argtypes = [C.c_int] + [p] * 10 + [i64] * 3
        _lib.ox_sip.argtypes = [p] * 14 + [i64] * 4 + [C.c_double, i64]
    return _lib


def _c(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a):
    return None if a is None else a.ctypes.data


def rowaligned_tri(sub1, main, sup1):
    bsz, n = main.shape
    d = np.zeros((bsz, n)); d[:, 1:] = sub1
    f = np.zeros((bsz, n)); f[:, :n - 1] = sup1
    return d, _c(main), f


def rowaligned_penta(sub2, sub1, main, sup1, sup2, m=2):
    bsz, n = main.shape
    c = np.zeros((bsz, n)); c[:, m:] = sub2
    d = np.zeros((bsz, n)); d[:, 1:] = sub1
    f = np.zeros((bsz, n)); f[:, :n - 1] = sup1
    g = np.zeros((bsz, n)); g[:, :n - m] = sup2
    return c, d, _c(main), f, g


def ntdm(d, e, f, b):
    """Row-aligned inputs -> (x, status, index)."""
    d, e, f, b = map(_c, (d, e, f, b))
    bsz, n = e.shape
    x = np.empty((bsz, n)); st = np.empty(bsz, np.int32); ix = np.empty(bsz, np.int32)
    lib().ox_ntdm(_p(d), _p(e), _p(f), _p(b), _p(x), _p(st), _p(ix), bsz, n, n)
    return x, st, ix


def penta(mod, c, d, e, f, g, b):
    c, d, e, f, g, b = map(_c, (c, d, e, f, g, b))
    bsz, n = e.shape
    x = np.empty((bsz, n)); st = np.empty(bsz, np.int32); ix = np.empty(bsz, np.int32)
    nz = np.empty(bsz, np.int64)
    lib().ox_penta(int(mod), _p(c), _p(d), _p(e), _p(f), _p(g), _p(b), _p(x), _p(st), _p(ix),
                   _p(nz), bsz, n, n)
    return x, st, ix, nz


def sip(c, d, e, f, g, b, tol, m=2, alpha=0.0, max_iter=500):
    c, d, e, f, g, b = map(_c, (c, d, e, f, g, b))
    bsz, n = e.shape
    tol = np.ascontiguousarray(np.broadcast_to(np.asarray(tol, np.float64), (bsz,)))
    x = np.empty((bsz, n)); bx = np.empty((bsz, n))
    it = np.empty(bsz, np.int64); res = np.empty(bsz); bres = np.empty(bsz)
    st = np.empty(bsz, np.int32); ix = np.empty(bsz, np.int32)
    lib().ox_sip(_p(c), _p(d), _p(e), _p(f), _p(g), _p(b), _p(tol), _p(x), _p(bx), _p(it),
                 _p(res), _p(bres), _p(st), _p(ix), bsz, n, n, m, float(alpha), max_iter)
    return dict(x=x, best_x=bx, iterations=it, residual=res, best_residual=bres, status=st,
                index=ix)


def threads():
    return lib().ox_threads()
