"""Batched restatement of the reference's direct solvers (NTDM, NPDM, MNPDM).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Arrays are batched along axis 0 and keep the reference's per-diagonal
lengths (core.py:117-152): for a pentadiagonal system of order n,
``sub2 (B,n-2), sub1 (B,n-1), main (B,n), sup1 (B,n-1), sup2 (B,n-2)``;
row i uses ``sub2[i-2], sub1[i-1], main[i], sup1[i], sup2[i]``
(core.py:157-164).  Every elementwise numpy operation is one IEEE binary64
rounding, exactly like the CPython float arithmetic of ``_elim.py``; the
operation order below follows the reference line by line, so results are
bit-identical (asserted against reference-generated golden vectors in
``tests/test_oracle_golden.py``).

Failure semantics: where the reference raises ``ZeroPivot(i)`` at the first
exactly-zero pivot (``_elim.py:26-27``) the batched oracle records
``status[s] = STATUS_ZERO_PIVOT``, ``index[s] = i`` and fills ``x[s]`` with
NaN.
"""

from __future__ import annotations

import numpy as np

from . import STATUS_OK, STATUS_REDUCTION_PIVOT, STATUS_ZERO_PIVOT


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class _PivotTracker:
    def __init__(self, batch):
        self.status = np.full(batch, STATUS_OK, dtype=np.int32)
        self.index = np.full(batch, -1, dtype=np.int32)

    def check(self, i, pivot):
        hit = (pivot == 0.0) & (self.status == STATUS_OK)
        if hit.any():
            self.status[hit] = STATUS_ZERO_PIVOT
            self.index[hit] = i

    def finish(self, x):
        bad = self.status != STATUS_OK
        if bad.any():
            x[bad] = np.nan
        return x


def ntdm(sub1, main, sup1, rhs):
    """Thomas with reciprocal pivots: ``tri_factor_recip`` + ``tri_solve_recip``
    (_elim.py:90-122) as called by ``solve_ntdm`` (direct.py:103-113).

    Returns (x, status, index).
    """
    d, e, f, b = _f64(sub1), _f64(main), _f64(sup1), _f64(rhs)
    bsz, n = e.shape
    trk = _PivotTracker(bsz)
    rec = np.empty((bsz, n))
    low = np.zeros((bsz, n))
    with np.errstate(all="ignore"):
        trk.check(0, e[:, 0])                       # _elim.py:101
        rec[:, 0] = 1.0 / e[:, 0]                   # _elim.py:102
        for i in range(1, n):                       # _elim.py:103-108
            li = d[:, i - 1] * rec[:, i - 1]
            mi = e[:, i] - li * f[:, i - 1]
            low[:, i] = li
            trk.check(i, mi)
            rec[:, i] = 1.0 / mi
        y = np.empty((bsz, n))                      # _elim.py:114-117
        y[:, 0] = b[:, 0]
        for i in range(1, n):
            y[:, i] = b[:, i] - low[:, i] * y[:, i - 1]
        x = np.empty((bsz, n))                      # _elim.py:118-121
        x[:, n - 1] = y[:, n - 1] * rec[:, n - 1]
        for i in range(n - 2, -1, -1):
            x[:, i] = (y[:, i] - f[:, i] * x[:, i + 1]) * rec[:, i]
    return trk.finish(x), trk.status, trk.index


def penta_factor(sub2, sub1, main, sup1, sup2):
    """Banded Doolittle LU, ``penta_factor`` (_elim.py:30-62) with the
    raising zero-pivot policy of ``lu_penta`` (direct.py:42-63).

    Returns row-aligned (mu, l1, l2, phi, psi, status, index); absent slots
    are 0.0 exactly as ``lu_penta`` stores them (direct.py:57-63).
    """
    c, d, e, f, g = _f64(sub2), _f64(sub1), _f64(main), _f64(sup1), _f64(sup2)
    bsz, n = e.shape
    trk = _PivotTracker(bsz)
    mu = np.zeros((bsz, n))
    l1 = np.zeros((bsz, n))
    l2 = np.zeros((bsz, n))
    phi = np.zeros((bsz, n))
    psi = np.zeros((bsz, n))
    with np.errstate(all="ignore"):
        trk.check(0, e[:, 0])
        mu[:, 0] = e[:, 0]                          # _elim.py:44
        phi[:, 0] = f[:, 0]
        psi[:, 0] = g[:, 0]
        l1[:, 1] = d[:, 0] / mu[:, 0]               # _elim.py:47
        m1 = e[:, 1] - l1[:, 1] * phi[:, 0]
        trk.check(1, m1)
        mu[:, 1] = m1
        phi[:, 1] = f[:, 1] - l1[:, 1] * psi[:, 0]  # _elim.py:50
        if n >= 4:
            psi[:, 1] = g[:, 1]
        for i in range(2, n):                       # _elim.py:53-61
            li2 = c[:, i - 2] / mu[:, i - 2]
            li1 = (d[:, i - 1] - li2 * phi[:, i - 2]) / mu[:, i - 1]
            mi = e[:, i] - li2 * psi[:, i - 2] - li1 * phi[:, i - 1]
            l2[:, i] = li2
            l1[:, i] = li1
            trk.check(i, mi)
            mu[:, i] = mi
            if i <= n - 2:
                phi[:, i] = f[:, i] - li1 * psi[:, i - 1]
            if i <= n - 3:
                psi[:, i] = g[:, i]
    return mu, l1, l2, phi, psi, trk.status, trk.index


def penta_forward(l1, l2, rhs):
    """Unit-lower solve, ``penta_forward`` (_elim.py:65-73); l1/l2 row-aligned."""
    b = _f64(rhs)
    bsz, n = b.shape
    y = np.empty((bsz, n))
    with np.errstate(all="ignore"):
        y[:, 0] = b[:, 0]
        y[:, 1] = b[:, 1] - l1[:, 1] * y[:, 0]
        for i in range(2, n):
            y[:, i] = b[:, i] - l1[:, i] * y[:, i - 1] - l2[:, i] * y[:, i - 2]
    return y


def penta_backward(mu, phi, psi, y):
    """Upper solve dividing by the pivots, ``penta_backward`` (_elim.py:76-87)."""
    bsz, n = y.shape
    x = np.empty((bsz, n))
    with np.errstate(all="ignore"):
        x[:, n - 1] = y[:, n - 1] / mu[:, n - 1]
        x[:, n - 2] = (y[:, n - 2] - phi[:, n - 2] * x[:, n - 1]) / mu[:, n - 2]
        for i in range(n - 3, -1, -1):
            x[:, i] = (y[:, i] - phi[:, i] * x[:, i + 1] - psi[:, i] * x[:, i + 2]) / mu[:, i]
    return x


def npdm(sub2, sub1, main, sup1, sup2, rhs):
    """``solve_npdm`` (direct.py:73-81): lu_penta + forward_sub + backward_sub."""
    mu, l1, l2, phi, psi, status, index = penta_factor(sub2, sub1, main, sup1, sup2)
    y = penta_forward(l1, l2, rhs)
    x = penta_backward(mu, phi, psi, y)
    bad = status != STATUS_OK
    x[bad] = np.nan
    return x, status, index


def mnpdm(sub2, sub1, main, sup1, sup2, rhs):
    """``mnpdm_sweep`` (_elim.py:125-190) as called by ``solve_mnpdm``
    (direct.py:84-100).  Returns (x, status, index, nz_sub2)."""
    c, d, e, f, g, b = (_f64(v) for v in (sub2, sub1, main, sup1, sup2, rhs))
    bsz, n = e.shape
    trk = _PivotTracker(bsz)
    rec = np.zeros((bsz, n))
    l1 = np.zeros((bsz, n))
    l2 = np.zeros((bsz, n))
    has2 = np.zeros((bsz, n), dtype=bool)
    phi = np.zeros((bsz, n))
    psi = np.zeros((bsz, n))
    nz = np.zeros(bsz, dtype=np.int64)
    with np.errstate(all="ignore"):
        trk.check(0, e[:, 0])                       # _elim.py:146
        rec[:, 0] = 1.0 / e[:, 0]
        phi[:, 0] = f[:, 0]
        psi[:, 0] = g[:, 0]
        l1[:, 1] = d[:, 0] * rec[:, 0]              # _elim.py:150
        m1 = e[:, 1] - l1[:, 1] * phi[:, 0]
        trk.check(1, m1)
        rec[:, 1] = 1.0 / m1
        phi[:, 1] = f[:, 1] - l1[:, 1] * psi[:, 0]
        if n >= 4:
            psi[:, 1] = g[:, 1]
        for i in range(2, n):                       # _elim.py:158-176
            ci = c[:, i - 2]
            nzc = ci != 0.0
            nz += nzc
            li2 = ci * rec[:, i - 2]
            ti = np.where(nzc, d[:, i - 1] - li2 * phi[:, i - 2], d[:, i - 1])
            li1 = ti * rec[:, i - 1]
            mi = e[:, i] - li1 * phi[:, i - 1]
            mi = np.where(nzc, mi - li2 * psi[:, i - 2], mi)
            trk.check(i, mi)
            l2[:, i] = np.where(nzc, li2, 0.0)
            has2[:, i] = nzc
            l1[:, i] = li1
            rec[:, i] = 1.0 / mi
            if i <= n - 2:
                phi[:, i] = f[:, i] - li1 * psi[:, i - 1]
            if i <= n - 3:
                psi[:, i] = g[:, i]
        y = np.empty((bsz, n))                      # _elim.py:177-184
        y[:, 0] = b[:, 0]
        y[:, 1] = b[:, 1] - l1[:, 1] * y[:, 0]
        for i in range(2, n):
            yi = b[:, i] - l1[:, i] * y[:, i - 1]
            y[:, i] = np.where(has2[:, i], yi - l2[:, i] * y[:, i - 2], yi)
        x = np.empty((bsz, n))                      # _elim.py:185-189
        x[:, n - 1] = y[:, n - 1] * rec[:, n - 1]
        x[:, n - 2] = (y[:, n - 2] - phi[:, n - 2] * x[:, n - 1]) * rec[:, n - 2]
        for i in range(n - 3, -1, -1):
            x[:, i] = (y[:, i] - phi[:, i] * x[:, i + 1] - psi[:, i] * x[:, i + 2]) * rec[:, i]
    return trk.finish(x), trk.status, trk.index, nz


def tri_matvec(sub1, main, sup1, x):
    """Row-fused T @ x, float path of ``tri_matvec`` (core.py:273-284)."""
    x = _f64(x)
    out = _f64(main) * x
    out[:, 1:] += _f64(sub1) * x[:, :-1]
    out[:, :-1] += _f64(sup1) * x[:, 1:]
    return out


def penta_matvec(sub2, sub1, main, sup1, sup2, x):
    """Row-fused A @ x, float path of ``penta_matvec`` (core.py:243-256)."""
    x = _f64(x)
    out = _f64(main) * x
    out[:, 1:] += _f64(sub1) * x[:, :-1]
    out[:, :-1] += _f64(sup1) * x[:, 1:]
    out[:, 2:] += _f64(sub2) * x[:, :-2]
    out[:, :-2] += _f64(sup2) * x[:, 2:]
    return out


def residual_inf_tri(sub1, main, sup1, x, b):
    """``inf_norm(residual(t, x, b))`` per system (core.py:303-321)."""
    with np.errstate(all="ignore"):
        r = _f64(b) - tri_matvec(sub1, main, sup1, x)
        return np.max(np.abs(r), axis=1)


def residual_inf_penta(sub2, sub1, main, sup1, sup2, x, b):
    with np.errstate(all="ignore"):
        r = _f64(b) - penta_matvec(sub2, sub1, main, sup1, sup2, x)
        return np.max(np.abs(r), axis=1)


# closed-form op counters (direct.py:52-53, 98-99, 111-112)
def ops_ntdm(n):
    return {"adds": 0, "subs": 3 * n - 3, "muls": 5 * n - 4, "divs": n}


def ops_npdm(n):
    return {"adds": 0, "subs": (4 * n - 7) + (2 * n - 3) + (2 * n - 3),
            "muls": (4 * n - 7) + (2 * n - 3) + (2 * n - 3),
            "divs": (2 * n - 3) + n}


def ops_mnpdm(n, nz):
    return {"adds": 0, "subs": 5 * n - 7 + 3 * nz, "muls": 7 * n - 8 + 4 * nz, "divs": n}


def pd_to_td(sub2, sub1, main, sup1, sup2, rhs):
    """``pd_to_td`` (direct.py:116-165), batched: sub2 entries eliminated in
    ascending rows against the row above, then sup2 entries in descending rows
    against the row below, each only where the entry is nonzero (is_zero
    skips), with the reference's per-system CounterBox tallies.

    Returns (sub1', main', sup1', rhs', ops (B,3) = muls/subs/divs, status,
    index); a ReductionPivotZero(i) leaves status 8 / index i and NaN rows.
    """
    c, d, e, f, g, r = (_f64(a).copy() for a in (sub2, sub1, main, sup1, sup2, rhs))
    bsz, n = e.shape
    ops = np.zeros((bsz, 3), dtype=np.int64)
    status = np.full(bsz, STATUS_OK, dtype=np.int32)
    index = np.full(bsz, -1, dtype=np.int32)
    live = np.ones(bsz, dtype=bool)
    with np.errstate(all="ignore"):
        for i in range(2, n):                              # direct.py:134-152
            ci = c[:, i - 2]
            act = live & (ci != 0.0)
            piv = d[:, i - 2]
            bad = act & (piv == 0.0)
            status[bad], index[bad], live[bad] = STATUS_REDUCTION_PIVOT, i, False
            act &= ~bad
            m = ci / piv
            d[act, i - 1] = d[act, i - 1] - m[act] * e[act, i - 1]
            e[act, i] = e[act, i] - m[act] * f[act, i - 1]
            ops[act] += (2, 2, 1)
            if i - 1 <= n - 3:
                ga = g[:, i - 1]
                act_g = act & (ga != 0.0)
                f[act_g, i] = f[act_g, i] - m[act_g] * ga[act_g]
                ops[act_g] += (1, 1, 0)
            r[act, i] = r[act, i] - m[act] * r[act, i - 1]
            ops[act] += (1, 1, 0)
            c[act, i - 2] = 0.0
        for i in range(n - 3, -1, -1):                     # direct.py:153-164
            gi = g[:, i]
            act = live & (gi != 0.0)
            piv = f[:, i + 1]
            bad = act & (piv == 0.0)
            status[bad], index[bad], live[bad] = STATUS_REDUCTION_PIVOT, i, False
            act &= ~bad
            m = gi / piv
            e[act, i] = e[act, i] - m[act] * d[act, i]
            f[act, i] = f[act, i] - m[act] * e[act, i + 1]
            r[act, i] = r[act, i] - m[act] * r[act, i + 1]
            ops[act] += (3, 3, 1)
            g[act, i] = 0.0
    for a in (d, e, f, r):
        a[~live] = np.nan
    return d, e, f, r, ops, status, index


def pd2td_ntdm(sub2, sub1, main, sup1, sup2, rhs):
    """``solve_pd2td_ntdm`` (direct.py:168-177): reduce, then NTDM on the
    reduced system.  Returns (x, status, index, reduction ops (B,3))."""
    d, e, f, r, ops, status, index = pd_to_td(sub2, sub1, main, sup1, sup2, rhs)
    ok = status == STATUS_OK
    x = np.full(e.shape, np.nan)
    if ok.any():
        xs, st2, ix2 = ntdm(d[ok], e[ok], f[ok], r[ok])
        x[ok] = xs
        status[ok], index[ok] = st2, ix2
    return x, status, index, ops
