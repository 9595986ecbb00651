"""Batched restatement of ILU(0), the defect matrix and Stone's SIP.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

The reference (``iterative.py``) is hard-wired to the pentadiagonal offsets
-2..+2.  This restatement takes the outer offset as a stride ``m``:

* ``m == 2`` reproduces the reference bit-for-bit (``ilu0_penta``
  iterative.py:62-124, ``_factor_product_diagonals``/``defect_matrix``
  152-200, ``_sweep_apply`` 203-236, ``forward_sub``/``backward_sub`` 127-149,
  ``sip_solve`` 255-308); pinned by ``tests/test_oracle_golden.py``.
* ``m >= 3`` is the five-point-stencil generalisation (grid width m): L has
  offsets -1, -m, U has +1, +m, and L U has fill at +-(m-1).  ``alpha`` is
  Stone's partial-cancellation parameter (absent from the reference, SURVEY
  D1); ``alpha == 0`` is pure pattern-restricted ILU(0).  The same
  pattern-restriction rules as the reference apply (multipliers only where A
  is structurally nonzero, iterative.py:80-114).  These rows are restated, not
  reference-pinned: DESIGN.md "SIP extension".

Diagonals are ROW-ALIGNED (B, n) arrays inside this module: ``lo1[:, i]`` is
the (i, i-1) entry, ``lom[:, i]`` the (i, i-m) entry, ``up1[:, i]`` the
(i, i+1) entry, ``upm[:, i]`` the (i, i+m) entry; out-of-range slots are 0.
"""

from __future__ import annotations

import numpy as np

from . import (STATUS_DIVERGED, STATUS_MAX_ITER, STATUS_OK, STATUS_ZERO_PIVOT)

DIVERGENCE_FACTOR = 1e6                         # iterative.py:29


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def row_aligned(sub_m, sub1, main, sup1, sup_m, m):
    """Reference-length diagonals -> row-aligned (B, n) arrays (core.py:157-164)."""
    main = _f64(main)
    bsz, n = main.shape
    lom = np.zeros((bsz, n)); lo1 = np.zeros((bsz, n))
    up1 = np.zeros((bsz, n)); upm = np.zeros((bsz, n))
    lom[:, m:] = _f64(sub_m)
    lo1[:, 1:] = _f64(sub1)
    up1[:, :n - 1] = _f64(sup1)
    upm[:, :n - m] = _f64(sup_m)
    return lom, lo1, main.copy(), up1, upm


def ilu0(sub_m, sub1, main, sup1, sup_m, m=2, alpha=0.0):
    """Pattern-restricted ILU(0) / Stone factorisation.

    Returns dict(mu, l1, l2, phi, psi) row-aligned plus status, index.
    m == 2, alpha == 0: ``ilu0_penta`` (iterative.py:62-124) bit-for-bit.
    """
    if m == 2 and alpha != 0.0:
        raise ValueError("alpha != 0 is defined for stride m >= 3 only")
    a2, a1, e, c1, c2 = row_aligned(sub_m, sub1, main, sup1, sup_m, m)
    bsz, n = e.shape
    mu = np.zeros((bsz, n)); l1 = np.zeros((bsz, n)); l2 = np.zeros((bsz, n))
    phi = np.zeros((bsz, n)); psi = np.zeros((bsz, n))
    status = np.zeros(bsz, dtype=np.int32)
    index = np.full(bsz, -1, dtype=np.int32)
    with np.errstate(all="ignore"):
        for i in range(n):
            has2 = (a2[:, i] != 0.0) if i >= m else np.zeros(bsz, bool)
            has1 = (a1[:, i] != 0.0) if i >= 1 else np.zeros(bsz, bool)
            if m == 2:
                # iterative.py:80-114
                li2 = a2[:, i] / mu[:, i - 2] if i >= 2 else np.zeros(bsz)
                t = np.where(has2, a1[:, i] - li2 * phi[:, i - 2], a1[:, i]) if i >= 2 else a1[:, i]
                li1 = t / mu[:, i - 1] if i >= 1 else np.zeros(bsz)
                mi = e[:, i]
                if i >= 2:
                    mi = np.where(has2, mi - li2 * psi[:, i - 2], mi)
                if i >= 1:
                    mi = np.where(has1, mi - li1 * phi[:, i - 1], mi)
                if i <= n - 2:
                    fi = c1[:, i]
                    upd = (fi != 0.0) & has1
                    phi[:, i] = np.where(upd, fi - li1 * psi[:, i - 1], fi) if i >= 1 else fi
                if i <= n - 3:
                    psi[:, i] = c2[:, i]
            else:
                if i >= m:
                    den2 = mu[:, i - m] if alpha == 0.0 else mu[:, i - m] + alpha * phi[:, i - m]
                    li2 = a2[:, i] / den2
                else:
                    li2 = np.zeros(bsz)
                if i >= 1:
                    den1 = mu[:, i - 1] if alpha == 0.0 else mu[:, i - 1] + alpha * psi[:, i - 1]
                    li1 = a1[:, i] / den1
                else:
                    li1 = np.zeros(bsz)
                mi = e[:, i]
                if i >= m:
                    mi = np.where(has2, mi - li2 * psi[:, i - m], mi)
                if i >= 1:
                    mi = np.where(has1, mi - li1 * phi[:, i - 1], mi)
                if alpha != 0.0:
                    comp = np.zeros(bsz)
                    if i >= m:
                        comp = np.where(has2, comp + li2 * phi[:, i - m], comp)
                    if i >= 1:
                        comp = np.where(has1, comp + li1 * psi[:, i - 1], comp)
                    mi = mi + alpha * comp
                if i <= n - 2:
                    fi = c1[:, i]
                    if alpha != 0.0 and i >= m:
                        fi = np.where((fi != 0.0) & has2, fi - alpha * (li2 * phi[:, i - m]), fi)
                    phi[:, i] = fi
                if i <= n - m - 1:
                    gi = c2[:, i]
                    if alpha != 0.0 and i >= 1:
                        gi = np.where((gi != 0.0) & has1, gi - alpha * (li1 * psi[:, i - 1]), gi)
                    psi[:, i] = gi
            hit = (mi == 0.0) & (status == STATUS_OK)
            status[hit] = STATUS_ZERO_PIVOT
            index[hit] = i
            mu[:, i] = mi
            l1[:, i] = np.where(has1, li1, 0.0)
            l2[:, i] = np.where(has2, li2, 0.0)
    return dict(mu=mu, l1=l1, l2=l2, phi=phi, psi=psi, m=m), status, index


def defect(f, sub_m, sub1, main, sup1, sup_m):
    """K = L U - A, row-aligned diagonals keyed by offset.

    m == 2: ``_factor_product_diagonals`` + ``defect_matrix``
    (iterative.py:152-200), five diagonals.  m >= 3: seven diagonals
    (offsets 0, +-1, +-(m-1), +-m).
    """
    m = f["m"]
    mu, l1, l2, phi, psi = f["mu"], f["l1"], f["l2"], f["phi"], f["psi"]
    a2, a1, e, c1, c2 = row_aligned(sub_m, sub1, main, sup1, sup_m, m)
    bsz, n = mu.shape
    k = {}
    with np.errstate(all="ignore"):
        p_m = np.zeros((bsz, n)); p_m[:, m:] = l2[:, m:] * mu[:, :n - m]
        p_1 = np.zeros((bsz, n)); p_1[:, 1:] = l1[:, 1:] * mu[:, :n - 1]
        p_0 = mu.copy()
        p_0[:, 1:] += l1[:, 1:] * phi[:, :n - 1]
        p_0[:, m:] += l2[:, m:] * psi[:, :n - m]
        p1 = phi.copy()
        p1[:, n - 1] = 0.0
        pm = psi.copy()
        pm[:, n - m:] = 0.0
        if m == 2:
            p_1[:, 2:] += l2[:, 2:] * phi[:, :n - 2]        # iterative.py:164
            p1[:, 1:n - 1] += l1[:, 1:n - 1] * psi[:, :n - 2]  # iterative.py:168
        else:
            p_mm1 = np.zeros((bsz, n)); p_mm1[:, m:] = l2[:, m:] * phi[:, :n - m]
            p_pm1 = np.zeros((bsz, n))
            p_pm1[:, 1:n - m + 1] = l1[:, 1:n - m + 1] * psi[:, :n - m]
            k[-(m - 1)] = p_mm1
            k[m - 1] = p_pm1
        k[-m] = p_m - a2
        k[-1] = p_1 - a1
        k[0] = p_0 - e
        k[1] = p1 - c1
        k[m] = pm - c2
    # out-of-range slots of the differences are exactly 0 - 0 = 0
    return k


def sweep_apply(diags, m, x):
    """A @ x as accumulating diagonal sweeps from zero, ``_sweep_apply``
    (iterative.py:203-221): order main, -1, +1, -m, +m [, -(m-1), +(m-1)]."""
    x = _f64(x)
    bsz, n = x.shape
    out = np.zeros((bsz, n))
    with np.errstate(all="ignore"):
        out += diags[0] * x
        out[:, 1:] += diags[-1][:, 1:] * x[:, :-1]
        out[:, :-1] += diags[1][:, :-1] * x[:, 1:]
        out[:, m:] += diags[-m][:, m:] * x[:, :-m]
        out[:, :-m] += diags[m][:, :-m] * x[:, m:]
        if m != 2 and -(m - 1) in diags:
            q = m - 1
            out[:, q:] += diags[-q][:, q:] * x[:, :-q]
            out[:, :-q] += diags[q][:, :-q] * x[:, q:]
    return out


def a_diags(sub_m, sub1, main, sup1, sup_m, m):
    a2, a1, e, c1, c2 = row_aligned(sub_m, sub1, main, sup1, sup_m, m)
    return {-m: a2, -1: a1, 0: e, 1: c1, m: c2}


def forward_sub(f, v):
    """L y = v, ``penta_forward`` (_elim.py:65-73) with the outer offset m."""
    m = f["m"]
    l1, l2 = f["l1"], f["l2"]
    v = _f64(v)
    bsz, n = v.shape
    y = np.empty((bsz, n))
    with np.errstate(all="ignore"):
        y[:, 0] = v[:, 0]
        for i in range(1, n):
            t = v[:, i] - l1[:, i] * y[:, i - 1]
            if i >= m:
                t = t - l2[:, i] * y[:, i - m]
            y[:, i] = t
    return y


def backward_sub(f, y):
    """U x = y, ``penta_backward`` (_elim.py:76-87) with the outer offset m."""
    m = f["m"]
    mu, phi, psi = f["mu"], f["phi"], f["psi"]
    bsz, n = y.shape
    x = np.empty((bsz, n))
    with np.errstate(all="ignore"):
        x[:, n - 1] = y[:, n - 1] / mu[:, n - 1]
        for i in range(n - 2, -1, -1):
            t = y[:, i] - phi[:, i] * x[:, i + 1]
            if i + m <= n - 1:
                t = t - psi[:, i] * x[:, i + m]
            x[:, i] = t / mu[:, i]
    return x


def sip(sub_m, sub1, main, sup1, sup_m, rhs, tol, max_iter, m=2, alpha=0.0,
        x0=None, record_history=False, apply_l=None, apply_u=None):
    """``sip_solve`` (iterative.py:255-308), batched with per-system tolerance.

    ``tol`` is a scalar or a (B,) array.  Each system iterates exactly as the
    reference would on its own and is frozen once it leaves the loop.
    Returns dict(x, iterations, residual, best_x, best_residual, status,
    index, history).  ``apply_l``/``apply_u`` replace the substitutions (the
    Hotelling-Bodewig variant, inverse.py:284-298).
    """
    b = _f64(rhs)
    bsz, n = b.shape
    tol = np.broadcast_to(np.asarray(tol, dtype=np.float64), (bsz,)).copy()
    f, st, idx = ilu0(sub_m, sub1, main, sup1, sup_m, m, alpha)
    kd = defect(f, sub_m, sub1, main, sup1, sup_m)
    ad = a_diags(sub_m, sub1, main, sup1, sup_m, m)
    x = np.zeros((bsz, n)) if x0 is None else _f64(x0).copy()
    with np.errstate(all="ignore"):
        res = b - sweep_apply(ad, m, x)
        r = np.max(np.abs(res), axis=1)
    r0 = r.copy()
    k = np.zeros(bsz, dtype=np.int64)
    best_x = x.copy()
    best = r.copy()
    status = st.copy()
    index = idx.copy()
    active = (status == STATUS_OK) & (r >= tol)
    history = []
    fl = apply_l or (lambda v: forward_sub(f, v))
    fu = apply_u or (lambda v: backward_sub(f, v))
    while active.any():
        maxed = active & (k >= max_iter)
        status[maxed] = STATUS_MAX_ITER
        active &= ~maxed
        if not active.any():
            break
        with np.errstate(all="ignore"):
            new_rhs = sweep_apply(kd, m, x) + b
            y = fl(new_rhs)
            xn = fu(y)
            rn = np.max(np.abs(b - sweep_apply(ad, m, xn)), axis=1)
        x[active] = xn[active]
        r[active] = rn[active]
        k[active] += 1
        if record_history:
            history.append(np.where(active, rn, np.nan))
        imp = active & (rn < best)
        best_x[imp] = xn[imp]
        best[imp] = rn[imp]
        dv = active & (r0 > 0) & (rn > DIVERGENCE_FACTOR * r0)
        status[dv] = STATUS_DIVERGED
        active &= ~dv
        active &= r >= tol
    return dict(x=x, iterations=k, residual=r, best_x=best_x, best_residual=best,
                status=status, index=index, history=history, factors=f, defect=kd)
