"""High-precision oracle for the symbolic solvers.  TEST INFRASTRUCTURE ONLY.

The reference's exact solvers return x = A^{-1} b exactly (exact.py:1-14,
278-307: the t-substituted elimination is LU of A + t*D and the limit t -> 0
is A^{-1} b for nonsingular A).  At config-3 sizes the reference itself takes
hours per system, so full-size parity is checked against
``limit_solve_mp``: banded Gaussian elimination with partial pivoting in
mpmath at ``dps`` decimal digits, rounded to binary64 -- float(A^{-1} b) up to
10^-dps relative.  Small-N cases are pinned to the reference's own exact
outputs (tests/golden/exact.npz).
"""

from __future__ import annotations

import mpmath
import numpy as np


def limit_solve_mp(diags, offsets, rhs, dps=50):
    """diags: reference-length 1-D arrays for the given offsets; one system."""
    n = len(rhs)
    with mpmath.workdps(dps):
        kl = -min(offsets)
        ku = max(offsets)
        # rows as dicts col -> value (band grows to ku + kl with pivoting)
        rows = [dict() for _ in range(n)]
        for d, off in zip(diags, offsets):
            for idx, v in enumerate(d):
                i = idx - min(off, 0)
                if v != 0.0:
                    rows[i][i + off] = mpmath.mpf(float(v))
        b = [mpmath.mpf(float(v)) for v in rhs]
        for k in range(n):
            # partial pivot among rows k..k+kl
            cand = range(k, min(n, k + kl + 1))
            p = max(cand, key=lambda r: abs(rows[r].get(k, 0)))
            if rows[p].get(k, 0) == 0:
                raise ZeroDivisionError("singular")
            if p != k:
                rows[k], rows[p] = rows[p], rows[k]
                b[k], b[p] = b[p], b[k]
            piv = rows[k][k]
            for r in range(k + 1, min(n, k + kl + 1)):
                f = rows[r].get(k, 0)
                if f == 0:
                    continue
                m = f / piv
                for c, v in rows[k].items():
                    if c >= k:
                        rows[r][c] = rows[r].get(c, 0) - m * v
                rows[r].pop(k, None)
                b[r] = b[r] - m * b[k]
        x = [mpmath.mpf(0)] * n
        for k in range(n - 1, -1, -1):
            acc = b[k]
            for c, v in rows[k].items():
                if c > k:
                    acc -= v * x[c]
            x[k] = acc / rows[k][k]
        return np.array([float(v) for v in x])


def frexp_fraction(v):
    """(mantissa, exponent) of an exact rational: v = m * 2**e, |m| in
    [0.5, 1) correctly rounded to binary64 (0 -> (0.0, 0))."""
    from fractions import Fraction
    v = Fraction(v)
    if v == 0:
        return 0.0, 0
    e = v.numerator.bit_length() - v.denominator.bit_length()
    if abs(v) >= Fraction(2) ** e:
        e += 1
    if abs(v) < Fraction(2) ** (e - 1):
        e -= 1
    return float(v / Fraction(2) ** e), e


def det_band_mp(diags, offsets, dps=60):
    """det(A) by banded Gaussian elimination with partial pivoting in mpmath
    (sign of the row permutation times the product of U's diagonal); the
    reference's exact_det_band returns det(A) exactly (exact.py:254-275), so
    this equals it to 10^-dps relative.  Returns (mantissa, exponent) as
    frexp_fraction."""
    from fractions import Fraction
    n = max(len(d) - min(o, 0) for d, o in zip(diags, offsets)) if diags else 0
    n = len(diags[offsets.index(0)])
    with mpmath.workdps(dps):
        kl = -min(offsets)
        rows = [dict() for _ in range(n)]
        for d, off in zip(diags, offsets):
            for idx, v in enumerate(d):
                i = idx - min(off, 0)
                if v != 0.0:
                    rows[i][i + off] = mpmath.mpf(float(v))
        det = mpmath.mpf(1)
        for k in range(n):
            cand = range(k, min(n, k + kl + 1))
            p = max(cand, key=lambda r: abs(rows[r].get(k, 0)))
            if rows[p].get(k, 0) == 0:
                return 0.0, 0
            if p != k:
                rows[k], rows[p] = rows[p], rows[k]
                det = -det
            piv = rows[k][k]
            det *= piv
            for r in range(k + 1, min(n, k + kl + 1)):
                f = rows[r].get(k, 0)
                if f == 0:
                    continue
                m = f / piv
                for c, v in rows[k].items():
                    if c >= k:
                        rows[r][c] = rows[r].get(c, 0) - m * v
                rows[r].pop(k, None)
        m, e = mpmath.frexp(det)
        return float(m), int(e)


def rcond_lapack(diags, offsets):
    """Reciprocal 1-norm condition estimate by LAPACK itself (scipy 1.18.1's
    bundled LAPACK: dgttrf + dgtcon for offsets -1..1, dgbtrf + dgbcon for
    -2..2), anorm = max column sum -- the checker of the GPU estimator (the
    reference has no condition estimator)."""
    import scipy.linalg.lapack as lp
    n = len(diags[offsets.index(0)])
    cols = np.zeros(n)
    for d, off in zip(diags, offsets):
        d = np.abs(np.asarray(d, dtype=np.float64))
        if off >= 0:
            cols[off:off + len(d)] += d        # A[i, i+off] sits in column i+off
        else:
            cols[:len(d)] += d                 # A[i-off... row i, column i+off
    anorm = float(np.max(cols))
    if len(offsets) == 3:
        dl, d, du = (np.asarray(diags[offsets.index(o)], dtype=np.float64) for o in (-1, 0, 1))
        dl2, d2, du2, du22, ipiv, info = lp.dgttrf(dl, d, du)
        if info > 0:
            return 0.0
        rc, info = lp.dgtcon(dl2, d2, du2, du22, ipiv, anorm, norm="1")
        return float(rc)
    kl = ku = 2
    ab = np.zeros((2 * kl + ku + 1, n))
    for d, off in zip(diags, offsets):
        for idx, v in enumerate(d):
            i = idx - min(off, 0)
            j = i + off
            ab[kl + ku + i - j, j] = v
    lub, ipiv, info = lp.dgbtrf(ab, kl, ku)
    if info > 0:
        return 0.0
    rc, info = lp.dgbcon(kl, ku, lub, ipiv, anorm, norm="1")
    return float(rc)


def rcond_dense(diags, offsets):
    """Exact 1/(||A||_1 ||A^-1||_1) by a dense inverse (small n only)."""
    n = len(diags[offsets.index(0)])
    a = np.zeros((n, n))
    for d, off in zip(diags, offsets):
        for idx, v in enumerate(d):
            i = idx - min(off, 0)
            a[i, i + off] = v
    return 1.0 / (np.linalg.norm(a, 1) * np.linalg.norm(np.linalg.inv(a), 1))
