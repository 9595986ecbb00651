"""Seeded synthetic workloads for the five BASELINE.json configurations.

The reference ships no generator (its ``bench`` module is declared but absent,
SPEC.md:403-471), so these restate BASELINE.json
``configs`` literally.  Every generator draws from
``numpy.random.default_rng(seed)`` in a fixed order and returns host arrays in
the reference's per-diagonal lengths (core.py:117-152), batched on axis 0:

* tridiagonal: ``(sub1 (B,n-1), main (B,n), sup1 (B,n-1), rhs (B,n))``
* pentadiagonal: ``(sub2 (B,n-2), sub1, main, sup1, sup2 (B,n-2), rhs)``
* strided five-point (SIP): ``(subm (B,n-m), sub1, main, sup1, supm (B,n-m), rhs)``

Off-diagonals are drawn row-aligned (B, n) with the out-of-range end entries
set to 0, then cut to reference lengths, so the main diagonal's dominance
margin sees exactly the stored entries.
"""

from __future__ import annotations

import numpy as np


def _rng(seed):
    return np.random.default_rng(seed)


def td_dominant(batch, n, seed=0, rng=None):
    """Config 1 (and the ADI coefficients): sub/sup ~ U[-1,1] (ends 0),
    main = |sub| + |sup| + 1 + U[0,1], rhs ~ U[-1,1]."""
    rng = rng or _rng(seed)
    sub = rng.uniform(-1.0, 1.0, (batch, n))
    sub[:, 0] = 0.0
    sup = rng.uniform(-1.0, 1.0, (batch, n))
    sup[:, n - 1] = 0.0
    main = np.abs(sub) + np.abs(sup) + 1.0 + rng.uniform(0.0, 1.0, (batch, n))
    rhs = rng.uniform(-1.0, 1.0, (batch, n))
    return (np.ascontiguousarray(sub[:, 1:]), main, np.ascontiguousarray(sup[:, :-1]), rhs)


def pd_dominant(batch, n, seed=1, sparse_outer=False, rng=None):
    """Config 2: +-1, +-2 ~ U[-1,1] (ends 0), main = sum|off| + 1 + U[0,1].

    ``sparse_outer`` is the MNPDM family (literal row reading):
    the +-2 diagonals are zero except rows 0, 1 (their sup2 entries) and rows
    n-2, n-1 (their sub2 entries), so nz(sub2) = 2.  The main diagonal is
    formed from the entries actually kept.
    """
    rng = rng or _rng(seed)
    s2 = rng.uniform(-1.0, 1.0, (batch, n)); s2[:, :2] = 0.0
    s1 = rng.uniform(-1.0, 1.0, (batch, n)); s1[:, 0] = 0.0
    p1 = rng.uniform(-1.0, 1.0, (batch, n)); p1[:, n - 1] = 0.0
    p2 = rng.uniform(-1.0, 1.0, (batch, n)); p2[:, n - 2:] = 0.0
    u = rng.uniform(0.0, 1.0, (batch, n))
    rhs = rng.uniform(-1.0, 1.0, (batch, n))
    if sparse_outer:
        keep_s2 = np.zeros(n, bool); keep_s2[n - 2:] = True
        keep_p2 = np.zeros(n, bool); keep_p2[:2] = True
        s2 = np.where(keep_s2, s2, 0.0)
        p2 = np.where(keep_p2, p2, 0.0)
    main = np.abs(s2) + np.abs(s1) + np.abs(p1) + np.abs(p2) + 1.0 + u
    return (np.ascontiguousarray(s2[:, 2:]), np.ascontiguousarray(s1[:, 1:]), main,
            np.ascontiguousarray(p1[:, :-1]), np.ascontiguousarray(p2[:, :-2]), rhs)


def zero_pivot_rows(rng, batch, n, count=8, spacing=4, tail=3):
    """``count`` sorted rows per system, pairwise >= ``spacing`` apart and not
    in the last ``tail`` rows."""
    span = n - tail - (count - 1) * (spacing - 1)
    if span < count:
        raise ValueError(f"n={n} too small for {count} zero rows at spacing {spacing}")
    rows = np.empty((batch, count), dtype=np.int64)
    for s in range(batch):
        base = np.sort(rng.choice(span, size=count, replace=False))
        rows[s] = base + np.arange(count) * (spacing - 1)
    return rows


def td_symbolic(batch, n, seed=2, zeros=8, rng=None):
    """Config 3, tridiagonal: every entry ~ U[-1,1] (non-dominant), with
    ``zeros`` decoupled rows where A[i,i-1] = A[i,i] = 0, which makes the
    elimination pivot exactly 0 in every arithmetic.
    Returns (sub1, main, sup1, rhs, zero_rows)."""
    rng = rng or _rng(seed)
    sub = rng.uniform(-1.0, 1.0, (batch, n)); sub[:, 0] = 0.0
    main = rng.uniform(-1.0, 1.0, (batch, n))
    sup = rng.uniform(-1.0, 1.0, (batch, n)); sup[:, n - 1] = 0.0
    rhs = rng.uniform(-1.0, 1.0, (batch, n))
    rows = zero_pivot_rows(rng, batch, n, zeros) if zeros else np.zeros((batch, 0), np.int64)
    bidx = np.repeat(np.arange(batch), rows.shape[1])
    sub[bidx, rows.ravel()] = 0.0
    main[bidx, rows.ravel()] = 0.0
    return (np.ascontiguousarray(sub[:, 1:]), main, np.ascontiguousarray(sup[:, :-1]), rhs, rows)


def pd_symbolic(batch, n, seed=2, zeros=8, rng=None):
    """Config 3, pentadiagonal: as ``td_symbolic`` with A[i,i-2] = A[i,i-1] =
    A[i,i] = 0 on the decoupled rows.  Returns (sub2, sub1, main, sup1, sup2,
    rhs, zero_rows)."""
    rng = rng or _rng(seed)
    s2 = rng.uniform(-1.0, 1.0, (batch, n)); s2[:, :2] = 0.0
    s1 = rng.uniform(-1.0, 1.0, (batch, n)); s1[:, 0] = 0.0
    main = rng.uniform(-1.0, 1.0, (batch, n))
    p1 = rng.uniform(-1.0, 1.0, (batch, n)); p1[:, n - 1] = 0.0
    p2 = rng.uniform(-1.0, 1.0, (batch, n)); p2[:, n - 2:] = 0.0
    rhs = rng.uniform(-1.0, 1.0, (batch, n))
    rows = zero_pivot_rows(rng, batch, n, zeros) if zeros else np.zeros((batch, 0), np.int64)
    bidx = np.repeat(np.arange(batch), rows.shape[1])
    for arr in (s2, s1, main):
        arr[bidx, rows.ravel()] = 0.0
    return (np.ascontiguousarray(s2[:, 2:]), np.ascontiguousarray(s1[:, 1:]), main,
            np.ascontiguousarray(p1[:, :-1]), np.ascontiguousarray(p2[:, :-2]), rhs, rows)


def five_point(batch, n, m, seed=3, r=0.25, kmin=0.5, kmax=2.0, rng=None):
    """Config 4: one implicit step of u_t = div(k grad u) on an (n/m) x m grid,
    A = I + r * (-div k grad)_h with r = dt/h^2.

    Cell (p, q) is row i = p*m + q (q fastest): neighbours q+-1 are offsets
    +-1, p+-1 are offsets +-m.  Face coefficient = harmonic mean of the two
    cell k (k ~ U[kmin, kmax] per cell); a boundary face uses the cell's own k
    with a zero Dirichlet ghost.  m = 2 is the "ladder" twin whose +-1
    diagonal is zero every other row.  Returns
    (subm, sub1, main, sup1, supm, rhs) in reference lengths.
    """
    if n % m:
        raise ValueError("n must be a multiple of the grid width m")
    rng = rng or _rng(seed)
    rows = n // m
    k = rng.uniform(kmin, kmax, (batch, rows, m))
    rhs = rng.uniform(-1.0, 1.0, (batch, n))
    kx = 2.0 * k[:, :, 1:] * k[:, :, :-1] / (k[:, :, 1:] + k[:, :, :-1])   # faces q|q+1
    ky = 2.0 * k[:, 1:, :] * k[:, :-1, :] / (k[:, 1:, :] + k[:, :-1, :])   # faces p|p+1
    diag = np.zeros((batch, rows, m))
    diag[:, :, 1:] += kx
    diag[:, :, :-1] += kx
    diag[:, 1:, :] += ky
    diag[:, :-1, :] += ky
    diag[:, :, 0] += k[:, :, 0]
    diag[:, :, m - 1] += k[:, :, m - 1]
    diag[:, 0, :] += k[:, 0, :]
    diag[:, rows - 1, :] += k[:, rows - 1, :]
    main = (1.0 + r * diag).reshape(batch, n)
    off1 = np.zeros((batch, rows, m))
    off1[:, :, :m - 1] = -r * kx                       # (i, i+1) within a grid row
    off1 = off1.reshape(batch, n)[:, :n - 1]
    offm = (-r * ky).reshape(batch, n - m)
    return (offm.copy(), off1.copy(), main, off1.copy(), offm.copy(), rhs)


def sip_tolerance(rhs, rel=1e-8):
    """Relative stopping rule of config 4 as per-system absolute tolerances:
    x0 = 0 => r0 = b, so ||r||_inf < rel * ||b||_inf."""
    return rel * np.max(np.abs(rhs), axis=1)


def adi_step(n, seed=0):
    """Config 5 coefficients: x-sweep (B=n systems of order n) and y-sweep
    tridiagonal coefficients drawn as config 1 from one ``seed`` stream
    (x-sweep first).  The y-sweep rhs is the x-sweep output.  Returns
    ((sub1, main, sup1, rhs) for x, (sub1, main, sup1) for y)."""
    rng = _rng(seed)
    xs = td_dominant(n, n, rng=rng)
    ys = td_dominant(n, n, rng=rng)[:3]
    return xs, ys
