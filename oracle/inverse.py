"""Restatement of the dense Hotelling-Bodewig inversion and SIP-HB.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Follows ``hb_invert_dense`` (inverse.py:94-119), ``dense_lower_factor`` /
``dense_upper_factor`` (72-87, generalised to the outer offset m) and the
dense branch of ``sip_hb_solve`` (205-241, 274-302).  The products go through
numpy.matmul (BLAS), as in the reference, so this path is NOT bit-reproducible
(SURVEY 8c "parity unpinned at the BLAS boundary"); parity is checked through
iteration counts, the inversion residual and the SIP-HB solution tolerance.
"""

from __future__ import annotations

import numpy as np

from . import STATUS_MAX_ITER, STATUS_OK, STATUS_ZERO_DIAG
from .iterative import sip


def dense_lower(f):
    """Unit-lower L as a dense (B, n, n) array (inverse.py:72-78)."""
    l1, l2, m = f["l1"], f["l2"], f["m"]
    bsz, n = l1.shape
    out = np.zeros((bsz, n, n))
    r = np.arange(n)
    out[:, r, r] = 1.0
    out[:, r[1:], r[1:] - 1] = l1[:, 1:]
    out[:, r[m:], r[m:] - m] = l2[:, m:]
    return out


def dense_upper(f):
    """Upper U as a dense (B, n, n) array (inverse.py:81-87)."""
    mu, phi, psi, m = f["mu"], f["phi"], f["psi"], f["m"]
    bsz, n = mu.shape
    out = np.zeros((bsz, n, n))
    r = np.arange(n)
    out[:, r, r] = mu
    out[:, r[:n - 1], r[:n - 1] + 1] = phi[:, :n - 1]
    out[:, r[:n - m], r[:n - m] + m] = psi[:, :n - m]
    return out


def hb_invert_dense(m, tol=1e-12, max_iter=200):
    """X <- X (2I - M X) from X0 = diag(1/m_ii) (inverse.py:94-119), one matrix.

    Returns (X, iterations, residual_inf, history, status)."""
    m = np.asarray(m, dtype=np.float64)
    n = m.shape[0]
    diag = np.diagonal(m)
    zero_rows = np.nonzero(diag == 0.0)[0]
    if zero_rows.size:
        return None, 0, np.inf, (), STATUS_ZERO_DIAG
    x = np.diag(1.0 / diag)
    eye = np.eye(n)
    history = []
    for it in range(max_iter + 1):
        p = m @ x
        r = float(np.max(np.sum(np.abs(eye - p), axis=1)))
        history.append(r)
        if r < tol:
            return x, it, r, tuple(history), STATUS_OK
        x = x @ (2.0 * eye - p)
    return x, max_iter, history[-1], tuple(history), STATUS_MAX_ITER


def sip_hb(sub_m, sub1, main, sup1, sup_m, rhs, tol, max_iter, m=2, alpha=0.0):
    """Dense-mode ``sip_hb_solve`` (inverse.py:205-302), batched.

    The inversion tolerance is the per-system SIP tolerance, as in the
    reference (inverse.py:235-236)."""
    from .iterative import ilu0
    f, st, idx = ilu0(sub_m, sub1, main, sup1, sup_m, m, alpha)
    bsz = f["mu"].shape[0]
    tol = np.broadcast_to(np.asarray(tol, dtype=np.float64), (bsz,))
    lo, up = dense_lower(f), dense_upper(f)
    xl = np.empty_like(lo)
    xu = np.empty_like(up)
    inv_iters = np.zeros((bsz, 2), dtype=np.int64)
    inv_res = np.zeros((bsz, 2))
    for s in range(bsz):
        xl[s], inv_iters[s, 0], inv_res[s, 0], _, _ = hb_invert_dense(lo[s], tol[s])
        xu[s], inv_iters[s, 1], inv_res[s, 1], _, _ = hb_invert_dense(up[s], tol[s])
    out = sip(sub_m, sub1, main, sup1, sup_m, rhs, tol, max_iter, m, alpha,
              apply_l=lambda v: np.einsum("bij,bj->bi", xl, v),
              apply_u=lambda v: np.einsum("bij,bj->bi", xu, v))
    out["inv_iterations"] = inv_iters
    out["inv_residual"] = inv_res
    out["xl"], out["xu"] = xl, xu
    return out
