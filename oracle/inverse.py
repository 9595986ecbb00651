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


# ---------------------------------------------------------------------------
# banded ("array implementation") HB: inverse.py:41-61, 122-195, 242-272
# ---------------------------------------------------------------------------
STATUS_STAGNATED = 9


def band_mul_tri(a_diags, b_diags, n, w_out, side):
    """_band_mul_tri (inverse.py:122-137), same op order: out[r] accumulated
    from zeros over j ascending, one rounding per multiply and per add."""
    p, q = len(a_diags) - 1, len(b_diags) - 1
    out = []
    for r in range(w_out + 1):
        res = np.zeros(n - r)
        for j in range(max(0, r - q), min(p, r) + 1):
            lo = r - j
            if side == "lower":
                res = res + a_diags[j][lo:lo + (n - r)] * b_diags[lo][:n - r]
            else:
                res = res + a_diags[j][:n - r] * b_diags[lo][j:j + (n - r)]
        out.append(res)
    return out


def band_residual_norm(p_diags):
    """_band_residual_norm (inverse.py:140-145)."""
    r = float(np.max(np.abs(1.0 - p_diags[0])))
    for d in p_diags[1:]:
        if d.size:
            r = max(r, float(np.max(np.abs(d))))
    return r


def factor_diags(f, s, side):
    """reference-length diagonals of factor `side` of system s (row-aligned
    oracle factors, iterative.ilu0): lower (1, l_sub1, l_sub2), upper (u_main,
    u_sup1, u_sup2) -- BandFactors, core.py:208-223."""
    n = f["mu"].shape[1]
    if side == "lower":
        return (np.ones(n), f["l1"][s, 1:], f["l2"][s, 2:])
    return (f["mu"][s], f["phi"][s, :n - 1], f["psi"][s, :n - 2])


def hb_invert_banded(m_diags, side, w=2, tol=1e-12, max_iter=200):
    """hb_invert_banded (inverse.py:148-195), one factor.  Returns (diags,
    iterations, residual, history, status): OK -> the converged iterate;
    STAGNATED -> the best report (Stagnated(best)); MAX_ITER -> best.inverse
    with the last residual (MaxIterationsExceeded(best.inverse, h[-1]));
    ZERO_DIAG -> (None, first zero row, ...)."""
    n = len(m_diags[0])
    if side == "lower":
        x0 = np.ones(n)
    else:
        zero = np.nonzero(m_diags[0] == 0.0)[0]
        if zero.size:
            return None, int(zero[0]), np.nan, (), STATUS_ZERO_DIAG
        x0 = 1.0 / m_diags[0]
    x = [x0] + [np.zeros(n - j) for j in range(1, w + 1)]
    history, best = [], None
    for it in range(max_iter + 1):
        p = band_mul_tri(m_diags, x, n, w, side)
        r = band_residual_norm(p)
        history.append(r)
        if best is None or r < best[2]:
            best = (x, it, r)
        if r < tol:
            return x, it, r, tuple(history), STATUS_OK
        if len(history) > 3 and r > 0.99 * history[-4]:
            return best[0], best[1], best[2], tuple(history), STATUS_STAGNATED
        s = [-d for d in p]
        s[0] = 2.0 + s[0]
        x = band_mul_tri(x, s, n, w, side)
    return best[0], max_iter, history[-1], tuple(history), STATUS_MAX_ITER


def band_matvec(diags, side, v):
    """BandedApproxInverse.matvec (inverse.py:49-61)."""
    n = len(diags[0])
    out = diags[0] * v
    for j in range(1, len(diags)):
        if side == "lower":
            out[j:] += diags[j] * v[:n - j]
        else:
            out[:n - j] += diags[j] * v[j:]
    return out


def band_true_residual(m_diags, x_diags, side):
    """||I - M X||_inf (max row sum) of a band inverse: the untruncated band
    product (offsets 0..w+2) summed along rows."""
    n = len(m_diags[0])
    w = len(x_diags) - 1
    p = band_mul_tri(m_diags, x_diags, n, min(w + 2, n - 1), side)
    rows = np.abs(1.0 - p[0])
    for r in range(1, len(p)):
        if side == "lower":
            rows[r:] += np.abs(p[r])       # entry (k + r, k) lies in row k + r
        else:
            rows[:n - r] += np.abs(p[r])   # entry (k, k + r) lies in row k
    return float(np.max(rows))


def sip_hb_banded(sub2, sub1, main, sup1, sup2, rhs, tol, max_iter, w=None, cap=None,
                  max_inv_iter=200):
    """sip_hb_solve(mode="banded") (inverse.py:242-272 + 274-302), batched.

    w >= 2: the reference's explicit width.  w None: auto width 2, 4, ... up to
    cap with the TRUE-residual acceptance rule of this build (the reference
    widens on stagnation only, which never triggers -- SURVEY D8)."""
    from .iterative import ilu0
    f, st, idx = ilu0(sub2, sub1, main, sup1, sup2, 2, 0.0)
    bsz, n = f["mu"].shape
    tol = np.broadcast_to(np.asarray(tol, dtype=np.float64), (bsz,))
    cap = min(cap or (n - 1), n - 1)
    inv = {}
    info = {"inv_w": np.zeros((bsz, 2), np.int64), "inv_status": np.zeros((bsz, 2), np.int32)}
    for s in range(bsz):
        for c, side in enumerate(("lower", "upper")):
            md = factor_diags(f, s, side)
            ww = w if w else min(2, cap)
            while True:
                d, it, r, h, stt = hb_invert_banded(md, side, ww, float(tol[s]), max_inv_iter)
                if w or stt not in (STATUS_OK, STATUS_STAGNATED) or ww >= cap:
                    break
                if band_true_residual(md, d, side) < tol[s]:
                    break
                ww = min(2 * ww, cap)
            inv[(s, side)] = d
            info["inv_w"][s, c] = ww
            info["inv_status"][s, c] = stt
    out = sip(sub2, sub1, main, sup1, sup2, rhs, tol, max_iter, 2, 0.0,
              apply_l=lambda v: np.stack([band_matvec(inv[(s, "lower")], "lower", v[s])
                                          for s in range(bsz)]),
              apply_u=lambda v: np.stack([band_matvec(inv[(s, "upper")], "upper", v[s])
                                          for s in range(bsz)]))
    out.update(info)
    return out
