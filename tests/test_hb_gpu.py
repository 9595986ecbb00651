"""GPU parity of the Hotelling-Bodewig inversion (DMMA) and SIP-HB against the
reference's own outputs (golden) and the numpy/BLAS restatement.  The
reference's HB products go through BLAS, so parity is iteration counts +
tolerance, not bits."""

import numpy as np
import pytest
import torch

from oracle import inverse as H
from oracle import iterative as I
from paper_1804_09666_b200 import (DenseCapExceeded, PentaMatrix, SipConfig, StencilMatrix,
                                   hb_invert_factors, sip_hb_solve)
from paper_1804_09666_b200 import workloads as W

pytestmark = pytest.mark.gpu
PD = ("sub2", "sub1", "main", "sup1", "sup2", "rhs")


def host(t):
    return t.detach().cpu().numpy()


@pytest.mark.parametrize("layout", ["interleaved", "system"])
def test_sip_hb_golden(cuda, golden, layout):
    g = golden("inverse")
    a = [g[f"hb_{k}"] for k in PD]
    A = PentaMatrix.from_diagonals(*a[:5], layout=layout)
    rep = sip_hb_solve(A, a[5], SipConfig(tolerance=g["hb_tol"], max_iterations=500))
    assert (host(rep.status) == 0).all()
    assert np.array_equal(host(rep.iterations), g["hb_k"])
    assert np.array_equal(host(rep.inv_iterations)[:, 0], g["hb_linv_iters"])
    assert np.array_equal(host(rep.inv_iterations)[:, 1], g["hb_uinv_iters"])
    x = host(rep.x)
    assert np.abs(x - g["hb_x"]).max() <= 1e-11 * np.abs(g["hb_x"]).max()
    assert np.all(host(rep.residual_inf) < g["hb_tol"])
    # ops: the reference's dense-apply tally, 4N^2 + 20N - 24 per iteration
    ops = np.stack([host(v) for v in (rep.ops.adds, rep.ops.subs, rep.ops.muls)], axis=1)
    assert np.array_equal(ops, g["hb_ops"][:, :3]) and (g["hb_ops"][:, 3] == 0).all()


@pytest.mark.parametrize("m,rows,alpha", [(2, 128, 0.0), (16, 24, 0.5), (32, 64, 0.5)])
def test_hb_inverses_match_restatement(cuda, m, rows, alpha):
    n = m * rows
    p = W.five_point(3, n, m, seed=8)
    tol = W.sip_tolerance(p[5])
    A = StencilMatrix.from_diagonals(*p[:5], m=m)
    xl, xu, its, res, st, _ = hb_invert_factors(A, tol, alpha=alpha)
    f, _, _ = I.ilu0(*p[:5], m=m, alpha=alpha)
    lo, up = H.dense_lower(f), H.dense_upper(f)
    for s in range(3):
        ref_l = H.hb_invert_dense(lo[s], tol[s])
        ref_u = H.hb_invert_dense(up[s], tol[s])
        assert host(its)[s, 0] == ref_l[1] and host(its)[s, 1] == ref_u[1]
        assert np.abs(host(xl)[s] - ref_l[0]).max() <= 1e-12 * np.abs(ref_l[0]).max()
        assert np.abs(host(xu)[s] - ref_u[0]).max() <= 1e-12 * np.abs(ref_u[0]).max()
        assert host(res)[s, 0] < tol[s] and host(res)[s, 1] < tol[s]


def test_sip_hb_stencil_matches_sip(cuda):
    """SIP-HB and SIP reach the same iterate count and solution (probe P9)."""
    m, n = 32, 2048
    p = W.five_point(8, n, m, seed=3)
    tol = W.sip_tolerance(p[5])
    A = StencilMatrix.from_diagonals(*p[:5], m=m)
    from paper_1804_09666_b200 import sip_solve
    r1 = sip_solve(A, p[5], SipConfig(tolerance=tol, max_iterations=500, alpha=0.5))
    r2 = sip_hb_solve(A, p[5], SipConfig(tolerance=tol, max_iterations=500, alpha=0.5))
    assert (host(r2.status) == 0).all()
    assert np.all(np.abs(host(r1.iterations) - host(r2.iterations)) <= 1)
    assert np.abs(host(r1.x) - host(r2.x)).max() <= 1e-7 * np.abs(host(r1.x)).max()


def test_dense_cap(cuda):
    p = W.five_point(1, 64, 2)
    with pytest.raises(DenseCapExceeded):
        sip_hb_solve(PentaMatrix.from_diagonals(*p[:5]), p[5], dense_cap=32)


def test_hb_inverses_ignore_stale_workspace(cuda):
    """A workspace full of NaN bytes (left by an earlier call) must not leak
    into the exported inverses: the off-triangle is exactly zero."""
    import torch
    from paper_1804_09666_b200 import _lib
    from paper_1804_09666_b200.core import workspace
    m, n = 16, 384
    p = W.five_point(2, n, m, seed=8)
    tol = W.sip_tolerance(p[5])
    ws = workspace(_lib.lib().bx_hb_workspace_bytes(2, n), torch.device("cuda", 0))
    ws.fill_(0xFF)  # NaN pattern in every double
    xl, xu, its, _, st, _ = hb_invert_factors(StencilMatrix.from_diagonals(*p[:5], m=m), tol,
                                              alpha=0.5)
    assert (host(st) == 0).all()
    xl, xu = host(xl), host(xu)
    assert np.all(np.isfinite(xl)) and np.all(np.isfinite(xu))
    assert np.all(np.triu(xl, 1) == 0.0) and np.all(np.tril(xu, -1) == 0.0)


# ---- hb_invert_dense on a caller's dense matrices (inverse.py:94-119) -------
def test_hb_invert_dense_spec_case(cuda, golden):
    """[[1, 0], [3, 1]] inverts in one iteration (reference run)."""
    from paper_1804_09666_b200 import hb_invert_dense
    g = golden("inverse")
    r = hb_invert_dense(np.array([[1.0, 0.0], [3.0, 1.0]]))
    assert r.iterations == int(g["hb_spec_iters"])
    assert np.array_equal(r.inverse, g["hb_spec_inv"])
    assert r.residual_inf < 1e-12 and len(r.residual_history) == r.iterations + 1


def test_hb_invert_dense_ilu_factors_match_reference_counts(cuda, golden):
    """dense_lower_factor / dense_upper_factor of the ILU(0) factors, then
    hb_invert_dense: the reference's iteration counts (golden), inverses within
    rounding of the numpy restatement."""
    from oracle import inverse as OI
    from paper_1804_09666_b200 import (dense_lower_factor, dense_upper_factor, hb_invert_dense,
                                       ilu0_penta)
    g = golden("inverse")
    a = [g[f"hb_{k}"] for k in PD]
    for s in range(a[0].shape[0]):
        A = PentaMatrix.from_diagonals(*(v[s] for v in a[:5]))
        f = ilu0_penta(A)
        for dense, key in ((dense_lower_factor, "hb_linv_iters"), (dense_upper_factor, "hb_uinv_iters")):
            M = dense(f)
            r = hb_invert_dense(M, float(g["hb_tol"][s]))
            assert r.iterations == int(g[key][s])
            rx, rit, _, _, _ = OI.hb_invert_dense(M, float(g["hb_tol"][s]))
            assert r.iterations == rit
            assert np.abs(r.inverse - rx).max() <= 1e-12 * np.abs(rx).max()


def test_hb_invert_dense_batched_general_and_errors(cuda):
    from oracle import inverse as OI
    from paper_1804_09666_b200 import MaxIterationsExceeded, ZeroDiagonal, hb_invert_dense
    rng = np.random.default_rng(4)
    B, n = 5, 150            # not a multiple of the 64-wide tiles; non-triangular
    M = np.eye(n)[None] + 0.3 / n * rng.uniform(-1, 1, (B, n, n))
    M[:, np.arange(n), np.arange(n)] += rng.uniform(0.5, 2.0, (B, n))
    r = hb_invert_dense(torch.from_numpy(M).cuda(), 1e-13)
    assert (host(r.status) == 0).all()
    for s in range(B):
        rx, rit, _, _, _ = OI.hb_invert_dense(M[s], 1e-13)
        assert int(r.iterations[s]) == rit
        x = host(r.inverse[s])
        assert np.abs(x - rx).max() <= 1e-12 * np.abs(rx).max()
        assert np.abs(np.eye(n) - M[s] @ x).sum(axis=1).max() < 1e-13
    Z = M.copy()
    Z[2, 7, 7] = 0.0
    rz = hb_invert_dense(Z)
    assert host(rz.status).tolist() == [0, 0, 5, 0, 0] and int(rz.index[2]) == 7
    with pytest.raises(ZeroDiagonal) as e:
        hb_invert_dense(Z[2])
    assert e.value.index == 7
    with pytest.raises(MaxIterationsExceeded) as e:
        hb_invert_dense(M[0], 1e-13, max_iter=1)
    assert e.value.iterations == 1
