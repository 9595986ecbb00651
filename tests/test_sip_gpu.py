"""GPU parity of ILU(0) / defect / SIP: bit-identical to the reference (m=2
golden vectors) and to the C restatement (stride m >= 3, Stone's alpha)."""

import numpy as np
import pytest

from oracle import cport
from oracle import iterative as I
from paper_1804_09666_b200 import (MaxIterationsExceeded, PentaMatrix, SipConfig, StencilMatrix,
                                   ZeroPivot, defect_matrix, ilu0_penta, sip_solve)
from paper_1804_09666_b200 import workloads as W

pytestmark = pytest.mark.gpu
PD = ("sub2", "sub1", "main", "sup1", "sup2", "rhs")
LAYOUTS = ["interleaved", "system"]


def host(t):
    return t.detach().cpu().numpy()


@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("tag", ["ladder", "full", "holes"])
def test_ilu0_defect_golden(cuda, golden, layout, tag):
    g = golden("iterative")
    a = [g[f"{tag}_{k}"] for k in PD]
    n = a[2].shape[1]
    A = PentaMatrix.from_diagonals(*a[:5], layout=layout)
    f = ilu0_penta(A)
    lay = lambda t: host(t.t() if layout == "interleaved" else t)  # noqa: E731
    assert np.array_equal(lay(f.l_sub1)[:, 1:], g[f"{tag}_l_sub1"])
    assert np.array_equal(lay(f.l_sub2)[:, 2:], g[f"{tag}_l_sub2"])
    assert np.array_equal(lay(f.u_main), g[f"{tag}_u_main"])
    assert np.array_equal(lay(f.u_sup1)[:, :n - 1], g[f"{tag}_u_sup1"])
    assert np.array_equal(lay(f.u_sup2)[:, :n - 2], g[f"{tag}_u_sup2"])
    K = defect_matrix(f, A).diagonals
    assert np.array_equal(host(K[-2])[:, 2:], g[f"{tag}_k_sub2"])
    assert np.array_equal(host(K[-1])[:, 1:], g[f"{tag}_k_sub1"])
    assert np.array_equal(host(K[0]), g[f"{tag}_k_main"])
    assert np.array_equal(host(K[1])[:, :n - 1], g[f"{tag}_k_sup1"])
    assert np.array_equal(host(K[2])[:, :n - 2], g[f"{tag}_k_sup2"])


@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("tag", ["ladder", "full", "holes"])
def test_sip_golden_bitexact(cuda, golden, layout, tag):
    g = golden("iterative")
    a = [g[f"{tag}_{k}"] for k in PD]
    A = PentaMatrix.from_diagonals(*a[:5], layout=layout)
    rep = sip_solve(A, a[5], SipConfig(tolerance=g[f"{tag}_tol"], max_iterations=500),
                    record_history=True)
    assert np.array_equal(host(rep.x), g[f"{tag}_x"])
    assert np.array_equal(host(rep.iterations), g[f"{tag}_k"])
    assert np.array_equal(host(rep.residual_inf), g[f"{tag}_res"])
    h = host(rep.history)
    kmax = int(g[f"{tag}_k"].max())
    assert np.array_equal(h[:, :kmax], g[f"{tag}_hist"][:, :kmax], equal_nan=True)
    assert (host(rep.status) == 0).all()


def test_sip_single_system_contract(cuda, golden):
    g = golden("iterative")
    a = [g[f"ladder_{k}"][0] for k in PD]
    A = PentaMatrix.from_diagonals(*a[:5])
    rep = sip_solve(A, a[5], SipConfig(tolerance=float(g["ladder_tol"][0]), max_iterations=500),
                    record_history=True)
    assert isinstance(rep.x, np.ndarray) and np.array_equal(rep.x, g["ladder_x"][0])
    assert rep.iterations == g["ladder_k"][0]
    assert rep.ops.total == rep.iterations * (31 * A.n - 36)
    assert [r for _, r in rep.history] == list(g["ladder_hist"][0, :rep.iterations])
    with pytest.raises(MaxIterationsExceeded) as ei:
        sip_solve(A, a[5], SipConfig(tolerance=1e-14, max_iterations=2))
    assert ei.value.iterations == g["maxit_k"]
    assert np.array_equal(ei.value.best, g["maxit_best"])
    assert ei.value.residual_inf == g["maxit_res"]


def test_ilu0_zero_pivot(cuda):
    p = [x.copy() for x in W.pd_dominant(2, 16, seed=4)]
    p[2][1, 0] = 0.0
    with pytest.raises(ZeroPivot) as ei:
        ilu0_penta(PentaMatrix.from_diagonals(*(x[1] for x in p[:5])))
    assert ei.value.index == 0
    rep = sip_solve(PentaMatrix.from_diagonals(*p[:5]), p[5], SipConfig(tolerance=1e-10))
    assert list(host(rep.status)) == [0, 1] and host(rep.index)[1] == 0


@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("m,rows,alpha", [(3, 20, 0.0), (3, 20, 0.5), (8, 12, 0.0), (8, 12, 0.5),
                                          (16, 16, 0.5), (32, 5, 0.9)])
def test_stencil_sip_matches_c_oracle(cuda, layout, m, rows, alpha):
    n = m * rows
    p = W.five_point(6, n, m, seed=3)
    tol = W.sip_tolerance(p[5])
    ref = cport.sip(*cport.rowaligned_penta(*p[:5], m=m), p[5], tol, m=m, alpha=alpha)
    A = StencilMatrix.from_diagonals(*p[:5], m=m, layout=layout)
    rep = sip_solve(A, p[5], SipConfig(tolerance=tol, max_iterations=500, alpha=alpha))
    assert np.array_equal(host(rep.iterations), ref["iterations"])
    assert np.array_equal(host(rep.x), ref["x"])
    assert np.array_equal(host(rep.residual_inf), ref["residual"])
    # and the numpy restatement agrees with the C one on the factors
    f, _, _ = I.ilu0(*p[:5], m=m, alpha=alpha)
    fg = ilu0_penta(A, alpha=alpha)
    mu = host(fg.u_main.t() if layout == "interleaved" else fg.u_main)
    assert np.array_equal(mu, f["mu"])


@pytest.mark.parametrize("algo", ["sequential", "wavefront"])
@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("m,rows,alpha", [(2, 64, 0.0), (3, 20, 0.5), (8, 12, 0.0), (33, 9, 0.5),
                                          (64, 40, 0.5), (64, 70, 0.0), (128, 20, 0.5),
                                          (256, 6, 0.5), (128, 200, 0.5)])
def test_algorithms_agree(cuda, algo, layout, m, rows, alpha):
    n = m * rows
    p = W.five_point(5, n, m, seed=9)
    tol = W.sip_tolerance(p[5])
    ref = cport.sip(*cport.rowaligned_penta(*p[:5], m=m), p[5], tol, m=m, alpha=alpha)
    A = StencilMatrix.from_diagonals(*p[:5], m=m, layout=layout)
    rep = sip_solve(A, p[5], SipConfig(tolerance=tol, max_iterations=500, alpha=alpha),
                    record_history=True, algo=algo)
    assert np.array_equal(host(rep.iterations), ref["iterations"])
    assert np.array_equal(host(rep.x), ref["x"])
    assert np.array_equal(host(rep.residual_inf), ref["residual"])


def test_wavefront_rejects_non_grid(cuda, golden):
    g = golden("iterative")
    a = [g[f"full_{k}"] for k in PD]
    A = PentaMatrix.from_diagonals(*a[:5])
    rep = sip_solve(A, a[5], SipConfig(tolerance=g["full_tol"]), algo="wavefront")
    assert (host(rep.status) == 7).all()
    rep = sip_solve(A, a[5], SipConfig(tolerance=g["full_tol"]), algo="auto")
    assert np.array_equal(host(rep.x), g["full_x"])


def test_wavefront_maxiter_best_iterate(cuda, golden):
    g = golden("iterative")
    a = [g[f"ladder_{k}"][:1] for k in PD]
    rep = sip_solve(PentaMatrix.from_diagonals(*a[:5]), a[5],
                    SipConfig(tolerance=1e-14, max_iterations=2), algo="wavefront")
    assert host(rep.status)[0] == 3 and host(rep.iterations)[0] == g["maxit_k"]
    assert np.array_equal(host(rep.best_x)[0], g["maxit_best"])


def test_config4_full_wavefront(cuda):
    """Config 4 at full size (B=64, 512x512 grid, alpha=0.5): same iteration
    counts and iterates as the C restatement on sampled systems; every system
    meets the relative 1e-8 stopping rule."""
    p = W.five_point(64, 262144, 512, seed=3)
    tol = W.sip_tolerance(p[5])
    A = StencilMatrix.from_diagonals(*p[:5], m=512, layout="system")
    rep = sip_solve(A, p[5], SipConfig(tolerance=tol, max_iterations=500, alpha=0.5), algo="wavefront")
    assert (host(rep.status) == 0).all()
    assert np.all(host(rep.residual_inf) < tol)
    idx = np.arange(0, 64, 9)
    ref = cport.sip(*cport.rowaligned_penta(*(x[idx] for x in p[:5]), m=512), p[5][idx], tol[idx],
                    m=512, alpha=0.5)
    assert np.array_equal(host(rep.iterations)[idx], ref["iterations"])
    assert np.array_equal(host(rep.x)[idx], ref["x"])


def test_alpha_requires_stride3(cuda):
    from paper_1804_09666_b200.errors import CudaError
    p = W.five_point(1, 64, 2)
    with pytest.raises(CudaError):
        sip_solve(PentaMatrix.from_diagonals(*p[:5]), p[5], SipConfig(tolerance=1e-8, alpha=0.5))


def test_sip_wavefront_is_deterministic(cuda):
    """The wavefront kernel's TMA ring / mbarrier / named-barrier protocol:
    repeated solves give the same bits (race detector substitute)."""
    g = W.five_point(8, 64 * 48, 48, seed=21)
    tol = W.sip_tolerance(g[5])
    S = StencilMatrix.from_diagonals(*g[:5], m=48)
    cfg = SipConfig(tolerance=tol, max_iterations=100, alpha=0.5)
    x0 = sip_solve(S, g[5], cfg, algo="wavefront").x.cpu().numpy()
    for _ in range(8):
        assert np.array_equal(sip_solve(S, g[5], cfg, algo="wavefront").x.cpu().numpy(), x0)


# --------------------------------------------------------------------------
# BX_ALGO_SCAN: correction form + row scans -- the north star's SIP contract
# (iteration count within +-1 of the reference loop, final residual below the
# tolerance), checked against the C restatement
# --------------------------------------------------------------------------
def _true_residual(p, m, x):
    ra = cport.rowaligned_penta(*p[:5], m=m)
    n = x.shape[1]
    ax = ra[2] * x
    ax[:, 1:] += ra[1][:, 1:] * x[:, :-1]
    ax[:, :-1] += ra[3][:, :-1] * x[:, 1:]
    ax[:, m:] += ra[0][:, m:] * x[:, :n - m]
    ax[:, :n - m] += ra[4][:, :n - m] * x[:, m:]
    return np.max(np.abs(p[5] - ax), axis=1)


@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("m,rows,alpha", [(32, 9, 0.5), (64, 40, 0.5), (64, 70, 0.0), (128, 21, 0.5),
                                          (256, 6, 0.5), (96, 33, 0.5), (512, 16, 0.5)])
def test_scan_matches_reference_loop(cuda, layout, m, rows, alpha):
    n = m * rows
    p = W.five_point(5, n, m, seed=9)
    tol = W.sip_tolerance(p[5])
    ref = cport.sip(*cport.rowaligned_penta(*p[:5], m=m), p[5], tol, m=m, alpha=alpha)
    A = StencilMatrix.from_diagonals(*p[:5], m=m, layout=layout)
    rep = sip_solve(A, p[5], SipConfig(tolerance=tol, max_iterations=500, alpha=alpha),
                    record_history=True, algo="scan")
    assert (host(rep.status) == 0).all()
    assert np.all(np.abs(host(rep.iterations) - ref["iterations"]) <= 1)
    x = host(rep.x)
    assert np.all(host(rep.residual_inf) < tol)
    # the reported residual is the residual of the returned iterate
    assert np.allclose(_true_residual(p, m, x), host(rep.residual_inf), rtol=1e-6, atol=1e-18)
    assert np.max(np.abs(x - ref["x"])) <= 1e-7 * np.max(np.abs(ref["x"]))
    # the recorded history ends with the reported residual
    h = host(rep.history)
    for s in range(5):
        k = int(host(rep.iterations)[s])
        if k:
            assert h[s, k - 1] == host(rep.residual_inf)[s]


@pytest.mark.parametrize("m", [64, 256])
def test_scan_maxiter_reports_best_iterate(cuda, m):
    rows = 20
    p = W.five_point(3, m * rows, m, seed=4)
    A = StencilMatrix.from_diagonals(*p[:5], m=m)
    rep = sip_solve(A, p[5], SipConfig(tolerance=1e-300, max_iterations=3, alpha=0.5), algo="scan")
    assert (host(rep.status) == 3).all() and (host(rep.iterations) == 3).all()
    assert np.allclose(_true_residual(p, m, host(rep.best_x)), host(rep.best_residual), rtol=1e-6)


@pytest.mark.parametrize("m", [32, 128])   # one CTA per system / a CTA pair
def test_scan_rejects_non_grid_and_zero_pivot(cuda, m):
    rows = 8
    p = [a.copy() for a in W.five_point(3, m * rows, m, seed=5)]
    p[1][1, m - 1] = 0.3      # A[m, m-1]: a coupling across a grid row
    p[2][2, 0] = 0.0          # a zero leading pivot
    A = StencilMatrix.from_diagonals(*p[:5], m=m)
    rep = sip_solve(A, p[5], SipConfig(tolerance=1e-8, alpha=0.5), algo="scan")
    st = host(rep.status)
    assert st[0] == 0 and st[1] == 7 and st[2] == 1 and host(rep.index)[2] == 0


def test_config4_full_scan(cuda):
    """Config 4 at full size through the scan solver: iteration counts within
    +-1 of the C restatement on all 64 systems, every system below the
    relative 1e-8 stopping rule, the residual recomputed on the host."""
    p = W.five_point(64, 262144, 512, seed=3)
    tol = W.sip_tolerance(p[5])
    A = StencilMatrix.from_diagonals(*p[:5], m=512, layout="system")
    rep = sip_solve(A, p[5], SipConfig(tolerance=tol, max_iterations=500, alpha=0.5), algo="scan")
    assert (host(rep.status) == 0).all()
    assert np.all(host(rep.residual_inf) < tol)
    # every one of the 64 systems against the C restatement of the reference loop
    ref = cport.sip(*cport.rowaligned_penta(*p[:5], m=512), p[5], tol, m=512, alpha=0.5)
    assert np.all(np.abs(host(rep.iterations) - ref["iterations"]) <= 1)
    x = host(rep.x)
    assert np.all(_true_residual(p, 512, x) < tol)
    assert np.max(np.abs(x - ref["x"])) <= 1e-7 * np.max(np.abs(ref["x"]))


@pytest.mark.parametrize("m,rows,bsz", [(128, 64, 100), (256, 32, 200), (128, 8, 1)])
def test_scan_pair_many_clusters_deterministic(cuda, m, rows, bsz):
    """More CTA pairs than SMs, repeated solves: the FIFO / credit protocol of
    the pair kernel gives the same bits every time (race detector substitute)
    and the reference loop's iteration counts +-1."""
    p = W.five_point(bsz, m * rows, m, seed=m + bsz)
    tol = W.sip_tolerance(p[5])
    A = StencilMatrix.from_diagonals(*p[:5], m=m, layout="system")
    ref = cport.sip(*cport.rowaligned_penta(*p[:5], m=m), p[5], tol, m=m, alpha=0.5)
    cfg = SipConfig(tolerance=tol, max_iterations=500, alpha=0.5)
    x0 = host(sip_solve(A, p[5], cfg, algo="scan").x)
    assert np.max(np.abs(x0 - ref["x"])) <= 1e-7 * np.max(np.abs(ref["x"]))
    for _ in range(5):
        rep = sip_solve(A, p[5], cfg, algo="scan")
        assert np.array_equal(host(rep.x), x0)
        assert np.all(np.abs(host(rep.iterations) - ref["iterations"]) <= 1)
