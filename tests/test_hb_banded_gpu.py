"""GPU parity of the banded Hotelling-Bodewig path:
hb_invert_banded and sip_hb_solve(mode="banded") against the reference's own
outputs (tests/golden/hbband.npz, bit for bit) and, for the automatic width
(true-residual widening), against the oracle restatement."""

import numpy as np
import pytest

from oracle import inverse as H
from oracle.iterative import ilu0
from paper_1804_09666_b200 import (MaxIterationsExceeded, PentaMatrix, SipConfig, Stagnated,
                                   hb_invert_banded, ilu0_penta, sip_hb_solve)
from paper_1804_09666_b200 import workloads as W

pytestmark = pytest.mark.gpu
HBB = ("sub2", "sub1", "main", "sup1", "sup2", "rhs")


def host(t):
    return t.detach().cpu().numpy()


@pytest.mark.parametrize("layout", ["interleaved", "system"])
def test_hb_invert_banded_golden(cuda, golden, layout):
    g = golden("hbband")
    p = [g[f"hbb_{k}"] for k in HBB]
    fac = ilu0_penta(PentaMatrix.from_diagonals(*p[:5], layout=layout))
    for side in ("lower", "upper"):
        for w in (2, 3, 6):
            for t in ("d", "t"):
                tol = np.full(2, 1e-12) if t == "d" else g["hbb_tol"]
                rep = hb_invert_banded(fac, side, w, tol)
                xd = host(rep.inverse.diags)
                for s in range(2):
                    key = f"inv_{s}_{side}_{w}_{t}"
                    gx = g[key + "_x"]
                    for j in range(w + 1):
                        assert np.array_equal(xd[s, j, :p[2].shape[1] - j], gx[j, :p[2].shape[1] - j])
                    assert int(rep.iterations[s]) == g[key + "_it"]
                    assert float(rep.residual_inf[s]) == g[key + "_res"]
                    assert int(rep.status[s]) == g[key + "_st"]
                    h = host(rep.residual_history[s])
                    assert np.array_equal(h[~np.isnan(h)], g[key + "_hist"])


def test_hb_invert_banded_single_contract(cuda, golden):
    g = golden("hbband")
    p = [g[f"hbb_{k}"] for k in HBB]
    fac = ilu0_penta(PentaMatrix.from_diagonals(*[d[0] for d in p[:5]]))
    rep = hb_invert_banded(fac, "upper", 3, float(g["hbb_tol"][0]))
    assert rep.iterations == g["inv_0_upper_3_t_it"] and rep.residual_inf == g["inv_0_upper_3_t_res"]
    v = np.linspace(-1.0, 1.0, p[2].shape[1])
    gx = g["inv_0_upper_3_t_x"]
    ref = H.band_matvec([gx[j, :p[2].shape[1] - j] for j in range(4)], "upper", v)
    assert np.array_equal(host(rep.inverse.matvec(v)), ref)
    # a stagnating factor raises Stagnated carrying the best report: an
    # iteration capped before convergence with an impossible tolerance
    with pytest.raises((Stagnated, MaxIterationsExceeded)):
        hb_invert_banded(fac, "lower", 2, 0.0, max_iter=6)


@pytest.mark.parametrize("w", [3, 6, 12])
def test_sip_hb_banded_explicit_width_golden(cuda, golden, w):
    """explicit hb_bandwidth: same best iterate / count / residual as the
    reference, which stalls (MaxIterationsExceeded) at these widths."""
    g = golden("hbband")
    p = [g[f"hbb_{k}"] for k in HBB]
    A = PentaMatrix.from_diagonals(*p[:5])
    rep = sip_hb_solve(A, p[5], SipConfig(tolerance=g["hbb_tol"], max_iterations=60), mode="banded",
                       hb_bandwidth=w)
    for s in range(2):
        key = f"sip_{s}_{w}"
        assert int(rep.status[s]) == g[key + "_st"]
        assert np.array_equal(host(rep.best_x[s]), g[key + "_x"])
        assert int(rep.iterations[s]) == g[key + "_k"]
        assert float(rep.best_residual[s]) == g[key + "_res"]
    with pytest.raises(MaxIterationsExceeded):
        sip_hb_solve(PentaMatrix.from_diagonals(*[d[0] for d in p[:5]]), p[5][0],
                     SipConfig(tolerance=float(g["hbb_tol"][0]), max_iterations=60),
                     mode="banded", hb_bandwidth=w)


@pytest.mark.parametrize("n,bsz", [(128, 2), (2048, 8)])
def test_sip_hb_banded_auto_width(cuda, n, bsz):
    """automatic width: true-residual widening converges (the reference's
    never widens and stalls); iterates, counts and widths equal
    the oracle restatement bit for bit."""
    p = W.five_point(bsz, n, 2, seed=3)
    tol = W.sip_tolerance(p[5])
    rep = sip_hb_solve(PentaMatrix.from_diagonals(*p[:5], layout="system"), p[5],
                       SipConfig(tolerance=tol, max_iterations=200), mode="banded")
    o = H.sip_hb_banded(*p, tol, 200, w=None, cap=256)
    assert (host(rep.status) == 0).all()
    assert np.array_equal(host(rep.iterations), o["iterations"])
    assert np.array_equal(host(rep.hb_bandwidth), o["inv_w"])
    assert np.array_equal(host(rep.x), o["x"])
    assert (host(rep.residual_inf) < tol).all()


def test_sip_hb_banded_width32_converges_golden(cuda, golden):
    """hb_bandwidth=32: the reference converges (k = 6); same iterate bits,
    count, residual and op tally (band applies, inverse.py:48-61)."""
    g = golden("hbband")
    p = [g[f"hbb_{k}"] for k in HBB]
    A = PentaMatrix.from_diagonals(*p[:5])
    rep = sip_hb_solve(A, p[5], SipConfig(tolerance=g["hbb_tol"], max_iterations=60), mode="banded",
                       hb_bandwidth=32)
    for s in range(2):
        key = f"sip_{s}_32"
        assert int(rep.status[s]) == 0 == int(g[key + "_st"])
        assert np.array_equal(host(rep.x[s]), g[key + "_x"])
        assert int(rep.iterations[s]) == g[key + "_k"]
        assert float(rep.residual_inf[s]) == float(g[key + "_res"])
        assert [int(rep.ops.adds[s]), int(rep.ops.subs[s]), int(rep.ops.muls[s]),
                int(rep.ops.divs)] == g[key + "_ops"].tolist()
