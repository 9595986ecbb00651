"""The oracle is pinned to the reference: golden vectors produced by running
bandix 0.1.0 itself (tests/golden/make_golden.py) must be reproduced
BIT-FOR-BIT by the batched restatement."""

import numpy as np
import pytest

from oracle import STATUS_MAX_ITER, STATUS_ZERO_PIVOT
from oracle import direct as D
from oracle import inverse as H
from oracle import iterative as I

PD = ("sub2", "sub1", "main", "sup1", "sup2", "rhs")


def eq(a, b):
    return np.array_equal(a, b, equal_nan=True)


def test_ntdm_config1_sample(golden):
    g = golden("direct")
    x, st, ix = D.ntdm(g["ntdm_sub1"], g["ntdm_main"], g["ntdm_sup1"], g["ntdm_rhs"])
    assert eq(x, g["ntdm_x"])
    res = D.residual_inf_tri(g["ntdm_sub1"], g["ntdm_main"], g["ntdm_sup1"], x, g["ntdm_rhs"])
    assert eq(res, g["ntdm_res"])
    n = x.shape[1]
    assert sum(D.ops_ntdm(n).values()) == g["ntdm_ops"][0] == 9 * n - 7


def test_ntdm_spec_and_edges(golden):
    g = golden("direct")
    x, *_ = D.ntdm([[-1.0, -1.0]], [[2.0, 2.0, 2.0]], [[-1.0, -1.0]], [[1.0, 0.0, 1.0]])
    assert eq(x, g["ntdm_spec_x"]) and np.allclose(x, 1.0)
    x, *_ = D.ntdm(g["ntdm2_sub1"], g["ntdm2_main"], g["ntdm2_sup1"], g["ntdm2_rhs"])
    assert eq(x, g["ntdm2_x"])


def test_ntdm_zero_pivots(golden):
    g = golden("direct")
    x, st, ix = D.ntdm(g["ntdmz_sub1"], g["ntdmz_main"], g["ntdmz_sup1"], g["ntdmz_rhs"])
    assert eq(st, g["ntdmz_status"]) and eq(ix, g["ntdmz_index"])
    assert list(st) == [STATUS_ZERO_PIVOT, STATUS_ZERO_PIVOT, 0] and list(ix) == [0, 5, -1]
    assert eq(x, g["ntdmz_x"])


@pytest.mark.parametrize("tag", ["pd", "pds", "pd3", "pd4", "pd5", "pdz"])
def test_penta_direct(golden, tag):
    g = golden("direct")
    a = [g[f"{tag}_{k}"] for k in PD]
    x, st, ix = D.npdm(*a)
    x2, st2, ix2, nz = D.mnpdm(*a)
    assert eq(x, g[f"{tag}_npdm_x"])
    assert eq(x2, g[f"{tag}_mnpdm_x"])
    if tag == "pdz":
        assert eq(st, g["pdz_npdm_status"]) and eq(ix, g["pdz_npdm_index"])
        assert eq(st2, g["pdz_mnpdm_status"]) and eq(ix2, g["pdz_mnpdm_index"])
    if tag in ("pd", "pds"):
        n = x.shape[1]
        assert sum(D.ops_npdm(n).values()) == g[f"{tag}_npdm_ops"][0] == 19 * n - 29
        assert sum(D.ops_mnpdm(n, int(nz[0])).values()) == g[f"{tag}_mnpdm_ops"][0]
        res = D.residual_inf_penta(*a[:5], x, a[5])
        assert eq(res, g[f"{tag}_npdm_res"])
    if tag == "pds":
        assert (nz == 2).all()


@pytest.mark.parametrize("tag", ["ladder", "full", "holes"])
def test_ilu0_defect_sip(golden, tag):
    g = golden("iterative")
    a = [g[f"{tag}_{k}"] for k in PD]
    n = a[2].shape[1]
    f, st, ix = I.ilu0(*a[:5], m=2)
    assert eq(f["l1"][:, 1:], g[f"{tag}_l_sub1"]) and eq(f["l2"][:, 2:], g[f"{tag}_l_sub2"])
    assert eq(f["mu"], g[f"{tag}_u_main"])
    assert eq(f["phi"][:, :n - 1], g[f"{tag}_u_sup1"]) and eq(f["psi"][:, :n - 2], g[f"{tag}_u_sup2"])
    k = I.defect(f, *a[:5])
    assert eq(k[-2][:, 2:], g[f"{tag}_k_sub2"]) and eq(k[-1][:, 1:], g[f"{tag}_k_sub1"])
    assert eq(k[0], g[f"{tag}_k_main"])
    assert eq(k[1][:, :n - 1], g[f"{tag}_k_sup1"]) and eq(k[2][:, :n - 2], g[f"{tag}_k_sup2"])
    r = I.sip(*a, tol=g[f"{tag}_tol"], max_iter=500, record_history=True)
    assert eq(r["x"], g[f"{tag}_x"])
    assert eq(r["iterations"], g[f"{tag}_k"])
    assert eq(r["residual"], g[f"{tag}_res"])
    hist = np.stack(r["history"], axis=1)
    kmax = hist.shape[1]
    assert eq(hist, g[f"{tag}_hist"][:, :kmax])


def test_sip_max_iterations(golden):
    g = golden("iterative")
    a = [g[f"ladder_{k}"][:1] for k in PD]
    r = I.sip(*a, tol=1e-14, max_iter=2)
    assert r["status"][0] == STATUS_MAX_ITER and r["iterations"][0] == g["maxit_k"]
    assert eq(r["best_x"][0], g["maxit_best"]) and r["best_residual"][0] == g["maxit_res"]


def test_hb_dense(golden):
    g = golden("inverse")
    a = [g[f"hb_{k}"] for k in PD]
    r = H.sip_hb(*a, tol=g["hb_tol"], max_iter=500)
    assert eq(r["iterations"], g["hb_k"])
    assert eq(r["inv_iterations"][:, 0], g["hb_linv_iters"])
    assert eq(r["inv_iterations"][:, 1], g["hb_uinv_iters"])
    # BLAS-ordered products: tolerance, not bits
    assert np.abs(r["x"] - g["hb_x"]).max() <= 1e-12 * np.abs(g["hb_x"]).max()
    x, it, res, hist, st = H.hb_invert_dense(np.array([[1.0, 0.0], [3.0, 1.0]]))
    assert it == g["hb_spec_iters"] == 1 and eq(x, g["hb_spec_inv"])


PD2TD_TAGS = ["dense", "sparse", "n3", "n4", "n5", "fail"]


@pytest.mark.parametrize("tag", PD2TD_TAGS)
def test_pd2td_restatement(golden, tag):
    """pd_to_td + solve_pd2td_ntdm restatement == the reference, bit for bit
    (reduced diagonals, rhs, per-system op tallies, x, ReductionPivotZero /
    ZeroPivot rows)."""
    from oracle import direct as D
    g = golden("pd2td")
    p = [g[f"{tag}_{k}"] for k in ("sub2", "sub1", "main", "sup1", "sup2", "rhs")]
    d, e, f, r, ops, st, ix = D.pd_to_td(*p)
    red_ok = g[f"{tag}_status"] != 8
    for a, k in ((d, "td"), (e, "te"), (f, "tf"), (r, "tr")):
        assert np.array_equal(a[red_ok], g[f"{tag}_{k}"][red_ok])
    assert np.array_equal(ops[red_ok], g[f"{tag}_ops"][red_ok])
    x, st2, ix2, _ = D.pd2td_ntdm(*p)
    assert np.array_equal(x, g[f"{tag}_x"], equal_nan=True)
    assert np.array_equal(st2, g[f"{tag}_status"]) and np.array_equal(ix2, g[f"{tag}_index"])
    ok = st2 == 0
    n = p[2].shape[1]
    # report op total = reduction + NTDM 9N-7 (direct.py:176)
    assert np.array_equal(ops[ok].sum(axis=1) + 9 * n - 7, g[f"{tag}_tot"][ok])


DET_CASES = [("tds", 3), ("td0", 3), ("tdd", 3), ("pds", 5), ("pd0", 5), ("pdd", 5)]


@pytest.mark.parametrize("tag,nd", DET_CASES)
def test_det_band_oracle(golden, tag, nd):
    """oracle det_band_mp (pivoted, 60 digits) reproduces the reference's exact
    determinant (exact_det_band, rounded to binary64) and its op counts."""
    from oracle.exact import det_band_mp
    g = golden("det")
    offs = [-1, 0, 1] if nd == 3 else [-2, -1, 0, 1, 2]
    n = g[f"{tag}_d{nd // 2}"].shape[1]
    for s in range(g[f"{tag}_mant"].shape[0]):
        diags = [g[f"{tag}_d{k}"][s] for k in range(nd)]
        # reference-length diagonals (golden stores the reference's arrays)
        m, e = det_band_mp(diags, offs)
        assert e == g[f"{tag}_expo"][s]
        assert abs(m - g[f"{tag}_mant"][s]) <= 2 * np.spacing(abs(g[f"{tag}_mant"][s]))
        ops = (4 * n - 7 + (n - 1)) + (4 * n - 7) + (2 * n - 3) if nd == 5 else \
            (2 * n - 2 + (n - 1)) + (n - 1) + n
        assert ops == g[f"{tag}_ops"][s]
    assert g["sing_mant"] == 0.0


HBB = ("sub2", "sub1", "main", "sup1", "sup2", "rhs")


def test_hb_banded_restatement(golden):
    """oracle hb_invert_banded reproduces the reference's banded HB bit for bit
    (inverse, iterations, residual, history, status) on both factors, widths
    2/3/6, two tolerances."""
    from oracle.iterative import ilu0
    g = golden("hbband")
    p = [g[f"hbb_{k}"] for k in HBB]
    f, _, _ = ilu0(*p[:5], 2, 0.0)
    for s in range(2):
        for side in ("lower", "upper"):
            for w in (2, 3, 6):
                for t in ("d", "t"):
                    tl = 1e-12 if t == "d" else float(g["hbb_tol"][s])
                    key = f"inv_{s}_{side}_{w}_{t}"
                    x, it, r, h, st = H.hb_invert_banded(H.factor_diags(f, s, side), side, w, tl)
                    gx = g[key + "_x"]
                    for j in range(w + 1):
                        assert eq(x[j], gx[j, :len(x[j])])
                    assert it == g[key + "_it"] and r == g[key + "_res"] and st == g[key + "_st"]
                    assert eq(np.asarray(h), g[key + "_hist"])


def test_sip_hb_banded_restatement(golden):
    """explicit-width SIP-HB (mode="banded"): the reference stalls at
    MaxIterationsExceeded; the restatement returns the same best iterate,
    count and residual bit for bit."""
    g = golden("hbband")
    p = [g[f"hbb_{k}"] for k in HBB]
    for w in (3, 6, 12):
        o = H.sip_hb_banded(*p, g["hbb_tol"], 60, w=w)
        for s in range(2):
            key = f"sip_{s}_{w}"
            assert o["status"][s] == g[key + "_st"] == STATUS_MAX_ITER
            assert eq(o["best_x"][s], g[key + "_x"])
            assert o["iterations"][s] == g[key + "_k"]
            assert o["best_residual"][s] == g[key + "_res"]
    # the reference's auto mode never widens and stalls too
    assert g["sip_0_auto_st"] == STATUS_MAX_ITER and g["sip_1_auto_st"] == STATUS_MAX_ITER
    # this build's true-residual widening converges
    o = H.sip_hb_banded(*p, g["hbb_tol"], 60, w=None)
    assert (o["status"] == 0).all() and (o["residual"] < g["hbb_tol"]).all()


# the 50-digit pivoted limit solve that stands in for the reference's exact
# solvers at config-3 size (tests/test_exact_gpu.py) is pinned to the
# reference's own exact results: exact.npz and the wider round-2 set exact2.npz
@pytest.mark.parametrize("name,tag,nd", [("exact2", "td_a", 3), ("exact2", "td_b", 3), ("exact2", "td_c", 3),
                                         ("exact2", "pd_a", 5), ("exact2", "pd_b", 5), ("exact2", "pd_c", 5)])
def test_limit_solve_oracle_reproduces_reference_exact_solves(golden, name, tag, nd):
    from oracle.exact import limit_solve_mp
    g = golden(name)
    d = [g[f"{tag}_in{j}"] for j in range(nd + 1)]
    offs = [-1, 0, 1] if nd == 3 else [-2, -1, 0, 1, 2]
    for s in range(d[0].shape[0]):
        x = limit_solve_mp([q[s] for q in d[:nd]], offs, d[nd][s])
        ref = g[f"{tag}_x"][s]
        assert np.max(np.abs(x - ref)) <= 1e-14 * np.max(np.abs(ref)), (tag, s)


def test_limit_solve_oracle_first_golden_set(golden):
    from oracle.exact import limit_solve_mp
    g = golden("exact")
    for s in range(3):
        x = limit_solve_mp([g["stdm_sub1"][s], g["stdm_main"][s], g["stdm_sup1"][s]], [-1, 0, 1],
                           g["stdm_rhs"][s])
        assert np.max(np.abs(x - g["stdm_x"][s])) <= 1e-14 * np.max(np.abs(g["stdm_x"][s]))
    keys = ("sub2", "sub1", "main", "sup1", "sup2")
    for s in range(2):
        x = limit_solve_mp([g[f"spdm_{k}"][s] for k in keys], [-2, -1, 0, 1, 2], g["spdm_rhs"][s])
        assert np.max(np.abs(x - g["spdm_x"][s])) <= 1e-14 * np.max(np.abs(g["spdm_x"][s]))
