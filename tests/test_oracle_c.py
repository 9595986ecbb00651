"""The C restatement (CPU baseline / reference arm) is pinned bit-for-bit to
the reference golden vectors and to the numpy restatement."""

import numpy as np
import pytest

from oracle import cport
from oracle import iterative as I
from paper_1804_09666_b200 import workloads as W

PD = ("sub2", "sub1", "main", "sup1", "sup2", "rhs")


def test_c_ntdm_golden(golden):
    g = golden("direct")
    d, e, f = cport.rowaligned_tri(g["ntdm_sub1"], g["ntdm_main"], g["ntdm_sup1"])
    x, st, ix = cport.ntdm(d, e, f, g["ntdm_rhs"])
    assert np.array_equal(x, g["ntdm_x"])
    d, e, f = cport.rowaligned_tri(g["ntdmz_sub1"], g["ntdmz_main"], g["ntdmz_sup1"])
    x, st, ix = cport.ntdm(d, e, f, g["ntdmz_rhs"])
    assert np.array_equal(st, g["ntdmz_status"]) and np.array_equal(ix, g["ntdmz_index"])


@pytest.mark.parametrize("tag", ["pd", "pds", "pd3", "pd4", "pd5", "pdz"])
def test_c_penta_golden(golden, tag):
    g = golden("direct")
    a = [g[f"{tag}_{k}"] for k in PD]
    r = cport.rowaligned_penta(*a[:5])
    for mod, kind in ((0, "npdm"), (1, "mnpdm")):
        x, st, ix, nz = cport.penta(mod, *r, a[5])
        assert np.array_equal(x, g[f"{tag}_{kind}_x"], equal_nan=True)


@pytest.mark.parametrize("tag", ["ladder", "full", "holes"])
def test_c_sip_golden(golden, tag):
    g = golden("iterative")
    a = [g[f"{tag}_{k}"] for k in PD]
    r = cport.sip(*cport.rowaligned_penta(*a[:5]), a[5], g[f"{tag}_tol"])
    assert np.array_equal(r["x"], g[f"{tag}_x"])
    assert np.array_equal(r["iterations"], g[f"{tag}_k"])
    assert np.array_equal(r["residual"], g[f"{tag}_res"])


@pytest.mark.parametrize("m,rows,alpha", [(3, 12, 0.5), (8, 10, 0.0), (8, 10, 0.5), (16, 6, 0.9)])
def test_c_sip_stride_matches_numpy(m, rows, alpha):
    p = W.five_point(3, m * rows, m, seed=3)
    tol = W.sip_tolerance(p[5])
    r1 = I.sip(*p, tol=tol, max_iter=500, m=m, alpha=alpha)
    r2 = cport.sip(*cport.rowaligned_penta(*p[:5], m=m), p[5], tol, m=m, alpha=alpha)
    assert np.array_equal(r1["x"], r2["x"])
    assert np.array_equal(r1["iterations"], r2["iterations"])
