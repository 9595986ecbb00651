"""GPU parity of pd_to_td / solve_pd2td_ntdm (direct.py:116-177): bit-identical
to the reference's own outputs (golden) and to the restatement at scale."""

import numpy as np
import pytest

from oracle import direct as D
from paper_1804_09666_b200 import (PentaMatrix, ReductionPivotZero, ZeroPivot, pd_to_td,
                                   solve_pd2td_ntdm)
from paper_1804_09666_b200 import workloads as W

pytestmark = pytest.mark.gpu
PD = ("sub2", "sub1", "main", "sup1", "sup2", "rhs")
TAGS = ["dense", "sparse", "n3", "n4", "n5", "fail"]


def host(t):
    return t.detach().cpu().numpy()


@pytest.mark.parametrize("layout", ["interleaved", "system"])
@pytest.mark.parametrize("tag", TAGS)
def test_pd2td_golden(cuda, golden, tag, layout):
    g = golden("pd2td")
    p = [g[f"{tag}_{k}"] for k in PD]
    A = PentaMatrix.from_diagonals(*p[:5], layout=layout)
    red = pd_to_td(A, p[5])
    st = host(red.status)
    ok = g[f"{tag}_status"] != 8
    assert np.array_equal(st != 0, ~ok)
    assert np.array_equal(host(red.index)[~ok], g[f"{tag}_index"][~ok])
    assert np.array_equal(host(red.tri.sub1)[ok], g[f"{tag}_td"][ok])
    assert np.array_equal(host(red.tri.main)[ok], g[f"{tag}_te"][ok])
    assert np.array_equal(host(red.tri.sup1)[ok], g[f"{tag}_tf"][ok])
    assert np.array_equal(host(red.rhs)[ok], g[f"{tag}_tr"][ok])
    ops = np.stack([host(red.ops.muls), host(red.ops.subs), host(red.ops.divs)], axis=1)
    assert np.array_equal(ops[ok], g[f"{tag}_ops"][ok])
    rep = solve_pd2td_ntdm(A, p[5])
    assert np.array_equal(host(rep.x), g[f"{tag}_x"], equal_nan=True)
    assert np.array_equal(host(rep.status), g[f"{tag}_status"])
    assert np.array_equal(host(rep.index), g[f"{tag}_index"])
    good = g[f"{tag}_status"] == 0
    assert np.array_equal(host(rep.residual_inf)[good], g[f"{tag}_res"][good])
    assert np.array_equal(host(rep.ops.total)[good], g[f"{tag}_tot"][good])


def test_pd2td_single_system_raises(cuda, golden):
    g = golden("pd2td")
    p = [g[f"fail_{k}"] for k in PD]
    one = lambda s: [a[s] for a in p]  # noqa: E731
    with pytest.raises(ReductionPivotZero) as e:
        pd_to_td(PentaMatrix.from_diagonals(*one(0)[:5]), one(0)[5])
    assert e.value.index == 2
    with pytest.raises(ReductionPivotZero) as e:
        solve_pd2td_ntdm(PentaMatrix.from_diagonals(*one(1)[:5]), one(1)[5])
    assert e.value.index == 21
    with pytest.raises(ZeroPivot) as e:
        solve_pd2td_ntdm(PentaMatrix.from_diagonals(*one(2)[:5]), one(2)[5])
    assert e.value.index == 0
    tri, rhs, ops = pd_to_td(PentaMatrix.from_diagonals(*one(3)[:5]), one(3)[5])
    assert np.array_equal(np.asarray(tri.main[0].cpu()), g["fail_te"][3])
    assert (ops.muls, ops.subs, ops.divs) == tuple(int(v) for v in g["fail_ops"][3])
    rep = solve_pd2td_ntdm(PentaMatrix.from_diagonals(*one(3)[:5]), one(3)[5])
    assert np.array_equal(rep.x, g["fail_x"][3])


@pytest.mark.parametrize("sparse", [False, True])
def test_pd2td_config2_sample_vs_restatement(cuda, sparse):
    """Config-2 shape (N = 4096), full and sparse outer: bit-identical to the
    restatement (itself pinned to the reference above)."""
    p = W.pd_dominant(64, 4096, seed=1, sparse_outer=sparse)
    x_ref, st_ref, ix_ref, ops_ref = D.pd2td_ntdm(*p)
    for layout in ("interleaved", "system"):
        rep = solve_pd2td_ntdm(PentaMatrix.from_diagonals(*p[:5], layout=layout), p[5])
        assert np.array_equal(host(rep.x), x_ref)
        assert (host(rep.status) == 0).all()
        red_total = ops_ref.sum(axis=1) + 9 * 4096 - 7
        assert np.array_equal(host(rep.ops.total), red_total)
