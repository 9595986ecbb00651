"""Band building blocks through the C ABI, against the oracle restatement of
the reference (bit-identical: same operation order, one rounding each):
lu_penta (direct.py:42-63), forward_sub / backward_sub (iterative.py:127-149),
penta_matvec / tri_matvec / residual / inf_norm / outer_nonzero_count
(core.py:243-334); factor once, solve many right-hand sides."""
import numpy as np
import pytest
import torch

from oracle import direct as D
from paper_1804_09666_b200 import (CounterBox, PentaMatrix, StencilMatrix, TriMatrix, ZeroPivot,
                                   backward_sub, backward_sub_batched, forward_sub, ilu0_penta,
                                   inf_norm, lu_penta, matvec, outer_nonzero_count, penta_matvec,
                                   residual, solve_npdm, tri_matvec)
from paper_1804_09666_b200 import workloads as W

pytestmark = pytest.mark.gpu
LAYOUTS = ["interleaved", "system"]


def host(t):
    return t.detach().cpu().numpy()


@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("n", [3, 4, 5, 257])
def test_lu_penta_bitexact(cuda, layout, n):
    p = W.pd_dominant(6, n, seed=n)
    mu, l1, l2, phi, psi, st, ix = D.penta_factor(*p[:5])
    f = lu_penta(PentaMatrix.from_diagonals(*p[:5], layout=layout))
    assert (host(f.status) == 0).all()
    rl1, rl2, rmu, rphi, rpsi = (host(v) for v in f.ref())
    assert np.array_equal(rmu, mu)
    assert np.array_equal(rl1, l1[:, 1:]) and np.array_equal(rl2, l2[:, 2:])
    assert np.array_equal(rphi, phi[:, :n - 1]) and np.array_equal(rpsi, psi[:, :n - 2])


@pytest.mark.parametrize("layout", LAYOUTS)
def test_factor_once_solve_many(cuda, layout):
    """lu_penta + forward_sub + backward_sub == solve_npdm (the reference's
    composition, direct.py:73-81) bit for bit, for several right-hand sides."""
    n = 1000
    p = W.pd_dominant(8, n, seed=7)
    A = PentaMatrix.from_diagonals(*p[:5], layout=layout)
    f = lu_penta(A)
    rng = np.random.default_rng(0)
    for _ in range(3):
        b = rng.uniform(-1, 1, (8, n))
        x_ref, _, _ = D.npdm(*p[:5], b)
        y = forward_sub(f, b)
        x, st, ix = backward_sub_batched(f, y)
        assert np.array_equal(host(x), x_ref)
        assert (host(st) == 0).all()
        assert np.array_equal(host(solve_npdm(A, b).x), x_ref)
    # the oracle's own sweeps on the oracle's factors
    mu, l1, l2, phi, psi, _, _ = D.penta_factor(*p[:5])
    assert np.array_equal(host(forward_sub(f, b)), D.penta_forward(l1, l2, b))


def test_single_system_api_and_zero_pivot(cuda):
    p = [a[:1].copy() for a in W.pd_dominant(1, 50, seed=3)]
    A = PentaMatrix.from_diagonals(*(a[0] for a in p[:5]))
    box = CounterBox()
    f = lu_penta(A, box)
    y = forward_sub(f, p[5][0], box)
    x = backward_sub(f, y, box)
    x_ref, _, _ = D.npdm(*p)
    assert isinstance(x, np.ndarray) and np.array_equal(x, x_ref[0])
    assert box.counter.total == 19 * 50 - 29        # 10N-17 + 4N-6 + 5N-6
    q = [a.copy() for a in p]
    q[2][0, 0] = 0.0
    with pytest.raises(ZeroPivot) as e:
        lu_penta(PentaMatrix.from_diagonals(*(a[0] for a in q[:5])))
    assert e.value.index == 0


@pytest.mark.parametrize("m,alpha", [(2, 0.0), (16, 0.5)])
def test_sweeps_on_ilu0_factors(cuda, m, alpha):
    """forward_sub / backward_sub on ILU(0) factors of a stride-m five-point
    band: the oracle's sweeps with the same factors, bit for bit."""
    rows = 24
    n = m * rows
    g = W.five_point(4, n, m, seed=5)
    S = StencilMatrix.from_diagonals(*g[:5], m=m)
    f = ilu0_penta(S, alpha=alpha)
    y = host(forward_sub(f, g[5]))
    x, st, _ = backward_sub_batched(f, y)
    # reference recurrences with the device factors (row-aligned)
    l1, l2, mu, phi, psi = (host(v).T if f.layout == 0 else host(v)
                            for v in (f.l_sub1, f.l_sub2, f.u_main, f.u_sup1, f.u_sup2))
    b = g[5]
    yr = np.empty_like(b)
    yr[:, 0] = b[:, 0]
    for i in range(1, n):
        yr[:, i] = b[:, i] - l1[:, i] * yr[:, i - 1]
        if i >= m:
            yr[:, i] = yr[:, i] - l2[:, i] * yr[:, i - m]
    assert np.array_equal(y, yr)
    xr = np.empty_like(b)
    xr[:, n - 1] = yr[:, n - 1] / mu[:, n - 1]
    for i in range(n - 2, -1, -1):
        v = yr[:, i] - phi[:, i] * xr[:, i + 1]
        if i <= n - 1 - m:
            v = v - psi[:, i] * xr[:, i + m]
        xr[:, i] = v / mu[:, i]
    assert np.array_equal(host(x), xr) and (host(st) == 0).all()


@pytest.mark.parametrize("layout", LAYOUTS)
def test_matvec_residual_norm(cuda, layout):
    n = 300
    p = W.pd_dominant(5, n, seed=2)
    A = PentaMatrix.from_diagonals(*p[:5], layout=layout)
    x = np.random.default_rng(1).uniform(-1, 1, (5, n))
    assert np.array_equal(host(penta_matvec(A, x)), D.penta_matvec(*p[:5], x))
    assert np.array_equal(host(matvec(A, x)), D.penta_matvec(*p[:5], x))
    r = residual(A, x, p[5])
    assert np.array_equal(host(r), p[5] - D.penta_matvec(*p[:5], x))
    assert np.array_equal(host(inf_norm(r)), D.residual_inf_penta(*p[:5], x, p[5]))
    t = W.td_dominant(5, n, seed=2)
    T = TriMatrix.from_diagonals(*t[:3], layout=layout)
    assert np.array_equal(host(tri_matvec(T, x)), D.tri_matvec(*t[:3], x))
    box = CounterBox()
    residual(T, x, t[3], box)
    assert (box.counter.muls, box.counter.adds, box.counter.subs) == (3 * n - 2, 2 * n - 2, n)
    assert inf_norm([]) == 0 and inf_norm(np.array([1.0, -3.0])) == 3.0


def test_outer_nonzero_count(cuda):
    p = W.pd_dominant(3, 40, seed=4, sparse_outer=True)
    A = PentaMatrix.from_diagonals(*p[:5])
    k = host(outer_nonzero_count(A))
    assert k.tolist() == [int(np.count_nonzero(p[0][s]) + np.count_nonzero(p[4][s])) for s in range(3)]
    A1 = PentaMatrix.from_diagonals(*(a[0] for a in p[:5]))
    assert outer_nonzero_count(A1) == int(np.count_nonzero(p[0][0]) + np.count_nonzero(p[4][0]))
