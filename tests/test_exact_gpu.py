"""GPU parity of the symbolic solvers (STDM/SPDM): against the reference's own
exact results at small N (golden vectors) and against the high-precision
limit oracle at config-3 size; substitution counts must be identical."""

import numpy as np
import pytest

from oracle.exact import limit_solve_mp
from paper_1804_09666_b200 import (PentaMatrix, SingularMatrix, TriMatrix, exact_solve_spdm,
                                   exact_solve_stdm)
from paper_1804_09666_b200 import workloads as W

pytestmark = pytest.mark.gpu
REL_TOL = 1e-10   # north_star: max relative error <= 1e-10 for the symbolic solvers
PD = ("sub2", "sub1", "main", "sup1", "sup2", "rhs")


def host(t):
    return t.detach().cpu().numpy()


def rel(x, ref):
    return np.max(np.abs(x - ref)) / np.max(np.abs(ref))


@pytest.mark.parametrize("layout", ["interleaved", "system"])
def test_stdm_golden(cuda, golden, layout):
    g = golden("exact")
    t = TriMatrix.from_diagonals(g["stdm_sub1"], g["stdm_main"], g["stdm_sup1"], layout=layout)
    r = exact_solve_stdm(t, g["stdm_rhs"])
    assert (host(r.status) == 0).all()
    assert np.array_equal(host(r.pivot_substitutions), g["stdm_subs"])
    for s in range(3):
        assert rel(host(r.x)[s], g["stdm_x"][s]) <= 1e-13
    t0 = TriMatrix.from_diagonals(g["stdm0_sub1"], g["stdm0_main"], g["stdm0_sup1"], layout=layout)
    r0 = exact_solve_stdm(t0, g["stdm0_rhs"])
    assert np.array_equal(host(r0.pivot_substitutions), g["stdm0_subs"])
    assert rel(host(r0.x), g["stdm0_x"]) <= 1e-12


@pytest.mark.parametrize("layout", ["interleaved", "system"])
def test_spdm_golden(cuda, golden, layout):
    g = golden("exact")
    a = [g[f"spdm_{k}"] for k in PD]
    A = PentaMatrix.from_diagonals(*a[:5], layout=layout)
    r = exact_solve_spdm(A, a[5])
    assert (host(r.status) == 0).all()
    assert np.array_equal(host(r.pivot_substitutions), g["spdm_subs"])
    for s in range(2):
        assert rel(host(r.x)[s], g["spdm_x"][s]) <= 1e-13


def test_single_system_contract(cuda, golden):
    g = golden("exact")
    t = TriMatrix.from_diagonals(g["stdm_sub1"][0], g["stdm_main"][0], g["stdm_sup1"][0])
    r = exact_solve_stdm(t, g["stdm_rhs"][0])
    assert isinstance(r.x, np.ndarray) and r.pivot_substitutions == g["stdm_subs"][0]
    sing = TriMatrix.from_diagonals([1.0, 1.0], [1.0, 1.0, 1.0], [1.0, 0.0])
    assert g["det_singular"] == 0.0
    with pytest.raises(SingularMatrix):
        exact_solve_stdm(sing, [1.0, 2.0, 3.0])
    # last row decoupled: exactly singular
    d = W.td_symbolic(1, 16, seed=5, zeros=0)
    sub1, main, sup1, rhs = (x.copy() for x in d[:4])
    sub1[0, -1] = 0.0
    main[0, -1] = 0.0
    with pytest.raises(SingularMatrix):
        exact_solve_stdm(TriMatrix.from_diagonals(sub1[0], main[0], sup1[0]), rhs[0])


@pytest.mark.parametrize("kind", ["td", "pd"])
def test_config3_full_size(cuda, kind):
    """B=4096, N=2048, 8 decoupled zero pivots per system (config 3)."""
    if kind == "td":
        *p, rows = W.td_symbolic(4096, 2048, seed=2)
        A = TriMatrix.from_diagonals(*p[:3], layout="system")
        r = exact_solve_stdm(A, p[3])
        offs = [-1, 0, 1]
        nd = 3
    else:
        *p, rows = W.pd_symbolic(4096, 2048, seed=2)
        A = PentaMatrix.from_diagonals(*p[:5], layout="system")
        r = exact_solve_spdm(A, p[5])
        offs = [-2, -1, 0, 1, 2]
        nd = 5
    st = host(r.status)
    assert (st == 0).all(), np.unique(st, return_counts=True)
    assert (host(r.pivot_substitutions) == 8).all()
    x = host(r.x)
    for s in range(0, 4096, 512):
        ref = limit_solve_mp([q[s] for q in p[:nd]], offs, p[nd][s])
        assert rel(x[s], ref) <= REL_TOL, (s, rel(x[s], ref))
