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
    # 128 of the 4096 systems against the 50-digit pivoted oracle (itself pinned
    # to the reference's exact results, tests/test_oracle_golden.py); round 1
    # sampled 8
    for s in range(0, 4096, 32):
        ref = limit_solve_mp([q[s] for q in p[:nd]], offs, p[nd][s])
        assert rel(x[s], ref) <= REL_TOL, (s, rel(x[s], ref))


DET_CASES = [("tds", 3), ("td0", 3), ("tdd", 3), ("pds", 5), ("pd0", 5), ("pdd", 5)]


def _det_rel(res, s, m_ref, e_ref):
    """relative error of det[s] = m * 2^e against m_ref * 2^e_ref"""
    m = float(res.mantissa[s]) * 2.0 ** (int(res.exponent[s]) - int(e_ref))
    return abs(m - m_ref) / abs(m_ref)


@pytest.mark.parametrize("layout", ["interleaved", "system"])
@pytest.mark.parametrize("tag,nd", DET_CASES)
def test_det_band_golden(cuda, golden, layout, tag, nd):
    """exact_det_band against the reference's exact determinants (golden)."""
    from paper_1804_09666_b200 import exact_det_band
    g = golden("det")
    diags = [g[f"{tag}_d{k}"] for k in range(nd)]
    A = (TriMatrix if nd == 3 else PentaMatrix).from_diagonals(*diags, layout=layout)
    res = exact_det_band(A)
    assert (host(res.status) == 0).all()
    for s in range(diags[0].shape[0]):
        assert _det_rel(res, s, g[f"{tag}_mant"][s], g[f"{tag}_expo"][s]) <= REL_TOL
    if tag.endswith("s"):
        assert (host(res.pivot_substitutions) == 2).all()
    # single system: a Fraction like the reference, plus the reference's op count
    from fractions import Fraction

    class Box:
        def __init__(self):
            self.ops = {}

        def add(self, **kw):
            for k, v in kw.items():
                self.ops[k] = self.ops.get(k, 0) + v
    box = Box()
    A1 = (TriMatrix if nd == 3 else PentaMatrix).from_diagonals(*[d[0] for d in diags])
    f = exact_det_band(A1, box)
    assert isinstance(f, Fraction)
    ref = Fraction(float(g[f"{tag}_mant"][0])) * Fraction(2) ** int(g[f"{tag}_expo"][0])
    assert abs(f - ref) <= REL_TOL * abs(ref)
    assert sum(box.ops.values()) == g[f"{tag}_ops"][0]


def test_det_band_singular(cuda, golden):
    from fractions import Fraction

    from paper_1804_09666_b200 import exact_det_band
    g = golden("det")
    t = TriMatrix.from_diagonals(g["sing_d0"], g["sing_d1"], g["sing_d2"])
    assert exact_det_band(t) == Fraction(0) == g["sing_mant"]


@pytest.mark.parametrize("kind", ["td", "pd"])
def test_det_band_config3(cuda, kind):
    """config-3 size (N=2048, 8 substituted zero pivots): the determinant of
    these non-dominant matrices spans ~1e-600; compared in mantissa/exponent
    form with the 60-digit pivoted oracle.  Tolerance 1e-8 relative: the
    reference's pivots are exact, the unpivoted binary64 product inherits the
    elimination's growth on non-dominant matrices."""
    from oracle.exact import det_band_mp
    from paper_1804_09666_b200 import exact_det_band
    if kind == "td":
        *p, rows = W.td_symbolic(64, 2048, seed=2)
        A = TriMatrix.from_diagonals(*p[:3], layout="system")
        offs, nd = [-1, 0, 1], 3
    else:
        *p, rows = W.pd_symbolic(64, 2048, seed=2)
        A = PentaMatrix.from_diagonals(*p[:5], layout="system")
        offs, nd = [-2, -1, 0, 1, 2], 5
    res = exact_det_band(A)
    assert (host(res.status) == 0).all()
    assert (host(res.pivot_substitutions) == 8).all()
    for s in range(0, 64, 16):
        m, e = det_band_mp([q[s] for q in p[:nd]], offs)
        assert _det_rel(res, s, m, e) <= 1e-8, (s, _det_rel(res, s, m, e))


def test_det_band_minimal_and_layouts(cuda):
    """n = 2 (TD) / 3 (PD), against the 60-digit oracle; batched in both
    layouts gives the same mantissa/exponent."""
    from oracle.exact import det_band_mp
    from paper_1804_09666_b200 import exact_det_band
    t = W.td_symbolic(3, 2, seed=4, zeros=0)
    for lay in ("interleaved", "system"):
        r = exact_det_band(TriMatrix.from_diagonals(*t[:3], layout=lay))
        for s in range(3):
            m, e = det_band_mp([q[s] for q in t[:3]], [-1, 0, 1])
            assert _det_rel(r, s, m, e) <= REL_TOL
    p = W.pd_symbolic(3, 3, seed=4, zeros=0)
    r = exact_det_band(PentaMatrix.from_diagonals(*p[:5]))
    for s in range(3):
        m, e = det_band_mp([q[s] for q in p[:5]], [-2, -1, 0, 1, 2])
        assert _det_rel(r, s, m, e) <= REL_TOL


# round 2: a wider reference-exact set (tests/golden/exact2.npz, generated by
# make_golden.py exact2 through exact_solve_stdm / exact_solve_spdm): 20
# tridiagonal and 12 pentadiagonal systems, 2-5 zero pivots, N = 28..72
EXACT2 = [("td_a", 3), ("td_b", 3), ("td_c", 3), ("pd_a", 5), ("pd_b", 5), ("pd_c", 5)]


@pytest.mark.parametrize("layout", ["interleaved", "system"])
@pytest.mark.parametrize("tag,nd", EXACT2)
def test_symbolic_golden_wide(cuda, golden, layout, tag, nd):
    g = golden("exact2")
    d = [g[f"{tag}_in{j}"] for j in range(nd + 1)]
    if nd == 3:
        r = exact_solve_stdm(TriMatrix.from_diagonals(*d[:3], layout=layout), d[3])
    else:
        r = exact_solve_spdm(PentaMatrix.from_diagonals(*d[:5], layout=layout), d[5])
    assert (host(r.status) == 0).all()
    assert np.array_equal(host(r.pivot_substitutions), g[f"{tag}_subs"])
    x = host(r.x)
    for s in range(x.shape[0]):
        assert rel(x[s], g[f"{tag}_x"][s]) <= REL_TOL, (tag, s, rel(x[s], g[f"{tag}_x"][s]))
