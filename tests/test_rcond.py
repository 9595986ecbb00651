"""Condition gate: the LAPACK checker against exact
condition numbers (CPU) and the GPU estimator against LAPACK (dgtcon /
dgbcon) on the same systems."""

import numpy as np
import pytest

from oracle.exact import rcond_dense, rcond_lapack
from paper_1804_09666_b200 import workloads as W

TD = [-1, 0, 1]
PD = [-2, -1, 0, 1, 2]


def cases(bsz, n, seed):
    yield "td", TD, W.td_symbolic(bsz, n, seed=seed, zeros=0)[:3]
    yield "pd", PD, W.pd_symbolic(bsz, n, seed=seed, zeros=0)[:5]
    yield "tdd", TD, W.td_dominant(bsz, n, seed=seed)[:3]
    yield "pdd", PD, W.pd_dominant(bsz, n, seed=seed)[:5]


def test_lapack_checker_bounds_the_exact_condition():
    # Hager-Higham underestimates ||A^-1||_1: rcond_est >= rcond_exact, and
    # stays within a small factor of it on these families
    for _, offs, p in cases(6, 48, 3):
        for s in range(6):
            d = [q[s] for q in p]
            est, ex = rcond_lapack(d, offs), rcond_dense(d, offs)
            assert est >= ex * (1 - 1e-10)
            assert est <= 10 * ex


@pytest.mark.gpu
@pytest.mark.parametrize("layout", ["interleaved", "system"])
def test_rcond_gpu_vs_lapack(cuda, layout):
    from paper_1804_09666_b200 import PentaMatrix, TriMatrix, rcond_band
    for name, offs, p in cases(64, 300, 7):
        A = (TriMatrix if len(offs) == 3 else PentaMatrix).from_diagonals(*p, layout=layout)
        rc, st, _ = rcond_band(A)
        rc = rc.cpu().numpy()
        assert (st.cpu().numpy() == 0).all()
        ref = np.array([rcond_lapack([q[s] for q in p], offs) for s in range(64)])
        rel = np.abs(rc - ref) / ref
        # same factorisation and the same dlacn2 path: agreement to rounding,
        # except where rounding flips a sign decision of the iteration
        assert np.mean(rel <= 1e-8) >= 0.95, (name, np.sort(rel)[-5:])
        assert np.all(rc <= 3 * ref) and np.all(rc >= ref / 3), name
    # single system: a float; an exactly singular matrix: 0
    t = TriMatrix.from_diagonals([1.0, 1.0], [1.0, 1.0, 1.0], [1.0, 0.0])
    assert rcond_band(t) == 0.0
    d = W.td_dominant(1, 50, seed=1)
    assert abs(rcond_band(TriMatrix.from_diagonals(*[q[0] for q in d[:3]]))
               - rcond_lapack([q[0] for q in d[:3]], TD)) <= 1e-8 * rcond_lapack([q[0] for q in d[:3]], TD)


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["td", "pd"])
def test_rcond_config3(cuda, kind):
    """config-3 size (N = 2048, 8 decoupled zero pivots: nonsingular, not
    dominant): the estimate the symbolic solvers' errors are read against."""
    from paper_1804_09666_b200 import PentaMatrix, TriMatrix, rcond_band
    if kind == "td":
        *p, rows = W.td_symbolic(32, 2048, seed=2)
        A, offs, nd = TriMatrix.from_diagonals(*p[:3], layout="system"), TD, 3
    else:
        *p, rows = W.pd_symbolic(32, 2048, seed=2)
        A, offs, nd = PentaMatrix.from_diagonals(*p[:5], layout="system"), PD, 5
    rc, st, _ = rcond_band(A)
    rc = rc.cpu().numpy()
    assert (st.cpu().numpy() == 0).all()
    for s in range(0, 32, 8):
        ref = rcond_lapack([q[s] for q in p[:nd]], offs)
        assert rc[s] <= 3 * ref and rc[s] >= ref / 3, (s, rc[s], ref)
