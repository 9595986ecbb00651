"""Diagnostic: per-factor deviation of the DMMA HB inverses from the restatement."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import inverse as H, iterative as I
from paper_1804_09666_b200 import StencilMatrix, hb_invert_factors
from paper_1804_09666_b200 import workloads as W
for m, rows, alpha in [(2, 128, 0.0), (16, 24, 0.5), (16, 24, 0.0), (32, 64, 0.5), (8, 40, 0.0)]:
    n = m * rows
    p = W.five_point(3, n, m, seed=8)
    tol = W.sip_tolerance(p[5])
    A = StencilMatrix.from_diagonals(*p[:5], m=m)
    xl, xu, its, res, st, _ = hb_invert_factors(A, tol, alpha=alpha)
    xl, xu, its = xl.cpu().numpy(), xu.cpu().numpy(), its.cpu().numpy()
    f, _, _ = I.ilu0(*p[:5], m=m, alpha=alpha)
    lo, up = H.dense_lower(f), H.dense_upper(f)
    for s in range(3):
        rl = H.hb_invert_dense(lo[s], tol[s]); ru = H.hb_invert_dense(up[s], tol[s])
        dl = np.abs(xl[s] - rl[0]); du = np.abs(xu[s] - ru[0])
        iu = np.unravel_index(np.argmax(du), du.shape)
        print(m, rows, alpha, s, "its", its[s], rl[1], ru[1], "dl %.2e du %.2e at %s gpu %r ref %r" % (
            dl.max(), du.max(), iu, xu[s][iu], ru[0][iu]))
