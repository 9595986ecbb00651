"""Developer harness for compute-sanitizer (not product code): one small
invocation of the kernels that use clusters / DSMEM / st.async / mbarriers /
cp.async.bulk rings -- the partitioned direct kernel (part_kernel, K=1 and
K=2, 1-CTA and 4-CTA clusters), the SIP wavefront kernel (sip_wave_kernel),
the re-solve pass and the HB DMMA GEMMs -- each checked against the oracle."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import cport  # noqa: E402
from oracle import direct as D  # noqa: E402
from paper_1804_09666_b200 import (PentaMatrix, SipConfig, StencilMatrix, TriMatrix,  # noqa: E402
                                   hb_invert_dense, sip_solve, solve_npdm, solve_ntdm)
from paper_1804_09666_b200 import workloads as W  # noqa: E402

for n in (900, 4096):
    p = W.pd_dominant(3, n, seed=n)
    p[2][1, 64] = 0.0                     # a flagged system -> the re-solve pass runs
    x = solve_npdm(PentaMatrix.from_diagonals(*p[:5], layout="system"), p[5], algo="partitioned").x
    xr, _, _ = D.npdm(*p)
    assert np.abs(x.cpu().numpy() - xr).max() <= 1e-9 * np.abs(xr).max()
    t = W.td_dominant(3, n, seed=n)
    x = solve_ntdm(TriMatrix.from_diagonals(*t[:3], layout="system"), t[3], algo="partitioned").x
    xr, _, _ = D.ntdm(*t)
    assert np.abs(x.cpu().numpy() - xr).max() <= 1e-9 * np.abs(xr).max()
g = W.five_point(2, 64 * 32, 32, seed=3)
tol = W.sip_tolerance(g[5])
rep = sip_solve(StencilMatrix.from_diagonals(*g[:5], m=32), g[5], SipConfig(tolerance=tol, max_iterations=50,
                                                                           alpha=0.5), algo="wavefront")
ref = cport.sip(*cport.rowaligned_penta(*g[:5], m=32), g[5], tol, m=32, alpha=0.5)
assert np.array_equal(rep.x.cpu().numpy(), ref["x"])
M = np.eye(100) + 0.001 * np.random.default_rng(0).uniform(-1, 1, (100, 100))
r = hb_invert_dense(M)
assert np.abs(np.eye(100) - M @ r.inverse).max() < 1e-12
print("sanitize case ok")
