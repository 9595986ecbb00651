"""Developer probe: scan-SIP time per grid row against the grid width m (same
row count): tells whether a sweep is bound by bytes per SM (time ~ m) or by the
per-row chain (time ~ const)."""
import sys, os
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_09666_b200 import SipConfig, StencilMatrix, sip_solve, workloads as W

R = 512
for m in (64, 128, 256, 512):
    p = W.five_point(64, m * R, m, seed=3)
    tol = W.sip_tolerance(p[5])
    A = StencilMatrix.from_diagonals(*p[:5], m=m, layout="system")
    cfg = SipConfig(tolerance=tol, max_iterations=500, alpha=0.5)
    for algo in ("scan", "wavefront"):
        rep = sip_solve(A, p[5], cfg, algo=algo)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            rep = sip_solve(A, p[5], cfg, algo=algo)
        e1.record(); torch.cuda.synchronize()
        k = float(rep.iterations.double().mean())
        print(f"m={m:4d} {algo:9s} {e0.elapsed_time(e1)/3:8.2f} ms per solve (incl. host-side wrapper), mean k={k:.1f}")
