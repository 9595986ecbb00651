import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_1804_09666_b200 import SipConfig, StencilMatrix, sip_solve, workloads as W
m = int(sys.argv[1]); R = 512
p = W.five_point(64, m * R, m, seed=3)
tol = W.sip_tolerance(p[5])
A = StencilMatrix.from_diagonals(*p[:5], m=m, layout="system")
rep = sip_solve(A, p[5], SipConfig(tolerance=tol, max_iterations=500, alpha=0.5), algo="scan")
torch.cuda.synchronize()
