import sys, torch
sys.path.insert(0, '.')
from paper_1804_09666_b200 import StencilMatrix, SipConfig, sip_solve, workloads as W
g = W.five_point(64, 262144, 512, seed=3)
A = StencilMatrix.from_diagonals(*g[:5], m=512, layout="system")
cfg = SipConfig(tolerance=W.sip_tolerance(g[5]), max_iterations=1, alpha=0.5)
for _ in range(3):
    r = sip_solve(A, g[5], cfg)
torch.cuda.synchronize()
print("ok")
