import sys, time, torch, numpy as np
sys.path.insert(0, '.')
from paper_1804_09666_b200 import StencilMatrix, SipConfig, sip_solve, workloads as W
g = W.five_point(64, 262144, 512, seed=3)
A = StencilMatrix.from_diagonals(*g[:5], m=512, layout="system")
b = torch.from_numpy(g[5]).cuda()
cfg = SipConfig(tolerance=W.sip_tolerance(g[5]), max_iterations=8, alpha=0.5)
for _ in range(2): sip_solve(A, b, cfg)
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(3): r = sip_solve(A, b, cfg)
torch.cuda.synchronize(); print("ms", (time.perf_counter() - t0) / 3 * 1e3)
