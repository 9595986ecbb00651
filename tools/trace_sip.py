"""Developer tool: phase clocks of the wavefront SIP kernel (BX_SIP_TRACE build
via tools/variant_lib.py), config-4 shape.  Not used by the product."""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1804_09666_b200 import StencilMatrix, SipConfig, sip_solve, workloads as W, _lib
L = _lib.lib()
B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
m = int(sys.argv[2]) if len(sys.argv) > 2 else 512
g = W.five_point(B, m * m, m, seed=3)
A = StencilMatrix.from_diagonals(*g[:5], m=m, layout="system")
cfg = SipConfig(tolerance=W.sip_tolerance(g[5]), max_iterations=500, alpha=0.5)
for _ in range(2):
    r = sip_solve(A, g[5], cfg)
torch.cuda.synchronize()
buf = np.zeros((64, 40), dtype=np.int64)
steps = 2 * m - 1
L.bx_sip_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
L.bx_sip_trace_read(buf.ctypes.data, buf.nbytes)
k = int(r.iterations.max())
b = buf[0]
print("iterations", k, "setup(+r0) cycles", b[1] - b[0], " to first iteration", b[2] - b[1])
for it in range(k):
    f = b[3 + 2 * it] - b[2 + 2 * it]
    nx = b[2 + 2 * (it + 1)] if it + 1 < k else b[39]
    print(f"  it {it}: forward {f} backward+residual {nx - b[3 + 2 * it]}")
print("producer: waiting on empty", b[37], "cycles, issuing", b[38], "cycles")
print("total", b[39] - b[0], "cycles; per step fwd/bwd",
      (b[3] - b[2]) / steps, (b[4] - b[3]) / (steps + 1))
