import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_1804_09666_b200 import TriMatrix, PentaMatrix, workloads as W
from paper_1804_09666_b200.exact import rcond_band, exact_det_band
for kind in ("td", "pd"):
    rng = np.random.default_rng(2)
    if kind == "td":
        *d, rhs, rows = W.td_symbolic(4096, 2048, rng=rng)
        A = TriMatrix.from_diagonals(*d, layout="interleaved")
    else:
        *d, rhs, rows = W.pd_symbolic(4096, 2048, rng=rng)
        A = PentaMatrix.from_diagonals(*d, layout="interleaved")
    for name, fn in (("rcond", lambda: rcond_band(A)), ("det", lambda: exact_det_band(A))):
        fn(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        print(kind, name, f"{e0.elapsed_time(e1):.3f} ms")
