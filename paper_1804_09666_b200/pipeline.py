"""Host-to-host batched solves through the C ABI, pipelined over PCIe.

For data that lives in (pinned) host memory -- the end-to-end use of the
library -- the batch is cut into chunks of systems; chunk k+1 is copied in
while chunk k is solved and chunk k-1 is copied out, on alternating CUDA
streams, so the run time approaches max(H2D, D2H) instead of their sum plus
the solve.  Storage is system-major row-aligned (each system's rows
contiguous), so a chunk is one contiguous slice of every array.
"""

from __future__ import annotations

import torch

from . import _lib
from .core import ptr


def outer_lists(sub2, sup2):
    """Host (numpy) twin of bx_outer_compact_f64 for system-major row-aligned
    (B, n) sub2 / sup2: per system the rows whose sub2 (i >= 2) or sup2
    (i <= n-3) is nonzero, in row order, padded with row -1.  Returns
    (rows int32 (B, k), sub2 values (B, k), sup2 values (B, k))."""
    import numpy as np
    B, n = sub2.shape
    i = np.arange(n)
    s2 = np.where(i >= 2, sub2, 0.0)
    p2 = np.where(i <= n - 3, sup2, 0.0)
    mask = (s2 != 0.0) | (p2 != 0.0)
    cnt = mask.sum(axis=1)
    k = max(int(cnt.max()) if B else 0, 1)
    rows = np.full((B, k), -1, dtype=np.int32)
    vs = np.zeros((B, k))
    vp = np.zeros((B, k))
    bi, ri = np.nonzero(mask)
    pos = np.arange(len(bi)) - np.repeat(np.cumsum(cnt) - cnt, cnt)
    rows[bi, pos] = ri
    vs[bi, pos] = s2[bi, ri]
    vp[bi, pos] = p2[bi, ri]
    return rows, vs, vp


class HostPipeline:
    """Reusable device staging for `solver` ("ntdm" | "npdm" | "mnpdm" |
    "mnpdm_sparse": sub1/main/sup1/rhs plus the outer_lists of every system)."""

    def __init__(self, solver, n, chunk, device, algo="partitioned", nslots=3, outer_k=0):
        self.solver, self.n, self.chunk, self.dev = solver, n, chunk, device
        self.ndiag = 3 if solver in ("ntdm", "mnpdm_sparse") else 5
        self.outer_k = max(outer_k, 1)
        self.algo = {"sequential": _lib.ALGO_SEQUENTIAL, "partitioned": _lib.ALGO_PARTITIONED}[algo]
        f64 = dict(dtype=torch.float64, device=device)
        self.slots = [dict(ins=[torch.empty((chunk, n), **f64) for _ in range(self.ndiag + 1)],
                           x=torch.empty((chunk, n), **f64),
                           st=torch.empty(chunk, dtype=torch.int32, device=device),
                           ix=torch.empty(chunk, dtype=torch.int32, device=device),
                           nz=torch.empty(chunk, dtype=torch.int64, device=device),
                           stream=torch.cuda.Stream(device=device),
                           done=torch.cuda.Event(),
                           orow=torch.empty((chunk, self.outer_k), dtype=torch.int32, device=device),
                           os2=torch.empty((chunk, self.outer_k), **f64),
                           op2=torch.empty((chunk, self.outer_k), **f64))
                      for _ in range(nslots)]
        L = _lib.lib()
        nbytes = 0 if solver == "mnpdm_sparse" else \
            L.bx_workspace_bytes(_lib.SOLVER[solver], chunk, n, _lib.LAYOUT_SYSTEM_MAJOR, self.algo)
        self.ws = [torch.empty(max(nbytes, 8), dtype=torch.uint8, device=device) for _ in range(nslots)]

    def run(self, host_ins, host_x, status=None, host_outer=None):
        """host_ins: ndiag diagonals + rhs, pinned (B, n) system-major
        row-aligned; host_x: pinned (B, n) output.  Returns after queueing;
        call torch.cuda.synchronize() (or wait on the last slot) to finish."""
        B, n = host_x.shape
        L = _lib.lib()
        cur = torch.cuda.current_stream(self.dev)
        for k, c0 in enumerate(range(0, B, self.chunk)):
            c1 = min(B, c0 + self.chunk)
            m = c1 - c0
            sl = self.slots[k % len(self.slots)]
            ws = self.ws[k % len(self.slots)]
            s = sl["stream"]
            s.wait_event(sl["done"])          # slot's previous chunk fully drained
            s.wait_stream(cur)
            with torch.cuda.stream(s):
                for h, d in zip(host_ins, sl["ins"]):
                    d[:m].copy_(h[c0:c1], non_blocking=True)
                a = [ptr(t) for t in sl["ins"]]
                tail = (m, n, n, _lib.LAYOUT_SYSTEM_MAJOR, self.algo, ptr(ws), ws.numel(), s.cuda_stream)
                if self.solver == "mnpdm_sparse":
                    for h, d in zip(host_outer, (sl["orow"], sl["os2"], sl["op2"])):
                        d[:m].copy_(h[c0:c1], non_blocking=True)
                    rc = L.bx_mnpdm_sparse_f64(ptr(sl["orow"]), ptr(sl["os2"]), ptr(sl["op2"]),
                                               self.outer_k, *a, ptr(sl["x"]), ptr(sl["st"]),
                                               ptr(sl["ix"]), ptr(sl["nz"]), m, n, n,
                                               _lib.LAYOUT_SYSTEM_MAJOR, s.cuda_stream)
                elif self.solver == "ntdm":
                    rc = L.bx_ntdm_f64(*a, ptr(sl["x"]), ptr(sl["st"]), ptr(sl["ix"]), *tail)
                elif self.solver == "npdm":
                    rc = L.bx_npdm_f64(*a, ptr(sl["x"]), ptr(sl["st"]), ptr(sl["ix"]), *tail)
                else:
                    rc = L.bx_mnpdm_f64(*a, ptr(sl["x"]), ptr(sl["st"]), ptr(sl["ix"]), ptr(sl["nz"]),
                                        *tail)
                _lib.check(rc, self.solver)
                host_x[c0:c1].copy_(sl["x"][:m], non_blocking=True)
                if status is not None:
                    status[c0:c1].copy_(sl["st"][:m], non_blocking=True)
                sl["done"].record(s)
        for sl in self.slots:
            cur.wait_event(sl["done"])
