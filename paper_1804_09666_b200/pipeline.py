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


class HostPipeline:
    """Reusable device staging for `solver` ("ntdm" | "npdm" | "mnpdm")."""

    def __init__(self, solver, n, chunk, device, algo="partitioned", nslots=3):
        self.solver, self.n, self.chunk, self.dev = solver, n, chunk, device
        self.ndiag = 3 if solver == "ntdm" else 5
        self.algo = {"sequential": _lib.ALGO_SEQUENTIAL, "partitioned": _lib.ALGO_PARTITIONED}[algo]
        f64 = dict(dtype=torch.float64, device=device)
        self.slots = [dict(ins=[torch.empty((chunk, n), **f64) for _ in range(self.ndiag + 1)],
                           x=torch.empty((chunk, n), **f64),
                           st=torch.empty(chunk, dtype=torch.int32, device=device),
                           ix=torch.empty(chunk, dtype=torch.int32, device=device),
                           nz=torch.empty(chunk, dtype=torch.int64, device=device),
                           stream=torch.cuda.Stream(device=device),
                           done=torch.cuda.Event())
                      for _ in range(nslots)]
        L = _lib.lib()
        nbytes = L.bx_workspace_bytes(_lib.SOLVER[solver], chunk, n, _lib.LAYOUT_SYSTEM_MAJOR, self.algo)
        self.ws = [torch.empty(max(nbytes, 8), dtype=torch.uint8, device=device) for _ in range(nslots)]

    def run(self, host_ins, host_x, status=None):
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
                if self.solver == "ntdm":
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
