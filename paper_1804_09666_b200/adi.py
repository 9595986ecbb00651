"""One ADI time step of a 2-D parabolic problem (BASELINE.json config 5):
N tridiagonal systems along x, then N along y whose right-hand sides are the
x-sweep output (the paper's "N SLAEs d times per time step", PAPER.md:64-67;
the reference itself has no ADI driver).

Storage: the grid u[y][x] (x fastest).  The x-sweep systems are the rows
y (system-major for the C ABI); the y-sweep systems are the columns x, so
the x-sweep output is transposed once on the GPU (bx_transpose_f64) into
system-major [x][y] and the y-sweep result comes back as u[x][y].

Multi-GPU (strong scaling): rank r owns grid rows [r*ny/G, (r+1)*ny/G) for the
x-sweep and grid columns [r*nx/G, (r+1)*nx/G) for the y-sweep; the one
exchange between the sweeps is an all-to-all of the transposed x-sweep output
(NCCL over NVLink on the GPU path).  The exchange is larger than a rank's
sweep at 8 GPUs, so the x-sweep runs in ``chunks`` slices of the
rank's rows: slice c is solved and transposed, its all-to-all is queued
asynchronously (NCCL's stream picks it up after the transpose) and slice c+1
is solved meanwhile; the y-sweep starts when the last slice has arrived.
The solver, the transpose and the process group are injected so the exchange
logic is tested with gloo on CPU.
"""

from __future__ import annotations

import torch

from . import _lib


class CudaBackend:
    """Partitioned NTDM (system-major) + smem-tiled transpose, via the C ABI."""

    def __init__(self, device):
        self.device = device
        self._ws = {}

    def tri_solve(self, sub1, main, sup1, rhs, out):
        from .core import ptr, stream_handle
        B, n = main.shape
        status = torch.empty(B, dtype=torch.int32, device=self.device)
        ws = self._ws.get((B, n))
        if ws is None:  # flags + re-solve scratch of the partitioned path, allocated once
            nbytes = _lib.lib().bx_workspace_bytes(_lib.SOLVER["ntdm"], B, n, _lib.LAYOUT_SYSTEM_MAJOR,
                                                   _lib.ALGO_PARTITIONED)
            ws = self._ws[(B, n)] = torch.empty(max(int(nbytes), 256), dtype=torch.uint8,
                                                device=self.device)
        _lib.call("bx_ntdm_f64", ptr(sub1), ptr(main), ptr(sup1), ptr(rhs), ptr(out), ptr(status),
                  None, B, n, main.stride(0), _lib.LAYOUT_SYSTEM_MAJOR, _lib.ALGO_PARTITIONED,
                  ptr(ws), ws.numel(), stream_handle())
        return status

    def transpose(self, src, dst):
        from .core import ptr, stream_handle
        r, c = src.shape
        _lib.call("bx_transpose_f64", ptr(src), ptr(dst), r, c, src.stride(0), dst.stride(0), 1, 0, 0,
                  stream_handle())


class ADIStep:
    """x-sweep -> (exchange) -> y-sweep for one rank.

    xs: (sub1, main, sup1) row-aligned, shape (ny_local, nx): this rank's rows.
    ys: (sub1, main, sup1) row-aligned, shape (nx_local, ny): this rank's columns.
    chunks: slices of the x-sweep whose exchanges overlap the next slice's
    solve (multi-rank only; clipped to ny_local).
    """

    def __init__(self, xs, ys, group=None, backend=None, chunks=4):
        self.xs, self.ys = xs, ys
        self.group = group
        self.world = torch.distributed.get_world_size(group) if group is not None else 1
        self.nyl, self.nx = xs[1].shape
        self.nxl, self.ny = ys[1].shape
        if self.nyl * self.world != self.ny or self.nxl * self.world != self.nx:
            raise ValueError("grid must split evenly over the ranks")
        dev = xs[1].device
        self.backend = backend or CudaBackend(dev)
        f64 = dict(dtype=torch.float64, device=dev)
        self.X = torch.empty((self.nyl, self.nx), **f64)
        self.U = torch.empty((self.nxl, self.ny), **f64)
        if self.world == 1:
            self.XT = torch.empty((self.nx, self.nyl), **f64)
            return
        nch = max(1, min(int(chunks), self.nyl))
        edges = [self.nyl * c // nch for c in range(nch + 1)]
        self.slices = [(edges[c], edges[c + 1]) for c in range(nch) if edges[c + 1] > edges[c]]
        # per slice: its transposed block [x][rows of the slice] (contiguous: block r
        # of it goes to rank r) and what the other ranks send for the same rows
        self.XTc = [torch.empty((self.nx, b - a), **f64) for a, b in self.slices]
        self.recv = [torch.empty((self.world, self.nxl, b - a), **f64) for a, b in self.slices]
        self.Y = torch.empty((self.nxl, self.ny), **f64)

    def __call__(self, rhs):
        be = self.backend
        if self.world == 1:
            st_x = be.tri_solve(*self.xs, rhs, self.X)        # x-sweep
            be.transpose(self.X, self.XT)                      # [x][y]
            st_y = be.tri_solve(*self.ys, self.XT, self.U)     # y-sweep
            return self.U, st_x, st_y
        works, st_parts = [], []
        for (a, b), xt, rv in zip(self.slices, self.XTc, self.recv):
            st_parts.append(be.tri_solve(*(d[a:b] for d in self.xs), rhs[a:b], self.X[a:b]))
            be.transpose(self.X[a:b], xt)                      # [x][rows a..b)
            # block r of xt (the grid columns rank r owns) goes to rank r; queued
            # behind the transpose, it runs while the next slice is solved
            works.append(torch.distributed.all_to_all_single(rv.view(-1), xt.view(-1),
                                                             group=self.group, async_op=True))
        Yv = self.Y.view(self.nxl, self.world, self.nyl)
        for (a, b), rv, w in zip(self.slices, self.recv, works):
            w.wait()
            Yv[:, :, a:b].copy_(rv.transpose(0, 1))            # rows a..b) of every source rank
        st_y = be.tri_solve(*self.ys, self.Y, self.U)          # y-sweep
        return self.U, torch.cat(st_parts), st_y
