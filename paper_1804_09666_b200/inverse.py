"""Hotelling-Bodewig inversion of the ILU(0) factors and SIP-HB -- the
reference's ``bandix.inverse`` dense mode (inverse.py:94-119, 205-302) over
the CUDA C ABI.  The triangular X X P products run on the FP64 tensor cores
(DMMA).  Host-driven iteration: these calls synchronise the stream.

``mode="banded"`` (the reference's array implementation, inverse.py:122-195)
is not part of the hot path and raises InvalidInput.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .core import SolveReport, _as_batch, _Timer, ptr, stream_handle, vector_from_layout, \
    vector_to_layout, workspace
from .errors import (DenseCapExceeded, DimensionMismatch, InvalidInput, MaxIterationsExceeded,
                     STATUS_MAX_ITER, STATUS_OK, exception_for)
from .iterative import SipConfig, _as_stencil, _sip_ops


def _tol(cfg, B, dev):
    return torch.as_tensor(np.broadcast_to(np.asarray(cfg.tolerance, dtype=np.float64), (B,)).copy(),
                           device=dev)


def hb_invert_factors(a, tol=1e-12, max_iter=200, *, alpha=0.0):
    """Dense inverses of the ILU(0) factors L, U of every system.

    Returns (X_L, X_U, iterations (B, 2), residual (B, 2), status, index) with
    X_* dense (B, n, n) device tensors; iterations/residual follow
    hb_invert_dense's (iteration, r) for L (column 0) and U (column 1)."""
    s = _as_stencil(a)
    B, n, dev = s.batch, s.n, s.device
    tl = _tol(SipConfig(tolerance=tol), B, dev)
    xl = torch.empty((B, n, n), dtype=torch.float64, device=dev)
    xu = torch.empty((B, n, n), dtype=torch.float64, device=dev)
    it = torch.empty(2 * B, dtype=torch.int64, device=dev)
    rs = torch.empty(2 * B, dtype=torch.float64, device=dev)
    st = torch.empty(B, dtype=torch.int32, device=dev)
    ix = torch.empty(B, dtype=torch.int32, device=dev)
    ws = workspace(_lib.lib().bx_hb_workspace_bytes(B, n), dev)
    _lib.call("bx_hb_invert_f64", *(ptr(v) for v in s.rowaligned()), ptr(tl), ptr(xl), ptr(xu),
              ptr(it), ptr(rs), ptr(st), ptr(ix), B, n, s.m, float(alpha), int(max_iter), s.ld,
              s.layout, ptr(ws), ws.numel(), stream_handle())
    its = torch.stack([it[:B], it[B:]], dim=1)
    res = torch.stack([rs[:B], rs[B:]], dim=1)
    return xl, xu, its, res, st, ix


def sip_hb_solve(a, b, cfg: SipConfig | None = None, mode: str = "dense", hb_bandwidth=None,
                 dense_cap: int = 8000, record_history: bool = False, *,
                 max_inv_iter: int = 200) -> SolveReport:
    """SIP with the substitutions replaced by the HB inverses (inverse.py:205-302)."""
    cfg = cfg or SipConfig()
    s = _as_stencil(a)
    if mode not in ("dense", "banded"):
        raise InvalidInput(f"unknown mode {mode!r}")
    if mode == "banded":
        raise InvalidInput("banded HB mode is not built (SURVEY 8f row f3); use mode='dense'")
    B, n, m, dev = s.batch, s.n, s.m, s.device
    bb, _ = _as_batch(b, "rhs")
    if bb.shape[1] != n:
        raise DimensionMismatch(f"rhs length {bb.shape[1]}, expected {n}")
    if n > dense_cap:
        raise DenseCapExceeded(n, dense_cap)
    b_store = vector_to_layout(bb, n, s.layout, dev)
    tl = _tol(cfg, B, dev)
    x = s.new_vector()
    use_x0 = 0
    if cfg.initial_guess is not None:
        g, _ = _as_batch(cfg.initial_guess, "initial_guess")
        x.copy_(vector_to_layout(np.broadcast_to(g, (B, n)), n, s.layout, dev))
        use_x0 = 1
    best_x = s.new_vector()
    iters = torch.zeros(B, dtype=torch.int64, device=dev)
    res = torch.empty(B, dtype=torch.float64, device=dev)
    best_res = torch.empty(B, dtype=torch.float64, device=dev)
    st = torch.empty(B, dtype=torch.int32, device=dev)
    ix = torch.empty(B, dtype=torch.int32, device=dev)
    hist = torch.full((B, cfg.max_iterations), float("nan"), dtype=torch.float64, device=dev) \
        if record_history else None
    inv_it = torch.empty(2 * B, dtype=torch.int64, device=dev)
    inv_res = torch.empty(2 * B, dtype=torch.float64, device=dev)
    ws = workspace(_lib.lib().bx_hb_workspace_bytes(B, n), dev)
    timer = _Timer()
    _lib.call("bx_sip_hb_f64", *(ptr(v) for v in s.rowaligned()), ptr(b_store), ptr(tl), ptr(x),
              ptr(best_x), ptr(iters), ptr(res), ptr(best_res), ptr(st), ptr(ix), ptr(hist),
              ptr(inv_it), ptr(inv_res), B, n, m, float(cfg.alpha), int(cfg.max_iterations),
              int(max_inv_iter), use_x0, s.ld, s.layout, ptr(ws), ws.numel(), stream_handle())
    timer.end()
    xv = vector_from_layout(x, s.layout)
    if s.single:
        code = int(st[0])
        k = int(iters[0])
        if code == STATUS_MAX_ITER:
            bx1 = vector_from_layout(best_x, s.layout)[0].cpu().numpy()
            raise MaxIterationsExceeded(bx1, float(best_res[0]), k)
        if code != STATUS_OK:
            raise exception_for(code, int(ix[0]), residual=float(res[0]), iterations=k)
        history = tuple((i + 1, float(v)) for i, v in enumerate(hist[0, :k].cpu().numpy())) \
            if record_history else ()
        x1 = xv[0].cpu().numpy()
        x1.setflags(write=False)
        return SolveReport(x=x1, iterations=k, residual_inf=float(res[0]), ops=_sip_ops(n, k),
                           wall_seconds=timer.seconds(), history=history)
    rep = SolveReport(x=xv, iterations=iters, residual_inf=res, ops=_sip_ops(n, iters),
                      wall_seconds=timer.seconds(), history=hist if record_history else (),
                      status=st, index=ix, x_storage=x)
    rep.best_x = vector_from_layout(best_x, s.layout)
    rep.inv_iterations = torch.stack([inv_it[:B], inv_it[B:]], dim=1)
    rep.inv_residual = torch.stack([inv_res[:B], inv_res[B:]], dim=1)
    return rep
