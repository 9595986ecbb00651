"""Hotelling-Bodewig inversion of the ILU(0) factors and SIP-HB -- the
reference's ``bandix.inverse`` dense mode (inverse.py:94-119, 205-302) over
the CUDA C ABI.  The triangular X X P products run on the FP64 tensor cores
(DMMA).  Host-driven iteration: these calls synchronise the stream.

``mode="banded"`` / :func:`hb_invert_banded` -- the reference's array
implementation (inverse.py:41-61, 122-195, 242-272):
band-truncated products in the reference's op order (bit-exact), with one
deliberate change in the automatic width: a width is accepted when the TRUE
residual ||I - M X||_inf is below the tolerance (the reference's criterion,
stagnation of the truncated iteration, never fires -- SURVEY D8).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Any

import numpy as np
import torch

from . import _lib
from .core import BandFactors, OpCounter, SolveReport, _as_batch, _Timer, default_device, ptr, \
    stream_handle, \
    vector_from_layout, vector_to_layout, workspace
from .errors import (DenseCapExceeded, DimensionMismatch, InvalidInput, MaxIterationsExceeded,
                     STATUS_MAX_ITER, STATUS_OK, STATUS_STAGNATED, STATUS_ZERO_DIAG, Stagnated,
                     ZeroDiagonal, exception_for)
from .iterative import SipConfig, _as_stencil



def _sweep_ops(n):
    """_sweep_apply: 5N-6 muls, 5N-6 adds (iterative.py:203-214)."""
    return 5 * n - 6


def _banded_apply_muls(n, w):
    """BandedApproxInverse.matvec: sum_{j<=w} (N - j) muls, that minus N adds
    (inverse.py:48-61); w may be a per-system tensor."""
    return (w + 1) * n - w * (w + 1) // 2


def _sip_hb_ops(n, k, mode="dense", w_lower=None, w_upper=None):
    """SolveReport.ops of sip_hb_solve: the CounterBox tally of its loop body
    (inverse.py:284-290) per iteration -- defect sweep, vec add, the two
    inverse applies, A sweep, vec sub.  Dense applies count N^2 muls and
    N(N-1) adds each (inverse.py:198-202): 4N^2 + 20N - 24 per iteration;
    banded applies count their band (inverse.py:48-61).  Pinned to the
    reference's own counts (tests/golden: hb_ops, sip_*_32_ops)."""
    sw = _sweep_ops(n)
    if mode == "dense":
        ml = mu = n * n
    else:
        ml, mu = _banded_apply_muls(n, w_lower), _banded_apply_muls(n, w_upper)
    muls = (2 * sw + ml + mu) * k
    adds = (2 * sw + n + (ml - n) + (mu - n)) * k
    return OpCounter(adds=adds, subs=n * k, muls=muls, divs=0)

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
        return _sip_hb_banded(s, b, cfg, hb_bandwidth, record_history, max_inv_iter)
    B, n, m, dev = s.batch, s.n, s.m, s.device
    bb, _ = _as_batch(b, "rhs")
    if bb.shape[1] != n:
        raise DimensionMismatch(f"rhs length {bb.shape[1]}, expected {n}")
    if n > dense_cap:
        raise DenseCapExceeded(n, dense_cap)
    b_store = vector_to_layout(bb, n, s.layout, dev, s.ld)
    tl = _tol(cfg, B, dev)
    x = s.new_vector()
    use_x0 = 0
    if cfg.initial_guess is not None:
        g, _ = _as_batch(cfg.initial_guess, "initial_guess")
        x.copy_(vector_to_layout(np.broadcast_to(g, (B, n)), n, s.layout, dev, s.ld))
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
        return SolveReport(x=x1, iterations=k, residual_inf=float(res[0]), ops=_sip_hb_ops(n, k),
                           wall_seconds=timer.seconds(), history=history)
    rep = SolveReport(x=xv, iterations=iters, residual_inf=res, ops=_sip_hb_ops(n, iters),
                      wall_seconds=timer.seconds(), history=hist if record_history else (),
                      status=st, index=ix, x_storage=x)
    rep.best_x = vector_from_layout(best_x, s.layout)
    rep.inv_iterations = torch.stack([inv_it[:B], inv_it[B:]], dim=1)
    rep.inv_residual = torch.stack([inv_res[:B], inv_res[B:]], dim=1)
    return rep


# ---------------------------------------------------------------------------
# banded mode (inverse.py:41-61, 122-195, 242-272)
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class BandedApproxInverse:
    """Triangular band approximation of an inverse, offsets 0..w on one side
    (inverse.py:41-61).  ``diags``: (B, w+1, n) device tensor; diagonal j of
    system s holds n-j entries (lower: (k+j, k), upper: (k, k+j))."""

    n: int
    side: str
    diags: Any
    w: int

    def matvec(self, v):
        """out = d0 * v, then out[i] += d_j[i-j] v[i-j] (lower) / d_j[i] v[i+j]
        (upper) for j = 1..w, in the reference's order (inverse.py:49-61);
        v: (n,) or (B, n)."""
        v = torch.as_tensor(v, dtype=torch.float64, device=self.diags.device)
        one = v.dim() == 1
        vv = v.reshape(-1, self.n)
        out = self.diags[:, 0, :] * vv
        n = self.n
        for j in range(1, self.w + 1):
            d = self.diags[:, j, :n - j]
            if self.side == "lower":
                out[:, j:] = out[:, j:] + d * vv[:, :n - j]
            else:
                out[:, :n - j] = out[:, :n - j] + d * vv[:, j:]
        return out[0] if one else out


@dataclass
class InversionReport:
    """inverse.py:64-69 (batched: iterations/residual_inf/status per system)."""

    inverse: Any
    iterations: Any
    residual_inf: Any
    residual_history: Any = ()
    status: Any = None
    index: Any = None


def hb_invert_dense(m, tol=1e-12, max_iter: int = 200, *, record_history: bool = True):
    """Quadratically convergent inversion X <- X (2I - M X) of dense square
    matrices (inverse.py:94-119): X0 = diag(1/m_ii), stop when ||I - M X||_inf
    < tol.  One (n, n) matrix: an InversionReport with a numpy inverse, and
    ZeroDiagonal / MaxIterationsExceeded(best, residual, max_iter) exactly as
    the reference.  A batch (B, n, n): device tensors and per-system status.
    Both products per iteration are DMMA GEMMs (bx_hb_invert_dense_f64)."""
    single = False
    if isinstance(m, torch.Tensor):
        t = m.detach().to(torch.float64)
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(m, dtype=np.float64)))
    if t.dim() == 2:
        t, single = t.unsqueeze(0), True
    if t.dim() != 3 or t.shape[1] != t.shape[2]:
        raise InvalidInput("dense inversion needs a square matrix")
    dev = t.device if t.is_cuda else default_device()
    t = t.to(dev).contiguous()
    B, n = t.shape[0], t.shape[1]
    tl = torch.as_tensor(np.broadcast_to(np.asarray(tol, dtype=np.float64), (B,)).copy(), device=dev)
    x = torch.empty((B, n, n), dtype=torch.float64, device=dev)
    it = torch.zeros(B, dtype=torch.int64, device=dev)
    rs = torch.empty(B, dtype=torch.float64, device=dev)
    hist = torch.empty((B, max_iter + 1), dtype=torch.float64, device=dev) if record_history else None
    st = torch.empty(B, dtype=torch.int32, device=dev)
    ix = torch.empty(B, dtype=torch.int32, device=dev)
    ws = workspace(_lib.lib().bx_hb_invert_dense_workspace_bytes(B, n), dev)
    _lib.call("bx_hb_invert_dense_f64", ptr(t), n, n, n * n, B, ptr(tl), int(max_iter), ptr(x), n,
              n * n, ptr(it), ptr(rs), ptr(hist), ptr(st), ptr(ix), ptr(ws), ws.numel(),
              stream_handle())
    if single:
        code, k, r = int(st[0]), int(it[0]), float(rs[0])
        x1 = x[0].cpu().numpy()
        if code == STATUS_ZERO_DIAG:
            raise ZeroDiagonal(int(ix[0]))
        if code == STATUS_MAX_ITER:
            raise MaxIterationsExceeded(x1, r, int(max_iter))
        h = tuple(float(v) for v in hist[0, :k + 1].cpu().numpy()) if record_history else ()
        return InversionReport(x1, k, r, h)
    return InversionReport(x, it, rs, hist if record_history else (), status=st, index=ix)


def dense_lower_factor(factors: BandFactors):
    """Unit-lower L as dense (B, n, n) device tensors -- or one (n, n) numpy
    array for a single system (inverse.py:72-78); outer offset factors.m."""
    return _dense_factor(factors, lower=True)


def dense_upper_factor(factors: BandFactors):
    """U as dense (B, n, n) / (n, n) (inverse.py:81-87)."""
    return _dense_factor(factors, lower=False)


def _dense_factor(f: BandFactors, lower: bool):
    l1, lm, mu, p1, pm = f.ref()
    B, n, m = l1.shape[0], f.n, f.m
    out = torch.zeros((B, n, n), dtype=torch.float64, device=mu.device)
    i = torch.arange(n, device=mu.device)
    if lower:
        out[:, i, i] = 1.0
        out[:, i[1:], i[:-1]] = l1
        out[:, i[m:], i[:n - m]] = lm
    else:
        out[:, i, i] = mu
        out[:, i[:-1], i[1:]] = p1
        out[:, i[:n - m], i[m:]] = pm
    if getattr(f, "single", False):
        return out[0].cpu().numpy()
    return out


def hb_invert_banded(factors: BandFactors, side: str, w: int = 2, tol=1e-12,
                     max_iter: int = 200) -> InversionReport:
    """Band-truncated Hotelling-Bodewig sweep for one triangular ILU(0) factor
    of every system (inverse.py:148-195), bit-for-bit the reference's
    iteration.  Single system: returns the report or raises Stagnated(best) /
    MaxIterationsExceeded / ZeroDiagonal like the reference; batched: per-system
    ``status`` (OK, STAGNATED, MAX_ITER, ZERO_DIAG) and the inverse the
    reference would hand back (the best one on stagnation)."""
    if w < 2:
        raise InvalidInput("banded inversion needs bandwidth w >= 2")
    if side not in ("lower", "upper"):
        raise InvalidInput(f"unknown side {side!r}")
    if getattr(factors, "m", 2) != 2:
        raise InvalidInput("banded inversion covers the pentadiagonal factors (m = 2)")
    layout = getattr(factors, "layout", _lib.LAYOUT_INTERLEAVED)
    mu = factors.u_main
    B = mu.shape[1] if layout == _lib.LAYOUT_INTERLEAVED else mu.shape[0]
    n, dev = factors.n, mu.device
    if w > n - 1:
        raise InvalidInput(f"bandwidth {w} exceeds n-1 = {n - 1}")
    tl = torch.as_tensor(np.broadcast_to(np.asarray(tol, dtype=np.float64), (B,)).copy(), device=dev)
    xd = torch.empty((B, w + 1, n), dtype=torch.float64, device=dev)
    it = torch.empty(B, dtype=torch.int64, device=dev)
    rs = torch.empty(B, dtype=torch.float64, device=dev)
    hist = torch.empty((B, max_iter + 1), dtype=torch.float64, device=dev)
    st = torch.empty(B, dtype=torch.int32, device=dev)
    ix = torch.empty(B, dtype=torch.int32, device=dev)
    ws = workspace(_lib.lib().bx_hb_banded_workspace_bytes(B, n, w), dev)
    _lib.call("bx_hb_invert_banded_f64", ptr(mu), ptr(factors.l_sub1), ptr(factors.l_sub2),
              ptr(factors.u_sup1), ptr(factors.u_sup2), 0 if side == "lower" else 1, int(w), ptr(tl),
              int(max_iter), ptr(xd), ptr(it), ptr(rs), ptr(hist), ptr(st), ptr(ix), B, n,
              mu.stride(0), layout, ptr(ws), ws.numel(), stream_handle())
    inv = BandedApproxInverse(n, side, xd, w)
    if getattr(factors, "single", False):
        code = int(st[0])
        h = hist[0].cpu().numpy()
        h = tuple(float(v) for v in h[~np.isnan(h)])
        rep = InversionReport(inv, int(it[0]), float(rs[0]), h)
        if code == STATUS_STAGNATED:
            raise Stagnated(rep)
        if code == STATUS_MAX_ITER:
            raise MaxIterationsExceeded(inv, float(rs[0]), int(max_iter))
        if code != STATUS_OK:
            raise exception_for(code, int(ix[0]))
        return rep
    return InversionReport(inv, it, rs, hist, st, ix)


def _sip_hb_banded(s, b, cfg, hb_bandwidth, record_history, max_inv_iter, w_cap=None):
    """sip_hb_solve(mode="banded") (inverse.py:242-272 + 274-302)."""
    if s.m != 2:
        raise InvalidInput("banded SIP-HB covers the pentadiagonal case (m = 2)")
    if cfg.alpha:
        raise InvalidInput("banded SIP-HB is the reference's ILU(0) (alpha = 0)")
    B, n, dev = s.batch, s.n, s.device
    bb, _ = _as_batch(b, "rhs")
    if bb.shape[1] != n:
        raise DimensionMismatch(f"rhs length {bb.shape[1]}, expected {n}")
    w = 0 if hb_bandwidth is None else int(hb_bandwidth)
    if w == 1 or w < 0:
        raise InvalidInput("banded inversion needs bandwidth w >= 2")
    w = min(w, n - 1) if w else 0
    cap = int(w_cap) if w_cap else (w if w else min(n - 1, 256))
    b_store = vector_to_layout(bb, n, s.layout, dev, s.ld)
    tl = _tol(cfg, B, dev)
    x = s.new_vector()
    use_x0 = 0
    if cfg.initial_guess is not None:
        g, _ = _as_batch(cfg.initial_guess, "initial_guess")
        x.copy_(vector_to_layout(np.broadcast_to(g, (B, n)), n, s.layout, dev, s.ld))
        use_x0 = 1
    best_x = s.new_vector()
    iters = torch.zeros(B, dtype=torch.int64, device=dev)
    res = torch.empty(B, dtype=torch.float64, device=dev)
    best_res = torch.empty(B, dtype=torch.float64, device=dev)
    st = torch.empty(B, dtype=torch.int32, device=dev)
    ix = torch.empty(B, dtype=torch.int32, device=dev)
    hist = torch.full((B, cfg.max_iterations), float("nan"), dtype=torch.float64, device=dev) \
        if record_history else None
    wu = torch.empty(2 * B, dtype=torch.int64, device=dev)
    inv_it = torch.empty(2 * B, dtype=torch.int64, device=dev)
    inv_res = torch.empty(2 * B, dtype=torch.float64, device=dev)
    inv_tr = torch.empty(2 * B, dtype=torch.float64, device=dev)
    ws = workspace(_lib.lib().bx_hb_banded_workspace_bytes(B, n, cap), dev)
    timer = _Timer()
    _lib.call("bx_sip_hb_banded_f64", *(ptr(v) for v in s.rowaligned()), ptr(b_store), ptr(tl),
              ptr(x), ptr(best_x), ptr(iters), ptr(res), ptr(best_res), ptr(st), ptr(ix), ptr(hist),
              w, cap, ptr(wu), ptr(inv_it), ptr(inv_res), ptr(inv_tr), B, n,
              int(cfg.max_iterations), int(max_inv_iter), use_x0, s.ld, s.layout, ptr(ws),
              ws.numel(), stream_handle())
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
        return SolveReport(x=x1, iterations=k, residual_inf=float(res[0]),
                           ops=_sip_hb_ops(n, k, "banded", int(wu[0]), int(wu[B])),
                           wall_seconds=timer.seconds(), history=history)
    rep = SolveReport(x=xv, iterations=iters, residual_inf=res,
                      ops=_sip_hb_ops(n, iters, "banded", wu[:B], wu[B:]),
                      wall_seconds=timer.seconds(), history=hist if record_history else (),
                      status=st, index=ix, x_storage=x)
    rep.best_x = vector_from_layout(best_x, s.layout)
    rep.best_residual = best_res
    rep.hb_bandwidth = torch.stack([wu[:B], wu[B:]], dim=1)
    rep.inv_iterations = torch.stack([inv_it[:B], inv_it[B:]], dim=1)
    rep.inv_residual = torch.stack([inv_res[:B], inv_res[B:]], dim=1)
    rep.inv_true_residual = torch.stack([inv_tr[:B], inv_tr[B:]], dim=1)
    return rep
