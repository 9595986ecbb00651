"""ILU(0) and Stone's strongly implicit procedure (SIP) -- the reference's
``bandix.iterative`` entry points (iterative.py:32-308) over the CUDA C ABI.

Generalisation: the outer offset is a stride
``m`` (``PentaMatrix`` is m = 2, exactly the reference; ``StencilMatrix``
carries m >= 3, the five-point stencil of an (n/m) x m grid) and
``SipConfig.alpha`` is Stone's partial-cancellation parameter (m >= 3 only;
alpha = 0 is pure ILU(0)).

Results are bit-identical to the reference (m = 2) and to the oracle's
restatement (m >= 3): the same operation order, one rounding per operation.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Any, Optional, Sequence

import numpy as np
import torch

from . import _lib
from .core import (LAYOUTS, BandFactors, OpCounter, PentaMatrix, SolveReport, _as_batch, _Band,
                   _Timer, default_device, pack_rows, ptr, stream_handle, unpack_rows,
                   vector_from_layout, vector_to_layout, workspace)
from .errors import (DimensionMismatch, InvalidInput, MaxIterationsExceeded, STATUS_DIVERGED,
                     STATUS_MAX_ITER, STATUS_OK, exception_for)

ALGOS = {"sequential": _lib.ALGO_SEQUENTIAL, "wavefront": 2, "auto": 3, "scan": 4}


@dataclass(frozen=True)
class SipConfig:
    """Stopping control (iterative.py:32-48).

    ``tolerance``: the errorMargin of the residual test, a scalar or one
    value per system (relative stopping = tol_s * ||b_s||_inf with x0 = 0).
    ``alpha``: Stone's parameter (extension; requires stride m >= 3).
    """

    tolerance: Any = 1e-12
    max_iterations: int = 10_000
    initial_guess: Optional[Sequence] = None
    alpha: float = 0.0

    def __post_init__(self):
        tol = np.asarray(self.tolerance, dtype=np.float64)
        if not np.all(tol > 0):
            raise InvalidInput("tolerance must be positive")
        if self.max_iterations < 1:
            raise InvalidInput("max_iterations must be at least 1")


class StencilMatrix(_Band):
    """Batched five-point band with outer offset m (offsets -m, -1, 0, +1, +m).

    Reference-length diagonals: subm (n-m), sub1 (n-1), main (n), sup1 (n-1),
    supm (n-m); row i uses subm[i-m], sub1[i-1], main[i], sup1[i], supm[i].
    m = 2 is the reference's ``PentaMatrix``.
    """

    names = ("subm", "sub1", "main", "sup1", "supm")

    def __init__(self, n, batch, diags, layout, single, device, m):
        self.m = m
        self.offsets = (-m, -1, 0, 1, m)
        super().__init__(n, batch, diags, layout, single, device)

    @staticmethod
    def from_diagonals(subm, sub1, main, sup1, supm, m, *, layout="interleaved", device=None):
        if m < 2:
            raise InvalidInput("stride m must be >= 2")
        lay = LAYOUTS[layout] if isinstance(layout, str) else layout
        device = torch.device(device) if device is not None else default_device()
        conv = [_as_batch(a, nm) for a, nm in zip((subm, sub1, main, sup1, supm), StencilMatrix.names)]
        single = all(s for _, s in conv)
        mats = [x for x, _ in conv]
        batch, n = mats[2].shape
        if n <= m:
            raise InvalidInput(f"stencil needs n > m (n={n}, m={m})")
        for x, off, nm in zip(mats, (-m, -1, 0, 1, m), StencilMatrix.names):
            if x.shape != (batch, n - abs(off)):
                raise InvalidInput(f"diagonal lengths do not match n={n} ({nm} has {tuple(x.shape)})")
        diags = [pack_rows(x, n, -off if off < 0 else 0, lay, device, batch)
                 for x, off in zip(mats, (-m, -1, 0, 1, m))]
        return StencilMatrix(n, batch, diags, lay, single, device, m)

    @staticmethod
    def from_penta(a: PentaMatrix):
        return StencilMatrix(a.n, a.batch, list(a.rowaligned()), a.layout, a.single, a.device, 2)


def _as_stencil(a):
    if isinstance(a, StencilMatrix):
        return a
    if isinstance(a, PentaMatrix):
        return StencilMatrix.from_penta(a)
    raise TypeError("expected a PentaMatrix or StencilMatrix")


@dataclass(frozen=True)
class DefectMatrix:
    """K = L U - A (iterative.py:51-55); ``diagonals`` keyed by offset,
    row-aligned (B, n) device tensors in the matrix layout."""

    diagonals: dict
    m: int


def _factor_call(a: StencilMatrix, alpha):
    B, n, m = a.batch, a.n, a.m
    dev = a.device
    outs = [a.new_vector() for _ in range(12)]
    status = torch.empty(B, dtype=torch.int32, device=dev)
    index = torch.empty(B, dtype=torch.int32, device=dev)
    nbytes = _lib.lib().bx_workspace_bytes(_lib.SOLVER["sip"], B, n, a.layout, 0)
    ws = workspace(nbytes, dev)
    d = a.rowaligned()
    _lib.call("bx_ilu0_f64", *(ptr(x) for x in d), *(ptr(x) for x in outs), ptr(status), ptr(index),
              B, n, m, float(alpha), a.ld, a.layout, ptr(ws), ws.numel(), stream_handle())
    return outs, status, index


def ilu0_penta(a, counter=None, *, alpha=0.0):
    """Pattern-restricted ILU(0) (iterative.py:62-124); Stone's alpha for m >= 3.

    Returns ``BandFactors`` with row-aligned device diagonals (views in the
    reference's lengths via ``.ref()``).  Raises ``ZeroPivot`` for a single
    system; batched calls carry ``status``/``index`` on the factors."""
    s = _as_stencil(a)
    outs, status, index = _factor_call(s, alpha)
    if s.single and int(status[0]) != STATUS_OK:
        raise exception_for(int(status[0]), int(index[0]))
    mu, l1, l2, phi, psi = outs[:5]
    f = BandFactors(s.n, l1, l2, mu, phi, psi, m=s.m)
    object.__setattr__(f, "status", status)
    object.__setattr__(f, "index", index)
    object.__setattr__(f, "layout", s.layout)
    object.__setattr__(f, "single", s.single)
    object.__setattr__(f, "batch", s.batch)
    object.__setattr__(f, "_defect", outs[5:])
    return f


def _factor_vec(f: BandFactors, v, what):
    vb, single = _as_batch(v, what)
    if vb.shape[1] != f.n:
        raise DimensionMismatch(f"{what} length {vb.shape[1]}, expected {f.n}")
    ld = getattr(f, "ld", None) or f.u_main.stride(0)
    return vector_to_layout(vb, f.n, f.layout, f.u_main.device, ld), single, ld


def _factor_out(f: BandFactors, store, single):
    v = vector_from_layout(store, f.layout)
    if single and getattr(f, "single", single):
        out = v[0].detach().cpu().numpy()
        out.setflags(write=False)
        return out
    return v


def forward_sub(factors: BandFactors, rhs, counter=None):
    """One sweep of L y = rhs, unit lower with two subdiagonals (iterative.py:
    127-137 -> penta_forward): 4N-6 ops, the reference's operation order
    (bit-identical).  Factors from lu_penta or ilu0_penta (outer offset m)."""
    f = factors
    b, single, ld = _factor_vec(f, rhs, "rhs")
    y = torch.empty_like(b)
    B = b.shape[1] if f.layout == _lib.LAYOUT_INTERLEAVED else b.shape[0]
    _lib.call("bx_forward_sub_f64", f.m, ptr(f.l_sub1), ptr(f.l_sub2), ptr(b), ptr(y), B, f.n, ld,
              f.layout, stream_handle())
    if counter is not None:
        counter.add(muls=2 * f.n - 3, subs=2 * f.n - 3)
    return _factor_out(f, y, single)


def backward_sub(factors: BandFactors, y, counter=None):
    """One sweep of U x = y with the pivots plus two superdiagonals
    (iterative.py:140-149 -> penta_backward): 5N-6 ops, bit-identical; a zero
    pivot raises ZeroPivot(first) for one system (batches: ``.status`` /
    ``.index`` on the returned tensor's owner -- see backward_sub_batched)."""
    x, status, index, single = _backward(factors, y, counter)
    if single and int(status[0]) != STATUS_OK:
        raise exception_for(int(status[0]), int(index[0]))
    return _factor_out(factors, x, single)


def backward_sub_batched(factors: BandFactors, y, counter=None):
    """backward_sub for a batch: (x, status, index) device tensors."""
    x, status, index, _ = _backward(factors, y, counter)
    return vector_from_layout(x, factors.layout), status, index


def _backward(f, y, counter):
    ys, single, ld = _factor_vec(f, y, "rhs")
    x = torch.empty_like(ys)
    B = ys.shape[1] if f.layout == _lib.LAYOUT_INTERLEAVED else ys.shape[0]
    status = torch.empty(B, dtype=torch.int32, device=ys.device)
    index = torch.empty(B, dtype=torch.int32, device=ys.device)
    _lib.call("bx_backward_sub_f64", f.m, ptr(f.u_main), ptr(f.u_sup1), ptr(f.u_sup2), ptr(ys), ptr(x),
              ptr(status), ptr(index), B, f.n, ld, f.layout, stream_handle())
    if counter is not None:
        counter.add(muls=2 * f.n - 3, subs=2 * f.n - 3, divs=f.n)
    return x, status, index, single


def defect_matrix(factors: BandFactors, a, counter=None) -> DefectMatrix:
    """K = L U - A (iterative.py:186-200): offsets -m, -1, 0, +1, +m and, for
    m >= 3, the dropped fill at +-(m-1)."""
    s = _as_stencil(a)
    if factors.n != s.n:
        raise DimensionMismatch(f"factors for n={factors.n}, matrix n={s.n}")
    ks = getattr(factors, "_defect", None)
    if ks is None:
        ks = _factor_call(s, 0.0)[0][5:]
    m = s.m
    keys = (-m, -1, 0, 1, m) if m == 2 else (-m, -1, 0, 1, m, -(m - 1), m - 1)
    diags = {k: vector_from_layout(v, s.layout) for k, v in zip(keys, ks)}
    return DefectMatrix(diags, m)


def sip_solve(a, b, cfg: SipConfig | None = None, record_history: bool = False, *,
              algo="auto") -> SolveReport:
    """Stone's strongly implicit procedure (iterative.py:255-308), batched.

    Loop per system: newRHS = K x + b, forward/backward substitution, then the
    recomputed residual b - A x; runs while ||r||_inf >= tolerance, raising
    (single system) or reporting (batched status) MaxIterationsExceeded /
    Diverged exactly as the reference.  ``ops`` is the reference's loop-body
    count 31N - 36 per iteration (iterative.py:262-264, m = 2).

    ``algo``: "sequential" (one thread per system, any band), "wavefront"
    (grid-structured systems: one CTA per system walks the grid's
    anti-diagonals), "auto" (wavefront when every system is a grid), or "scan"
    (grid-structured systems, throughput path: the same iteration in
    correction form with row-parallel scans -- iteration counts within +-1
    of the reference and the residual below the tolerance, not bit parity)."""
    cfg = cfg or SipConfig()
    s = _as_stencil(a)
    B, n, m = s.batch, s.n, s.m
    dev = s.device
    bb, _ = _as_batch(b, "rhs")
    if bb.shape[1] != n:
        raise DimensionMismatch(f"rhs length {bb.shape[1]}, expected {n}")
    if bb.shape[0] != B:
        raise DimensionMismatch(f"rhs batch {bb.shape[0]} != {B}")
    b_store = vector_to_layout(bb, n, s.layout, dev, s.ld)
    tol = torch.as_tensor(np.broadcast_to(np.asarray(cfg.tolerance, dtype=np.float64), (B,)).copy(),
                          device=dev)
    x = s.new_vector()
    use_x0 = 0
    if cfg.initial_guess is not None:
        g, _ = _as_batch(cfg.initial_guess, "initial_guess")
        if g.shape[1] != n:
            raise DimensionMismatch("initial guess has wrong length")
        x.copy_(vector_to_layout(np.broadcast_to(g, (B, n)) if not isinstance(g, torch.Tensor)
                                 else g.expand(B, n), n, s.layout, dev, s.ld))
        use_x0 = 1
    best_x = s.new_vector()
    iters = torch.zeros(B, dtype=torch.int64, device=dev)
    res = torch.empty(B, dtype=torch.float64, device=dev)
    best_res = torch.empty(B, dtype=torch.float64, device=dev)
    status = torch.empty(B, dtype=torch.int32, device=dev)
    index = torch.empty(B, dtype=torch.int32, device=dev)
    hist = (torch.full((B, cfg.max_iterations), float("nan"), dtype=torch.float64, device=dev)
            if record_history else None)
    al = ALGOS[algo] if isinstance(algo, str) else int(algo)
    nbytes = _lib.lib().bx_sip_workspace_bytes(B, n, m)
    ws = workspace(nbytes, dev)
    d = s.rowaligned()
    timer = _Timer()
    _lib.call("bx_sip_f64", *(ptr(v) for v in d), ptr(b_store), ptr(tol), ptr(x), ptr(best_x),
              ptr(iters), ptr(res), ptr(best_res), ptr(status), ptr(index), ptr(hist), B, n, m,
              float(cfg.alpha), int(cfg.max_iterations), use_x0, s.ld, s.layout, al, ptr(ws),
              ws.numel(), stream_handle())
    timer.end()
    xv = vector_from_layout(x, s.layout)
    if s.single:
        st = int(status[0])
        k = int(iters[0])
        if st == STATUS_MAX_ITER:
            bx1 = vector_from_layout(best_x, s.layout)[0].cpu().numpy()
            raise MaxIterationsExceeded(bx1, float(best_res[0]), k)
        if st != STATUS_OK:
            raise exception_for(st, int(index[0]), residual=float(res[0]), iterations=k)
        history = ()
        if record_history:
            h = hist[0, :k].cpu().numpy()
            history = tuple((i + 1, float(v)) for i, v in enumerate(h))
        x1 = xv[0].cpu().numpy()
        x1.setflags(write=False)
        return SolveReport(x=x1, iterations=k, residual_inf=float(res[0]),
                           ops=_sip_ops(n, k), wall_seconds=timer.seconds(), history=history,
                           status=status.cpu().numpy(), index=index.cpu().numpy())
    rep = SolveReport(x=xv, iterations=iters, residual_inf=res, ops=_sip_ops(n, iters),
                      wall_seconds=timer.seconds(), history=hist if record_history else (),
                      status=status, index=index, x_storage=x)
    rep.best_x = vector_from_layout(best_x, s.layout)
    rep.best_residual = best_res
    return rep


def _sip_ops(n, k):
    """Per-iteration loop-body tally of the reference (iterative.py:262-264):
    sweeps 2 x (5N-6 muls + 5N-6 adds), vec add N, forward 4N-6, backward
    5N-6 (N divs), vec sub N  ->  31N-36 per iteration."""
    muls = (2 * (5 * n - 6) + (2 * n - 3) + (2 * n - 3)) * k
    adds = (2 * (5 * n - 6) + n) * k
    subs = ((2 * n - 3) + (2 * n - 3) + n) * k
    divs = n * k
    return OpCounter(adds=adds, subs=subs, muls=muls, divs=divs)
