"""Direct band solvers (NTDM, NPDM, MNPDM) -- the reference's ``bandix.direct``
entry points (direct.py:73-113) over the CUDA C ABI.

Each call solves ONE system when given 1-D inputs (returning host values and
raising ``ZeroPivot`` exactly as the reference does) or a batch of systems
when given 2-D inputs / batched containers (per-system ``status``/``index``
instead of exceptions).

``algo``:
  * ``"sequential"`` (default) -- the reference's operation order, one thread
    per system: results are bit-identical to bandix.
  * ``"partitioned"`` -- on-chip partitioned elimination for throughput;
    agrees with the reference within the north-star tolerance (<= 1e-10
    relative on nonsingular, well-conditioned systems), not bitwise.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .core import (BandFactors, OpCounter, OuterSparsePenta, PentaMatrix, SolveReport, TriMatrix,
                   _Timer, ptr, stream_handle, vector_from_layout, workspace)
from .errors import DimensionMismatch, STATUS_OK, exception_for
from collections import namedtuple

ALGOS = {"sequential": _lib.ALGO_SEQUENTIAL, "partitioned": _lib.ALGO_PARTITIONED}


def _algo(algo):
    if isinstance(algo, str):
        if algo not in ALGOS:
            raise ValueError(f"unknown algo {algo!r}; expected one of {sorted(ALGOS)}")
        return ALGOS[algo]
    return int(algo)


def _coerce(a, kind):
    if kind == "tri" and not isinstance(a, TriMatrix):
        raise TypeError("expected a bandix_b200 TriMatrix")
    if kind == "penta" and not isinstance(a, PentaMatrix):
        raise TypeError("expected a bandix_b200 PentaMatrix")
    return a


def lu_penta(a: PentaMatrix, counter=None) -> BandFactors:
    """Doolittle factorisation restricted to the band (direct.py:42-63): 10N-17
    ops, the reference's operation order (penta_factor, _elim.py:30-62) -- the
    factors are bit-identical.  Factor once, then ``forward_sub`` /
    ``backward_sub`` (iterative.py) for every right-hand side.  One system
    raises ZeroPivot(i); a batch carries ``status`` / ``index``."""
    a = _coerce(a, "penta")
    outs = [a.new_vector() for _ in range(5)]   # mu, l1, l2, phi, psi
    status = torch.empty(a.batch, dtype=torch.int32, device=a.device)
    index = torch.empty(a.batch, dtype=torch.int32, device=a.device)
    _lib.call("bx_lu_penta_f64", *(ptr(v) for v in a.rowaligned()), *(ptr(v) for v in outs),
              ptr(status), ptr(index), a.batch, a.n, a.ld, a.layout, stream_handle())
    if counter is not None:
        counter.add(muls=4 * a.n - 7, subs=4 * a.n - 7, divs=2 * a.n - 3)
    if a.single and int(status[0]) != STATUS_OK:
        raise exception_for(int(status[0]), int(index[0]))
    mu, l1, l2, phi, psi = outs
    f = BandFactors(a.n, l1, l2, mu, phi, psi, m=2)
    for k, v in (("status", status), ("index", index), ("layout", a.layout), ("single", a.single),
                 ("batch", a.batch), ("ld", a.ld), ("device", a.device)):
        object.__setattr__(f, k, v)
    return f


def ops_ntdm(n):
    """9N-7 (direct.py:111-112)."""
    return OpCounter(muls=5 * n - 4, subs=3 * n - 3, divs=n)


def ops_npdm(n):
    """19N-29: lu_penta 10N-17 + forward 4N-6 + backward 5N-6 (direct.py:52-53;
    iterative.py:134, 146)."""
    return OpCounter(muls=8 * n - 13, subs=8 * n - 13, divs=3 * n - 3)


def ops_mnpdm(n, nz):
    """13N-15 + 7 nz(sub2) (direct.py:98-99); nz may be a per-system array."""
    return OpCounter(muls=7 * n - 8 + 4 * nz, subs=5 * n - 7 + 3 * nz, divs=n)


def _scalar(v):
    if isinstance(v, torch.Tensor):
        return int(v.reshape(-1)[0].item())
    return int(np.asarray(v).reshape(-1)[0])


def _finish(a, x_store, status, index, timer, b_store, ops, residual):
    res = None
    if residual:
        res = torch.empty(a.batch, dtype=torch.float64, device=a.device)
        diags = a.rowaligned()
        if isinstance(a, TriMatrix):
            c = g = None
            d, e, f = diags
            bw = 1
        else:
            c, d, e, f, g = diags
            bw = 2
        _lib.call("bx_residual_inf_f64", bw, ptr(c), ptr(d), ptr(e), ptr(f), ptr(g), ptr(x_store),
                  ptr(b_store), ptr(res), a.batch, a.n, a.ld, a.layout, stream_handle())
    x = vector_from_layout(x_store, a.layout)
    rep = SolveReport(x=x, iterations=0, residual_inf=res, ops=ops, wall_seconds=timer,
                      status=status, index=index, x_storage=x_store)
    if a.single:
        st = int(status[0])
        if st != STATUS_OK:
            raise exception_for(st, int(index[0]))
        ops1 = OpCounter(*(_scalar(v) for v in (ops.adds, ops.subs, ops.muls, ops.divs)))
        x1 = x[0].detach().cpu().numpy()
        x1.setflags(write=False)
        return SolveReport(x=x1, iterations=0,
                           residual_inf=float(res[0]) if res is not None else float("nan"),
                           ops=ops1, wall_seconds=timer.seconds(),
                           status=status.cpu().numpy(), index=index.cpu().numpy())
    rep.wall_seconds = timer.seconds() if timer is not None else float("nan")
    return rep


def solve_ntdm(t: TriMatrix, b, *, algo="sequential", residual=True) -> SolveReport:
    """Thomas solve with reciprocal-normalised pivots: 9N-7 ops (direct.py:103-113)."""
    t = _coerce(t, "tri")
    b_store = t.rhs(b)
    x = t.new_vector()
    status = torch.empty(t.batch, dtype=torch.int32, device=t.device)
    index = torch.empty(t.batch, dtype=torch.int32, device=t.device)
    al = _algo(algo)
    nbytes = _lib.lib().bx_workspace_bytes(_lib.SOLVER["ntdm"], t.batch, t.n, t.layout, al)
    ws = workspace(nbytes, t.device)
    d, e, f = t.rowaligned()
    timer = _Timer()
    _lib.call("bx_ntdm_f64", ptr(d), ptr(e), ptr(f), ptr(b_store), ptr(x), ptr(status), ptr(index),
              t.batch, t.n, t.ld, t.layout, al, ptr(ws), ws.numel(), stream_handle())
    timer.end()
    return _finish(t, x, status, index, timer, b_store, ops_ntdm(t.n), residual)


def solve_npdm(a: PentaMatrix, b, *, algo="sequential", residual=True) -> SolveReport:
    """Pentadiagonal solve via banded LU plus substitutions: 19N-29 ops (direct.py:73-81)."""
    a = _coerce(a, "penta")
    b_store = a.rhs(b)
    x = a.new_vector()
    status = torch.empty(a.batch, dtype=torch.int32, device=a.device)
    index = torch.empty(a.batch, dtype=torch.int32, device=a.device)
    al = _algo(algo)
    nbytes = _lib.lib().bx_workspace_bytes(_lib.SOLVER["npdm"], a.batch, a.n, a.layout, al)
    ws = workspace(nbytes, a.device)
    c, d, e, f, g = a.rowaligned()
    timer = _Timer()
    _lib.call("bx_npdm_f64", ptr(c), ptr(d), ptr(e), ptr(f), ptr(g), ptr(b_store), ptr(x),
              ptr(status), ptr(index), a.batch, a.n, a.ld, a.layout, al, ptr(ws), ws.numel(),
              stream_handle())
    timer.end()
    return _finish(a, x, status, index, timer, b_store, ops_npdm(a.n), residual)


def solve_mnpdm(a: PentaMatrix, b, *, algo="sequential", residual=True) -> SolveReport:
    """Sparsity-aware pentadiagonal solve: 13N-15 + 7 nz(sub2) ops (direct.py:84-100).

    ``a`` may be ``PentaMatrix.sparse_outer()``: the partitioned algorithm then
    streams only sub1/main/sup1/rhs plus the outer-row lists (the sequential,
    bit-exact algorithm runs on the dense source)."""
    if isinstance(a, OuterSparsePenta):
        if _algo(algo) != _lib.ALGO_PARTITIONED:
            return solve_mnpdm(a.dense, b, algo=algo, residual=residual)
        b_store = a.rhs(b)
        x = a.new_vector()
        status = torch.empty(a.batch, dtype=torch.int32, device=a.device)
        index = torch.empty(a.batch, dtype=torch.int32, device=a.device)
        nz = torch.zeros(a.batch, dtype=torch.int64, device=a.device)
        _, d, e, f, _ = a.rowaligned()
        timer = _Timer()
        _lib.call("bx_mnpdm_sparse_f64", ptr(a.rows), ptr(a.vals_sub2), ptr(a.vals_sup2), a.k,
                  ptr(d), ptr(e), ptr(f), ptr(b_store), ptr(x), ptr(status), ptr(index), ptr(nz),
                  a.batch, a.n, a.ld, a.layout, stream_handle())
        timer.end()
        return _finish(a.dense, x, status, index, timer, b_store, ops_mnpdm(a.n, nz), residual)
    a = _coerce(a, "penta")
    b_store = a.rhs(b)
    x = a.new_vector()
    status = torch.empty(a.batch, dtype=torch.int32, device=a.device)
    index = torch.empty(a.batch, dtype=torch.int32, device=a.device)
    nz = torch.zeros(a.batch, dtype=torch.int64, device=a.device)
    al = _algo(algo)
    nbytes = _lib.lib().bx_workspace_bytes(_lib.SOLVER["mnpdm"], a.batch, a.n, a.layout, al)
    ws = workspace(nbytes, a.device)
    c, d, e, f, g = a.rowaligned()
    timer = _Timer()
    _lib.call("bx_mnpdm_f64", ptr(c), ptr(d), ptr(e), ptr(f), ptr(g), ptr(b_store), ptr(x),
              ptr(status), ptr(index), ptr(nz), a.batch, a.n, a.ld, a.layout, al, ptr(ws),
              ws.numel(), stream_handle())
    timer.end()
    return _finish(a, x, status, index, timer, b_store, ops_mnpdm(a.n, nz), residual)


ReductionResult = namedtuple("ReductionResult", "tri rhs ops status index")


def pd_to_td(a: PentaMatrix, b):
    """Gaussian reduction of pentadiagonal systems to tridiagonal ones
    (direct.py:116-165), the reference's operation order (bit-identical).

    One system (1-D inputs): returns ``(TriMatrix, rhs, OpCounter)`` like the
    reference and raises ``ReductionPivotZero(i)``.  A batch: returns
    ``ReductionResult(tri, rhs, ops, status, index)`` with per-system
    ``OpCounter`` tensors and status ``STATUS_REDUCTION_PIVOT`` / index."""
    a = _coerce(a, "penta")
    b_store = a.rhs(b)
    lay = a.layout
    shape = (a.n, a.batch) if lay == _lib.LAYOUT_INTERLEAVED else (a.batch, a.n)
    out = [torch.empty(shape, dtype=torch.float64, device=a.device) for _ in range(4)]
    ops = torch.zeros((a.batch, 3), dtype=torch.int64, device=a.device)
    status = torch.empty(a.batch, dtype=torch.int32, device=a.device)
    index = torch.empty(a.batch, dtype=torch.int32, device=a.device)
    c, d, e, f, g = a.rowaligned()
    _lib.call("bx_pd2td_f64", ptr(c), ptr(d), ptr(e), ptr(f), ptr(g), ptr(b_store),
              *(ptr(t) for t in out), ptr(ops), ptr(status), ptr(index), a.batch, a.n, a.ld,
              out[0].stride(0), lay, stream_handle())
    tri = TriMatrix.from_rowaligned(out[0], out[1], out[2], layout=lay)
    counter = OpCounter(adds=0, subs=ops[:, 1], muls=ops[:, 0], divs=ops[:, 2])
    rhs = vector_from_layout(out[3], lay)
    if a.single:
        st = int(status[0])
        if st != STATUS_OK:
            raise exception_for(st, int(index[0]))
        tri.single = True
        c1 = OpCounter(0, int(ops[0, 1]), int(ops[0, 0]), int(ops[0, 2]))
        r1 = rhs[0].detach().cpu().numpy()
        r1.setflags(write=False)
        return tri, r1, c1
    return ReductionResult(tri, rhs, counter, status, index)


def solve_pd2td_ntdm(a: PentaMatrix, b, *, residual=True) -> SolveReport:
    """Reduce to tridiagonal, then the Thomas method (direct.py:168-177); the
    report residual is taken against the original pentadiagonal system and the
    op count is the reduction's plus NTDM's 9N-7."""
    a = _coerce(a, "penta")
    b_store = a.rhs(b)
    x = a.new_vector()
    ops = torch.zeros((a.batch, 3), dtype=torch.int64, device=a.device)
    status = torch.empty(a.batch, dtype=torch.int32, device=a.device)
    index = torch.empty(a.batch, dtype=torch.int32, device=a.device)
    nbytes = _lib.lib().bx_workspace_bytes(_lib.SOLVER["pd2td"], a.batch, a.n, a.layout, 0)
    ws = workspace(nbytes, a.device)
    c, d, e, f, g = a.rowaligned()
    timer = _Timer()
    _lib.call("bx_pd2td_ntdm_f64", ptr(c), ptr(d), ptr(e), ptr(f), ptr(g), ptr(b_store), ptr(x),
              ptr(ops), ptr(status), ptr(index), a.batch, a.n, a.ld, a.layout, ptr(ws), ws.numel(),
              stream_handle())
    timer.end()
    red = OpCounter(adds=0, subs=ops[:, 1], muls=ops[:, 0], divs=ops[:, 2])
    return _finish(a, x, status, index, timer, b_store, red.merged(ops_ntdm(a.n)), residual)


def check_rhs(n, b):
    if len(b) != n:
        raise DimensionMismatch(f"rhs length {len(b)}, expected {n}")
