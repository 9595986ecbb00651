"""Batched band-matrix containers and result records (host side of the C ABI).

Mirrors the reference's value types (``bandix.core``, core.py:69-235) with a
batch axis and GPU residency:

* ``TriMatrix`` / ``PentaMatrix`` keep the reference constructor
  ``from_diagonals(...)`` and argument conventions (reference-length diagonals:
  sub2[i-2], sub1[i-1], main[i], sup1[i], sup2[i] for row i, core.py:117-183),
  accept one system (1-D sequences, exactly the reference call) or a batch
  (2-D, one system per row), and hold the diagonals on the GPU in the C ABI's
  ROW-ALIGNED storage: every diagonal has n rows, row i holds equation i's
  coefficient.  Default layout is interleaved ``(n, B)`` (system index
  fastest); ``layout="system"`` keeps ``(B, n)``.
* ``SolveReport`` carries x, iterations, residual_inf, ops, wall_seconds,
  history (core.py:226-235) plus the per-system ``status``/``index`` that
  replace exceptions in batched calls.
* ``OpCounter`` is the reference's closed-form operation tally (core.py:69-102).

Inputs are never mutated (the reference freezes them, core.py:48-53).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from fractions import Fraction
from typing import Any, Optional

import numpy as np
import torch

from . import _lib
from .errors import (DimensionMismatch, InvalidInput, STATUS_OK, exception_for)

LAYOUTS = {"interleaved": _lib.LAYOUT_INTERLEAVED, "system": _lib.LAYOUT_SYSTEM_MAJOR}


def default_device():
    if not torch.cuda.is_available():
        from .errors import CudaError
        raise CudaError("bandix_b200 needs a CUDA device (there is no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _as_batch(v, what):
    """-> (float64 numpy/torch 2-D array, single_flag)."""
    if isinstance(v, torch.Tensor):
        t = v.detach().to(torch.float64)
        if t.dim() == 1:
            return t.unsqueeze(0), True
        if t.dim() == 2:
            return t, False
        raise InvalidInput(f"{what}: expected 1-D or 2-D, got shape {tuple(t.shape)}")
    if not isinstance(v, np.ndarray) and len(v) and isinstance(v[0], Fraction):
        v = [float(q) for q in v]          # exact inputs are evaluated in binary64
    a = np.asarray(v, dtype=np.float64)
    if a.ndim == 1:
        return a[None, :], True
    if a.ndim == 2:
        return a, False
    raise InvalidInput(f"{what}: expected 1-D or 2-D, got shape {a.shape}")


def _to_device(a, device):
    if isinstance(a, torch.Tensor):
        return a.to(device=device, dtype=torch.float64)
    return torch.from_numpy(np.ascontiguousarray(a)).to(device=device)


def padded_ld(n):
    """System-major leading dimension of the band containers: n rounded up to
    4 doubles, so every system starts 32-byte aligned (the streaming
    partitioned kernel's vector loads, bx_direct_stream.cu)."""
    return (n + 3) // 4 * 4


def _system_major(batch, n, ld, device):
    ld = n if ld is None else ld
    return torch.zeros((batch, ld), dtype=torch.float64, device=device)[:, :n]


def pack_rows(arr, n, first_row, layout, device, batch, ld=None):
    """Reference-length diagonal (B, L) -> row-aligned device storage whose
    rows first_row .. first_row+L-1 hold it (other slots zero); system-major
    storage with leading dimension ld (default n)."""
    t = _to_device(arr, device)
    if t.shape[0] != batch:
        raise DimensionMismatch(f"batch {t.shape[0]} != {batch}")
    L = t.shape[1]
    if layout == _lib.LAYOUT_INTERLEAVED:
        out = torch.zeros((n, batch), dtype=torch.float64, device=device)
        out[first_row:first_row + L].copy_(t.t())
    else:
        out = _system_major(batch, n, ld, device)
        out[:, first_row:first_row + L].copy_(t)
    return out


def unpack_rows(t, first_row, length, layout):
    """Row-aligned device storage -> (B, L) view in reference indexing."""
    if layout == _lib.LAYOUT_INTERLEAVED:
        return t[first_row:first_row + length].t()
    return t[:, first_row:first_row + length]


def vector_to_layout(v, n, layout, device, ld=None):
    """(B, n) host/device vector -> device storage of the layout (system-major:
    leading dimension ld, default n)."""
    t = _to_device(v, device)
    if t.shape[1] != n:
        raise DimensionMismatch(f"rhs has length {t.shape[1]}, expected {n}")
    if layout == _lib.LAYOUT_INTERLEAVED:
        return t.t().contiguous()
    if ld is None or ld == n:
        return t.contiguous()
    out = _system_major(t.shape[0], n, ld, device)
    out.copy_(t)
    return out


def vector_from_layout(t, layout):
    """Device storage -> (B, n) view."""
    return t.t() if layout == _lib.LAYOUT_INTERLEAVED else t


def _ld(t, layout):
    return t.stride(0)


class _Band:
    """Common machinery of the batched containers."""

    names: tuple = ()
    offsets: tuple = ()

    def __init__(self, n, batch, diags, layout, single, device):
        self.n = n
        self.batch = batch
        self._diags = diags            # row-aligned device tensors, same shape/stride
        self.layout = layout
        self.single = single
        self.device = device
        self.exact = False
        t = diags[0]
        for d in diags:
            if d.shape != t.shape or d.stride() != t.stride() or d.dtype != torch.float64:
                raise InvalidInput("diagonals must share shape, stride and dtype float64")
        self.ld = t.stride(0)
        if t.stride(1) != 1:
            raise InvalidInput("row-aligned storage must be contiguous along its last axis")

    @classmethod
    def _build(cls, arrays, n_from, min_n, layout, device):
        lay = LAYOUTS[layout] if isinstance(layout, str) else layout
        device = torch.device(device) if device is not None else default_device()
        conv = [_as_batch(a, nm) for a, nm in zip(arrays, cls.names)]
        single = all(s for _, s in conv)
        mats = [m for m, _ in conv]
        batch = mats[0].shape[0]
        n = mats[n_from].shape[1]
        if n < min_n:
            raise InvalidInput(f"{cls.__name__} semantics need n >= {min_n}, got {n}")
        for m, off, nm in zip(mats, cls.offsets, cls.names):
            if m.shape[0] != batch:
                raise InvalidInput(f"{nm}: batch {m.shape[0]} != {batch}")
            if m.shape[1] != n - abs(off):
                raise InvalidInput(f"diagonal lengths do not match n={n} ({nm} has {m.shape[1]})")
        ld = padded_ld(n) if lay == _lib.LAYOUT_SYSTEM_MAJOR else None
        diags = [pack_rows(m, n, -off if off < 0 else 0, lay, device, batch, ld)
                 for m, off in zip(mats, cls.offsets)]
        return n, batch, diags, lay, single, device

    def diagonals(self):
        """Reference-length (B, L) views of the stored diagonals (core.py:145-146)."""
        out = []
        for d, off in zip(self._diags, self.offsets):
            first = -off if off < 0 else 0
            out.append(unpack_rows(d, first, self.n - abs(off), self.layout))
        return tuple(out)

    def rowaligned(self):
        return tuple(self._diags)

    def rhs(self, b):
        """Validate and lay out a right-hand side (or batch of them)."""
        bb, single = _as_batch(b, "rhs")
        if bb.shape[0] != self.batch:
            raise DimensionMismatch(f"rhs batch {bb.shape[0]} != {self.batch}")
        if bb.shape[1] != self.n:
            raise DimensionMismatch(f"rhs length {bb.shape[1]}, expected {self.n}")
        return vector_to_layout(bb, self.n, self.layout, self.device, self.ld)

    def new_vector(self):
        """Solution storage with the container's layout and leading dimension."""
        if self.layout == _lib.LAYOUT_INTERLEAVED:
            return torch.empty((self.n, self.batch), dtype=torch.float64, device=self.device)
        return torch.empty((self.batch, self.ld), dtype=torch.float64, device=self.device)[:, :self.n]

    def to_dense(self):
        """Dense (B, n, n) float64 host copy, for oracles and small reports (core.py:148-155)."""
        out = np.zeros((self.batch, self.n, self.n))
        for d, off in zip(self.diagonals(), self.offsets):
            dd = d.detach().cpu().numpy()
            for idx in range(dd.shape[1]):
                i = idx - min(off, 0)
                out[:, i, i + off] = dd[:, idx]
        return out


class TriMatrix(_Band):
    """Batched tridiagonal systems (offsets -1..+1), n >= 2 (core.py:167-202)."""

    names = ("sub1", "main", "sup1")
    offsets = (-1, 0, 1)

    @staticmethod
    def from_diagonals(sub1, main, sup1, exact=None, *, layout="interleaved", device=None):
        n, batch, diags, lay, single, dev = TriMatrix._build((sub1, main, sup1), 1, 2, layout, device)
        return TriMatrix(n, batch, diags, lay, single, dev)

    @staticmethod
    def from_rowaligned(sub1, main, sup1, layout="interleaved"):
        """Wrap device tensors already in the C ABI's row-aligned storage."""
        lay = LAYOUTS[layout] if isinstance(layout, str) else layout
        n, batch = (main.shape if lay == _lib.LAYOUT_INTERLEAVED else main.shape[::-1])
        return TriMatrix(n, batch, [sub1, main, sup1], lay, False, main.device)

    @property
    def sub1(self):
        return self.diagonals()[0]

    @property
    def main(self):
        return self.diagonals()[1]

    @property
    def sup1(self):
        return self.diagonals()[2]


class PentaMatrix(_Band):
    """Batched pentadiagonal systems (offsets -2..+2), n >= 3 (core.py:117-164)."""

    names = ("sub2", "sub1", "main", "sup1", "sup2")
    offsets = (-2, -1, 0, 1, 2)

    @staticmethod
    def from_diagonals(sub2, sub1, main, sup1, sup2, exact=None, *, layout="interleaved",
                       device=None):
        n, batch, diags, lay, single, dev = PentaMatrix._build(
            (sub2, sub1, main, sup1, sup2), 2, 3, layout, device)
        return PentaMatrix(n, batch, diags, lay, single, dev)

    @staticmethod
    def from_rowaligned(sub2, sub1, main, sup1, sup2, layout="interleaved"):
        lay = LAYOUTS[layout] if isinstance(layout, str) else layout
        n, batch = (main.shape if lay == _lib.LAYOUT_INTERLEAVED else main.shape[::-1])
        return PentaMatrix(n, batch, [sub2, sub1, main, sup1, sup2], lay, False, main.device)

    def sparse_outer(self, max_per_system=None):
        """The same systems with the +-2 diagonals held as a row-sorted list per
        system (MNPDM's case: only K rows carry outer entries, PAPER Remark 2,
        _elim.py:125-190).  Built once on the device (like a factorisation
        reused across time steps); ``solve_mnpdm`` then streams 40 B/row
        instead of 56.  Returns ``OuterSparsePenta``."""
        return OuterSparsePenta(self, max_per_system)

    @property
    def sub2(self):
        return self.diagonals()[0]

    @property
    def sub1(self):
        return self.diagonals()[1]

    @property
    def main(self):
        return self.diagonals()[2]

    @property
    def sup1(self):
        return self.diagonals()[3]

    @property
    def sup2(self):
        return self.diagonals()[4]


class OuterSparsePenta:
    """Pentadiagonal systems whose sub2/sup2 are kept as per-system lists of
    (row, sub2, sup2) in row order (``rows`` (B, k) int32, -1 pads); sub1, main,
    sup1 stay row-aligned (shared with the source matrix)."""

    def __init__(self, a, max_per_system=None):
        if not isinstance(a, PentaMatrix):
            raise TypeError("sparse_outer needs a PentaMatrix")
        self.dense = a
        self.n, self.batch, self.layout, self.single, self.device = (a.n, a.batch, a.layout,
                                                                    a.single, a.device)
        self.ld = a.ld
        c, _, _, _, g = a.rowaligned()
        count = torch.empty(a.batch, dtype=torch.int32, device=a.device)
        _lib.call("bx_outer_compact_f64", ptr(c), ptr(g), ptr(count), None, None, None, 0, a.batch,
                  a.n, a.ld, a.layout, stream_handle())
        k = int(count.max()) if a.batch else 0
        if max_per_system is not None and k > max_per_system:
            raise InvalidInput(f"{k} outer rows in a system exceed max_per_system={max_per_system}")
        self.k = k
        self.count = count
        self.rows = torch.empty((a.batch, max(k, 1)), dtype=torch.int32, device=a.device)
        self.vals_sub2 = torch.empty((a.batch, max(k, 1)), dtype=torch.float64, device=a.device)
        self.vals_sup2 = torch.empty((a.batch, max(k, 1)), dtype=torch.float64, device=a.device)
        if k:
            _lib.call("bx_outer_compact_f64", ptr(c), ptr(g), ptr(count), ptr(self.rows),
                      ptr(self.vals_sub2), ptr(self.vals_sup2), k, a.batch, a.n, a.ld, a.layout,
                      stream_handle())

    def rowaligned(self):
        return self.dense.rowaligned()

    def rhs(self, b):
        return self.dense.rhs(b)

    def new_vector(self):
        return self.dense.new_vector()


@dataclass(frozen=True)
class OpCounter:
    """Scalar-operation tally (core.py:69-102), closed form per method."""

    adds: Any = 0
    subs: Any = 0
    muls: Any = 0
    divs: Any = 0

    @property
    def total(self):
        return self.adds + self.subs + self.muls + self.divs

    def plus(self, adds=0, subs=0, muls=0, divs=0):
        return OpCounter(self.adds + adds, self.subs + subs, self.muls + muls, self.divs + divs)

    def merged(self, other):
        return self.plus(other.adds, other.subs, other.muls, other.divs)

    def as_dict(self):
        return {"adds": self.adds, "subs": self.subs, "muls": self.muls, "divs": self.divs,
                "total": self.total}


class _Timer:
    """CUDA-event stopwatch on the current stream; read lazily."""

    def __init__(self):
        self.start = torch.cuda.Event(enable_timing=True)
        self.stop = torch.cuda.Event(enable_timing=True)
        self.start.record()

    def end(self):
        self.stop.record()
        return self

    def seconds(self):
        self.stop.synchronize()
        return self.start.elapsed_time(self.stop) / 1e3


@dataclass
class SolveReport:
    """Outcome of a (batched) solve (core.py:226-235).

    Batched: ``x`` is a (B, n) device tensor (a view of the layout storage),
    ``iterations``/``residual_inf``/``status``/``index`` are (B,) device
    tensors.  Single-system calls return host values exactly like the
    reference (numpy x, float residual, int iterations) and raise instead of
    reporting a status.
    """

    x: Any
    iterations: Any
    residual_inf: Any
    ops: OpCounter
    wall_seconds: float
    history: tuple = ()
    status: Any = None
    index: Any = None
    x_storage: Any = field(default=None, repr=False)

    def ok(self):
        return bool((self.status == STATUS_OK).all())

    def raise_for_status(self):
        """Raise the reference exception for the first failing system."""
        st = self.status.detach().cpu().numpy() if isinstance(self.status, torch.Tensor) else np.asarray(self.status)
        bad = np.nonzero(st != STATUS_OK)[0]
        if bad.size:
            s = int(bad[0])
            ix = self.index.detach().cpu().numpy() if isinstance(self.index, torch.Tensor) else np.asarray(self.index)
            it = self.iterations
            it_s = int(it[s]) if hasattr(it, "__len__") else it
            res = self.residual_inf
            res_s = float(res[s]) if hasattr(res, "__len__") else res
            raise exception_for(int(st[s]), int(ix[s]), best=None, residual=res_s, iterations=it_s)


@dataclass(frozen=True)
class BandFactors:
    """Banded (I)LU factors, row-aligned device storage (core.py:208-223):
    row i of l_sub1 / l_sub2 holds L(i, i-1) / L(i, i-m), of u_main /
    u_sup1 / u_sup2 U(i, i) / U(i, i+1) / U(i, i+m).  Producers attach
    ``layout``, ``batch``, ``single``, ``status`` and ``index``."""

    n: int
    l_sub1: Any
    l_sub2: Any
    u_main: Any
    u_sup1: Any
    u_sup2: Any
    m: int = 2
    exact: bool = False

    def ref(self):
        """(l_sub1, l_sub2, u_main, u_sup1, u_sup2) as (B, len) views in the
        reference's unpadded lengths n-1, n-m, n, n-1, n-m."""
        lay, n, m = getattr(self, "layout", _lib.LAYOUT_INTERLEAVED), self.n, self.m
        return (unpack_rows(self.l_sub1, 1, n - 1, lay), unpack_rows(self.l_sub2, m, n - m, lay),
                unpack_rows(self.u_main, 0, n, lay), unpack_rows(self.u_sup1, 0, n - 1, lay),
                unpack_rows(self.u_sup2, 0, n - m, lay))


class CounterBox:
    """Mutable holder threading an OpCounter through a call (core.py:105-114)."""

    __slots__ = ("counter",)

    def __init__(self):
        self.counter = OpCounter()

    def add(self, adds=0, subs=0, muls=0, divs=0):
        self.counter = self.counter.plus(adds, subs, muls, divs)


# ---- band helpers of the reference's core.py (243-334) ------------------------
def _vec_in(a, x, what="vector"):
    """x for band container a -> (storage in a's layout / ld, single flag)."""
    xb, single = _as_batch(x, what)
    if xb.shape[1] != a.n:
        raise DimensionMismatch(f"{what} has length {xb.shape[1]}, expected {a.n}")
    if xb.shape[0] != a.batch:
        raise DimensionMismatch(f"{what} batch {xb.shape[0]} != {a.batch}")
    return vector_to_layout(xb, a.n, a.layout, a.device, a.ld), single


def _vec_out(a, store, single):
    v = vector_from_layout(store, a.layout)
    if single:
        out = v[0].detach().cpu().numpy()
        out.setflags(write=False)
        return out
    return v


def _band_matvec(a, x, b=None):
    """bx_band_matvec_f64: A x, or b - A x when b is given (device storage)."""
    xs, single = _vec_in(a, x)
    bs = _vec_in(a, b, "rhs")[0] if b is not None else None
    y = a.new_vector()
    diags = a.rowaligned()
    if len(diags) == 3:
        bw, m, (c, d, e, f, g) = 1, 2, (None,) + tuple(diags) + (None,)
    else:
        bw, m, (c, d, e, f, g) = 2, getattr(a, "m", 2), diags
    _lib.call("bx_band_matvec_f64", bw, m, ptr(c), ptr(d), ptr(e), ptr(f), ptr(g), ptr(xs), ptr(bs),
              ptr(y), a.batch, a.n, a.ld, a.layout, stream_handle())
    return _vec_out(a, y, single and a.single)


def penta_matvec(a, x, counter=None):
    """A @ x for pentadiagonal A (core.py:243-268): 5N-6 muls, 4N-6 adds;
    the reference's float order (main, sub1, sup1, sub2, sup2), bit-identical."""
    if counter is not None:
        counter.add(muls=5 * a.n - 6, adds=4 * a.n - 6)
    return _band_matvec(a, x)


def tri_matvec(t, x, counter=None):
    """T @ x for tridiagonal T (core.py:271-289): 3N-2 muls, 2N-2 adds."""
    if counter is not None:
        counter.add(muls=3 * t.n - 2, adds=2 * t.n - 2)
    return _band_matvec(t, x)


def matvec(a, x, counter=None):
    """core.py:292-295."""
    return penta_matvec(a, x, counter) if isinstance(a, PentaMatrix) else tri_matvec(a, x, counter)


def residual(a, x, b, counter=None):
    """b - A @ x, entrywise (core.py:307-316): matvec ops + N subs."""
    if counter is not None:
        if isinstance(a, PentaMatrix):
            counter.add(muls=5 * a.n - 6, adds=4 * a.n - 6)
        else:
            counter.add(muls=3 * a.n - 2, adds=2 * a.n - 2)
        counter.add(subs=a.n)
    return _band_matvec(a, x, b)


def inf_norm(v):
    """Maximum absolute entry; the empty vector has norm 0 (core.py:298-304).
    A 2-D batch gives one norm per row (NaN propagates, as numpy.max)."""
    if isinstance(v, torch.Tensor):
        if v.numel() == 0:
            return 0 if v.dim() < 2 else torch.zeros(v.shape[0], dtype=torch.float64, device=v.device)
        return torch.amax(v.abs(), dim=-1) if v.dim() == 2 else float(torch.amax(v.abs()))
    a = np.asarray(v, dtype=np.float64)
    if a.size == 0:
        return 0
    return np.max(np.abs(a), axis=-1) if a.ndim == 2 else float(np.max(np.abs(a)))


def outer_nonzero_count(a):
    """Rows with a structurally nonzero sub2 entry plus rows with a nonzero
    sup2 entry (core.py:319-334): exact zero test on the stored data.  An int
    for a single system, a (B,) tensor for a batch."""
    sub2, _, _, _, sup2 = a.diagonals()
    k = torch.count_nonzero(sub2, dim=1) + torch.count_nonzero(sup2, dim=1)
    return int(k[0]) if a.single else k


_WS_CACHE: dict = {}


def workspace(nbytes, device):
    """Reusable scratch buffer (grown on demand, never shrunk)."""
    key = (device.index if device.index is not None else torch.cuda.current_device())
    buf = _WS_CACHE.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)
        _WS_CACHE[key] = buf
    return buf


def stream_handle():
    return torch.cuda.current_stream().cuda_stream


def ptr(t: Optional[torch.Tensor]):
    return None if t is None else t.data_ptr()
