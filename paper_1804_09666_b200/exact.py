"""Symbolic solvers SPDM / STDM -- the reference's ``bandix.exact`` entry
points (exact.py:278-307) over the CUDA C ABI.

Zero pivots are replaced by the indeterminate t and the solution is
evaluated in the limit t -> 0, as in the reference; the rational functions of
t are carried as truncated Laurent series with binary64 coefficients
(DESIGN.md "symbolic solvers").  Conventions that differ from the reference,
by design:

* inputs are binary64 (a float is an exact rational; the reference demands
  Fraction input and raises InvalidInput for floats, exact.py:232-236) and
  x is returned in binary64 -- the correctly-rounded exact answer up to the
  conditioning of the system, not a tuple of Fractions;
* batched calls report SingularMatrix / window overflow per system in
  ``status`` instead of raising.
"""

from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction
from typing import Any

import numpy as np
import torch

from . import _lib
from .core import OpCounter, PentaMatrix, TriMatrix, _as_batch, ptr, stream_handle, \
    vector_from_layout, vector_to_layout, workspace
from .errors import InvalidInput, STATUS_OK, exception_for


@dataclass
class ExactSolveResult:
    """Solution plus the number of zero pivots replaced by t (exact.py:213-218)."""

    x: Any
    pivot_substitutions: Any
    status: Any = None
    index: Any = None


def _rhs(a, b):
    bb, _ = _as_batch(b, "rhs")
    if bb.shape[1] != a.n:
        raise InvalidInput(f"rhs length {bb.shape[1]} does not match n={a.n}")
    if bb.shape[0] != a.batch:
        raise InvalidInput(f"rhs batch {bb.shape[0]} != {a.batch}")
    return vector_to_layout(bb, a.n, a.layout, a.device, a.ld)


def _solve(kind, a, b):
    b_store = _rhs(a, b)
    x = a.new_vector()
    dev = a.device
    status = torch.empty(a.batch, dtype=torch.int32, device=dev)
    index = torch.empty(a.batch, dtype=torch.int32, device=dev)
    subs = torch.empty(a.batch, dtype=torch.int32, device=dev)
    solver = "stdm" if kind == 1 else "spdm"
    nbytes = _lib.lib().bx_workspace_bytes(_lib.SOLVER[solver], a.batch, a.n, a.layout, 0)
    ws = workspace(nbytes, dev)
    if kind == 1:
        d, e, f = a.rowaligned()
        _lib.call("bx_stdm_f64", ptr(d), ptr(e), ptr(f), ptr(b_store), ptr(x), ptr(status),
                  ptr(index), ptr(subs), a.batch, a.n, a.ld, a.layout, ptr(ws), ws.numel(),
                  stream_handle())
    else:
        c, d, e, f, g = a.rowaligned()
        _lib.call("bx_spdm_f64", ptr(c), ptr(d), ptr(e), ptr(f), ptr(g), ptr(b_store), ptr(x),
                  ptr(status), ptr(index), ptr(subs), a.batch, a.n, a.ld, a.layout, ptr(ws),
                  ws.numel(), stream_handle())
    xv = vector_from_layout(x, a.layout)
    if a.single:
        st = int(status[0])
        if st != STATUS_OK:
            raise exception_for(st, int(index[0]))
        x1 = xv[0].cpu().numpy()
        x1.setflags(write=False)
        return ExactSolveResult(x1, int(subs[0]), status.cpu().numpy(), index.cpu().numpy())
    return ExactSolveResult(xv, subs, status, index)


def exact_solve_stdm(t: TriMatrix, b) -> ExactSolveResult:
    """Symbolic tridiagonal solve (exact.py:296-307)."""
    if not isinstance(t, TriMatrix):
        raise TypeError("expected a TriMatrix")
    return _solve(1, t, b)


def exact_solve_spdm(a: PentaMatrix, b) -> ExactSolveResult:
    """Symbolic pentadiagonal solve (exact.py:278-293)."""
    if not isinstance(a, PentaMatrix):
        raise TypeError("expected a PentaMatrix")
    return _solve(2, a, b)


@dataclass
class BandDeterminant:
    """Batched exact_det_band result: det[s] = mantissa[s] * 2**exponent[s]
    (|mantissa| in [0.5, 1) or 0: products of thousands of pivots leave the
    binary64 range), plus the substitution count and status per system."""

    mantissa: Any
    exponent: Any
    pivot_substitutions: Any
    status: Any
    index: Any

    def sign(self):
        return torch.sign(self.mantissa)

    def log2abs(self):
        """log2 |det| (-inf for a zero determinant)."""
        return torch.log2(self.mantissa.abs()) + self.exponent.to(self.mantissa.dtype)

    def to_fraction(self, s: int = 0) -> Fraction:
        """det of system s as the exact rational value of the binary64 result."""
        m = float(self.mantissa[s])
        e = int(self.exponent[s])
        return Fraction(m) * (Fraction(2) ** e)


def _det_ops(a) -> OpCounter:
    """Closed-form op count of exact_det_band (exact.py:266-272)."""
    n = a.n
    if isinstance(a, PentaMatrix):
        return OpCounter(muls=4 * n - 7 + (n - 1), subs=4 * n - 7, divs=2 * n - 3)
    return OpCounter(muls=2 * n - 2 + (n - 1), subs=n - 1, divs=n)


def exact_det_band(a, counter=None):
    """Determinant of a band matrix from the t-substituted pivots at t -> 0
    (exact.py:254-275).  Zero is a valid return: the nonsingularity test of
    the symbolic solvers is det != 0.

    Single system (1-D diagonals): a ``Fraction`` like the reference -- the
    exact rational value of the binary64 determinant (inputs are binary64,
    the module's convention).  Batched: a :class:`BandDeterminant`.
    ``counter`` (an object with ``add(**ops)``, e.g. the reference's
    CounterBox) receives the reference's closed-form op counts."""
    if isinstance(a, TriMatrix):
        bw, diags = 1, (None,) + tuple(a.rowaligned()) + (None,)
    elif isinstance(a, PentaMatrix):
        bw, diags = 2, tuple(a.rowaligned())
    else:
        raise TypeError("expected a TriMatrix or PentaMatrix")
    dev = a.device
    mant = torch.empty(a.batch, dtype=torch.float64, device=dev)
    expo = torch.empty(a.batch, dtype=torch.int64, device=dev)
    status = torch.empty(a.batch, dtype=torch.int32, device=dev)
    index = torch.empty(a.batch, dtype=torch.int32, device=dev)
    subs = torch.empty(a.batch, dtype=torch.int32, device=dev)
    _lib.call("bx_det_band_f64", bw, *(ptr(d) for d in diags), ptr(mant), ptr(expo), ptr(status),
              ptr(index), ptr(subs), a.batch, a.n, a.ld, a.layout, stream_handle())
    if counter is not None:
        ops = _det_ops(a)
        counter.add(muls=ops.muls * a.batch, subs=ops.subs * a.batch, divs=ops.divs * a.batch)
    res = BandDeterminant(mant, expo, subs, status, index)
    if a.single:
        st = int(status[0])
        if st != STATUS_OK:
            raise exception_for(st, int(index[0]))
        return res.to_fraction(0)
    return res


def rcond_band(a):
    """Reciprocal 1-norm condition estimate of every system, LAPACK's
    convention (dgtcon / dgbcon, norm '1'): the condition
    gate next to exact_det_band, against which config-3 errors are read
    (SURVEY H7).  Single system: a float (0.0 when exactly singular);
    batched: (rcond (B,), status, index) device tensors."""
    if isinstance(a, TriMatrix):
        bw, diags = 1, (None,) + tuple(a.rowaligned()) + (None,)
    elif isinstance(a, PentaMatrix):
        bw, diags = 2, tuple(a.rowaligned())
    else:
        raise TypeError("expected a TriMatrix or PentaMatrix")
    dev = a.device
    rc = torch.empty(a.batch, dtype=torch.float64, device=dev)
    status = torch.empty(a.batch, dtype=torch.int32, device=dev)
    index = torch.empty(a.batch, dtype=torch.int32, device=dev)
    ws = workspace(_lib.lib().bx_rcond_workspace_bytes(bw, a.batch, a.n), dev)
    _lib.call("bx_rcond_band_f64", bw, *(ptr(d) for d in diags), ptr(rc), ptr(status), ptr(index),
              a.batch, a.n, a.ld, a.layout, ptr(ws), ws.numel(), stream_handle())
    if a.single:
        return float(rc[0])
    return rc, status, index
