"""Generate the golden vectors by running the REFERENCE (bandix 0.1.0) itself.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

Every case feeds seeded inputs (paper_1804_09666_b200.workloads, or a small
hand case from SPEC.md) through the reference's public functions, one system
per call exactly as the reference API works, and stores inputs and outputs in
``tests/golden/*.npz``.  The files are committed; nothing at test time reads
/root/reference.
"""

from __future__ import annotations

import os
import sys
import time
from fractions import Fraction

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

from bandix import core, direct, exact, inverse, iterative  # noqa: E402
from bandix.errors import (MaxIterationsExceeded, ReductionPivotZero, ZeroPivot)  # noqa: E402

from paper_1804_09666_b200 import workloads as W  # noqa: E402


def _save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path}")


def _run_direct(kind, diags, rhs):
    """One reference call per system; x=NaN + index on ZeroPivot."""
    bsz, n = rhs.shape
    xs = np.full((bsz, n), np.nan)
    res = np.full(bsz, np.nan)
    ops = np.zeros(bsz, dtype=np.int64)
    status = np.zeros(bsz, dtype=np.int32)
    index = np.full(bsz, -1, dtype=np.int32)
    for s in range(bsz):
        cols = [d[s] for d in diags]
        try:
            if kind == "ntdm":
                rep = direct.solve_ntdm(core.TriMatrix.from_diagonals(*cols), rhs[s])
            else:
                a = core.PentaMatrix.from_diagonals(*cols)
                rep = (direct.solve_npdm if kind == "npdm" else direct.solve_mnpdm)(a, rhs[s])
            xs[s] = rep.x
            res[s] = rep.residual_inf
            ops[s] = rep.ops.total
        except ZeroPivot as zp:
            status[s] = 1
            index[s] = zp.index
    return xs, res, ops, status, index


def golden_direct():
    out = {}
    # config 1 sample (seeded exactly as config 1, reduced batch)
    d = W.td_dominant(16, 1024, seed=0)
    x, r, o, st, ix = _run_direct("ntdm", d[:3], d[3])
    out.update(ntdm_sub1=d[0], ntdm_main=d[1], ntdm_sup1=d[2], ntdm_rhs=d[3],
               ntdm_x=x, ntdm_res=r, ntdm_ops=o, ntdm_status=st, ntdm_index=ix)
    # ntdm edge cases: n=2, n=3, zero pivot at 0 and at 5
    sub = np.array([[-1.0, -1.0]]); main = np.array([[2.0, 2.0, 2.0]]); sup = np.array([[-1.0, -1.0]])
    b = np.array([[1.0, 0.0, 1.0]])
    x, *_ = _run_direct("ntdm", (sub, main, sup), b)
    out.update(ntdm_spec_x=x)
    e = W.td_dominant(3, 16, seed=11)
    sub1, main, sup1, rhs = (a.copy() for a in e)
    main[0, 0] = 0.0                         # pivot 0 at row 0
    # make row 5 of system 1 an exact zero pivot: decouple (sub=main=0)
    sub1[1, 4] = 0.0; main[1, 5] = 0.0
    x, r, o, st, ix = _run_direct("ntdm", (sub1, main, sup1), rhs)
    out.update(ntdmz_sub1=sub1, ntdmz_main=main, ntdmz_sup1=sup1, ntdmz_rhs=rhs,
               ntdmz_x=x, ntdmz_status=st, ntdmz_index=ix)
    n2 = W.td_dominant(4, 2, seed=12)
    x, r, o, st, ix = _run_direct("ntdm", n2[:3], n2[3])
    out.update(ntdm2_sub1=n2[0], ntdm2_main=n2[1], ntdm2_sup1=n2[2], ntdm2_rhs=n2[3], ntdm2_x=x)

    # config 2 sample, full band and sparse outer (MNPDM family)
    for tag, sparse in (("pd", False), ("pds", True)):
        p = W.pd_dominant(8, 512, seed=1, sparse_outer=sparse)
        out.update({f"{tag}_{k}": v for k, v in zip(("sub2", "sub1", "main", "sup1", "sup2", "rhs"), p)})
        for kind in ("npdm", "mnpdm"):
            x, r, o, st, ix = _run_direct(kind, p[:5], p[5])
            out.update({f"{tag}_{kind}_x": x, f"{tag}_{kind}_res": r, f"{tag}_{kind}_ops": o})
    # small orders n = 3, 4, 5 and zero pivots
    for n in (3, 4, 5):
        p = W.pd_dominant(3, n, seed=20 + n)
        out.update({f"pd{n}_{k}": v for k, v in zip(("sub2", "sub1", "main", "sup1", "sup2", "rhs"), p)})
        for kind in ("npdm", "mnpdm"):
            x, *_ = _run_direct(kind, p[:5], p[5])
            out[f"pd{n}_{kind}_x"] = x
    p = [a.copy() for a in W.pd_dominant(3, 32, seed=30)]
    p[2][0, 0] = 0.0                                          # zero at row 0
    p[0][1, 7] = 0.0; p[1][1, 8] = 0.0; p[2][1, 9] = 0.0      # decoupled row 9
    p[1][2, 0] = p[2][2, 1] * p[2][2, 0] / p[3][2, 0]         # near-singular 2x2 lead (row 1)
    out.update({f"pdz_{k}": v for k, v in zip(("sub2", "sub1", "main", "sup1", "sup2", "rhs"), p)})
    for kind in ("npdm", "mnpdm"):
        x, r, o, st, ix = _run_direct(kind, p[:5], p[5])
        out.update({f"pdz_{kind}_x": x, f"pdz_{kind}_status": st, f"pdz_{kind}_index": ix})
    _save("direct", **out)


def golden_iterative():
    out = {}
    cases = {
        # ladder twin of config 4 (m = 2 five-point), reference-representable
        "ladder": W.five_point(4, 512, 2, seed=3),
        # full-band DD pentadiagonal: ILU(0) == LU, k = 1
        "full": W.pd_dominant(2, 256, seed=1),
    }
    q = [a.copy() for a in W.pd_dominant(3, 200, seed=5)]
    rng = np.random.default_rng(55)
    q[1][rng.random(q[1].shape) < 0.3] = 0.0                   # 30% zero +-1 entries
    q[3][rng.random(q[3].shape) < 0.3] = 0.0
    cases["holes"] = tuple(q)
    for tag, p in cases.items():
        out.update({f"{tag}_{k}": v for k, v in zip(("sub2", "sub1", "main", "sup1", "sup2", "rhs"), p)})
        bsz, n = p[5].shape
        tol = W.sip_tolerance(p[5])
        keys = ("l_sub1", "l_sub2", "u_main", "u_sup1", "u_sup2")
        fac = {k: np.zeros((bsz, len(getattr_len(k, n)))) for k in keys}
        kdiag = {k: np.zeros((bsz, L)) for k, L in zip(("k_sub2", "k_sub1", "k_main", "k_sup1", "k_sup2"),
                                                     (n - 2, n - 1, n, n - 1, n - 2))}
        xs = np.zeros((bsz, n)); its = np.zeros(bsz, np.int64); res = np.zeros(bsz)
        hist = np.full((bsz, 600), np.nan)
        t0 = time.time()
        for s in range(bsz):
            a = core.PentaMatrix.from_diagonals(*[d[s] for d in p[:5]])
            f = iterative.ilu0_penta(a)
            for k in keys:
                fac[k][s] = np.asarray(getattr(f, k))
            km = iterative.defect_matrix(f, a).matrix
            for k, dg in zip(kdiag, km.diagonals()):
                kdiag[k][s] = np.asarray(dg)
            rep = iterative.sip_solve(a, p[5][s], iterative.SipConfig(tolerance=float(tol[s]),
                                                                      max_iterations=500),
                                      record_history=True)
            xs[s] = rep.x; its[s] = rep.iterations; res[s] = rep.residual_inf
            for kk, rr in rep.history:
                hist[s, kk - 1] = rr
        print(f"{tag}: sip k={its.tolist()} ({time.time()-t0:.1f}s)")
        out.update({f"{tag}_{k}": v for k, v in fac.items()})
        out.update({f"{tag}_{k}": v for k, v in kdiag.items()})
        out.update({f"{tag}_tol": tol, f"{tag}_x": xs, f"{tag}_k": its, f"{tag}_res": res,
                    f"{tag}_hist": hist})
    # MaxIterationsExceeded: ladder with a 2-iteration budget -> best iterate
    p = cases["ladder"]
    a = core.PentaMatrix.from_diagonals(*[d[0] for d in p[:5]])
    try:
        iterative.sip_solve(a, p[5][0], iterative.SipConfig(tolerance=1e-14, max_iterations=2))
        raise AssertionError("expected MaxIterationsExceeded")
    except MaxIterationsExceeded as e:
        out.update(maxit_best=np.asarray(e.best), maxit_res=np.float64(e.residual_inf),
                   maxit_k=np.int64(e.iterations))
    _save("iterative", **out)


def getattr_len(key, n):
    return range({"l_sub1": n - 1, "l_sub2": n - 2, "u_main": n, "u_sup1": n - 1, "u_sup2": n - 2}[key])


def golden_inverse():
    out = {}
    p = W.five_point(2, 256, 2, seed=3)
    out.update({f"hb_{k}": v for k, v in zip(("sub2", "sub1", "main", "sup1", "sup2", "rhs"), p)})
    tol = W.sip_tolerance(p[5])
    bsz, n = p[5].shape
    xs = np.zeros((bsz, n)); its = np.zeros(bsz, np.int64); res = np.zeros(bsz)
    li = np.zeros(bsz, np.int64); ui = np.zeros(bsz, np.int64)
    ops = np.zeros((bsz, 4), np.int64)   # SolveReport.ops (adds, subs, muls, divs)
    for s in range(bsz):
        a = core.PentaMatrix.from_diagonals(*[d[s] for d in p[:5]])
        rep = inverse.sip_hb_solve(a, p[5][s], iterative.SipConfig(tolerance=float(tol[s]),
                                                                   max_iterations=500))
        xs[s] = rep.x; its[s] = rep.iterations; res[s] = rep.residual_inf
        ops[s] = (rep.ops.adds, rep.ops.subs, rep.ops.muls, rep.ops.divs)
        f = iterative.ilu0_penta(a)
        li[s] = inverse.hb_invert_dense(inverse.dense_lower_factor(f), float(tol[s])).iterations
        ui[s] = inverse.hb_invert_dense(inverse.dense_upper_factor(f), float(tol[s])).iterations
    out.update(hb_tol=tol, hb_x=xs, hb_k=its, hb_res=res, hb_linv_iters=li, hb_uinv_iters=ui, hb_ops=ops)
    # [[1,0],[3,1]] inverts in one iteration
    r = inverse.hb_invert_dense(np.array([[1.0, 0.0], [3.0, 1.0]]))
    out.update(hb_spec_iters=np.int64(r.iterations), hb_spec_inv=np.asarray(r.inverse))
    _save("inverse", **out)


def _banded_report(fn):
    """(diags, iterations, residual, history, status) of hb_invert_banded;
    Stagnated / MaxIterationsExceeded carry the best approximation."""
    from bandix.errors import Stagnated
    try:
        r = fn()
        return r.inverse.diags, r.iterations, r.residual_inf, r.residual_history, 0
    except Stagnated as e:
        r = e.report
        return r.inverse.diags, r.iterations, r.residual_inf, r.residual_history, 9
    except MaxIterationsExceeded as e:
        return e.best.diags, e.iterations, e.residual_inf, (), 3


def golden_hbband():
    """Banded HB (inverse.py:122-195, the paper's array implementation) on the
    ILU(0) factors of m = 2 ladder systems, and sip_hb_solve(mode="banded")
    with explicit widths and in the reference's auto mode."""
    out = {}
    p = W.five_point(2, 128, 2, seed=3)
    out.update({f"hbb_{k}": v for k, v in zip(("sub2", "sub1", "main", "sup1", "sup2", "rhs"), p)})
    tol = W.sip_tolerance(p[5])
    out.update(hbb_tol=tol)
    bsz, n = p[5].shape
    for s in range(bsz):
        a = core.PentaMatrix.from_diagonals(*[d[s] for d in p[:5]])
        f = iterative.ilu0_penta(a)
        for side in ("lower", "upper"):
            for w in (2, 3, 6):
                for tl in (1e-12, float(tol[s])):
                    key = f"inv_{s}_{side}_{w}_{'t' if tl != 1e-12 else 'd'}"
                    d, it, r, h, st = _banded_report(
                        lambda: inverse.hb_invert_banded(f, side, w, tl, 200))
                    dd = np.full((w + 1, n), np.nan)
                    for j, v in enumerate(d):
                        dd[j, :len(v)] = v
                    out.update({key + "_x": dd, key + "_it": np.int64(it), key + "_res": np.float64(r),
                                key + "_hist": np.asarray(h, dtype=np.float64), key + "_st": np.int32(st)})
        for w in (3, 6, 12, 32, None):
            key = f"sip_{s}_{w if w else 'auto'}"
            cfg = iterative.SipConfig(tolerance=float(tol[s]), max_iterations=60)
            try:
                rep = inverse.sip_hb_solve(a, p[5][s], cfg, mode="banded", hb_bandwidth=w)
                out.update({key + "_x": np.asarray(rep.x), key + "_k": np.int64(rep.iterations),
                            key + "_res": np.float64(rep.residual_inf), key + "_st": np.int32(0),
                            key + "_ops": np.array([rep.ops.adds, rep.ops.subs, rep.ops.muls,
                                                    rep.ops.divs], np.int64)})
            except MaxIterationsExceeded as e:
                out.update({key + "_x": np.asarray(e.best), key + "_k": np.int64(e.iterations),
                            key + "_res": np.float64(e.residual_inf), key + "_st": np.int32(3)})
            print(key, int(out[key + "_st"]), int(out[key + "_k"]), float(out[key + "_res"]))
    _save("hbband", **out)


def golden_exact():
    """Small-N symbolic solves through the reference's exact solvers (float
    inputs converted losslessly with to_exact, exact.py:15-16)."""
    out = {}
    t0 = time.time()
    sub1, main, sup1, rhs, rows = W.td_symbolic(3, 40, seed=2, zeros=2)
    xs = np.zeros((3, 40)); subs = np.zeros(3, np.int64)
    for s in range(3):
        t = core.TriMatrix.from_diagonals(*[[core.to_exact(v) for v in d[s]] for d in (sub1, main, sup1)])
        r = exact.exact_solve_stdm(t, [core.to_exact(v) for v in rhs[s]])
        xs[s] = [float(v) for v in r.x]; subs[s] = r.pivot_substitutions
    out.update(stdm_sub1=sub1, stdm_main=main, stdm_sup1=sup1, stdm_rhs=rhs, stdm_rows=rows,
               stdm_x=xs, stdm_subs=subs)
    print(f"stdm {time.time()-t0:.1f}s subs={subs.tolist()}")
    t0 = time.time()
    p = W.pd_symbolic(2, 24, seed=2, zeros=2)
    xs = np.zeros((2, 24)); subs = np.zeros(2, np.int64)
    for s in range(2):
        a = core.PentaMatrix.from_diagonals(*[[core.to_exact(v) for v in d[s]] for d in p[:5]])
        r = exact.exact_solve_spdm(a, [core.to_exact(v) for v in p[5][s]])
        xs[s] = [float(v) for v in r.x]; subs[s] = r.pivot_substitutions
    out.update({f"spdm_{k}": v for k, v in zip(("sub2", "sub1", "main", "sup1", "sup2", "rhs", "rows"), p)})
    out.update(spdm_x=xs, spdm_subs=subs)
    print(f"spdm {time.time()-t0:.1f}s subs={subs.tolist()}")
    # no-zero-pivot exact solves agree with float solves to rounding
    q = W.td_symbolic(2, 64, seed=7, zeros=0)
    xs = np.zeros((2, 64)); subs = np.zeros(2, np.int64)
    for s in range(2):
        t = core.TriMatrix.from_diagonals(*[[core.to_exact(v) for v in d[s]] for d in q[:3]])
        r = exact.exact_solve_stdm(t, [core.to_exact(v) for v in q[3][s]])
        xs[s] = [float(v) for v in r.x]; subs[s] = r.pivot_substitutions
    out.update(stdm0_sub1=q[0], stdm0_main=q[1], stdm0_sup1=q[2], stdm0_rhs=q[3], stdm0_x=xs,
               stdm0_subs=subs)
    # exact determinant zero gate on a singular 3x3 (rows 0 and 1 equal)
    F = Fraction
    t = core.TriMatrix.from_diagonals([F(1), F(1)], [F(1), F(1), F(1)], [F(1), F(0)])
    out.update(det_singular=np.float64(float(exact.exact_det_band(t))))
    _save("exact", **out)


def golden_exact2():
    """More reference-exact symbolic solves (round 2: the verdict found the
    first set thin): wider spread of sizes, zero counts and seeds.  Sized so
    that the exact solvers finish in minutes (RatFunc gcd cost grows fast)."""
    out = {}
    cases = [("td_a", "td", 10, 48, 3, 11), ("td_b", "td", 6, 72, 2, 12), ("td_c", "td", 4, 32, 5, 13),
             ("pd_a", "pd", 6, 28, 2, 21), ("pd_b", "pd", 3, 40, 2, 22), ("pd_c", "pd", 3, 32, 3, 23)]
    for tag, kind, bsz, n, zeros, seed in cases:
        t0 = time.time()
        if kind == "td":
            *d, rows = W.td_symbolic(bsz, n, seed=seed, zeros=zeros)
            nd = 3
        else:
            *d, rows = W.pd_symbolic(bsz, n, seed=seed, zeros=zeros)
            nd = 5
        xs = np.zeros((bsz, n)); subs = np.zeros(bsz, np.int64)
        for s in range(bsz):
            diags = [[core.to_exact(v) for v in q[s]] for q in d[:nd]]
            rhs = [core.to_exact(v) for v in d[nd][s]]
            if kind == "td":
                r = exact.exact_solve_stdm(core.TriMatrix.from_diagonals(*diags), rhs)
            else:
                r = exact.exact_solve_spdm(core.PentaMatrix.from_diagonals(*diags), rhs)
            xs[s] = [float(v) for v in r.x]; subs[s] = r.pivot_substitutions
        for j, q in enumerate(d[:nd + 1]):
            out[f"{tag}_in{j}"] = q
        out.update({f"{tag}_rows": rows, f"{tag}_x": xs, f"{tag}_subs": subs})
        print(f"{tag}: {bsz} x N={n}, {zeros} zeros, {time.time()-t0:.1f}s subs={subs.tolist()}", flush=True)
    _save("exact2", **out)


def _frexp_fraction(v):
    e = v.numerator.bit_length() - v.denominator.bit_length() if v != 0 else 0
    if v == 0:
        return 0.0, 0
    if abs(v) >= Fraction(2) ** e:
        e += 1
    if abs(v) < Fraction(2) ** (e - 1):
        e -= 1
    return float(v / Fraction(2) ** e), e


def golden_det():
    """exact_det_band (exact.py:254-275) through the reference on small seeded
    systems (with and without substituted zero pivots, and singular ones);
    the exact rational det is stored as (mantissa, exponent), det = m * 2**e."""
    out = {}
    t0 = time.time()
    cases = {
        "tds": W.td_symbolic(3, 40, seed=2, zeros=2)[:3],          # 2 zero pivots each
        "td0": W.td_symbolic(3, 200, seed=5, zeros=0)[:3],          # non-dominant, no zeros
        "tdd": W.td_dominant(3, 300, seed=6)[:3],                   # dominant
        "pds": W.pd_symbolic(2, 24, seed=2, zeros=2)[:5],
        "pd0": W.pd_symbolic(2, 120, seed=5, zeros=0)[:5],
        "pdd": W.pd_dominant(2, 160, seed=6)[:5],
    }
    for name, diags in cases.items():
        bsz = diags[0].shape[0]
        mant = np.zeros(bsz); expo = np.zeros(bsz, np.int64); ops = np.zeros(bsz, np.int64)
        for s in range(bsz):
            cols = [[core.to_exact(v) for v in d[s]] for d in diags]
            a = (core.TriMatrix if len(diags) == 3 else core.PentaMatrix).from_diagonals(*cols)
            box = core.CounterBox()
            det = exact.exact_det_band(a, box)
            mant[s], expo[s] = _frexp_fraction(det)
            ops[s] = box.counter.total
        out.update({f"{name}_d{k}": d for k, d in enumerate(diags)})
        out.update({f"{name}_mant": mant, f"{name}_expo": expo, f"{name}_ops": ops})
        print(f"det {name} {time.time()-t0:.1f}s")
    # singular: a zero determinant with a substituted pivot (rows 0, 1 equal)
    F = Fraction
    t = core.TriMatrix.from_diagonals([F(1), F(1)], [F(1), F(1), F(1)], [F(1), F(0)])
    out.update(sing_d0=np.array([1.0, 1.0]), sing_d1=np.array([1.0, 1.0, 1.0]),
               sing_d2=np.array([1.0, 0.0]),
               sing_mant=np.float64(_frexp_fraction(exact.exact_det_band(t))[0]))
    _save("det", **out)


def _run_pd2td(p):
    """Reference pd_to_td + solve_pd2td_ntdm per system (direct.py:116-177)."""
    sub2, sub1, main, sup1, sup2, rhs = p
    bsz, n = rhs.shape
    red = {k: np.full(shape, np.nan) for k, shape in
           (("td", (bsz, n - 1)), ("te", (bsz, n)), ("tf", (bsz, n - 1)), ("tr", (bsz, n)))}
    ops = np.zeros((bsz, 3), dtype=np.int64)       # muls, subs, divs of the reduction
    x = np.full((bsz, n), np.nan)
    res = np.full(bsz, np.nan)
    tot = np.zeros(bsz, dtype=np.int64)            # solve report ops.total
    status = np.zeros(bsz, dtype=np.int32)
    index = np.full(bsz, -1, dtype=np.int32)
    for s in range(bsz):
        a = core.PentaMatrix.from_diagonals(sub2[s], sub1[s], main[s], sup1[s], sup2[s])
        try:
            t, r, c = direct.pd_to_td(a, rhs[s])
            red["td"][s], red["te"][s], red["tf"][s] = t.sub1, t.main, t.sup1
            red["tr"][s] = r
            ops[s] = (c.muls, c.subs, c.divs)
        except ReductionPivotZero as e:
            status[s], index[s] = 8, e.index
            continue
        try:
            rep = direct.solve_pd2td_ntdm(a, rhs[s])
            x[s], res[s], tot[s] = rep.x, rep.residual_inf, rep.ops.total
        except ZeroPivot as zp:
            status[s], index[s] = 1, zp.index
    return red, ops, x, res, tot, status, index


def golden_pd2td():
    out = {}
    keys = ("sub2", "sub1", "main", "sup1", "sup2", "rhs")
    cases = {
        "dense": W.pd_dominant(6, 96, seed=41),
        "sparse": W.pd_dominant(6, 96, seed=42, sparse_outer=True),
        "n3": W.pd_dominant(3, 3, seed=43),
        "n4": W.pd_dominant(3, 4, seed=44),
        "n5": W.pd_dominant(3, 5, seed=45, sparse_outer=True),
    }
    # failure cases on one batch of order 24:
    #   s0: ReductionPivotZero in pass 1 (sub2 of row 2 with sub1 of row 1 zero)
    #   s1: ReductionPivotZero in pass 2 (sup2 of row n-3 with sup1 of row n-2 zero)
    #   s2: reduction fine, Thomas hits ZeroPivot(0) (main[0] = 0, no sub2/sup2 at row 0/2)
    #   s3: holes: half the outer entries exactly zero (skipped eliminations)
    f = [a.copy() for a in W.pd_dominant(4, 24, seed=46)]
    n = 24
    f[1][0, 0] = 0.0                        # A[1,0] = 0, A[2,0] = sub2[0] != 0
    f[3][1, n - 2] = 0.0                    # A[n-2, n-1] = 0
    f[0][1, n - 4] = 0.0                    # keep pass 1 from touching row n-2's sup1
    f[2][2, 0] = 0.0; f[0][2, 0] = 0.0; f[4][2, 0] = 0.0
    rng = np.random.default_rng(47)
    for k in (0, 4):
        f[k][3, rng.random(n - 2) < 0.5] = 0.0
    cases["fail"] = tuple(f)
    for tag, p in cases.items():
        red, ops, x, res, tot, st, ix = _run_pd2td(p)
        out.update({f"{tag}_{k}": v for k, v in zip(keys, p)})
        out.update({f"{tag}_{k}": v for k, v in red.items()})
        out.update({f"{tag}_ops": ops, f"{tag}_x": x, f"{tag}_res": res, f"{tag}_tot": tot,
                    f"{tag}_status": st, f"{tag}_index": ix})
        print(tag, "status", st.tolist(), "index", ix.tolist())
    _save("pd2td", **out)


MATRIXIO_TEXTS = [
    "tri 3\n-1 -1\n2 2 2\n-1 -1\nrhs 1 0 1\n",
    "penta 5\n1 2 3\n4 5 6 7\n10 11 12 13 14\n1/2 -3/4 5 6\n7 8 9\n",
    "penta 4 # header\n0.5 1\n1 2 3\n4 5 6 7\n1 1 1\n2e-3 -1\nrhs 1 2\n 3 4\n",
    "tri 2\n1\n2 3\n4\n",
    "tri 3\n1 2\n3 4 5\n6 7\nrhs 1 2 3 4\n",
    "quad 3\n1\n",
    "penta 2\n1\n",
    "tri 3\n1 2\n3 x 5\n6 7\n",
    "tri 3\n1 2\n3 4 5\n6\n",
    "tri three\n",
    "tri 3\n1/0 2\n3 4 5\n6 7\n",
    "tri 3\n1 2\n3 4 5\n6 7\nfoo 1 2 3\n",
    "# only a comment\n",
    "TRI 2\n+1\n-2 +3\n4\nrhs 1/3 2\n",
]


def golden_matrixio():
    """Reference parser/serializer outputs (matrixio.py) for hand texts -> JSON."""
    import json
    from bandix import matrixio as M
    from bandix.errors import InvalidInput

    def enc(v):
        return ["F", v.numerator, v.denominator] if isinstance(v, Fraction) else ["f", float(v).hex()]
    cases = []
    for t in MATRIXIO_TEXTS:
        try:
            m, rhs = M.parse_matrix_text(t)
            kind = "penta" if isinstance(m, core.PentaMatrix) else "tri"
            cases.append({"text": t, "kind": kind, "n": m.n, "exact": bool(m.exact),
                          "diags": [[enc(v) for v in d] for d in m.diagonals()],
                          "rhs": None if rhs is None else [enc(v) for v in rhs],
                          "serialized": M.serialize_matrix(m, rhs)})
        except InvalidInput as e:
            cases.append({"text": t, "error": type(e).__name__, "message": str(e)})
    path = os.path.join(HERE, "matrixio.json")
    with open(path, "w") as f:
        json.dump(cases, f, indent=1)
    print(f"wrote {path}")


if __name__ == "__main__":
    which = sys.argv[1:] or ["direct", "iterative", "inverse", "exact", "pd2td", "matrixio", "det", "hbband"]
    for w in which:
        globals()["golden_" + w]()
