"""Developer tool: pure-Python mirror of bx_exact.cu's truncated-Laurent
elimination, for debugging the window/precision logic on small cases."""
import sys

import numpy as np

LO, HI = -4, 4
NC = HI - LO + 1
EXACT = 1000   # "top" of a series that is an exact Laurent polynomial inside the window


class LS:
    def __init__(self, c=None, top=EXACT):
        self.c = np.zeros(NC) if c is None else np.array(c, dtype=float)
        self.top = top

    @staticmethod
    def const(v):
        r = LS(); r.c[-LO] = v; return r

    @staticmethod
    def t():
        r = LS(); r.c[1 - LO] = 1.0; return r

    def ord(self):
        for k in range(NC):
            if k + LO <= self.top and self.c[k] != 0.0:
                return k + LO
        return HI + 1

    def is_zero(self):
        return self.ord() > min(self.top, HI)

    def deg(self):
        for k in range(NC - 1, -1, -1):
            if self.c[k] != 0.0:
                return k + LO
        return LO - 1

    def scale(self, s):
        return LS(self.c * s, self.top)

    def sub(self, o):
        return LS(self.c - o.c, min(self.top, o.top))

    def mul(self, o, ovf):
        oa, ob = self.ord(), o.ord()
        r = LS()
        if oa > self.top or ob > o.top:
            return r
        if oa + ob < LO:
            ovf.append(("mul", oa, ob))
        for i in range(NC):
            for j in range(NC):
                k = i + j + LO
                if 0 <= k < NC and i + LO <= self.top and j + LO <= o.top:
                    r.c[k] += self.c[i] * o.c[j]
        if self.top >= EXACT and o.top >= EXACT:
            r.top = EXACT if self.deg() + o.deg() <= HI else HI
        else:
            r.top = min(self.top + ob, o.top + oa, HI)
        return r

    def inv(self, ovf):
        v = self.ord()
        r = LS()
        if v > min(self.top, HI):
            ovf.append(("inv0",))
            return LS(np.full(NC, np.nan))
        if -v < LO:
            ovf.append(("inv", v))
        b0 = self.c[v - LO]
        d = []
        for k in range(NC):
            acc = 0.0
            for j in range(1, k + 1):
                bi = v + j - LO
                bj = self.c[bi] if (0 <= bi < NC and v + j <= self.top) else 0.0
                acc += bj * d[k - j]
            d.append(1.0 / b0 if k == 0 else -acc / b0)
            o = k - v
            if LO <= o <= HI:
                r.c[o - LO] = d[k]
        if self.top >= EXACT and self.deg() == v:   # exact monomial: exact inverse
            r.top = EXACT
        else:
            r.top = min(HI, self.top - 2 * v)
        return r

    def clamp(self, lo):
        for k in range(NC):
            if k + LO < lo:
                self.c[k] = 0.0


def spdm(c, d, e, f, g, b, verbose=False):
    n = len(e)
    ovf = []
    nsub = 0; ordsum = 0
    MU, PH, Y = [], [], []
    for i in range(n):
        if i == 0:
            mu = LS.const(e[0]); ph = LS.const(f[0]); y = LS.const(b[0])
        elif i == 1:
            l1 = LS.const(d[1]).mul(MU[0].inv(ovf), ovf)
            mu = LS.const(e[1]).sub(l1.mul(PH[0], ovf))
            ph = LS.const(f[1]).sub(l1.scale(g[0]))
            y = LS.const(b[1]).sub(l1.mul(Y[0], ovf))
        else:
            l2 = MU[i - 2].inv(ovf).scale(c[i])
            l1 = LS.const(d[i]).sub(l2.mul(PH[i - 2], ovf)).mul(MU[i - 1].inv(ovf), ovf)
            mu = LS.const(e[i]).sub(l2.scale(g[i - 2])).sub(l1.mul(PH[i - 1], ovf))
            ph = LS.const(f[i]).sub(l1.scale(g[i - 1])) if i <= n - 2 else LS.const(0.0)
            y = LS.const(b[i]).sub(l1.mul(Y[i - 1], ovf)).sub(l2.mul(Y[i - 2], ovf))
        mu.clamp(-ordsum)
        if mu.is_zero():
            mu = LS.t(); nsub += 1
        ordsum += mu.ord()
        if verbose:
            print(i, "mu ord", mu.ord(), "top", mu.top, "ph top", ph.top, "y ord/top", y.ord(), y.top, ovf[-1:] )
        MU.append(mu); PH.append(ph); Y.append(y)
    x = [None] * n
    x1 = Y[n - 1].mul(MU[n - 1].inv(ovf), ovf); x1.clamp(0); x[n - 1] = x1
    x2 = x1
    x1 = Y[n - 2].sub(PH[n - 2].mul(x2, ovf)).mul(MU[n - 2].inv(ovf), ovf); x1.clamp(0); x[n - 2] = x1
    for i in range(n - 3, -1, -1):
        num = Y[i].sub(PH[i].mul(x1, ovf)).sub(x2.scale(g[i]))
        xi = num.mul(MU[i].inv(ovf), ovf); xi.clamp(0)
        if xi.top < 0:
            ovf.append(("xtop", i, xi.top))
        x[i] = xi; x2 = x1; x1 = xi
    return np.array([v.c[-LO] for v in x]), nsub, ordsum, ovf


if __name__ == "__main__":
    g = np.load("tests/golden/exact.npz")
    s = 0
    a = [g[f"spdm_{k}"][s] for k in ("sub2", "sub1", "main", "sup1", "sup2", "rhs")]
    n = len(a[2])
    c = np.zeros(n); c[2:] = a[0]
    d = np.zeros(n); d[1:] = a[1]
    f = np.zeros(n); f[:n - 1] = a[3]
    gg = np.zeros(n); gg[:n - 2] = a[4]
    x, nsub, ordsum, ovf = spdm(c, d, a[2], f, gg, a[5], verbose="-v" in sys.argv)
    print("rows", g["spdm_rows"][s], "subs", nsub, "ordsum", ordsum, "ovf", ovf[:5])
    print("err", np.max(np.abs(x - g["spdm_x"][s])) / np.max(np.abs(g["spdm_x"][s])))


def pivots_pd(c, d, e, f, g):
    """Symbolic pivot recurrence of penta_factor only (no y / x)."""
    n = len(e)
    ovf = []
    nsub = 0; ordsum = 0
    MU, PH = [], []
    for i in range(n):
        if i == 0:
            mu = LS.const(e[0]); ph = LS.const(f[0])
        elif i == 1:
            l1 = LS.const(d[1]).mul(MU[0].inv(ovf), ovf)
            mu = LS.const(e[1]).sub(l1.mul(PH[0], ovf))
            ph = LS.const(f[1]).sub(l1.scale(g[0]))
        else:
            l2 = MU[i - 2].inv(ovf).scale(c[i])
            l1 = LS.const(d[i]).sub(l2.mul(PH[i - 2], ovf)).mul(MU[i - 1].inv(ovf), ovf)
            mu = LS.const(e[i]).sub(l2.scale(g[i - 2])).sub(l1.mul(PH[i - 1], ovf))
            ph = LS.const(f[i]).sub(l1.scale(g[i - 1])) if i <= n - 2 else LS.const(0.0)
        mu.clamp(-ordsum)
        if mu.is_zero():
            if mu.top < EXACT and mu.top < HI:
                ovf.append(("undetermined", i))
            mu = LS.t(); nsub += 1
        ordsum += mu.ord()
        MU.append(mu); PH.append(ph)
    return nsub, ordsum, ovf, min(m.top for m in MU)
