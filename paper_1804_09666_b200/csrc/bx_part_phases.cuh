// Chunk phases shared by the partitioned direct solvers (bx_direct_part.cu:
// two-port tree; bx_direct_halo.cu: interface iteration).  Thread t of a CTA
// of T threads owns M consecutive rows of one system of half-bandwidth K;
// the per-row state (Q = 1 + 2K doubles) lives in shared memory as
// state[(q * M + j) * T + t] (thread-fastest: conflict-free).
//   down    Gaussian elimination of the chunk against its own normalised rows
//           with the coupling to the K unknowns left of it carried as a spike W
//   up      upward elimination carrying the right spike V, after which
//           x_j = d_j - W_j . L - V_j . R   (L / R: the K unknowns just outside)
//   port    the chunk's two-port (first / last K rows)
//   write_x phase 3 given L and R
// The arithmetic replaces _elim.py:30-122 (a different elimination order:
// results agree with the reference to rounding, not bitwise).
#pragma once
#include "bx_common.cuh"
#include "bx_twoport.cuh"

#ifndef BX_PART_LA_SP
#define BX_PART_LA_SP 1  // ... of the sparse-outer variant (2 spills under the 168-register cap: 0.497 vs 0.460 ms)
#endif
#ifndef BX_PART_LA
#define BX_PART_LA 1  // input groups in flight ahead of the elimination (measured: 1 > 2 > 3)
#endif
#ifndef BX_SP_REG_ENTRIES
#define BX_SP_REG_ENTRIES 2  // sparse outer entries of a thread held in registers (more: loads;
                             // 4 spill under the interface kernel's 168-register cap)
#endif
#ifndef BX_P3_UNROLL
#define BX_P3_UNROLL 2  // row groups of phase 3 unrolled together (measured: 2 >= 4 > 1)
#endif
#define BX_PRAGMA_(x) _Pragma(#x)
#define BX_UNROLL(n) BX_PRAGMA_(unroll n)
#ifndef BX_TR
#define BX_TR(slot) \
  do {              \
  } while (0)
#endif

namespace bx {
namespace part {

// +-2 diagonals held sparse (MNPDM's case): per system a row-sorted list of
// the rows where sub2 or sup2 is nonzero, k slots per system (row -1 pads)
struct Outer {
  const int32_t *rows;
  const double *sub2, *sup2;
  int64_t k;
};

// status word of a system the interface-iteration pass hands to the tree
// pass when there is no workspace for separate marks (sparse-outer entry)
constexpr int32_t kRetryMark = 0x7f;

template <int K, int M, int T, bool VEC, bool SP, class Lay>
struct Chunk {
  static constexpr int G = 4;
  static_assert(M % G == 0, "M must be a multiple of 4");

  // s: system, base: first row of this thread's chunk; bad: first zero /
  // non-finite chunk-local pivot (-1: none); nzc: rows with sub2 != 0
  //
  // TT ("top tracking"): the chunk's first K unknowns are carried along as
  // affine functions of L and the K newest unknowns,
  //     x_a = al_a - om_a . L - P_a x_{j+1} - Q_a x_{j+2}      (after row j),
  // advanced with every normalised row (substitute x_j:  al -= P y_j,
  // om -= P W_j, (P, Q) <- (Q - P p_j, -P q_j); started from x_a itself), so
  // that after the last row they are affine in (L, R): the chunk's two-port
  // comes out of the down sweep alone (no up sweep, no second pass over the
  // state) and phase 3 is a back-substitution from R (write_x_backsub).
  template <bool TT = false>
  static __device__ __forceinline__ void down(
      double *__restrict__ state, const int t, const int64_t s, const int64_t base, const int64_t n,
      const Lay lay, const double *__restrict__ c2p, const double *__restrict__ c1p,
      const double *__restrict__ ep, const double *__restrict__ f1p,
      const double *__restrict__ f2p, const double *__restrict__ bp, const Outer outer,
      int32_t &bad, int &nzc, TwoPort<K> *port = nullptr) {
    auto st = [&](int q, int j) -> double & { return state[(q * M + j) * T + t]; };
    double tal[K], tom[K][K], tP[K], tQ[K];
#pragma unroll
    for (int a = 0; a < K; ++a) {
      tal[a] = 0.0;
      tP[a] = a == 0 ? -1.0 : 0.0;
      tQ[a] = a == 1 ? -1.0 : 0.0;
#pragma unroll
      for (int k = 0; k < K; ++k) tom[a][k] = 0.0;
    }
  // ---------------- phase 1: downward elimination --------------------------
  // Gaussian elimination of the chunk against its own normalised rows:
  // x_{j-2} is eliminated with row j-2, then x_{j-1} with row j-1, and the
  // row is scaled by 1/mu (MUFU seed + Newton, rcp).  Stored (normalised):
  //   x_j + p x_{j+1} + q x_{j+2} + W.L = y
  // (measured: 20 FP64 ops/row beat the division-free variant's 37, whose
  // shorter dependent chain does not pay for its extra issue slots)
  bad = -1;
  nzc = 0;
  // carried rows j-1 (f1, g1, y1, W1) and j-2: p, q, y, W of the stored rows
  double f1 = 0, g1 = 0, y1 = 0, f2 = 0, g2 = 0, y2 = 0;
  double W1[K], W2[K];
#pragma unroll
  for (int k = 0; k < K; ++k) W1[k] = W2[k] = 0.0;
  if (K == 2) { W2[0] = -1.0; W1[K - 1] = -1.0; }
  else W1[0] = -1.0;
  // register ring of input groups, LA groups in flight ahead of the one being
  // eliminated; the g loop is fully unrolled so the ring slots are fixed
  // registers (a copy between loop iterations would wait for the load)
  // (sparse outer diagonals: four arrays per group instead of six -- a second
  // group of lookahead fits the same registers)
  constexpr int LA0 = (SP && K == 2) ? BX_PART_LA_SP : BX_PART_LA;
  constexpr int LA = LA0 < M / G ? LA0 : M / G - 1 > 0 ? M / G - 1 : 1;
  constexpr int RG = LA + 1;
  struct Grp {
    double a2[G], a1[G], e[G], c1[G], c2[G], b[G];
  } ring[RG];
  auto load_group = [&](int g, Grp &gr) {
    double(&A2)[G] = gr.a2;
    double(&A1)[G] = gr.a1;
    double(&E)[G] = gr.e;
    double(&C1)[G] = gr.c1;
    double(&C2)[G] = gr.c2;
    double(&Bv)[G] = gr.b;
    const int64_t i0 = base + g * G;
    if (VEC && i0 + G <= n) {
      if (K == 2 && !SP) ld4(c2p + lay(i0, s), A2);
      ld4(c1p + lay(i0, s), A1);
      ld4(ep + lay(i0, s), E);
      ld4(f1p + lay(i0, s), C1);
      if (K == 2 && !SP) ld4(f2p + lay(i0, s), C2);
      ld4(bp + lay(i0, s), Bv);
      // (slots outside the matrix are masked where the group is consumed:
      // touching the registers here would wait for the load)
    } else {
#pragma unroll
      for (int u = 0; u < G; ++u) {
        const int64_t i = i0 + u;
        const bool in = i < n;
        A2[u] = (K == 2 && !SP && in && i >= 2) ? ldg(c2p + lay(i, s)) : 0.0;
        A1[u] = (in && i >= 1) ? ldg(c1p + lay(i, s)) : 0.0;
        E[u] = in ? ldg(ep + lay(i, s)) : 1.0;  // padding rows: identity
        C1[u] = (in && i <= n - 2) ? ldg(f1p + lay(i, s)) : 0.0;
        C2[u] = (K == 2 && !SP && in && i <= n - 3) ? ldg(f2p + lay(i, s)) : 0.0;
        Bv[u] = in ? ldg(bp + lay(i, s)) : 0.0;
      }
    }
  };
  // sparse outer diagonals: the slice [ob, oe) of this system's sorted list
  // that falls in this thread's rows (empty for almost every thread); the
  // first 8 list rows are fetched with independent loads (one round trip)
  int ob = 0, oe = 0;
  auto outer_slice = [&]() {
    const int32_t *orow = outer.rows + s * outer.k;
    const int k = (int)outer.k;
    int32_t r8[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) r8[q] = q < k ? __ldg(orow + q) : -1;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      ob += (r8[q] >= 0 && r8[q] < base) ? 1 : 0;
      oe += (r8[q] >= 0 && r8[q] < base + M) ? 1 : 0;
    }
    if (k > 8 && oe == 8) {  // long lists: continue the walk
      ob = min(ob, 8);
      while (ob < k && orow[ob] >= 0 && orow[ob] < base) ++ob;
      oe = ob;
      while (oe < k && orow[oe] >= 0 && orow[oe] < base + M) ++oe;
    }
  };
  // this thread's first NE entries in registers (rows compared per row, no
  // memory access on the elimination chain); more fall back to loads
  constexpr int NE = BX_SP_REG_ENTRIES;
  int32_t er[NE];
  double es2[NE], ep2[NE];
#pragma unroll
  for (int q = 0; q < NE; ++q) { er[q] = -1; es2[q] = ep2[q] = 0.0; }
  auto outer_regs = [&]() {
#pragma unroll
    for (int q = 0; q < NE; ++q)
      if (ob + q < oe) {
        const int64_t o = s * outer.k + ob + q;
        er[q] = __ldg(outer.rows + o);
        es2[q] = __ldg(outer.sub2 + o);
        ep2[q] = __ldg(outer.sup2 + o);
      }
  };


  const bool first = base == 0;                             // rows 0, 1 of the system
  const int rend = (int)min(n - base, (int64_t)(M + 4));     // n - base, clamped
#pragma unroll
  for (int g = 0; g < LA && g < M / G; ++g) load_group(g, ring[g]);
  if (SP) {  // after the first input loads are in flight
    outer_slice();
    outer_regs();
  }
#pragma unroll
  for (int g = 0; g < M / G; ++g) {
    if (g + LA < M / G) load_group(g + LA, ring[(g + LA) % RG]);
    const Grp &cur = ring[g % RG];
#pragma unroll
    for (int u = 0; u < G; ++u) {
    const int j = g * G + u;
    const int64_t i = base + j;  // slots outside the matrix are never trusted:
    // chunk bases are multiples of M, so only rows j < 2 of the first chunk
    // can fall left of the matrix; the right edge is a 32-bit test on rend
    double a2 = (K != 2 || SP) ? 0.0 : cur.a2[u];
    double a1 = cur.a1[u];
    if (j < 2 && first) {
      a2 = 0.0;
      if (j < 1) a1 = 0.0;
    }
    const double e = cur.e[u];
    const double c1 = j > rend - 2 ? 0.0 : cur.c1[u];
    double c2 = (K != 2 || SP || j > rend - 3) ? 0.0 : cur.c2[u];
    if (SP) {  // branch-free for the register entries (the row loop stays one block)
#pragma unroll
      for (int q = 0; q < NE; ++q) {
        const bool h = er[q] == (int32_t)i;
        a2 = h ? (i < 2 ? 0.0 : es2[q]) : a2;
        c2 = h ? (i > n - 3 ? 0.0 : ep2[q]) : c2;
      }
    }
    if (SP && oe - ob > NE) {
      for (int q = ob + NE; q < oe; ++q)
        if (outer.rows[s * outer.k + q] == (int32_t)i) {
          a2 = i < 2 ? 0.0 : outer.sub2[s * outer.k + q];
          c2 = i > n - 3 ? 0.0 : outer.sup2[s * outer.k + q];
        }
    }
    const double b = cur.b[u];
    // reciprocal form on normalised carried rows (p, q, y, w); rows -2, -1
    // are the virtual rows x_{-2} - L_0 = 0, x_{-1} - L_{K-1} = 0
    double mu, c1p, yy, ww[K];
    if (K == 2) {
      nzc += (a2 != 0.0);
      const double t1 = fma(-a2, f2, a1);
      const double e2 = fma(-a2, g2, e);
      const double y2p = fma(-a2, y2, b);
      mu = fma(-t1, f1, e2);
      c1p = fma(-t1, g1, c1);
      yy = fma(-t1, y1, y2p);
#pragma unroll
      for (int k = 0; k < K; ++k) ww[k] = fma(-t1, W1[k], -a2 * W2[k]);
    } else {
      mu = fma(-a1, f1, e);
      c1p = c1;
      yy = fma(-a1, y1, b);
      ww[0] = -a1 * W1[0];
    }
    if (mu == 0.0 || !isfinite(mu)) {
      if (bad < 0) bad = (int32_t)(base + j);
      mu = 1.0;
    }
    const double r = rcp(mu);
    const double pn = c1p * r, qn = c2 * r, yn = yy * r;
    st(0, j) = pn;
    if (K == 2) st(1, j) = qn;
    st(K, j) = yn;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const double w = ww[k] * r;
      st(K + 1 + k, j) = w;
      W2[k] = W1[k];
      W1[k] = w;
    }
    if (TT) {
#pragma unroll
      for (int a = 0; a < K; ++a) {
        const double P = tP[a];
        tal[a] = fma(-P, yn, tal[a]);
#pragma unroll
        for (int k = 0; k < K; ++k) tom[a][k] = fma(-P, W1[k], tom[a][k]);  // W1 = this row's W
        tP[a] = K == 2 ? fma(-P, pn, tQ[a]) : -P * pn;
        tQ[a] = -P * qn;
      }
    }
    f2 = f1; g2 = g1; y2 = y1;
    f1 = pn; g1 = qn; y1 = yn;
    }
  }
  if (TT) {
    // F: x_a = al - om.L - (P, Q).R ; E: the last K normalised rows
#pragma unroll
    for (int a = 0; a < K; ++a) {
      port->F.g.v[a] = tal[a];
#pragma unroll
      for (int k = 0; k < K; ++k) port->F.A.m[a][k] = -tom[a][k];
      port->F.B.m[a][0] = -tP[a];
      if (K == 2) port->F.B.m[a][K - 1] = -tQ[a];
    }
    port->E = port_E_rows(f2, g2, y2, W2, f1, g1, y1, W1);
  }
  }

  // E side of a two-port from the chunk's last normalised rows M-2 (p2, q2, y2,
  // w2; K = 2 only) and M-1 (p1, q1, y1, w1):  x_{M-1} = y1 - w1.L - (p1, q1).R,
  // x_{M-2} = y2 - w2.L - p2 x_{M-1} - q2 R_0
  static __device__ __forceinline__ Port<K> port_E_rows(double p2, double q2, double y2,
                                                        const double *w2, double p1, double q1,
                                                        double y1, const double *w1) {
    Port<K> E;
    E.g.v[K - 1] = y1;
#pragma unroll
    for (int k = 0; k < K; ++k) E.A.m[K - 1][k] = -w1[k];
    E.B.m[K - 1][0] = -p1;
    if (K == 2) {
      E.B.m[K - 1][K - 1] = -q1;
      E.g.v[0] = fma(-p2, y1, y2);
#pragma unroll
      for (int k = 0; k < K; ++k) E.A.m[0][k] = -fma(-p2, w1[k], w2[k]);
      E.B.m[0][0] = -fma(-p2, p1, q2);
      E.B.m[0][K - 1] = p2 * q1;
    }
    return E;
  }
  // ... of chunk c, read from the state left by down<true> (any thread's rows)
  static __device__ __forceinline__ Port<K> port_E_state(const double *__restrict__ state,
                                                         const int c) {
    auto at = [&](int q, int j) -> double { return state[(q * M + j) * T + c]; };
    double w1[K], w2[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      w1[k] = at(K + 1 + k, M - 1);
      w2[k] = K == 2 ? at(K + 1 + k, M - 2) : 0.0;
    }
    return port_E_rows(K == 2 ? at(0, M - 2) : 0.0, K == 2 ? at(1, M - 2) : 0.0,
                       K == 2 ? at(K, M - 2) : 0.0, w2, at(0, M - 1), K == 2 ? at(1, M - 1) : 0.0,
                       at(K, M - 1), w1);
  }

  static __device__ __forceinline__ void up(double *__restrict__ state, const int t) {
    auto st = [&](int q, int j) -> double & { return state[(q * M + j) * T + t]; };
  // ---------------- phase 1b: upward elimination ---------------------------
  // x_j = d_j - W_j.L - V_j.R ; state slots after: 0:d, 1..K: W, K+1..2K: V
  {
    double d1 = 0, d2 = 0, Wu1[K], Wu2[K], V1[K], V2[K];
#pragma unroll
    for (int k = 0; k < K; ++k) Wu1[k] = Wu2[k] = V1[k] = V2[k] = 0.0;
#pragma unroll
    for (int j = M - 1; j >= 0; --j) {
      const double p = st(0, j);
      const double q = K == 2 ? st(1, j) : 0.0;
      const double y = st(K, j);
      double W[K];
#pragma unroll
      for (int k = 0; k < K; ++k) W[k] = st(K + 1 + k, j);
      double d, Wu[K], V[K];
      if (j == M - 1) {
        d = y;
#pragma unroll
        for (int k = 0; k < K; ++k) Wu[k] = W[k];
        V[0] = p;
        if (K == 2) V[1] = q;
      } else if (K == 2 && j == M - 2) {
        d = fma(-p, d1, y);
#pragma unroll
        for (int k = 0; k < K; ++k) Wu[k] = fma(-p, Wu1[k], W[k]);
        V[0] = fma(-p, V1[0], q);
        V[1] = -p * V1[1];
      } else {
        // row j+2 terms first: the row j+1 results (newest) enter last
        d = K == 2 ? fma(-p, d1, fma(-q, d2, y)) : fma(-p, d1, y);
#pragma unroll
        for (int k = 0; k < K; ++k) {
          Wu[k] = K == 2 ? fma(-p, Wu1[k], fma(-q, Wu2[k], W[k])) : fma(-p, Wu1[k], W[k]);
          V[k] = K == 2 ? fma(-p, V1[k], -q * V2[k]) : -p * V1[k];
        }
      }
      st(0, j) = d;
#pragma unroll
      for (int k = 0; k < K; ++k) { st(1 + k, j) = Wu[k]; st(1 + K + k, j) = V[k]; }
      d2 = d1; d1 = d;
#pragma unroll
      for (int k = 0; k < K; ++k) { Wu2[k] = Wu1[k]; Wu1[k] = Wu[k]; V2[k] = V1[k]; V1[k] = V[k]; }
    }
  }
  }

  // two-port of chunk c (any thread's rows): F from rows 0..K-1, E from M-K..M-1
  static __device__ __forceinline__ Port<K> port_side(const double *__restrict__ state, const int c,
                                                      const int j0) {
    Port<K> p;
#pragma unroll
    for (int a = 0; a < K; ++a) {
      p.g.v[a] = state[(0 * M + j0 + a) * T + c];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        p.A.m[a][k] = -state[((1 + k) * M + j0 + a) * T + c];
        p.B.m[a][k] = -state[((1 + K + k) * M + j0 + a) * T + c];
      }
    }
    return p;
  }
  static __device__ __forceinline__ TwoPort<K> port(const double *__restrict__ state, const int t) {
    TwoPort<K> p;
    p.F = port_side(state, t, 0);
    p.E = port_side(state, t, M - K);
    return p;
  }

  static __device__ __forceinline__ void write_x(const double *__restrict__ state, const int t,
                                                 const int64_t s, const int64_t base,
                                                 const int64_t n, const Lay lay,
                                                 double *__restrict__ xp, const Vec<K> &L,
                                                 const Vec<K> &R) {
    auto st = [&](int q, int j) -> double { return state[(q * M + j) * T + t]; };
  // ---------------- phase 3: x_j = d - W.L - V.R -----------------------------
BX_UNROLL(BX_P3_UNROLL)
  for (int g = 0; g < M / G; ++g) {
    double xv[G];
#pragma unroll
    for (int u = 0; u < G; ++u) {
      const int j = g * G + u;
      double v = st(0, j);
#pragma unroll
      for (int k = 0; k < K; ++k) v = fma(-st(1 + k, j), L.v[k], fma(-st(1 + K + k, j), R.v[k], v));
      xv[u] = v;
    }
    const int64_t i0 = base + g * G;
    if (VEC && i0 + G <= n) {
      st4(xp + lay(i0, s), xv);
    } else {
#pragma unroll
      for (int u = 0; u < G; ++u)
        if (i0 + u < n) xp[lay(i0 + u, s)] = xv[u];
    }
  }
  }

  // phase 3 after down<true>: back-substitution from R through the normalised
  // rows,  x_j = y_j - W_j.L - p_j x_{j+1} - q_j x_{j+2}  (newest unknown last)
  static __device__ __forceinline__ void write_x_backsub(const double *__restrict__ state,
                                                         const int t, const int64_t s,
                                                         const int64_t base, const int64_t n,
                                                         const Lay lay, double *__restrict__ xp,
                                                         const Vec<K> &L, const Vec<K> &R) {
    auto st = [&](int q, int j) -> double { return state[(q * M + j) * T + t]; };
    double X1 = R.v[0], X2 = K == 2 ? R.v[K - 1] : 0.0;
BX_UNROLL(BX_P3_UNROLL)
    for (int g = M / G - 1; g >= 0; --g) {
      double xv[G];
#pragma unroll
      for (int u = G - 1; u >= 0; --u) {
        const int j = g * G + u;
        double v = st(K, j);
#pragma unroll
        for (int k = 0; k < K; ++k) v = fma(-st(K + 1 + k, j), L.v[k], v);
        if (K == 2) v = fma(-st(1, j), X2, v);
        v = fma(-st(0, j), X1, v);
        xv[u] = v;
        X2 = X1;
        X1 = v;
      }
      const int64_t i0 = base + g * G;
      if (VEC && i0 + G <= n) {
        st4(xp + lay(i0, s), xv);
      } else {
#pragma unroll
        for (int u = 0; u < G; ++u)
          if (i0 + u < n) xp[lay(i0 + u, s)] = xv[u];
      }
    }
  }
};

}  // namespace part
}  // namespace bx
