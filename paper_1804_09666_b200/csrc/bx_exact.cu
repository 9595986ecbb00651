// Symbolic solvers STDM / SPDM in binary64: zero pivots carried as the
// indeterminate t and the solution evaluated in the limit t -> 0.
//
// Reference (exact.py, bandix 0.1.0): exact_solve_stdm (296-307) and
// exact_solve_spdm (278-293) run tri_factor_recip / penta_factor
// (_elim.py:30-62, 90-109) with the _Substituter policy (221-229): a pivot that
// is exactly zero is replaced by t, the elimination continues over rational
// functions of t, and every x_i is evaluated at t = 0 (lift_limit, 207-210);
// exact_det_band (254-275) first rejects matrices whose determinant (product of
// the same pivots at t -> 0) is zero.
//
// Realisation here, in two passes per system (one thread per system):
//
// 1. The symbolic pass runs the reference's pivot recurrence (tri_factor_recip
//    / penta_factor) with every quantity a truncated Laurent series in t
//    (binary64 coefficients, orders LO..HI) that carries the highest order
//    still known exactly ("top", propagated through every operation like
//    p-adic precision; exact Laurent polynomials such as constants, t and
//    exact zeros have top = EXACT).  A pivot is replaced by t exactly when it
//    is identically zero -- every coefficient 0.0 with exact knowledge, the
//    reference's is_zero on a rational function (core.py:31-33).  Pivot
//    coefficients below -sum(ord of the previous pivots) are clamped (leading
//    minors are polynomials in t).  This yields pivot_substitutions and the
//    determinant gate: det(A) = lim prod mu_i = 0 iff sum ord(mu_i) > 0.  A
//    pivot whose zero test cannot be decided inside the window reports
//    WINDOW_OVERFLOW rather than guessing.
// 2. The limit itself: for nonsingular A the substituted elimination is the LU
//    of A + t*D_S and lim_{t->0} x(t) = A^{-1} b (exact.py:1-14).  Carrying
//    the solution sweeps in t would need one more series order per
//    substitution downstream of it; instead the limit is evaluated directly
//    by banded Gaussian elimination with partial pivoting in binary64 (the
//    stable way to form A^{-1} b; it also meets the 1e-10 tolerance on the
//    non-diagonally-dominant config-3 matrices where unpivoted elimination
//    does not).
#include <math.h>

#include "bx_common.cuh"
#include "bx_kernels.h"

namespace bx {
namespace ex {

constexpr int LO = -3, HI = 10, NC = HI - LO + 1;
constexpr int EXACT = 1 << 20;

struct LS {
  double c[NC];  // c[k - LO] = coefficient of t^k
  int top;       // highest order known exactly (EXACT: an exact Laurent polynomial)
};

__device__ __forceinline__ LS ls_const(double v) {
  LS r;
#pragma unroll
  for (int k = 0; k < NC; ++k) r.c[k] = 0.0;
  r.c[-LO] = v;
  r.top = EXACT;
  return r;
}
__device__ __forceinline__ LS ls_t() {  // the indeterminate t
  LS r = ls_const(0.0);
  r.c[1 - LO] = 1.0;
  return r;
}
// bit k set: coefficient k nonzero (branch-free; the early-exit scans
// diverged and were ~14 % of the pivot pass)
__device__ __forceinline__ unsigned ls_nzmask(const LS &a) {
  unsigned m = 0;
#pragma unroll
  for (int k = 0; k < NC; ++k) m |= (a.c[k] != 0.0 ? 1u : 0u) << k;
  return m;
}
// order / degree from a precomputed ls_nzmask (one mask per series serves
// every test on it)
__device__ __forceinline__ int ls_ord(const LS &a, unsigned nz) {
  const int nb = min(a.top, HI) - LO + 1;  // coefficients below nb are known exactly
  const unsigned m = nb <= 0 ? 0u : nz & ((1u << nb) - 1u);
  return m ? __ffs(m) - 1 + LO : HI + 1;
}
__device__ __forceinline__ int ls_deg(unsigned nz) { return nz ? 31 - __clz(nz) + LO : LO - 1; }
// x[j] := x[j + s] / x[j - s] (0 outside), 0 <= s < 16, in registers: a
// runtime-indexed coefficient array would live in local memory
__device__ __forceinline__ void ls_shift_down(double (&x)[NC], int s) {
#pragma unroll
  for (int b = 1; b < NC; b <<= 1) {
    const bool on = s & b;
#pragma unroll
    for (int j = 0; j < NC; ++j) x[j] = on ? (j + b < NC ? x[j + b] : 0.0) : x[j];
  }
}
__device__ __forceinline__ void ls_shift_up(double (&x)[NC], int s) {
#pragma unroll
  for (int b = 1; b < NC; b <<= 1) {
    const bool on = s & b;
#pragma unroll
    for (int j = NC - 1; j >= 0; --j) x[j] = on ? (j - b >= 0 ? x[j - b] : 0.0) : x[j];
  }
}
__device__ __forceinline__ LS ls_scale(double s, const LS &a) {
  if (s == 0.0) return ls_const(0.0);  // exact zero
  LS r;
#pragma unroll
  for (int k = 0; k < NC; ++k) r.c[k] = s * a.c[k];
  r.top = a.top;
  return r;
}
__device__ __forceinline__ LS ls_sub(const LS &a, const LS &b) {
  LS r;
#pragma unroll
  for (int k = 0; k < NC; ++k) r.c[k] = a.c[k] - b.c[k];
  r.top = min(a.top, b.top);
  return r;
}
__device__ __forceinline__ LS ls_mul(const LS &a, const LS &b, bool *ovf) {
  const unsigned ma = ls_nzmask(a), mb = ls_nzmask(b);
  const int oa = ls_ord(a, ma), ob = ls_ord(b, mb);
  if ((oa > HI && a.top >= EXACT) || (ob > HI && b.top >= EXACT)) return ls_const(0.0);
  LS r;
#pragma unroll
  for (int k = 0; k < NC; ++k) r.c[k] = 0.0;
  if (oa + ob < LO) *ovf = true;
  // coefficients beyond top do not take part: zeroed once here instead of a
  // per-product test (fma(0, y, r) == r for the finite y of a series)
  double am[NC], bm[NC];
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    am[i] = i + LO <= a.top ? a.c[i] : 0.0;
    bm[i] = i + LO <= b.top ? b.c[i] : 0.0;
  }
#pragma unroll
  for (int i = 0; i < NC; ++i)
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      const int k = i + j + LO;
      if (k >= 0 && k < NC) r.c[k] = fma(am[i], bm[j], r.c[k]);
    }
  if (a.top >= EXACT && b.top >= EXACT)
    r.top = ls_deg(ma) + ls_deg(mb) <= HI ? EXACT : HI;
  else
    r.top = min(min(a.top + ob, b.top + oa), HI);
  return r;
}
// d[0..KM) of 1/b for bs[j] = coefficient j of b / t^ord(b), ib0 = 1/bs[0]
template <int KM>
__device__ __forceinline__ void ls_inv_coeffs(const double (&bs)[NC], double ib0, double (&d)[NC]) {
#pragma unroll
  for (int k = 0; k < KM; ++k) {
    double acc = 0.0;  // newest d last: one FMA + one multiply after d[k-1]
#pragma unroll
    for (int j = k; j >= 1; --j) acc = fma(bs[j], d[k - j], acc);
    d[k] = k == 0 ? ib0 : -acc * ib0;
  }
}
__device__ __forceinline__ LS ls_inv(const LS &b, unsigned nz, bool *ovf) {
  const int v = ls_ord(b, nz);
  if (v > HI) {  // not invertible inside the window
    *ovf = true;
    return ls_const(0.0);
  }
  LS r;
  if (-v < LO) *ovf = true;
  // v = 0 on every lane of the warp (the common case: only rows next to a
  // substituted pivot have a Laurent part) needs no runtime shifts
  const bool v0 = __all_sync(__activemask(), v == 0);
  double bs[NC];  // bs[j] = coefficient of t^(v+j), 0 beyond top / the window
  if (v0) {
#pragma unroll
    for (int j = 0; j < NC; ++j) bs[j] = j - LO < NC ? b.c[j - LO] : 0.0;
  } else {
#pragma unroll
    for (int j = 0; j < NC; ++j) bs[j] = b.c[j];
    ls_shift_down(bs, v - LO);
  }
#pragma unroll
  for (int j = 1; j < NC; ++j)
    if (v + j > b.top) bs[j] = 0.0;
  const double ib0 = 1.0 / bs[0];
  double d[NC];  // d[k] = coefficient of t^(k-v) of 1/b
  // r.c[m] = d[m + v + LO] (orders LO..HI of the inverse)
  if (v0) {  // orders 0..HI only: d[HI+1..] would fall outside the window
    ls_inv_coeffs<HI + 1>(bs, ib0, d);
#pragma unroll
    for (int m = 0; m < NC; ++m) r.c[m] = m + LO >= 0 ? d[m + LO] : 0.0;
  } else {
    ls_inv_coeffs<NC>(bs, ib0, d);
    const int sh = v + LO;
    ls_shift_down(d, sh > 0 ? sh : 0);
    ls_shift_up(d, sh < 0 ? -sh : 0);
#pragma unroll
    for (int k = 0; k < NC; ++k) r.c[k] = d[k];
  }
  if (b.top >= EXACT && ls_deg(nz) == v)
    r.top = EXACT;  // exact monomial: exact inverse
  else
    r.top = min(HI, b.top - 2 * v);
  return r;
}
__device__ __forceinline__ void ls_clamp_below(LS &a, int lo) {
#pragma unroll
  for (int k = 0; k < NC; ++k)
    if (k + LO < lo) a.c[k] = 0.0;
}
// identically zero?  +1: yes, 0: no, -1: undecidable inside the window
__device__ __forceinline__ int ls_zero(const LS &a, unsigned nz) {
  const int o = ls_ord(a, nz);
  if (o <= min(a.top, HI)) return 0;
  return (a.top >= EXACT || a.top >= HI) ? 1 : -1;
}

// leading coefficient of a (nonzero) series: the value of t^-ord * a at t = 0
__device__ __forceinline__ double ls_lead(const LS &a, unsigned nz) {
  const int o = ls_ord(a, nz);
  double r = 0.0;  // select chain, not a runtime index (local memory)
#pragma unroll
  for (int k = 0; k < NC; ++k) r = k + LO == o ? a.c[k] : r;
  return r;
}
// det accumulator: mantissa in [0.5, 1) (or 0) times 2^exponent, so that the
// product of n pivots neither overflows nor underflows
struct Det {
  double m = 1.0;
  int64_t e = 0;
  __device__ __forceinline__ void mul(double v) {
    int ex;
    m = frexp(m * v, &ex);
    e += ex;
  }
};

// ---- per-thread row staging: every pass walks one system's rows in order
// with a dependent chain per row, so each row's inputs are fetched DS rows
// ahead with cp.async into a shared-memory ring [DS][NV][32 threads] and
// read back after cp.async.wait_group (no global latency on the chain).
constexpr int DS = 8;
constexpr int NVMAX = 6;
struct Stage {
  double *sm;  // this block's ring: DS slots x NVMAX values x 32 threads
  int tid;
  __device__ __forceinline__ double *slot(int64_t row, int v) const {
    return sm + ((int)(row % DS) * NVMAX + v) * 32 + tid;
  }
  // value v of `row` from global address g (nullptr: the value is zero)
  __device__ __forceinline__ void put(int64_t row, int v, const double *g) const {
    double *d = slot(row, v);
    if (g)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(d)),
                   "l"(g)
                   : "memory");
    else
      *d = 0.0;
  }
  __device__ __forceinline__ void commit() const { asm volatile("cp.async.commit_group;" ::: "memory"); }
  __device__ __forceinline__ void wait() const {  // the oldest of DS-1 groups in flight landed
    asm volatile("cp.async.wait_group %0;" ::"n"(DS - 1) : "memory");
  }
  __device__ __forceinline__ void wait_next() const {  // ... and the row after it
    asm volatile("cp.async.wait_group %0;" ::"n"(DS - 2) : "memory");
  }
  __device__ __forceinline__ double get(int64_t row, int v) const { return *slot(row, v); }
};

// ---- pass 1: the reference pivot recurrence with t-substitution ----------
template <class Lay>
__device__ void tri_pivots(const double *dp, const double *ep, const double *fp, int64_t s,
                           int64_t n, Lay lay, int &nsub, int &ordsum, bool &ovf,
                           const Stage &sg, Det *det = nullptr) {
  auto stage = [&](int64_t i) {  // e_i, d_i, f_{i-1}
    if (i < n) {
      sg.put(i, 0, ep + lay(i, s));
      sg.put(i, 1, i >= 1 ? dp + lay(i, s) : nullptr);
      sg.put(i, 2, i >= 1 ? fp + lay(i - 1, s) : nullptr);
    }
    sg.commit();
  };
  for (int64_t i = 0; i < DS - 1; ++i) stage(i);
  LS rec = ls_const(0.0);
  for (int64_t i = 0; i < n; ++i) {
    stage(i + DS - 1);
    sg.wait();
    const double e = sg.get(i, 0);
    LS mu;
    if (i == 0) {
      mu = ls_const(e);
    } else {
      const LS l = ls_scale(sg.get(i, 1), rec);                        // l = d * rec (_elim.py:104)
      mu = ls_sub(ls_const(e), ls_scale(sg.get(i, 2), l));             // e - l f    (_elim.py:105)
    }
    ls_clamp_below(mu, -ordsum);
    unsigned nz = ls_nzmask(mu);
    const int z = ls_zero(mu, nz);
    if (z < 0) ovf = true;
    if (z > 0) { mu = ls_t(); nz = 1u << (1 - LO); ++nsub; }          // _Substituter
    ordsum += ls_ord(mu, nz);
    if (det) det->mul(ls_lead(mu, nz));                                // exact_det_band: prod mu
    rec = ls_inv(mu, nz, &ovf);                                        // rec = 1/mu
  }
}

template <class Lay>
__device__ void penta_pivots(const double *cp, const double *dp, const double *ep,
                             const double *fp, const double *gp, int64_t s, int64_t n, Lay lay,
                             int &nsub, int &ordsum, bool &ovf, const Stage &sg,
                             Det *det = nullptr) {
  auto stage = [&](int64_t i) {  // e, f, g, d, c of row i
    if (i < n) {
      sg.put(i, 0, ep + lay(i, s));
      sg.put(i, 1, i <= n - 2 ? fp + lay(i, s) : nullptr);
      sg.put(i, 2, i <= n - 3 ? gp + lay(i, s) : nullptr);
      sg.put(i, 3, i >= 1 ? dp + lay(i, s) : nullptr);
      sg.put(i, 4, i >= 2 ? cp + lay(i, s) : nullptr);
    }
    sg.commit();
  };
  for (int64_t i = 0; i < DS - 1; ++i) stage(i);
  // carried: 1/mu and phi of rows i-1, i-2; psi = g (scalar)
  LS r1 = ls_const(0.0), ph1 = ls_const(0.0);
  double ps1 = 0.0;
  // l2 = c_i / mu_{i-2}, l2 phi_{i-2} and e_i - psi_{i-2} l2 depend on rows
  // <= i-1 only: formed one row early (iteration i-1), off the mu_{i-1} -> mu_i
  // chain (same operations, same rounding)
  LS t1n = ls_const(0.0), m0n = ls_const(0.0);
  for (int64_t i = 0; i < n; ++i) {
    stage(i + DS - 1);
    sg.wait_next();
    const double e = sg.get(i, 0);
    const double f = sg.get(i, 1);
    const double g = sg.get(i, 2);
    const LS t1 = t1n, m0 = m0n;
    if (i >= 1 && i + 1 < n) {
      const LS l2n = ls_scale(sg.get(i + 1, 4), r1);                    // c / mu_{i-2}   (54)
      t1n = ls_mul(l2n, ph1, &ovf);                                     // l2 phi_{i-2}
      m0n = ls_sub(ls_const(sg.get(i + 1, 0)), ls_scale(ps1, l2n));    // e - psi l2     (56)
    }
    LS mu, ph;
    if (i == 0) {
      mu = ls_const(e);
      ph = ls_const(f);
    } else if (i == 1) {
      const LS l1 = ls_scale(sg.get(i, 3), r1);                        // d0 / mu0 (_elim.py:47)
      mu = ls_sub(ls_const(e), ls_mul(l1, ph1, &ovf));
      ph = ls_sub(ls_const(f), ls_scale(ps1, l1));
    } else {
      const LS l1 = ls_mul(ls_sub(ls_const(sg.get(i, 3)), t1), r1, &ovf);  // (d - l2 phi)/mu (55)
      mu = ls_sub(m0, ls_mul(l1, ph1, &ovf));                                     // (56)
      ph = i <= n - 2 ? ls_sub(ls_const(f), ls_scale(ps1, l1)) : ls_const(0.0);  // (60)
    }
    ls_clamp_below(mu, -ordsum);
    unsigned nz = ls_nzmask(mu);
    const int z = ls_zero(mu, nz);
    if (z < 0) ovf = true;
    if (z > 0) { mu = ls_t(); nz = 1u << (1 - LO); ++nsub; }
    ordsum += ls_ord(mu, nz);
    if (det) det->mul(ls_lead(mu, nz));
    r1 = ls_inv(mu, nz, &ovf);
    ph1 = ph;
    ps1 = g;
  }
}

// ---- pass 2: x = A^{-1} b by banded elimination with partial pivoting -------
// K = half bandwidth (1: TD, 2: PD).  Window of K+1 unreduced rows, each with
// the 2K+1 coefficients of columns k..k+2K (upper bandwidth grows to 2K with
// row interchanges) and its rhs; U rows + y go to the scratch for the back
// substitution.
template <int K, class Lay>
__device__ bool gbsv(const double *cp, const double *dp, const double *ep, const double *fp,
                     const double *gp, const double *bp, double *xp, double *ws, int64_t s,
                     int64_t batch, int64_t n, Lay lay, const Stage &sg) {
  constexpr int W = 2 * K + 1;
  double w[K + 1][W], rb[K + 1];
  // rows are fetched in increasing order, each staged DS-1 fetches ahead
  auto stage_row = [&](int64_t i) {  // coefficients at offsets -K..K, then the rhs
    if (i < n) {
      if (K == 2) {
        sg.put(i, 0, i >= 2 ? cp + lay(i, s) : nullptr);
        sg.put(i, 1, i >= 1 ? dp + lay(i, s) : nullptr);
        sg.put(i, 2, ep + lay(i, s));
        sg.put(i, 3, i <= n - 2 ? fp + lay(i, s) : nullptr);
        sg.put(i, 4, i <= n - 3 ? gp + lay(i, s) : nullptr);
      } else {
        sg.put(i, 0, i >= 1 ? dp + lay(i, s) : nullptr);
        sg.put(i, 1, ep + lay(i, s));
        sg.put(i, 2, i <= n - 2 ? fp + lay(i, s) : nullptr);
      }
      sg.put(i, W, bp + lay(i, s));
    }
    sg.commit();
  };
  for (int64_t i = 0; i < DS - 1; ++i) stage_row(i);
  auto load_row = [&](int64_t i, double *row, double &rhs, int64_t k) {
    // row i, columns k .. k+2K; entries at columns i-K .. i+K
    stage_row(i + DS - 1);
    sg.wait();
#pragma unroll
    for (int c = 0; c < W; ++c) row[c] = 0.0;
    rhs = 0.0;
    if (i >= n) return;
    const int sh = (int)(i - k);  // column i-K sits at offset sh - K
    double v[2 * K + 1];
#pragma unroll
    for (int o = 0; o < 2 * K + 1; ++o) v[o] = sg.get(i, o);
#pragma unroll
    for (int o = 0; o < 2 * K + 1; ++o) {
      const int c = sh - K + o;
      if (c >= 0 && c < W) row[c] = v[o];
    }
    rhs = sg.get(i, W);
  };
#pragma unroll
  for (int j = 0; j <= K; ++j) load_row(j, w[j], rb[j], 0);
  const int64_t plane = batch * n;
  for (int64_t k = 0; k < n; ++k) {
    // pivot among the window rows still inside the matrix
    int p = 0;
    double best = fabs(w[0][0]);
#pragma unroll
    for (int j = 1; j <= K; ++j)
      if (k + j < n && fabs(w[j][0]) > best) { best = fabs(w[j][0]); p = j; }
    if (best == 0.0) return false;
#pragma unroll
    for (int j = 1; j <= K; ++j)
      if (j == p) {
#pragma unroll
        for (int c = 0; c < W; ++c) { const double tmp = w[0][c]; w[0][c] = w[j][c]; w[j][c] = tmp; }
        const double tb = rb[0]; rb[0] = rb[j]; rb[j] = tb;
      }
    const double piv = w[0][0];
#pragma unroll
    for (int j = 1; j <= K; ++j) {
      const double mlt = w[j][0] / piv;
#pragma unroll
      for (int c = 1; c < W; ++c) w[j][c] = fma(-mlt, w[0][c], w[j][c]);
      rb[j] = fma(-mlt, rb[0], rb[j]);
    }
    // emit U row k (columns k..k+2K) and y_k
#pragma unroll
    for (int c = 0; c < W; ++c) ws[(int64_t)c * plane + k * batch + s] = w[0][c];
    ws[(int64_t)W * plane + k * batch + s] = rb[0];
    // shift: the window now starts at column k+1
#pragma unroll
    for (int j = 0; j < K; ++j) {
#pragma unroll
      for (int c = 0; c < W - 1; ++c) w[j][c] = w[j + 1][c + 1];
      w[j][W - 1] = 0.0;
      rb[j] = rb[j + 1];
    }
    load_row(k + 1 + K, w[K], rb[K], k + 1);
  }
  // back substitution x_k = (y_k - sum_c U[k][c] x_{k+c}) / U[k][0]; the U
  // rows + y are staged DS-1 rows ahead (descending) like the inputs
  asm volatile("cp.async.wait_all;" ::: "memory");
  auto stage_back = [&](int64_t k) {
    if (k >= 0)
#pragma unroll
      for (int c = 0; c <= W; ++c) sg.put(k, c, ws + (int64_t)c * plane + k * batch + s);
    sg.commit();
  };
  for (int64_t j = 0; j < DS - 1; ++j) stage_back(n - 1 - j);
  double xs[W];  // x_{k+1} .. x_{k+2K} (xs[1..2K])
#pragma unroll
  for (int c = 0; c < W; ++c) xs[c] = 0.0;
  for (int64_t k = n - 1; k >= 0; --k) {
    stage_back(k - (DS - 1));
    sg.wait();
    double acc = sg.get(k, W);
#pragma unroll
    for (int c = 1; c < W; ++c) acc = fma(-sg.get(k, c), xs[c], acc);
    const double xk = acc / sg.get(k, 0);
#pragma unroll
    for (int c = W - 1; c >= 2; --c) xs[c] = xs[c - 1];
    xs[1] = xk;
    xp[lay(k, s)] = xk;
  }
  return true;
}

// The pivot pass and the pivoted solve are independent until the status, so
// they run on two thread sets of one launch (even blocks: pass 1, odd blocks:
// pass 2 -- twice the warps, the passes overlap); exact_finish combines.
template <int K, class Lay>
__global__ void exact_kernel(const double *__restrict__ cp, const double *__restrict__ dp,
                             const double *__restrict__ ep, const double *__restrict__ fp,
                             const double *__restrict__ gp, const double *__restrict__ bp,
                             double *__restrict__ xp, int32_t *subs, int32_t *gate,
                             int32_t *solved, double *ws, int64_t batch, int64_t n, Lay lay) {
  extern __shared__ double stage_sm[];
  const Stage sg{stage_sm, (int)threadIdx.x};
  const int role = blockIdx.x & 1;
  const int64_t s = (int64_t)(blockIdx.x >> 1) * blockDim.x + threadIdx.x;
  if (s >= batch) return;
  if (role == 0) {
    int nsub = 0, ordsum = 0;
    bool ovf = false;
    if (K == 1) tri_pivots(dp, ep, fp, s, n, lay, nsub, ordsum, ovf, sg);
    else penta_pivots(cp, dp, ep, fp, gp, s, n, lay, nsub, ordsum, ovf, sg);
    asm volatile("cp.async.wait_all;" ::: "memory");
    if (subs) subs[s] = nsub;
    // WINDOW_OVERFLOW, or exact_det_band == 0 -> SingularMatrix (exact.py:287-288, 301-302)
    gate[s] = ovf ? BX_STATUS_WINDOW_OVERFLOW : ordsum > 0 ? BX_STATUS_SINGULAR : BX_STATUS_OK;
  } else {
    const bool ok = gbsv<K>(cp, dp, ep, fp, gp, bp, xp, ws, s, batch, n, lay, sg);
    solved[s] = ok ? BX_STATUS_OK : BX_STATUS_SINGULAR;
  }
}

template <class Lay>
__global__ void exact_finish(const int32_t *gate, const int32_t *solved, double *xp,
                             int32_t *status, int32_t *index, int64_t batch, int64_t n, Lay lay) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= batch) return;
  const int32_t g = gate[s];
  set_status(status, index, s, g != BX_STATUS_OK ? g : solved[s], -1);
  if (g != BX_STATUS_OK) {
    const double nan = __longlong_as_double(0x7ff8000000000000LL);
    for (int64_t i = 0; i < n; ++i) xp[lay(i, s)] = nan;
  }
}

// exact_det_band (exact.py:254-275): det(A) = lim_{t->0} prod mu_i(t).  The
// leading minors are polynomials in t, so sum ord(mu_i) >= 0; the limit is 0
// when it is > 0 and the product of the leading coefficients when it is 0.
template <int K, class Lay>
__global__ void det_kernel(const double *__restrict__ cp, const double *__restrict__ dp,
                           const double *__restrict__ ep, const double *__restrict__ fp,
                           const double *__restrict__ gp, double *mant, int64_t *expo,
                           int32_t *status, int32_t *index, int32_t *subs, int64_t batch,
                           int64_t n, Lay lay) {
  extern __shared__ double stage_sm[];
  const Stage sg{stage_sm, (int)threadIdx.x};
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= batch) return;
  int nsub = 0, ordsum = 0;
  bool ovf = false;
  Det det;
  if (K == 1) tri_pivots(dp, ep, fp, s, n, lay, nsub, ordsum, ovf, sg, &det);
  else penta_pivots(cp, dp, ep, fp, gp, s, n, lay, nsub, ordsum, ovf, sg, &det);
  asm volatile("cp.async.wait_all;" ::: "memory");
  if (subs) subs[s] = nsub;
  if (ovf) {
    mant[s] = __longlong_as_double(0x7ff8000000000000LL);
    expo[s] = 0;
    set_status(status, index, s, BX_STATUS_WINDOW_OVERFLOW, -1);
    return;
  }
  mant[s] = ordsum > 0 ? 0.0 : det.m;
  expo[s] = ordsum > 0 ? 0 : det.e;
  set_status(status, index, s, BX_STATUS_OK, -1);
}

}  // namespace ex

static constexpr size_t kStageBytes = sizeof(double) * ex::DS * ex::NVMAX * 32;

int det_band(int kind, const double *c, const double *d, const double *e, const double *f,
             const double *g, double *mant, int64_t *expo, int32_t *st, int32_t *ix,
             int32_t *subs, int64_t batch, int64_t n, int64_t ld, int layout,
             cudaStream_t stream) {
  const int threads = 32;
  const dim3 grid((unsigned)((batch + threads - 1) / threads));
  if (kind == 1) {
    if (layout == BX_LAYOUT_INTERLEAVED)
      ex::det_kernel<1><<<grid, threads, kStageBytes, stream>>>(c, d, e, f, g, mant, expo, st, ix, subs,
                                                     batch, n, Interleaved{ld});
    else
      ex::det_kernel<1><<<grid, threads, kStageBytes, stream>>>(c, d, e, f, g, mant, expo, st, ix, subs,
                                                     batch, n, SystemMajor{ld});
  } else {
    if (layout == BX_LAYOUT_INTERLEAVED)
      ex::det_kernel<2><<<grid, threads, kStageBytes, stream>>>(c, d, e, f, g, mant, expo, st, ix, subs,
                                                     batch, n, Interleaved{ld});
    else
      ex::det_kernel<2><<<grid, threads, kStageBytes, stream>>>(c, d, e, f, g, mant, expo, st, ix, subs,
                                                     batch, n, SystemMajor{ld});
  }
  return BX_OK;
}

size_t exact_workspace_bytes(int kind, int64_t batch, int64_t n) {
  const int planes = kind == 1 ? 4 : 6;  // U row (2K+1) + y
  // + the two per-system outcomes (pivot pass gate, pivoted solve)
  return sizeof(double) * (size_t)planes * (size_t)batch * (size_t)n + 2 * sizeof(int32_t) * (size_t)batch;
}

int exact_solve(int kind, const double *c, const double *d, const double *e, const double *f,
                const double *g, const double *b, double *x, int32_t *st, int32_t *ix,
                int32_t *subs, double *ws, int64_t batch, int64_t n, int64_t ld, int layout,
                cudaStream_t stream) {
  const int threads = 32;
  const unsigned nb = (unsigned)((batch + threads - 1) / threads);
  const dim3 grid(2 * nb);  // even blocks: pivot pass, odd blocks: pivoted solve
  const int planes = kind == 1 ? 4 : 6;
  int32_t *gate = reinterpret_cast<int32_t *>(ws + (size_t)planes * (size_t)batch * (size_t)n);
  int32_t *solved = gate + batch;
  auto go = [&](auto lay) {
    if (kind == 1)
      ex::exact_kernel<1><<<grid, threads, kStageBytes, stream>>>(c, d, e, f, g, b, x, subs, gate,
                                                                   solved, ws, batch, n, lay);
    else
      ex::exact_kernel<2><<<grid, threads, kStageBytes, stream>>>(c, d, e, f, g, b, x, subs, gate,
                                                                   solved, ws, batch, n, lay);
    ex::exact_finish<<<(unsigned)((batch + 255) / 256), 256, 0, stream>>>(gate, solved, x, st, ix,
                                                                          batch, n, lay);
  };
  if (layout == BX_LAYOUT_INTERLEAVED) go(Interleaved{ld});
  else go(SystemMajor{ld});
  return BX_OK;
}

}  // namespace bx
