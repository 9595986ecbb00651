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
__device__ __forceinline__ int ls_ord(const LS &a) {
  const int lim = min(a.top, HI);
#pragma unroll
  for (int k = 0; k < NC; ++k)
    if (k + LO <= lim && a.c[k] != 0.0) return k + LO;
  return HI + 1;
}
__device__ __forceinline__ int ls_deg(const LS &a) {
#pragma unroll
  for (int k = NC - 1; k >= 0; --k)
    if (a.c[k] != 0.0) return k + LO;
  return LO - 1;
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
  const int oa = ls_ord(a), ob = ls_ord(b);
  if ((oa > HI && a.top >= EXACT) || (ob > HI && b.top >= EXACT)) return ls_const(0.0);
  LS r;
#pragma unroll
  for (int k = 0; k < NC; ++k) r.c[k] = 0.0;
  if (oa + ob < LO) *ovf = true;
#pragma unroll
  for (int i = 0; i < NC; ++i)
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      const int k = i + j + LO;
      if (k >= 0 && k < NC && i + LO <= a.top && j + LO <= b.top) r.c[k] = fma(a.c[i], b.c[j], r.c[k]);
    }
  if (a.top >= EXACT && b.top >= EXACT)
    r.top = ls_deg(a) + ls_deg(b) <= HI ? EXACT : HI;
  else
    r.top = min(min(a.top + ob, b.top + oa), HI);
  return r;
}
__device__ __forceinline__ LS ls_inv(const LS &b, bool *ovf) {
  const int v = ls_ord(b);
  if (v > HI) {  // not invertible inside the window
    *ovf = true;
    return ls_const(0.0);
  }
  LS r;
#pragma unroll
  for (int k = 0; k < NC; ++k) r.c[k] = 0.0;
  if (-v < LO) *ovf = true;
  const double ib0 = 1.0 / b.c[v - LO];
  double d[NC];
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    double acc = 0.0;
#pragma unroll
    for (int j = 1; j <= k; ++j) {
      const int bi = v + j - LO;
      const double bj = (bi >= 0 && bi < NC && v + j <= b.top) ? b.c[bi] : 0.0;
      acc = fma(bj, d[k - j], acc);
    }
    d[k] = k == 0 ? ib0 : -acc * ib0;
    const int ord = k - v;
    if (ord >= LO && ord <= HI) r.c[ord - LO] = d[k];
  }
  if (b.top >= EXACT && ls_deg(b) == v)
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
__device__ __forceinline__ int ls_zero(const LS &a) {
  const int o = ls_ord(a);
  if (o <= min(a.top, HI)) return 0;
  return (a.top >= EXACT || a.top >= HI) ? 1 : -1;
}

// leading coefficient of a (nonzero) series: the value of t^-ord * a at t = 0
__device__ __forceinline__ double ls_lead(const LS &a) {
  const int o = ls_ord(a);
  return o <= HI ? a.c[o - LO] : 0.0;
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

// ---- pass 1: the reference pivot recurrence with t-substitution ----------
template <class Lay>
__device__ void tri_pivots(const double *dp, const double *ep, const double *fp, int64_t s,
                           int64_t n, Lay lay, int &nsub, int &ordsum, bool &ovf, Det *det = nullptr) {
  LS rec = ls_const(0.0);
  for (int64_t i = 0; i < n; ++i) {
    const double e = ldg(ep + lay(i, s));
    LS mu;
    if (i == 0) {
      mu = ls_const(e);
    } else {
      const LS l = ls_scale(ldg(dp + lay(i, s)), rec);                 // l = d * rec (_elim.py:104)
      mu = ls_sub(ls_const(e), ls_scale(ldg(fp + lay(i - 1, s)), l));  // e - l f    (_elim.py:105)
    }
    ls_clamp_below(mu, -ordsum);
    const int z = ls_zero(mu);
    if (z < 0) ovf = true;
    if (z > 0) { mu = ls_t(); ++nsub; }                                // _Substituter
    ordsum += ls_ord(mu);
    if (det) det->mul(ls_lead(mu));                                    // exact_det_band: prod mu
    rec = ls_inv(mu, &ovf);                                            // rec = 1/mu
  }
}

template <class Lay>
__device__ void penta_pivots(const double *cp, const double *dp, const double *ep,
                             const double *fp, const double *gp, int64_t s, int64_t n, Lay lay,
                             int &nsub, int &ordsum, bool &ovf, Det *det = nullptr) {
  // carried: 1/mu and phi of rows i-1, i-2; psi = g (scalar)
  LS r1 = ls_const(0.0), r2 = ls_const(0.0), ph1 = ls_const(0.0), ph2 = ls_const(0.0);
  double ps1 = 0.0, ps2 = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double e = ldg(ep + lay(i, s));
    const double f = i <= n - 2 ? ldg(fp + lay(i, s)) : 0.0;
    const double g = i <= n - 3 ? ldg(gp + lay(i, s)) : 0.0;
    LS mu, ph;
    if (i == 0) {
      mu = ls_const(e);
      ph = ls_const(f);
    } else if (i == 1) {
      const LS l1 = ls_scale(ldg(dp + lay(i, s)), r1);                 // d0 / mu0 (_elim.py:47)
      mu = ls_sub(ls_const(e), ls_mul(l1, ph1, &ovf));
      ph = ls_sub(ls_const(f), ls_scale(ps1, l1));
    } else {
      const LS l2 = ls_scale(ldg(cp + lay(i, s)), r2);                 // c / mu_{i-2}   (54)
      const LS l1 = ls_mul(ls_sub(ls_const(ldg(dp + lay(i, s))), ls_mul(l2, ph2, &ovf)), r1,
                           &ovf);                                       // (d - l2 phi)/mu (55)
      mu = ls_sub(ls_sub(ls_const(e), ls_scale(ps2, l2)), ls_mul(l1, ph1, &ovf));  // (56)
      ph = i <= n - 2 ? ls_sub(ls_const(f), ls_scale(ps1, l1)) : ls_const(0.0);  // (60)
    }
    ls_clamp_below(mu, -ordsum);
    const int z = ls_zero(mu);
    if (z < 0) ovf = true;
    if (z > 0) { mu = ls_t(); ++nsub; }
    ordsum += ls_ord(mu);
    if (det) det->mul(ls_lead(mu));
    r2 = r1;
    r1 = ls_inv(mu, &ovf);
    ph2 = ph1; ph1 = ph;
    ps2 = ps1; ps1 = g;
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
                     int64_t batch, int64_t n, Lay lay) {
  constexpr int W = 2 * K + 1;
  double w[K + 1][W], rb[K + 1];
  auto load_row = [&](int64_t i, double *row, double &rhs, int64_t k) {
    // row i, columns k .. k+2K; entries at columns i-K .. i+K
#pragma unroll
    for (int c = 0; c < W; ++c) row[c] = 0.0;
    rhs = 0.0;
    if (i >= n) return;
    const int sh = (int)(i - k);  // column i-K sits at offset sh - K
    double v[2 * K + 1];
    if (K == 2) {
      v[0] = i >= 2 ? ldg(cp + lay(i, s)) : 0.0;
      v[1] = i >= 1 ? ldg(dp + lay(i, s)) : 0.0;
      v[2] = ldg(ep + lay(i, s));
      v[3] = i <= n - 2 ? ldg(fp + lay(i, s)) : 0.0;
      v[4] = i <= n - 3 ? ldg(gp + lay(i, s)) : 0.0;
    } else {
      v[0] = i >= 1 ? ldg(dp + lay(i, s)) : 0.0;
      v[1] = ldg(ep + lay(i, s));
      v[2] = i <= n - 2 ? ldg(fp + lay(i, s)) : 0.0;
    }
#pragma unroll
    for (int o = 0; o < 2 * K + 1; ++o) {
      const int c = sh - K + o;
      if (c >= 0 && c < W) row[c] = v[o];
    }
    rhs = ldg(bp + lay(i, s));
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
  // back substitution x_k = (y_k - sum_c U[k][c] x_{k+c}) / U[k][0]
  double xs[W];  // x_{k+1} .. x_{k+2K} (xs[1..2K])
#pragma unroll
  for (int c = 0; c < W; ++c) xs[c] = 0.0;
  for (int64_t k = n - 1; k >= 0; --k) {
    double acc = ws[(int64_t)W * plane + k * batch + s];
#pragma unroll
    for (int c = 1; c < W; ++c) acc = fma(-ws[(int64_t)c * plane + k * batch + s], xs[c], acc);
    const double xk = acc / ws[k * batch + s];
#pragma unroll
    for (int c = W - 1; c >= 2; --c) xs[c] = xs[c - 1];
    xs[1] = xk;
    xp[lay(k, s)] = xk;
  }
  return true;
}

template <int K, class Lay>
__global__ void exact_kernel(const double *__restrict__ cp, const double *__restrict__ dp,
                             const double *__restrict__ ep, const double *__restrict__ fp,
                             const double *__restrict__ gp, const double *__restrict__ bp,
                             double *__restrict__ xp, int32_t *status, int32_t *index,
                             int32_t *subs, double *ws, int64_t batch, int64_t n, Lay lay) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= batch) return;
  int nsub = 0, ordsum = 0;
  bool ovf = false;
  if (K == 1) tri_pivots(dp, ep, fp, s, n, lay, nsub, ordsum, ovf);
  else penta_pivots(cp, dp, ep, fp, gp, s, n, lay, nsub, ordsum, ovf);
  if (subs) subs[s] = nsub;
  const double nan = __longlong_as_double(0x7ff8000000000000LL);
  if (ovf) {
    set_status(status, index, s, BX_STATUS_WINDOW_OVERFLOW, -1);
    for (int64_t i = 0; i < n; ++i) xp[lay(i, s)] = nan;
    return;
  }
  if (ordsum > 0) {  // exact_det_band == 0 -> SingularMatrix (exact.py:287-288, 301-302)
    set_status(status, index, s, BX_STATUS_SINGULAR, -1);
    for (int64_t i = 0; i < n; ++i) xp[lay(i, s)] = nan;
    return;
  }
  const bool ok = gbsv<K>(cp, dp, ep, fp, gp, bp, xp, ws, s, batch, n, lay);
  set_status(status, index, s, ok ? BX_STATUS_OK : BX_STATUS_SINGULAR, -1);
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
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= batch) return;
  int nsub = 0, ordsum = 0;
  bool ovf = false;
  Det det;
  if (K == 1) tri_pivots(dp, ep, fp, s, n, lay, nsub, ordsum, ovf, &det);
  else penta_pivots(cp, dp, ep, fp, gp, s, n, lay, nsub, ordsum, ovf, &det);
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

int det_band(int kind, const double *c, const double *d, const double *e, const double *f,
             const double *g, double *mant, int64_t *expo, int32_t *st, int32_t *ix,
             int32_t *subs, int64_t batch, int64_t n, int64_t ld, int layout,
             cudaStream_t stream) {
  const int threads = 32;
  const dim3 grid((unsigned)((batch + threads - 1) / threads));
  if (kind == 1) {
    if (layout == BX_LAYOUT_INTERLEAVED)
      ex::det_kernel<1><<<grid, threads, 0, stream>>>(c, d, e, f, g, mant, expo, st, ix, subs,
                                                     batch, n, Interleaved{ld});
    else
      ex::det_kernel<1><<<grid, threads, 0, stream>>>(c, d, e, f, g, mant, expo, st, ix, subs,
                                                     batch, n, SystemMajor{ld});
  } else {
    if (layout == BX_LAYOUT_INTERLEAVED)
      ex::det_kernel<2><<<grid, threads, 0, stream>>>(c, d, e, f, g, mant, expo, st, ix, subs,
                                                     batch, n, Interleaved{ld});
    else
      ex::det_kernel<2><<<grid, threads, 0, stream>>>(c, d, e, f, g, mant, expo, st, ix, subs,
                                                     batch, n, SystemMajor{ld});
  }
  return BX_OK;
}

size_t exact_workspace_bytes(int kind, int64_t batch, int64_t n) {
  const int planes = kind == 1 ? 4 : 6;  // U row (2K+1) + y
  return sizeof(double) * (size_t)planes * (size_t)batch * (size_t)n;
}

int exact_solve(int kind, const double *c, const double *d, const double *e, const double *f,
                const double *g, const double *b, double *x, int32_t *st, int32_t *ix,
                int32_t *subs, double *ws, int64_t batch, int64_t n, int64_t ld, int layout,
                cudaStream_t stream) {
  const int threads = 32;
  const dim3 grid((unsigned)((batch + threads - 1) / threads));
  if (kind == 1) {
    if (layout == BX_LAYOUT_INTERLEAVED)
      ex::exact_kernel<1><<<grid, threads, 0, stream>>>(c, d, e, f, g, b, x, st, ix, subs, ws,
                                                       batch, n, Interleaved{ld});
    else
      ex::exact_kernel<1><<<grid, threads, 0, stream>>>(c, d, e, f, g, b, x, st, ix, subs, ws,
                                                       batch, n, SystemMajor{ld});
  } else {
    if (layout == BX_LAYOUT_INTERLEAVED)
      ex::exact_kernel<2><<<grid, threads, 0, stream>>>(c, d, e, f, g, b, x, st, ix, subs, ws,
                                                       batch, n, Interleaved{ld});
    else
      ex::exact_kernel<2><<<grid, threads, 0, stream>>>(c, d, e, f, g, b, x, st, ix, subs, ws,
                                                       batch, n, SystemMajor{ld});
  }
  return BX_OK;
}

}  // namespace bx
