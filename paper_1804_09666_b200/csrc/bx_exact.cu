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
// Realisation here: every quantity is a truncated Laurent series in t with
// binary64 coefficients for orders LO..HI, plus the highest order that is
// still exact ("top", tracked through every operation like p-adic precision:
// a division by a series of order v loses 2v orders at the top).  Because the
// result x(t) = A(t)^{-1} b is analytic at 0 (A nonsingular), its negative
// orders are rounding residue and are clamped; pivot coefficients below
// -sum(ord of the previous pivots) are clamped as well (leading minors are
// polynomials in t), which keeps the valuation of pivots exact.  A pivot is
// "identically zero" when every exact coefficient is 0.0 -- the reference's
// is_zero on a rational function (core.py:31-33).  The determinant gate is the
// order of the pivot product: det(A) = 0 iff sum ord(mu_i) > 0.
//
// One thread per system (latency-bound, config 3 is parity-first); the series
// of rec/mu, phi and y live in an interleaved scratch between the sweeps.
#include <math.h>

#include "bx_common.cuh"
#include "bx_kernels.h"

namespace bx {
namespace ex {

constexpr int LO = -4, HI = 4, NC = HI - LO + 1;

struct LS {
  double c[NC];  // c[k - LO] = coefficient of t^k
  int top;       // highest exact order
};

__device__ __forceinline__ LS ls_const(double v) {
  LS r;
#pragma unroll
  for (int k = 0; k < NC; ++k) r.c[k] = 0.0;
  r.c[-LO] = v;
  r.top = HI;
  return r;
}
__device__ __forceinline__ LS ls_t() {  // the indeterminate t
  LS r = ls_const(0.0);
  r.c[1 - LO] = 1.0;
  return r;
}
// lowest order with a nonzero exact coefficient; HI+1 if identically zero
__device__ __forceinline__ int ls_ord(const LS &a) {
#pragma unroll
  for (int k = 0; k < NC; ++k)
    if (k + LO <= a.top && a.c[k] != 0.0) return k + LO;
  return HI + 1;
}
__device__ __forceinline__ bool ls_is_zero(const LS &a) { return ls_ord(a) > a.top; }

__device__ __forceinline__ LS ls_scale(double s, const LS &a) {
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
// a*b truncated to the window; *ovf set if an exact nonzero product term falls below LO
__device__ __forceinline__ LS ls_mul(const LS &a, const LS &b, bool *ovf) {
  const int oa = ls_ord(a), ob = ls_ord(b);
  LS r;
#pragma unroll
  for (int k = 0; k < NC; ++k) r.c[k] = 0.0;
  if (oa > a.top || ob > b.top) {  // a zero factor
    r.top = HI;
    return r;
  }
  if (oa + ob < LO) *ovf = true;
#pragma unroll
  for (int i = 0; i < NC; ++i) {
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      const int k = i + j + LO;  // order (i+LO)+(j+LO) -> index k - LO
      if (k >= 0 && k < NC && i + LO <= a.top && j + LO <= b.top)
        r.c[k] = fma(a.c[i], b.c[j], r.c[k]);
    }
  }
  r.top = min(a.top + ob, b.top + oa);
  r.top = min(r.top, HI);
  return r;
}
// 1/b for b not identically zero
__device__ __forceinline__ LS ls_inv(const LS &b, bool *ovf) {
  const int v = ls_ord(b);
  LS r;
#pragma unroll
  for (int k = 0; k < NC; ++k) r.c[k] = 0.0;
  if (-v < LO) *ovf = true;
  const double b0 = b.c[v - LO];
  const double ib0 = 1.0 / b0;
  // 1/b = t^{-v} sum_k d_k t^k,  d_0 = 1/b_v,  d_k = -(sum_{j=1..k} b_{v+j} d_{k-j}) / b_v
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
  r.top = min(HI, b.top - 2 * v);
  return r;
}
__device__ __forceinline__ void ls_clamp_below(LS &a, int lo) {
#pragma unroll
  for (int k = 0; k < NC; ++k)
    if (k + LO < lo) a.c[k] = 0.0;
}

// scratch: NQ series planes (+ a top plane per series), interleaved [n][batch]
struct Store {
  double *base;
  int64_t batch, n;
  __device__ __forceinline__ double *plane(int p) const { return base + (int64_t)p * batch * n; }
  __device__ __forceinline__ void put(int q, int64_t i, int64_t s, const LS &a) const {
#pragma unroll
    for (int k = 0; k < NC; ++k) plane(q * (NC + 1) + k)[i * batch + s] = a.c[k];
    plane(q * (NC + 1) + NC)[i * batch + s] = (double)a.top;
  }
  __device__ __forceinline__ LS get(int q, int64_t i, int64_t s) const {
    LS a;
#pragma unroll
    for (int k = 0; k < NC; ++k) a.c[k] = plane(q * (NC + 1) + k)[i * batch + s];
    a.top = (int)plane(q * (NC + 1) + NC)[i * batch + s];
    return a;
  }
};

// ---------------------------------------------------------------------------
// STDM: tri_factor_recip + tri_solve_recip with the t-substitution policy
// ---------------------------------------------------------------------------
template <class Lay>
__global__ void stdm_kernel(const double *__restrict__ dp, const double *__restrict__ ep,
                            const double *__restrict__ fp, const double *__restrict__ bp,
                            double *__restrict__ xp, int32_t *status, int32_t *index,
                            int32_t *subs, Store S, int64_t batch, int64_t n, Lay lay) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= batch) return;
  bool ovf = false;
  int nsub = 0, ordsum = 0;
  LS rec, y;
  // forward: rec_i = 1/mu_i, y_i = b_i - l_i y_{i-1}  (_elim.py:98-117)
  for (int64_t i = 0; i < n; ++i) {
    LS mu;
    const double e = ldg(ep + lay(i, s));
    const double b = ldg(bp + lay(i, s));
    LS l;
    if (i == 0) {
      mu = ls_const(e);
      y = ls_const(b);
    } else {
      l = ls_scale(ldg(dp + lay(i, s)), rec);                                  // l = d * rec
      mu = ls_sub(ls_const(e), ls_scale(ldg(fp + lay(i - 1, s)), l));          // e - l f
      y = ls_sub(ls_const(b), ls_mul(l, y, &ovf));                             // b - l y
    }
    ls_clamp_below(mu, -ordsum);
    if (ls_is_zero(mu)) {  // _Substituter: exact zero pivot -> t
      mu = ls_t();
      ++nsub;
    }
    ordsum += ls_ord(mu);
    rec = ls_inv(mu, &ovf);
    S.put(0, i, s, rec);
    S.put(1, i, s, y);
  }
  if (subs) subs[s] = nsub;
  if (ordsum > 0) {  // exact_det_band(t) == 0 -> SingularMatrix (exact.py:301-302)
    set_status(status, index, s, BX_STATUS_SINGULAR, -1);
    for (int64_t i = 0; i < n; ++i) xp[lay(i, s)] = __longlong_as_double(0x7ff8000000000000LL);
    return;
  }
  // backward: x_i = (y_i - f_i x_{i+1}) rec_i  (_elim.py:118-121), x analytic at 0
  LS x = ls_mul(S.get(1, n - 1, s), S.get(0, n - 1, s), &ovf);
  ls_clamp_below(x, 0);
  if (x.top < 0) ovf = true;
  xp[lay(n - 1, s)] = x.c[-LO];
  for (int64_t i = n - 2; i >= 0; --i) {
    const LS yi = S.get(1, i, s), ri = S.get(0, i, s);
    x = ls_mul(ls_sub(yi, ls_scale(ldg(fp + lay(i, s)), x)), ri, &ovf);
    ls_clamp_below(x, 0);
    if (x.top < 0) ovf = true;
    xp[lay(i, s)] = x.c[-LO];
  }
  set_status(status, index, s, ovf ? BX_STATUS_WINDOW_OVERFLOW : BX_STATUS_OK, -1);
}

// ---------------------------------------------------------------------------
// SPDM: penta_factor + _penta_substitute_solve (exact.py:239-251)
// ---------------------------------------------------------------------------
template <class Lay>
__global__ void spdm_kernel(const double *__restrict__ cp, const double *__restrict__ dp,
                            const double *__restrict__ ep, const double *__restrict__ fp,
                            const double *__restrict__ gp, const double *__restrict__ bp,
                            double *__restrict__ xp, int32_t *status, int32_t *index,
                            int32_t *subs, Store S, int64_t batch, int64_t n, Lay lay) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= batch) return;
  bool ovf = false;
  int nsub = 0, ordsum = 0;
  // carried rows i-1, i-2: mu, phi, y (series) and psi (= g, scalar)
  LS mu1, mu2, ph1, ph2, y1, y2;
  double ps1 = 0.0, ps2 = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double e = ldg(ep + lay(i, s));
    const double b = ldg(bp + lay(i, s));
    const double f = i <= n - 2 ? ldg(fp + lay(i, s)) : 0.0;
    const double g = i <= n - 3 ? ldg(gp + lay(i, s)) : 0.0;
    LS mu, ph, y;
    if (i == 0) {
      mu = ls_const(e);
      ph = ls_const(f);
      y = ls_const(b);
    } else if (i == 1) {
      const LS l1 = ls_mul(ls_const(ldg(dp + lay(i, s))), ls_inv(mu1, &ovf), &ovf);   // d0/mu0
      mu = ls_sub(ls_const(e), ls_mul(l1, ph1, &ovf));
      ph = ls_sub(ls_const(f), ls_scale(ps1, l1));
      y = ls_sub(ls_const(b), ls_mul(l1, y1, &ovf));
    } else {
      const LS l2 = ls_scale(ldg(cp + lay(i, s)), ls_inv(mu2, &ovf));                 // c/mu_{i-2}
      const LS l1 = ls_mul(ls_sub(ls_const(ldg(dp + lay(i, s))), ls_mul(l2, ph2, &ovf)),
                           ls_inv(mu1, &ovf), &ovf);                                    // (d - l2 phi)/mu
      mu = ls_sub(ls_sub(ls_const(e), ls_scale(ps2, l2)), ls_mul(l1, ph1, &ovf));
      ph = i <= n - 2 ? ls_sub(ls_const(f), ls_scale(ps1, l1)) : ls_const(0.0);
      y = ls_sub(ls_sub(ls_const(b), ls_mul(l1, y1, &ovf)), ls_mul(l2, y2, &ovf));
    }
    ls_clamp_below(mu, -ordsum);
    if (ls_is_zero(mu)) {
      mu = ls_t();
      ++nsub;
    }
    ordsum += ls_ord(mu);
    S.put(0, i, s, mu);
    S.put(1, i, s, ph);
    S.put(2, i, s, y);
    mu2 = mu1; mu1 = mu;
    ph2 = ph1; ph1 = ph;
    y2 = y1; y1 = y;
    ps2 = ps1; ps1 = g;
  }
  if (subs) subs[s] = nsub;
  if (ordsum > 0) {
    set_status(status, index, s, BX_STATUS_SINGULAR, -1);
    for (int64_t i = 0; i < n; ++i) xp[lay(i, s)] = __longlong_as_double(0x7ff8000000000000LL);
    return;
  }
  // x_{n-1} = y/mu ; x_{n-2} = (y - phi x1)/mu ; x_i = (y - phi x1 - psi x2)/mu
  LS x1 = ls_mul(S.get(2, n - 1, s), ls_inv(S.get(0, n - 1, s), &ovf), &ovf);
  ls_clamp_below(x1, 0);
  if (x1.top < 0) ovf = true;
  xp[lay(n - 1, s)] = x1.c[-LO];
  LS x2 = x1;
  x1 = ls_mul(ls_sub(S.get(2, n - 2, s), ls_mul(S.get(1, n - 2, s), x2, &ovf)),
              ls_inv(S.get(0, n - 2, s), &ovf), &ovf);
  ls_clamp_below(x1, 0);
  if (x1.top < 0) ovf = true;
  xp[lay(n - 2, s)] = x1.c[-LO];
  for (int64_t i = n - 3; i >= 0; --i) {
    const double g = ldg(gp + lay(i, s));
    LS num = ls_sub(ls_sub(S.get(2, i, s), ls_mul(S.get(1, i, s), x1, &ovf)), ls_scale(g, x2));
    LS xi = ls_mul(num, ls_inv(S.get(0, i, s), &ovf), &ovf);
    ls_clamp_below(xi, 0);
    if (xi.top < 0) ovf = true;
    xp[lay(i, s)] = xi.c[-LO];
    x2 = x1;
    x1 = xi;
  }
  set_status(status, index, s, ovf ? BX_STATUS_WINDOW_OVERFLOW : BX_STATUS_OK, -1);
}

}  // namespace ex

size_t exact_workspace_bytes(int kind, int64_t batch, int64_t n) {
  const int nq = kind == 1 ? 2 : 3;  // STDM: rec, y ; SPDM: mu, phi, y
  return sizeof(double) * (size_t)nq * (ex::NC + 1) * (size_t)batch * (size_t)n;
}

int exact_solve(int kind, const double *c, const double *d, const double *e, const double *f,
                const double *g, const double *b, double *x, int32_t *st, int32_t *ix,
                int32_t *subs, double *ws, int64_t batch, int64_t n, int64_t ld, int layout,
                cudaStream_t stream) {
  ex::Store S{ws, batch, n};
  const int threads = 32;
  const dim3 grid((unsigned)((batch + threads - 1) / threads));
  if (kind == 1) {
    if (layout == BX_LAYOUT_INTERLEAVED)
      ex::stdm_kernel<<<grid, threads, 0, stream>>>(d, e, f, b, x, st, ix, subs, S, batch, n,
                                                    Interleaved{ld});
    else
      ex::stdm_kernel<<<grid, threads, 0, stream>>>(d, e, f, b, x, st, ix, subs, S, batch, n,
                                                    SystemMajor{ld});
  } else {
    if (layout == BX_LAYOUT_INTERLEAVED)
      ex::spdm_kernel<<<grid, threads, 0, stream>>>(c, d, e, f, g, b, x, st, ix, subs, S, batch, n,
                                                    Interleaved{ld});
    else
      ex::spdm_kernel<<<grid, threads, 0, stream>>>(c, d, e, f, g, b, x, st, ix, subs, S, batch, n,
                                                    SystemMajor{ld});
  }
  return BX_OK;
}

}  // namespace bx
