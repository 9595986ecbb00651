// Band-matrix building blocks of the reference exposed as batched entry
// points (SURVEY 8a rows a3-a5, a8 helpers), in the reference's operation
// order with one IEEE rounding per operation (bit-identical results):
//   band_matvec   A x / b - A x     penta_matvec / tri_matvec / residual
//                                   (core.py:243-314, float branch: the array
//                                   sweeps main, sub1, sup1, sub2, sup2)
//   lu_penta      banded Doolittle  penta_factor via lu_penta (_elim.py:30-62,
//                                   direct.py:42-63): mu, l1, l2, phi, psi
//   forward_sub   L y = rhs         penta_forward (_elim.py:65-73,
//                                   iterative.py:127-137)
//   backward_sub  U x = y           penta_backward (_elim.py:76-87,
//                                   iterative.py:140-149)
// The sweeps take an outer stride m (the reference's pentadiagonal is m = 2;
// m >= 3 serves the grid ILU(0) factors of iterative.ilu0_penta).  One
// thread per system walks its rows (the recurrences are sequential);
// interleaved storage makes every row access of a warp one coalesced segment.
#include "bx_common.cuh"
#include "bx_kernels.h"

namespace bx {
namespace bops {

constexpr int kThreads = 64;

// y = A x  (rhs == nullptr)  or  y = rhs - A x, one element per thread
template <class Lay>
__global__ void __launch_bounds__(256)
matvec_kernel(int bw, int64_t m, const double *__restrict__ c, const double *__restrict__ d,
              const double *__restrict__ e, const double *__restrict__ f,
              const double *__restrict__ g, const double *__restrict__ x,
              const double *__restrict__ b, double *__restrict__ y, int64_t batch, int64_t n,
              bool sys_fastest, Lay lay) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= batch * n) return;
  // index order that keeps a warp's accesses contiguous in the layout
  const int64_t s = sys_fastest ? t % batch : t / n;
  const int64_t i = sys_fastest ? t / batch : t % n;
  double acc = mul(ldg(e + lay(i, s)), ldg(x + lay(i, s)));                          // main
  if (i >= 1) acc = add(acc, mul(ldg(d + lay(i, s)), ldg(x + lay(i - 1, s))));       // sub1
  if (i <= n - 2) acc = add(acc, mul(ldg(f + lay(i, s)), ldg(x + lay(i + 1, s))));   // sup1
  if (bw == 2) {
    if (i >= m) acc = add(acc, mul(ldg(c + lay(i, s)), ldg(x + lay(i - m, s))));     // sub_m
    if (i <= n - 1 - m) acc = add(acc, mul(ldg(g + lay(i, s)), ldg(x + lay(i + m, s))));  // sup_m
  }
  y[lay(i, s)] = b ? sub(ldg(b + lay(i, s)), acc) : acc;
}

// penta_factor (m = 2) with the raising zero-pivot policy of lu_penta; the
// structurally absent slots (l1[0], l2[0..1], phi[n-1], psi[n-2..]) are 0
template <class Lay>
__global__ void __launch_bounds__(kThreads)
lu_penta_kernel(const double *__restrict__ c, const double *__restrict__ d,
                const double *__restrict__ e, const double *__restrict__ f,
                const double *__restrict__ g, double *__restrict__ mu, double *__restrict__ l1,
                double *__restrict__ l2, double *__restrict__ phi, double *__restrict__ psi,
                int32_t *status, int32_t *index, int64_t batch, int64_t n, Lay lay) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= batch) return;
  int32_t bad = -1;
  auto chk = [&](int64_t i, double v) {
    if (v == 0.0 && bad < 0) bad = (int32_t)i;
  };
  // carried: mu, phi, psi of rows i-1 (1) and i-2 (2)
  double m0 = ldg(e + lay(0, s));
  chk(0, m0);
  double ph0 = ldg(f + lay(0, s)), ps0 = n >= 3 ? ldg(g + lay(0, s)) : 0.0;  // _elim.py:44-46
  mu[lay(0, s)] = m0;
  l1[lay(0, s)] = 0.0;
  l2[lay(0, s)] = 0.0;
  phi[lay(0, s)] = ph0;
  psi[lay(0, s)] = ps0;
  const double l11 = dvd(ldg(d + lay(1, s)), m0);                      // _elim.py:47
  const double m1 = sub(ldg(e + lay(1, s)), mul(l11, ph0));            // _elim.py:48
  chk(1, m1);
  const double ph1 = n >= 3 ? sub(ldg(f + lay(1, s)), mul(l11, ps0)) : 0.0;  // _elim.py:50
  const double ps1 = n >= 4 ? ldg(g + lay(1, s)) : 0.0;                // _elim.py:51-52
  mu[lay(1, s)] = m1;
  l1[lay(1, s)] = l11;
  l2[lay(1, s)] = 0.0;
  phi[lay(1, s)] = ph1;
  psi[lay(1, s)] = ps1;
  double mu2 = m0, mu1 = m1, phi2 = ph0, phi1 = ph1, psi2 = ps0, psi1 = ps1;
  for (int64_t i = 2; i < n; ++i) {                                    // _elim.py:53-61
    const double li2 = dvd(ldg(c + lay(i, s)), mu2);
    const double li1 = dvd(sub(ldg(d + lay(i, s)), mul(li2, phi2)), mu1);
    const double mi = sub(sub(ldg(e + lay(i, s)), mul(li2, psi2)), mul(li1, phi1));
    chk(i, mi);
    const double phn = i <= n - 2 ? sub(ldg(f + lay(i, s)), mul(li1, psi1)) : 0.0;
    const double psn = i <= n - 3 ? ldg(g + lay(i, s)) : 0.0;
    mu[lay(i, s)] = mi;
    l1[lay(i, s)] = li1;
    l2[lay(i, s)] = li2;
    phi[lay(i, s)] = phn;
    psi[lay(i, s)] = psn;
    mu2 = mu1; mu1 = mi;
    phi2 = phi1; phi1 = phn;
    psi2 = psi1; psi1 = psn;
  }
  set_status(status, index, s, bad < 0 ? BX_STATUS_OK : BX_STATUS_ZERO_PIVOT, bad);
}

// L y = rhs: y_0 = b_0; y_i = b_i - l1_i y_{i-1} (i < m); y_i = (b_i - l1_i y_{i-1}) - lm_i y_{i-m}
template <class Lay>
__global__ void __launch_bounds__(kThreads)
forward_kernel(int64_t m, const double *__restrict__ l1, const double *__restrict__ lm,
               const double *__restrict__ b, double *__restrict__ y, int64_t batch, int64_t n,
               Lay lay) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= batch) return;
  double prev = ldg(b + lay(0, s));
  y[lay(0, s)] = prev;
  for (int64_t i = 1; i < n; ++i) {
    double v = sub(ldg(b + lay(i, s)), mul(ldg(l1 + lay(i, s)), prev));
    if (i >= m) v = sub(v, mul(ldg(lm + lay(i, s)), y[lay(i - m, s)]));
    y[lay(i, s)] = v;
    prev = v;
  }
}

// U x = y: ZeroPivot(first zero pivot) before any division (_elim.py:80-82);
// x_{n-1} = y/mu; x_i = ((y - phi x_{i+1}) - psi x_{i+m}) / mu
template <class Lay>
__global__ void __launch_bounds__(kThreads)
backward_kernel(int64_t m, const double *__restrict__ mu, const double *__restrict__ phi,
                const double *__restrict__ psi, const double *__restrict__ y,
                double *__restrict__ x, int32_t *status, int32_t *index, int64_t batch, int64_t n,
                Lay lay) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= batch) return;
  for (int64_t i = 0; i < n; ++i)
    if (ldg(mu + lay(i, s)) == 0.0) {
      set_status(status, index, s, BX_STATUS_ZERO_PIVOT, (int32_t)i);
      const double nan = __longlong_as_double(0x7ff8000000000000LL);
      for (int64_t j = 0; j < n; ++j) x[lay(j, s)] = nan;
      return;
    }
  double next = dvd(ldg(y + lay(n - 1, s)), ldg(mu + lay(n - 1, s)));
  x[lay(n - 1, s)] = next;
  for (int64_t i = n - 2; i >= 0; --i) {
    double v = sub(ldg(y + lay(i, s)), mul(ldg(phi + lay(i, s)), next));
    if (i <= n - 1 - m) v = sub(v, mul(ldg(psi + lay(i, s)), x[lay(i + m, s)]));
    next = dvd(v, ldg(mu + lay(i, s)));
    x[lay(i, s)] = next;
  }
  set_status(status, index, s, BX_STATUS_OK, -1);
}

inline dim3 sys_grid(int64_t batch) { return dim3((unsigned)((batch + kThreads - 1) / kThreads)); }

}  // namespace bops

void band_matvec(int bw, int64_t m, const double *c, const double *d, const double *e,
                 const double *f, const double *g, const double *x, const double *b, double *y,
                 int64_t batch, int64_t n, int64_t ld, int layout, cudaStream_t stream) {
  const int64_t tot = batch * n;
  const dim3 grid((unsigned)((tot + 255) / 256));
  if (layout == BX_LAYOUT_INTERLEAVED)
    bops::matvec_kernel<<<grid, 256, 0, stream>>>(bw, m, c, d, e, f, g, x, b, y, batch, n, true,
                                                   Interleaved{ld});
  else
    bops::matvec_kernel<<<grid, 256, 0, stream>>>(bw, m, c, d, e, f, g, x, b, y, batch, n, false,
                                                   SystemMajor{ld});
}

void lu_penta(const double *c, const double *d, const double *e, const double *f, const double *g,
              double *mu, double *l1, double *l2, double *phi, double *psi, int32_t *st,
              int32_t *ix, int64_t batch, int64_t n, int64_t ld, int layout, cudaStream_t stream) {
  if (layout == BX_LAYOUT_INTERLEAVED)
    bops::lu_penta_kernel<<<bops::sys_grid(batch), bops::kThreads, 0, stream>>>(
        c, d, e, f, g, mu, l1, l2, phi, psi, st, ix, batch, n, Interleaved{ld});
  else
    bops::lu_penta_kernel<<<bops::sys_grid(batch), bops::kThreads, 0, stream>>>(
        c, d, e, f, g, mu, l1, l2, phi, psi, st, ix, batch, n, SystemMajor{ld});
}

void forward_sub(int64_t m, const double *l1, const double *lm, const double *b, double *y,
                 int64_t batch, int64_t n, int64_t ld, int layout, cudaStream_t stream) {
  if (layout == BX_LAYOUT_INTERLEAVED)
    bops::forward_kernel<<<bops::sys_grid(batch), bops::kThreads, 0, stream>>>(m, l1, lm, b, y, batch,
                                                                             n, Interleaved{ld});
  else
    bops::forward_kernel<<<bops::sys_grid(batch), bops::kThreads, 0, stream>>>(m, l1, lm, b, y, batch,
                                                                             n, SystemMajor{ld});
}

void backward_sub(int64_t m, const double *mu, const double *phi, const double *psi, const double *y,
                  double *x, int32_t *st, int32_t *ix, int64_t batch, int64_t n, int64_t ld,
                  int layout, cudaStream_t stream) {
  if (layout == BX_LAYOUT_INTERLEAVED)
    bops::backward_kernel<<<bops::sys_grid(batch), bops::kThreads, 0, stream>>>(
        m, mu, phi, psi, y, x, st, ix, batch, n, Interleaved{ld});
  else
    bops::backward_kernel<<<bops::sys_grid(batch), bops::kThreads, 0, stream>>>(
        m, mu, phi, psi, y, x, st, ix, batch, n, SystemMajor{ld});
}

}  // namespace bx
