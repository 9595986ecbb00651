// Banded ("array implementation") Hotelling-Bodewig inversion of the ILU(0)
// factors -- hb_invert_banded (inverse.py:122-195) and the banded apply of
// BandedApproxInverse.matvec (41-61), reference op order, bit-exact:
//
//   * _band_mul_tri (122-137): out[r] = sum_{j} a[j] * b[r-j], truncated to
//     offsets 0..w, accumulated from 0.0 in ascending j with one rounding per
//     multiply and per add (numpy elementwise, no FMA);
//   * _band_residual_norm (140-145): max(|1 - P_0|, max_r |P_r|);
//   * S = -P, S_0 = 2 + S_0 (inverse.py:193-194), folded into the second
//     product's operand fetch.
//
// Storage: diagonal r of factor f at X[(f*(cap+1) + r)*n + k], k < n - r,
// with the reference's indexing -- lower: entry (k+r, k); upper: (k, k+r).
// M (the factor itself, offsets 0..2) is read from the ILU(0) planes of
// bx_sip.cu ([n][batch] interleaved, row-aligned).
#include <math.h>
#include <string.h>

#include <vector>

#include "bx_common.cuh"
#include "bx_kernels.h"

namespace bx {
namespace hbb {

// ILU(0) factor planes (bx_sip.cu): MU, L1, L2, PHI, PSI
enum { MU = 0, L1, L2, PHI, PSI };

// diagonal j (0..2) of factor f at position k (reference diag arrays)
__device__ __forceinline__ double mdiag(const double *fac, int lower, int j, int64_t k, int64_t s,
                                        int64_t batch, int64_t n) {
  const int64_t pl = batch * n;
  if (lower) {  // unit-lower L: (1, l_sub1, l_sub2); l_sub1[k] = L(k+1, k)
    if (j == 0) return 1.0;
    return fac[(j == 1 ? L1 : L2) * pl + (k + j) * batch + s];
  }
  return fac[(j == 0 ? MU : j == 1 ? PHI : PSI) * pl + k * batch + s];  // U(k, k+j)
}

// X_0: lower ones, upper 1/diag (inverse.py:170-181); other diagonals zero.
// Zero upper diagonal -> ZeroDiagonal(first row) (inverse.py:175-177).
__global__ void band_init_kernel(double *X, const double *fac, const int *act, int nact,
                                 int64_t batch, int64_t n, int64_t cap, int64_t w, int *zero_row) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)nact * (w + 1) * n) return;
  const int f = act[idx % nact];
  const int64_t rk = idx / nact, r = rk / n, k = rk % n;
  const int lower = f < batch;
  const int64_t s = lower ? f : f - batch;
  double v = 0.0;
  if (r == 0) {
    if (lower) {
      v = 1.0;
    } else {
      const double d = mdiag(fac, 0, 0, k, s, batch, n);
      if (d == 0.0) atomicMin(zero_row + f, (int)k);
      v = __ddiv_rn(1.0, d);
    }
  }
  X[((int64_t)f * (cap + 1) + r) * n + k] = v;
}

// P = M X (M: offsets 0..2), truncated to 0..w  (_band_mul_tri(m, x))
__global__ void band_mx_kernel(const double *__restrict__ fac, const double *__restrict__ X,
                               double *__restrict__ P, const int *act, int nact, int64_t batch,
                               int64_t n, int64_t cap, int64_t w) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)nact * (w + 1) * n) return;
  const int f = act[idx % nact];
  const int64_t rk = idx / nact, r = rk / n, i = rk % n;
  if (i >= n - r) return;
  const int lower = f < batch;
  const int64_t s = lower ? f : f - batch;
  const double *x = X + (int64_t)f * (cap + 1) * n;
  double acc = 0.0;
  const int64_t j0 = r - w > 0 ? r - w : 0, j1 = r < 2 ? r : 2;
  for (int64_t j = j0; j <= j1; ++j) {
    const int64_t l = r - j;
    const double t = lower ? __dmul_rn(mdiag(fac, 1, (int)j, l + i, s, batch, n), x[l * n + i])
                           : __dmul_rn(mdiag(fac, 0, (int)j, i, s, batch, n), x[l * n + j + i]);
    acc = __dadd_rn(acc, t);
  }
  P[((int64_t)f * (cap + 1) + r) * n + i] = acc;
}

// Xn = X S with S = -P, S_0 = 2 + S_0, truncated to 0..w (_band_mul_tri(x, s))
__global__ void band_xs_kernel(const double *__restrict__ X, const double *__restrict__ P,
                               double *__restrict__ Xn, const int *act, int nact, int64_t batch,
                               int64_t n, int64_t cap, int64_t w) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)nact * (w + 1) * n) return;
  const int f = act[idx % nact];
  const int64_t rk = idx / nact, r = rk / n, i = rk % n;
  if (i >= n - r) return;
  const int lower = f < batch;
  const double *x = X + (int64_t)f * (cap + 1) * n;
  const double *p = P + (int64_t)f * (cap + 1) * n;
  auto S = [&](int64_t l, int64_t k) {
    return l == 0 ? __dadd_rn(2.0, -p[k]) : -p[l * n + k];
  };
  double acc = 0.0;
  for (int64_t j = 0; j <= r; ++j) {  // p = q = w >= r
    const int64_t l = r - j;
    const double t = lower ? __dmul_rn(x[j * n + l + i], S(l, i)) : __dmul_rn(x[j * n + i], S(l, j + i));
    acc = __dadd_rn(acc, t);
  }
  Xn[((int64_t)f * (cap + 1) + r) * n + i] = acc;
}

__device__ __forceinline__ unsigned long long nan_high_bits(double r) {
  if (r != r) r = __longlong_as_double(0x7ff8000000000000LL);
  return (unsigned long long)__double_as_longlong(r);
}

// _band_residual_norm: max(|1 - P_0|, max_{r>=1} |P_r|)
__global__ void band_resid_kernel(const double *__restrict__ P, const int *act, int nact,
                                  unsigned long long *rbits, int64_t batch, int64_t n, int64_t cap,
                                  int64_t w) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)nact * (w + 1) * n) return;
  const int f = act[idx % nact];
  const int64_t rk = idx / nact, r = rk / n, i = rk % n;
  if (i >= n - r) return;
  const double v = P[((int64_t)f * (cap + 1) + r) * n + i];
  const double a = r == 0 ? fabs(__dsub_rn(1.0, v)) : fabs(v);
  atomicMax(rbits + f, nan_high_bits(a));
}

// true residual ||I - M X||_inf (max row sum over the full product band
// 0..w+2): the widening criterion of the auto mode
__global__ void band_true_resid_kernel(const double *__restrict__ fac, const double *__restrict__ X,
                                       const int *act, int nact, unsigned long long *rbits,
                                       int64_t batch, int64_t n, int64_t cap, int64_t w) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)nact * n) return;
  const int f = act[idx % nact];
  const int64_t row = idx / nact;
  const int lower = f < batch;
  const int64_t s = lower ? f : f - batch;
  const double *x = X + (int64_t)f * (cap + 1) * n;
  double sum = 0.0;
  for (int64_t r = 0; r <= w + 2; ++r) {
    // entry of M X on diagonal r in this row: lower (row, row-r), upper (row, row+r)
    const int64_t k = lower ? row - r : row;  // reference diag position
    if (k < 0 || k >= n - r) continue;
    double acc = 0.0;
    const int64_t j0 = r - w > 0 ? r - w : 0, j1 = r < 2 ? r : 2;
    for (int64_t j = j0; j <= j1; ++j) {
      const int64_t l = r - j;
      acc = lower ? fma(mdiag(fac, 1, (int)j, l + k, s, batch, n), x[l * n + k], acc)
                  : fma(mdiag(fac, 0, (int)j, k, s, batch, n), x[l * n + j + k], acc);
    }
    sum += r == 0 ? fabs(1.0 - acc) : fabs(acc);
  }
  atomicMax(rbits + f, nan_high_bits(sum));
}

__global__ void band_copy_kernel(const double *src, double *dst, const int *act, int nact,
                                 int64_t n, int64_t cap, int64_t w) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)nact * (w + 1) * n) return;
  const int f = act[idx % nact];
  const int64_t rk = idx / nact;
  const int64_t o = (int64_t)f * (cap + 1) * n + rk;
  dst[o] = src[o];
}

// BandedApproxInverse.matvec (inverse.py:49-61): out = d0 * v, then
// out[i] += d_j[i-j] v[i-j] (lower) / d_j[i] v[i+j] (upper), j = 1..w.
// v, out: [n][batch] vectors; factor f = s (lower) or batch + s (upper).
__global__ void band_apply_kernel(const double *__restrict__ X, const int64_t *__restrict__ wf,
                                  const double *__restrict__ v, double *__restrict__ out,
                                  const int *act, int nact, int64_t batch, int64_t n, int64_t cap,
                                  int upper) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)nact * n) return;
  const int64_t s = act[idx % nact], i = idx / nact;
  const int64_t f = upper ? batch + s : s;
  const double *x = X + f * (cap + 1) * n;
  const int64_t w = wf[f];
  double acc = __dmul_rn(x[i], v[i * batch + s]);
  for (int64_t j = 1; j <= w; ++j) {
    if (!upper && i >= j) acc = __dadd_rn(acc, __dmul_rn(x[j * n + i - j], v[(i - j) * batch + s]));
    if (upper && i < n - j) acc = __dadd_rn(acc, __dmul_rn(x[j * n + i], v[(i + j) * batch + s]));
  }
  out[i * batch + s] = acc;
}

// caller's row-aligned factor diagonals (layout) -> ILU planes [n][batch]
template <class Lay>
__global__ void factors_to_planes_kernel(const double *mu, const double *l1, const double *l2,
                                         const double *phi, const double *psi, double *fac,
                                         int64_t batch, int64_t n, Lay lay) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= batch * n) return;
  const int64_t i = idx / batch, s = idx % batch, pl = batch * n;
  fac[MU * pl + idx] = mu ? mu[lay(i, s)] : 0.0;
  fac[L1 * pl + idx] = l1 ? l1[lay(i, s)] : 0.0;
  fac[L2 * pl + idx] = l2 ? l2[lay(i, s)] : 0.0;
  fac[PHI * pl + idx] = phi ? phi[lay(i, s)] : 0.0;
  fac[PSI * pl + idx] = psi ? psi[lay(i, s)] : 0.0;
}

inline unsigned blocks(int64_t work, int threads = 256) {
  return (unsigned)((work + threads - 1) / threads);
}

}  // namespace hbb

size_t hb_band_bytes(int64_t batch, int64_t n, int64_t cap) {
  // X, Xn, P, best (doubles) + per-factor width
  return sizeof(double) * 4 * (size_t)(2 * batch) * (size_t)(cap + 1) * (size_t)n +
         sizeof(int64_t) * (size_t)(2 * batch) + 256;
}

// One banded inversion round at width w for the factors in `act`; results
// (the reference's InversionReport / exceptions) per factor in the host
// arrays.  X ends holding, per factor, the approximation the reference
// returns: the converged iterate, or `best` on Stagnated / MaxIterations.
int hb_band_invert_round(const double *fac, double *X, double *Xn, double *P, double *Best,
                         int *dact, int *dzero, unsigned long long *rbits,
                         const std::vector<int> &act0, const double *tol_f, int64_t batch,
                         int64_t n, int64_t cap, int64_t w, int64_t max_iter, int64_t *iters,
                         double *resid, int *status, int *zero_row,
                         std::vector<std::vector<double>> *hist, cudaStream_t st) {
  using namespace hbb;
  const int F = (int)(2 * batch);
  std::vector<int> act = act0;
  if (act.empty()) return BX_OK;
  int na = (int)act.size();
  std::vector<int> zr(F, 0x7fffffff);
  cudaMemcpyAsync(dzero, zr.data(), sizeof(int) * F, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(dact, act.data(), sizeof(int) * na, cudaMemcpyHostToDevice, st);
  band_init_kernel<<<blocks((int64_t)na * (w + 1) * n), 256, 0, st>>>(X, fac, dact, na, batch, n,
                                                                       cap, w, dzero);
  cudaMemcpyAsync(zr.data(), dzero, sizeof(int) * F, cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  {
    std::vector<int> keep;
    for (int f : act) {
      if (zr[f] != 0x7fffffff) {
        status[f] = BX_STATUS_ZERO_DIAG;
        zero_row[f] = zr[f];
        iters[f] = 0;
        resid[f] = NAN;
      } else {
        keep.push_back(f);
      }
    }
    act.swap(keep);
  }
  std::vector<double> best_r(F, INFINITY);
  std::vector<int64_t> best_it(F, 0);
  std::vector<std::vector<double>> h(F);
  std::vector<unsigned long long> bits(F);
  for (int64_t it = 0; it <= max_iter && !act.empty(); ++it) {
    na = (int)act.size();
    cudaMemcpyAsync(dact, act.data(), sizeof(int) * na, cudaMemcpyHostToDevice, st);
    cudaMemsetAsync(rbits, 0, sizeof(unsigned long long) * F, st);
    const unsigned g = blocks((int64_t)na * (w + 1) * n);
    band_mx_kernel<<<g, 256, 0, st>>>(fac, X, P, dact, na, batch, n, cap, w);
    band_resid_kernel<<<g, 256, 0, st>>>(P, dact, na, rbits, batch, n, cap, w);
    cudaMemcpyAsync(bits.data(), rbits, sizeof(unsigned long long) * F, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    std::vector<int> improved, next;
    for (int f : act) {
      double r;
      memcpy(&r, &bits[f], sizeof r);
      h[f].push_back(r);
      if (r < best_r[f]) {
        best_r[f] = r;
        best_it[f] = it;
        improved.push_back(f);
      }
      const size_t L = h[f].size();
      if (r < tol_f[f]) {  // converged: the current iterate is returned
        status[f] = BX_STATUS_OK;
        iters[f] = it;
        resid[f] = r;
      } else if (L > 3 && r > 0.99 * h[f][L - 1 - 3]) {  // Stagnated(best)
        status[f] = BX_STATUS_STAGNATED;
        iters[f] = best_it[f];
        resid[f] = best_r[f];
      } else if (it == max_iter) {  // MaxIterationsExceeded(best.inverse, history[-1])
        status[f] = BX_STATUS_MAX_ITER;
        iters[f] = max_iter;
        resid[f] = r;
      } else {
        next.push_back(f);
      }
    }
    if (!improved.empty()) {
      const int ni = (int)improved.size();
      cudaMemcpyAsync(dact, improved.data(), sizeof(int) * ni, cudaMemcpyHostToDevice, st);
      band_copy_kernel<<<blocks((int64_t)ni * (w + 1) * n), 256, 0, st>>>(X, Best, dact, ni, n,
                                                                           cap, w);
    }
    if (!next.empty()) {
      const int nn = (int)next.size();
      cudaMemcpyAsync(dact, next.data(), sizeof(int) * nn, cudaMemcpyHostToDevice, st);
      band_xs_kernel<<<blocks((int64_t)nn * (w + 1) * n), 256, 0, st>>>(X, P, Xn, dact, nn, batch,
                                                                         n, cap, w);
      band_copy_kernel<<<blocks((int64_t)nn * (w + 1) * n), 256, 0, st>>>(Xn, X, dact, nn, n, cap,
                                                                           w);
    }
    act.swap(next);
  }
  // stagnated / max-iteration factors return the best approximation
  std::vector<int> use_best;
  for (int f : act0)
    if (status[f] == BX_STATUS_STAGNATED || status[f] == BX_STATUS_MAX_ITER) use_best.push_back(f);
  if (!use_best.empty()) {
    const int nb = (int)use_best.size();
    cudaMemcpyAsync(dact, use_best.data(), sizeof(int) * nb, cudaMemcpyHostToDevice, st);
    band_copy_kernel<<<blocks((int64_t)nb * (w + 1) * n), 256, 0, st>>>(Best, X, dact, nb, n, cap,
                                                                         w);
  }
  if (hist)
    for (int f : act0) (*hist)[f] = h[f];
  cudaStreamSynchronize(st);
  return bxh::check_launch("banded hotelling-bodewig");
}

// true residual ||I - M X||_inf of the factors in act (host array out)
int hb_band_true_residual(const double *fac, const double *X, int *dact, unsigned long long *rbits,
                          const std::vector<int> &act, int64_t batch, int64_t n, int64_t cap,
                          int64_t w, double *out, cudaStream_t st) {
  using namespace hbb;
  const int F = (int)(2 * batch);
  if (act.empty()) return BX_OK;
  const int na = (int)act.size();
  cudaMemcpyAsync(dact, act.data(), sizeof(int) * na, cudaMemcpyHostToDevice, st);
  cudaMemsetAsync(rbits, 0, sizeof(unsigned long long) * F, st);
  band_true_resid_kernel<<<blocks((int64_t)na * n), 256, 0, st>>>(fac, X, dact, na, rbits, batch,
                                                                   n, cap, w);
  std::vector<unsigned long long> bits(F);
  cudaMemcpyAsync(bits.data(), rbits, sizeof(unsigned long long) * F, cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  for (int f : act) memcpy(&out[f], &bits[f], sizeof(double));
  return bxh::check_launch("banded hotelling-bodewig residual");
}

int hb_band_factor_planes(const double *mu, const double *l1, const double *l2, const double *phi,
                          const double *psi, double *fac, int64_t batch, int64_t n, int64_t ld,
                          int layout, cudaStream_t st) {
  const unsigned g = hbb::blocks(batch * n);
  if (layout == BX_LAYOUT_INTERLEAVED)
    hbb::factors_to_planes_kernel<<<g, 256, 0, st>>>(mu, l1, l2, phi, psi, fac, batch, n,
                                                     Interleaved{ld});
  else
    hbb::factors_to_planes_kernel<<<g, 256, 0, st>>>(mu, l1, l2, phi, psi, fac, batch, n,
                                                     SystemMajor{ld});
  return BX_OK;
}

int hb_band_apply(const double *X, const int64_t *wf, const double *v, double *out, const int *act,
                  int nact, int64_t batch, int64_t n, int64_t cap, int upper, cudaStream_t st) {
  hbb::band_apply_kernel<<<hbb::blocks((int64_t)nact * n), 256, 0, st>>>(X, wf, v, out, act, nact,
                                                                         batch, n, cap, upper);
  return BX_OK;
}

}  // namespace bx

namespace bx {

// ---------------------------------------------------------------------------
// hb_invert_banded entry (factors given): one side of every system
// ---------------------------------------------------------------------------
namespace hbb {
struct BandWs {
  double *fac, *X, *Xn, *P, *Best;
  int *act, *zero;
  unsigned long long *rbits;
};
inline char *align256(char *p) { return (char *)(((uintptr_t)p + 255) & ~(uintptr_t)255); }
// fac_bytes: the factor planes in front; then 4 band buffers for 2*batch
// factors of cap+1 diagonals; ints and residual bits
inline BandWs carve_band(void *ws, size_t fac_bytes, int64_t batch, int64_t n, int64_t cap) {
  char *p = (char *)ws;
  BandWs w;
  w.fac = (double *)p;
  p = align256(p + fac_bytes);
  const size_t band = sizeof(double) * (size_t)(2 * batch) * (size_t)(cap + 1) * (size_t)n;
  w.X = (double *)p; p = align256(p + band);
  w.Xn = (double *)p; p = align256(p + band);
  w.P = (double *)p; p = align256(p + band);
  w.Best = (double *)p; p = align256(p + band);
  w.act = (int *)p; p += sizeof(int) * 2 * batch;
  w.zero = (int *)p; p += sizeof(int) * 2 * batch;
  w.rbits = (unsigned long long *)align256(p);
  return w;
}
inline size_t band_ws_bytes(size_t fac_bytes, int64_t batch, int64_t n, int64_t cap) {
  return fac_bytes + 4 * (sizeof(double) * (size_t)(2 * batch) * (size_t)(cap + 1) * (size_t)n) +
         sizeof(int) * 4 * (size_t)batch + sizeof(unsigned long long) * 2 * (size_t)batch +
         8 * 256;
}
}  // namespace hbb

size_t hb_band_invert_workspace_bytes(int64_t batch, int64_t n, int64_t w) {
  return hbb::band_ws_bytes(sizeof(double) * 5 * (size_t)batch * (size_t)n, batch, n, w);
}

int hb_band_invert(const double *mu, const double *l1, const double *l2, const double *phi,
                   const double *psi, int side, int64_t w, const double *tol, int64_t max_iter,
                   double *xdiags, int64_t *iterations, double *residual, double *history,
                   int32_t *status, int32_t *index, int64_t batch, int64_t n, int64_t ld,
                   int layout, void *workspace, cudaStream_t st) {
  hbb::BandWs ws = hbb::carve_band(workspace, sizeof(double) * 5 * (size_t)batch * (size_t)n,
                                   batch, n, w);
  hb_band_factor_planes(mu, l1, l2, phi, psi, ws.fac, batch, n, ld, layout, st);
  const int F = (int)(2 * batch);
  std::vector<double> tolh(batch), tolf(F, 0.0);
  cudaMemcpyAsync(tolh.data(), tol, sizeof(double) * batch, cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  std::vector<int> act;
  for (int64_t s = 0; s < batch; ++s) {
    const int f = (int)(side ? batch + s : s);
    act.push_back(f);
    tolf[f] = tolh[s];
  }
  std::vector<int64_t> it(F, 0);
  std::vector<double> rs(F, NAN);
  std::vector<int> stf(F, BX_STATUS_OK), zr(F, -1);
  std::vector<std::vector<double>> hist(F);
  int rc = hb_band_invert_round(ws.fac, ws.X, ws.Xn, ws.P, ws.Best, ws.act, ws.zero, ws.rbits, act,
                                tolf.data(), batch, n, w, w, max_iter, it.data(), rs.data(),
                                stf.data(), zr.data(), &hist, st);
  if (rc) return rc;
  const int f0 = side ? (int)batch : 0;
  if (xdiags)
    cudaMemcpyAsync(xdiags, ws.X + (size_t)f0 * (w + 1) * n,
                    sizeof(double) * (size_t)batch * (w + 1) * n, cudaMemcpyDeviceToDevice, st);
  std::vector<int32_t> so(batch), io(batch);
  for (int64_t s = 0; s < batch; ++s) {
    so[s] = stf[f0 + s];
    io[s] = so[s] == BX_STATUS_ZERO_DIAG ? zr[f0 + s] : -1;
  }
  if (iterations) cudaMemcpyAsync(iterations, it.data() + f0, sizeof(int64_t) * batch, cudaMemcpyHostToDevice, st);
  if (residual) cudaMemcpyAsync(residual, rs.data() + f0, sizeof(double) * batch, cudaMemcpyHostToDevice, st);
  if (status) cudaMemcpyAsync(status, so.data(), sizeof(int32_t) * batch, cudaMemcpyHostToDevice, st);
  if (index) cudaMemcpyAsync(index, io.data(), sizeof(int32_t) * batch, cudaMemcpyHostToDevice, st);
  if (history) {
    std::vector<double> h((size_t)batch * (max_iter + 1), NAN);
    for (int64_t s = 0; s < batch; ++s)
      for (size_t j = 0; j < hist[f0 + s].size(); ++j) h[(size_t)s * (max_iter + 1) + j] = hist[f0 + s][j];
    cudaMemcpyAsync(history, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice, st);
  }
  cudaStreamSynchronize(st);
  return bxh::check_launch("bx_hb_invert_banded_f64");
}

}  // namespace bx
