// ILU(0) / Stone factorisation, defect matrix and the strongly implicit
// procedure (SIP, Algorithm 1 of the paper), sequential-per-system kernels.
//
// Reference: iterative.py (bandix 0.1.0)
//   ilu0_penta          62-124   (pattern-restricted ILU(0), modified Doolittle)
//   _factor_product_diagonals / defect_matrix  152-200   (K = L U - A)
//   _sweep_apply        203-236   (A x as accumulating diagonal sweeps from 0)
//   forward_sub / backward_sub   127-149  (penta_forward/backward, _elim.py:65-87)
//   sip_solve           255-308   (the iteration with best-iterate tracking,
//                                   MaxIterationsExceeded and Diverged)
// generalised to an outer offset m (row-aligned diagonals subm[i] = A[i,i-m],
// supm[i] = A[i,i+m]); m = 2 is the reference bit-for-bit, m >= 3 adds the
// fill diagonals +-(m-1) to K and Stone's alpha (oracle/iterative.py states
// the same recurrences).  One thread per system, every operation rounded once
// (bx::mul/sub/add/dvd), so results are bit-identical to the oracle.
//
// The grid-structured fast path (anti-diagonal wavefront, one CTA per system)
// is bx_sip_wave.cu.
#include <math.h>

#include "bx_common.cuh"
#include "bx_kernels.h"

namespace bx {
namespace sip {

constexpr int kThreads = 32;

// scratch planes (interleaved [n][batch]) used by the sequential SIP
enum Plane { MU = 0, L1, L2, PHI, PSI, KM, K1N, K0, K1P, KP, KQN, KQP, YV, XB, kPlanes };

struct Planes {
  double *base;
  int64_t batch, n;
  __device__ __forceinline__ double *operator()(int p) const { return base + (int64_t)p * batch * n; }
};

// ---------------------------------------------------------------------------
// ILU(0) (m == 2: iterative.py:80-114 verbatim) / Stone with alpha (m >= 3)
// ---------------------------------------------------------------------------
template <class Lay>
__device__ bool ilu0_one(const double *a2p, const double *a1p, const double *ep,
                         const double *c1p, const double *c2p, Planes P, int64_t s, int64_t n,
                         int64_t m, double alpha, Lay lay, int32_t *bad_row) {
  const Scratch ws{P.batch};
  double *mu = P(MU), *fl1 = P(L1), *fl2 = P(L2), *phi = P(PHI), *psi = P(PSI);
  double mu1 = 0.0, phi1 = 0.0, psi1 = 0.0;  // row i-1
  for (int64_t i = 0; i < n; ++i) {
    const double a2 = i >= m ? ldg(a2p + lay(i, s)) : 0.0;
    const double a1 = i >= 1 ? ldg(a1p + lay(i, s)) : 0.0;
    const double e = ldg(ep + lay(i, s));
    const bool has2 = i >= m && a2 != 0.0;
    const bool has1 = i >= 1 && a1 != 0.0;
    double li2 = 0.0, li1 = 0.0, mi, ph = 0.0, ps = 0.0;
    if (m == 2) {
      const double mum = i >= 2 ? mu[ws(i - 2, s)] : 0.0;
      const double phm = i >= 2 ? phi[ws(i - 2, s)] : 0.0;
      const double psm = i >= 2 ? psi[ws(i - 2, s)] : 0.0;
      if (has2) li2 = dvd(a2, mum);
      if (has1) {
        double t = a1;
        if (has2) t = sub(t, mul(li2, phm));
        li1 = dvd(t, mu1);
      }
      mi = e;
      if (has2) mi = sub(mi, mul(li2, psm));
      if (has1) mi = sub(mi, mul(li1, phi1));
      if (i <= n - 2) {
        double fi = ldg(c1p + lay(i, s));
        if (fi != 0.0 && has1) fi = sub(fi, mul(li1, psi1));
        ph = fi;
      }
      ps = i <= n - 3 ? ldg(c2p + lay(i, s)) : 0.0;
    } else {
      const double mum = i >= m ? mu[ws(i - m, s)] : 0.0;
      const double phm = i >= m ? phi[ws(i - m, s)] : 0.0;
      const double psm = i >= m ? psi[ws(i - m, s)] : 0.0;
      if (has2) li2 = dvd(a2, alpha == 0.0 ? mum : add(mum, mul(alpha, phm)));
      if (has1) li1 = dvd(a1, alpha == 0.0 ? mu1 : add(mu1, mul(alpha, psi1)));
      mi = e;
      if (has2) mi = sub(mi, mul(li2, psm));
      if (has1) mi = sub(mi, mul(li1, phi1));
      if (alpha != 0.0) {
        double comp = 0.0;
        if (has2) comp = add(comp, mul(li2, phm));
        if (has1) comp = add(comp, mul(li1, psi1));
        mi = add(mi, mul(alpha, comp));
      }
      if (i <= n - 2) {
        double fi = ldg(c1p + lay(i, s));
        if (alpha != 0.0 && fi != 0.0 && has2) fi = sub(fi, mul(alpha, mul(li2, phm)));
        ph = fi;
      }
      if (i <= n - m - 1) {
        double gi = ldg(c2p + lay(i, s));
        if (alpha != 0.0 && gi != 0.0 && has1) gi = sub(gi, mul(alpha, mul(li1, psi1)));
        ps = gi;
      }
    }
    if (mi == 0.0) {
      *bad_row = (int32_t)i;
      return false;
    }
    mu[ws(i, s)] = mi;
    fl1[ws(i, s)] = has1 ? li1 : 0.0;
    fl2[ws(i, s)] = has2 ? li2 : 0.0;
    phi[ws(i, s)] = ph;
    psi[ws(i, s)] = ps;
    mu1 = mi; phi1 = ph; psi1 = ps;
  }
  return true;
}

// K = L U - A  (iterative.py:152-200; m >= 3 adds the +-(m-1) fill)
template <class Lay>
__device__ void defect_one(const double *a2p, const double *a1p, const double *ep,
                           const double *c1p, const double *c2p, Planes P, int64_t s, int64_t n,
                           int64_t m, Lay lay) {
  const Scratch ws{P.batch};
  const double *mu = P(MU), *l1 = P(L1), *l2 = P(L2), *phi = P(PHI), *psi = P(PSI);
  for (int64_t i = 0; i < n; ++i) {
    const double l1i = l1[ws(i, s)], l2i = l2[ws(i, s)], mui = mu[ws(i, s)];
    double pm = i >= m ? mul(l2i, mu[ws(i - m, s)]) : 0.0;
    double p_1 = i >= 1 ? mul(l1i, mu[ws(i - 1, s)]) : 0.0;
    if (m == 2 && i >= 2) p_1 = add(p_1, mul(l2i, phi[ws(i - 2, s)]));
    double p0 = mui;
    if (i >= 1) p0 = add(p0, mul(l1i, phi[ws(i - 1, s)]));
    if (i >= m) p0 = add(p0, mul(l2i, psi[ws(i - m, s)]));
    double p1 = i <= n - 2 ? phi[ws(i, s)] : 0.0;
    if (m == 2 && i >= 1 && i <= n - 2) p1 = add(p1, mul(l1i, psi[ws(i - 1, s)]));
    const double pp = i <= n - m - 1 ? psi[ws(i, s)] : 0.0;
    P(KM)[ws(i, s)] = sub(pm, i >= m ? ldg(a2p + lay(i, s)) : 0.0);
    P(K1N)[ws(i, s)] = sub(p_1, i >= 1 ? ldg(a1p + lay(i, s)) : 0.0);
    P(K0)[ws(i, s)] = sub(p0, ldg(ep + lay(i, s)));
    P(K1P)[ws(i, s)] = sub(p1, i <= n - 2 ? ldg(c1p + lay(i, s)) : 0.0);
    P(KP)[ws(i, s)] = sub(pp, i <= n - m - 1 ? ldg(c2p + lay(i, s)) : 0.0);
    if (m != 2) {
      P(KQN)[ws(i, s)] = i >= m ? mul(l2i, phi[ws(i - m, s)]) : 0.0;
      P(KQP)[ws(i, s)] = (i >= 1 && i <= n - m) ? mul(l1i, psi[ws(i - 1, s)]) : 0.0;
    }
  }
}

// acc from 0: main, -1, +1, -m, +m [, -(m-1), +(m-1)]  (iterative.py:213-221)
template <class XL, class DL>
__device__ __forceinline__ double sweep_row(const double *d0, const double *dn1, const double *dp1,
                                            const double *dnm, const double *dpm,
                                            const double *dnq, const double *dpq, DL dl,
                                            const double *x, XL xl, int64_t i, int64_t s,
                                            int64_t n, int64_t m) {
  double acc = add(0.0, mul(d0[dl(i, s)], x[xl(i, s)]));
  if (i >= 1) acc = add(acc, mul(dn1[dl(i, s)], x[xl(i - 1, s)]));
  if (i <= n - 2) acc = add(acc, mul(dp1[dl(i, s)], x[xl(i + 1, s)]));
  if (i >= m) acc = add(acc, mul(dnm[dl(i, s)], x[xl(i - m, s)]));
  if (i + m <= n - 1) acc = add(acc, mul(dpm[dl(i, s)], x[xl(i + m, s)]));
  if (dnq) {
    const int64_t q = m - 1;
    if (i >= q) acc = add(acc, mul(dnq[dl(i, s)], x[xl(i - q, s)]));
    if (i + q <= n - 1) acc = add(acc, mul(dpq[dl(i, s)], x[xl(i + q, s)]));
  }
  return acc;
}

template <class Lay>
__device__ double residual_norm(const double *a2p, const double *a1p, const double *ep,
                                const double *c1p, const double *c2p, const double *bp,
                                const double *x, Scratch xl, int64_t s, int64_t n, int64_t m,
                                Lay lay) {
  double r = 0.0;
  bool nan = false;
  for (int64_t i = 0; i < n; ++i) {
    const double ax = sweep_row(ep, a1p, c1p, a2p, c2p, (const double *)nullptr,
                                (const double *)nullptr, lay, x, xl, i, s, n, m);
    const double v = fabs(sub(ldg(bp + lay(i, s)), ax));
    nan |= v != v;
    r = v > r ? v : r;
  }
  return nan ? __longlong_as_double(0x7ff8000000000000LL) : r;
}

template <class Lay>
__global__ void __launch_bounds__(kThreads)
sip_seq_kernel(const double *__restrict__ a2p, const double *__restrict__ a1p,
               const double *__restrict__ ep, const double *__restrict__ c1p,
               const double *__restrict__ c2p, const double *__restrict__ bp,
               const double *__restrict__ tol, double *__restrict__ xout,
               double *__restrict__ best_x, int64_t *iters, double *res, double *best_res,
               int32_t *status, int32_t *index, double *history, Planes P, int64_t batch,
               int64_t n, int64_t m, double alpha, int64_t max_iter, int use_x0, Lay lay,
               int factor_only) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= batch) return;
  const Scratch ws{batch};
  int32_t bad = -1;
  if (!ilu0_one(a2p, a1p, ep, c1p, c2p, P, s, n, m, alpha, lay, &bad)) {
    set_status(status, index, s, BX_STATUS_ZERO_PIVOT, bad);
    if (iters) iters[s] = 0;
    return;
  }
  defect_one(a2p, a1p, ep, c1p, c2p, P, s, n, m, lay);
  if (factor_only) {
    set_status(status, index, s, BX_STATUS_OK, -1);
    return;
  }
  const double *mu = P(MU), *l1 = P(L1), *l2 = P(L2), *phi = P(PHI), *psi = P(PSI);
  const double *kq_n = m != 2 ? P(KQN) : nullptr, *kq_p = m != 2 ? P(KQP) : nullptr;
  double *y = P(YV);
  // ping-pong iterates in scratch: plane XB and the plane after the last one
  double *X[2] = {P(XB) + batch * n, P(XB)};
  for (int64_t i = 0; i < n; ++i) X[0][ws(i, s)] = use_x0 ? xout[lay(i, s)] : 0.0;
  int cur = 0;
  int best_loc = 0;  // 0/1: ping-pong buffer holding the best iterate; 2: best_x
  double r = residual_norm(a2p, a1p, ep, c1p, c2p, bp, X[0], ws, s, n, m, lay);
  const double r0 = r;
  double best = r;
  int64_t k = 0;
  int32_t st = BX_STATUS_OK;
  const double tl = tol[s];
  while (r >= tl) {
    if (k >= max_iter) { st = BX_STATUS_MAX_ITER; break; }
    const int nxt = cur ^ 1;
    if (best_loc == nxt) {  // about to overwrite the best iterate: keep it
      if (best_x)
        for (int64_t i = 0; i < n; ++i) best_x[lay(i, s)] = X[nxt][ws(i, s)];
      best_loc = 2;
    }
    const double *xo = X[cur];
    double *xn = X[nxt];
    // newRHS = K x + b ; forward substitution (iterative.py:293-294)
    double y1 = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      const double kx = sweep_row(P(K0), P(K1N), P(K1P), P(KM), P(KP), kq_n, kq_p, ws, xo, ws, i,
                                  s, n, m);
      const double v = add(kx, ldg(bp + lay(i, s)));
      double t = i >= 1 ? sub(v, mul(l1[ws(i, s)], y1)) : v;
      if (i >= m) t = sub(t, mul(l2[ws(i, s)], y[ws(i - m, s)]));
      y[ws(i, s)] = t;
      y1 = t;
    }
    // backward substitution (iterative.py:295)
    double x1 = 0.0;
    for (int64_t i = n - 1; i >= 0; --i) {
      double t = y[ws(i, s)];
      if (i <= n - 2) t = sub(t, mul(phi[ws(i, s)], x1));
      if (i + m <= n - 1) t = sub(t, mul(psi[ws(i, s)], xn[ws(i + m, s)]));
      x1 = dvd(t, mu[ws(i, s)]);
      xn[ws(i, s)] = x1;
    }
    // recomputed residual (iterative.py:296-297)
    r = residual_norm(a2p, a1p, ep, c1p, c2p, bp, xn, ws, s, n, m, lay);
    cur = nxt;
    ++k;
    if (history) history[s * max_iter + (k - 1)] = r;
    if (r < best) { best = r; best_loc = cur; }
    if (r0 > 0 && r > 1e6 * r0) { st = BX_STATUS_DIVERGED; break; }
  }
  for (int64_t i = 0; i < n; ++i) xout[lay(i, s)] = X[cur][ws(i, s)];
  if (best_x && best_loc != 2)
    for (int64_t i = 0; i < n; ++i) best_x[lay(i, s)] = X[best_loc][ws(i, s)];
  if (iters) iters[s] = k;
  if (res) res[s] = r;
  if (best_res) best_res[s] = best;
  set_status(status, index, s, st, -1);
}

// copy the factor / defect planes out in the caller's layout (row-aligned);
// the 12 output pointers travel by value as a kernel parameter (no device
// staging buffer, no copies, no stream synchronisation)
struct ExportArgs {
  double *outs[12];
  int which[12];
};

template <class Lay>
__global__ void export_planes_kernel(Planes P, const ExportArgs args, int64_t batch, int64_t n,
                                     Lay lay) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= batch * n) return;
  const int64_t i = idx / batch, s = idx % batch;
#pragma unroll
  for (int c = 0; c < 12; ++c)
    if (args.outs[c]) args.outs[c][lay(i, s)] = P(args.which[c])[i * batch + s];
}

}  // namespace sip

size_t sip_workspace_bytes(int64_t batch, int64_t n) {
  return sizeof(double) * (size_t)batch * (size_t)n * (sip::kPlanes + 1);
}

template <class Lay>
static void launch_sip(const double *a2, const double *a1, const double *e, const double *c1,
                       const double *c2, const double *b, const double *tol, double *x,
                       double *best_x, int64_t *iters, double *res, double *best_res,
                       int32_t *st, int32_t *ix, double *hist, double *ws, int64_t batch,
                       int64_t n, int64_t m, double alpha, int64_t max_iter, int use_x0, Lay lay,
                       int factor_only, cudaStream_t stream) {
  sip::Planes P{ws, batch, n};
  const dim3 grid((unsigned)((batch + sip::kThreads - 1) / sip::kThreads));
  sip::sip_seq_kernel<Lay><<<grid, sip::kThreads, 0, stream>>>(
      a2, a1, e, c1, c2, b, tol, x, best_x, iters, res, best_res, st, ix, hist, P, batch, n, m,
      alpha, max_iter, use_x0, lay, factor_only);
}

int sip_seq(const double *a2, const double *a1, const double *e, const double *c1,
            const double *c2, const double *b, const double *tol, double *x, double *best_x,
            int64_t *iters, double *res, double *best_res, int32_t *st, int32_t *ix,
            double *hist, double *ws, int64_t batch, int64_t n, int64_t m, double alpha,
            int64_t max_iter, int use_x0, int64_t ld, int layout, int factor_only,
            cudaStream_t stream) {
  if (layout == BX_LAYOUT_INTERLEAVED)
    launch_sip(a2, a1, e, c1, c2, b, tol, x, best_x, iters, res, best_res, st, ix, hist, ws,
               batch, n, m, alpha, max_iter, use_x0, Interleaved{ld}, factor_only, stream);
  else
    launch_sip(a2, a1, e, c1, c2, b, tol, x, best_x, iters, res, best_res, st, ix, hist, ws,
               batch, n, m, alpha, max_iter, use_x0, SystemMajor{ld}, factor_only, stream);
  return BX_OK;
}

// factors (mu, l1, l2, phi, psi) and defect diagonals (K_{-m}, K_{-1}, K_0,
// K_{+1}, K_{+m}, K_{-(m-1)}, K_{+(m-1)}) -> caller arrays (NULL skips)
int sip_export(double *ws, int64_t batch, int64_t n, double *const *outs12, int64_t ld,
               int layout, cudaStream_t stream) {
  static const int which[12] = {sip::MU, sip::L1, sip::L2, sip::PHI, sip::PSI, sip::KM,
                                sip::K1N, sip::K0, sip::K1P, sip::KP, sip::KQN, sip::KQP};
  sip::ExportArgs args;
  for (int c = 0; c < 12; ++c) {
    args.outs[c] = outs12[c];
    args.which[c] = which[c];
  }
  sip::Planes P{ws, batch, n};
  const int64_t tot = batch * n;
  const dim3 grid((unsigned)((tot + 255) / 256));
  if (layout == BX_LAYOUT_INTERLEAVED)
    sip::export_planes_kernel<<<grid, 256, 0, stream>>>(P, args, batch, n, Interleaved{ld});
  else
    sip::export_planes_kernel<<<grid, 256, 0, stream>>>(P, args, batch, n, SystemMajor{ld});
  return bxh::check_launch("bx_ilu0_f64 export");
}

}  // namespace bx
