// SIP on grid-structured systems: anti-diagonal wavefront, one CTA per system.
//
// A stride-m five-point band whose +-1 couplings never cross a grid row
// (A[i,i-1] = 0 when i % m == 0, A[i,i+1] = 0 when i % m == m-1) is the
// natural ordering of an (n/m) x m grid: row i is cell (p, q) = (i / m, i % m).
// Every recurrence of ILU(0) and of the triangular solves then only reaches
// (p, q-1) and (p-1, q) (forward) or (p, q+1) and (p+1, q) (backward), so all
// cells of an anti-diagonal t = p + q are independent.  Thread q of the CTA
// owns grid column q; the CTA walks t = 0 .. R+m-2 (R = n/m rows) with one
// barrier per step, exchanging the neighbouring column's value through shared
// memory.  Every cell executes exactly the operation sequence of the
// sequential kernel (bx_sip.cu) / the oracle, so iterates, residuals and
// iteration counts are the same bits; the only difference is that products
// with a structurally zero coefficient that would reach across a grid row are
// skipped, which can change the sign of an exactly-zero intermediate and
// nothing else.
//
// Storage is "skewed" per system: plane[t][q] = value of cell (t-q, q), so at
// every step the CTA reads and writes one contiguous row of m doubles per
// plane (coalesced).  A, b, the factors, the defect K and the iterates are
// converted once in the setup pass; iterations then stream the planes.
//   reference: ilu0_penta / defect_matrix / sip_solve (iterative.py:62-308)
#include <math.h>

#include "bx_common.cuh"
#include "bx_kernels.h"

namespace bx {
namespace sipw {

enum Plane {
  PA2 = 0, PA1, PE, PC1, PC2, PB,   // A and b
  PL1, PL2, PMU, PPHI, PPSI,        // factors
  PK0, PKN1, PKP1, PKNM, PKPM, PKNQ, PKPQ,  // defect, sweep order
  PY, PXA, PXB, PXBEST, kPlanes
};

struct Skew {
  double *ws;
  int64_t batch, m, T, mp;  // T = R + m - 1 slices; mp = row stride (m rounded up to even)
  __device__ __forceinline__ double *at(int p, int64_t s, int64_t t) const {
    return ws + (((int64_t)p * batch + s) * T + t) * mp;
  }
};

// ---- TMA bulk copies into a shared-memory ring, completion on mbarriers ----
__device__ __forceinline__ unsigned smem_u32(const void *p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ double nan_max(double a, double b) {
  if (a != a || b != b) return __longlong_as_double(0x7ff8000000000000LL);
  return a > b ? a : b;
}

constexpr int NPL = 11;  // plane rows per ring stage

template <class Lay>
__global__ void __launch_bounds__(512) sip_wave_kernel(const double *__restrict__ a2p, const double *__restrict__ a1p,
                                const double *__restrict__ ep, const double *__restrict__ c1p,
                                const double *__restrict__ c2p, const double *__restrict__ bp,
                                const double *__restrict__ tol, double *__restrict__ xout,
                                double *__restrict__ best_x, int64_t *iters, double *res,
                                double *best_res, int32_t *status, int32_t *index,
                                double *history, Skew S, int64_t n, double alpha,
                                int64_t max_iter, int use_x0, Lay lay, int nst) {
  extern __shared__ double sh[];
  const int64_t m = S.m, R = n / m, T = S.T;
  const int q = threadIdx.x;
  const int64_t s = blockIdx.x;
  __shared__ int s_bad, s_notgrid, s_go, s_bestcopy;
  __shared__ double s_red[32];
  if (q == 0) { s_bad = 0x7fffffff; s_notgrid = 0; }
  __syncthreads();

  // ---------------- setup: skew A, b, x0; ILU(0)/Stone; defect ------------
  {
    double *smu = sh, *sphi = sh + 3 * m, *spsi = sh + 6 * m;
    double mu_u = 0, phi_u = 0, psi_u = 0;  // own column, previous cell (p-1, q)
    for (int64_t t = 0; t < T; ++t) {
      const int64_t p = t - q;
      const bool valid = p >= 0 && p < R;
      if (valid) {
        const int64_t i = p * m + q;
        const double a2 = i >= m ? ldg(a2p + lay(i, s)) : 0.0;
        const double a1 = i >= 1 ? ldg(a1p + lay(i, s)) : 0.0;
        const double e = ldg(ep + lay(i, s));
        const double c1 = i <= n - 2 ? ldg(c1p + lay(i, s)) : 0.0;
        const double c2 = i <= n - m - 1 ? ldg(c2p + lay(i, s)) : 0.0;
        if ((q == 0 && a1 != 0.0) || (q == m - 1 && c1 != 0.0)) s_notgrid = 1;
        const int sl = (int)((t + 2) % 3);  // slot of step t-1
        const double mu_l = q >= 1 ? smu[sl * m + q - 1] : 0.0;
        const double phi_l = q >= 1 ? sphi[sl * m + q - 1] : 0.0;
        const double psi_l = q >= 1 ? spsi[sl * m + q - 1] : 0.0;
        const bool has2 = i >= m && a2 != 0.0;
        const bool has1 = i >= 1 && a1 != 0.0;  // implies q >= 1 on a grid
        double li2 = 0.0, li1 = 0.0, mi, ph = 0.0, ps = 0.0;
        if (m == 2) {
          if (has2) li2 = dvd(a2, mu_u);
          if (has1) {
            double tt = a1;
            if (has2) tt = sub(tt, mul(li2, phi_u));
            li1 = dvd(tt, mu_l);
          }
          mi = e;
          if (has2) mi = sub(mi, mul(li2, psi_u));
          if (has1) mi = sub(mi, mul(li1, phi_l));
          if (i <= n - 2) {
            double fi = c1;
            if (fi != 0.0 && has1) fi = sub(fi, mul(li1, psi_l));
            ph = fi;
          }
          ps = i <= n - 3 ? c2 : 0.0;
        } else {
          if (has2) li2 = dvd(a2, alpha == 0.0 ? mu_u : add(mu_u, mul(alpha, phi_u)));
          if (has1) li1 = dvd(a1, alpha == 0.0 ? mu_l : add(mu_l, mul(alpha, psi_l)));
          mi = e;
          if (has2) mi = sub(mi, mul(li2, psi_u));
          if (has1) mi = sub(mi, mul(li1, phi_l));
          if (alpha != 0.0) {
            double comp = 0.0;
            if (has2) comp = add(comp, mul(li2, phi_u));
            if (has1) comp = add(comp, mul(li1, psi_l));
            mi = add(mi, mul(alpha, comp));
          }
          if (i <= n - 2) {
            double fi = c1;
            if (alpha != 0.0 && fi != 0.0 && has2) fi = sub(fi, mul(alpha, mul(li2, phi_u)));
            ph = fi;
          }
          if (i <= n - m - 1) {
            double gi = c2;
            if (alpha != 0.0 && gi != 0.0 && has1) gi = sub(gi, mul(alpha, mul(li1, psi_l)));
            ps = gi;
          }
        }
        if (mi == 0.0) atomicMin(&s_bad, (int)i);
        const double l1 = has1 ? li1 : 0.0, l2 = has2 ? li2 : 0.0;
        // defect K = LU - A (iterative.py:152-200); cross-row products are
        // structural zeros and are skipped
        double pm = i >= m ? mul(l2, mu_u) : 0.0;
        double p_1 = (i >= 1 && q >= 1) ? mul(l1, mu_l) : 0.0;
        if (m == 2 && i >= 2) p_1 = add(p_1, mul(l2, phi_u));
        double p0 = mi;
        if (i >= 1 && q >= 1) p0 = add(p0, mul(l1, phi_l));
        if (i >= m) p0 = add(p0, mul(l2, psi_u));
        double p1 = i <= n - 2 ? ph : 0.0;
        if (m == 2 && i >= 1 && i <= n - 2 && q >= 1) p1 = add(p1, mul(l1, psi_l));
        const double pp = i <= n - m - 1 ? ps : 0.0;
        *(S.at(PKNM, s, t) + q) = sub(pm, i >= m ? a2 : 0.0);
        *(S.at(PKN1, s, t) + q) = sub(p_1, i >= 1 ? a1 : 0.0);
        *(S.at(PK0, s, t) + q) = sub(p0, e);
        *(S.at(PKP1, s, t) + q) = sub(p1, i <= n - 2 ? c1 : 0.0);
        *(S.at(PKPM, s, t) + q) = sub(pp, i <= n - m - 1 ? c2 : 0.0);
        if (m != 2) {
          *(S.at(PKNQ, s, t) + q) = i >= m ? mul(l2, phi_u) : 0.0;
          *(S.at(PKPQ, s, t) + q) = (i >= 1 && i <= n - m && q >= 1) ? mul(l1, psi_l) : 0.0;
        }
        *(S.at(PA2, s, t) + q) = a2;
        *(S.at(PA1, s, t) + q) = a1;
        *(S.at(PE, s, t) + q) = e;
        *(S.at(PC1, s, t) + q) = c1;
        *(S.at(PC2, s, t) + q) = c2;
        *(S.at(PB, s, t) + q) = ldg(bp + lay(i, s));
        *(S.at(PL1, s, t) + q) = l1;
        *(S.at(PL2, s, t) + q) = l2;
        *(S.at(PMU, s, t) + q) = mi;
        *(S.at(PPHI, s, t) + q) = ph;
        *(S.at(PPSI, s, t) + q) = ps;
        *(S.at(PXA, s, t) + q) = use_x0 ? xout[lay(i, s)] : 0.0;
        const int ws_ = (int)(t % 3);
        smu[ws_ * m + q] = mi;
        sphi[ws_ * m + q] = ph;
        spsi[ws_ * m + q] = ps;
        mu_u = mi; phi_u = ph; psi_u = ps;
      }
      __syncthreads();
    }
  }
  if (s_notgrid || s_bad != 0x7fffffff) {
    if (q == 0) {
      if (s_notgrid) set_status(status, index, s, BX_STATUS_NOT_GRID, -1);
      else set_status(status, index, s, BX_STATUS_ZERO_PIVOT, s_bad);
      if (iters) iters[s] = 0;
    }
    return;
  }

  double *xs = sh;          // [4][m] window of the previous iterate
  double *ys = sh + 4 * m;  // [3][m]
  double *xn = sh + 7 * m;  // [4][m] window of the new iterate
  // ring of NST stages x NPL plane rows (padded stride mp), filled by TMA bulk copies
  const int64_t mp = S.mp;
  double *ring = sh + 11 * m + (11 * m & 1);
  uint64_t *bars = reinterpret_cast<uint64_t *>(ring + (int64_t)nst * NPL * mp);
  auto R_ = [&](int stage, int j) { return ring + ((int64_t)stage * NPL + j) * mp; };
  auto valid_cell = [&](int64_t t) { const int64_t p = t - q; return p >= 0 && p < R; };
  if (q == 0)
    for (int i = 0; i < nst; ++i) mbar_init(bars + i);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.global;" ::: "memory");  // setup's plane writes -> TMA reads
  __syncthreads();
  // ring bookkeeping (identical in every thread): stage index + phase parity
  int i_stg = 0, u_stg = 0;
  unsigned u_par = 0;
  const int lane = q & 31;
  const int width = m < 32 ? (int)m : 32;  // lanes present in warp 0
  const unsigned wmask = width == 32 ? 0xffffffffu : ((1u << width) - 1u);
  // per phase, lane j of warp 0 owns plane row j: base pointer, slice offset, ring slot
  const double *my_base = nullptr;
  const int *rw_planes = nullptr, *rw_offs = nullptr;
  int my_off = 0, my_cnt = 0;
  auto set_rows = [&](const int *planes, const int *offs, int cnt) {
    my_cnt = cnt;
    rw_planes = planes;
    rw_offs = offs;
    if (lane < cnt) { my_base = S.at(planes[lane], s, 0); my_off = offs[lane]; }
  };
  // valid columns of slice u, widened to 16-byte alignment: [a0, a0 + nb/8)
  auto span = [&](int u, int &a0, unsigned &nb) {
    nb = 0;
    a0 = 0;
    if (u >= 0 && u < (int)T) {
      const int qlo = u - (int)R + 1 > 0 ? u - (int)R + 1 : 0, qhi = u < (int)m - 1 ? u : (int)m - 1;
      if (qlo <= qhi) {
        a0 = qlo & ~1;
        nb = (unsigned)(((qhi + 2) & ~1) - a0) * (unsigned)sizeof(double);
      }
    }
  };
  // warp 0: queue the rows of step slice tb (row j uses slice tb + off_j)
  auto issue = [&](int tb) {
    if (width >= my_cnt) {  // one row per lane
      unsigned nb = 0;
      int a0 = 0;
      if (lane < my_cnt) span(tb + my_off, a0, nb);
      const unsigned bytes = __reduce_add_sync(wmask, nb);
      if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect(bars + i_stg, bytes);
      }
      __syncwarp(wmask);
      if (nb)
        bulk_g2s(R_(i_stg, lane) + a0, my_base + (int64_t)(tb + my_off) * mp + a0, nb, bars + i_stg);
    } else {  // narrow grids (m < rows per step): lanes loop over rows
      unsigned bytes = 0, nb;
      int a0;
      for (int j = 0; j < my_cnt; ++j) {
        span(tb + rw_offs[j], a0, nb);
        bytes += nb;
      }
      if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect(bars + i_stg, bytes);
      }
      __syncwarp(wmask);
      for (int j = lane; j < my_cnt; j += width) {
        const int u = tb + rw_offs[j];
        span(u, a0, nb);
        if (nb) bulk_g2s(R_(i_stg, j) + a0, S.at(rw_planes[j], s, u) + a0, nb, bars + i_stg);
      }
    }
    i_stg = i_stg + 1 == nst ? 0 : i_stg + 1;
  };
  auto wait_stage = [&]() -> int {
    const int stg = u_stg;
    mbar_wait(bars + stg, u_par);
    if (++u_stg == nst) { u_stg = 0; u_par ^= 1u; }
    return stg;
  };

  // residual of cell (slice tt, column q) from a window w[4][m] of x slices
  // tt-1..tt+1 and the row's A/b values (iterative.py:213-221 order, acc from 0)
  auto residual_from = [&](const double *w, int64_t tt, double a2, double a1, double e,
                           double c1, double c2, double bb) -> double {
    const int64_t p = tt - q, i = p * m + q;
    auto X = [&](int64_t sl, int col) { return w[(int)(((sl % 4) + 4) % 4) * m + col]; };
    double acc = add(0.0, mul(e, X(tt, q)));
    if (i >= 1) {
      if (q >= 1) acc = add(acc, mul(a1, X(tt - 1, q - 1)));
      else if (m == 2) acc = add(acc, mul(a1, X(tt, q + 1)));
    }
    if (i <= n - 2) {
      if (q <= m - 2) acc = add(acc, mul(c1, X(tt + 1, q + 1)));
      else if (m == 2) acc = add(acc, mul(c1, X(tt, q - 1)));
    }
    if (i >= m) acc = add(acc, mul(a2, X(tt - 1, q)));
    if (i + m <= n - 1) acc = add(acc, mul(c2, X(tt + 1, q)));
    return fabs(sub(bb, acc));
  };
  auto residual_cell = [&](const double *w, int64_t tt) -> double {
    return residual_from(w, tt, *(S.at(PA2, s, tt) + q), *(S.at(PA1, s, tt) + q),
                         *(S.at(PE, s, tt) + q), *(S.at(PC1, s, tt) + q), *(S.at(PC2, s, tt) + q),
                         *(S.at(PB, s, tt) + q));
  };

  auto block_max = [&](double v) -> double {
    for (int o = 16; o > 0; o >>= 1) v = nan_max(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if ((q & 31) == 0) s_red[q >> 5] = v;
    __syncthreads();
    double r = 0.0;
    const int nw = (int)((m + 31) / 32);
    for (int w = 0; w < nw; ++w) r = nan_max(r, s_red[w]);
    return r;
  };

  // initial residual of x0 (iterative.py:279-283)
  double rloc = 0.0;
  if (!use_x0) {
    // x0 = 0: every product of the sweep is a signed zero and 0 + (+-0) = +0,
    // so b - A x0 == b exactly and r0 = max |b|
    for (int64_t t = 0; t < T; ++t)
      if (valid_cell(t)) rloc = nan_max(rloc, fabs(*(S.at(PB, s, t) + q)));
  } else {
    for (int64_t t = 0; t < T + 1; ++t) {
      if (t < T) xn[(int)(t % 4) * m + q] = valid_cell(t) ? *(S.at(PXA, s, t) + q) : 0.0;
      __syncthreads();
      if (t >= 1 && valid_cell(t - 1)) rloc = nan_max(rloc, residual_cell(xn, t - 1));
    }
  }
  double r = block_max(rloc);
  const double r0 = r;
  double best = r;
  int64_t k = 0;
  int32_t st = BX_STATUS_OK;
  int cur = 0, best_loc = 0;
  const double tl = tol[s];
  const int XP[3] = {PXA, PXB, PXBEST};

  while (true) {
    if (q == 0) {
      s_go = 0;
      s_bestcopy = 0;
      if (r >= tl) {
        if (k >= max_iter) st = BX_STATUS_MAX_ITER;
        else s_go = 1;
      }
      if (s_go && best_loc == (cur ^ 1)) s_bestcopy = 1;
    }
    __syncthreads();
    if (!s_go) break;
    const int nxt = cur ^ 1;
    if (s_bestcopy) {  // the buffer about to be overwritten holds the best iterate
      for (int64_t t = 0; t < T; ++t)
        if (valid_cell(t)) *(S.at(PXBEST, s, t) + q) = *(S.at(XP[nxt], s, t) + q);
      best_loc = 2;
    }
    const int xo = XP[cur], xw = XP[nxt];
    // ---- forward: newRHS = K x + b, then L y = newRHS (iterative.py:293-294)
    // ring rows per step t: K (7), b, l1, l2 at slice t; x_old at slice t+1
    const int fpl[NPL] = {PK0, PKN1, PKP1, PKNM, PKPM, PKNQ, PKPQ, PB, PL1, PL2, xo};
    const int foff[NPL] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 1};
    if (q < 32) {
      set_rows(fpl, foff, NPL);
      for (int t = 0; t < nst - 1 && t < (int)T; ++t) issue(t);
    }
    xs[0 * m + q] = valid_cell(0) ? *(S.at(xo, s, 0) + q) : 0.0;
    double y_u = 0.0;  // own column, previous cell
    for (int64_t t = 0; t < T; ++t) {
      const int stg = wait_stage();
      if (t + 1 < T) xs[(int)((t + 1) % 4) * m + q] = valid_cell(t + 1) ? R_(stg, 10)[q] : 0.0;
      __syncthreads();
      if (q < 32 && t + nst - 1 < T) issue((int)(t + nst - 1));
      if (valid_cell(t)) {
        const int64_t p = t - q, i = p * m + q;
        auto X = [&](int64_t sl, int col) { return xs[(int)(((sl % 4) + 4) % 4) * m + col]; };
        double acc = add(0.0, mul(R_(stg, 0)[q], X(t, q)));
        if (i >= 1) {
          if (q >= 1) acc = add(acc, mul(R_(stg, 1)[q], X(t - 1, q - 1)));
          else if (m == 2) acc = add(acc, mul(R_(stg, 1)[q], X(t, q + 1)));
        }
        if (i <= n - 2) {
          if (q <= m - 2) acc = add(acc, mul(R_(stg, 2)[q], X(t + 1, q + 1)));
          else if (m == 2) acc = add(acc, mul(R_(stg, 2)[q], X(t, q - 1)));
        }
        if (i >= m) acc = add(acc, mul(R_(stg, 3)[q], X(t - 1, q)));
        if (i + m <= n - 1) acc = add(acc, mul(R_(stg, 4)[q], X(t + 1, q)));
        if (m != 2) {
          if (i >= m - 1 && q <= m - 2 && p >= 1) acc = add(acc, mul(R_(stg, 5)[q], X(t, q + 1)));
          if (i + m - 1 <= n - 1 && q >= 1) acc = add(acc, mul(R_(stg, 6)[q], X(t, q - 1)));
        }
        const double v = add(acc, R_(stg, 7)[q]);
        double y = v;
        if (i >= 1 && q >= 1) y = sub(y, mul(R_(stg, 8)[q], ys[(int)((t + 2) % 3) * m + q - 1]));
        if (i >= m) y = sub(y, mul(R_(stg, 9)[q], y_u));
        *(S.at(PY, s, t) + q) = y;
        ys[(int)(t % 3) * m + q] = y;
        y_u = y;
      }
    }
    asm volatile("fence.proxy.async.global;" ::: "memory");  // y rows -> TMA reads below
    __syncthreads();
    // ---- backward U x = y (iterative.py:295) + fused residual (296-297)
    // ring rows per step (t = T-1-j): y, phi, psi, mu at t; A (5), b at t+1
    const int bpl[10] = {PY, PPHI, PPSI, PMU, PA2, PA1, PE, PC1, PC2, PB};
    const int boff[10] = {0, 0, 0, 0, 1, 1, 1, 1, 1, 1};
    if (q < 32) {
      set_rows(bpl, boff, 10);
      for (int64_t j = 0; j < nst - 1 && j <= T; ++j) issue((int)(T - 1 - j));
    }
    double x_d = 0.0;  // own column, next cell (p+1, q)
    rloc = 0.0;
    for (int64_t j = 0; j <= T; ++j) {
      const int64_t t = T - 1 - j;
      const int stg = wait_stage();
      if (t >= 0 && valid_cell(t)) {
        const int64_t p = t - q, i = p * m + q;
        double v = R_(stg, 0)[q];
        if (i <= n - 2 && q <= m - 2)
          v = sub(v, mul(R_(stg, 1)[q], xn[(int)((t + 1) % 4) * m + q + 1]));
        if (i + m <= n - 1) v = sub(v, mul(R_(stg, 2)[q], x_d));
        const double xv = dvd(v, R_(stg, 3)[q]);
        *(S.at(xw, s, t) + q) = xv;
        xn[(int)(t % 4) * m + q] = xv;
        x_d = xv;
      } else if (t >= 0) {
        xn[(int)(t % 4) * m + q] = 0.0;
      }
      __syncthreads();
      if (q < 32 && j + nst - 1 <= T) issue((int)(T - 1 - (j + nst - 1)));
      if (t + 1 <= T - 1 && valid_cell(t + 1))
        rloc = nan_max(rloc, residual_from(xn, t + 1, R_(stg, 4)[q], R_(stg, 5)[q], R_(stg, 6)[q],
                                           R_(stg, 7)[q], R_(stg, 8)[q], R_(stg, 9)[q]));
    }
    asm volatile("fence.proxy.async.global;" ::: "memory");  // x rows -> next forward's TMA
    r = block_max(rloc);
    cur = nxt;
    ++k;
    if (q == 0 && history) history[s * max_iter + (k - 1)] = r;
    if (r < best) { best = r; best_loc = cur; }
    if (r0 > 0 && r > 1e6 * r0) { st = BX_STATUS_DIVERGED; break; }
  }
  // ---- outputs in the caller's layout
  for (int64_t t = 0; t < T; ++t) {
    if (!valid_cell(t)) continue;
    const int64_t i = (t - q) * m + q;
    xout[lay(i, s)] = *(S.at(XP[cur], s, t) + q);
    if (best_x) best_x[lay(i, s)] = *(S.at(XP[best_loc], s, t) + q);
  }
  if (q == 0) {
    if (iters) iters[s] = k;
    if (res) res[s] = r;
    if (best_res) best_res[s] = best;
    set_status(status, index, s, st, -1);
  }
}

// grid-structure check: any A[i,i-1] != 0 with i % m == 0, or A[i,i+1] != 0
// with i % m == m-1 (those couplings would cross a grid row)
template <class Lay>
__global__ void grid_check_kernel(const double *__restrict__ a1p, const double *__restrict__ c1p,
                                  int64_t batch, int64_t n, int64_t m, Lay lay, int *flag) {
  const int64_t rows = n / m;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < batch * rows * 2;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = idx / (rows * 2), r = (idx / 2) % rows;
    if (idx & 1) {
      const int64_t i = r * m + m - 1;
      if (i <= n - 2 && ldg(c1p + lay(i, s)) != 0.0) atomicOr(flag, 1);
    } else {
      const int64_t i = r * m;
      if (i >= 1 && ldg(a1p + lay(i, s)) != 0.0) atomicOr(flag, 1);
    }
  }
}

}  // namespace sipw

bool sip_is_grid(const double *a1, const double *c1, int64_t batch, int64_t n, int64_t m,
                 int64_t ld, int layout, cudaStream_t stream) {
  if (m < 2 || n % m != 0 || m > 512) return false;
  int *flag = nullptr;
  if (cudaMallocAsync((void **)&flag, sizeof(int), stream) != cudaSuccess) return false;
  cudaMemsetAsync(flag, 0, sizeof(int), stream);
  const int64_t work = batch * (n / m) * 2;
  const unsigned grid = (unsigned)(work / 256 + 1 < 4096 ? work / 256 + 1 : 4096);
  if (layout == BX_LAYOUT_INTERLEAVED)
    sipw::grid_check_kernel<<<grid, 256, 0, stream>>>(a1, c1, batch, n, m, Interleaved{ld}, flag);
  else
    sipw::grid_check_kernel<<<grid, 256, 0, stream>>>(a1, c1, batch, n, m, SystemMajor{ld}, flag);
  int h = 1;
  cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, stream);
  cudaStreamSynchronize(stream);
  cudaFreeAsync(flag, stream);
  return h == 0;
}

static int64_t sipw_mp(int64_t m) { return (m + 1) & ~(int64_t)1; }

size_t sip_wave_workspace_bytes(int64_t batch, int64_t n, int64_t m) {
  if (m < 2 || n % m) return 0;
  const int64_t T = n / m + m - 1;
  return sizeof(double) * (size_t)sipw::kPlanes * (size_t)batch * (size_t)T * (size_t)sipw_mp(m) + 256;
}

int sip_wave(const double *a2, const double *a1, const double *e, const double *c1,
             const double *c2, const double *b, const double *tol, double *x, double *best_x,
             int64_t *iters, double *res, double *best_res, int32_t *st, int32_t *ix,
             double *hist, double *ws, int64_t batch, int64_t n, int64_t m, double alpha,
             int64_t max_iter, int use_x0, int64_t ld, int layout, cudaStream_t stream) {
  if (n % m != 0 || m > 512) {
    bxh::set_error("wavefront SIP needs n %% m == 0 and m <= 512 (n=%lld, m=%lld)",
                   (long long)n, (long long)m);
    return BX_ERR_UNSUPPORTED;
  }
  const int64_t mp = sipw_mp(m);
  // workspace base 16-byte aligned for the TMA copies
  double *base = (double *)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  sipw::Skew S{base, batch, m, n / m + m - 1, mp};
  // ring stages: as many as fit next to the 11 m window doubles (<= 4)
  const size_t win = sizeof(double) * (size_t)(11 * m + 1);
  const size_t stage = sizeof(double) * (size_t)sipw::NPL * (size_t)mp;
  int nst = (int)((200 * 1024 - win) / stage);
  if (nst > 4) nst = 4;
  if (nst < 2) {
    bxh::set_error("wavefront SIP: grid width m=%lld too large for the shared-memory ring",
                   (long long)m);
    return BX_ERR_UNSUPPORTED;
  }
  const size_t smem = win + stage * nst + sizeof(uint64_t) * nst + 16;
  if (layout == BX_LAYOUT_INTERLEAVED) {
    auto k = sipw::sip_wave_kernel<Interleaved>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<(unsigned)batch, (unsigned)m, smem, stream>>>(a2, a1, e, c1, c2, b, tol, x, best_x, iters,
                                                     res, best_res, st, ix, hist, S, n, alpha,
                                                     max_iter, use_x0, Interleaved{ld}, nst);
  } else {
    auto k = sipw::sip_wave_kernel<SystemMajor>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<(unsigned)batch, (unsigned)m, smem, stream>>>(a2, a1, e, c1, c2, b, tol, x, best_x, iters,
                                                     res, best_res, st, ix, hist, S, n, alpha,
                                                     max_iter, use_x0, SystemMajor{ld}, nst);
  }
  return BX_OK;
}

}  // namespace bx
