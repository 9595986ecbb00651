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
#include <stdlib.h>

#include "bx_common.cuh"
#include "bx_kernels.h"

#ifdef BX_SIP_TRACE
__device__ long long g_sip_trace[64][40];
extern "C" int bx_sip_trace_read(void *host, size_t bytes) {
  return (int)cudaMemcpyFromSymbol(host, g_sip_trace, bytes < sizeof(g_sip_trace) ? bytes : sizeof(g_sip_trace));
}
#define SIP_TR(slot)                                                                      \
  do {                                                                                    \
    if (threadIdx.x == 0 && blockIdx.x < 64 && (slot) < 40) g_sip_trace[blockIdx.x][slot] = clock64(); \
  } while (0)
#else
#define SIP_TR(slot) \
  do {               \
  } while (0)
#endif

namespace bx {
namespace sipw {

enum Plane {
  PA2 = 0, PA1, PE, PC1, PC2, PB,   // A and b
  PL1, PL2, PMU, PPHI, PPSI,        // factors
  PK0, PKN1, PKP1, PKNM, PKPM, PKNQ, PKPQ,  // defect, sweep order
  PY, PXA, PXB, PXBEST, kPlanes
};

// Workspace of one system (doubles), laid out so that every wavefront step
// streams two contiguous blocks:
//   FG[t]  slice t, 10 rows of width W(t): K0 KN1 KP1 KNM KPM KNQ KPQ b l1 l2
//   BG[t]  t = -1..T-1: 3 rows of width W(t) (phi psi mu of slice t) then
//          6 rows of width W(t+1) (a2 a1 e c1 c2 b of slice t+1)
//   then full-stride planes (T x mp): y, x_a, x_b, x_best
// A row holds the valid cells (t-q, q), q = qlo(t) .. qlo(t)+nv(t)-1, of its
// slice; W(t) = nv(t) rounded up to even keeps every row 16-byte aligned.
struct Skew {
  double *ws;
  int64_t batch, m, T, mp, R;
  int64_t P;        // sum of W(t) over the slices
  int64_t per_sys;  // doubles per system
  const int64_t *pw;  // pw[t] = sum of W(u) for u < t, t = 0..T (device table)
  __device__ __forceinline__ int width(int t) const {
    if (t < 0 || t >= (int)T) return 0;
    int nv = t + 1;
    if ((int)m < nv) nv = (int)m;
    if ((int)R < nv) nv = (int)R;
    if ((int)T - t < nv) nv = (int)T - t;
    return nv + (nv & 1);
  }
  __device__ __forceinline__ int qlo(int t) const { return t - (int)R + 1 > 0 ? t - (int)R + 1 : 0; }
  __device__ __forceinline__ double *fg(int64_t s) const { return ws + s * per_sys; }
  // block offsets: FG[t] = 10 pw[t]; BG[t] = 3 pw[t] + 6 pw[t+1] (BG[-1] = 0)
  __device__ __forceinline__ int64_t fg_off(int t) const { return 10 * pw[t]; }
  __device__ __forceinline__ int64_t bg_off(int t) const { return t < 0 ? 0 : 3 * pw[t] + 6 * pw[t + 1]; }
  __device__ __forceinline__ double *bg(int64_t s) const { return fg(s) + 10 * P; }
  // full-stride planes only (PY, PXA, PXB, PXBEST)
  __device__ __forceinline__ double *at(int p, int64_t s, int64_t t) const {
    return fg(s) + 19 * P + ((int64_t)(p - PY) * T + t) * mp;
  }
};

// running block offsets while walking the slices upward: F = FG[t],
// Bm = BG[t-1], Bt = BG[t] (relative to fg(s) / bg(s))
struct Walk {
  int64_t F, Bm, Bt;
  __device__ __forceinline__ void start(const Skew &S) { F = 0; Bm = 0; Bt = 6 * (int64_t)S.width(0); }
  __device__ __forceinline__ void next(const Skew &S, int t) {  // from slice t to t+1
    F += 10 * (int64_t)S.width(t);
    Bm = Bt;
    Bt += 3 * (int64_t)S.width(t) + 6 * (int64_t)S.width(t + 1);
  }
};

// ---- TMA bulk copies into a shared-memory ring, completion on mbarriers ----
__device__ __forceinline__ unsigned smem_u32(const void *p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
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

__device__ __forceinline__ void mbar_wait_u32(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_u32(unsigned bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ double nan_max(double a, double b) {
  if (a != a || b != b) return __longlong_as_double(0x7ff8000000000000LL);
  return a > b ? a : b;
}

constexpr int NPL = 11;  // plane rows per ring stage

// pw[t] = sum_{u<t} W(u), t = 0..T (one thread; T is a few thousand at most)
__global__ void sip_prefix_kernel(Skew S) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int64_t acc = 0;
  int64_t *pw = const_cast<int64_t *>(S.pw);
  for (int t = 0; t <= (int)S.T; ++t) {
    pw[t] = acc;
    acc += S.width(t);
  }
}

// Data-parallel part of the setup, all SMs: gather A and b of every cell
// (t-q, q) into the packed slice rows (A/b rows of BG[t-1], b row of FG[t])
// with the reference's out-of-range zeros applied, and the initial iterate
// plane.  Rows of the original arrays are read where they lie; consecutive
// slices reuse the same sectors through L2.  The wavefront setup then reads
// A/b per step as contiguous rows.
template <class Lay>
__global__ void __launch_bounds__(512)
sip_pack_kernel(const double *__restrict__ a2p, const double *__restrict__ a1p,
                const double *__restrict__ ep, const double *__restrict__ c1p,
                const double *__restrict__ c2p, const double *__restrict__ bp,
                const double *__restrict__ x0, Skew S, int64_t n, int use_x0, Lay lay) {
  const int t = blockIdx.x;
  const int64_t s = blockIdx.y;
  const int mi = (int)S.m, Ri = (int)S.R;
  for (int q = threadIdx.x; q < mi; q += blockDim.x) {
    const int p = t - q;
    if ((unsigned)p >= (unsigned)Ri) continue;
    const int64_t i = (int64_t)p * mi + q;
    const int64_t li = lay(i, s);
    const bool pge1 = p >= 1, ige1 = pge1 || q >= 1, ilen2 = !(p == Ri - 1 && q == mi - 1),
               ple = p <= Ri - 2;
    const int Wt = S.width(t), Wm = S.width(t - 1), qo = q - S.qlo(t);
    double *ab = S.bg(s) + S.bg_off(t - 1) + 3 * Wm + qo;
    const double bb = ldg(bp + li);
    ab[0] = pge1 ? ldg(a2p + li) : 0.0;
    ab[Wt] = ige1 ? ldg(a1p + li) : 0.0;
    ab[2 * Wt] = ldg(ep + li);
    ab[3 * Wt] = ilen2 ? ldg(c1p + li) : 0.0;
    ab[4 * Wt] = ple ? ldg(c2p + li) : 0.0;
    ab[5 * Wt] = bb;
    S.fg(s)[S.fg_off(t) + 7 * Wt + qo] = bb;
    *(S.at(PXA, s, t) + q) = use_x0 ? x0[li] : 0.0;
  }
}

template <class Lay, bool M2>
__global__ void __launch_bounds__(544) sip_wave_kernel(const double *__restrict__ a2p, const double *__restrict__ a1p,
                                const double *__restrict__ ep, const double *__restrict__ c1p,
                                const double *__restrict__ c2p, const double *__restrict__ bp,
                                const double *__restrict__ tol, double *__restrict__ xout,
                                double *__restrict__ best_x, int64_t *iters, double *res,
                                double *best_res, int32_t *status, int32_t *index,
                                double *history, Skew S, int64_t n, double alpha,
                                int64_t max_iter, int use_x0, Lay lay, int nst,
                                double *__restrict__ nat, int32_t *__restrict__ setup_ok) {
  // nat != nullptr: setup only, for the scan solver (bx_sip_scan.cu) -- the
  // factors also leave in natural order, planes [l1 l2 mu phi psi][batch][n],
  // setup_ok[s] says whether system s has them
  extern __shared__ double sh[];
  SIP_TR(0);
  const int64_t m = S.m, R = n / m, T = S.T;
  const int q = threadIdx.x;
  const int64_t s = blockIdx.x;
  __shared__ int s_bad, s_notgrid, s_go, s_bestcopy;
  __shared__ double s_red[32];
  if (q == 0) { s_bad = 0x7fffffff; s_notgrid = 0; }
  __syncthreads();

  // ---------------- setup: skew A, b, x0; ILU(0)/Stone; defect ------------
  // The six input values of each thread's cell DS steps ahead are staged in
  // shared memory with cp.async (stage area = the later TMA ring), so the
  // per-step recurrence never waits a full global-memory round trip.
  double rb0 = 0.0;  // max |b| of the own cells (r0 when x0 = 0)
  {
    // lean per-step loop: 32-bit grid indices, grid-form boundary tests
    // (i = p m + q), rotating smem slots, incremental addresses
    double *smu = sh, *sphi = sh + 3 * m, *spsi = sh + 6 * m;
    double *stg_in = sh + 11 * m + (11 * m & 1);  // [DS][6][m]
    constexpr int DS = 4;
    const int mi_ = (int)m, Ri = (int)R, Ti = (int)T;
    const bool live = q < m;
    const bool qge1 = q >= 1, qlast = q == mi_ - 1, qfirst = q == 0;
    // A/b of cell (tt-q, q) from the packed rows BG[tt-1] (sip_pack_kernel):
    // the six rows of a slice are contiguous in q, so every copy is coalesced
    auto stage_cell = [&](int tt) {
      const int pp = tt - q;
      if (live && tt < Ti && (unsigned)pp < (unsigned)Ri) {
        const int W1 = S.width(tt), W0 = S.width(tt - 1);
        const double *src = S.bg(s) + S.bg_off(tt - 1) + 3 * W0 + (q - S.qlo(tt));
        const unsigned d = smem_u32(stg_in + ((tt % DS) * 6) * mi_ + q);
        const unsigned dm = (unsigned)(mi_ * sizeof(double));
#pragma unroll
        for (int a = 0; a < 6; ++a)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d + a * dm), "l"(src + a * W1)
                       : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    for (int tt = 0; tt < DS - 1; ++tt) stage_cell(tt);
    double mu_u = 0, phi_u = 0, psi_u = 0;  // own column, previous cell (p-1, q)
    // slots of the left neighbour's factors: previous step (read) / this step (write)
    int sl_prev = 2 * mi_, sl_cur = 0;  // (t-1) % 3 * m, t % 3 * m at t = 0
    int64_t F = 0, Bm = 0, Bt = 6 * (int64_t)S.width(0);
    int Wm = 0, Wt = S.width(0);
    const bool stone = alpha != 0.0;
    for (int t = 0; t < Ti; ++t) {
      stage_cell(t + DS - 1);
      asm volatile("cp.async.wait_group %0;" ::"n"(DS - 1) : "memory");
      const int p = t - q;
      const int Wn = S.width(t + 1);
      if (live && (unsigned)p < (unsigned)Ri) {
        const double *in = stg_in + ((t % DS) * 6) * mi_ + q;
        const bool pge1 = p >= 1, plast = p == Ri - 1, ple = p <= Ri - 2;
        const bool ige1 = pge1 || qge1;                 // i >= 1
        const bool ilen2 = !(plast && qlast);           // i <= n - 2
        const double a2 = pge1 ? in[0] : 0.0;           // i >= m
        const double a1 = ige1 ? in[mi_] : 0.0;
        const double e = in[2 * mi_];
        const double c1 = ilen2 ? in[3 * mi_] : 0.0;
        const double c2 = ple ? in[4 * mi_] : 0.0;      // i <= n - m - 1
        if ((qfirst && a1 != 0.0) || (qlast && c1 != 0.0)) s_notgrid = 1;
        const double mu_l = qge1 ? smu[sl_prev + q - 1] : 0.0;
        const double phi_l = qge1 ? sphi[sl_prev + q - 1] : 0.0;
        const double psi_l = qge1 ? spsi[sl_prev + q - 1] : 0.0;
        const bool has2 = pge1 && a2 != 0.0;
        const bool has1 = ige1 && a1 != 0.0;  // implies q >= 1 on a grid
        double li2 = 0.0, li1 = 0.0, mi, ph = 0.0, ps = 0.0;
        if (M2) {
          if (has2) li2 = dvd(a2, mu_u);
          if (has1) {
            double tt = a1;
            if (has2) tt = sub(tt, mul(li2, phi_u));
            li1 = dvd(tt, mu_l);
          }
          mi = e;
          if (has2) mi = sub(mi, mul(li2, psi_u));
          if (has1) mi = sub(mi, mul(li1, phi_l));
          if (ilen2) {
            double fi = c1;
            if (fi != 0.0 && has1) fi = sub(fi, mul(li1, psi_l));
            ph = fi;
          }
          ps = ple ? c2 : 0.0;                          // i <= n - 3 (m = 2)
        } else {
          if (has2) li2 = dvd(a2, stone ? add(mu_u, mul(alpha, phi_u)) : mu_u);
          if (has1) li1 = dvd(a1, stone ? add(mu_l, mul(alpha, psi_l)) : mu_l);
          mi = e;
          if (has2) mi = sub(mi, mul(li2, psi_u));
          if (has1) mi = sub(mi, mul(li1, phi_l));
          if (stone) {
            double comp = 0.0;
            if (has2) comp = add(comp, mul(li2, phi_u));
            if (has1) comp = add(comp, mul(li1, psi_l));
            mi = add(mi, mul(alpha, comp));
          }
          if (ilen2) {
            double fi = c1;
            if (stone && fi != 0.0 && has2) fi = sub(fi, mul(alpha, mul(li2, phi_u)));
            ph = fi;
          }
          if (ple) {
            double gi = c2;
            if (stone && gi != 0.0 && has1) gi = sub(gi, mul(alpha, mul(li1, psi_l)));
            ps = gi;
          }
        }
        if (mi == 0.0) atomicMin(&s_bad, p * mi_ + q);
        const double l1 = has1 ? li1 : 0.0, l2 = has2 ? li2 : 0.0;
        // defect K = LU - A (iterative.py:152-200); cross-row products are
        // structural zeros and are skipped
        if (nat) {
          // scan solver: the factors in natural order are all it needs (no
          // defect K, no packed planes); consecutive steps fill neighbouring
          // words of a sector, merged in L2
          const int64_t pl = (int64_t)gridDim.x * n;
          double *o = nat + s * n + (int64_t)p * mi_ + q;
          o[0] = l1;
          o[pl] = l2;
          o[2 * pl] = mi;  // (the scan solver inverts the plane in a pass of its own)
          o[3 * pl] = ph;
          o[4 * pl] = ps;
        } else {
        const double pm = pge1 ? mul(l2, mu_u) : 0.0;
        double p_1 = (ige1 && qge1) ? mul(l1, mu_l) : 0.0;
        if (M2 && pge1) p_1 = add(p_1, mul(l2, phi_u));           // i >= 2
        double p0 = mi;
        if (ige1 && qge1) p0 = add(p0, mul(l1, phi_l));
        if (pge1) p0 = add(p0, mul(l2, psi_u));
        double p1 = ilen2 ? ph : 0.0;
        if (M2 && ige1 && ilen2 && qge1) p1 = add(p1, mul(l1, psi_l));
        const double pp = ple ? ps : 0.0;
        const int qo = q - S.qlo(t);
        double *fgp = S.fg(s) + F + qo;
        double *up = S.bg(s) + Bt + qo;
        fgp[3 * Wt] = sub(pm, pge1 ? a2 : 0.0);                  // KNM
        fgp[Wt] = sub(p_1, ige1 ? a1 : 0.0);                     // KN1
        fgp[0] = sub(p0, e);                                     // K0
        fgp[2 * Wt] = sub(p1, ilen2 ? c1 : 0.0);                 // KP1
        fgp[4 * Wt] = sub(pp, ple ? c2 : 0.0);                   // KPM
        if (!M2) {
          fgp[5 * Wt] = pge1 ? mul(l2, phi_u) : 0.0;                                  // KNQ
          fgp[6 * Wt] = ((ige1 && (ple || (plast && qfirst))) && qge1) ? mul(l1, psi_l) : 0.0;  // KPQ
        }
        const double bb = in[5 * mi_];
        rb0 = nan_max(rb0, fabs(bb));
        fgp[8 * Wt] = l1;   // (b row 7 and the A/b rows come from sip_pack_kernel)
        fgp[9 * Wt] = l2;
        up[0] = ph;
        up[Wt] = ps;
        up[2 * Wt] = mi;
        }
        smu[sl_cur + q] = mi;
        sphi[sl_cur + q] = ph;
        spsi[sl_cur + q] = ps;
        mu_u = mi; phi_u = ph; psi_u = ps;
      }
      // slice walk: FG[t+1], BG[t] (= A/b of t+1), BG[t+1]
      F += 10 * (int64_t)Wt;
      Bm = Bt;
      Bt += 3 * (int64_t)Wt + 6 * (int64_t)Wn;
      Wm = Wt;
      Wt = Wn;
      sl_prev = sl_cur;
      sl_cur = sl_cur == 2 * mi_ ? 0 : sl_cur + mi_;
      __syncthreads();
    }
    asm volatile("cp.async.wait_all;" ::: "memory");  // staging area becomes the TMA ring
  }
  if (s_notgrid || s_bad != 0x7fffffff) {
    if (q == 0) {
      if (s_notgrid) set_status(status, index, s, BX_STATUS_NOT_GRID, -1);
      else set_status(status, index, s, BX_STATUS_ZERO_PIVOT, s_bad);
      if (iters) iters[s] = 0;
      if (setup_ok) setup_ok[s] = 0;
    }
    return;
  }
  if (nat) {
    if (q == 0) setup_ok[s] = 1;
    return;
  }

  SIP_TR(1);
  // (the forward keeps the previous iterate's window in registers)
  double *ys = sh + 4 * m;  // [3][m]
  double *xn = sh + 7 * m;  // [4][m] window of the new iterate
  // ring of NST stages x NPL plane rows (padded stride mp), filled by TMA bulk
  // copies that a dedicated producer warp issues; full[] completes on the
  // copies' bytes, empty[] when every consumer warp has finished the stage
  const int mp = (int)S.mp;
  double *ring = sh + 11 * m + (11 * m & 1);
  uint64_t *full = reinterpret_cast<uint64_t *>(ring + (int64_t)nst * NPL * mp);
  uint64_t *empty = full + nst;
  const int NCW = (int)((m + 31) / 32), NCT = NCW * 32;  // consumer warps / threads
  const bool producer = q >= NCT;
  const int lane = q & 31;
  auto R_ = [&](int stage, int j) { return ring + (stage * NPL + j) * mp; };
  auto valid_cell = [&](int64_t t) { const int64_t p = t - q; return q < m && p >= 0 && p < R; };
  if (q == 0)
    for (int i = 0; i < nst; ++i) { mbar_init(full + i, 1); mbar_init(empty + i, NCW); }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.global;" ::: "memory");  // setup's plane writes -> TMA reads
  __syncthreads();
  // ring bookkeeping: producer (issue side) and consumers (use side) walk the
  // same stage sequence; parity flips at every wrap
  int p_stg = 0, c_stg = 0;
  unsigned p_par = 0, c_par = 0;
  // producer: wait until the consumers released the stage, then queue one
  // contiguous group block (lane 0) and one full-stride row's valid range
  // (lane 1) for the step; both complete on the stage's full barrier
#ifdef BX_SIP_TRACE
  long long tr_wait = 0, tr_issue = 0;
#endif
  auto produce = [&](const double *gsrc, unsigned gbytes, const double *rowp, int rslice) {
#ifdef BX_SIP_TRACE
    const long long c0 = clock64();
#endif
    mbar_wait(empty + p_stg, p_par ^ 1u);  // first round passes (fresh barrier)
#ifdef BX_SIP_TRACE
    const long long c1 = clock64();
    tr_wait += c1 - c0;
#endif
    unsigned rb_ = 0;
    int a0 = 0;
    if (rowp != nullptr && rslice >= 0 && rslice < (int)T) {
      a0 = S.qlo(rslice) & ~1;
      const int qhi = rslice < (int)m - 1 ? rslice : (int)m - 1;
      rb_ = (unsigned)(((qhi + 2) & ~1) - a0) * (unsigned)sizeof(double);
    }
    if (lane == 0) {
      mbar_expect(full + p_stg, gbytes + rb_);
      if (gbytes) bulk_g2s(R_(p_stg, 0), gsrc, gbytes, full + p_stg);
    } else if (lane == 1 && rb_) {
      bulk_g2s(R_(p_stg, 10) + a0, rowp + (int64_t)rslice * mp + a0, rb_, full + p_stg);
    }
    __syncwarp();
    if (++p_stg == nst) { p_stg = 0; p_par ^= 1u; }
#ifdef BX_SIP_TRACE
    tr_issue += clock64() - c1;
#endif
  };
  const unsigned full_u = smem_u32(full), empty_u = smem_u32(empty);
  auto consume_wait = [&]() -> int {
    const int stg = c_stg;
    mbar_wait_u32(full_u + 8u * (unsigned)stg, c_par);
    return stg;
  };
  auto consume_release = [&]() {
    __syncwarp();
    if (lane == 0) mbar_arrive_u32(empty_u + 8u * (unsigned)c_stg);
    if (++c_stg == nst) { c_stg = 0; c_par ^= 1u; }
  };

  // consumer-only barrier (named barrier 1): the producer warp runs ahead
  auto cons_sync = [&]() { asm volatile("bar.sync 1, %0;" ::"r"(NCT) : "memory"); };

  // residual of cell (slice tt, column q) from a window w[4][m] of x slices
  // tt-1..tt+1 and the row's A/b values (iterative.py:213-221 order, acc from 0)
  auto residual_from = [&](const double *w, int tt, double a2, double a1, double e,
                           double c1, double c2, double bb) -> double {
    const int p = tt - q;
    const int64_t i = (int64_t)p * m + q;
    auto X = [&](int sl, int col) { return w[(sl & 3) * (int)m + col]; };
    double acc = add(0.0, mul(e, X(tt, q)));
    if (i >= 1) {
      if (q >= 1) acc = add(acc, mul(a1, X(tt - 1, q - 1)));
      else if (m == 2) acc = add(acc, mul(a1, X(tt, q + 1)));
    }
    if (i <= n - 2) {
      if (q <= m - 2) acc = add(acc, mul(c1, X(tt + 1, q + 1)));
      else if (m == 2) acc = add(acc, mul(c1, X(tt, q - 1)));
    }
    if (p >= 1) acc = add(acc, mul(a2, X(tt - 1, q)));
    if (p <= (int)R - 2) acc = add(acc, mul(c2, X(tt + 1, q)));
    return fabs(sub(bb, acc));
  };
  // A/b of slice tt live in BG[tt-1] (offset Bm of the walk at slice tt)
  auto residual_cell = [&](const double *w, int tt, int64_t Bm) -> double {
    const int Wt = S.width(tt), Wm = S.width(tt - 1);
    const double *ab = S.bg(s) + Bm + 3 * Wm + (q - S.qlo(tt));
    return residual_from(w, tt, ab[0], ab[Wt], ab[2 * Wt], ab[3 * Wt], ab[4 * Wt], ab[5 * Wt]);
  };

  auto block_max = [&](double v) -> double {
    for (int o = 16; o > 0; o >>= 1) v = nan_max(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if ((q & 31) == 0) s_red[q >> 5] = v;
    __syncthreads();
    double r = 0.0;
    for (int w = 0; w < NCW; ++w) r = nan_max(r, s_red[w]);
    return r;
  };

  // initial residual of x0 (iterative.py:279-283)
  double rloc = 0.0;
  {
    Walk W;
    W.start(S);
    if (!use_x0) {
      // x0 = 0: every product of the sweep is a signed zero and 0 + (+-0) = +0,
      // so b - A x0 == b exactly and r0 = max |b| (taken during the setup)
      rloc = rb0;
    } else {
      int64_t Bprev = 0;  // BG offset for slice t-1's A/b (= walk Bm at slice t-1)
      for (int t = 0; t < (int)T + 1; ++t) {
        if (t < (int)T && q < m) xn[(t % 4) * m + q] = valid_cell(t) ? *(S.at(PXA, s, t) + q) : 0.0;
        __syncthreads();
        if (t >= 1 && valid_cell(t - 1)) rloc = nan_max(rloc, residual_cell(xn, t - 1, Bprev));
        Bprev = W.Bm;
        if (t < (int)T) W.next(S, t);
      }
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
  const int Ti = (int)T, Ri = (int)R, mi_ = (int)m;
  const int p_hi = Ri - 2;  // cells with p <= p_hi have a +m neighbour

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
      asm volatile("fence.proxy.async.global;" ::: "memory");
      __syncthreads();
    }
    SIP_TR(2 + 2 * (int)k);
    const int xo = XP[cur], xw = XP[nxt];
    // ---- forward: newRHS = K x + b, then L y = newRHS (iterative.py:293-294)
    // ring rows per step t: K (7), b, l1, l2 at slice t; x_old at slice t+1
    if (producer) {
      const double *xrow = S.at(xo, s, 0);
      int64_t F = 0;
      for (int t = 0; t < Ti; ++t) {
        const int Wt = S.width(t);
        produce(S.fg(s) + F, (unsigned)(10 * Wt * sizeof(double)), xrow, t + 1);
        F += 10 * Wt;
      }
    } else {
      // lean per-step loop: incremental slice geometry, grid-form boundary
      // tests (i = p m + q), 32-bit indices.  The old iterate's 3x3 window
      // (columns q-1..q+1, slices t-1..t+1) lives in registers, read from the
      // staged plane row, so K x + b of the step is formed before the
      // barrier; only y = v - l1 y(left) - l2 y(up) follows it.
      const bool live = q < m;
      double *py = S.at(PY, s, 0) + q;
      auto x_at = [&](const double *row, int tt, int qq) -> double {  // 0 outside the grid
        const int pp = tt - qq;
        return (qq >= 0 && qq < mi_ && (unsigned)pp < (unsigned)Ri) ? row[qq] : 0.0;
      };
      const double *xrow0 = S.at(xo, s, 0);
      double xm_l = 0.0, xm_c = 0.0;                       // slice t-1: q-1, q
      double x0_l = x_at(xrow0, 0, q - 1), x0_c = x_at(xrow0, 0, q), x0_r = x_at(xrow0, 0, q + 1);
      double y_u = 0.0;  // own column, previous cell
      const bool qge1 = q >= 1, qlem2 = q <= mi_ - 2, qlast = q == mi_ - 1, qfirst = q == 0;
      double *yprev = ys + mi_, *ycur = ys;  // slices t-1, t
      const int stage_d = NPL * mp;
      int Wt = S.width(0), qlo_t = 0;
      for (int t = 0; t < Ti; ++t, py += mp) {
        const int stg = consume_wait();
        const double *stage = ring + stg * stage_d;
        const int p = t - q;
        double xp_l = 0.0, xp_c = 0.0, xp_r = 0.0;  // slice t+1: q-1, q, q+1
        if (live && t + 1 < Ti) {
          const double *xr = stage + 10 * mp;
          xp_l = x_at(xr, t + 1, q - 1);
          xp_c = x_at(xr, t + 1, q);
          xp_r = x_at(xr, t + 1, q + 1);
        }
        const bool cell = live && (unsigned)p < (unsigned)Ri;
        const double *rb = stage + (q - qlo_t);
        const bool pge1 = p >= 1;
        double v = 0.0;
        if (cell) {
          const bool plast = p == Ri - 1, phi_ok = p <= p_hi;
          double acc = add(0.0, mul(rb[0], x0_c));
          if (pge1 || qge1) {                                   // i >= 1
            if (qge1) acc = add(acc, mul(rb[Wt], xm_l));
            else if (M2) acc = add(acc, mul(rb[Wt], x0_r));
          }
          if (!(plast && qlast)) {                              // i <= n - 2
            if (qlem2) acc = add(acc, mul(rb[2 * Wt], xp_r));
            else if (M2) acc = add(acc, mul(rb[2 * Wt], x0_l));
          }
          if (pge1) acc = add(acc, mul(rb[3 * Wt], xm_c));
          if (phi_ok) acc = add(acc, mul(rb[4 * Wt], xp_c));
          if (!M2) {
            if ((pge1 || qlast) && qlem2 && pge1) acc = add(acc, mul(rb[5 * Wt], x0_r));
            if ((phi_ok || (plast && qfirst)) && qge1) acc = add(acc, mul(rb[6 * Wt], x0_l));
          }
          v = add(acc, rb[7 * Wt]);
        }
        cons_sync();  // y of slice t-1 (yprev) written by the left neighbour
        if (cell) {
          double y = v;
          if ((pge1 || qge1) && qge1) y = sub(y, mul(rb[8 * Wt], yprev[q - 1]));
          if (pge1) y = sub(y, mul(rb[9 * Wt], y_u));
          *py = y;
          ycur[q] = y;
          y_u = y;
        }
        consume_release();
        Wt = S.width(t + 1);
        qlo_t += t + 1 >= Ri ? 1 : 0;
        xm_l = x0_l; xm_c = x0_c;
        x0_l = xp_l; x0_c = xp_c; x0_r = xp_r;
        double *ty = yprev; yprev = ycur; ycur = ty;
      }
      asm volatile("fence.proxy.async.global;" ::: "memory");  // y rows -> TMA reads below
    }
    __syncthreads();
    SIP_TR(3 + 2 * (int)k);
    // ---- backward U x = y (iterative.py:295) + fused residual (296-297)
    // ring rows per step (t = T-1-j): y, phi, psi, mu at t; A (5), b at t+1
    rloc = 0.0;
    if (producer) {
      const double *yrow = S.at(PY, s, 0);
      int64_t B = 9 * S.P - 3 * (int64_t)S.width(Ti - 1);  // BG[T-1]
      for (int t = Ti - 1; t >= -1; --t) {
        const int64_t sz = 3 * (int64_t)S.width(t) + 6 * (int64_t)S.width(t + 1);
        produce(S.bg(s) + B, (unsigned)(sz * sizeof(double)), yrow, t);
        B -= 3 * (int64_t)S.width(t - 1) + 6 * (int64_t)S.width(t);
      }
    } else {
      const bool live = q < m;
      double *px = S.at(xw, s, 0) + q + (int64_t)(Ti - 1) * mp;
      double x_d = 0.0;  // own column, next cell (p+1, q)
      const bool qge1 = q >= 1, qlem2 = q <= mi_ - 2, qlast = q == mi_ - 1;
      // window of the new iterate: slices t, t+1, t+2 (and t+3, being retired)
      double *n0 = xn + ((Ti - 1) & 3) * mi_, *n1 = xn + (Ti & 3) * mi_,
             *n2 = xn + ((Ti + 1) & 3) * mi_, *n3 = xn + ((Ti + 2) & 3) * mi_;
      const int stage_d = NPL * mp;
      int Wt = S.width(Ti - 1), W1 = 0, qlo_t = S.qlo(Ti - 1), qlo_1 = S.qlo(Ti);
      for (int j = 0; j <= Ti; ++j, px -= mp) {
        const int t = Ti - 1 - j;
        const int stg = consume_wait();
        const double *stage = ring + stg * stage_d;
        const int p = t - q;
        if (live && t >= 0) {
          if ((unsigned)p < (unsigned)Ri) {
            const double *ub = stage + (q - qlo_t);                 // phi psi mu of slice t
            double v = stage[10 * mp + q];                          // y
            if (!(p == Ri - 1 && qlast) && qlem2) v = sub(v, mul(ub[0], n1[q + 1]));
            if (p <= p_hi) v = sub(v, mul(ub[Wt], x_d));
            const double xv = dvd(v, ub[2 * Wt]);
            *px = xv;
            n0[q] = xv;
            x_d = xv;
          } else {
            n0[q] = 0.0;
          }
        }
        cons_sync();
        if (live && t + 1 <= Ti - 1 && (unsigned)(p + 1) < (unsigned)Ri) {
          // residual of slice t+1 (iterative.py:213-221 order, acc from 0)
          const double *ab = stage + 3 * Wt + (q - qlo_1);          // A, b of slice t+1
          const int pp = p + 1;
          double acc = add(0.0, mul(ab[2 * W1], n1[q]));
          if (pp >= 1 || qge1) {
            if (qge1) acc = add(acc, mul(ab[W1], n0[q - 1]));
            else if (M2) acc = add(acc, mul(ab[W1], n1[q + 1]));
          }
          if (!(pp == Ri - 1 && qlast)) {
            if (qlem2) acc = add(acc, mul(ab[3 * W1], n2[q + 1]));
            else if (M2) acc = add(acc, mul(ab[3 * W1], n1[q - 1]));
          }
          if (pp >= 1) acc = add(acc, mul(ab[0], n0[q]));
          if (pp <= p_hi) acc = add(acc, mul(ab[4 * W1], n2[q]));
          rloc = nan_max(rloc, fabs(sub(ab[5 * W1], acc)));
        }
        consume_release();
        W1 = Wt;
        Wt = S.width(t - 1);
        qlo_1 = qlo_t;
        qlo_t -= (t - 1 >= Ri - 1 && qlo_t > 0) ? 1 : 0;
        double *tw = n3; n3 = n2; n2 = n1; n1 = n0; n0 = tw;
      }
      asm volatile("fence.proxy.async.global;" ::: "memory");  // x rows -> next forward's TMA
    }
    r = block_max(rloc);
    cur = nxt;
    ++k;
    if (q == 0 && history) history[s * max_iter + (k - 1)] = r;
    if (r < best) { best = r; best_loc = cur; }
    if (r0 > 0 && r > 1e6 * r0) { st = BX_STATUS_DIVERGED; break; }
  }
#ifdef BX_SIP_TRACE
  if (producer && lane == 0 && blockIdx.x < 64) { g_sip_trace[blockIdx.x][37] = tr_wait; g_sip_trace[blockIdx.x][38] = tr_issue; }
#endif
  SIP_TR(39);
  // ---- outputs in the caller's layout: column q's cells (p, q), slice p + q;
  // eight loads in flight per thread (one at a time left the loop latency-bound)
  if (q < m) {
    const double *xc = S.at(XP[cur], s, 0) + q, *xb = S.at(XP[best_loc], s, 0) + q;
    constexpr int U = 8;
    for (int64_t p0 = 0; p0 < R; p0 += U) {
      double v[U], w[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t p = p0 + u;
        v[u] = p < R ? xc[(p + q) * S.mp] : 0.0;
        w[u] = (best_x && p < R) ? xb[(p + q) * S.mp] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t p = p0 + u;
        if (p >= R) break;
        const int64_t i = p * m + q;
        xout[lay(i, s)] = v[u];
        if (best_x) best_x[lay(i, s)] = w[u];
      }
    }
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
                 int64_t ld, int layout, void *scratch, cudaStream_t stream) {
  // scratch: >= 4 bytes of the caller's workspace (no allocation on this path)
  if (m < 2 || n % m != 0 || m > 512 || scratch == nullptr) return false;
  int *flag = reinterpret_cast<int *>(scratch);
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
  return h == 0;
}

static int64_t sipw_mp(int64_t m) { return (m + 1) & ~(int64_t)1; }

// packed per-system layout (see Skew): sum of the even-rounded slice widths
static sipw::Skew sipw_layout(double *base, int64_t batch, int64_t n, int64_t m) {
  sipw::Skew S{};
  S.ws = base;
  S.batch = batch;
  S.m = m;
  S.R = n / m;
  S.T = S.R + m - 1;
  S.mp = sipw_mp(m);
  int64_t P = 0;
  for (int64_t t = 0; t < S.T; ++t) {
    int64_t nv = t + 1;
    if (m < nv) nv = m;
    if (S.R < nv) nv = S.R;
    if (S.T - t < nv) nv = S.T - t;
    P += nv + (nv & 1);
  }
  S.P = P;
  S.per_sys = 19 * P + 4 * S.T * S.mp;
  return S;
}

// workspace: [prefix table pw (T+1 int64, padded to 256 B)] [systems]
static size_t sipw_pw_bytes(int64_t T) { return ((size_t)(T + 1) * sizeof(int64_t) + 255) & ~(size_t)255; }

size_t sip_wave_workspace_bytes(int64_t batch, int64_t n, int64_t m) {
  if (m < 2 || n % m) return 0;
  const sipw::Skew S = sipw_layout(nullptr, batch, n, m);
  return sipw_pw_bytes(S.T) + sizeof(double) * (size_t)batch * (size_t)S.per_sys + 256;
}

int sip_wave(const double *a2, const double *a1, const double *e, const double *c1,
             const double *c2, const double *b, const double *tol, double *x, double *best_x,
             int64_t *iters, double *res, double *best_res, int32_t *st, int32_t *ix,
             double *hist, double *ws, int64_t batch, int64_t n, int64_t m, double alpha,
             int64_t max_iter, int use_x0, int64_t ld, int layout, cudaStream_t stream,
             double *nat, int32_t *setup_ok) {
  if (n % m != 0 || m > 512) {
    bxh::set_error("wavefront SIP needs n %% m == 0 and m <= 512 (n=%lld, m=%lld)",
                   (long long)n, (long long)m);
    return BX_ERR_UNSUPPORTED;
  }
  const int64_t mp = sipw_mp(m);
  // workspace base 16-byte aligned for the TMA copies
  double *base = (double *)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  sipw::Skew S = sipw_layout(nullptr, batch, n, m);
  S.pw = reinterpret_cast<const int64_t *>(base);
  S.ws = reinterpret_cast<double *>(reinterpret_cast<char *>(base) + sipw_pw_bytes(S.T));
  // ring stages: as many as fit next to the 11 m window doubles (<= 4)
  const size_t win = sizeof(double) * (size_t)(11 * m + 1);
  const size_t stage = sizeof(double) * (size_t)sipw::NPL * (size_t)mp;
  int nst = (int)((200 * 1024 - win) / stage);
  if (nst > 4) nst = 4;
  if (const char *env = getenv("BX_SIP_NST")) nst = nst < atoi(env) ? nst : atoi(env);  // dev knob
  if (nst < 2) {
    bxh::set_error("wavefront SIP: grid width m=%lld too large for the shared-memory ring",
                   (long long)m);
    return BX_ERR_UNSUPPORTED;
  }
  sipw::sip_prefix_kernel<<<1, 32, 0, stream>>>(S);
  {
    const unsigned pthreads = (unsigned)(m < 512 ? ((m + 31) / 32) * 32 : 512);
    const dim3 pgrid((unsigned)S.T, (unsigned)batch);
    if (layout == BX_LAYOUT_INTERLEAVED)
      sipw::sip_pack_kernel<<<pgrid, pthreads, 0, stream>>>(a2, a1, e, c1, c2, b, x, S, n, use_x0,
                                                           Interleaved{ld});
    else
      sipw::sip_pack_kernel<<<pgrid, pthreads, 0, stream>>>(a2, a1, e, c1, c2, b, x, S, n, use_x0,
                                                           SystemMajor{ld});
  }
  const size_t ring = stage * nst + sizeof(uint64_t) * 2 * nst + 16;
  const size_t staging = sizeof(double) * 4 * 6 * (size_t)m + 16;  // setup cp.async stages (DS = 4)
  const size_t smem = win + (ring > staging ? ring : staging);
  // consumer warps (one thread per grid column) + one TMA producer warp
  const unsigned threads = (unsigned)(((m + 31) / 32) * 32 + 32);
  if (layout == BX_LAYOUT_INTERLEAVED) {
    auto k = m == 2 ? sipw::sip_wave_kernel<Interleaved, true> : sipw::sip_wave_kernel<Interleaved, false>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<(unsigned)batch, threads, smem, stream>>>(a2, a1, e, c1, c2, b, tol, x, best_x, iters,
                                                 res, best_res, st, ix, hist, S, n, alpha,
                                                 max_iter, use_x0, Interleaved{ld}, nst, nat, setup_ok);
  } else {
    auto k = m == 2 ? sipw::sip_wave_kernel<SystemMajor, true> : sipw::sip_wave_kernel<SystemMajor, false>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<(unsigned)batch, threads, smem, stream>>>(a2, a1, e, c1, c2, b, tol, x, best_x, iters,
                                                 res, best_res, st, ix, hist, S, n, alpha,
                                                 max_iter, use_x0, SystemMajor{ld}, nst, nat, setup_ok);
  }
  return BX_OK;
}

}  // namespace bx
