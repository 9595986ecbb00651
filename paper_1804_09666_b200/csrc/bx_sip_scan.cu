// SIP on grid-structured systems, throughput path (BX_ALGO_SCAN): row-parallel
// scan sweeps in correction form, one CTA per system.
//
// Same iteration as sip_solve (iterative.py:255-308) in exact arithmetic:
// with L U = A + K,   x_{k+1} = (LU)^-1 (K x_k + b) = x_k + (LU)^-1 (b - A x_k),
// so one pass over the grid rows forms r = b - A x_k (whose max norm is the
// loop's residual of x_k), and solves L y = r on the fly; a second pass solves
// U d = y upwards and writes x_{k+1} = x_k + d.  The defect matrix K is never
// read (104 -> 128 B per cell and iteration against the wavefront kernel's
// 184), and the rounding differs from Algorithm 1's: the contract is the
// north star's "same iteration count +-1, final residual below the
// tolerance", not bit parity (that is bx_sip.cu / bx_sip_wave.cu).
//
// Parallelism: thread q owns grid column q.  Inside a grid row the forward
// recurrence  y_q = c_q - l1_q y_{q-1}  (c_q = r_q - lm_q y_{p-1,q} is local)
// is a first-order linear recurrence: an inclusive scan of the affine maps
// y -> c + a y over the row (warp shuffles, then the warp totals), one CTA
// barrier per grid row.  A sweep therefore costs R = n/m scans of depth
// log2(m) instead of the wavefront's R + m - 1 dependent steps with half the
// threads idle.  The backward recurrence d_q = (y_q - psi_q d_{p+1,q}) / mu_q -
// (phi_q / mu_q) d_{q+1} is the mirror image.  Inputs of the next rows are
// prefetched into registers while a row is scanned.
//
// Grids of 128 columns and more are split over a CTA pair (two SMs per system)
// as a feed-forward pipeline, sip_scan_pair_kernel below.
//
// The factors come from the wavefront kernel's setup pass (ILU(0) / Stone
// alpha, bit-identical to ilu0_penta, iterative.py:62-124), which also leaves
// them in natural order for this kernel (1/mu instead of mu).
#include <stdlib.h>

#include "bx_common.cuh"
#include "bx_kernels.h"

namespace bx {
namespace sipscan {

constexpr int kST = 4;  // grid rows in flight: cp.async ring stages in shared memory

// natural-order planes [batch][n]
struct Nat {
  const double *l1, *l2, *rmu, *phi, *psi;
  double *y, *x[3];
};

__device__ __forceinline__ double nan_max(double a, double b) {
  return (b > a || b != b) ? b : a;  // NaN sticks
}

// inclusive scan step of affine maps F(y) = B + A y: own segment after the
// segment `d` lanes away (up: lower lanes come first; down: higher lanes)
template <bool UP>
__device__ __forceinline__ void warp_scan(double &A, double &B, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const double Ao = UP ? __shfl_up_sync(0xffffffffu, A, d) : __shfl_down_sync(0xffffffffu, A, d);
    const double Bo = UP ? __shfl_up_sync(0xffffffffu, B, d) : __shfl_down_sync(0xffffffffu, B, d);
    const bool has = UP ? lane >= d : lane + d < 32;  // (selects: the warp stays converged)
    const double Bn = fma(A, Bo, B), An = A * Ao;
    B = has ? Bn : B;
    A = has ? An : A;
  }
}

// value entering warp `warp` from the warps before (UP) / after (!UP) it:
// scan of the warp totals tot[w] = (A, B) from the value `start` that enters
// the first warp in scan order (0 at a system edge, the neighbouring CTA's
// boundary value in the CTA-pair kernel)
template <bool UP>
__device__ __forceinline__ double carry_in(const double2 *tot, int warp, int lane, int nw,
                                           double start = 0.0) {
  // Fast path: the previous warp's map forgets what entered it (|A| * |carry|
  // is below the rounding of B: dominant rows decay by the 32 cells of a warp),
  // so the value leaving it is its B alone.  Checked per row, exact otherwise.
  const int prev = UP ? warp - 1 : warp + 1;
  if (prev >= 0 && prev < nw) {
    const double2 v = tot[prev];
    const int pp = UP ? prev - 1 : prev + 1;
    const double bprev = (pp >= 0 && pp < nw) ? fabs(tot[pp].y) : fabs(start);
    if (fabs(v.x) * bprev <= 0x1p-60 * fabs(v.y) && fabs(v.x) <= 0x1p-40) return v.y;
  } else {
    return start;
  }
  const int j = UP ? lane : nw - 1 - lane;  // lane 0 holds the first warp in scan order
  double A = 0.0, B = 0.0;
  if (lane < nw) {
    const double2 v = tot[j];
    A = v.x;
    B = v.y;
  }
  warp_scan<true>(A, B, lane);
  const int src = (UP ? warp : nw - 1 - warp) - 1;  // inclusive result of the warp before this one
  const double a = __shfl_sync(0xffffffffu, A, src < 0 ? 0 : src);
  const double c = __shfl_sync(0xffffffffu, B, src < 0 ? 0 : src);
  return src < 0 ? start : fma(a, start, c);
}

// C doubles at p (32-byte vector access when VEC: C == 4, aligned)
template <int C, bool VEC>
__device__ __forceinline__ void ldC(const double *p, double *o) {
  if (VEC && C == 4) {
    asm volatile("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];"
                 : "=d"(o[0]), "=d"(o[1]), "=d"(o[2]), "=d"(o[3])
                 : "l"(p));
  } else {
#pragma unroll
    for (int c = 0; c < C; ++c) o[c] = p[c];
  }
}
template <int C, bool VEC>
__device__ __forceinline__ void stC(double *p, const double *v) {
  if (VEC && C == 4) {
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(v[0]), "d"(v[1]),
                 "d"(v[2]), "d"(v[3])
                 : "memory");
  } else {
#pragma unroll
    for (int c = 0; c < C; ++c) p[c] = v[c];
  }
}

__device__ __forceinline__ unsigned smem_u32(const void *p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
// C doubles global -> shared, asynchronously (16-byte copies when W16)
template <int C, bool W16>
__device__ __forceinline__ void cpC(double *dst, const double *src) {
  if (W16 && C % 2 == 0) {
#pragma unroll
    for (int c = 0; c < C; c += 2)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst + c)), "l"(src + c)
                   : "memory");
  } else {
#pragma unroll
    for (int c = 0; c < C; ++c)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst + c)), "l"(src + c)
                   : "memory");
  }
}

// Thread tq owns the C grid columns C tq .. C tq + C - 1 (m / C threads): its
// own cells are composed serially, the threads' maps by the warp scan, the
// warps' by carry_in.  C = 1 is the default (measured fastest, see sip_scan):
// C > 1 trades warps for fewer instructions per cell and loses.
// VEC: the caller's arrays allow 32-byte accesses (system-major, aligned).
template <class Lay, int C, bool VEC>
__global__ void __launch_bounds__(512 / C)
sip_scan_kernel(const double *__restrict__ a2p, const double *__restrict__ a1p,
                const double *__restrict__ ep, const double *__restrict__ c1p,
                const double *__restrict__ c2p, const double *__restrict__ bp,
                const double *__restrict__ tol, double *__restrict__ xout,
                double *__restrict__ best_x, int64_t *iters, double *res, double *best_res,
                int32_t *status, int32_t *index, double *history, Nat N,
                const int32_t *__restrict__ setup_ok, int64_t n, int m, int64_t max_iter,
                int use_x0, Lay lay) {
  const int64_t s = blockIdx.x;
  if (!setup_ok[s]) return;  // not a grid / zero pivot: reported by the setup pass
  const int tq = threadIdx.x, lane = tq & 31, warp = tq >> 5, nw = (m / C) >> 5;
  const int q0 = C * tq;  // first own column
  const int R = (int)(n / m);
  extern __shared__ double sh[];
  double *xrow = sh;                                          // [2][m + 2] (zero ends)
  double2 *tot = reinterpret_cast<double2 *>(sh + 2 * (m + 2));  // [2][nw]
  double *red = sh + 2 * (m + 2) + 4 * nw;                     // [32]
  double *ring = red + 32;                                    // [kST][9][m] staged rows (own columns)
  const int64_t o = s * n;  // this system's planes
  if (tq < 2) {
    xrow[tq * (m + 2)] = 0.0;
    xrow[tq * (m + 2) + m + 1] = 0.0;
  }

  // ---- initial iterate -> buffer 0 ----------------------------------------
  for (int p = 0; p < R; ++p) {
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const int64_t i = (int64_t)p * m + q0 + c;
      N.x[0][o + i] = use_x0 ? xout[lay(i, s)] : 0.0;
    }
  }
  __syncthreads();

  // CTA-wide max of the per-thread residuals (NaN propagates)
  auto block_max = [&](double v) -> double {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v = nan_max(v, __shfl_xor_sync(0xffffffffu, v, d));
    __syncthreads();  // red reusable
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double r = red[0];
    for (int w = 1; w < nw; ++w) r = nan_max(r, red[w]);
    return r;
  };
  // caller arrays: this thread's C values of row i0.. into its ring slots
  auto cp_in = [&](double *dst, const double *base, int64_t i0) {
    if (VEC) {
      cpC<C, true>(dst, base + lay(i0, s));
    } else {
#pragma unroll
      for (int c = 0; c < C; ++c) cpC<1, false>(dst + c, base + lay(i0 + c, s));
    }
  };
  auto commit = [] { asm volatile("cp.async.commit_group;" ::: "memory"); };
  auto wait_row = [] { asm volatile("cp.async.wait_group %0;" ::"n"(kST - 1) : "memory"); };

  // ---- forward pass: r = b - A x, ||r||_inf, L y = r ------------------------
  auto forward = [&](const double *__restrict__ x) -> double {
    // ring slot of row p: [a2 a1 e c1 c2 b l1 l2 x(p+1)][m]; every thread stages
    // and later reads only its own columns (no barrier, just the copy groups)
    auto stage = [&](int p) {
      if (p < R) {
        double *dst = ring + (int64_t)(p % kST) * 9 * m + q0;
        const int64_t i0 = (int64_t)p * m + q0;
        cp_in(dst, a2p, i0);
        cp_in(dst + m, a1p, i0);
        cp_in(dst + 2 * m, ep, i0);
        cp_in(dst + 3 * m, c1p, i0);
        cp_in(dst + 4 * m, c2p, i0);
        cp_in(dst + 5 * m, bp, i0);
        cpC<C, true>(dst + 6 * m, N.l1 + o + i0);
        cpC<C, true>(dst + 7 * m, N.l2 + o + i0);
        if (p + 1 < R) {
          cpC<C, true>(dst + 8 * m, x + o + i0 + m);
        } else {
#pragma unroll
          for (int c = 0; c < C; ++c) dst[8 * m + c] = 0.0;
        }
      }
      commit();
    };
    for (int u = 0; u < kST - 1; ++u) stage(u);
    double xm[C], x0[C], yab[C], rmax = 0.0;
    ldC<C, true>(x + o + q0, x0);
#pragma unroll
    for (int c = 0; c < C; ++c) {
      xm[c] = yab[c] = 0.0;
      xrow[q0 + c + 1] = x0[c];
    }
    __syncthreads();
    for (int p = 0; p < R; ++p) {
      {
        {
          stage(p + kST - 1);
          wait_row();
          struct {
            double a2[C], a1[C], e[C], c1[C], c2[C], b[C], l1[C], l2[C], xn[C];
          } d;
          {
            const double *src = ring + (int64_t)(p % kST) * 9 * m + q0;
#pragma unroll
            for (int c = 0; c < C; ++c) {
              d.a2[c] = src[c]; d.a1[c] = src[m + c]; d.e[c] = src[2 * m + c];
              d.c1[c] = src[3 * m + c]; d.c2[c] = src[4 * m + c]; d.b[c] = src[5 * m + c];
              d.l1[c] = src[6 * m + c]; d.l2[c] = src[7 * m + c]; d.xn[c] = src[8 * m + c];
            }
          }
          double *xr = xrow + (p & 1) * (m + 2), *xw = xrow + ((p + 1) & 1) * (m + 2);
          // next row's values for the neighbours (visible after this row's barrier)
#pragma unroll
          for (int c = 0; c < C; ++c) xw[q0 + c + 1] = d.xn[c];
          const double xl = xr[q0], xrr = xr[q0 + C + 1];
          const bool row0 = p == 0, rowl = p == R - 1;
          double a[C], bb[C];
#pragma unroll
          for (int c = 0; c < C; ++c) {
            // reference out-of-range entries: A[i, i-m] (p = 0), A[0, -1], A[n-1, n], A[i, i+m]
            const double a2 = row0 ? 0.0 : d.a2[c];
            const double a1 = (row0 && q0 + c == 0) ? 0.0 : d.a1[c];
            const double c1 = (rowl && q0 + c == m - 1) ? 0.0 : d.c1[c];
            const double c2 = rowl ? 0.0 : d.c2[c];
            double ax = d.e[c] * x0[c];
            ax = fma(a1, c == 0 ? xl : x0[c > 0 ? c - 1 : 0], ax);
            ax = fma(c1, c == C - 1 ? xrr : x0[c < C - 1 ? c + 1 : 0], ax);
            ax = fma(a2, xm[c], ax);
            ax = fma(c2, d.xn[c], ax);
            const double r = d.b[c] - ax;
            rmax = nan_max(rmax, fabs(r));
            a[c] = -d.l1[c];
            bb[c] = fma(-d.l2[c], yab[c], r);
          }
          // the thread's cells composed left to right, then the threads', the warps'
          double A = a[0], B = bb[0];
#pragma unroll
          for (int c = 1; c < C; ++c) {
            B = fma(a[c], B, bb[c]);
            A *= a[c];
          }
          warp_scan<true>(A, B, lane);
          if (lane == 31) tot[(p & 1) * nw + warp] = make_double2(A, B);
          const double Ap = __shfl_up_sync(0xffffffffu, A, 1), Bp = __shfl_up_sync(0xffffffffu, B, 1);
          __syncthreads();
          const double cw = carry_in<true>(tot + (p & 1) * nw, warp, lane, nw);
          double yin = lane == 0 ? cw : fma(Ap, cw, Bp);  // y of the column left of the thread's
          double y[C];
#pragma unroll
          for (int c = 0; c < C; ++c) {
            yin = fma(a[c], yin, bb[c]);
            y[c] = yin;
            yab[c] = yin;
            xm[c] = x0[c];
            x0[c] = d.xn[c];
          }
          stC<C, true>(N.y + o + (int64_t)p * m + q0, y);
        }
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    return block_max(rmax);
  };

  // ---- backward pass: U d = y, x_new = x + d --------------------------------
  auto backward = [&](const double *__restrict__ x, double *__restrict__ xn) {
    auto stage = [&](int p) {  // ring slot: [y 1/mu phi psi x][m]
      if (p >= 0) {
        double *dst = ring + (int64_t)(p % kST) * 9 * m + q0;
        const int64_t i0 = o + (int64_t)p * m + q0;
        cpC<C, true>(dst, N.y + i0);
        cpC<C, true>(dst + m, N.rmu + i0);
        cpC<C, true>(dst + 2 * m, N.phi + i0);
        cpC<C, true>(dst + 3 * m, N.psi + i0);
        cpC<C, true>(dst + 4 * m, x + i0);
      }
      commit();
    };
    for (int u = 0; u < kST - 1; ++u) stage(R - 1 - u);
    double dbl[C];  // d of the row below, own columns
#pragma unroll
    for (int c = 0; c < C; ++c) dbl[c] = 0.0;
    for (int p = R - 1; p >= 0; --p) {
      {
        {
          stage(p - (kST - 1));
          wait_row();
          struct {
            double y[C], rmu[C], phi[C], psi[C], x[C];
          } d;
          {
            const double *src = ring + (int64_t)(p % kST) * 9 * m + q0;
#pragma unroll
            for (int c = 0; c < C; ++c) {
              d.y[c] = src[c]; d.rmu[c] = src[m + c]; d.phi[c] = src[2 * m + c];
              d.psi[c] = src[3 * m + c]; d.x[c] = src[4 * m + c];
            }
          }
          double a[C], bb[C];
#pragma unroll
          for (int c = 0; c < C; ++c) {
            a[c] = -d.phi[c] * d.rmu[c];
            bb[c] = fma(-d.psi[c], dbl[c], d.y[c]) * d.rmu[c];
          }
          // composed right to left: d_q = bb_q + a_q d_{q+1}
          double A = a[C - 1], B = bb[C - 1];
#pragma unroll
          for (int c = C - 2; c >= 0; --c) {
            B = fma(a[c], B, bb[c]);
            A *= a[c];
          }
          warp_scan<false>(A, B, lane);
          if (lane == 0) tot[(p & 1) * nw + warp] = make_double2(A, B);
          const double Ap = __shfl_down_sync(0xffffffffu, A, 1), Bp = __shfl_down_sync(0xffffffffu, B, 1);
          __syncthreads();
          const double cw = carry_in<false>(tot + (p & 1) * nw, warp, lane, nw);
          double din = lane == 31 ? cw : fma(Ap, cw, Bp);  // d of the column right of the thread's
          double xo[C];
#pragma unroll
          for (int c = C - 1; c >= 0; --c) {
            din = fma(a[c], din, bb[c]);
            dbl[c] = din;
            xo[c] = d.x[c] + din;
          }
          stC<C, true>(xn + o + (int64_t)p * m + q0, xo);
        }
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();  // x_new complete before the next forward pass reads neighbours' cells
  };

  // ---- the reference loop (iterative.py:290-304) -----------------------------
  int cur = 0, best_buf = 0;
  double r = forward(N.x[0]);
  const double r0 = r, tl = tol[s];
  double best = r;
  int64_t k = 0;
  int32_t st = BX_STATUS_OK;
  while (r >= tl) {
    if (k >= max_iter) { st = BX_STATUS_MAX_ITER; break; }
    int nxt = 0;
    while (nxt == cur || nxt == best_buf) ++nxt;  // never overwrite the best iterate
    backward(N.x[cur], N.x[nxt]);
    cur = nxt;
    r = forward(N.x[cur]);
    ++k;
    if (history && tq == 0) history[s * max_iter + (k - 1)] = r;
    if (r < best) { best = r; best_buf = cur; }
    if (r0 > 0 && r > 1e6 * r0) { st = BX_STATUS_DIVERGED; break; }
  }
  for (int p = 0; p < R; ++p) {
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const int64_t i = (int64_t)p * m + q0 + c;
      xout[lay(i, s)] = N.x[cur][o + i];
      if (best_x) best_x[lay(i, s)] = N.x[best_buf][o + i];
    }
  }
  if (tq == 0) {
    if (iters) iters[s] = k;
    if (res) res[s] = r;
    if (best_res) best_res[s] = best;
    set_status(status, index, s, st, -1);
  }
}

// ----------------------------------------------------------------------------
// CTA-pair variant: the grid columns of a system split over the two CTAs of a
// cluster (two SMs pull the planes; one SM's ~20 B/clk was the single-CTA
// kernel's bound together with its per-row chain).  The split is a feed-
// forward pipeline: in the forward sweep the left half never needs anything
// from the right half -- it pushes the y of its last column into the right
// CTA's FIFO (st.async + mbarrier complete_tx) and runs ahead; the right CTA
// takes it as the start value of its row scan.  Backwards the roles swap.
// Credits (remote mbarrier arrives) keep the producer at most kFifo rows
// ahead; DSMEM latency stays off both chains.  One thread per column.
// ----------------------------------------------------------------------------
constexpr int kFifo = 8;

__device__ __forceinline__ void mbar_init(uint64_t *b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t *b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "W_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W_%=;\n}" ::"r"(smem_u32(b)), "r"(parity)
      : "memory");
}
__device__ __forceinline__ unsigned peer_addr(const void *p, int rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <class Lay>
__global__ void __launch_bounds__(256)
sip_scan_pair_kernel(const double *__restrict__ a2p, const double *__restrict__ a1p,
                     const double *__restrict__ ep, const double *__restrict__ c1p,
                     const double *__restrict__ c2p, const double *__restrict__ bp,
                     const double *__restrict__ tol, double *__restrict__ xout,
                     double *__restrict__ best_x, int64_t *iters, double *res, double *best_res,
                     int32_t *status, int32_t *index, double *history, Nat N,
                     const int32_t *__restrict__ setup_ok, int64_t n, int m, int64_t max_iter,
                     int use_x0, Lay lay, int nc) {
  // nc CTAs (2 or 4) of a cluster in a chain: rank r takes the boundary value
  // of rank r - 1 in the forward sweep and of rank r + 1 in the backward one
  const int64_t s = blockIdx.x / nc;
  if (!setup_ok[s]) return;  // (every CTA of the cluster)
  unsigned rank_;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank_));
  const int rank = (int)rank_;
  const bool hasL = rank > 0, hasR = rank < nc - 1;
  const int mh = m / nc;                  // columns of this CTA
  const int tq = threadIdx.x, lane = tq & 31, warp = tq >> 5, nw = mh >> 5;
  const int q = rank * mh + tq;           // own grid column
  const int R = (int)(n / m);
  extern __shared__ double sh[];
  double *xrow = sh;                                             // [2][mh + 2]
  double2 *tot = reinterpret_cast<double2 *>(sh + 2 * (mh + 2));  // [2][nw]
  double *red = sh + 2 * (mh + 2) + 4 * nw;                      // [32]
  double *rmx = red + 32;                                        // [2] residual max per sweep parity
  double *fifo = rmx + 2;                                        // [2 directions][kFifo]
  uint64_t *full = reinterpret_cast<uint64_t *>(fifo + 2 * kFifo);  // [2][kFifo]
  uint64_t *fre = full + 2 * kFifo;                              // [2][kFifo] credits
  double *ring = reinterpret_cast<double *>(fre + 2 * kFifo);     // [kST][9][mh] + edge [kST][2]
  double *edge = ring + kST * 9 * mh;
  const int64_t o = s * n;
  if (tq == 0) {
    for (int i = 0; i < 2 * kFifo; ++i) {
      mbar_init(full + i, 1);
      mbar_init(fre + i, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int p = 0; p < R; ++p) {
    const int64_t i = (int64_t)p * m + q;
    N.x[0][o + i] = use_x0 ? xout[lay(i, s)] : 0.0;
  }
  __syncthreads();
  cluster_sync_all();  // barriers live, initial iterate visible to the peer

  auto block_max = [&](double v) -> double {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v = nan_max(v, __shfl_xor_sync(0xffffffffu, v, d));
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double r = red[0];
    for (int w = 1; w < nw; ++w) r = nan_max(r, red[w]);
    return r;
  };
  auto commit = [] { asm volatile("cp.async.commit_group;" ::: "memory"); };
  auto wait_row = [] { asm volatile("cp.async.wait_group %0;" ::"n"(kST - 1) : "memory"); };
  auto cp8 = [](double *dst, const double *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
  };
  // producer side of a direction (0 forward, 1 backward): value of row number
  // `cnt` of that direction into the peer's FIFO
  auto push = [&](int dir, int cnt, double v) {
    const int peer = dir == 0 ? rank + 1 : rank - 1;
    const int slot = dir * kFifo + cnt % kFifo;
    if (cnt >= kFifo) mbar_wait(fre + slot, (unsigned)((cnt / kFifo - 1) & 1));  // the slot was read
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];"
                 ::"r"(peer_addr(fifo + slot, peer)), "d"(v), "r"(peer_addr(full + slot, peer))
                 : "memory");
  };
  auto credit = [&](int dir, int cnt) {  // consumer: row `cnt` of `dir` has been read by every thread
    const int peer = dir == 0 ? rank - 1 : rank + 1;
    const int slot = dir * kFifo + cnt % kFifo;
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];"
                 ::"r"(peer_addr(fre + slot, peer))
                 : "memory");
  };
  int nf = 0, nb = 0;  // rows of the forward / backward direction processed so far

  // ---- forward: values flow from rank r to rank r + 1 -------------------------------
  auto forward = [&](const double *__restrict__ x, int par) -> double {
    auto stage = [&](int p) {
      if (p < R) {
        double *dst = ring + (int64_t)(p % kST) * 9 * mh + tq;
        const int64_t i0 = (int64_t)p * m + q;
        cp8(dst, a2p + lay(i0, s));
        cp8(dst + mh, a1p + lay(i0, s));
        cp8(dst + 2 * mh, ep + lay(i0, s));
        cp8(dst + 3 * mh, c1p + lay(i0, s));
        cp8(dst + 4 * mh, c2p + lay(i0, s));
        cp8(dst + 5 * mh, bp + lay(i0, s));
        cp8(dst + 6 * mh, N.l1 + o + i0);
        cp8(dst + 7 * mh, N.l2 + o + i0);
        if (p + 1 < R) cp8(dst + 8 * mh, x + o + i0 + m);
        else dst[8 * mh] = 0.0;
        // the neighbouring CTA's boundary column of the next row
        if (tq == 0 && hasL) {
          if (p + 1 < R) cp8(edge + (p % kST) * 2, x + o + i0 + m - 1);
          else edge[(p % kST) * 2] = 0.0;
        }
        if (tq == mh - 1 && hasR) {
          if (p + 1 < R) cp8(edge + (p % kST) * 2 + 1, x + o + i0 + m + 1);
          else edge[(p % kST) * 2 + 1] = 0.0;
        }
      }
      commit();
    };
    for (int u = 0; u < kST - 1; ++u) stage(u);
    double xm = 0.0, x0 = x[o + q], yab = 0.0, rmax = 0.0;
    xrow[tq + 1] = x0;
    if (tq == 0) xrow[0] = hasL ? x[o + q - 1] : 0.0;
    if (tq == mh - 1) xrow[mh + 1] = hasR ? x[o + q + 1] : 0.0;
    __syncthreads();
    for (int p = 0; p < R; ++p, ++nf) {
      stage(p + kST - 1);
      wait_row();
      const int fslot = nf % kFifo;
      if (hasL && tq == 0) mbar_expect(full + fslot, 8);
      const double *src = ring + (int64_t)(p % kST) * 9 * mh + tq;
      const double xp = src[8 * mh];
      double *xr = xrow + (p & 1) * (mh + 2), *xw = xrow + ((p + 1) & 1) * (mh + 2);
      xw[tq + 1] = xp;
      if (tq == 0) xw[0] = hasL ? edge[(p % kST) * 2] : 0.0;
      if (tq == mh - 1) xw[mh + 1] = hasR ? edge[(p % kST) * 2 + 1] : 0.0;
      const double xl = xr[tq], xrr = xr[tq + 2];
      const bool row0 = p == 0, rowl = p == R - 1;
      const double a2 = row0 ? 0.0 : src[0];
      const double a1 = (row0 && q == 0) ? 0.0 : src[mh];
      const double c1 = (rowl && q == m - 1) ? 0.0 : src[3 * mh];
      const double c2 = rowl ? 0.0 : src[4 * mh];
      double ax = src[2 * mh] * x0;
      ax = fma(a1, xl, ax);
      ax = fma(c1, xrr, ax);
      ax = fma(a2, xm, ax);
      ax = fma(c2, xp, ax);
      const double r = src[5 * mh] - ax;
      rmax = nan_max(rmax, fabs(r));
      double A = -src[6 * mh], B = fma(-src[7 * mh], yab, r);
      warp_scan<true>(A, B, lane);
      if (lane == 31) tot[(p & 1) * nw + warp] = make_double2(A, B);
      __syncthreads();
      double start = 0.0;
      if (hasL) {
        // (the sweep's previous row: every thread read it before this row's barrier;
        // the last row of a sweep is credited after the loop)
        if (tq == 0 && p > 0) credit(0, nf - 1);
        mbar_wait(full + fslot, (unsigned)((nf / kFifo) & 1));
        start = fifo[fslot];
      }
      const double y = fma(A, carry_in<true>(tot + (p & 1) * nw, warp, lane, nw, start), B);
      N.y[o + (int64_t)p * m + q] = y;
      if (hasR && tq == mh - 1) push(0, nf, y);
      yab = y;
      xm = x0;
      x0 = xp;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    double rl = block_max(rmax);  // (its barriers: every thread has read the last FIFO slot)
    if (hasL && tq == 0) credit(0, nf - 1);
    if (tq == 0) rmx[par] = rl;
    cluster_sync_all();
    double rall = 0.0;  // the same reduction order in every CTA: identical loop decisions
    for (int c = 0; c < nc; ++c) {
      double rp;
      asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(rp) : "r"(peer_addr(rmx + par, c)));
      rall = nan_max(rall, rp);
    }
    return rall;
  };

  // ---- backward: values flow from rank r to rank r - 1 ------------------------------
  auto backward = [&](const double *__restrict__ x, double *__restrict__ xn) {
    auto stage = [&](int p) {
      if (p >= 0) {
        double *dst = ring + (int64_t)(p % kST) * 9 * mh + tq;
        const int64_t i0 = o + (int64_t)p * m + q;
        cp8(dst, N.y + i0);
        cp8(dst + mh, N.rmu + i0);
        cp8(dst + 2 * mh, N.phi + i0);
        cp8(dst + 3 * mh, N.psi + i0);
        cp8(dst + 4 * mh, x + i0);
      }
      commit();
    };
    for (int u = 0; u < kST - 1; ++u) stage(R - 1 - u);
    double dbl = 0.0;
    for (int p = R - 1; p >= 0; --p, ++nb) {
      stage(p - (kST - 1));
      wait_row();
      const int bslot = kFifo + nb % kFifo;
      if (hasR && tq == 0) mbar_expect(full + bslot, 8);
      const double *src = ring + (int64_t)(p % kST) * 9 * mh + tq;
      const double rmu = src[mh];
      double A = -src[2 * mh] * rmu, B = fma(-src[3 * mh], dbl, src[0]) * rmu;
      warp_scan<false>(A, B, lane);
      if (lane == 0) tot[(p & 1) * nw + warp] = make_double2(A, B);
      __syncthreads();
      double start = 0.0;
      if (hasR) {
        if (tq == 0 && p < R - 1) credit(1, nb - 1);
        mbar_wait(full + bslot, (unsigned)((nb / kFifo) & 1));
        start = fifo[bslot];
      }
      const double dl = fma(A, carry_in<false>(tot + (p & 1) * nw, warp, lane, nw, start), B);
      xn[o + (int64_t)p * m + q] = src[4 * mh] + dl;
      if (hasL && tq == 0) push(1, nb, dl);
      dbl = dl;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    if (hasR && tq == 0) credit(1, nb - 1);
    cluster_sync_all();  // x_new of every part visible before the next forward sweep
  };

  int cur = 0, best_buf = 0, par = 0;
  double r = forward(N.x[0], par);
  par ^= 1;
  const double r0 = r, tl = tol[s];
  double best = r;
  int64_t k = 0;
  int32_t st = BX_STATUS_OK;
  while (r >= tl) {
    if (k >= max_iter) { st = BX_STATUS_MAX_ITER; break; }
    int nxt = 0;
    while (nxt == cur || nxt == best_buf) ++nxt;
    backward(N.x[cur], N.x[nxt]);
    cur = nxt;
    r = forward(N.x[cur], par);
    par ^= 1;
    ++k;
    if (history && tq == 0 && rank == 0) history[s * max_iter + (k - 1)] = r;
    if (r < best) { best = r; best_buf = cur; }
    if (r0 > 0 && r > 1e6 * r0) { st = BX_STATUS_DIVERGED; break; }
  }
  for (int p = 0; p < R; ++p) {
    const int64_t i = (int64_t)p * m + q;
    xout[lay(i, s)] = N.x[cur][o + i];
    if (best_x) best_x[lay(i, s)] = N.x[best_buf][o + i];
  }
  if (tq == 0 && rank == 0) {
    if (iters) iters[s] = k;
    if (res) res[s] = r;
    if (best_res) best_res[s] = best;
    set_status(status, index, s, st, -1);
  }
  cluster_sync_all();  // no CTA leaves while its peer may still address its shared memory
}

// mu -> 1/mu in place over the natural plane (systems the setup rejected are skipped)
__global__ void invert_plane_kernel(double *mu, const int32_t *__restrict__ setup_ok, int64_t n,
                                    int64_t total) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x)
    if (setup_ok[i / n]) mu[i] = 1.0 / mu[i];
}

}  // namespace sipscan

// workspace after the wavefront solver's: setup flags | 9 natural planes
static size_t scan_flag_bytes(int64_t batch) { return ((size_t)batch * 4 + 255) & ~(size_t)255; }

bool sip_scan_applicable(int64_t n, int64_t m) { return m >= 32 && m <= 512 && m % 32 == 0 && n % m == 0; }

size_t sip_scan_workspace_bytes(int64_t batch, int64_t n, int64_t m) {
  if (!sip_scan_applicable(n, m)) return 0;
  return sip_wave_workspace_bytes(batch, n, m) + 256 + scan_flag_bytes(batch) +
         sizeof(double) * 9 * (size_t)batch * (size_t)n;
}

int sip_scan(const double *a2, const double *a1, const double *e, const double *c1,
             const double *c2, const double *b, const double *tol, double *x, double *best_x,
             int64_t *iters, double *res, double *best_res, int32_t *st, int32_t *ix,
             double *hist, double *ws, int64_t batch, int64_t n, int64_t m, double alpha,
             int64_t max_iter, int use_x0, int64_t ld, int layout, cudaStream_t stream) {
  if (!sip_scan_applicable(n, m)) {
    bxh::set_error("scan SIP needs a grid width m that is a multiple of 32 in [32, 512] and "
                   "n %% m == 0 (n=%lld, m=%lld)", (long long)n, (long long)m);
    return BX_ERR_UNSUPPORTED;
  }
  char *base = reinterpret_cast<char *>(ws) + ((sip_wave_workspace_bytes(batch, n, m) + 255) & ~(size_t)255);
  int32_t *ok = reinterpret_cast<int32_t *>(base);
  double *nat = reinterpret_cast<double *>(base + scan_flag_bytes(batch));
  const size_t pl = (size_t)batch * (size_t)n;
  // setup: ILU(0) / Stone in the wavefront kernel, factors also in natural order
  int rc = sip_wave(a2, a1, e, c1, c2, b, tol, x, best_x, iters, res, best_res, st, ix, hist, ws,
                    batch, n, m, alpha, max_iter, use_x0, ld, layout, stream, nat, ok);
  if (rc != BX_OK) return rc;
  sipscan::invert_plane_kernel<<<148 * 8, 256, 0, stream>>>(nat + 2 * pl, ok, n, (int64_t)pl);
  sipscan::Nat N{nat, nat + pl, nat + 2 * pl, nat + 3 * pl, nat + 4 * pl, nat + 5 * pl,
                 {nat + 6 * pl, nat + 7 * pl, nat + 8 * pl}};
  const size_t smem = sizeof(double) * (size_t)(2 * (m + 2) + 4 * (m / 32) + 32 + sipscan::kST * 9 * m);
  // columns per thread: measured on config 4 (m = 512): C = 1 7.47 ms, C = 2 8.04, C = 4 11.3
  // (fewer warps leave the per-row instruction stream of a warp exposed)
  int C = 1;
  const unsigned grid = (unsigned)batch;
  // CTA pair per system (two SMs per system) when the halves are whole warps
  // (developer knob BX_SCAN_PAIR: 0 = one CTA per system, 4 = four)
  static const int pair = getenv("BX_SCAN_PAIR") ? atoi(getenv("BX_SCAN_PAIR")) : 1;
  if (pair && m % 64 == 0 && m >= 128) {
    // 2 CTAs per system; 4 (BX_SCAN_PAIR=4, developer knob) measured slower on
    // config 4: 6.06 vs 5.79 ms (two CTAs share an SM, the chain gets longer)
    const int nc = (pair == 4 && m % 128 == 0 && m >= 256) ? 4 : 2;
    const int mh = (int)m / nc;
    const size_t psmem = sizeof(double) * (size_t)(2 * (mh + 2) + 4 * (mh / 32) + 32 + 2 + 2 * sipscan::kFifo) +
                         sizeof(uint64_t) * 4 * sipscan::kFifo +
                         sizeof(double) * (size_t)(sipscan::kST * 9 * mh + sipscan::kST * 2);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(nc * batch));
    cfg.blockDim = dim3((unsigned)mh);
    cfg.dynamicSmemBytes = psmem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = nc;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t err;
    if (layout == BX_LAYOUT_INTERLEAVED) {
      auto kern = sipscan::sip_scan_pair_kernel<Interleaved>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psmem);
      err = cudaLaunchKernelEx(&cfg, kern, a2, a1, e, c1, c2, b, tol, x, best_x, iters, res, best_res,
                               st, ix, hist, N, (const int32_t *)ok, n, (int)m, max_iter, use_x0,
                               Interleaved{ld}, nc);
    } else {
      auto kern = sipscan::sip_scan_pair_kernel<SystemMajor>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psmem);
      err = cudaLaunchKernelEx(&cfg, kern, a2, a1, e, c1, c2, b, tol, x, best_x, iters, res, best_res,
                               st, ix, hist, N, (const int32_t *)ok, n, (int)m, max_iter, use_x0,
                               SystemMajor{ld}, nc);
    }
    if (err != cudaSuccess) {
      bxh::set_error("scan SIP (CTA pair) launch: %s", cudaGetErrorString(err));
      return BX_ERR_CUDA;
    }
    return BX_OK;
  }
  if (const char *env = getenv("BX_SCAN_C")) {  // developer knob
    const int c = atoi(env);
    if ((c == 1 || c == 2 || c == 4) && m % (32 * c) == 0) C = c;
  }
  auto a32 = [](const void *p) { return ((uintptr_t)p & 31u) == 0; };
  const bool vec = layout == BX_LAYOUT_SYSTEM_MAJOR && C >= 2 && ld % 4 == 0 && a32(a2) && a32(a1) &&
                   a32(e) && a32(c1) && a32(c2) && a32(b);
#define BX_SCAN_LAUNCH(LAY, CC, VV, layv)                                                          \
  do {                                                                                             \
    cudaFuncSetAttribute(sipscan::sip_scan_kernel<LAY, CC, VV>,                                     \
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);                   \
    sipscan::sip_scan_kernel<LAY, CC, VV><<<grid, (unsigned)(m / CC), smem, stream>>>(              \
        a2, a1, e, c1, c2, b, tol, x, best_x, iters, res, best_res, st, ix, hist, N, ok, n, (int)m, \
        max_iter, use_x0, layv);                                                                    \
  } while (0)
  if (layout == BX_LAYOUT_INTERLEAVED) {
    if (C == 4) BX_SCAN_LAUNCH(Interleaved, 4, false, Interleaved{ld});
    else if (C == 2) BX_SCAN_LAUNCH(Interleaved, 2, false, Interleaved{ld});
    else BX_SCAN_LAUNCH(Interleaved, 1, false, Interleaved{ld});
  } else {
    if (vec && C == 4) BX_SCAN_LAUNCH(SystemMajor, 4, true, SystemMajor{ld});
    else if (vec && C == 2) BX_SCAN_LAUNCH(SystemMajor, 2, true, SystemMajor{ld});
    else if (C == 4) BX_SCAN_LAUNCH(SystemMajor, 4, false, SystemMajor{ld});
    else if (C == 2) BX_SCAN_LAUNCH(SystemMajor, 2, false, SystemMajor{ld});
    else BX_SCAN_LAUNCH(SystemMajor, 1, false, SystemMajor{ld});
  }
#undef BX_SCAN_LAUNCH
  return BX_OK;
}

}  // namespace bx
