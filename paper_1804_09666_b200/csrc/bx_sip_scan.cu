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
// The factors come from the wavefront kernel's setup pass (ILU(0) / Stone
// alpha, bit-identical to ilu0_penta, iterative.py:62-124), which also leaves
// them in natural order for this kernel (1/mu instead of mu).
#include <stdlib.h>

#include "bx_common.cuh"
#include "bx_kernels.h"

namespace bx {
namespace sipscan {

constexpr int kST = 4;  // grid rows in flight: cp.async ring stages in shared memory
constexpr int kAhead = 24;  // rows the L2 prefetcher CTA runs in front of its solver

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
// scan of the warp totals tot[w] = (A, B), start value 0
template <bool UP>
__device__ __forceinline__ double carry_in(const double2 *tot, int warp, int lane, int nw) {
  // Fast path: the previous warp's map forgets what entered it (|A| * |carry|
  // is below the rounding of B: dominant rows decay by the 32 cells of a warp),
  // so the value leaving it is its B alone.  Checked per row, exact otherwise.
  const int prev = UP ? warp - 1 : warp + 1;
  if (prev >= 0 && prev < nw) {
    const double2 v = tot[prev];
    const int pp = UP ? prev - 1 : prev + 1;
    const double bprev = (pp >= 0 && pp < nw) ? fabs(tot[pp].y) : 0.0;
    if (fabs(v.x) * bprev <= 0x1p-60 * fabs(v.y) && fabs(v.x) <= 0x1p-40) return v.y;
  } else {
    return 0.0;
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
  const double c = __shfl_sync(0xffffffffu, B, src < 0 ? 0 : src);
  return src < 0 ? 0.0 : c;
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
                int use_x0, Lay lay, int *prog, int64_t batch) {
  // CTAs batch .. 2 batch - 1 (only when prog != nullptr; an experiment that is
  // off by default, see sip_scan): L2 prefetchers, one per system, on SMs the
  // solve leaves idle.  A solving CTA is fed at what
  // one SM can pull from HBM on its own requests (~20 B/clk measured); its
  // prefetcher walks kAhead rows in front of it (the solver publishes its
  // position in prog[s]) and bulk-prefetches the rows of the planes whose
  // addresses do not depend on the iteration, so the solver's copies hit L2.
  if (blockIdx.x >= batch) {
    const int64_t sp = blockIdx.x - batch;
    if (threadIdx.x >= 32 || !setup_ok[sp]) return;
    const int R = (int)(n / m), lane = threadIdx.x;
    const int64_t o = sp * n;
    const double *fw[8] = {a2p + lay(0, sp), a1p + lay(0, sp), ep + lay(0, sp), c1p + lay(0, sp),
                           c2p + lay(0, sp), bp + lay(0, sp), N.l1 + o, N.l2 + o};
    const double *bw[4] = {N.rmu + o, N.phi + o, N.psi + o, N.y + o};
    const double *mine_f = fw[lane & 7], *mine_b = bw[lane & 3];
    int ph = 0, i = 0;
    for (;;) {
      const int cur = *reinterpret_cast<volatile int *>(prog + sp);
      if (cur == 0x7fffffff) return;
      const int cph = cur / R, ci = cur % R;
      if (cph > ph) { ph = cph; i = ci; }
      if (i < R && i <= ci + kAhead) {
        const int row = (ph & 1) ? R - 1 - i : i;  // odd sweeps run upwards
        const double *src = ((ph & 1) ? mine_b : mine_f) + (int64_t)row * m;
        if (lane < ((ph & 1) ? 4 : 8))
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src),
                       "r"((unsigned)(m * sizeof(double)))
                       : "memory");
        ++i;
      } else {
        __nanosleep(100);
      }
    }
  }
  const int64_t s = blockIdx.x;
  if (!setup_ok[s]) {  // not a grid / zero pivot: reported by the setup pass
    if (prog && threadIdx.x == 0) prog[s] = 0x7fffffff;
    return;
  }
  int sweep = 0;  // sweeps started so far (even: forward, odd: backward)
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
          if (prog && tq == 0) *reinterpret_cast<volatile int *>(prog + s) = sweep * R + p;
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
    ++sweep;
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
          if (prog && tq == 0) *reinterpret_cast<volatile int *>(prog + s) = sweep * R + (R - 1 - p);
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
    ++sweep;
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
    if (prog) *reinterpret_cast<volatile int *>(prog + s) = 0x7fffffff;  // releases the prefetcher
    if (iters) iters[s] = k;
    if (res) res[s] = r;
    if (best_res) best_res[s] = best;
    set_status(status, index, s, st, -1);
  }
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
static size_t scan_flag_bytes(int64_t batch) { return ((size_t)batch * 8 + 255) & ~(size_t)255; }  // setup_ok | prog

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
  // L2 prefetcher CTAs (see sip_scan_kernel): when solvers and prefetchers are
  // all resident at once and the rows are 16-byte aligned (bulk prefetch)
  int *prog = nullptr;
  {
    // developer knob, off: measured on config 4 the prefetchers slow the solve (18.2 vs 7.47 ms)
    static const int pf = getenv("BX_SCAN_PF") ? atoi(getenv("BX_SCAN_PF")) : 0;
    auto a16 = [](const void *p) { return ((uintptr_t)p & 15u) == 0; };
    if (pf && layout == BX_LAYOUT_SYSTEM_MAJOR && 2 * batch <= 148 && ld % 2 == 0 && m % 2 == 0 &&
        a16(a2) && a16(a1) && a16(e) && a16(c1) && a16(c2) && a16(b)) {
      prog = ok + batch;
      cudaMemsetAsync(prog, 0, sizeof(int) * (size_t)batch, stream);
    }
  }
  const unsigned grid = (unsigned)(prog ? 2 * batch : batch);
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
        max_iter, use_x0, layv, prog, batch);                                                       \
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
