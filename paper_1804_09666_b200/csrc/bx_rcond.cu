// Reciprocal 1-norm condition estimate of banded systems (SURVEY 8f row f1:
// the condition gate that accompanies exact_det_band; SURVEY H7 asks for the
// per-system error to be reported with a condition estimate).
//
// LAPACK convention (dgtcon / dgbcon with norm = '1'):
//     rcond = 1 / (||A||_1 * est(||A^-1||_1)),
// A = P L U by banded Gaussian elimination with partial pivoting (U bandwidth
// 2K), est by Higham's modification of Hager's method (LAPACK dlacn2): at most
// five sign-vector iterations of A^-1 x / A^-T x plus the alternating-sign
// lower bound.  One thread per system; the factors, the iterate and the sign
// vector live in a [plane][n][batch] workspace (coalesced across systems).
#include <math.h>

#include "bx_common.cuh"
#include "bx_kernels.h"

namespace bx {
namespace rc {

template <int K>
struct Planes {
  static constexpr int W = 2 * K + 1;           // U row: columns k .. k+2K
  static constexpr int U0 = 0, L0 = W, PIV = W + K, X = W + K + 1, SG = W + K + 2;
  static constexpr int N = W + K + 3;
};

template <int K, class Lay>
__global__ void rcond_kernel(const double *__restrict__ cp, const double *__restrict__ dp,
                             const double *__restrict__ ep, const double *__restrict__ fp,
                             const double *__restrict__ gp, double *__restrict__ rcond,
                             int32_t *status, int32_t *index, double *ws, int64_t batch,
                             int64_t n, Lay lay) {
  using P = Planes<K>;
  constexpr int W = P::W;
  constexpr int DS = 8, NV = W + 1;  // staging ring: DS rows x NV values x 32 threads
  extern __shared__ double ring[];
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= batch) return;
  const int64_t pl = batch * n;
  auto Wsp = [&](int p, int64_t k) -> double & { return ws[(int64_t)p * pl + k * batch + s]; };
  constexpr int PF = 8;  // anorm: rows prefetched ahead into L1
  // coefficient of A at (i, i+o), o in -K..K (0 outside the matrix)
  auto A = [&](int64_t i, int o) -> double {
    if (i < 0 || i >= n || i + o < 0 || i + o >= n) return 0.0;
    if (K == 2) {
      const double *d = o == -2 ? cp : o == -1 ? dp : o == 0 ? ep : o == 1 ? fp : gp;
      return ldg(d + lay(i, s));
    }
    const double *d = o == -1 ? dp : o == 0 ? ep : fp;
    return ldg(d + lay(i, s));
  };
  auto pf_row = [&](int64_t i) {  // the 2K+1 coefficients of row i into L1
    if (i < 0 || i >= n) return;
    const double *dg[5] = {cp, dp, ep, fp, gp};
#pragma unroll
    for (int o = -K; o <= K; ++o) {
      const double *d = dg[o + 2];
      if (d) asm volatile("prefetch.global.L1 [%0];" ::"l"(d + lay(i, s)));
    }
  };
  auto put = [&](int64_t k, int v, int p, int64_t row) {
    double *d = ring + ((int)(k % DS) * NV + v) * 32 + threadIdx.x;
    if (row >= 0 && row < n)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(d)),
                   "l"(&Wsp(p, row))
                   : "memory");
    else
      *d = 0.0;
  };
  auto putp = [&](int64_t k, int v, const double *g) {  // g == nullptr: the value is 0
    double *d = ring + ((int)(k % DS) * NV + v) * 32 + threadIdx.x;
    if (g)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(d)),
                   "l"(g)
                   : "memory");
    else
      *d = 0.0;
  };
  auto get = [&](int64_t k, int v) -> double { return ring[((int)(k % DS) * NV + v) * 32 + threadIdx.x]; };
  auto commit = [] { asm volatile("cp.async.commit_group;" ::: "memory"); };
  auto wait = [] { asm volatile("cp.async.wait_group %0;" ::"n"(DS - 1) : "memory"); };
  // one pass: rows k = first, first + dir, ...; stage(k) puts row k's values
  auto pass = [&](int64_t first, int dir, auto stage, auto body) {
    for (int d = 0; d < DS - 1; ++d) {
      const int64_t k = first + (int64_t)d * dir;
      if (k >= 0 && k < n) stage(k);
      commit();
    }
    for (int64_t i = 0; i < n; ++i) {
      const int64_t k = first + i * dir, kn = k + (int64_t)(DS - 1) * dir;
      if (kn >= 0 && kn < n) stage(kn);
      commit();
      wait();
      body(k);
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  };
  // ||A||_1: max column sum
  double anorm = 0.0;
  for (int64_t c = 0; c < n; ++c) {
    pf_row(c + K + PF);
    double cs = 0.0;
#pragma unroll
    for (int o = -K; o <= K; ++o) cs += fabs(A(c + o, -o));
    anorm = cs > anorm || cs != cs ? cs : anorm;
  }
  // ---- P L U (window of K+1 unreduced rows, columns k .. k+2K) ------------
  double w[K + 1][W];
  auto load_row = [&](int64_t i, double *row, int64_t k) {
#pragma unroll
    for (int c = 0; c < W; ++c) row[c] = 0.0;
    if (i >= n) return;
#pragma unroll
    for (int o = -K; o <= K; ++o) {
      const int c = (int)(i + o - k);
      if (c >= 0 && c < W) row[c] = A(i, o);
    }
  };
#pragma unroll
  for (int j = 0; j <= K; ++j) load_row(j, w[j], 0);
  bool singular = false;
  int64_t zrow = -1;
  const double *dg[5] = {cp, dp, ep, fp, gp};
  pass(0, 1,
       [&](int64_t k) {  // row k+1+K, columns k+1 .. k+1+2K
         const int64_t i = k + 1 + K;
#pragma unroll
         for (int o = -K; o <= K; ++o) {
           const double *d = dg[o + 2];
           putp(k, K + o, (d && i < n && i + o >= 0 && i + o < n) ? d + lay(i, s) : nullptr);
         }
       },
       [&](int64_t k) {
    int p = 0;
    double best = fabs(w[0][0]);
#pragma unroll
    for (int j = 1; j <= K; ++j)
      if (k + j < n && fabs(w[j][0]) > best) { best = fabs(w[j][0]); p = j; }
    if (best == 0.0 && !singular) { singular = true; zrow = k; }
#pragma unroll
    for (int j = 1; j <= K; ++j)
      if (j == p) {
#pragma unroll
        for (int c = 0; c < W; ++c) { const double tmp = w[0][c]; w[0][c] = w[j][c]; w[j][c] = tmp; }
      }
    const double piv = w[0][0];
#pragma unroll
    for (int j = 1; j <= K; ++j) {
      const double mlt = piv != 0.0 ? w[j][0] / piv : 0.0;
      Wsp(P::L0 + j - 1, k) = mlt;
#pragma unroll
      for (int c = 1; c < W; ++c) w[j][c] = fma(-mlt, w[0][c], w[j][c]);
    }
#pragma unroll
    for (int c = 0; c < W; ++c) Wsp(P::U0 + c, k) = w[0][c];
    Wsp(P::PIV, k) = (double)p;
#pragma unroll
    for (int j = 0; j < K; ++j) {
#pragma unroll
      for (int c = 0; c < W - 1; ++c) w[j][c] = w[j + 1][c + 1];
      w[j][W - 1] = 0.0;
    }
#pragma unroll
    for (int c = 0; c < W; ++c) w[K][c] = get(k, c);
  });
  if (singular || anorm == 0.0) {  // LAPACK: rcond = 0 for an exactly singular U
    rcond[s] = 0.0;
    set_status(status, index, s, singular ? BX_STATUS_SINGULAR : BX_STATUS_OK,
               singular ? (int32_t)zrow : -1);
    return;
  }
  // ---- x := A^-1 x (trans = 0) or A^-T x (trans = 1), in place on plane X --
  // Every row step depends on the rows just solved: those are carried in
  // register windows (a global write read back one step later costs an L2
  // round trip per row), and each step's plane values are fetched DS rows
  // ahead with cp.async into a per-thread shared-memory ring (the plain loads
  // cannot be hoisted past the X stores: same workspace).  Same operations in
  // the same order as the plain loops.  Every value staged was written by an
  // earlier pass, or is read before this pass overwrites it.
  auto solve = [&](int trans) {
    if (!trans) {
      double win[K + 1];  // X[k .. k+K] as modified so far
#pragma unroll
      for (int j = 0; j <= K; ++j) win[j] = j < n ? Wsp(P::X, j) : 0.0;
      pass(0, 1,
           [&](int64_t k) {
             put(k, 0, P::PIV, k);
#pragma unroll
             for (int j = 1; j <= K; ++j) put(k, j, P::L0 + j - 1, k);
             put(k, K + 1, P::X, k + K + 1);
           },
           [&](int64_t k) {  // L: row swaps + eliminations
             const int p = (int)get(k, 0);
             double xk = win[0];
#pragma unroll
             for (int j = 1; j <= K; ++j)
               if (p == j) { const double t = win[j]; win[j] = xk; xk = t; }
             Wsp(P::X, k) = xk;
#pragma unroll
             for (int j = 1; j <= K; ++j)
               if (k + j < n) win[j] = fma(-get(k, j), xk, win[j]);
#pragma unroll
             for (int j = 0; j < K; ++j) win[j] = win[j + 1];
             win[K] = get(k, K + 1);
           });
      double r[W];  // r[c] = solved X[k + c], c = 1 .. 2K
#pragma unroll
      for (int c = 0; c < W; ++c) r[c] = 0.0;
      pass(n - 1, -1,
           [&](int64_t k) {
             put(k, 0, P::X, k);
#pragma unroll
             for (int c = 0; c < W; ++c) put(k, 1 + c, P::U0 + c, k);
           },
           [&](int64_t k) {  // U back substitution
             double acc = get(k, 0);
#pragma unroll
             for (int c = 1; c < W; ++c)
               if (k + c < n) acc = fma(-get(k, 1 + c), r[c], acc);
             const double xk = acc / get(k, 1);
             Wsp(P::X, k) = xk;
#pragma unroll
             for (int c = W - 1; c >= 2; --c) r[c] = r[c - 1];
             r[1] = xk;
           });
    } else {
      double q[W];  // q[c] = solved X[k - c]
#pragma unroll
      for (int c = 0; c < W; ++c) q[c] = 0.0;
      pass(0, 1,
           [&](int64_t k) {
             put(k, 0, P::X, k);
#pragma unroll
             for (int c = 0; c < W; ++c) put(k, 1 + c, P::U0 + c, k - c);
           },
           [&](int64_t k) {  // U^T forward
             double acc = get(k, 0);
#pragma unroll
             for (int c = 1; c < W; ++c)
               if (k - c >= 0) acc = fma(-get(k, 1 + c), q[c], acc);
             const double xk = acc / get(k, 1);
             Wsp(P::X, k) = xk;
#pragma unroll
             for (int c = W - 1; c >= 2; --c) q[c] = q[c - 1];
             q[1] = xk;
           });
      double v[K + 1];  // v[j] = current X[k + j], j = 1 .. K
#pragma unroll
      for (int j = 0; j <= K; ++j) v[j] = 0.0;
      pass(n - 1, -1,
           [&](int64_t k) {
             put(k, 0, P::X, k);
             put(k, 1, P::PIV, k);
#pragma unroll
             for (int j = 1; j <= K; ++j) put(k, 1 + j, P::L0 + j - 1, k);
           },
           [&](int64_t k) {  // L^T backward, swaps undone in reverse
             double xk = get(k, 0);  // untouched by the later steps' swaps (indices > k)
#pragma unroll
             for (int j = 1; j <= K; ++j)
               if (k + j < n) xk = fma(-get(k, 1 + j), v[j], xk);
             const int p = (int)get(k, 1);
             double xnew = xk;
#pragma unroll
             for (int j = 1; j <= K; ++j)
               if (p == j) { xnew = v[j]; v[j] = xk; }
             if (k + K < n) Wsp(P::X, k + K) = v[K];  // leaves the window: final
#pragma unroll
             for (int j = K; j >= 2; --j) v[j] = v[j - 1];
             v[1] = xnew;
           });
#pragma unroll
      for (int j = 1; j <= K; ++j)
        if (j - 1 < n) Wsp(P::X, j - 1) = v[j];
    }
  };
  auto asum = [&]() {
    double a = 0.0;
    pass(0, 1, [&](int64_t k) { put(k, 0, P::X, k); }, [&](int64_t k) { a += fabs(get(k, 0)); });
    return a;
  };
  auto signs = [&]() {  // x := sign(x), remembered in SG
    pass(0, 1, [&](int64_t k) { put(k, 0, P::X, k); },
         [&](int64_t k) {
           const double sg = get(k, 0) >= 0.0 ? 1.0 : -1.0;
           Wsp(P::X, k) = sg;
           Wsp(P::SG, k) = sg;
         });
  };
  auto iamax = [&]() {  // first index of max |x|
    int64_t j = 0;
    double b = -1.0;
    pass(0, 1, [&](int64_t k) { put(k, 0, P::X, k); },
         [&](int64_t k) {
           const double v = fabs(get(k, 0));
           if (v > b) { b = v; j = k; }
         });
    return j;
  };
  auto unit = [&](int64_t j) {
    for (int64_t k = 0; k < n; ++k) Wsp(P::X, k) = k == j ? 1.0 : 0.0;
  };
  // ---- dlacn2 (norm '1': kase 1 = A^-1 x, kase 2 = A^-T x) ---------------
  for (int64_t k = 0; k < n; ++k) Wsp(P::X, k) = 1.0 / (double)n;
  solve(0);
  double est;
  if (n == 1) {
    est = fabs(Wsp(P::X, 0));
  } else {
    est = asum();
    signs();
    solve(1);
    int64_t j = iamax();
    int iter = 2;
    while (true) {
      unit(j);
      solve(0);
      const double estold = est;
      est = asum();
      bool same = true;
      pass(0, 1, [&](int64_t k) { put(k, 0, P::X, k); put(k, 1, P::SG, k); },
           [&](int64_t k) { same = same && (get(k, 0) >= 0.0 ? 1.0 : -1.0) == get(k, 1); });
      if (same || est <= estold) break;  // repeated sign vector / no increase (dlacn2 70-90)
      signs();
      solve(1);
      const int64_t jlast = j;
      j = iamax();
      if (Wsp(P::X, jlast) != fabs(Wsp(P::X, j)) && iter < 5) {
        ++iter;
        continue;
      }
      break;
    }
    // alternating-sign lower bound
    double alt = 1.0;
    for (int64_t k = 0; k < n; ++k) {
      Wsp(P::X, k) = alt * (1.0 + (double)k / (double)(n - 1));
      alt = -alt;
    }
    solve(0);
    const double temp = 2.0 * (asum() / (double)(3 * n));
    if (temp > est) est = temp;
  }
  rcond[s] = est != 0.0 ? (1.0 / est) / anorm : 0.0;
  set_status(status, index, s, BX_STATUS_OK, -1);
}

}  // namespace rc

size_t rcond_workspace_bytes(int kind, int64_t batch, int64_t n) {
  const int planes = kind == 1 ? rc::Planes<1>::N : rc::Planes<2>::N;
  return sizeof(double) * (size_t)planes * (size_t)batch * (size_t)n;
}

int rcond_band(int kind, const double *c, const double *d, const double *e, const double *f,
               const double *g, double *rcond, int32_t *st, int32_t *ix, double *ws,
               int64_t batch, int64_t n, int64_t ld, int layout, cudaStream_t stream) {
  const int threads = 32;
  const dim3 grid((unsigned)((batch + threads - 1) / threads));
  if (kind == 1) {
    if (layout == BX_LAYOUT_INTERLEAVED)
      rc::rcond_kernel<1><<<grid, threads, sizeof(double) * 8 * 4 * 32, stream>>>(c, d, e, f, g, rcond, st, ix, ws, batch, n,
                                                       Interleaved{ld});
    else
      rc::rcond_kernel<1><<<grid, threads, sizeof(double) * 8 * 4 * 32, stream>>>(c, d, e, f, g, rcond, st, ix, ws, batch, n,
                                                       SystemMajor{ld});
  } else {
    if (layout == BX_LAYOUT_INTERLEAVED)
      rc::rcond_kernel<2><<<grid, threads, sizeof(double) * 8 * 6 * 32, stream>>>(c, d, e, f, g, rcond, st, ix, ws, batch, n,
                                                       Interleaved{ld});
    else
      rc::rcond_kernel<2><<<grid, threads, sizeof(double) * 8 * 6 * 32, stream>>>(c, d, e, f, g, rcond, st, ix, ws, batch, n,
                                                       SystemMajor{ld});
  }
  return BX_OK;
}

}  // namespace bx
