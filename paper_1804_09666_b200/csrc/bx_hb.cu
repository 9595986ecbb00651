// Hotelling-Bodewig (Newton-Schulz) inversion of the ILU(0) triangular
// factors on the FP64 tensor cores (DMMA), and SIP with the substitutions
// replaced by products with those inverses.
//
// Reference (inverse.py, bandix 0.1.0):
//   dense_lower_factor / dense_upper_factor   72-87
//   hb_invert_dense                           94-119   X0 = diag(1/m_ii);
//       loop: P = M X; r = ||I - P||_inf; stop if r < tol; X <- X (2I - P)
//   sip_hb_solve (mode="dense")               205-241, 274-302
// The reference forms P and X(2I-P) with numpy.matmul (BLAS); results agree to
// rounding, not bitwise.
//
// B200 realisation:
//   * factors are batched: f < B are the unit-lower L_s, f >= B the upper U_s;
//     X is kept dense row-major per factor, only its triangle is ever touched;
//   * P = M X exploits the band of M (three diagonals: 3 FMAs per entry) and
//     produces the row sums of |I - P| in the same pass (atomicMax per factor);
//   * X <- 2X - X P is a triangular x triangular product: output tiles above
//     (below) the diagonal and K-blocks outside [J, I] are skipped, so only
//     N^3/3 of the dense 2N^3 flops are executed, on mma.sync.m16n8k16.f64
//     (DMMA) with cp.async double-buffered shared-memory tiles; the epilogue
//     fuses 2X - C.
#include <math.h>

#include "bx_common.cuh"
#include "bx_kernels.h"

namespace bx {
namespace hb {

constexpr int TM = 64, TN = 64, TK = 16, PADA = 4, PADB = 4;

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

__device__ __forceinline__ void dmma16816(double (&d)[4], const double (&a)[8], const double (&b)[4]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 "
      "{%0, %1, %2, %3}, {%4, %5, %6, %7, %8, %9, %10, %11}, {%12, %13, %14, %15}, "
      "{%0, %1, %2, %3};\n"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
        "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

// tile index -> (I, J) of the lower (I >= J) or upper (I <= J) triangle
__device__ __forceinline__ void tile_of(int t, int nb, bool lower, int &I, int &J) {
  // lower: row-by-row enumeration of (I, J), J <= I
  int i = (int)((sqrtf(8.0f * t + 1.0f) - 1.0f) * 0.5f);
  while ((i + 1) * (i + 2) / 2 <= t) ++i;
  while (i * (i + 1) / 2 > t) --i;
  const int j = t - i * (i + 1) / 2;
  if (lower) { I = i; J = j; } else { I = nb - 1 - i; J = nb - 1 - j; }
}

// Xn = 2 X - X P for active factors (triangular tiles only)
__global__ void __launch_bounds__(128)
hb_gemm_kernel(double *__restrict__ Xa, double *__restrict__ Xb, const int *__restrict__ parity,
               const double *__restrict__ P, const int *__restrict__ active_list, int64_t n, int nb,
               int nlower_factors) {
  __shared__ __align__(16) double As[2][TM][TK + PADA];
  __shared__ __align__(16) double Bs[2][TK][TN + PADB];
  const int f = active_list[blockIdx.y];
  const bool lower = f < nlower_factors;
  int I, J;
  tile_of(blockIdx.x, nb, lower, I, J);
  const size_t off = (size_t)f * n * n;
  const double *x = (parity[f] ? Xb : Xa) + off, *p = P + off;
  double *xn = (parity[f] ? Xa : Xb) + off;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  // K range: lower: blocks J..I ; upper: blocks I..J (in TM units)
  const int kb0 = (lower ? J : I) * TM, kb1 = (lower ? I : J) * TM + TM;  // [kb0, kb1)
  const int nk = (kb1 - kb0) / TK;
  const int row0 = I * TM, col0 = J * TN;

  auto load = [&](int kt, int buf) {
    const int k0 = kb0 + kt * TK;
    // A: 64 x 16 doubles = 512 x 16B; 128 threads x 4
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int e = tid + r * 128;        // 0..511
      const int row = e >> 3, c2 = (e & 7) * 2;
      cp_async16(&As[buf][row][c2], x + (size_t)(row0 + row) * n + k0 + c2);
    }
    // B: 16 x 64 doubles
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int e = tid + r * 128;
      const int row = e >> 5, c2 = (e & 31) * 2;
      cp_async16(&Bs[buf][row][c2], p + (size_t)(k0 + row) * n + col0 + c2);
    }
    cp_async_commit();
  };

  double acc[2][4][4];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[a][b][v] = 0.0;

  load(0, 0);
  for (int kt = 0; kt < nk; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < nk) {
      load(kt + 1, buf ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    double af[2][8], bf[4][4];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int v = 0; v < 8; ++v)
        af[a][v] = As[buf][wm + 16 * a + (lane >> 2) + 8 * (v & 1)][(lane & 3) + 4 * (v >> 1)];
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int v = 0; v < 4; ++v) bf[b][v] = Bs[buf][(lane & 3) + 4 * v][wn + 8 * b + (lane >> 2)];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) dmma16816(acc[a][b], af[a], bf[b]);
    __syncthreads();
  }
  // epilogue: Xn = 2 X - X P
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int r = row0 + wm + 16 * a + (lane >> 2) + 8 * (v >> 1);
        const int c = col0 + wn + 8 * b + 2 * (lane & 3) + (v & 1);
        const size_t idx = (size_t)r * n + c;
        xn[idx] = fma(2.0, x[idx], -acc[a][b][v]);
      }
}

// P = M X for active factors and r_f = max_i sum_j |delta_ij - P_ij| (inverse.py:90-91,112-113)
// factor f < B: L (unit diagonal, l1 = L(i,i-1), l2 = L(i,i-m)); f >= B: U (mu, phi, psi)
__global__ void __launch_bounds__(256)
hb_residual_kernel(const double *__restrict__ Xa, const double *__restrict__ Xb,
                   const int *__restrict__ parity, double *__restrict__ P,
                   const double *__restrict__ l1, const double *__restrict__ l2,
                   const double *__restrict__ mu, const double *__restrict__ phi,
                   const double *__restrict__ psi, const int *__restrict__ active_list,
                   unsigned long long *rnorm_bits, int64_t nr, int64_t n, int64_t m,
                   int64_t batch) {
  // nr = true order; n = padded order (rows >= nr are identity).  One warp
  // per row (8 rows per block): coalesced row sweeps, shuffle reductions.
  const int f = active_list[blockIdx.y];
  const int lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (i >= n) return;
  const bool lower = f < batch;
  const int64_t s = lower ? f : f - batch;
  const size_t off = (size_t)f * n * n;
  const double *x = (parity[f] ? Xb : Xa) + off;
  double *p = P + off;
  // factor coefficients of row i (row-aligned, interleaved [n][batch] scratch planes)
  double c0, c1, c2;
  int64_t k1, k2;
  if (i >= nr) {
    c0 = 1.0; c1 = c2 = 0.0; k1 = k2 = i;
  } else if (lower) {
    c0 = 1.0;
    c1 = i >= 1 ? l1[i * batch + s] : 0.0;
    c2 = i >= m ? l2[i * batch + s] : 0.0;
    k1 = i - 1; k2 = i - m;
  } else {
    c0 = mu[i * batch + s];
    c1 = i <= nr - 2 ? phi[i * batch + s] : 0.0;
    c2 = i + m <= nr - 1 ? psi[i * batch + s] : 0.0;
    k1 = i + 1; k2 = i + m;
  }
  double rsum = 0.0;
  const int64_t j0 = lower ? 0 : i, j1 = lower ? i + 1 : n;
  // the GEMM reads whole 64x64 diagonal tiles of P: keep their other triangle zero
  {
    const int64_t t0 = i & ~(int64_t)(TM - 1), t1 = t0 + TM;
    const int64_t z0 = lower ? i + 1 : t0, z1 = lower ? t1 : i;
    for (int64_t j = z0 + lane; j < z1; j += 32) p[i * n + j] = 0.0;
  }
  for (int64_t j = j0 + lane; j < j1; j += 32) {
    // X is triangular: entries of rows k1/k2 outside the triangle are zero by
    // definition (and are never stored in the ping-pong buffers)
    double v = c0 * x[i * n + j];
    const bool in1 = lower ? j <= k1 : j >= k1;
    const bool in2 = lower ? j <= k2 : j >= k2;
    if (c1 != 0.0 && in1) v = fma(c1, x[k1 * n + j], v);
    if (c2 != 0.0 && in2) v = fma(c2, x[k2 * n + j], v);
    p[i * n + j] = v;
    rsum += fabs((i == j ? 1.0 : 0.0) - v);
  }
  // row sum, then a max over rows via the ordered bits of a non-negative double
  for (int o = 16; o > 0; o >>= 1) rsum += __shfl_xor_sync(0xffffffffu, rsum, o);
  if (lane == 0) {
    if (rsum != rsum) rsum = INFINITY;
    atomicMax(rnorm_bits + f, (unsigned long long)__double_as_longlong(rsum));
  }
}

// X0 = diag(1/m_ii) (zero elsewhere in the triangle)
__global__ void hb_init_kernel(double *__restrict__ X, const double *__restrict__ mu,
                               int64_t nr, int64_t n, int64_t batch, int32_t *zero_diag) {
  const int f = blockIdx.y;
  const int64_t i = blockIdx.x;
  const bool lower = f < batch;
  const int64_t s = lower ? f : f - batch;
  double *x = X + (size_t)f * n * n + (size_t)i * n;
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) x[j] = 0.0;
  __syncthreads();
  if (threadIdx.x == 0) {
    const double d = (lower || i >= nr) ? 1.0 : mu[i * batch + s];
    if (d == 0.0) atomicMin(zero_diag + f, (int)i);
    x[i] = 1.0 / d;
  }
}

// ---------------------------------------------------------------------------
// SIP-HB iteration pieces (inverse.py:284-298)
// ---------------------------------------------------------------------------
// y_s = X v_s for one factor per CTA-row (triangular), v/y interleaved [n][batch]
__global__ void hb_apply_kernel(const double *__restrict__ Xa, const double *__restrict__ Xb,
                                const int *__restrict__ parity, const double *__restrict__ v,
                                double *__restrict__ y, const int *__restrict__ act, int64_t nr,
                                int64_t n, int64_t batch, int upper) {
  const int64_t s = act[blockIdx.y];
  const int64_t i = blockIdx.x;
  const int f = upper ? (int)(batch + s) : (int)s;
  const double *x = (parity[f] ? Xb : Xa) + (size_t)f * n * n + (size_t)i * n;
  const int64_t j0 = upper ? i : 0, j1 = upper ? nr : i + 1;
  double acc = 0.0;
  for (int64_t j = j0 + threadIdx.x; j < j1; j += blockDim.x) acc = fma(x[j], v[j * batch + s], acc);
  __shared__ double red[32];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    y[i * batch + s] = t;
  }
}

// the same product with the system's v staged once in shared memory (the
// interleaved v[j * batch + s] read costs a 32-byte sector per element) and
// APPLY_R rows per CTA, 4 rows per warp in flight (X rows are contiguous)
constexpr int APPLY_R = 32;
__global__ void __launch_bounds__(256)
hb_apply_smem_kernel(const double *__restrict__ Xa, const double *__restrict__ Xb,
                     const int *__restrict__ parity, const double *__restrict__ v,
                     double *__restrict__ y, const int *__restrict__ act, int64_t nr, int64_t n,
                     int64_t batch, int upper) {
  extern __shared__ double vs[];
  const int64_t s = act[blockIdx.y];
  const int64_t i0 = (int64_t)blockIdx.x * APPLY_R;
  const int64_t i1 = min(i0 + APPLY_R, nr);
  const int f = upper ? (int)(batch + s) : (int)s;
  const double *xf = (parity[f] ? Xb : Xa) + (size_t)f * n * n;
  // columns this row block touches: lower [0, i1), upper [i0, nr)
  const int64_t c0 = upper ? i0 : 0, c1 = upper ? nr : i1;
  for (int64_t j = c0 + threadIdx.x; j < c1; j += blockDim.x) vs[j - c0] = v[j * batch + s];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ib = i0 + warp * 4;
  if (ib >= i1) return;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  const double *xr[4];
  int64_t lo[4], hi[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int64_t i = min(ib + r, i1 - 1);
    xr[r] = xf + (size_t)i * n;
    lo[r] = upper ? i : 0;
    hi[r] = ib + r < i1 ? (upper ? nr : i + 1) : lo[r];  // rows past the block: empty
  }
  const int64_t jlo = upper ? ib : 0;
  const int64_t jhi = upper ? nr : min(ib + 4, i1);
  for (int64_t j = jlo + lane; j < jhi; j += 32) {
    const double vj = vs[j - c0];
#pragma unroll
    for (int r = 0; r < 4; ++r)
      if (j >= lo[r] && j < hi[r]) acc[r] = fma(ldg(xr[r] + j), vj, acc[r]);
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    double a = acc[r];
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0 && ib + r < i1) y[(ib + r) * batch + s] = a;
  }
}

}  // namespace hb

static inline int64_t hb_pad(int64_t n) { return (n + hb::TM - 1) / hb::TM * hb::TM; }

size_t hb_dense_bytes(int64_t batch, int64_t n) {
  const int64_t np_ = hb_pad(n);
  return sizeof(double) * 3 * (size_t)(2 * batch) * (size_t)np_ * (size_t)np_;
}

int hb_gemm(double *Xa, double *Xb, const int *parity, const double *P, const int *active_list,
            int nactive, int64_t n, int64_t batch, cudaStream_t stream) {
  const int64_t np_ = hb_pad(n);
  const int nb = (int)(np_ / hb::TM);
  const int tiles = nb * (nb + 1) / 2;
  hb::hb_gemm_kernel<<<dim3((unsigned)tiles, (unsigned)nactive), 128, 0, stream>>>(
      Xa, Xb, parity, P, active_list, np_, nb, (int)batch);
  return BX_OK;
}

int hb_residual(const double *Xa, const double *Xb, const int *parity, double *P, const double *l1,
                const double *l2, const double *mu, const double *phi, const double *psi,
                const int *active_list, int nactive, unsigned long long *rbits, int64_t n,
                int64_t m, int64_t batch, cudaStream_t stream) {
  const int64_t np_ = hb_pad(n);
  hb::hb_residual_kernel<<<dim3((unsigned)((np_ + 7) / 8), (unsigned)nactive), 256, 0, stream>>>(
      Xa, Xb, parity, P, l1, l2, mu, phi, psi, active_list, rbits, n, np_, m, batch);
  return BX_OK;
}

int hb_init(double *X, const double *mu, int64_t n, int64_t batch, int32_t *zero_diag,
            cudaStream_t stream) {
  const int64_t np_ = hb_pad(n);
  hb::hb_init_kernel<<<dim3((unsigned)np_, (unsigned)(2 * batch)), 256, 0, stream>>>(
      X, mu, n, np_, batch, zero_diag);
  return BX_OK;
}

int hb_apply(const double *Xa, const double *Xb, const int *parity, const double *v, double *y,
             const int *act, int nact, int64_t n, int64_t batch, int upper, cudaStream_t stream) {
  const int64_t np_ = hb_pad(n);
  const size_t smem = sizeof(double) * (size_t)n;
  if (smem <= 200 * 1024) {
    static size_t attr = 0;  // opt-in above 48 KB, set once per size class
    if (smem > 48 * 1024 && smem > attr) {
      cudaFuncSetAttribute(hb::hb_apply_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem);
      attr = smem;
    }
    hb::hb_apply_smem_kernel<<<dim3((unsigned)((n + hb::APPLY_R - 1) / hb::APPLY_R), (unsigned)nact),
                               256, smem, stream>>>(Xa, Xb, parity, v, y, act, n, np_, batch, upper);
  } else {
    hb::hb_apply_kernel<<<dim3((unsigned)n, (unsigned)nact), 128, 0, stream>>>(
        Xa, Xb, parity, v, y, act, n, np_, batch, upper);
  }
  return BX_OK;
}

int64_t hb_padded(int64_t n) { return hb_pad(n); }

}  // namespace bx
