// hb_invert_dense(m, tol, max_iter) for a caller's dense square matrices
// (inverse.py:94-119), batched: X0 = diag(1/m_ii); loop P = M X,
// r = ||I - P||_inf, stop when r < tol, X <- X (2I - P) = 2X - X P.  The
// reference forms P and X(2I - P) with numpy.matmul (BLAS), so results agree
// to rounding, not bitwise; iteration counts and statuses are the
// reference's.  Unlike the factor inversion of bx_hb.cu (banded M, triangular
// X), M here is a general dense matrix: both products are full GEMMs on the
// FP64 tensor cores (mma.sync m16n8k16 f64, DMMA), 64x64 output tiles,
// cp.async double-buffered 16-deep K slices, fused epilogues (2X - XP) and a
// fused |I - P| row-sum pass.  Orders are padded to a multiple of 64 with an
// identity block (P and X stay block-diagonal, the padding's residual is 0).
// Host-driven iteration (one residual read per iteration): synchronises.
#include <math.h>

#include <algorithm>
#include <vector>

#include "bx_common.cuh"
#include "bx_kernels.h"

namespace bx {
namespace hbd {

constexpr int TM = 64, TN = 64, TK = 16, PAD = 4;

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void dmma16816(double (&d)[4], const double (&a)[8], const double (&b)[4]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 "
      "{%0, %1, %2, %3}, {%4, %5, %6, %7, %8, %9, %10, %11}, {%12, %13, %14, %15}, "
      "{%0, %1, %2, %3};\n"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
        "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

// C = A B (MODE 0) or C = 2 A - A B (MODE 1) for the active systems; all
// matrices [np][np] row-major, system f at f * np * np
template <int MODE>
__global__ void __launch_bounds__(128)
gemm_kernel(const double *__restrict__ A, const double *__restrict__ B, double *__restrict__ C,
            const int *__restrict__ act, int64_t np_, int nb) {
  __shared__ __align__(16) double As[2][TM][TK + PAD];
  __shared__ __align__(16) double Bs[2][TK][TN + PAD];
  const int f = act[blockIdx.y];
  const int I = blockIdx.x / nb, J = blockIdx.x % nb;
  const size_t off = (size_t)f * np_ * np_;
  const double *a = A + off, *b = B + off;
  double *c = C + off;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  const int row0 = I * TM, col0 = J * TN;
  const int nk = (int)(np_ / TK);
  auto load = [&](int kt, int buf) {
    const int64_t k0 = (int64_t)kt * TK;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int e = tid + r * 128;
      const int row = e >> 3, c2 = (e & 7) * 2;
      cp_async16(&As[buf][row][c2], a + (size_t)(row0 + row) * np_ + k0 + c2);
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int e = tid + r * 128;
      const int row = e >> 5, c2 = (e & 31) * 2;
      cp_async16(&Bs[buf][row][c2], b + (size_t)(k0 + row) * np_ + col0 + c2);
    }
    asm volatile("cp.async.commit_group;");
  };
  double acc[2][4][4];
#pragma unroll
  for (int x = 0; x < 2; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[x][y][v] = 0.0;
  load(0, 0);
  for (int kt = 0; kt < nk; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < nk) {
      load(kt + 1, buf ^ 1);
      asm volatile("cp.async.wait_group 1;");
    } else {
      asm volatile("cp.async.wait_group 0;");
    }
    __syncthreads();
    double af[2][8], bf[4][4];
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
      for (int v = 0; v < 8; ++v)
        af[x][v] = As[buf][wm + 16 * x + (lane >> 2) + 8 * (v & 1)][(lane & 3) + 4 * (v >> 1)];
#pragma unroll
    for (int y = 0; y < 4; ++y)
#pragma unroll
      for (int v = 0; v < 4; ++v) bf[y][v] = Bs[buf][(lane & 3) + 4 * v][wn + 8 * y + (lane >> 2)];
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) dmma16816(acc[x][y], af[x], bf[y]);
    __syncthreads();
  }
#pragma unroll
  for (int x = 0; x < 2; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int r = row0 + wm + 16 * x + (lane >> 2) + 8 * (v >> 1);
        const int cc = col0 + wn + 8 * y + 2 * (lane & 3) + (v & 1);
        const size_t idx = (size_t)r * np_ + cc;
        c[idx] = MODE == 0 ? acc[x][y][v] : fma(2.0, a[idx], -acc[x][y][v]);
      }
}

// r_f = max_i sum_j |delta_ij - P_ij| (inverse.py:90-91): one warp per row,
// max over rows through the ordered bits of a non-negative double
__global__ void __launch_bounds__(256)
resid_kernel(const double *__restrict__ P, const int *__restrict__ act,
             unsigned long long *rbits, int64_t np_) {
  const int f = act[blockIdx.y];
  const int lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (i >= np_) return;
  const double *p = P + (size_t)f * np_ * np_ + (size_t)i * np_;
  double rs = 0.0;
  for (int64_t j = lane; j < np_; j += 32) rs += fabs((i == j ? 1.0 : 0.0) - p[j]);
  for (int o = 16; o > 0; o >>= 1) rs += __shfl_xor_sync(0xffffffffu, rs, o);
  if (lane == 0) {
    if (rs != rs) rs = INFINITY;
    atomicMax(rbits + f, (unsigned long long)__double_as_longlong(rs));
  }
}

// Mp = [[M, 0], [0, I]], X0 = diag(1/m_ii) (padding rows 1); zero_diag[f] =
// first i < n with m_ii == 0 (ZeroDiagonal, inverse.py:104-106)
__global__ void init_kernel(const double *__restrict__ M, int64_t n, int64_t ldm, int64_t sstride,
                            double *__restrict__ Mp, double *__restrict__ X, int64_t np_,
                            int32_t *zero_diag) {
  const int f = blockIdx.y;
  const int64_t i = blockIdx.x;
  double *mp = Mp + (size_t)f * np_ * np_ + (size_t)i * np_;
  double *x = X + (size_t)f * np_ * np_ + (size_t)i * np_;
  const double *m = M + (size_t)f * sstride + (size_t)i * ldm;
  for (int64_t j = threadIdx.x; j < np_; j += blockDim.x) {
    mp[j] = (i < n && j < n) ? m[j] : (i == j ? 1.0 : 0.0);
    x[j] = 0.0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const double d = i < n ? m[i] : 1.0;
    if (d == 0.0) atomicMin(zero_diag + f, (int)i);
    x[i] = 1.0 / d;
  }
}

__global__ void copy_out_kernel(const double *__restrict__ Xa, const double *__restrict__ Xb,
                                const int *__restrict__ parity, double *__restrict__ X, int64_t n,
                                int64_t ldx, int64_t sstride, int64_t np_) {
  const int f = blockIdx.y;
  const int64_t i = blockIdx.x;
  const double *src = (parity[f] ? Xb : Xa) + (size_t)f * np_ * np_ + (size_t)i * np_;
  double *dst = X + (size_t)f * sstride + (size_t)i * ldx;
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) dst[j] = src[j];
}

static int64_t pad(int64_t n) { return (n + TM - 1) / TM * TM; }

}  // namespace hbd

size_t hb_dense_invert_workspace_bytes(int64_t batch, int64_t n) {
  const int64_t np_ = hbd::pad(n);
  return sizeof(double) * 4 * (size_t)batch * (size_t)np_ * (size_t)np_ +
         (size_t)batch * (8 + 4 * 3) + 256;
}

int hb_dense_invert(const double *M, int64_t n, int64_t ldm, int64_t mstride, int64_t batch,
                    const double *tol, int64_t max_iter, double *X, int64_t ldx, int64_t xstride,
                    int64_t *iterations, double *residual, double *history, int32_t *status,
                    int32_t *index, void *ws, cudaStream_t st) {
  using namespace hbd;
  const int64_t np_ = pad(n);
  const int nb = (int)(np_ / TM);
  const size_t mat = (size_t)np_ * np_;
  double *Mp = reinterpret_cast<double *>(ws);
  double *Xa = Mp + batch * mat, *Xb = Xa + batch * mat, *P = Xb + batch * mat;
  unsigned long long *rbits = reinterpret_cast<unsigned long long *>(P + batch * mat);
  int32_t *zd = reinterpret_cast<int32_t *>(rbits + batch);
  int *act = reinterpret_cast<int *>(zd + batch);
  int *parity = act + batch;

  std::vector<int32_t> hz(batch, 0x7fffffff);
  cudaMemcpyAsync(zd, hz.data(), sizeof(int32_t) * batch, cudaMemcpyHostToDevice, st);
  init_kernel<<<dim3((unsigned)np_, (unsigned)batch), 256, 0, st>>>(M, n, ldm, mstride, Mp, Xa, np_, zd);
  std::vector<double> htol(batch);
  cudaMemcpyAsync(htol.data(), tol, sizeof(double) * batch, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(hz.data(), zd, sizeof(int32_t) * batch, cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  std::vector<int> par(batch, 0), active, hst(batch, BX_STATUS_OK), hix(batch, -1);
  std::vector<int64_t> hit(batch, 0);
  std::vector<double> hres(batch, NAN);
  std::vector<double> hhist(history ? (size_t)batch * (max_iter + 1) : 0, NAN);
  for (int64_t f = 0; f < batch; ++f) {
    if (hz[f] != 0x7fffffff) {
      hst[f] = BX_STATUS_ZERO_DIAG;
      hix[f] = hz[f];
    } else {
      active.push_back((int)f);
    }
  }
  std::vector<unsigned long long> hb(batch);
  for (int64_t it = 0; it <= max_iter && !active.empty(); ++it) {
    const int na = (int)active.size();
    cudaMemcpyAsync(act, active.data(), sizeof(int) * na, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(parity, par.data(), sizeof(int) * batch, cudaMemcpyHostToDevice, st);
    cudaMemsetAsync(rbits, 0, sizeof(unsigned long long) * batch, st);
    // P = M X: X is the current parity buffer of each system -- launch per
    // parity class (all active systems share the parity: they started together
    // and flip together)
    const double *Xc = par[active[0]] ? Xb : Xa;
    double *Xn = par[active[0]] ? Xa : Xb;
    gemm_kernel<0><<<dim3((unsigned)(nb * nb), (unsigned)na), 128, 0, st>>>(Mp, Xc, P, act, np_, nb);
    resid_kernel<<<dim3((unsigned)((np_ + 7) / 8), (unsigned)na), 256, 0, st>>>(P, act, rbits, np_);
    cudaMemcpyAsync(hb.data(), rbits, sizeof(unsigned long long) * batch, cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return bxh::check_launch("bx_hb_invert_dense_f64");
    std::vector<int> still;
    for (int f : active) {
      double r;
      memcpy(&r, &hb[f], 8);
      if (history) hhist[(size_t)f * (max_iter + 1) + it] = r;
      hres[f] = r;
      hit[f] = it;
      if (r < htol[f]) {
        hst[f] = BX_STATUS_OK;  // converged: X is the current iterate
      } else {
        still.push_back(f);
        if (it == max_iter) hst[f] = BX_STATUS_MAX_ITER;  // X updated once more, as the reference
      }
    }
    if (!still.empty()) {
      cudaMemcpyAsync(act, still.data(), sizeof(int) * still.size(), cudaMemcpyHostToDevice, st);
      gemm_kernel<1><<<dim3((unsigned)(nb * nb), (unsigned)still.size()), 128, 0, st>>>(Xc, P, Xn, act,
                                                                                        np_, nb);
      for (int f : still) par[f] ^= 1;
    }
    active.swap(still);
  }
  cudaMemcpyAsync(parity, par.data(), sizeof(int) * batch, cudaMemcpyHostToDevice, st);
  if (X)
    copy_out_kernel<<<dim3((unsigned)n, (unsigned)batch), 256, 0, st>>>(Xa, Xb, parity, X, n, ldx,
                                                                       xstride, np_);
  if (iterations) cudaMemcpyAsync(iterations, hit.data(), sizeof(int64_t) * batch, cudaMemcpyHostToDevice, st);
  if (residual) cudaMemcpyAsync(residual, hres.data(), sizeof(double) * batch, cudaMemcpyHostToDevice, st);
  if (history)
    cudaMemcpyAsync(history, hhist.data(), sizeof(double) * hhist.size(), cudaMemcpyHostToDevice, st);
  if (status) cudaMemcpyAsync(status, hst.data(), sizeof(int32_t) * batch, cudaMemcpyHostToDevice, st);
  if (index) cudaMemcpyAsync(index, hix.data(), sizeof(int32_t) * batch, cudaMemcpyHostToDevice, st);
  cudaStreamSynchronize(st);  // the host vectors above are the copies' sources
  return bxh::check_launch("bx_hb_invert_dense_f64");
}

}  // namespace bx
