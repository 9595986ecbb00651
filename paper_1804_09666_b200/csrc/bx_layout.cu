// Layout conversion between the C ABI's two storages (row-aligned diagonals):
// interleaved [n][batch] <-> system-major [batch][n] is a matrix transpose.
// Used by the ADI step (x-sweep output -> y-sweep input) and by the host
// wrappers.  Tiled through shared memory: both the read and the write side are
// coalesced 256-byte rows (32 doubles), the tile is padded against bank
// conflicts.  HBM-bound: 16 bytes of traffic per element.
#include "bx_common.cuh"
#include "bx_kernels.h"

namespace bx {

constexpr int TT = 32;

// dst[c][r] = src[r][c] for r < rows, c < cols (row strides lds, ldd)
__global__ void __launch_bounds__(256)
transpose_kernel(const double *__restrict__ src, double *__restrict__ dst, int64_t rows,
                 int64_t cols, int64_t lds, int64_t ldd, int64_t batch_stride_s,
                 int64_t batch_stride_d) {
  __shared__ double tile[TT][TT + 1];
  const int64_t r0 = (int64_t)blockIdx.y * TT, c0 = (int64_t)blockIdx.x * TT;
  const double *s = src + (int64_t)blockIdx.z * batch_stride_s;
  double *d = dst + (int64_t)blockIdx.z * batch_stride_d;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
#pragma unroll
  for (int k = 0; k < TT; k += 8) {
    const int64_t r = r0 + ty + k, c = c0 + tx;
    if (r < rows && c < cols) tile[ty + k][tx] = __ldg(s + r * lds + c);
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < TT; k += 8) {
    const int64_t c = c0 + ty + k, r = r0 + tx;
    if (r < rows && c < cols) d[c * ldd + r] = tile[tx][ty + k];
  }
}

int transpose(const double *src, double *dst, int64_t rows, int64_t cols, int64_t lds,
              int64_t ldd, int64_t nbatch, int64_t bss, int64_t bsd, cudaStream_t stream) {
  const dim3 grid((unsigned)((cols + TT - 1) / TT), (unsigned)((rows + TT - 1) / TT),
                  (unsigned)nbatch);
  transpose_kernel<<<grid, dim3(TT, 8), 0, stream>>>(src, dst, rows, cols, lds, ldd, bss, bsd);
  return BX_OK;
}

}  // namespace bx
