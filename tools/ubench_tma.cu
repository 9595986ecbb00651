// Developer microbenchmark: per-SM bulk-copy (TMA) streaming bandwidth with
// a producer warp + consumer warps ring, no compute.  Not part of the product.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned sa(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void stream(const double *src, size_t per_cta, int chunk, int pieces, int nst, unsigned long long *sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t *full = (uint64_t *)sm, *empty = full + 8;
  unsigned char *ring = sm + 256;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, ncw = blockDim.x / 32 - 1;
  if (tid == 0)
    for (int i = 0; i < nst; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(full + i)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(empty + i)), "r"(ncw));
    }
  __syncthreads();
  const char *base = (const char *)src + blockIdx.x * per_cta;
  const int steps = (int)(per_cta / chunk);
  unsigned long long acc = 0;
  if (warp == ncw) {  // producer
    int stg = 0; unsigned par = 0;
    for (int k = 0; k < steps; ++k) {
      asm volatile("{\n\t.reg .pred P;\nW1:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W1;\n}" ::"r"(sa(empty + stg)), "r"(par ^ 1u));
      if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(full + stg)), "r"((unsigned)chunk));
      __syncwarp();
      const int pb = chunk / pieces;  // chunk is a multiple of 16*pieces
      if (lane < pieces)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(ring + stg * chunk + lane * pb)), "l"(base + (size_t)k * chunk + lane * pb), "r"((unsigned)pb), "r"(sa(full + stg)) : "memory");
      if (++stg == nst) { stg = 0; par ^= 1u; }
    }
  } else {
    int stg = 0; unsigned par = 0;
    for (int k = 0; k < steps; ++k) {
      asm volatile("{\n\t.reg .pred P;\nW2:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W2;\n}" ::"r"(sa(full + stg)), "r"(par));
      acc += ((const unsigned long long *)(ring + stg * chunk))[tid];
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(empty + stg)));
      if (++stg == nst) { stg = 0; par ^= 1u; }
    }
  }
  if (acc == 0x1234) sink[0] = acc;
}

int main() {
  const size_t total = (size_t)4 << 30;
  double *src;
  unsigned long long *sink;
  cudaMalloc(&src, total);
  cudaMemset(src, 1, total);
  cudaMalloc(&sink, 8);
  for (int ctas : {64, 148}) {
    for (int chunk0 : {8192, 22528, 45056}) {
      for (int pieces : {1, 11}) {
        const int chunk = chunk0 / (16 * pieces) * (16 * pieces);
        for (int nst : {3, 4}) {
          if ((size_t)nst * chunk + 256 > 227 * 1024) continue;
          const size_t per_cta = (total / ctas) / chunk * chunk;
          const int smem = nst * chunk + 256;
          cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
          stream<<<ctas, 544, smem>>>(src, per_cta, chunk, pieces, nst, sink);
          cudaEvent_t a, b;
          cudaEventCreate(&a); cudaEventCreate(&b);
          cudaEventRecord(a);
          stream<<<ctas, 544, smem>>>(src, per_cta, chunk, pieces, nst, sink);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms; cudaEventElapsedTime(&ms, a, b);
          const double gbs = (double)per_cta * ctas / (ms / 1e3) / 1e9;
          printf("ctas=%3d chunk=%6d pieces=%2d nst=%d : %8.1f GB/s total, %6.1f GB/s per SM\n", ctas, chunk, pieces, nst, gbs, gbs / ctas);
        }
      }
    }
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
