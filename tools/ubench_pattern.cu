// Developer microbenchmark (not product code): HBM efficiency of the access
// patterns a partitioned band solve can use on system-major data (6 input
// arrays of B*n doubles, 1 output).  Pure memory (sums only).
//   coal   : grid-stride, consecutive lanes read consecutive 32 B (ideal)
//   chunk  : lane owns M consecutive rows, 4-row groups (32 B) per array,
//            LA groups of lookahead; optional re-read of the lane's rows
//   line   : lane owns M=16 rows; the whole 128-B line of each array is
//            requested back to back (4 x 32 B), then consumed
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void ld4(const double *p, double *o) {
  asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0, %1, %2, %3}, [%4];"
               : "=d"(o[0]), "=d"(o[1]), "=d"(o[2]), "=d"(o[3])
               : "l"(p));
}
__device__ __forceinline__ void st4(double *p, const double *v) {
  asm volatile("st.global.L1::no_allocate.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(v[0]),
               "d"(v[1]), "d"(v[2]), "d"(v[3])
               : "memory");
}

struct Arr {
  const double *a[6];
  double *x;
};

__global__ void coal(Arr A, long long n4) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x) {
    double v[6][4], o[4];
#pragma unroll
    for (int k = 0; k < 6; ++k) ld4(A.a[k] + 4 * i, v[k]);
#pragma unroll
    for (int u = 0; u < 4; ++u) o[u] = v[0][u] + v[1][u] + v[2][u] + v[3][u] + v[4][u] + v[5][u];
    st4(A.x + 4 * i, o);
  }
}

// one CTA of W warps per "system segment" of W*32*M rows
template <int W, int M, int LA, int REREAD>
__global__ void __launch_bounds__(W * 32) chunk(Arr A) {
  const long long base = (long long)blockIdx.x * (W * 32 * M) + (long long)threadIdx.x * M;
  constexpr int G = M / 4, RG = LA + 1;
  double r[RG][6][4];
  double acc = 0;
#pragma unroll
  for (int g = 0; g < LA && g < G; ++g)
#pragma unroll
    for (int k = 0; k < 6; ++k) ld4(A.a[k] + base + 4 * g, r[g % RG][k]);
#pragma unroll
  for (int g = 0; g < G; ++g) {
    if (g + LA < G)
#pragma unroll
      for (int k = 0; k < 6; ++k) ld4(A.a[k] + base + 4 * (g + LA), r[(g + LA) % RG][k]);
#pragma unroll
    for (int k = 0; k < 6; ++k)
#pragma unroll
      for (int u = 0; u < 4; ++u) acc = fma(acc, 0.5, r[g % RG][k][u]);
  }
  acc = __shfl_xor_sync(0xffffffffu, acc, 1) + acc;
  __syncthreads();
  if (REREAD) {
#pragma unroll
    for (int g = G - 1; g >= 0; --g) {
      double v[6][4];
#pragma unroll
      for (int k = 0; k < 6; ++k) ld4(A.a[k] + base + 4 * g, v[k]);
      double o[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) o[u] = acc + v[0][u] + v[1][u] + v[2][u] + v[3][u] + v[4][u] + v[5][u];
      st4(A.x + base + 4 * g, o);
    }
  } else {
#pragma unroll
    for (int g = G - 1; g >= 0; --g) {
      double o[4] = {acc, acc + 1, acc + 2, acc + 3};
      st4(A.x + base + 4 * g, o);
    }
  }
}

template <int W>
__global__ void __launch_bounds__(W * 32) line16(Arr A) {
  const long long base = (long long)blockIdx.x * (W * 32 * 16) + (long long)threadIdx.x * 16;
  double acc = 0;
  double v[2][4][4];
#pragma unroll
  for (int k = 0; k < 6; ++k) {
#pragma unroll
    for (int g = 0; g < 4; ++g) ld4(A.a[k] + base + 4 * g, v[k & 1][g]);
#pragma unroll
    for (int g = 0; g < 4; ++g)
#pragma unroll
      for (int u = 0; u < 4; ++u) acc = fma(acc, 0.5, v[k & 1][g][u]);
  }
  __syncthreads();
#pragma unroll
  for (int g = 3; g >= 0; --g) {
    double o[4] = {acc, acc + 1, acc + 2, acc + 3};
    st4(A.x + base + 4 * g, o);
  }
}

static cudaEvent_t e0, e1;
template <class F>
void timeit(const char *name, F launch, double bytes, int nb, int regs) {
  for (int i = 0; i < 3; ++i) launch();
  cudaEventRecord(e0);
  for (int i = 0; i < 10; ++i) launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= 10;
  printf("%-40s regs=%3d ctas/SM=%2d %.3f ms %5.0f GB/s frac %.3f %s\n", name, regs, nb, ms,
         bytes / ms / 1e6, bytes / ms / 1e6 / 6545.9, cudaGetErrorString(cudaGetLastError()));
}

template <int W, int M, int LA, int RR>
void run_chunk(Arr A, long long rows, int occ) {
  auto k = chunk<W, M, LA, RR>;
  int smem = occ > 0 ? 227 * 1024 / occ - 1024 : 0;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int nb;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, W * 32, smem);
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, k);
  char name[96];
  snprintf(name, sizeof name, "chunk W=%d M=%d LA=%d reread=%d occ=%d", W, M, LA, RR, occ);
  const int grid = (int)(rows / (W * 32 * M));
  timeit(name, [&] { k<<<grid, W * 32, smem>>>(A); }, rows * 56.0, nb, fa.numRegs);
}

int main() {
  const long long rows = 8192LL * 4096;
  Arr A;
  for (int i = 0; i < 6; ++i) {
    double *p;
    cudaMalloc(&p, rows * 8);
    cudaMemset(p, 0, rows * 8);
    A.a[i] = p;
  }
  cudaMalloc(&A.x, rows * 8);
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int bps : {2, 4, 8, 16}) {
    char name[64];
    snprintf(name, sizeof name, "coal 256 thr x %d CTA/SM", bps);
    timeit(name, [&] { coal<<<148 * bps, 256>>>(A, rows / 4); }, rows * 56.0, bps, 0);
  }
  for (int occ : {0, 1, 2, 4}) {
    run_chunk<8, 16, 1, 0>(A, rows, occ);
    run_chunk<8, 16, 1, 1>(A, rows, occ);
  }
  run_chunk<8, 16, 2, 0>(A, rows, 0);
  run_chunk<8, 16, 3, 0>(A, rows, 0);
  run_chunk<4, 32, 1, 0>(A, rows, 0);
  run_chunk<4, 32, 1, 1>(A, rows, 0);
  run_chunk<4, 32, 2, 0>(A, rows, 0);
  run_chunk<4, 32, 1, 0>(A, rows, 2);
  run_chunk<4, 32, 1, 1>(A, rows, 2);
  run_chunk<16, 8, 1, 0>(A, rows, 0);
  run_chunk<16, 8, 1, 1>(A, rows, 0);
  run_chunk<8, 8, 1, 0>(A, rows, 0);
  run_chunk<8, 8, 1, 1>(A, rows, 0);
  run_chunk<8, 4, 0, 0>(A, rows, 0);
  run_chunk<2, 64, 1, 0>(A, rows, 0);
  run_chunk<1, 128, 1, 0>(A, rows, 0);
  for (int occ : {0, 2, 4}) {
    auto k = line16<8>;
    int smem = occ > 0 ? 227 * 1024 / occ - 1024 : 0;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int nb;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, 256, smem);
    char name[64];
    snprintf(name, sizeof name, "line16 W=8 occ=%d", occ);
    timeit(name, [&] { k<<<(int)(rows / (256 * 16)), 256, smem>>>(A); }, rows * 56.0, nb, 0);
  }
  return 0;
}
