// Developer microbenchmark: FP64 pipe throughput per SM vs warps per SM and
// ILP, plus dependent DFMA / MUFU.RCP64H latency (clock64).  Not product code.
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void thr(double *sink, long long *cyc, int n) {
  double a[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) a[i] = 1.0 + threadIdx.x * 1e-9 + i * 1e-7;
  const double b = 0.9999999, c = 1e-9;
  __syncthreads();
  long long t0 = clock64();
  for (int k = 0; k < n; ++k) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) a[i] = fma(a[i], b, c);
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += a[i];
  if (s == 12345.0) sink[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void lat(long long *out, double *sink, int n) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.9999999, c = 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = fma(a, b, c);
  long long t1 = clock64();
  out[0] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    double r;
    asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a));
    a = r + 1.0;
  }
  t1 = clock64();
  out[1] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) a = 1.0 / a + 1.0;
  t1 = clock64();
  out[2] = t1 - t0;
  if (a == 12345.0) sink[0] = a;
}

int main() {
  double *sink;
  long long *cyc, h[256];
  cudaMalloc(&sink, 8);
  cudaMalloc(&cyc, 256 * 8);
  const int n = 4096;
  lat<<<1, 32>>>(cyc, sink, n);
  cudaMemcpy(h, cyc, 24, cudaMemcpyDeviceToHost);
  printf("latency: DFMA %.1f cyc, rcp.approx.f64+DADD %.1f cyc, 1.0/a+DADD %.1f cyc\n",
         (double)h[0] / n, (double)h[1] / n, (double)h[2] / n);
  for (int warps : {1, 2, 4, 5, 8, 16}) {
    for (int ilp : {1, 4, 8}) {
      if (ilp == 1) thr<1><<<148, warps * 32>>>(sink, cyc, n);
      if (ilp == 4) thr<4><<<148, warps * 32>>>(sink, cyc, n);
      if (ilp == 8) thr<8><<<148, warps * 32>>>(sink, cyc, n);
      cudaMemcpy(h, cyc, 148 * 8, cudaMemcpyDeviceToHost);
      double c = 0;
      for (int i = 0; i < 148; ++i) c += h[i];
      c /= 148;
      const double dfma = (double)warps * 32 * ilp * n;
      printf("warps/SM %2d ILP %d: %.2f DFMA lanes/clk/SM\n", warps, ilp, dfma / c);
    }
  }
  return 0;
}
