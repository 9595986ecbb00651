// Developer microbenchmark: dependent-chain latencies on this GPU (clock64),
// one warp, one CTA.  Not part of the product.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(long long *out, double *dsink, float *fsink, int n) {
  __shared__ int chase[1024];
  __shared__ double dchase[1024];
  const int t = threadIdx.x;
  for (int i = t; i < 1024; i += blockDim.x) { chase[i] = (i + 1) & 1023; dchase[i] = 1.0; }
  __syncthreads();
  double a = 1.0 + t * 1e-9, b = 0.999999, c = 1e-7;
  float fa = 1.0f + t * 1e-7f, fb = 0.9999f, fc = 1e-6f;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) a = fma(a, b, c);
  t1 = clock64();
  if (t == 0) out[0] = t1 - t0;
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) a = a + c;
  t1 = clock64();
  if (t == 0) out[1] = t1 - t0;
  // FFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) fa = fmaf(fa, fb, fc);
  t1 = clock64();
  if (t == 0) out[2] = t1 - t0;
  // LDS chain (int pointer chasing)
  int p = t & 1023;
  t0 = clock64();
  for (int i = 0; i < n; ++i) p = chase[p];
  t1 = clock64();
  if (t == 0) out[3] = t1 - t0;
  // SHFL chain (double)
  double s = a;
  t0 = clock64();
  for (int i = 0; i < n; ++i) s = __shfl_xor_sync(0xffffffffu, s, 1) + 0.0;
  t1 = clock64();
  if (t == 0) out[4] = t1 - t0;
  // DDIV chain
  double d = a;
  t0 = clock64();
  for (int i = 0; i < n / 8; ++i) d = 1.0 / (d + 0.5);
  t1 = clock64();
  if (t == 0) out[5] = (t1 - t0) * 8;
  // LDS.64 double chase: value feeds index
  double v = 0.0;
  int q = t;
  t0 = clock64();
  for (int i = 0; i < n; ++i) { v += dchase[q]; q = (q + (int)v) & 1023; }
  t1 = clock64();
  if (t == 0) out[6] = t1 - t0;
  // DMUL chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) a = a * b;
  t1 = clock64();
  if (t == 0) out[7] = t1 - t0;
  dsink[t] = a + s + d + v + p;
  fsink[t] = fa;
}

int main() {
  long long *out;
  double *ds;
  float *fs;
  cudaMalloc(&out, 16 * sizeof(long long));
  cudaMalloc(&ds, 1024 * sizeof(double));
  cudaMalloc(&fs, 1024 * sizeof(float));
  const int n = 4096;
  const char *names[] = {"DFMA", "DADD", "FFMA", "LDS.32 chase", "SHFL.64+DADD", "DDIV (1/x)", "LDS.64+DADD+IADD", "DMUL"};
  for (int warps : {1, 4, 8, 16}) {
    lat<<<1, 32 * warps>>>(out, ds, fs, n);
    lat<<<1, 32 * warps>>>(out, ds, fs, n);
    long long h[16];
    cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
    printf("warps/CTA=%d\n", warps);
    for (int i = 0; i < 8; ++i) printf("  %-18s %7.2f cycles/op\n", names[i], (double)h[i] / n);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
