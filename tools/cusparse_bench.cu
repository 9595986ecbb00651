// Comparator (not product code): the vendor library's batched band solvers
// on the same shapes as the bench workloads, same B200, same timing rules
// (CUDA events, warm-up, L2 larger than the inputs or flushed), to place the
// hand-written kernels against cuSPARSE:
//   config 1  NTDM  B=1024 N=1024   cusparseDgtsv2StridedBatch (system-major)
//                                   cusparseDgtsvInterleavedBatch algo 0/1
//   config 5  NTDM  B=8192 N=8192   same
//   config 2  NPDM  B=8192 N=4096   cusparseDgpsvInterleavedBatch (QR)
// Reported: ms per batched solve, systems/s, fraction of the HBM roofline
// (the same algorithmic bytes as bench.py: 40 B/row TD, 56 B/row PD, against
// MEASURED_PEAKS.json's 6545.9 GB/s), max relative residual of a sample.
//   nvcc -O3 -arch=sm_100a tools/cusparse_bench.cu -lcusparse -o tools/cusparse_bench
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#include <cuda_runtime.h>
#include <cusparse.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1); } } while (0)
#define CS(x) do { cusparseStatus_t s_ = (x); if (s_ != CUSPARSE_STATUS_SUCCESS) { printf("cuSPARSE %d at %d\n", (int)s_, __LINE__); exit(1); } } while (0)

static const double kPeak = 6545.9;  // GB/s, MEASURED_PEAKS.json hbm_gbs

// diagonally dominant data like paper_1804_09666_b200.workloads (uniform
// off-diagonals, main = sum|off| + 1 + U[0,1]); layout: system-major
// (element (s, i) at s*n + i) or interleaved (i*B + s)
__global__ void gen(double *d2, double *d1, double *d0, double *u1, double *u2, double *b, long long B,
                    long long n, int K, bool interleaved, unsigned seed) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < B * n;
       t += (long long)gridDim.x * blockDim.x) {
    const long long s = interleaved ? t % B : t / n, i = interleaved ? t / B : t % n;
    auto rnd = [&](unsigned k) {
      unsigned h = (unsigned)(s * 1315423911u) ^ (unsigned)(i * 2654435761u) ^ (seed + 97u * k);
      h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
      return (h & 0xffffff) / 16777216.0;
    };
    const double a1 = i >= 1 ? 2 * rnd(1) - 1 : 0.0, c1 = i <= n - 2 ? 2 * rnd(2) - 1 : 0.0;
    const double a2 = (K == 2 && i >= 2) ? 2 * rnd(3) - 1 : 0.0, c2 = (K == 2 && i <= n - 3) ? 2 * rnd(4) - 1 : 0.0;
    if (K == 2) { d2[t] = a2; u2[t] = c2; }
    d1[t] = a1; u1[t] = c1;
    d0[t] = fabs(a1) + fabs(c1) + fabs(a2) + fabs(c2) + 1.0 + rnd(5);
    b[t] = 2 * rnd(6) - 1;
  }
}

static double sample_residual(const std::vector<double> &d2, const std::vector<double> &d1,
                              const std::vector<double> &d0, const std::vector<double> &u1,
                              const std::vector<double> &u2, const std::vector<double> &b,
                              const std::vector<double> &x, long long B, long long n, int K,
                              bool il) {
  double worst = 0;
  for (long long s = 0; s < B; s += B / 8) {
    auto at = [&](const std::vector<double> &v, long long i) { return v[il ? i * B + s : s * n + i]; };
    double rmax = 0, xmax = 0;
    for (long long i = 0; i < n; ++i) {
      double acc = at(d0, i) * at(x, i);
      if (i >= 1) acc += at(d1, i) * at(x, i - 1);
      if (i <= n - 2) acc += at(u1, i) * at(x, i + 1);
      if (K == 2 && i >= 2) acc += at(d2, i) * at(x, i - 2);
      if (K == 2 && i <= n - 3) acc += at(u2, i) * at(x, i + 2);
      rmax = fmax(rmax, fabs(at(b, i) - acc));
      xmax = fmax(xmax, fabs(at(x, i)));
    }
    worst = fmax(worst, rmax / xmax);
  }
  return worst;
}

struct Case {
  const char *name;
  long long B, n;
  int K;      // 1 tri, 2 penta
  int kind;   // 0 gtsv2StridedBatch, 1 gtsvInterleavedBatch, 2 gpsvInterleavedBatch
  int algo;
};

int main() {
  cusparseHandle_t h;
  CS(cusparseCreate(&h));
  const Case cases[] = {
      {"cfg1 NTDM gtsv2StridedBatch", 1024, 1024, 1, 0, 0},
      {"cfg1 NTDM gtsvInterleavedBatch algo0 (Thomas)", 1024, 1024, 1, 1, 0},
      {"cfg1 NTDM gtsvInterleavedBatch algo1 (LU pivoting)", 1024, 1024, 1, 1, 1},
      {"cfg5 NTDM gtsv2StridedBatch", 8192, 8192, 1, 0, 0},
      {"cfg5 NTDM gtsvInterleavedBatch algo0 (Thomas)", 8192, 8192, 1, 1, 0},
      {"cfg5 NTDM gtsvInterleavedBatch algo1 (LU pivoting)", 8192, 8192, 1, 1, 1},
      {"cfg2 NPDM gpsvInterleavedBatch (QR)", 8192, 4096, 2, 2, 0},
  };
  double *scrub;
  CK(cudaMalloc(&scrub, 512ull << 20));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (const Case &c : cases) {
    const long long N = c.B * c.n;
    const bool il = c.kind != 0;
    double *a[6], *p[6];
    for (int k = 0; k < 6; ++k) {
      CK(cudaMalloc(&a[k], N * 8));
      CK(cudaMalloc(&p[k], N * 8));
    }
    gen<<<2048, 256>>>(p[0], p[1], p[2], p[3], p[4], p[5], c.B, c.n, c.K, il, 7u);
    CK(cudaDeviceSynchronize());
    size_t bufsz = 0;
    if (c.kind == 0)
      CS(cusparseDgtsv2StridedBatch_bufferSizeExt(h, (int)c.n, a[1], a[2], a[3], a[5], (int)c.B, (int)c.n, &bufsz));
    else if (c.kind == 1)
      CS(cusparseDgtsvInterleavedBatch_bufferSizeExt(h, c.algo, (int)c.n, a[1], a[2], a[3], a[5], (int)c.B, &bufsz));
    else
      CS(cusparseDgpsvInterleavedBatch_bufferSizeExt(h, 0, (int)c.n, a[0], a[1], a[2], a[3], a[4], a[5], (int)c.B, &bufsz));
    void *buf = nullptr;
    CK(cudaMalloc(&buf, bufsz + 256));
    auto restore = [&]() {
      for (int k = 0; k < 6; ++k) CK(cudaMemcpyAsync(a[k], p[k], N * 8, cudaMemcpyDeviceToDevice));
      CK(cudaMemsetAsync(scrub, 0, 512ull << 20));  // flush L2 (inputs < L2 for cfg1)
    };
    auto solve = [&]() {
      if (c.kind == 0) CS(cusparseDgtsv2StridedBatch(h, (int)c.n, a[1], a[2], a[3], a[5], (int)c.B, (int)c.n, buf));
      else if (c.kind == 1) CS(cusparseDgtsvInterleavedBatch(h, c.algo, (int)c.n, a[1], a[2], a[3], a[5], (int)c.B, buf));
      else CS(cusparseDgpsvInterleavedBatch(h, 0, (int)c.n, a[0], a[1], a[2], a[3], a[4], a[5], (int)c.B, buf));
    };
    for (int w = 0; w < 3; ++w) { restore(); solve(); }
    const int reps = 5;
    float tot = 0;
    for (int r = 0; r < reps; ++r) {
      restore();
      cudaEventRecord(e0);
      solve();
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      tot += ms;
    }
    const double ms = tot / reps;
    std::vector<std::vector<double>> hv(6, std::vector<double>(N));
    for (int k = 0; k < 6; ++k) CK(cudaMemcpy(hv[k].data(), p[k], N * 8, cudaMemcpyDeviceToHost));
    std::vector<double> x(N);
    CK(cudaMemcpy(x.data(), a[5], N * 8, cudaMemcpyDeviceToHost));
    const double res = sample_residual(hv[0], hv[1], hv[2], hv[3], hv[4], hv[5], x, c.B, c.n, c.K, il);
    const double bytes = (c.K == 1 ? 40.0 : 56.0) * N;
    printf("%-52s B=%5lld n=%5lld  %8.3f ms  %10.0f systems/s  %7.1f GB/s  roofline frac %.3f  rel.res %.1e\n",
           c.name, c.B, c.n, ms, c.B / (ms * 1e-3), bytes / ms / 1e6, bytes / ms / 1e6 / kPeak, res);
    for (int k = 0; k < 6; ++k) { cudaFree(a[k]); cudaFree(p[k]); }
    cudaFree(buf);
  }
  cusparseDestroy(h);
  return 0;
}
