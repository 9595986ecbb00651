// Developer harness (not product code): per-CTA phase clocks of the segment
// solver (bx_direct_seg.cu built with BX_SEG_TRACE).  Solves B random
// diagonally dominant band systems of order n, prints per-phase cycle
// statistics over CTAs.
//   BX_SEG_CFG=<cfg> tools/trace_seg K n B
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1804_09666_b200/csrc/bx_direct_seg.cu"

namespace bxh {
void set_error(const char *fmt, ...) { fprintf(stderr, "%s\n", fmt); }
int check_launch(const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { fprintf(stderr, "%s: %s\n", what, cudaGetErrorString(e)); return 2; }
  return 0;
}
}  // namespace bxh

__global__ void fill(double *p, long long n, unsigned seed, double scale, double shift) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    unsigned h = (unsigned)(i * 2654435761u) ^ seed;
    h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
    p[i] = shift + scale * ((h & 0xffffff) / 16777216.0 - 0.5);
  }
}

int main(int argc, char **argv) {
  const int K = argc > 1 ? atoi(argv[1]) : 2;
  const long long n = argc > 2 ? atoll(argv[2]) : 4096, B = argc > 3 ? atoll(argv[3]) : 8192;
  double *a[6], *x;
  for (int i = 0; i < 6; ++i) {
    cudaMalloc(&a[i], B * n * 8);
    fill<<<1024, 256>>>(a[i], B * n, 17 * i + 1, 1.0, i == K ? 5.0 : 0.0);
  }
  cudaMalloc(&x, B * n * 8);
  int32_t *flags;
  cudaMalloc(&flags, B * 8 * 4);
  int cs = 1;
  auto run = [&]() {
    if (K == 1) return bx::seg_solve(1, nullptr, a[0], a[1], a[2], nullptr, a[3], x, flags, nullptr, B, n, n, 0, &cs);
    return bx::seg_solve(2, a[0], a[1], a[2], a[3], a[4], a[5], x, flags, nullptr, B, n, n, 0, &cs);
  };
  for (int i = 0; i < 3; ++i) run();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  const int reps = 5;
  for (int i = 0; i < reps; ++i) run();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  std::vector<long long> tr(65536 * 8);
  cudaMemcpyFromSymbol(tr.data(), g_seg_trace, tr.size() * 8);
  const int nb = (int)std::min<long long>(B * cs, 65536);
  std::vector<double> ph[7];
  // concurrency: per SM, the number of CTAs alive at each CTA's start
  std::vector<std::vector<std::pair<long long, long long>>> per(256);
  for (int b = 0; b < nb; ++b) {
    const long long *r = &tr[b * 8];
    for (int k = 0; k < 4; ++k) ph[k].push_back(r[k + 1] - r[k]);
    ph[4].push_back(r[4] - r[0]);
    ph[5].push_back(r[5] - r[4]);
    ph[6].push_back(r[5] - r[0]);
    per[r[6] & 255].push_back({r[0], r[5]});
  }
  double occ = 0; long long cnt = 0;
  for (auto &v : per) {
    for (auto &a : v) {
      long long mid = (a.first + a.second) / 2; int live = 0;
      for (auto &b2 : v) live += (b2.first <= mid && mid < b2.second);
      occ += live; ++cnt;
    }
  }
  printf("  mean CTAs alive per SM at a CTA's midpoint: %.2f\n", occ / cnt);
  printf("K=%d n=%lld B=%lld cfg=%s csize=%d: %.3f ms, %.0f GB/s (frac %.3f), err=%s\n", K, n, B,
         getenv("BX_SEG_CFG") ? getenv("BX_SEG_CFG") : "auto", cs, ms,
         (2 * K + 3) * 8.0 * n * B / ms / 1e6, (2 * K + 3) * 8.0 * n * B / ms / 1e6 / 6545.9,
         cudaGetErrorString(cudaGetLastError()));
  const char *nm[7] = {"load", "phase1", "tree", "phase3", "to p3 end", "p3 end->exit", "lifetime"};
  for (int i = 0; i < 7; ++i) {
    std::sort(ph[i].begin(), ph[i].end());
    printf("  %-8s cycles: p10 %8.0f  median %8.0f  p90 %8.0f\n", nm[i], ph[i][nb / 10], ph[i][nb / 2], ph[i][nb * 9 / 10]);
  }
  return 0;
}
