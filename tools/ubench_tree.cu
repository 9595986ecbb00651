// Developer microbenchmark (not product code): latency of the in-warp
// boundary-lane two-port tree of bx_direct_seg.cu (one warp, clock64), and of
// its pieces: shuffles of a port, one half-merge, the full up/down sweeps.
#include <cstdio>
#include "../paper_1804_09666_b200/csrc/bx_direct_seg.cu"
namespace bxh {
void set_error(const char *, ...) {}
int check_launch(const char *) { return 0; }
}  // namespace bxh
using namespace bx::seg;
using bx::part::TwoPort;
using bx::part::Port;
using bx::part::Vec;

template <int K>
__global__ void kern(double *out, long long *cyc, int reps) {
  __shared__ double wst[2048];
  const int lane = threadIdx.x & 31;
  TwoPort<K> P;
  double *pp = reinterpret_cast<double *>(&P);
  for (int i = 0; i < (int)(sizeof(P) / 8); ++i) pp[i] = 0.01 * ((lane * 7 + i * 3) % 11) + (i % 5 == 0 ? 0.0 : 0.0);
  bool bad = false;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    Port<K> a = shfl_idx_t(P.E, (lane + 1) & 31);
    P.E.g.v[0] += a.g.v[0] * 1e-30;
  }
  long long t1 = clock64();
  for (int r = 0; r < reps; ++r) {
    Port<K> w, o;
    half_merge<K>(P.E, P.F, P.E, w, o);
    P.E.g.v[0] += o.g.v[0] * 1e-30;
  }
  long long t2 = clock64();
  for (int r = 0; r < reps; ++r) {
    TwoPort<K> Q = P;
    tree_up<K>(Q, 5, lane, wst, 64, 0, bad);
    P.F.g.v[0] += Q.F.g.v[0] * 1e-30;
  }
  long long t3 = clock64();
  for (int r = 0; r < reps; ++r) {
    Vec<K> L, R;
    for (int k = 0; k < K; ++k) L.v[k] = R.v[k] = 0.0;
    tree_down<K>(L, R, 5, lane, wst, 64, 0);
    P.F.g.v[0] += L.v[0] * 1e-30;
  }
  long long t4 = clock64();
  for (int r = 0; r < reps; ++r) {
    TwoPort<K> m;
    bx::part::MergeInfo<K> mi;
    bx::part::merge<K>(P, P, m, mi);
    P.E.g.v[0] += m.E.g.v[0] * 1e-30;
  }
  long long t5 = clock64();
  if (lane == 0) {
    cyc[0] = (t1 - t0) / reps; cyc[1] = (t2 - t1) / reps; cyc[2] = (t3 - t2) / reps; cyc[3] = (t4 - t3) / reps;
    cyc[4] = (t5 - t4) / reps;
  }
  out[threadIdx.x] = P.F.g.v[0] + P.E.g.v[0] + bad;
}

int main() {
  double *o; long long *c, h[8];
  cudaMalloc(&o, 4096); cudaMalloc(&c, 64);
  for (int K : {2, 1}) {
    for (int warps : {1, 4}) {
      if (K == 2) kern<2><<<1, 32 * warps>>>(o, c, 50); else kern<1><<<1, 32 * warps>>>(o, c, 50);
      cudaMemcpy(h, c, 40, cudaMemcpyDeviceToHost);
      printf("K=%d warps=%d: shfl-port %lld, half_merge %lld, tree_up(5) %lld, tree_down(5) %lld, full merge %lld cycles (%s)\n",
             K, warps, h[0], h[1], h[2], h[3], h[4], cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
