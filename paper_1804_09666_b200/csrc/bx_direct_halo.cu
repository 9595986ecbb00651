// Interface-iteration partitioned direct solver for banded systems of half-
// bandwidth K (K=1: NTDM, K=2: NPDM / MNPDM) -- the first pass of
// BX_ALGO_PARTITIONED.  Same solution contract as the reference solvers
// (solve_ntdm / solve_npdm / solve_mnpdm, direct.py:73-113; the elimination
// of _elim.py:30-190 in a different order): results agree with the reference
// to rounding (<= 1e-10 relative, north star), not bitwise.
//
// Chunks and their two-ports are those of bx_direct_part.cu (thread t owns M
// consecutive rows; after the down / up sweeps of bx_part_phases.cuh every
// row reads x_j = d_j - W_j.L - V_j.R).  What changes is the reduced system.
// Between adjacent chunks i and i+1 the interface unknowns are E_i (last K
// rows of chunk i) and F_{i+1} (first K rows of chunk i+1).  They couple
// strongly to each other and only through a whole chunk ("transmission") to
// the neighbouring interfaces:
//     E_i     = u.g + u.A E_{i-1} + u.B F_{i+2}
//     F_{i+1} = v.g + v.A E_{i-1} + v.B F_{i+2}          (iface() below)
// For the matrices the unpivoted reference solvers are meant for (diagonally
// dominant: the chunk's Green function decays), |u.A|, |u.B|, |v.A|, |v.B|
// are tiny (config 2, M = 16: <= 3e-5), so a block-Jacobi iteration over the
// interfaces converges by that factor per sweep: kNit sweeps replace the
// log-depth two-port tree and its cluster-wide exchange (measured: the tree
// and descent were ~18 K of a CTA's ~28 K cycle lifetime).
// Every thread holds one interface; a CTA needs only the kNit+1 nearest
// chunks of its two cluster neighbours (pushed once with st.async into its
// halo slots), whose interfaces it iterates redundantly.
//
// Guard: rho = max row sum of (|u.A| + |u.B|, |v.A| + |v.B|) over every
// interface the CTA uses bounds the error after kNit sweeps by rho^(kNit+1)
// (relative, max norm).  A system with rho > rho_max (2^-13: error <= 2^-52)
// or a non-finite rho is marked in retry[] and solved again by the two-port
// tree kernel (exact for any nonsingular reduced system); zero / non-finite
// chunk pivots flag the system for the reference-order re-solve exactly as
// in bx_direct_part.cu.  HBM traffic is the compulsory I/O.
#include <cooperative_groups.h>
#include <stdlib.h>

#include "bx_common.cuh"
#include "bx_kernels.h"
#include "bx_twoport.cuh"

namespace cg = cooperative_groups;

#ifdef BX_HALO_TRACE
// developer instrumentation (tools/trace_halo.py): per-CTA phase clocks
__device__ long long g_bx_halo_trace[4096][12];
extern "C" int bx_halo_trace_read(void *host, size_t bytes) {
  return (int)cudaMemcpyFromSymbol(host, g_bx_halo_trace,
                                   bytes < sizeof(g_bx_halo_trace) ? bytes : sizeof(g_bx_halo_trace));
}
#ifndef BX_HALO_TRACE_BASE
#define BX_HALO_TRACE_BASE 0
#endif
#define BX_TR(slot)                                                                   \
  do {                                                                                \
    const unsigned tb_ = blockIdx.x - BX_HALO_TRACE_BASE;                             \
    if (threadIdx.x == 0 && tb_ < 4096) g_bx_halo_trace[tb_][slot] = clock64();       \
  } while (0)
#endif

#include "bx_part_phases.cuh"

namespace bx {
namespace part {

constexpr int kNit = 3;       // interface sweeps
constexpr int kH = kNit + 1;  // halo chunks per side

// interface between chunk a (its E side) and the next chunk b (its F side):
// the first half of merge() -- u = a's E, v = b's F as affine functions of
// the unknowns beyond the two chunks (E of the chunk before a, F of the chunk
// after b)
template <int K>
__device__ __forceinline__ bool iface(const Port<K> &aE, const Port<K> &bF, MergeInfo<K> &mi) {
  Mat<K> S;
  const bool ok = inv_i_minus<K>(mm<K>(aE.B, bF.A), S);
  mi.u.g = mv<K>(S, vadd<K>(aE.g, mv<K>(aE.B, bF.g)));
  mi.u.A = mm<K>(S, aE.A);
  mi.u.B = mm<K>(S, mm<K>(aE.B, bF.B));
  mi.v.g = vadd<K>(bF.g, mv<K>(bF.A, mi.u.g));
  mi.v.A = mm<K>(bF.A, mi.u.A);
  mi.v.B = madd<K>(mm<K>(bF.A, mi.u.B), bF.B);
  return ok;
}

// max row sum of the interface's coupling to its neighbours (NaN propagates)
template <int K>
__device__ __forceinline__ double coupling(const MergeInfo<K> &mi) {
  double r = 0.0;
#pragma unroll
  for (int a = 0; a < K; ++a) {
    double su = 0.0, sv = 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      su += fabs(mi.u.A.m[a][k]) + fabs(mi.u.B.m[a][k]);
      sv += fabs(mi.v.A.m[a][k]) + fabs(mi.v.B.m[a][k]);
    }
    r = (su > r || su != su) ? su : r;
    r = (sv > r || sv != sv) ? sv : r;
  }
  return r;
}

template <int K>
__device__ __forceinline__ Port<K> zero_port() {
  Port<K> p;
#pragma unroll
  for (int a = 0; a < K; ++a) {
    p.g.v[a] = 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k) p.A.m[a][k] = p.B.m[a][k] = 0.0;
  }
  return p;
}

// shared memory (doubles): state[Q][M][T] | halo[2][kH] two-ports (side 0:
// chunks -kH..-1 of the left neighbour, side 1: chunks T..T+kH-1 of the right
// one) | itU, itV [T + 2 kH + 1][K] interface iterates (slot i + kH + 1 for
// interface i in [-kH-1, T+kH-1]; the two end slots stay zero) | misc
template <int K, int M, int T>
struct HaloSmem {
  static constexpr int Q = 1 + 2 * K;
  static constexpr int NP = (int)(sizeof(TwoPort<K>) / 8);
  static constexpr int NS = T + 2 * kH + 1;
  static constexpr int kState = Q * M * T;
  static constexpr int kHalo = 2 * kH * NP;
  static constexpr int kIt = NS * K;
  static constexpr size_t bytes = sizeof(double) * (size_t)(kState + kHalo + 2 * kIt + 8);
};

template <int K, int M, int T, bool VEC, bool SP, class Lay>
__global__ void __launch_bounds__(T)
halo_kernel(const double *__restrict__ c2p, const double *__restrict__ c1p,
            const double *__restrict__ ep, const double *__restrict__ f1p,
            const double *__restrict__ f2p, const double *__restrict__ bp,
            double *__restrict__ xp, int32_t *flags, int32_t *retry, int64_t *nz_out,
            int64_t batch, int64_t n, Lay lay, int csize, Outer outer, double rho_max) {
  using SM = HaloSmem<K, M, T>;
  using CH = Chunk<K, M, T, VEC, SP, Lay>;
  constexpr int H = kH, NP = SM::NP, NS = SM::NS;
  static_assert(T % 32 == 0 && T >= 2 * H, "T must be a multiple of 32");
  extern __shared__ __align__(16) double smem[];
  double *state = smem;
  double *halo = smem + SM::kState;
  double *itU = halo + SM::kHalo;
  double *itV = itU + SM::kIt;
  int *misc = reinterpret_cast<int *>(itV + SM::kIt);
  // misc: [0] nz counter (int), [2..3] halo mbarrier (8-byte slot)
  uint64_t *cbar = reinterpret_cast<uint64_t *>(misc + 2);

  const int t = threadIdx.x, lane = t & 31;
  const int crank = csize > 1 ? (int)cg::this_cluster().block_rank() : 0;
  const bool hasL = crank > 0, hasR = crank < csize - 1;
  const int64_t s = blockIdx.x / csize;
  const int64_t seg0 = (int64_t)crank * (T * M);
  const int64_t base = seg0 + (int64_t)t * M;
  if (t == 0) {
    misc[0] = 0;
    if (csize > 1) {
      // receives the neighbours' edge two-ports pushed with st.async
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(cbar)) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
  }
  if (csize > 1) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  for (int k = t; k < 2 * SM::kIt; k += T) itU[k] = 0.0;  // itU | itV are contiguous

  BX_TR(0);
  int32_t bad;
  int nzc;
  CH::down(state, t, s, base, n, lay, c2p, c1p, ep, f1p, f2p, bp, outer, bad, nzc);
  BX_TR(1);
  CH::up(state, t);
  BX_TR(2);

  // ---------------- halo exchange ---------------------------------------------
  // the first kH chunks go to the left neighbour (its side-1 slots), the last
  // kH to the right neighbour (its side-0 slots); each thread pushes its own
  // two-port (its own state rows: no CTA barrier needed first), completing
  // on the receiver's mbarrier.  A CTA exits only after its own halos arrived,
  // and nothing is pushed into a CTA that is not waiting for it.
  if (csize > 1) {
    asm volatile("barrier.cluster.wait.aligned;" ::: "memory");  // peers started: mbarriers live
    if (t == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(cbar)),
                   "r"((unsigned)(((hasL ? 1 : 0) + (hasR ? 1 : 0)) * H * NP * 8))
                   : "memory");
    const bool toL = hasL && t < H, toR = hasR && t >= T - H;
    if (toL || toR) {
      const TwoPort<K> own = CH::port(state, t);
      const double *v = reinterpret_cast<const double *>(&own);
      const int peer = toL ? crank - 1 : crank + 1;
      const double *slot = halo + ((toL ? 1 : 0) * H + (toL ? t : t - (T - H))) * NP;
      unsigned ra, rb;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_addr(slot)), "r"(peer));
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(smem_addr(cbar)), "r"(peer));
#pragma unroll
      for (int c = 0; c < NP; ++c)
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];"
                     ::"r"(ra + 8u * c), "d"(v[c]), "r"(rb)
                     : "memory");
    }
  }
  __syncthreads();  // every chunk's state rows are visible

  // ---------------- interfaces --------------------------------------------------
  // thread t: interface t (chunk t | t+1).  Left halo interfaces -kH..-1 are
  // held as second interfaces by threads 0..kH-1, right halo interfaces
  // T..T+kH-2 by threads T-kH..T-2.
  auto halo_port = [&](int side, int h) -> TwoPort<K> {
    TwoPort<K> p;
    double *v = reinterpret_cast<double *>(&p);
#pragma unroll
    for (int c = 0; c < NP; ++c) v[c] = halo[(side * H + h) * NP + c];
    return p;
  };
  bool ok = true;
  MergeInfo<K> mi, mi2;
  const Port<K> aE = CH::port_side(state, t, M - K);
  if (t < T - 1) ok &= iface<K>(aE, CH::port_side(state, t + 1, 0), mi);
  else if (!hasR) ok &= iface<K>(aE, zero_port<K>(), mi);
  BX_TR(3);
  if (hasL || hasR) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "W_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
        "@!p bra W_%=;\n}" ::"r"(smem_addr(cbar))
        : "memory");
  }
  BX_TR(4);
  if (t == T - 1 && hasR) ok &= iface<K>(aE, halo_port(1, 0).F, mi);
  int i2 = 0;
  bool sec = false;
  if (hasL && t < H) {
    const Port<K> bF = t < H - 1 ? halo_port(0, t + 1).F : CH::port_side(state, 0, 0);
    ok &= iface<K>(halo_port(0, t).E, bF, mi2);
    i2 = t - H;
    sec = true;
  } else if (hasR && t >= T - H && t < T - 1) {
    const int h = t - (T - H);
    ok &= iface<K>(halo_port(1, h).E, halo_port(1, h + 1).F, mi2);
    i2 = T + h;
    sec = true;
  }
  double rho = coupling<K>(mi);
  if (sec) {
    const double r2 = coupling<K>(mi2);
    rho = (r2 > rho || r2 != r2) ? r2 : rho;
  }

  // ---------------- block-Jacobi sweeps over the interfaces ---------------------
  auto ldv = [&](const double *a, int slot) -> Vec<K> {
    Vec<K> r;
#pragma unroll
    for (int k = 0; k < K; ++k) r.v[k] = a[slot * K + k];
    return r;
  };
  auto stv = [&](double *a, int slot, const Vec<K> &x) {
#pragma unroll
    for (int k = 0; k < K; ++k) a[slot * K + k] = x.v[k];
  };
  const int sl = t + H + 1, sl2 = i2 + H + 1;
  Vec<K> u = mi.u.g, v = mi.v.g;
  stv(itU, sl, u);
  stv(itV, sl, v);
  if (sec) {
    stv(itU, sl2, mi2.u.g);
    stv(itV, sl2, mi2.v.g);
  }
  __syncthreads();
#pragma unroll 1
  for (int it = 0; it < kNit; ++it) {
    const Vec<K> um = ldv(itU, sl - 1), vp = ldv(itV, sl + 1);
    Vec<K> um2, vp2;
    if (sec) {
      um2 = ldv(itU, sl2 - 1);
      vp2 = ldv(itV, sl2 + 1);
    }
    __syncthreads();
    u = apply<K>(mi.u, um, vp);
    v = apply<K>(mi.v, um, vp);
    stv(itU, sl, u);
    stv(itV, sl, v);
    if (sec) {
      stv(itU, sl2, apply<K>(mi2.u, um2, vp2));
      stv(itV, sl2, apply<K>(mi2.v, um2, vp2));
    }
    __syncthreads();
  }
  const Vec<K> L = ldv(itU, sl - 1), R = v;  // E of chunk t-1, F of chunk t+1
  BX_TR(5);

  // ---------------- phase 3 -------------------------------------------------------
  CH::write_x(state, t, s, base, n, lay, xp, L, R);
  BX_TR(6);

  // ---------------- flags / counters ----------------------------------------------
  // csize == 1: this CTA owns the system and writes its words itself (no
  // memsets in the launch); csize > 1: the launcher preset them to 0.
  if (!ok && bad < 0) bad = (int32_t)seg0;
  const bool any_bad = __syncthreads_or(bad >= 0);
  const bool any_slow = __syncthreads_or(!(rho <= rho_max));
  if (t == 0) {
    if (csize == 1) {
      flags[s] = any_bad ? BX_STATUS_ZERO_PIVOT : BX_STATUS_OK;
      retry[s] = any_slow ? 1 : 0;
    } else {
      if (any_bad) flags[s] = BX_STATUS_ZERO_PIVOT;
      if (any_slow) retry[s] = 1;
    }
  }
  if (K == 2 && nz_out) {
    nzc = __reduce_add_sync(0xffffffffu, nzc);
    if (lane == 0) atomicAdd(&misc[0], nzc);
    __syncthreads();
    if (t == 0) {
      if (csize == 1) nz_out[s] = misc[0];
      else atomicAdd(reinterpret_cast<unsigned long long *>(nz_out + s), (unsigned long long)misc[0]);
    }
  }
#ifdef BX_HALO_TRACE
  if (threadIdx.x == 0 && blockIdx.x - BX_HALO_TRACE_BASE < 4096u) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_bx_halo_trace[blockIdx.x - BX_HALO_TRACE_BASE][7] = clock64();
    g_bx_halo_trace[blockIdx.x - BX_HALO_TRACE_BASE][8] = smid;
  }
#endif
}

// ----------------------------------------------------------------------------
// launch configuration (the CTA shapes of bx_direct_part.cu)
// ----------------------------------------------------------------------------
static double rho_max_default() {
  static double v = -1.0;
  if (v < 0.0) {
    const char *env = getenv("BX_HALO_RHO");  // developer knob: 0 sends every system to the tree
    v = env ? atof(env) : 1.0 / 8192.0;       // 2^-13: rho^(kNit+1) <= 2^-52
  }
  return v;
}

template <int K, int M, int T, bool VEC, bool SP, class Lay>
static int halo_launch(const double *c2, const double *c1, const double *e, const double *f1,
                       const double *f2, const double *b, double *x, int32_t *flags,
                       int32_t *retry, int64_t *nz, int64_t batch, int64_t n, Lay lay,
                       cudaStream_t stream, Outer outer) {
  constexpr int rows = M * T;
  const int csize = (int)((n + rows - 1) / rows);
  if (csize > 8) return BX_ERR_UNSUPPORTED;  // (the tree kernel reports the limit)
  const size_t smem = HaloSmem<K, M, T>::bytes;
  auto kern = halo_kernel<K, M, T, VEC, SP, Lay>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (csize > 1) {  // flags | retry are contiguous (halo_solve's contract)
    cudaMemsetAsync(flags, 0, sizeof(int32_t) * 2 * (size_t)batch, stream);
    if (nz) cudaMemsetAsync(nz, 0, sizeof(int64_t) * (size_t)batch, stream);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(batch * csize));
  cfg.blockDim = dim3(T);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = csize;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t err = cudaLaunchKernelEx(&cfg, kern, c2, c1, e, f1, f2, b, x, flags, retry, nz, batch,
                                       n, lay, csize, outer, rho_max_default());
  if (err != cudaSuccess) {
    bxh::set_error("partitioned solver (interface iteration) launch: %s", cudaGetErrorString(err));
    return BX_ERR_CUDA;
  }
  return BX_OK;
}

template <int K, bool VEC, bool SP, class Lay>
static int halo_shapes(const double *c2, const double *c1, const double *e, const double *f1,
                       const double *f2, const double *b, double *x, int32_t *flags,
                       int32_t *retry, int64_t *nz, int64_t batch, int64_t n, Lay lay,
                       cudaStream_t stream, Outer o) {
  if (n <= 256) return halo_launch<K, 8, 32, VEC, SP, Lay>(c2, c1, e, f1, f2, b, x, flags, retry, nz, batch, n, lay, stream, o);
  if (n <= 512) return halo_launch<K, 8, 64, VEC, SP, Lay>(c2, c1, e, f1, f2, b, x, flags, retry, nz, batch, n, lay, stream, o);
  if (n <= 8192) return halo_launch<K, 16, 64, VEC, SP, Lay>(c2, c1, e, f1, f2, b, x, flags, retry, nz, batch, n, lay, stream, o);
  return halo_launch<K, 16, 128, VEC, SP, Lay>(c2, c1, e, f1, f2, b, x, flags, retry, nz, batch, n, lay, stream, o);
}

template <int K, bool SP>
static int halo_layouts(const double *c2, const double *c1, const double *e, const double *f1,
                        const double *f2, const double *b, double *x, int32_t *flags,
                        int32_t *retry, int64_t *nz, int64_t batch, int64_t n, int64_t ld,
                        int layout, cudaStream_t stream, Outer o) {
  auto a32 = [](const void *p) { return p == nullptr || ((uintptr_t)p & 31u) == 0; };
  if (layout == BX_LAYOUT_SYSTEM_MAJOR) {
    const bool vec = ld % 4 == 0 && a32(c2) && a32(c1) && a32(e) && a32(f1) && a32(f2) && a32(b) && a32(x);
    if (vec) return halo_shapes<K, true, SP>(c2, c1, e, f1, f2, b, x, flags, retry, nz, batch, n, SystemMajor{ld}, stream, o);
    return halo_shapes<K, false, SP>(c2, c1, e, f1, f2, b, x, flags, retry, nz, batch, n, SystemMajor{ld}, stream, o);
  }
  return halo_shapes<K, false, SP>(c2, c1, e, f1, f2, b, x, flags, retry, nz, batch, n, Interleaved{ld}, stream, o);
}

}  // namespace part

bool halo_enabled() {
  static int v = -1;
  if (v < 0) {
    const char *env = getenv("BX_PART_HALO");  // developer knob: 0 = two-port tree only
    v = env ? atoi(env) : 1;
  }
  return v != 0;
}

// flags[batch] | retry[batch] contiguous int32 words (retry = flags + batch).
// outer_rows != nullptr: the +-2 diagonals come from the sparse lists (K = 2).
int halo_solve(int K, const double *c2, const double *c1, const double *e, const double *f1,
               const double *f2, const double *b, double *x, int32_t *flags, int64_t *nz,
               int64_t batch, int64_t n, int64_t ld, int layout, cudaStream_t stream,
               const int32_t *outer_rows, const double *outer_sub2, const double *outer_sup2,
               int64_t outer_k) {
  int32_t *retry = flags + batch;
  const part::Outer o{outer_rows, outer_sub2, outer_sup2, outer_k};
  if (K == 1)
    return part::halo_layouts<1, false>(nullptr, c1, e, f1, nullptr, b, x, flags, retry, nullptr,
                                        batch, n, ld, layout, stream, o);
  if (outer_rows)
    return part::halo_layouts<2, true>(nullptr, c1, e, f1, nullptr, b, x, flags, retry, nz, batch,
                                       n, ld, layout, stream, o);
  return part::halo_layouts<2, false>(c2, c1, e, f1, f2, b, x, flags, retry, nz, batch, n, ld,
                                      layout, stream, o);
}

}  // namespace bx
