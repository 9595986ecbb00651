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
#include <stdio.h>
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

#ifndef BX_HALO_PF
#define BX_HALO_PF 1  // L2 bulk prefetch: 0 none, 1 own segment (measured 0.473 -> 0.462 ms cfg 2), 2 own + a later CTA's (slower)
#endif

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
// one) | per warp: itU, itV [kChain + 4][K] interface iterates (slot p + 1
// for position p of the warp's chain; slots 0 and kChain + 1 stay zero, slot
// kChain + 2 is the dump of lanes without a second interface; the F sides
// published across warp boundaries are overlaid on these arrays) | misc
constexpr int kChain = 32 + 2 * kH - 1;  // left halo kH | 32 primaries | right halo kH - 1
template <int K, int M, int T>
struct HaloSmem {
  static constexpr int Q = 1 + 2 * K;
  static constexpr int NP = (int)(sizeof(TwoPort<K>) / 8);
  static constexpr int NW = T / 32;
  static constexpr int kState = Q * M * T;
  static constexpr int kHalo = 2 * kH * NP;
  static constexpr int kIt = (kChain + 4) * K;  // one array of one warp (+1: the dump slot's right neighbour)
  // F sides published across every warp boundary inside the CTA: the kH-1
  // last chunks of the warp before it, the kH first chunks of the warp after
  static constexpr int kPub = (NW - 1) * (2 * kH - 1) * (NP / 2);
  static_assert(kPub <= 2 * NW * kIt, "pubF is overlaid on the iterate arrays");
  // (K=2, M=16, T=64: 45008 B -- 5 CTAs/SM need <= 44 KB each)
  static constexpr size_t bytes = sizeof(double) * (size_t)(kState + kHalo + 2 * NW * kIt + 2);
};

// Registers: at most 168 per thread, i.e. 12 warps per SM -- each SM sub-
// partition owns 16 K registers, so a warp of 169..255-register threads fits
// only twice per sub-partition (8 warps per SM = 4 of the 64-thread CTAs,
// measured), one of <= 168 three times.  K = 1 gets no hint: it needs 96
// (with a minimum of 6 blocks the compiler spent 154: 0.48 -> 0.51 ms on
// config 5; capped at 102 for 10 blocks it spilled: 0.60 ms).
template <int K, int M, int T, bool VEC, bool SP, class Lay>
__global__ void __launch_bounds__(T, K == 2 ? 384 / T : 0)
halo_kernel(const double *__restrict__ c2p, const double *__restrict__ c1p,
            const double *__restrict__ ep, const double *__restrict__ f1p,
            const double *__restrict__ f2p, const double *__restrict__ bp,
            double *__restrict__ xp, int32_t *flags, int32_t *retry, int32_t *nzpart,
            int64_t batch, int64_t n, Lay lay, int csize, Outer outer, double rho_max,
            int pf_ahead, int32_t *index, int64_t *nz_out) {
  // the retry pass and the re-solve kernel behind this one may become
  // resident as this grid drains (they wait for its completion themselves)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  using SM = HaloSmem<K, M, T>;
  using CH = Chunk<K, M, T, VEC, SP, Lay>;
  constexpr int H = kH, NP = SM::NP, NW = SM::NW;
  static_assert(T % 32 == 0 && T >= 2 * H, "T must be a multiple of 32");
  extern __shared__ __align__(16) double smem[];
  double *state = smem;
  double *halo = smem + SM::kState;
  double *itU = halo + SM::kHalo + (threadIdx.x >> 5) * 2 * SM::kIt;  // this warp's arrays
  double *itV = itU + SM::kIt;
  double *pubF = halo + SM::kHalo;  // overlaid on the iterate arrays (dead until the sweeps)
  int *misc = reinterpret_cast<int *>(halo + SM::kHalo + 2 * NW * SM::kIt);
  // misc: [0] nz counter (int), [2..3] halo mbarrier (8-byte slot)
  uint64_t *cbar = reinterpret_cast<uint64_t *>(misc + 2);

  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
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
#if BX_HALO_PF
  if (VEC && t < (K == 2 && !SP ? 6 : 4)) {
    // warm L2 with this CTA's segment of one array per thread (TMA bulk
    // prefetch, no registers): the per-group loads of the down sweep then see
    // L2 latency after the first group.  Bytes still leave HBM exactly once.
    const double *arr[6] = {bp, ep, c1p, f1p, c2p, f2p};
    const int64_t rows = min((int64_t)(T * M), n - seg0) & ~(int64_t)3;
    if (rows > 0) {
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(arr[t] + lay(seg0, s)),
                   "r"((unsigned)(rows * sizeof(double)))
                   : "memory");
#if BX_HALO_PF > 1
      // ... and with the segment of the CTA BX_HALO_PF_AHEAD launches later
      const int64_t bn = (int64_t)blockIdx.x + pf_ahead;
      if (bn < (int64_t)gridDim.x)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(arr[t] + lay((bn % csize) * (T * M), bn / csize)),
                     "r"((unsigned)(rows * sizeof(double)))
                     : "memory");
#endif
    }
  }
#endif

  BX_TR(0);
  int32_t bad;
  int nzc;
  TwoPort<K> port;  // this chunk's two-port, out of the down sweep (top tracking)
  CH::template down<true>(state, t, s, base, n, lay, c2p, c1p, ep, f1p, f2p, bp, outer, bad, nzc, &port);
  BX_TR(1);
  const int w0 = t - lane;  // the warp's first chunk
  if (NW > 1) {  // F sides the neighbouring warps will need
    int slot = -1;
    if (warp < NW - 1 && lane > 32 - H) slot = warp * (2 * H - 1) + (lane - (32 - H + 1));
    if (warp > 0 && lane < H) slot = (warp - 1) * (2 * H - 1) + (H - 1) + lane;
    if (slot >= 0) {
      const double *v = reinterpret_cast<const double *>(&port.F);
#pragma unroll
      for (int c = 0; c < NP / 2; ++c) pubF[slot * (NP / 2) + c] = v[c];
    }
  }
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
      const double *v = reinterpret_cast<const double *>(&port);
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
  __syncthreads();  // every chunk's state rows and the published F sides are visible

  // ---------------- interfaces --------------------------------------------------
  // Every warp iterates its own chain of interfaces without CTA barriers:
  //   positions 0..kH-1      the kH interfaces left of the warp's first chunk
  //                          (second interfaces of lanes 0..kH-1),
  //   positions kH..kH+31    interface (c | c+1) of the lane's own chunk c,
  //   positions kH+32..      the kH-1 interfaces right of the warp's last chunk
  //                          (second interfaces of lanes 32-kH..30).
  // Chunks outside the CTA come from the halo slots (cluster neighbours) or
  // are absent (system ends: zero ports, inert interfaces).
  auto halo_side = [&](int side, int h, bool isE) -> Port<K> {
    Port<K> p;
    double *v = reinterpret_cast<double *>(&p);
    const double *src = halo + (side * H + h) * NP + (isE ? NP / 2 : 0);  // TwoPort = {F, E}
#pragma unroll
    for (int c = 0; c < NP / 2; ++c) v[c] = src[c];
    return p;
  };
  auto F_other = [&](int c) -> Port<K> {  // F side of chunk c outside this warp
    if (c < 0) return hasL ? halo_side(0, c + H, false) : zero_port<K>();
    if (c >= T) return hasR ? halo_side(1, c - T, false) : zero_port<K>();
    const int slot = c < w0 ? (warp - 1) * (2 * H - 1) + (c - (w0 - (H - 1)))
                            : warp * (2 * H - 1) + (H - 1) + (c - (w0 + 32));
    Port<K> p;
    double *v = reinterpret_cast<double *>(&p);
#pragma unroll
    for (int q = 0; q < NP / 2; ++q) v[q] = pubF[slot * (NP / 2) + q];
    return p;
  };
  auto E_other = [&](int c) -> Port<K> {  // E side of chunk c outside this warp
    if (c < 0) return hasL ? halo_side(0, c + H, true) : zero_port<K>();
    if (c >= T) return hasR ? halo_side(1, c - T, true) : zero_port<K>();
    return CH::port_E_state(state, c);
  };
  bool ok = true;
  MergeInfo<K> mi, mi2;
  {  // lanes without a second interface carry an inert one (all zero)
    double *z = reinterpret_cast<double *>(&mi2);
#pragma unroll
    for (int c = 0; c < NP; ++c) z[c] = 0.0;
  }
  Port<K> Fnext, F0;  // F of the next lane's chunk, of the warp's first chunk
  {
    const double *src = reinterpret_cast<const double *>(&port.F);
    double *d1 = reinterpret_cast<double *>(&Fnext), *d0 = reinterpret_cast<double *>(&F0);
#pragma unroll
    for (int c = 0; c < NP / 2; ++c) {
      d1[c] = __shfl_down_sync(0xffffffffu, src[c], 1);
      d0[c] = __shfl_sync(0xffffffffu, src[c], 0);
    }
  }
  const bool prim_early = t < T - 1 || !hasR;  // needs nothing from the halo
  if (prim_early) ok &= iface<K>(port.E, lane < 31 ? Fnext : F_other(t + 1), mi);
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
  if (!prim_early) ok &= iface<K>(port.E, F_other(t + 1), mi);
  int pos2 = kChain + 1;  // dump slot
  if (lane < H) {
    const int c = w0 - H + lane;
    ok &= iface<K>(E_other(c), lane < H - 1 ? F_other(c + 1) : F0, mi2);
    pos2 = lane;
  } else if (lane >= 32 - H && lane < 31) {
    const int c = w0 + lane + H;
    ok &= iface<K>(E_other(c), F_other(c + 1), mi2);
    pos2 = lane + 2 * H;
  }
  double rho = coupling<K>(mi);
  {
    const double r2 = coupling<K>(mi2);
    rho = (r2 > rho || r2 != r2) ? r2 : rho;
  }

  if (NW > 1) __syncthreads();  // pubF (overlaid on the iterate arrays) has been read

  // ---------------- block-Jacobi sweeps over the warp's chain -------------------
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
  const int sl = H + lane + 1, sl2 = pos2 + 1;
  Vec<K> u = mi.u.g, v = mi.v.g;
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) itU[k] = itV[(kChain + 1) * K + k] = 0.0;
  }
  stv(itU, sl, u);
  stv(itV, sl, v);
  stv(itU, sl2, mi2.u.g);
  stv(itV, sl2, mi2.v.g);
  __syncwarp();
#pragma unroll 1
  for (int it = 0; it < kNit; ++it) {
    const Vec<K> um = ldv(itU, sl - 1), vp = ldv(itV, sl + 1);
    const Vec<K> um2 = ldv(itU, sl2 - 1), vp2 = ldv(itV, sl2 + 1);
    __syncwarp();
    u = apply<K>(mi.u, um, vp);
    v = apply<K>(mi.v, um, vp);
    stv(itU, sl, u);
    stv(itV, sl, v);
    stv(itU, sl2, apply<K>(mi2.u, um2, vp2));
    stv(itV, sl2, apply<K>(mi2.v, um2, vp2));
    __syncwarp();
  }
  const Vec<K> L = ldv(itU, sl - 1), R = v;  // E of chunk t-1, F of chunk t+1
  BX_TR(5);

  // ---------------- phase 3 -------------------------------------------------------
  CH::write_x_backsub(state, t, s, base, n, lay, xp, L, R);
  BX_TR(6);

  // ---------------- flags / counters ----------------------------------------------
  // every CTA owns word [s * csize + crank] of flags / retry / nzpart (no
  // presets, no atomics on global memory)
  if (!ok && bad < 0) bad = (int32_t)seg0;
  const bool slow = !(rho <= rho_max);
  const int64_t w = s * csize + crank;
  const bool rare = __syncthreads_or(bad >= 0 || slow);
  if (retry == nullptr) {
    // no workspace (sparse-outer entry): flags is the caller's status array,
    // preset to OK / -1 / 0 by the launcher when csize > 1.  A system with any
    // zero pivot or slow interface is handed to the tree pass, which then
    // writes its final status / index (bx_direct_part.cu, mark mode).
    if (csize == 1) {
      if (t == 0) {
        flags[s] = rare ? kRetryMark : BX_STATUS_OK;
        if (index) index[s] = -1;
      }
    } else if (rare && t == 0) {
      flags[s] = kRetryMark;
    }
    if (K == 2 && nz_out) {
      nzc = __reduce_add_sync(0xffffffffu, nzc);
      if (NW > 1) {
        if (lane == 0) atomicAdd(&misc[0], nzc);
        __syncthreads();
        nzc = misc[0];
      }
      if (t == 0) {
        if (csize == 1) nz_out[s] = nzc;
        else atomicAdd(reinterpret_cast<unsigned long long *>(nz_out + s), (unsigned long long)nzc);
      }
    }
    return;
  }
  if (t == 0) {
    flags[w] = BX_STATUS_OK;
    retry[w] = 0;
  }
  if (rare) {  // say which
    __syncthreads();
    if (bad >= 0) flags[w] = BX_STATUS_ZERO_PIVOT;
    if (slow) retry[w] = 1;
  }
  if (K == 2 && nzpart) {
    nzc = __reduce_add_sync(0xffffffffu, nzc);
    if (NW > 1) {
      if (lane == 0) atomicAdd(&misc[0], nzc);
      __syncthreads();
      nzc = misc[0];
    }
    if (t == 0) nzpart[w] = nzc;
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
                       int32_t *retry, int32_t *nzpart, int64_t batch, int64_t n, Lay lay,
                       cudaStream_t stream, Outer outer, int *csize_out, int32_t *index,
                       int64_t *nz_out) {
  constexpr int rows = M * T;
  const int csize = (int)((n + rows - 1) / rows);
  if (csize > 8) return BX_ERR_UNSUPPORTED;  // (the tree kernel reports the limit)
  *csize_out = csize;
  const size_t smem = HaloSmem<K, M, T>::bytes;
  auto kern = halo_kernel<K, M, T, VEC, SP, Lay>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  static const int pf_ahead = getenv("BX_HALO_PF_AHEAD") ? atoi(getenv("BX_HALO_PF_AHEAD")) : 740;
  if (getenv("BX_HALO_DEBUG")) {
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, T, smem);
    fprintf(stderr, "halo_kernel<K=%d,M=%d,T=%d>: smem %zu B, %d CTAs/SM, csize %d\n", K, M, T, smem, nb, csize);
  }
  if (!retry && csize > 1) {  // no-workspace mode: the caller's arrays carry the words
    cudaMemsetAsync(flags, 0, sizeof(int32_t) * (size_t)batch, stream);  // BX_STATUS_OK
    if (index) cudaMemsetAsync(index, 0xff, sizeof(int32_t) * (size_t)batch, stream);  // -1
    if (nz_out) cudaMemsetAsync(nz_out, 0, sizeof(int64_t) * (size_t)batch, stream);
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
  cudaError_t err = cudaLaunchKernelEx(&cfg, kern, c2, c1, e, f1, f2, b, x, flags, retry, nzpart, batch,
                                       n, lay, csize, outer, rho_max_default(), pf_ahead, index, nz_out);
  if (err != cudaSuccess) {
    bxh::set_error("partitioned solver (interface iteration) launch: %s", cudaGetErrorString(err));
    return BX_ERR_CUDA;
  }
  return BX_OK;
}

template <int K, bool VEC, bool SP, class Lay>
static int halo_shapes(const double *c2, const double *c1, const double *e, const double *f1,
                       const double *f2, const double *b, double *x, int32_t *flags,
                       int32_t *retry, int32_t *nzpart, int64_t batch, int64_t n, Lay lay,
                       cudaStream_t stream, Outer o, int *cs, int32_t *ix, int64_t *nzo) {
  if (n <= 256) return halo_launch<K, 8, 32, VEC, SP, Lay>(c2, c1, e, f1, f2, b, x, flags, retry, nzpart, batch, n, lay, stream, o, cs, ix, nzo);
  if (n <= 512) return halo_launch<K, 8, 64, VEC, SP, Lay>(c2, c1, e, f1, f2, b, x, flags, retry, nzpart, batch, n, lay, stream, o, cs, ix, nzo);
  if (n <= 8192) return halo_launch<K, 16, 64, VEC, SP, Lay>(c2, c1, e, f1, f2, b, x, flags, retry, nzpart, batch, n, lay, stream, o, cs, ix, nzo);
  return halo_launch<K, 16, 128, VEC, SP, Lay>(c2, c1, e, f1, f2, b, x, flags, retry, nzpart, batch, n, lay, stream, o, cs, ix, nzo);
}

template <int K, bool SP>
static int halo_layouts(const double *c2, const double *c1, const double *e, const double *f1,
                        const double *f2, const double *b, double *x, int32_t *flags,
                        int32_t *retry, int32_t *nzpart, int64_t batch, int64_t n, int64_t ld,
                        int layout, cudaStream_t stream, Outer o, int *cs, int32_t *ix,
                        int64_t *nzo) {
  auto a32 = [](const void *p) { return p == nullptr || ((uintptr_t)p & 31u) == 0; };
  if (layout == BX_LAYOUT_SYSTEM_MAJOR) {
    const bool vec = ld % 4 == 0 && a32(c2) && a32(c1) && a32(e) && a32(f1) && a32(f2) && a32(b) && a32(x);
    if (vec) return halo_shapes<K, true, SP>(c2, c1, e, f1, f2, b, x, flags, retry, nzpart, batch, n, SystemMajor{ld}, stream, o, cs, ix, nzo);
    return halo_shapes<K, false, SP>(c2, c1, e, f1, f2, b, x, flags, retry, nzpart, batch, n, SystemMajor{ld}, stream, o, cs, ix, nzo);
  }
  return halo_shapes<K, false, SP>(c2, c1, e, f1, f2, b, x, flags, retry, nzpart, batch, n, Interleaved{ld}, stream, o, cs, ix, nzo);
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

// flags / retry / nzpart: [batch][*csize] int32 words, one per CTA of a
// system's cluster (direct_fixup's fs = *csize convention).
// outer_rows != nullptr: the +-2 diagonals come from the sparse lists (K = 2).
// retry == nullptr: no workspace -- flags is the caller's status array, index /
// nz are written here, marked systems carry kRetryMark (see halo_kernel).
int halo_solve(int K, const double *c2, const double *c1, const double *e, const double *f1,
               const double *f2, const double *b, double *x, int32_t *flags, int32_t *retry,
               int32_t *nzpart, int64_t batch, int64_t n, int64_t ld, int layout,
               cudaStream_t stream, const int32_t *outer_rows, const double *outer_sub2,
               const double *outer_sup2, int64_t outer_k, int *csize, int32_t *index,
               int64_t *nz) {
  const part::Outer o{outer_rows, outer_sub2, outer_sup2, outer_k};
  if (K == 1)
    return part::halo_layouts<1, false>(nullptr, c1, e, f1, nullptr, b, x, flags, retry, nullptr,
                                        batch, n, ld, layout, stream, o, csize, index, nullptr);
  if (outer_rows || outer_k == 0 && !c2)
    return part::halo_layouts<2, true>(nullptr, c1, e, f1, nullptr, b, x, flags, retry, nzpart,
                                       batch, n, ld, layout, stream, o, csize, index, nz);
  return part::halo_layouts<2, false>(c2, c1, e, f1, f2, b, x, flags, retry, nzpart, batch, n, ld,
                                      layout, stream, o, csize, index, nz);
}

}  // namespace bx
