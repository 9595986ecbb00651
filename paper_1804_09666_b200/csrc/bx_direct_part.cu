// Partitioned ("two-port tree") direct solvers for banded systems of half-
// bandwidth K (K=1 tridiagonal: NTDM; K=2 pentadiagonal: NPDM / MNPDM).
//
// Throughput path (BX_ALGO_PARTITIONED).  Same solution contract as the
// reference solvers (solve_ntdm/solve_npdm/solve_mnpdm, direct.py:73-113),
// different elimination order, so results agree to rounding (north-star
// tolerance 1e-10 relative on nonsingular well-conditioned systems), not
// bitwise.  The bit-exact path is bx_direct_seq.cu.
//
// Decomposition (one system per cluster of C CTAs, all data on chip):
//   * thread t of a CTA owns a chunk of M consecutive rows;
//   * phase 1 (registers + smem): a downward elimination of the chunk with
//     the coupling to the K unknowns left of the chunk carried as a "left
//     spike" W, then an upward elimination carrying the right spike V, so that
//     every row of the chunk reads   x_j = d_j - W_j . L - V_j . R
//     with L / R the K unknowns just outside the chunk.  These 1+2K numbers
//     per row stay in shared memory.
//   * the chunk's first K and last K rows form a "two-port"
//         F = gF + AF L + BF R,   E = gE + AE L + BE R        (K-vectors, KxK)
//     Two adjacent segments merge into one two-port by eliminating their
//     shared interface (a KxK solve); a binary tree of merges over the CTA's
//     chunks (shared memory) and then over the cluster's CTAs (DSMEM)
//     reduces the system to its root, whose L = R = 0.
//   * the tree is descended to hand every chunk its L and R, and phase 3
//     writes x_j = d_j - W_j.L - V_j.R.
// HBM traffic is the compulsory I/O (K=2: 6 reads + 1 write per row; K=1:
// 4 + 1): intermediates never leave the SM.
#include <cooperative_groups.h>
#include <stdlib.h>

#include "bx_common.cuh"
#include "bx_kernels.h"
#include "bx_twoport.cuh"

namespace cg = cooperative_groups;

#ifdef BX_TRACE
// developer instrumentation (tools/trace_part.py): per-CTA phase clocks
__device__ long long g_bx_trace[4096][24];
extern "C" int bx_trace_read(void *host, size_t bytes) {
  return (int)cudaMemcpyFromSymbol(host, g_bx_trace, bytes < sizeof(g_bx_trace) ? bytes : sizeof(g_bx_trace));
}
#ifndef BX_TRACE_BASE
#define BX_TRACE_BASE 0
#endif
#define BX_TR(slot)                                                                  \
  do {                                                                               \
    const unsigned tb_ = blockIdx.x - BX_TRACE_BASE;                                 \
    if (threadIdx.x == 0 && tb_ < 4096) g_bx_trace[tb_][slot] = clock64();           \
  } while (0)
#else
#define BX_TR(slot) \
  do {              \
  } while (0)
#endif

#include "bx_part_phases.cuh"

namespace bx {
namespace part {

// per-row state kept in smem between the passes: Q = 1 + 2K doubles
//   down pass: p (x_{j+1} coeff), q (x_{j+2} coeff, K=2), y, W[K]  (normalised)
//   up pass  : d, W[K], V[K]
template <int K>
struct Cfg {
  static constexpr int Q = 1 + 2 * K;
};

// shared-memory layout (doubles): state[Q][M][T] | info[20][T] | wport[T/4] |
// wlr[T/4][2K] | croots[8] (cluster roots, pushed by every CTA) | misc
template <int K, int M, int T>
struct Smem {
  static constexpr int Q = Cfg<K>::Q;
  static constexpr int NW = T / 32;
  static constexpr int kState = Q * M * T;
  static constexpr int kInfo = T * (int)(sizeof(MergeInfo<K>) / 8);  // SoA, T nodes
  // in-warp tree levels (all warps); the remaining NU nodes are reduced by
  // warp 0.  K=2 merges are FP64-heavy: hand them to one warp early; K=1
  // merges are cheap: stay warp-parallel longer.
#ifndef BX_NLW2
#define BX_NLW2 2
#endif
  static constexpr int NLW = K == 2 ? BX_NLW2 : 5;
  static constexpr int NPW = 32 >> NLW;  // nodes per warp after the in-warp levels
  static constexpr int NIW = 32 - NPW;   // merge nodes per warp (in-warp levels)
  static constexpr int NU = NW * NPW;
  static constexpr int kWPort = NU * (int)(sizeof(TwoPort<K>) / 8);
  static constexpr int kWLR = NU * 2 * K;
  static constexpr int kRoots = 8 * (int)(sizeof(TwoPort<K>) / 8);
  static constexpr int kMisc = 8;
  static constexpr size_t bytes =
      sizeof(double) * (size_t)(kState + kInfo + kWPort + kWLR + kRoots + kMisc);
};

template <int K, int M, int T, bool VEC, bool SP, class Lay>
__global__ void __launch_bounds__(T)
part_kernel(const double *__restrict__ c2p, const double *__restrict__ c1p,
            const double *__restrict__ ep, const double *__restrict__ f1p,
            const double *__restrict__ f2p, const double *__restrict__ bp,
            double *__restrict__ xp, int32_t *status, int32_t *index, int64_t *nz_out,
            int64_t batch, int64_t n, Lay lay, int csize, Outer outer,
            const int32_t *__restrict__ only, int fs, int mark) {
  // only != nullptr: retry pass after the interface-iteration kernel
  // (bx_direct_halo.cu) -- a small persistent grid whose clusters walk the
  // batch and solve just the systems it marked (only[s * fs + r] != 0 for some
  // r < fs), OR-ing flags into status[s * fs]; fs = 1 otherwise.  mark != 0
  // (no workspace: the sparse-outer entry): `only` is the status array itself,
  // a system is marked by status[s] == mark and leaves with its final status /
  // index, exactly what this kernel writes without a first pass.
  // let the re-solve kernel behind this one become resident early; the retry
  // pass itself is such a dependent of the interface-iteration kernel
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (only) asm volatile("griddepcontrol.wait;" ::: "memory");
  using SM = Smem<K, M, T>;
  constexpr int NW = SM::NW;
  static_assert(T % 32 == 0 && (NW & (NW - 1)) == 0, "T must be 32 * power of two");
  extern __shared__ __align__(16) double smem[];
  double *state = smem;
  double *info = smem + SM::kState;
  TwoPort<K> *wport = reinterpret_cast<TwoPort<K> *>(smem + SM::kState + SM::kInfo);
  double *wlr = smem + SM::kState + SM::kInfo + SM::kWPort;
  TwoPort<K> *croots = reinterpret_cast<TwoPort<K> *>(wlr + SM::kWLR);
  int *misc = reinterpret_cast<int *>(wlr + SM::kWLR + SM::kRoots);

  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int crank = csize > 1 ? (int)cg::this_cluster().block_rank() : 0;
  const int64_t seg0 = (int64_t)crank * (T * M);
  const int64_t base = seg0 + (int64_t)t * M;
  using CH = Chunk<K, M, T, VEC, SP, Lay>;
  // misc: [0] nz counter (int), [1] cluster mbarrier (8-byte slot)
  uint64_t *cbar = reinterpret_cast<uint64_t *>(misc + 2);
  if (t == 0) {
    misc[0] = 0;
    if (csize > 1) {
      // receives the (csize - 1) peer roots pushed with st.async
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(cbar)) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
  }
  if (csize > 1) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");

  unsigned ph = 0;  // parity of the root mbarrier's current phase
  const int64_t nclus = gridDim.x / csize;
  for (int64_t s0 = blockIdx.x / csize; s0 < batch; s0 += only ? 32 * nclus : batch) {
  // retry pass: 32 of this cluster's systems are tested per round trip (every
  // warp of the cluster reads the same words: the walk is cluster-uniform)
  unsigned todo = 1u;
  if (only) {
    const int64_t sl = s0 + (int64_t)lane * nclus;
    bool marked = false;
    if (sl < batch)
      for (int r = 0; r < fs; ++r) marked |= mark ? only[sl * fs + r] == mark : only[sl * fs + r] != 0;
    todo = __ballot_sync(0xffffffffu, marked);
  }
  while (todo) {
  const int64_t s = s0 + (int64_t)(__ffs(todo) - 1) * nclus;
  todo &= todo - 1;
  BX_TR(0);
  // ---------------- phase 1: downward elimination (bx_part_phases.cuh) ------
  int32_t bad;
  int nzc;
  CH::down(state, t, s, base, n, lay, c2p, c1p, ep, f1p, f2p, bp, outer, bad, nzc);

  BX_TR(1);
  CH::up(state, t);

  BX_TR(2);
  // chunk two-port from the thread's own rows 0..K-1 (F) and M-K..M-1 (E)
  TwoPort<K> port = CH::port(state, t);

  // ---------------- tree ascent ---------------------------------------------
  // Levels 0..NLW-1 inside every warp (shuffles), then warp 0 alone reduces
  // the NU remaining nodes (shuffles again): for K=2 the upper levels then
  // cost one warp's issue slots instead of every warp's, and the other warps
  // leave the FP64 pipes to the co-resident CTA.  Merge-info nodes: in-warp
  // level l of warp w at info[w*NIW + (32 - (32 >> l)) + k], upper levels
  // after NW*NIW.
  constexpr int NU = SM::NU, NLW = SM::NLW, NPW = SM::NPW, NIW = SM::NIW;
  bool ok = true;
#pragma unroll 1
  for (int l = 0; l < NLW; ++l) {
    const int step = 1 << l;
    const TwoPort<K> other = shfl_down_port<K>(port, step);
    // divergence-free: every lane merges (inactive lanes discard), so the
    // warp stays converged for the next level's shuffles; inactive lanes park
    // their merge info in the spare node T-1
    const bool act = (lane & (2 * step - 1)) == 0;
    MergeInfo<K> mi;
    TwoPort<K> m;
    const bool okm = merge<K>(port, other, m, mi);
    ok &= okm || !act;
    store_info<K, T>(info, act ? warp * NIW + (32 - (32 >> l)) + (lane >> (l + 1)) : T - 1, mi);
    if (act) port = m;
  }
  BX_TR(3);
  if ((lane & ((1 << NLW) - 1)) == 0) wport[warp * NPW + (lane >> NLW)] = port;
  __syncthreads();
  if (NW >= 2 && warp < 2) {
    // upper levels on warps 0 and 1 together: warp 0 computes the u half of
    // every merge (S, u, merged E), warp 1 the mirrored v half (T, v, merged
    // F), on two SMSPs; nodes are merged in place in wport (level l reads
    // nodes 2k, 2k+1 and writes node k), two 64-thread named barriers a level
    const bool isU = warp == 0;
    int off = NW * NIW;
#pragma unroll 1
    for (int l = 0; (1 << l) < NU; ++l) {
      const int nm = NU >> (l + 1);
      const int k = lane < nm ? lane : 0;  // idle lanes redo merge 0 and discard
      Port<K> half, out;
      bool okm;
      if (isU) okm = merge_u<K>(wport[2 * k].E, wport[2 * k + 1].F, wport[2 * k + 1].E, half, out);
      else okm = merge_v<K>(wport[2 * k].E, wport[2 * k + 1].F, wport[2 * k].F, half, out);
      ok &= okm || lane >= nm;
      asm volatile("bar.sync 1, 64;" ::: "memory");  // level l read by both warps
      if (lane < nm) {
        store_port<K, T>(info, isU ? 0 : (int)(sizeof(Port<K>) / 8), off + lane, half);
        if (isU) wport[lane].E = out;
        else wport[lane].F = out;
      }
      asm volatile("bar.sync 1, 64;" ::: "memory");  // level l+1 complete
      off += nm;
    }
  } else if (NW == 1) {
    TwoPort<K> wp = wport[lane & (NU - 1)];
    int off = NW * NIW;
#pragma unroll 1
    for (int l = 0; (1 << l) < NU; ++l) {
      const int step = 1 << l;
      const TwoPort<K> other = shfl_down_port<K>(wp, step);
      const bool act = lane < NU && (lane & (2 * step - 1)) == 0;
      MergeInfo<K> mi;
      TwoPort<K> m;
      const bool okm = merge<K>(wp, other, m, mi);
      ok &= okm || !act;
      store_info<K, T>(info, act ? off + (lane >> (l + 1)) : T - 1, mi);
      if (act) wp = m;
      off += NU >> (l + 1);
    }
    if (lane == 0) wport[0] = wp;
  }

  BX_TR(4);
  // ---------------- cluster level -------------------------------------------
  Vec<K> Lseg, Rseg;
#pragma unroll
  for (int k = 0; k < K; ++k) Lseg.v[k] = Rseg.v[k] = 0.0;
  if (csize > 1 && warp == 0) {
    // every CTA pushes its segment root (wport[0], written by lane 0 above)
    // into slot [crank] of every peer with st.async, completing on the peer's
    // mbarrier: no cluster-wide barrier, no generic-proxy fence, and warps
    // 1..NW-1 never wait here.
    constexpr int NR = (int)(sizeof(TwoPort<K>) / 8);
    __syncwarp();
    asm volatile("barrier.cluster.wait.aligned;" ::: "memory");  // peers started (arrive at entry)
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(cbar)),
                   "r"((unsigned)((csize - 1) * NR * 8))
                   : "memory");
    if (lane < NR) {
      const double v = reinterpret_cast<const double *>(wport)[lane];
      double *slot = reinterpret_cast<double *>(&croots[crank]) + lane;
      *slot = v;
      const unsigned ls = smem_addr(slot), lb = smem_addr(cbar);
      for (int r = 0; r < csize; ++r) {
        if (r == crank) continue;
        unsigned ra, rb;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(ls), "r"(r));
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(lb), "r"(r));
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];"
                     ::"r"(ra), "d"(v), "r"(rb)
                     : "memory");
      }
    }
    // wait for the peers' roots (phase 0 of the mbarrier)
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "W_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra W_%=;\n}" ::"r"(smem_addr(cbar)), "r"(ph)
        : "memory");
    __syncwarp();
    if (lane == 0) {
      // segments left (P) and right (Q) of this one, merged in order; then
      // the three-segment system P | S | Q with L = R = 0 at the ends
      const TwoPort<K> S = croots[crank];
      TwoPort<K> P, Q, m;
      MergeInfo<K> mi;
      const bool hasP = crank > 0, hasQ = crank < csize - 1;
      if (hasP) {
        P = croots[0];
        for (int r = 1; r < crank; ++r) { ok &= merge<K>(P, croots[r], m, mi); P = m; }
      }
      if (hasQ) {
        Q = croots[crank + 1];
        for (int r = crank + 2; r < csize; ++r) { ok &= merge<K>(Q, croots[r], m, mi); Q = m; }
      }
      if (hasP && hasQ) {
        MergeInfo<K> m1, m2;
        TwoPort<K> PS, PSQ;
        ok &= merge<K>(P, S, PS, m1);
        ok &= merge<K>(PS, Q, PSQ, m2);
        Rseg = m2.v.g;                      // F of Q with root L = R = 0
        Lseg = vadd<K>(m1.u.g, mv<K>(m1.u.B, Rseg));  // E of P given R(PS) = F of Q
      } else if (hasQ) {
        ok &= merge<K>(S, Q, m, mi);
        Rseg = mi.v.g;
      } else {
        ok &= merge<K>(P, S, m, mi);
        Lseg = mi.u.g;
      }
    }
  }

#ifdef BX_TRACE
  {  // make the clock wait for the cluster-level results
    double d0, d1;
    asm volatile("mov.b64 %0, %1;" : "=d"(d0) : "d"(Lseg.v[0]));
    asm volatile("mov.b64 %0, %1;" : "=d"(d1) : "d"(Rseg.v[0]));
    if (d0 == 1.2345e300 && d1 == 1.2345e300) misc[1] = 1;
  }
  BX_TR(12);
  __syncwarp();
#endif
  BX_TR(5);
  // ---------------- tree descent -------------------------------------------
  if (warp == 0) {
    // root of the CTA (lane 0), then the upper levels (lanes 0..NU-1)
    Vec<K> L = Lseg, R = Rseg;
    constexpr int nlev = NU >= 32 ? 5 : NU >= 16 ? 4 : NU >= 8 ? 3 : NU >= 4 ? 2 : NU >= 2 ? 1 : 0;
    int offs[nlev > 0 ? nlev : 1];
    {
      int off = NW * NIW;
#pragma unroll
      for (int l = 0; l < nlev; ++l) { offs[l] = off; off += NU >> (l + 1); }
    }
#pragma unroll
    for (int l = nlev - 1; l >= 0; --l) {
      const int step = 1 << l;
      const bool act = lane < NU && (lane & (2 * step - 1)) == 0;
      // divergence-free: every lane loads and applies, inactive lanes discard
      const MergeInfo<K> mi = load_info<K, T>(info, offs[l] + ((lane & (NU - 1)) >> (l + 1)));
      Vec<K> uu = apply<K>(mi.u, L, R), vv = apply<K>(mi.v, L, R);
      if (!act) { uu = L; vv = R; }
      const Vec<K> pu = shfl_up_vec<K>(uu, step), pR = shfl_up_vec<K>(R, step);
      if (lane < NU && (lane & (2 * step - 1)) == step) { L = pu; R = pR; }
      if (act) R = vv;
    }
    if (lane < NU) {
#pragma unroll
      for (int k = 0; k < K; ++k) { wlr[lane * 2 * K + k] = L.v[k]; wlr[lane * 2 * K + K + k] = R.v[k]; }
    }
  }
  BX_TR(10);
  __syncthreads();
  BX_TR(11);
  Vec<K> L, R;
  {
    const int nd = warp * NPW + (lane >> NLW);  // this lane's node (used by lanes 2^NLW i)
#pragma unroll
    for (int k = 0; k < K; ++k) { L.v[k] = wlr[nd * 2 * K + k]; R.v[k] = wlr[nd * 2 * K + K + k]; }
  }
#pragma unroll 1
  for (int l = NLW - 1; l >= 0; --l) {
    const int step = 1 << l;
    const bool act = (lane & (2 * step - 1)) == 0;
    const MergeInfo<K> mi = load_info<K, T>(info, warp * NIW + (32 - (32 >> l)) + (lane >> (l + 1)));
    Vec<K> uu = apply<K>(mi.u, L, R), vv = apply<K>(mi.v, L, R);
    if (!act) { uu = L; vv = R; }
    const Vec<K> pu = shfl_up_vec<K>(uu, step), pR = shfl_up_vec<K>(R, step);
    if ((lane & (2 * step - 1)) == step) { L = pu; R = pR; }
    if (act) R = vv;
  }

  BX_TR(6);
  // ---------------- phase 3: x_j = d - W.L - V.R -----------------------------
  CH::write_x(state, t, s, base, n, lay, xp, L, R);

  BX_TR(7);
  // ---------------- status / counters ---------------------------------------
  // csize == 1: this CTA owns the system and writes status/index itself (no
  // memsets in the launch).  csize > 1: status/index were preset to OK/-1 by
  // the launcher; failing CTAs report the smallest failing row (atomicMin on
  // the unsigned view of index).
  if (!ok && bad < 0) bad = (int32_t)seg0;
  if (csize == 1) {
    if (t == 0) misc[1] = 0x7fffffff;
    const bool any_bad = __syncthreads_or(bad >= 0);
    if (any_bad) {
      if (bad >= 0) atomicMin(&misc[1], bad);
      __syncthreads();
    }
    if (t == 0 && (any_bad || !only || mark)) {
      if (status) status[s * fs] = any_bad ? BX_STATUS_ZERO_PIVOT : BX_STATUS_OK;
      if (index) index[s] = any_bad ? misc[1] : -1;
    }
  } else if (__syncthreads_or(bad >= 0)) {
    // (mark: the word still holds the mark, which the peers may yet have to
    // read -- add a bit now, rank 0 settles the word after the cluster barrier)
    if (mark) { if (bad >= 0) atomicOr(status + s, 0x80); }
    else if (status) status[s * fs] = BX_STATUS_ZERO_PIVOT;
    if (index && bad >= 0) atomicMin(reinterpret_cast<unsigned int *>(index + s), (unsigned int)bad);
  }
#ifdef BX_TRACE
  if (threadIdx.x == 0 && blockIdx.x - BX_TRACE_BASE < 4096u) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_bx_trace[blockIdx.x - BX_TRACE_BASE][8] = clock64();
    g_bx_trace[blockIdx.x - BX_TRACE_BASE][9] = smid;
  }
#endif
  if (K == 2 && nz_out) {
    nzc = __reduce_add_sync(0xffffffffu, nzc);
    if (lane == 0) atomicAdd(&misc[0], nzc);
    __syncthreads();
    if (t == 0) {
      if (csize == 1) nz_out[s] = misc[0];
      else atomicAdd(reinterpret_cast<unsigned long long *>(nz_out + s), (unsigned long long)misc[0]);
    }
  }
  if (only) {
    // next marked system: this one's shared memory (and, in a cluster, the
    // root slots the peers push into) must be done with everywhere first
    __syncthreads();
    if (csize > 1) {
      if (warp != 0) asm volatile("barrier.cluster.wait.aligned;" ::: "memory");  // pairs the arrive above
      asm volatile("barrier.cluster.arrive.aligned;" ::: "memory");
      asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
      if (mark && crank == 0 && t == 0) status[s] = (status[s] & 0x80) ? BX_STATUS_ZERO_PIVOT : BX_STATUS_OK;
      asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");  // "started" for the next one
      ph ^= 1u;
    }
  }
  }  // marked systems of this round
  }  // systems of this cluster
}

// ----------------------------------------------------------------------------
// launch configuration
// ----------------------------------------------------------------------------
static const Outer kNoOuter{nullptr, nullptr, nullptr, 0};


template <int K, int M, int T, bool VEC, class Lay, bool SP = false>
static int launch(const double *c2, const double *c1, const double *e, const double *f1,
                  const double *f2, const double *b, double *x, int32_t *st, int32_t *ix,
                  int64_t *nz, int64_t batch, int64_t n, Lay lay, cudaStream_t stream,
                  Outer outer = kNoOuter, const int32_t *only = nullptr, int fs = 1) {
  constexpr int rows = M * T;
  const int csize = (int)((n + rows - 1) / rows);
  if (csize > 8) {
    bxh::set_error("partitioned solver: n=%lld exceeds %d rows (8-CTA cluster)", (long long)n,
                   8 * rows);
    return BX_ERR_UNSUPPORTED;
  }
  size_t smem = Smem<K, M, T>::bytes;
#ifdef BX_TRACE
  if (getenv("BX_TRACE_SMEM")) smem = (size_t)atoi(getenv("BX_TRACE_SMEM"));  // occupancy experiments
#endif
  auto kern = part_kernel<K, M, T, VEC, SP, Lay>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (csize > 1 && !only) {  // single-CTA systems write status/index/nz in the kernel
    if (nz) cudaMemsetAsync(nz, 0, sizeof(int64_t) * (size_t)batch, stream);
    if (st) cudaMemsetAsync(st, 0, sizeof(int32_t) * (size_t)batch, stream);     // BX_STATUS_OK
    if (ix) cudaMemsetAsync(ix, 0xff, sizeof(int32_t) * (size_t)batch, stream);  // -1
  }
  cudaLaunchConfig_t cfg = {};
  // retry pass: a few clusters per SM walk the batch (launching batch * csize
  // CTAs that mostly exit at once cost 42 us on config 2)
  const int64_t nclus = only ? (batch < 2 * 148 ? batch : 2 * 148) : batch;
  cfg.gridDim = dim3((unsigned)(nclus * csize));
  cfg.blockDim = dim3(T);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = csize;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // retry pass only
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = only ? 2 : 1;
  // fs < 0: no-workspace retry (marks in the status array, see part_kernel)
  cudaError_t err = cudaLaunchKernelEx(&cfg, kern, c2, c1, e, f1, f2, b, x, st, ix, nz, batch, n,
                                       lay, csize, outer, only, fs < 0 ? 1 : fs, fs < 0 ? kRetryMark : 0);
  if (err != cudaSuccess) {
    bxh::set_error("partitioned solver launch: %s", cudaGetErrorString(err));
    return BX_ERR_CUDA;
  }
  return BX_OK;
}

// Above 1024 rows: 1024-row CTAs (T=64) or 2048-row CTAs (T=128)?  Measured
// on B200 (K=1,2; n = 1100..8192): the 1024-row shape wins whenever it pads
// fewer rows (n mod 2048 in (0, 1024]: 2500 rows 0.477 vs 0.608 ms) and, at
// equal padding, when its last CTA is at least half full (n=4096: 0.581 vs
// 0.592 ms; n=1500: 0.577 vs 0.553 ms the other way).  8-CTA cluster limit.
static bool use_1k_ctas(int64_t n) {
  if (n <= 1024) return true;
  if (n > 8192) return false;
  const int64_t r = (n - 1) % 2048 + 1;  // rows in the last 2048-row CTA
  return r <= 1024 || r - 1024 >= 512;
}

template <int K, bool VEC, class Lay>
static int dispatch2(const double *c2, const double *c1, const double *e, const double *f1,
                     const double *f2, const double *b, double *x, int32_t *st, int32_t *ix,
                     int64_t *nz, int64_t batch, int64_t n, Lay lay, cudaStream_t stream,
                     const int32_t *only, int fs) {
  // rows per CTA = M*T; small systems use small CTAs (many CTAs per SM).
  // BX_PART_CFG (developer knob, benchmarking only) forces one configuration.
  static int forced = -2;
  if (forced == -2) {
    const char *env = getenv("BX_PART_CFG");
    forced = env ? atoi(env) : -1;
  }
  switch (forced) {
    case 0: return launch<K, 8, 32, VEC, Lay>(c2, c1, e, f1, f2, b, x, st, ix, nz, batch, n, lay, stream, kNoOuter, only, fs);
    case 1: return launch<K, 8, 64, VEC, Lay>(c2, c1, e, f1, f2, b, x, st, ix, nz, batch, n, lay, stream, kNoOuter, only, fs);
    case 2: return launch<K, 8, 128, VEC, Lay>(c2, c1, e, f1, f2, b, x, st, ix, nz, batch, n, lay, stream, kNoOuter, only, fs);
    case 3: return launch<K, 16, 64, VEC, Lay>(c2, c1, e, f1, f2, b, x, st, ix, nz, batch, n, lay, stream, kNoOuter, only, fs);
    case 4: return launch<K, 16, 32, VEC, Lay>(c2, c1, e, f1, f2, b, x, st, ix, nz, batch, n, lay, stream, kNoOuter, only, fs);
    case 5: return launch<K, 32, 32, VEC, Lay>(c2, c1, e, f1, f2, b, x, st, ix, nz, batch, n, lay, stream, kNoOuter, only, fs);
    case 6: return launch<K, 16, 128, VEC, Lay>(c2, c1, e, f1, f2, b, x, st, ix, nz, batch, n, lay, stream, kNoOuter, only, fs);
    default: break;
  }
  if (n <= 256) return launch<K, 8, 32, VEC, Lay>(c2, c1, e, f1, f2, b, x, st, ix, nz, batch, n, lay, stream, kNoOuter, only, fs);
  if (n <= 512) return launch<K, 8, 64, VEC, Lay>(c2, c1, e, f1, f2, b, x, st, ix, nz, batch, n, lay, stream, kNoOuter, only, fs);
  if (use_1k_ctas(n)) return launch<K, 16, 64, VEC, Lay>(c2, c1, e, f1, f2, b, x, st, ix, nz, batch, n, lay, stream, kNoOuter, only, fs);
  return launch<K, 16, 128, VEC, Lay>(c2, c1, e, f1, f2, b, x, st, ix, nz, batch, n, lay, stream, kNoOuter, only, fs);
}

// sparse +-2 diagonals (MNPDM): default shapes only, K = 2
template <bool VEC, class Lay>
static int dispatch_sparse(const double *c1, const double *e, const double *f1, const double *b,
                           double *x, int32_t *st, int32_t *ix, int64_t *nz, int64_t batch,
                           int64_t n, Lay lay, cudaStream_t stream, Outer o,
                           const int32_t *only = nullptr, int fs = 1) {
  if (n <= 256)
    return launch<2, 8, 32, VEC, Lay, true>(nullptr, c1, e, f1, nullptr, b, x, st, ix, nz, batch, n, lay, stream, o, only, fs);
  if (n <= 512)
    return launch<2, 8, 64, VEC, Lay, true>(nullptr, c1, e, f1, nullptr, b, x, st, ix, nz, batch, n, lay, stream, o, only, fs);
  if (n <= 1024)  // the 1024-row shape measured slower here (n=4096: 0.668 vs 0.632 ms)
    return launch<2, 16, 64, VEC, Lay, true>(nullptr, c1, e, f1, nullptr, b, x, st, ix, nz, batch, n, lay, stream, o, only, fs);
  return launch<2, 16, 128, VEC, Lay, true>(nullptr, c1, e, f1, nullptr, b, x, st, ix, nz, batch, n, lay, stream, o, only, fs);
}

// one CTA per system: rows whose sub2 (i >= 2) or sup2 (i <= n-3) is nonzero,
// in row order (block-wide exclusive scan of per-thread counts); count[s]
// always, the entries only when capacity > 0 (row -1 pads the slots)
template <class Lay>
__global__ void __launch_bounds__(256)
outer_compact_kernel(const double *__restrict__ c2p, const double *__restrict__ f2p,
                     int32_t *count, int32_t *rows, double *vs2, double *vp2, int64_t cap,
                     int64_t n, Lay lay) {
  const int64_t s = blockIdx.x;
  const int t = threadIdx.x;
  const int64_t per = (n + 255) / 256, r0 = t * per, r1 = min(n, r0 + per);
  auto nzrow = [&](int64_t i) {
    const double a = i >= 2 ? ldg(c2p + lay(i, s)) : 0.0;
    const double c = i <= n - 3 ? ldg(f2p + lay(i, s)) : 0.0;
    return a != 0.0 || c != 0.0;
  };
  int cnt = 0;
  for (int64_t i = r0; i < r1; ++i) cnt += nzrow(i);
  __shared__ int wsum[8];
  int incl = cnt;
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if ((t & 31) >= o) incl += v;
  }
  if ((t & 31) == 31) wsum[t >> 5] = incl;
  __syncthreads();
  int off = incl - cnt;
  for (int w = 0; w < (t >> 5); ++w) off += wsum[w];
  if (t == 255) count[s] = off + cnt;
  if (cap <= 0) return;
  for (int64_t i = r0; i < r1 && off < cap; ++i) {
    if (!nzrow(i)) continue;
    rows[s * cap + off] = (int32_t)i;
    vs2[s * cap + off] = i >= 2 ? ldg(c2p + lay(i, s)) : 0.0;
    vp2[s * cap + off] = i <= n - 3 ? ldg(f2p + lay(i, s)) : 0.0;
    ++off;
  }
  __syncthreads();
  const int total = (int)min((int64_t)count[s], cap);
  for (int64_t j = total + t; j < cap; j += 256) {
    rows[s * cap + j] = -1;
    vs2[s * cap + j] = 0.0;
    vp2[s * cap + j] = 0.0;
  }
}

static bool aligned32(const void *p) { return p == nullptr || ((uintptr_t)p & 31u) == 0; }

template <int K, class Lay>
static int dispatch(const double *c2, const double *c1, const double *e, const double *f1,
                    const double *f2, const double *b, double *x, int32_t *st, int32_t *ix,
                    int64_t *nz, int64_t batch, int64_t n, Lay lay, cudaStream_t stream,
                    bool vec_ok, const int32_t *only = nullptr, int fs = 1) {
  vec_ok = vec_ok && aligned32(c2) && aligned32(c1) && aligned32(e) && aligned32(f1) &&
           aligned32(f2) && aligned32(b) && aligned32(x);
  if (vec_ok) return dispatch2<K, true>(c2, c1, e, f1, f2, b, x, st, ix, nz, batch, n, lay, stream, only, fs);
  return dispatch2<K, false>(c2, c1, e, f1, f2, b, x, st, ix, nz, batch, n, lay, stream, only, fs);
}

}  // namespace part

// Workspace of the partitioned path: per-system flags (zero / non-finite
// pivots of the partitioned elimination) and the re-solve scratch of
// direct_fixup (bx_direct_seq.cu).
// BX_PART_SEG=1 (developer knob, experiment): use the segment-resident kernel
// (bx_direct_seg.cu; measured slower than part_kernel)
static bool seg_enabled() {
  static int v = -1;
  if (v < 0) {
    const char *env = getenv("BX_PART_SEG");
    v = env ? atoi(env) : 0;
  }
  return v != 0;
}

static size_t flag_bytes(int64_t batch) { return ((size_t)batch * 8 * 4 + 255) / 256 * 256; }
size_t part_workspace_bytes(int bandwidth, int64_t batch, int64_t n) {
  return 3 * flag_bytes(batch) + 8 * fixup_scratch_doubles(bandwidth == 1 ? 0 : 1, n);
}

// workspace: flags [batch][8] | nz parts [batch][8] | retry marks [batch][8] |
// re-solve scratch
static void carve(double *ws, int64_t batch, int32_t *&flags, int32_t *&nzpart, int32_t *&retry,
                  double *&scratch) {
  char *p = reinterpret_cast<char *>(ws);
  flags = reinterpret_cast<int32_t *>(p);
  nzpart = reinterpret_cast<int32_t *>(p + flag_bytes(batch));
  retry = reinterpret_cast<int32_t *>(p + 2 * flag_bytes(batch));
  scratch = reinterpret_cast<double *>(p + 3 * flag_bytes(batch));
}

int ntdm_part(const double *d, const double *e, const double *f, const double *b, double *x,
              double *ws, int32_t *st, int32_t *ix, int64_t batch, int64_t n, int64_t ld, int layout,
              cudaStream_t stream) {
  int32_t *flags, *nzpart, *retry;
  double *scratch;
  carve(ws, batch, flags, nzpart, retry, scratch);
  const double *ptrs[] = {d, e, f, b, x};
  int rc = BX_ERR_UNSUPPORTED, fs = 1;
  if (seg_enabled() && seg_applicable(ptrs, 5, n, ld, layout))
    rc = seg_solve(1, nullptr, d, e, f, nullptr, b, x, flags, nullptr, batch, n, ld, stream, &fs);
  if (rc == BX_ERR_UNSUPPORTED) {
    fs = 1;
    // first pass: interface iteration; the tree then solves only what it marked
    const int32_t *only = nullptr;
    if (halo_enabled()) {
      rc = halo_solve(1, nullptr, d, e, f, nullptr, b, x, flags, retry, nullptr, batch, n, ld,
                      layout, stream, nullptr, nullptr, nullptr, 0, &fs);
      if (rc == BX_OK) only = retry;
      else if (rc != BX_ERR_UNSUPPORTED) return rc;
      else fs = 1;
    }
    if (layout == BX_LAYOUT_SYSTEM_MAJOR)
      rc = part::dispatch<1>(nullptr, d, e, f, nullptr, b, x, flags, nullptr, nullptr, batch, n,
                             SystemMajor{ld}, stream, ld % 4 == 0, only, fs);
    else
      rc = part::dispatch<1>(nullptr, d, e, f, nullptr, b, x, flags, nullptr, nullptr, batch, n,
                             Interleaved{ld}, stream, false, only, fs);
  }
  if (rc != BX_OK) return rc;
  direct_fixup(0, nullptr, d, e, f, nullptr, b, x, scratch, flags, fs, nullptr, st, ix, nullptr,
               batch, n, ld, layout, stream);
  return bxh::check_launch("partitioned solver re-solve");
}

int penta_part(bool mod, const double *c, const double *d, const double *e, const double *f,
               const double *g, const double *b, double *x, double *ws, int32_t *st, int32_t *ix,
               int64_t *nz, int64_t batch, int64_t n, int64_t ld, int layout, cudaStream_t stream) {
  int32_t *flags, *nzpart, *retry;
  double *scratch;
  carve(ws, batch, flags, nzpart, retry, scratch);
  const double *ptrs[] = {c, d, e, f, g, b, x};
  int rc = BX_ERR_UNSUPPORTED, fs = 1;
  bool seg = false, halo = false;
  if (seg_enabled() && seg_applicable(ptrs, 7, n, ld, layout)) {
    rc = seg_solve(2, c, d, e, f, g, b, x, flags, nz ? nzpart : nullptr, batch, n, ld, stream, &fs);
    seg = rc != BX_ERR_UNSUPPORTED;
  }
  if (!seg) {
    fs = 1;
    // first pass: interface iteration (it also counts nz, per CTA); the tree
    // then solves only the systems it marked
    const int32_t *only = nullptr;
    if (halo_enabled()) {
      rc = halo_solve(2, c, d, e, f, g, b, x, flags, retry, nz ? nzpart : nullptr, batch, n, ld,
                      layout, stream, nullptr, nullptr, nullptr, 0, &fs);
      if (rc == BX_OK) only = retry;
      else if (rc != BX_ERR_UNSUPPORTED) return rc;
      else fs = 1;
    }
    halo = only != nullptr;
    int64_t *tnz = only ? nullptr : nz;
    if (layout == BX_LAYOUT_SYSTEM_MAJOR)
      rc = part::dispatch<2>(c, d, e, f, g, b, x, flags, nullptr, tnz, batch, n, SystemMajor{ld},
                             stream, ld % 4 == 0, only, fs);
    else
      rc = part::dispatch<2>(c, d, e, f, g, b, x, flags, nullptr, tnz, batch, n, Interleaved{ld},
                             stream, false, only, fs);
  }
  if (rc != BX_OK) return rc;
  direct_fixup(mod ? 2 : 1, c, d, e, f, g, b, x, scratch, flags, fs, (seg || halo) && nz ? nzpart : nullptr,
               st, ix, nz, batch, n, ld, layout, stream);
  return bxh::check_launch("partitioned solver re-solve");
}

int outer_compact(const double *sub2, const double *sup2, int32_t *count, int32_t *rows,
                  double *vsub2, double *vsup2, int64_t cap, int64_t batch, int64_t n, int64_t ld,
                  int layout, cudaStream_t stream) {
  if (layout == BX_LAYOUT_SYSTEM_MAJOR)
    part::outer_compact_kernel<<<(unsigned)batch, 256, 0, stream>>>(sub2, sup2, count, rows, vsub2,
                                                                   vsup2, cap, n, SystemMajor{ld});
  else
    part::outer_compact_kernel<<<(unsigned)batch, 256, 0, stream>>>(sub2, sup2, count, rows, vsub2,
                                                                   vsup2, cap, n, Interleaved{ld});
  return BX_OK;
}

int mnpdm_sparse_part(const int32_t *rows, const double *vsub2, const double *vsup2, int64_t k,
                      const double *d, const double *e, const double *f, const double *b,
                      double *x, int32_t *st, int32_t *ix, int64_t *nz, int64_t batch, int64_t n,
                      int64_t ld, int layout, cudaStream_t stream) {
  const part::Outer o{rows, vsub2, vsup2, k};
  // first pass: interface iteration with the status array carrying the retry
  // marks (this entry has no workspace); the tree pass then solves the marked
  // systems and writes their final status / index
  const int32_t *only = nullptr;
  int fs = 1;
  if (halo_enabled() && st) {
    int cs = 1;
    const int rc = halo_solve(2, nullptr, d, e, f, nullptr, b, x, st, nullptr, nullptr, batch, n, ld,
                              layout, stream, rows, vsub2, vsup2, k, &cs, ix, nz);
    if (rc == BX_OK) {
      only = st;
      fs = -1;  // marks in the status array
      nz = nullptr;
    } else if (rc != BX_ERR_UNSUPPORTED) {
      return rc;
    }
  }
  if (layout == BX_LAYOUT_SYSTEM_MAJOR) {
    const bool vec = ld % 4 == 0 && part::aligned32(d) && part::aligned32(e) && part::aligned32(f) &&
                     part::aligned32(b) && part::aligned32(x);
    if (vec)
      return part::dispatch_sparse<true>(d, e, f, b, x, st, ix, nz, batch, n, SystemMajor{ld}, stream, o, only, fs);
    return part::dispatch_sparse<false>(d, e, f, b, x, st, ix, nz, batch, n, SystemMajor{ld}, stream, o, only, fs);
  }
  return part::dispatch_sparse<false>(d, e, f, b, x, st, ix, nz, batch, n, Interleaved{ld}, stream, o, only, fs);
}

size_t other_workspace_bytes(int solver, int64_t batch, int64_t n) {
  if (solver == BX_SOLVER_SIP) return sip_workspace_bytes(batch, n);
  if (solver == BX_SOLVER_STDM) return exact_workspace_bytes(1, batch, n);
  if (solver == BX_SOLVER_SPDM) return exact_workspace_bytes(2, batch, n);
  return 0;
}

}  // namespace bx
