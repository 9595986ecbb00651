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

#ifndef BX_PART_LA
#define BX_PART_LA 1  // input groups in flight ahead of the elimination (measured: 1 > 2 > 3)
#endif

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

// +-2 diagonals held sparse (MNPDM's case): per system a row-sorted list of
// the rows where sub2 or sup2 is nonzero, k slots per system (row -1 pads)
struct Outer {
  const int32_t *rows;
  const double *sub2, *sup2;
  int64_t k;
};

template <int K, int M, int T, bool VEC, bool SP, class Lay>
__global__ void __launch_bounds__(T)
part_kernel(const double *__restrict__ c2p, const double *__restrict__ c1p,
            const double *__restrict__ ep, const double *__restrict__ f1p,
            const double *__restrict__ f2p, const double *__restrict__ bp,
            double *__restrict__ xp, int32_t *status, int32_t *index, int64_t *nz_out,
            int64_t batch, int64_t n, Lay lay, int csize, Outer outer) {
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
  const int64_t s = blockIdx.x / csize;
  const int64_t seg0 = (int64_t)crank * (T * M);
  const int64_t base = seg0 + (int64_t)t * M;
  auto st = [&](int q, int j) -> double & { return state[(q * M + j) * T + t]; };
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

  BX_TR(0);
  // ---------------- phase 1: downward elimination --------------------------
  // Gaussian elimination of the chunk against its own normalised rows:
  // x_{j-2} is eliminated with row j-2, then x_{j-1} with row j-1, and the
  // row is scaled by 1/mu (MUFU seed + Newton, rcp).  Stored (normalised):
  //   x_j + p x_{j+1} + q x_{j+2} + W.L = y
  // (measured: 20 FP64 ops/row beat the division-free variant's 37, whose
  // shorter dependent chain does not pay for its extra issue slots)
  int32_t bad = -1;
  int nzc = 0;
  // carried rows j-1 (f1, g1, y1, W1) and j-2: p, q, y, W of the stored rows
  double f1 = 0, g1 = 0, y1 = 0, f2 = 0, g2 = 0, y2 = 0;
  double W1[K], W2[K];
#pragma unroll
  for (int k = 0; k < K; ++k) W1[k] = W2[k] = 0.0;
  if (K == 2) { W2[0] = -1.0; W1[K - 1] = -1.0; }
  else W1[0] = -1.0;
  constexpr int G = 4;
  static_assert(M % G == 0, "M must be a multiple of 4");
  // register ring of input groups, LA groups in flight ahead of the one being
  // eliminated; the g loop is fully unrolled so the ring slots are fixed
  // registers (a copy between loop iterations would wait for the load)
  constexpr int LA = BX_PART_LA < M / G ? BX_PART_LA : M / G - 1 > 0 ? M / G - 1 : 1;
  constexpr int RG = LA + 1;
  struct Grp {
    double a2[G], a1[G], e[G], c1[G], c2[G], b[G];
  } ring[RG];
  auto load_group = [&](int g, Grp &gr) {
    double(&A2)[G] = gr.a2;
    double(&A1)[G] = gr.a1;
    double(&E)[G] = gr.e;
    double(&C1)[G] = gr.c1;
    double(&C2)[G] = gr.c2;
    double(&Bv)[G] = gr.b;
    const int64_t i0 = base + g * G;
    if (VEC && i0 + G <= n) {
      if (K == 2 && !SP) ld4(c2p + lay(i0, s), A2);
      ld4(c1p + lay(i0, s), A1);
      ld4(ep + lay(i0, s), E);
      ld4(f1p + lay(i0, s), C1);
      if (K == 2 && !SP) ld4(f2p + lay(i0, s), C2);
      ld4(bp + lay(i0, s), Bv);
      // (slots outside the matrix are masked where the group is consumed:
      // touching the registers here would wait for the load)
    } else {
#pragma unroll
      for (int u = 0; u < G; ++u) {
        const int64_t i = i0 + u;
        const bool in = i < n;
        A2[u] = (K == 2 && !SP && in && i >= 2) ? ldg(c2p + lay(i, s)) : 0.0;
        A1[u] = (in && i >= 1) ? ldg(c1p + lay(i, s)) : 0.0;
        E[u] = in ? ldg(ep + lay(i, s)) : 1.0;  // padding rows: identity
        C1[u] = (in && i <= n - 2) ? ldg(f1p + lay(i, s)) : 0.0;
        C2[u] = (K == 2 && !SP && in && i <= n - 3) ? ldg(f2p + lay(i, s)) : 0.0;
        Bv[u] = in ? ldg(bp + lay(i, s)) : 0.0;
      }
    }
  };
  // sparse outer diagonals: the slice [ob, oe) of this system's sorted list
  // that falls in this thread's rows (empty for almost every thread); the
  // first 8 list rows are fetched with independent loads (one round trip)
  int ob = 0, oe = 0;
  auto outer_slice = [&]() {
    const int32_t *orow = outer.rows + s * outer.k;
    const int k = (int)outer.k;
    int32_t r8[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) r8[q] = q < k ? __ldg(orow + q) : -1;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      ob += (r8[q] >= 0 && r8[q] < base) ? 1 : 0;
      oe += (r8[q] >= 0 && r8[q] < base + M) ? 1 : 0;
    }
    if (k > 8 && oe == 8) {  // long lists: continue the walk
      ob = min(ob, 8);
      while (ob < k && orow[ob] >= 0 && orow[ob] < base) ++ob;
      oe = ob;
      while (oe < k && orow[oe] >= 0 && orow[oe] < base + M) ++oe;
    }
  };
  // this thread's first 4 entries in registers (rows compared per row, no
  // memory access on the elimination chain); more than 4 fall back to loads
  int32_t er[4] = {-1, -1, -1, -1};
  double es2[4] = {0, 0, 0, 0}, ep2[4] = {0, 0, 0, 0};
  auto outer_regs = [&]() {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (ob + q < oe) {
        const int64_t o = s * outer.k + ob + q;
        er[q] = __ldg(outer.rows + o);
        es2[q] = __ldg(outer.sub2 + o);
        ep2[q] = __ldg(outer.sup2 + o);
      }
  };


  const bool first = base == 0;                             // rows 0, 1 of the system
  const int rend = (int)min(n - base, (int64_t)(M + 4));     // n - base, clamped
#pragma unroll
  for (int g = 0; g < LA && g < M / G; ++g) load_group(g, ring[g]);
  if (SP) {  // after the first input loads are in flight
    outer_slice();
    outer_regs();
  }
#pragma unroll
  for (int g = 0; g < M / G; ++g) {
    if (g + LA < M / G) load_group(g + LA, ring[(g + LA) % RG]);
    const Grp &cur = ring[g % RG];
#pragma unroll
    for (int u = 0; u < G; ++u) {
    const int j = g * G + u;
    const int64_t i = base + j;  // slots outside the matrix are never trusted:
    // chunk bases are multiples of M, so only rows j < 2 of the first chunk
    // can fall left of the matrix; the right edge is a 32-bit test on rend
    double a2 = (K != 2 || SP) ? 0.0 : cur.a2[u];
    double a1 = cur.a1[u];
    if (j < 2 && first) {
      a2 = 0.0;
      if (j < 1) a1 = 0.0;
    }
    const double e = cur.e[u];
    const double c1 = j > rend - 2 ? 0.0 : cur.c1[u];
    double c2 = (K != 2 || SP || j > rend - 3) ? 0.0 : cur.c2[u];
    if (SP) {  // branch-free for the register entries (the row loop stays one block)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const bool h = er[q] == (int32_t)i;
        a2 = h ? (i < 2 ? 0.0 : es2[q]) : a2;
        c2 = h ? (i > n - 3 ? 0.0 : ep2[q]) : c2;
      }
    }
    if (SP && oe - ob > 4) {
      for (int q = ob + 4; q < oe; ++q)
        if (outer.rows[s * outer.k + q] == (int32_t)i) {
          a2 = i < 2 ? 0.0 : outer.sub2[s * outer.k + q];
          c2 = i > n - 3 ? 0.0 : outer.sup2[s * outer.k + q];
        }
    }
    const double b = cur.b[u];
    // reciprocal form on normalised carried rows (p, q, y, w); rows -2, -1
    // are the virtual rows x_{-2} - L_0 = 0, x_{-1} - L_{K-1} = 0
    double mu, c1p, yy, ww[K];
    if (K == 2) {
      nzc += (a2 != 0.0);
      const double t1 = fma(-a2, f2, a1);
      const double e2 = fma(-a2, g2, e);
      const double y2p = fma(-a2, y2, b);
      mu = fma(-t1, f1, e2);
      c1p = fma(-t1, g1, c1);
      yy = fma(-t1, y1, y2p);
#pragma unroll
      for (int k = 0; k < K; ++k) ww[k] = fma(-t1, W1[k], -a2 * W2[k]);
    } else {
      mu = fma(-a1, f1, e);
      c1p = c1;
      yy = fma(-a1, y1, b);
      ww[0] = -a1 * W1[0];
    }
    if (mu == 0.0 || !isfinite(mu)) {
      if (bad < 0) bad = (int32_t)(base + j);
      mu = 1.0;
    }
    const double r = rcp(mu);
    const double pn = c1p * r, qn = c2 * r, yn = yy * r;
    st(0, j) = pn;
    if (K == 2) st(1, j) = qn;
    st(K, j) = yn;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const double w = ww[k] * r;
      st(K + 1 + k, j) = w;
      W2[k] = W1[k];
      W1[k] = w;
    }
    f2 = f1; g2 = g1; y2 = y1;
    f1 = pn; g1 = qn; y1 = yn;
    }
  }

  BX_TR(1);
  // ---------------- phase 1b: upward elimination ---------------------------
  // x_j = d_j - W_j.L - V_j.R ; state slots after: 0:d, 1..K: W, K+1..2K: V
  {
    double d1 = 0, d2 = 0, Wu1[K], Wu2[K], V1[K], V2[K];
#pragma unroll
    for (int k = 0; k < K; ++k) Wu1[k] = Wu2[k] = V1[k] = V2[k] = 0.0;
#pragma unroll
    for (int j = M - 1; j >= 0; --j) {
      const double p = st(0, j);
      const double q = K == 2 ? st(1, j) : 0.0;
      const double y = st(K, j);
      double W[K];
#pragma unroll
      for (int k = 0; k < K; ++k) W[k] = st(K + 1 + k, j);
      double d, Wu[K], V[K];
      if (j == M - 1) {
        d = y;
#pragma unroll
        for (int k = 0; k < K; ++k) Wu[k] = W[k];
        V[0] = p;
        if (K == 2) V[1] = q;
      } else if (K == 2 && j == M - 2) {
        d = fma(-p, d1, y);
#pragma unroll
        for (int k = 0; k < K; ++k) Wu[k] = fma(-p, Wu1[k], W[k]);
        V[0] = fma(-p, V1[0], q);
        V[1] = -p * V1[1];
      } else {
        // row j+2 terms first: the row j+1 results (newest) enter last
        d = K == 2 ? fma(-p, d1, fma(-q, d2, y)) : fma(-p, d1, y);
#pragma unroll
        for (int k = 0; k < K; ++k) {
          Wu[k] = K == 2 ? fma(-p, Wu1[k], fma(-q, Wu2[k], W[k])) : fma(-p, Wu1[k], W[k]);
          V[k] = K == 2 ? fma(-p, V1[k], -q * V2[k]) : -p * V1[k];
        }
      }
      st(0, j) = d;
#pragma unroll
      for (int k = 0; k < K; ++k) { st(1 + k, j) = Wu[k]; st(1 + K + k, j) = V[k]; }
      d2 = d1; d1 = d;
#pragma unroll
      for (int k = 0; k < K; ++k) { Wu2[k] = Wu1[k]; Wu1[k] = Wu[k]; V2[k] = V1[k]; V1[k] = V[k]; }
    }
  }

  BX_TR(2);
  // chunk two-port from the thread's own rows 0..K-1 (F) and M-K..M-1 (E)
  TwoPort<K> port;
#pragma unroll
  for (int a = 0; a < K; ++a) {
    const int jf = a, je = M - K + a;
    port.F.g.v[a] = st(0, jf);
    port.E.g.v[a] = st(0, je);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      port.F.A.m[a][k] = -st(1 + k, jf);
      port.F.B.m[a][k] = -st(1 + K + k, jf);
      port.E.A.m[a][k] = -st(1 + k, je);
      port.E.B.m[a][k] = -st(1 + K + k, je);
    }
  }

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
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
        "@!p bra W_%=;\n}" ::"r"(smem_addr(cbar))
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
#pragma unroll 1
  for (int g = 0; g < M / G; ++g) {
    double xv[G];
#pragma unroll
    for (int u = 0; u < G; ++u) {
      const int j = g * G + u;
      double v = st(0, j);
#pragma unroll
      for (int k = 0; k < K; ++k) v = fma(-st(1 + k, j), L.v[k], fma(-st(1 + K + k, j), R.v[k], v));
      xv[u] = v;
    }
    const int64_t i0 = base + g * G;
    if (VEC && i0 + G <= n) {
      st4(xp + lay(i0, s), xv);
    } else {
#pragma unroll
      for (int u = 0; u < G; ++u)
        if (i0 + u < n) xp[lay(i0 + u, s)] = xv[u];
    }
  }

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
    if (t == 0) {
      if (status) status[s] = any_bad ? BX_STATUS_ZERO_PIVOT : BX_STATUS_OK;
      if (index) index[s] = any_bad ? misc[1] : -1;
    }
  } else if (__syncthreads_or(bad >= 0)) {
    if (status) status[s] = BX_STATUS_ZERO_PIVOT;
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
}

// ----------------------------------------------------------------------------
// launch configuration
// ----------------------------------------------------------------------------
template <int K, int M, int T, bool VEC, class Lay, bool SP = false>
static int launch(const double *c2, const double *c1, const double *e, const double *f1,
                  const double *f2, const double *b, double *x, int32_t *st, int32_t *ix,
                  int64_t *nz, int64_t batch, int64_t n, Lay lay, cudaStream_t stream,
                  Outer outer = Outer{nullptr, nullptr, nullptr, 0}) {
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
  if (csize > 1) {  // single-CTA systems write status/index/nz in the kernel
    if (nz) cudaMemsetAsync(nz, 0, sizeof(int64_t) * (size_t)batch, stream);
    if (st) cudaMemsetAsync(st, 0, sizeof(int32_t) * (size_t)batch, stream);     // BX_STATUS_OK
    if (ix) cudaMemsetAsync(ix, 0xff, sizeof(int32_t) * (size_t)batch, stream);  // -1
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
  cudaError_t err = cudaLaunchKernelEx(&cfg, kern, c2, c1, e, f1, f2, b, x, st, ix, nz, batch, n,
                                       lay, csize, outer);
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
                     int64_t *nz, int64_t batch, int64_t n, Lay lay, cudaStream_t stream) {
  // rows per CTA = M*T; small systems use small CTAs (many CTAs per SM).
  // BX_PART_CFG (developer knob, benchmarking only) forces one configuration.
  static int forced = -2;
  if (forced == -2) {
    const char *env = getenv("BX_PART_CFG");
    forced = env ? atoi(env) : -1;
  }
  switch (forced) {
    case 0: return launch<K, 8, 32, VEC, Lay>(c2, c1, e, f1, f2, b, x, st, ix, nz, batch, n, lay, stream);
    case 1: return launch<K, 8, 64, VEC, Lay>(c2, c1, e, f1, f2, b, x, st, ix, nz, batch, n, lay, stream);
    case 2: return launch<K, 8, 128, VEC, Lay>(c2, c1, e, f1, f2, b, x, st, ix, nz, batch, n, lay, stream);
    case 3: return launch<K, 16, 64, VEC, Lay>(c2, c1, e, f1, f2, b, x, st, ix, nz, batch, n, lay, stream);
    case 4: return launch<K, 16, 32, VEC, Lay>(c2, c1, e, f1, f2, b, x, st, ix, nz, batch, n, lay, stream);
    case 5: return launch<K, 32, 32, VEC, Lay>(c2, c1, e, f1, f2, b, x, st, ix, nz, batch, n, lay, stream);
    case 6: return launch<K, 16, 128, VEC, Lay>(c2, c1, e, f1, f2, b, x, st, ix, nz, batch, n, lay, stream);
    default: break;
  }
  if (n <= 256) return launch<K, 8, 32, VEC, Lay>(c2, c1, e, f1, f2, b, x, st, ix, nz, batch, n, lay, stream);
  if (n <= 512) return launch<K, 8, 64, VEC, Lay>(c2, c1, e, f1, f2, b, x, st, ix, nz, batch, n, lay, stream);
  if (use_1k_ctas(n)) return launch<K, 16, 64, VEC, Lay>(c2, c1, e, f1, f2, b, x, st, ix, nz, batch, n, lay, stream);
  return launch<K, 16, 128, VEC, Lay>(c2, c1, e, f1, f2, b, x, st, ix, nz, batch, n, lay, stream);
}

// sparse +-2 diagonals (MNPDM): default shapes only, K = 2
template <bool VEC, class Lay>
static int dispatch_sparse(const double *c1, const double *e, const double *f1, const double *b,
                           double *x, int32_t *st, int32_t *ix, int64_t *nz, int64_t batch,
                           int64_t n, Lay lay, cudaStream_t stream, Outer o) {
  if (n <= 256)
    return launch<2, 8, 32, VEC, Lay, true>(nullptr, c1, e, f1, nullptr, b, x, st, ix, nz, batch, n, lay, stream, o);
  if (n <= 512)
    return launch<2, 8, 64, VEC, Lay, true>(nullptr, c1, e, f1, nullptr, b, x, st, ix, nz, batch, n, lay, stream, o);
  if (n <= 1024)  // the 1024-row shape measured slower here (n=4096: 0.668 vs 0.632 ms)
    return launch<2, 16, 64, VEC, Lay, true>(nullptr, c1, e, f1, nullptr, b, x, st, ix, nz, batch, n, lay, stream, o);
  return launch<2, 16, 128, VEC, Lay, true>(nullptr, c1, e, f1, nullptr, b, x, st, ix, nz, batch, n, lay, stream, o);
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
                    bool vec_ok) {
  vec_ok = vec_ok && aligned32(c2) && aligned32(c1) && aligned32(e) && aligned32(f1) &&
           aligned32(f2) && aligned32(b) && aligned32(x);
  if (vec_ok) return dispatch2<K, true>(c2, c1, e, f1, f2, b, x, st, ix, nz, batch, n, lay, stream);
  return dispatch2<K, false>(c2, c1, e, f1, f2, b, x, st, ix, nz, batch, n, lay, stream);
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
  return 2 * flag_bytes(batch) + 8 * fixup_scratch_doubles(bandwidth == 1 ? 0 : 1, n);
}

// workspace: flags [batch][8] | nz parts [batch][8] | re-solve scratch
static void carve(double *ws, int64_t batch, int32_t *&flags, int32_t *&nzpart, double *&scratch) {
  char *p = reinterpret_cast<char *>(ws);
  flags = reinterpret_cast<int32_t *>(p);
  nzpart = reinterpret_cast<int32_t *>(p + flag_bytes(batch));
  scratch = reinterpret_cast<double *>(p + 2 * flag_bytes(batch));
}

int ntdm_part(const double *d, const double *e, const double *f, const double *b, double *x,
              double *ws, int32_t *st, int32_t *ix, int64_t batch, int64_t n, int64_t ld, int layout,
              cudaStream_t stream) {
  int32_t *flags, *nzpart;
  double *scratch;
  carve(ws, batch, flags, nzpart, scratch);
  const double *ptrs[] = {d, e, f, b, x};
  int rc = BX_ERR_UNSUPPORTED, fs = 1;
  if (seg_enabled() && seg_applicable(ptrs, 5, n, ld, layout))
    rc = seg_solve(1, nullptr, d, e, f, nullptr, b, x, flags, nullptr, batch, n, ld, stream, &fs);
  if (rc == BX_ERR_UNSUPPORTED) {
    fs = 1;
    if (layout == BX_LAYOUT_SYSTEM_MAJOR)
      rc = part::dispatch<1>(nullptr, d, e, f, nullptr, b, x, flags, nullptr, nullptr, batch, n,
                             SystemMajor{ld}, stream, ld % 4 == 0);
    else
      rc = part::dispatch<1>(nullptr, d, e, f, nullptr, b, x, flags, nullptr, nullptr, batch, n,
                             Interleaved{ld}, stream, false);
  }
  if (rc != BX_OK) return rc;
  direct_fixup(0, nullptr, d, e, f, nullptr, b, x, scratch, flags, fs, nullptr, st, ix, nullptr,
               batch, n, ld, layout, stream);
  return bxh::check_launch("partitioned solver re-solve");
}

int penta_part(bool mod, const double *c, const double *d, const double *e, const double *f,
               const double *g, const double *b, double *x, double *ws, int32_t *st, int32_t *ix,
               int64_t *nz, int64_t batch, int64_t n, int64_t ld, int layout, cudaStream_t stream) {
  int32_t *flags, *nzpart;
  double *scratch;
  carve(ws, batch, flags, nzpart, scratch);
  const double *ptrs[] = {c, d, e, f, g, b, x};
  int rc = BX_ERR_UNSUPPORTED, fs = 1;
  bool seg = false;
  if (seg_enabled() && seg_applicable(ptrs, 7, n, ld, layout)) {
    rc = seg_solve(2, c, d, e, f, g, b, x, flags, nz ? nzpart : nullptr, batch, n, ld, stream, &fs);
    seg = rc != BX_ERR_UNSUPPORTED;
  }
  if (!seg) {
    fs = 1;
    if (layout == BX_LAYOUT_SYSTEM_MAJOR)
      rc = part::dispatch<2>(c, d, e, f, g, b, x, flags, nullptr, nz, batch, n, SystemMajor{ld},
                             stream, ld % 4 == 0);
    else
      rc = part::dispatch<2>(c, d, e, f, g, b, x, flags, nullptr, nz, batch, n, Interleaved{ld},
                             stream, false);
  }
  if (rc != BX_OK) return rc;
  direct_fixup(mod ? 2 : 1, c, d, e, f, g, b, x, scratch, flags, fs, seg && nz ? nzpart : nullptr,
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
  if (layout == BX_LAYOUT_SYSTEM_MAJOR) {
    const bool vec = ld % 4 == 0 && part::aligned32(d) && part::aligned32(e) && part::aligned32(f) &&
                     part::aligned32(b) && part::aligned32(x);
    if (vec)
      return part::dispatch_sparse<true>(d, e, f, b, x, st, ix, nz, batch, n, SystemMajor{ld}, stream, o);
    return part::dispatch_sparse<false>(d, e, f, b, x, st, ix, nz, batch, n, SystemMajor{ld}, stream, o);
  }
  return part::dispatch_sparse<false>(d, e, f, b, x, st, ix, nz, batch, n, Interleaved{ld}, stream, o);
}

size_t other_workspace_bytes(int solver, int64_t batch, int64_t n) {
  if (solver == BX_SOLVER_SIP) return sip_workspace_bytes(batch, n);
  if (solver == BX_SOLVER_STDM) return exact_workspace_bytes(1, batch, n);
  if (solver == BX_SOLVER_SPDM) return exact_workspace_bytes(2, batch, n);
  return 0;
}

}  // namespace bx
