// Segment-resident partitioned direct solver for system-major band systems of
// half-bandwidth K (K=1: NTDM, K=2: NPDM / MNPDM) -- the throughput path of
// BX_ALGO_PARTITIONED.  Same solution contract as the reference solvers
// (solve_ntdm / solve_npdm / solve_mnpdm, direct.py:73-113; the elimination
// of _elim.py:30-190 in a different order): results agree with the reference
// to rounding (<= 1e-10 relative, north star), not bitwise.
//
// A system is cut into C segments of R = 32*W*M rows; one CTA of W warps per
// segment, the C CTAs of a system form a thread-block cluster.  Lane t of a
// CTA owns the M consecutive rows [t*M, t*M+M) of its segment.
//   load     the CTA copies its segment of every diagonal and of the rhs into
//            shared memory with coalesced 16-byte cp.async (each warp request
//            covers whole 128-byte lines: 4 L2 sectors per request, not the
//            one sector a lane's own rows would give), XOR-swizzled so that
//            the lanes' row-strided reads below are bank-conflict free.  The
//            segment stays resident: nothing is read from HBM twice.
//   phase 1  one forward pass over the lane's rows: elimination against the
//            chunk's own normalised rows with the left coupling carried as a
//            spike W (x_j + p_j x_{j+1} + q_j x_{j+2} + W_j.L = y_j) and the
//            first K unknowns carried forward as affine functions of L and the
//            two newest unknowns ("top tracking"): at the end the chunk's
//            first and last K unknowns are affine in (L, R) -- its two-port --
//            with O(1) registers.
//   tree     two-port merges: 5 levels inside each warp (shuffles, merge
//            infos in shared memory); the W*C warp roots of the cluster are
//            read by warp 0 of every CTA through distributed shared memory
//            and merged/descended redundantly (<= 32 leaves, one warp); then
//            the in-warp descent hands every lane its L and R.
//   phase 3  the same elimination with L folded into the start rows, then
//            back-substitution from R in registers; x overwrites the rhs
//            slot in shared memory and leaves with coalesced stores.
// HBM traffic is the compulsory I/O (K=2: 48 B read + 8 B written per row).
//
// Pivots that are zero or not finite in this elimination order (chunk-local
// pivots, interface determinants) flag the segment; direct_fixup
// (bx_direct_seq.cu) then re-solves flagged systems in the reference's
// operation order, so their status / index / x are the reference's
// (ZeroPivot(i) of _elim.py:26-27,57,107).
#include <stdlib.h>

#include "bx_common.cuh"
#include "bx_kernels.h"
#include "bx_twoport.cuh"

#ifdef BX_SEG_TRACE
// developer instrumentation (tools/trace_seg.cu): per-CTA phase clocks of lane 0
__device__ long long g_seg_trace[65536][8];
#define BX_ST(slot)                                                                     \
  do {                                                                                  \
    if (threadIdx.x == 0 && blockIdx.x < 65536u) g_seg_trace[blockIdx.x][slot] = clock64(); \
  } while (0)
#else
#define BX_ST(slot) \
  do {              \
  } while (0)
#endif

namespace bx {
namespace seg {

using part::MergeInfo;
using part::Port;
using part::rcp;
using part::TwoPort;
using part::Vec;

template <class T>
__device__ __forceinline__ T shfl_up_t(const T &v, int d) {
  T r;
  const double *s = reinterpret_cast<const double *>(&v);
  double *o = reinterpret_cast<double *>(&r);
#pragma unroll
  for (int i = 0; i < (int)(sizeof(T) / 8); ++i) o[i] = __shfl_up_sync(0xffffffffu, s[i], d);
  return r;
}
template <class T>
__device__ __forceinline__ T shfl_down_t(const T &v, int d) {
  T r;
  const double *s = reinterpret_cast<const double *>(&v);
  double *o = reinterpret_cast<double *>(&r);
#pragma unroll
  for (int i = 0; i < (int)(sizeof(T) / 8); ++i) o[i] = __shfl_down_sync(0xffffffffu, s[i], d);
  return r;
}
// structure-of-arrays POD of doubles: component c of slot k at base[c * stride + k]
template <class T>
__device__ __forceinline__ void soa_store(double *base, int stride, int k, const T &v) {
  const double *s = reinterpret_cast<const double *>(&v);
#pragma unroll
  for (int c = 0; c < (int)(sizeof(T) / 8); ++c) base[c * stride + k] = s[c];
}
template <class T>
__device__ __forceinline__ T soa_load(const double *base, int stride, int k) {
  T v;
  double *o = reinterpret_cast<double *>(&v);
#pragma unroll
  for (int c = 0; c < (int)(sizeof(T) / 8); ++c) o[c] = base[c * stride + k];
  return v;
}
// the same from a peer CTA of the cluster (distributed shared memory)
template <class T>
__device__ __forceinline__ T soa_load_peer(const double *base, int stride, int k, int rank) {
  T v;
  double *o = reinterpret_cast<double *>(&v);
  unsigned a;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(part::smem_addr(base + k)), "r"(rank));
#pragma unroll
  for (int c = 0; c < (int)(sizeof(T) / 8); ++c)
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(o[c]) : "r"(a + 8u * (unsigned)(c * stride)));
  return v;
}

// the interface determinant of merge(a, b) (merge() itself only reports == 0)
__device__ __forceinline__ bool good_det(const TwoPort<2> &a, const TwoPort<2> &b) {
  const double p00 = a.E.B.m[0][0] * b.F.A.m[0][0] + a.E.B.m[0][1] * b.F.A.m[1][0];
  const double p01 = a.E.B.m[0][0] * b.F.A.m[0][1] + a.E.B.m[0][1] * b.F.A.m[1][1];
  const double p10 = a.E.B.m[1][0] * b.F.A.m[0][0] + a.E.B.m[1][1] * b.F.A.m[1][0];
  const double p11 = a.E.B.m[1][0] * b.F.A.m[0][1] + a.E.B.m[1][1] * b.F.A.m[1][1];
  const double det = (1.0 - p00) * (1.0 - p11) - p01 * p10;
  return det != 0.0 && isfinite(det);
}
__device__ __forceinline__ bool good_det(const TwoPort<1> &a, const TwoPort<1> &b) {
  const double det = 1.0 - a.E.B.m[0][0] * b.F.A.m[0][0];
  return det != 0.0 && isfinite(det);
}

// two-port of an empty segment (F = R, E = L): the padding leaf of a tree
// whose leaf count is not a power of two; merging with it is the identity
template <int K>
__device__ __forceinline__ TwoPort<K> empty_port() {
  TwoPort<K> p;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    p.F.g.v[i] = p.E.g.v[i] = 0.0;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      p.F.A.m[i][j] = 0.0;
      p.F.B.m[i][j] = i == j ? 1.0 : 0.0;
      p.E.A.m[i][j] = i == j ? 1.0 : 0.0;
      p.E.B.m[i][j] = 0.0;
    }
  }
  return p;
}

// in-warp merge nodes: level l (0..4) has 16 >> l nodes; 31 per warp
__device__ __forceinline__ int node_id(int l, int lane) { return (32 - (32 >> l)) + (lane >> (l + 1)); }

// 1/a to ~1 ulp with one cubic correction of the MUFU seed (3 dependent
// DFMA after MUFU.RCP64H instead of the two Newton steps' 4): e = 1 - a r,
// r (1 + e + e^2) has relative error e^3
__device__ __forceinline__ double rcp3(double a) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a));
  double e = fma(-a, r, 1.0);
  e = fma(e, e, e);
  return fma(r, e, r);
}

// ---- boundary-lane two-port tree ---------------------------------------------
// A segment of leaves [a, b] keeps its F port (first K unknowns, affine in the
// segment's outer unknowns L, R) on its first lane a and its E port on its
// last lane b.  Merging children [a, m], [m+1, b] eliminates the interface
// (u = left child's E, v = right child's F): lane b computes u and the merged
// E, lane a the mirror image (v, merged F) -- the same code with the roles of
// L and R swapped (mirror = swap a port's A and B), so the warp executes ONE
// half-merge of ~80 FP64 ops per level instead of the full merge's ~135.
template <int K>
__device__ __forceinline__ Port<K> mirror(const Port<K> &p) {
  Port<K> r;
  r.g = p.g;
  r.A = p.B;
  r.B = p.A;
  return r;
}
template <int K>
__device__ __forceinline__ Port<K> sel_port(bool c, const Port<K> &x, const Port<K> &y) {
  Port<K> r;
  const double *xs = reinterpret_cast<const double *>(&x);
  const double *ys = reinterpret_cast<const double *>(&y);
  double *o = reinterpret_cast<double *>(&r);
#pragma unroll
  for (int i = 0; i < (int)(sizeof(Port<K>) / 8); ++i) o[i] = c ? xs[i] : ys[i];
  return r;
}
template <class T>
__device__ __forceinline__ T shfl_idx_t(const T &v, int src) {
  T r;
  const double *s = reinterpret_cast<const double *>(&v);
  double *o = reinterpret_cast<double *>(&r);
#pragma unroll
  for (int i = 0; i < (int)(sizeof(T) / 8); ++i) o[i] = __shfl_sync(0xffffffffu, s[i], src);
  return r;
}
// x = X(L, y), y = Y(x, R)  =>  x = w(L, R) with w = S (X.g + X.B Y.g) + S X.A L
// + S X.B Y.B R, S = (I - X.B Y.A)^-1; out = Z(x, R).  Returns det != 0, finite.
template <int K>
__device__ __forceinline__ bool half_merge(const Port<K> &X, const Port<K> &Y, const Port<K> &Z,
                                           Port<K> &w, Port<K> &out) {
  using part::mm;
  using part::mv;
  using part::vadd;
  using part::madd;
  part::Mat<K> S;
  const part::Mat<K> P = mm<K>(X.B, Y.A);
  double det;
  if (K == 1) {
    det = 1.0 - P.m[0][0];
    S.m[0][0] = rcp3(det);
  } else {
    const double a = 1.0 - P.m[0][0], b = -P.m[0][1], c = -P.m[1][0], d = 1.0 - P.m[K - 1][K - 1];
    det = fma(a, d, -b * c);
    const double r = rcp3(det);
    S.m[0][0] = d * r;
    S.m[0][K - 1] = -b * r;
    S.m[K - 1][0] = -c * r;
    S.m[K - 1][K - 1] = a * r;
  }
  w.g = mv<K>(S, vadd<K>(X.g, mv<K>(X.B, Y.g)));
  w.A = mm<K>(S, X.A);
  w.B = mm<K>(S, mm<K>(X.B, Y.B));
  out.g = vadd<K>(Z.g, mv<K>(Z.A, w.g));
  out.A = mm<K>(Z.A, w.A);
  out.B = madd<K>(mm<K>(Z.A, w.B), Z.B);
  return det != 0.0 && isfinite(det);
}
// up-sweep over the first 2^levels lanes; w ports of level j, segment k, role
// (0 = first lane, 1 = last lane) at slot wbase + 2 * node_id(j, lane) + role
template <int K>
__device__ __forceinline__ void tree_up(TwoPort<K> &P, int levels, int lane, double *wst, int wstride,
                                        int wbase, bool &bad) {
#pragma unroll 1
  for (int j = 0; j < levels; ++j) {
    const int span = 2 << j, a = lane & ~(span - 1), b = a + span - 1, m = a + (span >> 1) - 1;
    const Port<K> aE = shfl_idx_t(P.E, m);      // left child's E
    const Port<K> bF = shfl_idx_t(P.F, m + 1);  // right child's F
    const bool isA = lane == a, isB = lane == b;
    const Port<K> X = sel_port(isA, mirror(bF), aE);
    const Port<K> Y = sel_port(isA, mirror(aE), bF);
    const Port<K> Z = sel_port(isA, mirror(P.F), P.E);
    Port<K> w, out;
    const bool ok = half_merge<K>(X, Y, Z, w, out);
    if (isA) P.F = mirror(out);
    if (isB) P.E = out;
    if (isA || isB) {
      bad |= !ok;
      soa_store(wst, wstride, wbase + 2 * node_id(j, lane) + (isB ? 1 : 0), w);
    }
  }
}
// descent: role lanes hold their segment's (L, R); at the end every lane
// holds its leaf's
template <int K>
__device__ __forceinline__ void tree_down(Vec<K> &L, Vec<K> &R, int levels, int lane, const double *wst,
                                          int wstride, int wbase) {
#pragma unroll 1
  for (int j = levels - 1; j >= 0; --j) {
    const int span = 2 << j, a = lane & ~(span - 1), b = a + span - 1, m = a + (span >> 1) - 1;
    const bool isA = lane == a, isB = lane == b;
    if (isA || isB) {
      const Port<K> wp = soa_load<Port<K>>(wst, wstride, wbase + 2 * node_id(j, lane) + (isB ? 1 : 0));
      // A: v (right child's F) = wp(R, L) mirrored; B: u (left child's E) = wp(L, R)
      const Vec<K> x = part::apply<K>(wp, isA ? R : L, isA ? L : R);
      if (isA) R = x;  // A keeps (L, v): the left child's boundaries
      else L = x;      // B keeps (u, R): the right child's
    }
    const Vec<K> La = shfl_idx_t(L, a), Ra = shfl_idx_t(R, a);
    const Vec<K> Lb = shfl_idx_t(L, b), Rb = shfl_idx_t(R, b);
    if (lane == m && !isA) { L = La; R = Ra; }
    if (lane == m + 1 && !isB) { L = Lb; R = Rb; }
  }
}

template <int K, int W, int M>
struct Layout {
  static constexpr int T = W * 32;
  static constexpr int R = T * M;              // rows per segment
  static constexpr int NA = 2 * K + 2;         // diagonals + rhs
  static constexpr int NI = (int)(sizeof(MergeInfo<K>) / 8);
  static constexpr int NP = (int)(sizeof(TwoPort<K>) / 8);
  static constexpr int kIn = NA * R;           // [NA][R] swizzled rows
  static constexpr int NW = (int)(sizeof(Port<K>) / 8);
  static constexpr int kInfo = NW * W * 64;    // [NW][W*64] in-warp tree w ports (62 per warp)
  static constexpr int kUInfo = NW * 64;       // upper tree w ports
  static constexpr int kWPort = NP * W;        // this CTA's warp roots [NP][W]
  static constexpr int kWLR = 2 * K * W;       // per-warp L, R
  static constexpr size_t bytes = 8 * (size_t)(kIn + kInfo + kUInfo + kWPort + kWLR);
};

// 16-byte chunk q of a segment row array (rows 2q, 2q+1) lives at chunk
// phys(q): the low 3 bits are XORed with the owning lane's low 3 bits, so
// 8 consecutive lanes reading the same chunk of their own rows hit 8
// different 16-byte bank groups, and 8 consecutive chunks written by
// consecutive threads stay a permutation of one 128-byte bank row.
template <int M>
__device__ __forceinline__ int phys(int q) {
  constexpr int SW = M == 16 ? 3 : 4;  // log2(M / 2)
  return q ^ ((q >> SW) & 7);
}

template <int K>
struct Grp {
  double a2[4], a1[4], e[4], c1[4], c2[4], b[4];
};

// carried state of the two newest normalised rows (1 = row j-1, 2 = row
// j-2): x_i + f x_{i+1} + g x_{i+2} + W.L = y; plus row j-1's unnormalised
// x_{j} coefficient cp1 and reciprocal pivot r1, so that the next pivot is
// one DFMA after r1 (the pivot recurrence is the kernel's latency chain)
template <int K, bool SPIKE>
struct Fwd {
  double f1, g1, y1, f2, g2, y2, cp1, r1;
  double W1[K], W2[K];
};

template <int K, bool SPIKE>
__device__ __forceinline__ void fwd_start(Fwd<K, SPIKE> &s) {
  s.f1 = s.g1 = s.y1 = s.f2 = s.g2 = s.y2 = s.cp1 = s.r1 = 0.0;
}

// one elimination step: row j against the two stored rows before it
template <int K, bool SPIKE>
__device__ __forceinline__ void elim_row(Fwd<K, SPIKE> &s, double a2, double a1, double e,
                                         double c1, double c2, double b, double &pn, double &qn,
                                         double &yn, double *wn, bool &bad) {
  double mu, c1p, yy, ww[K];
  if (K == 2) {
    const double t1 = fma(-a2, s.f2, a1);
    const double e2 = fma(-a2, s.g2, e);
    const double b2 = fma(-a2, s.y2, b);
    mu = fma(-(t1 * s.cp1), s.r1, e2);  // e2 - t1 f1 with f1 = cp1 r1
    c1p = fma(-t1, s.g1, c1);
    yy = fma(-t1, s.y1, b2);
    if (SPIKE) {
#pragma unroll
      for (int k = 0; k < K; ++k) ww[k] = fma(-t1, s.W1[k], -a2 * s.W2[k]);
    }
  } else {
    mu = fma(-(a1 * s.cp1), s.r1, e);
    c1p = c1;
    yy = fma(-a1, s.y1, b);
    if (SPIKE) ww[0] = -a1 * s.W1[0];
  }
  bad |= !(mu != 0.0 && isfinite(mu));  // off the chain: a bad system is re-solved anyway
  const double r = rcp3(mu);
  pn = c1p * r;
  qn = K == 2 ? c2 * r : 0.0;
  yn = yy * r;
  if (SPIKE) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      wn[k] = ww[k] * r;
      s.W2[k] = s.W1[k];
      s.W1[k] = wn[k];
    }
  }
  s.f2 = s.f1; s.g2 = s.g1; s.y2 = s.y1;
  s.f1 = pn; s.g1 = qn; s.y1 = yn;
  s.cp1 = c1p; s.r1 = r;
}

template <int K, int W, int M>
__global__ void __launch_bounds__(W * 32)
seg_kernel(const double *__restrict__ c2p, const double *__restrict__ c1p,
           const double *__restrict__ ep, const double *__restrict__ f1p,
           const double *__restrict__ f2p, const double *__restrict__ bp,
           double *__restrict__ xp, int32_t *__restrict__ flags, int32_t *__restrict__ nzpart,
           int n, int64_t ld, int csize) {
  using LY = Layout<K, W, M>;
  constexpr int T = LY::T, R = LY::R, NA = LY::NA, G = 4, NG = M / G, HM = M / 2;
  constexpr int S = 16, NSC = M / S, SG = S / G;
  static_assert(M == 16 || M == 32, "M in {16, 32}");
  extern __shared__ __align__(128) double smem[];
  double *in = smem;
  double *info = in + LY::kIn;
  double *uinfo = info + LY::kInfo;
  double *wport = uinfo + LY::kUInfo;
  double *wlr = wport + LY::kWPort;

  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  int crank = 0;
  if (csize > 1) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  const int64_t s = blockIdx.x / csize;
  const int64_t sb = s * ld;
  const int seg0 = crank * R;
  const int base = seg0 + t * M;  // first system row of this lane's chunk
  const int rend = n - base;      // rows of the chunk inside the matrix (may be <= 0)
  const bool first = base == 0;

  const double *arrs[NA];
  if (K == 2) {
    arrs[0] = c2p; arrs[1] = c1p; arrs[2] = ep; arrs[3] = f1p; arrs[K == 2 ? 4 : 0] = f2p; arrs[NA - 1] = bp;
  } else {
    arrs[0] = c1p; arrs[1] = ep; arrs[2] = f1p; arrs[NA - 1] = bp;
  }

  BX_ST(0);
  // ---------------- load the segment (coalesced, swizzled) ------------------
#pragma unroll
  for (int a = 0; a < NA; ++a) {
#pragma unroll 4
    for (int q = t; q < R / 2; q += T) {
      const int row = seg0 + 2 * q;
      const int v = n - row;
      const unsigned bytes = (unsigned)min(max(v * 8, 0), 16);
      const double *src = arrs[a] + sb + (v > 0 ? row : 0);
      const unsigned dst = part::smem_addr(in + a * R + 2 * phys<M>(q));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  BX_ST(1);

  // group g (rows 4g..4g+3 of the lane's chunk) from shared memory
  auto read_group = [&](int g, Grp<K> &gr) {
    double *dd[NA];
    if (K == 2) {
      dd[0] = gr.a2; dd[1] = gr.a1; dd[2] = gr.e; dd[3] = gr.c1; dd[K == 2 ? 4 : 0] = gr.c2; dd[NA - 1] = gr.b;
    } else {
      dd[0] = gr.a1; dd[1] = gr.e; dd[2] = gr.c1; dd[NA - 1] = gr.b;
#pragma unroll
      for (int u = 0; u < 4; ++u) gr.a2[u] = gr.c2[u] = 0.0;
    }
    const int q0 = t * HM + 2 * g;
#pragma unroll
    for (int a = 0; a < NA; ++a) {
      const double2 v0 = *reinterpret_cast<const double2 *>(in + a * R + 2 * phys<M>(q0));
      const double2 v1 = *reinterpret_cast<const double2 *>(in + a * R + 2 * phys<M>(q0 + 1));
      dd[a][0] = v0.x; dd[a][1] = v0.y; dd[a][2] = v1.x; dd[a][3] = v1.y;
    }
  };
  // coefficient masks: slots outside the matrix are never trusted; rows >= n
  // are identity rows
  auto coeffs = [&](const Grp<K> &cur, int u, int j, double &a2, double &a1, double &e, double &c1,
                    double &c2, double &b) {
    a2 = K == 2 ? cur.a2[u] : 0.0;
    a1 = cur.a1[u];
    if (j < 2 && first) {
      a2 = 0.0;
      if (j < 1) a1 = 0.0;
    }
    e = j >= rend ? 1.0 : cur.e[u];
    c1 = j > rend - 2 ? 0.0 : cur.c1[u];
    c2 = (K != 2 || j > rend - 3) ? 0.0 : cur.c2[u];
    b = cur.b[u];
  };

  bool bad = false;
  int nzc = 0;

  // ---------------- phase 1: one forward pass, O(1) state ------------------
  Fwd<K, true> fs;
  fwd_start(fs);
#pragma unroll
  for (int k = 0; k < K; ++k) fs.W1[k] = fs.W2[k] = 0.0;
  if (K == 2) {  // virtual rows x_{-2} - L_0 = 0, x_{-1} - L_1 = 0
    fs.W2[0] = -1.0;
    fs.W1[1] = -1.0;
  } else {
    fs.W1[0] = -1.0;
  }
  double tg[K], tA[K][K], tc[K][K];  // x_tt = tg + tA.L + tc[0] x_{j+1} + tc[1] x_{j+2}
  Fwd<K, true> ck;                   // forward state after row S-1 (M = 2S)
  // Row loops are rolled (one 4-row group body): every CTA runs this code
  // once, and a fully unrolled kernel (~150 KB of SASS) was bound by
  // instruction-cache misses.
  auto track = [&](int tt, double pn, double qn, double yn, const double *wn) {
    const double c0 = tc[tt][0];
    tg[tt] = fma(c0, yn, tg[tt]);
#pragma unroll
    for (int k = 0; k < K; ++k) tA[tt][k] = fma(-c0, wn[k], tA[tt][k]);
    if (K == 2) {
      tc[tt][0] = fma(-c0, pn, tc[tt][K - 1]);
      tc[tt][K - 1] = -c0 * qn;
    } else {
      tc[tt][0] = -c0 * pn;
    }
  };
  {
    Grp<K> cur;
    read_group(0, cur);
#pragma unroll
    for (int u = 0; u < G; ++u) {  // group 0: the tracked rows start here
      double a2, a1, e, c1, c2, b;
      coeffs(cur, u, u, a2, a1, e, c1, c2, b);
      if (K == 2) nzc += (a2 != 0.0 && u < rend) ? 1 : 0;
      double pn, qn, yn, wn[K];
      elim_row<K, true>(fs, a2, a1, e, c1, c2, b, pn, qn, yn, wn, bad);
#pragma unroll
      for (int tt = 0; tt < K; ++tt) {
        if (tt == u) {
          tg[tt] = yn;
#pragma unroll
          for (int k = 0; k < K; ++k) tA[tt][k] = -wn[k];
          tc[tt][0] = -pn;
          if (K == 2) tc[tt][K - 1] = -qn;
        } else if (tt < u) {
          track(tt, pn, qn, yn, wn);
        }
      }
    }
  }
#pragma unroll 1
  for (int g = 1; g < NG; ++g) {
    Grp<K> cur;
    read_group(g, cur);
#pragma unroll
    for (int u = 0; u < G; ++u) {
      const int j = g * G + u;
      double a2, a1, e, c1, c2, b;
      coeffs(cur, u, j, a2, a1, e, c1, c2, b);
      if (K == 2) nzc += (a2 != 0.0 && j < rend) ? 1 : 0;
      double pn, qn, yn, wn[K];
      elim_row<K, true>(fs, a2, a1, e, c1, c2, b, pn, qn, yn, wn, bad);
#pragma unroll
      for (int tt = 0; tt < K; ++tt) track(tt, pn, qn, yn, wn);
    }
    if (NSC == 2 && g == S / G - 1) ck = fs;
  }
  // the chunk's two-port: F = first K unknowns, E = last K, affine in L, R
  TwoPort<K> P;
#pragma unroll
  for (int tt = 0; tt < K; ++tt) {
    P.F.g.v[tt] = tg[tt];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      P.F.A.m[tt][k] = tA[tt][k];
      P.F.B.m[tt][k] = tc[tt][k];
    }
  }
  if (K == 2) {
    // x_{M-1} = y1 - W1.L - f1 R0 - g1 R1 ; x_{M-2} = y2 - W2.L - f2 x_{M-1} - g2 R0
    P.E.g.v[1] = fs.y1;
    P.E.g.v[0] = fma(-fs.f2, fs.y1, fs.y2);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      P.E.A.m[1][k] = -fs.W1[k];
      P.E.A.m[0][k] = fma(fs.f2, fs.W1[k], -fs.W2[k]);
    }
    P.E.B.m[1][0] = -fs.f1;
    P.E.B.m[1][K - 1] = -fs.g1;
    P.E.B.m[0][0] = fma(fs.f2, fs.f1, -fs.g2);
    P.E.B.m[0][K - 1] = fs.f2 * fs.g1;
  } else {
    P.E.g.v[0] = fs.y1;
    P.E.A.m[0][0] = -fs.W1[0];
    P.E.B.m[0][0] = -fs.f1;
  }
  BX_ST(2);

  // ---------------- tree ------------------------------------------------------
#ifdef BX_SEG_NOTREE  // developer bound: skip the reduced solve (wrong x)
  Vec<K> myL, myR;
#pragma unroll
  for (int k = 0; k < K; ++k) myL.v[k] = myR.v[k] = P.F.g.v[k] * 1e-30;
  if (csize > 1) {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  }
#else
  tree_up<K>(P, 5, lane, info, W * 64, warp * 64, bad);
  if (lane == 0) soa_store(wport, 2 * W, 2 * warp, P.F);       // warp root: F on lane 0,
  if (lane == 31) soa_store(wport, 2 * W, 2 * warp + 1, P.E);  // E on lane 31
  if (csize > 1) {  // warp roots of the whole cluster visible (and every peer running)
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  } else {
    __syncthreads();
  }
  // upper tree over the cluster's W*C warp roots (padded to a power of two
  // with empty segments), computed by warp 0 of every CTA
  if (warp == 0) {
    const int leaves = W * csize;
    int lv = 0;
    while ((1 << lv) < leaves) ++lv;
    TwoPort<K> Q = empty_port<K>();
    if (lane < leaves) {
      const int r = lane / W, w = lane % W;
      if (r == crank) {
        Q.F = soa_load<Port<K>>(wport, 2 * W, 2 * w);
        Q.E = soa_load<Port<K>>(wport, 2 * W, 2 * w + 1);
      } else {
        Q.F = soa_load_peer<Port<K>>(wport, 2 * W, 2 * w, r);
        Q.E = soa_load_peer<Port<K>>(wport, 2 * W, 2 * w + 1, r);
      }
    }
    tree_up<K>(Q, lv, lane, uinfo, 64, 0, bad);
    Vec<K> uL, uR;  // the system's outer boundaries are L = R = 0
#pragma unroll
    for (int k = 0; k < K; ++k) uL.v[k] = uR.v[k] = 0.0;
    tree_down<K>(uL, uR, lv, lane, uinfo, 64, 0);
    if (lane / W == crank && lane < leaves) {
#pragma unroll
      for (int k = 0; k < K; ++k) {
        wlr[(lane % W) * 2 * K + k] = uL.v[k];
        wlr[(lane % W) * 2 * K + K + k] = uR.v[k];
      }
    }
  }
  if (csize > 1) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");  // peers' roots read
  __syncthreads();
  Vec<K> myL, myR;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    myL.v[k] = wlr[warp * 2 * K + k];
    myR.v[k] = wlr[warp * 2 * K + K + k];
  }
  tree_down<K>(myL, myR, 5, lane, info, W * 64, warp * 64);
#endif
  BX_ST(3);

  // ---------------- phase 3: eliminate with L folded, back-substitute ------
  // p, q, y of row j go to the dead e, c1, b slots of row j (its inputs have
  // been consumed); the back-substitution reads them and writes x_j over y_j
  double xn1 = myR.v[0], xn2 = K == 2 ? myR.v[K - 1] : 0.0;
  constexpr int AP = K == 2 ? 2 : 1, AQ = K == 2 ? 3 : 2, AY = NA - 1;  // e, c1, b slots
  auto slot = [&](int a, int j) -> double & {
    return in[a * R + 2 * phys<M>(t * HM + (j >> 1)) + (j & 1)];
  };
#pragma unroll 1
  for (int sc = NSC - 1; sc >= 0; --sc) {
    Fwd<K, false> fw;
    fwd_start(fw);
    if (sc == 0) {  // virtual start rows carry L
      if (K == 2) {
        fw.y2 = myL.v[0];
        fw.y1 = myL.v[K - 1];
      } else {
        fw.y1 = myL.v[0];
        fw.y2 = 0.0;
      }
    } else {  // checkpoint after row S-1, L folded into y
      fw.f1 = ck.f1; fw.g1 = ck.g1; fw.f2 = ck.f2; fw.g2 = ck.g2; fw.cp1 = ck.cp1; fw.r1 = ck.r1;
      double y1 = ck.y1, y2 = ck.y2;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        y1 = fma(-ck.W1[k], myL.v[k], y1);
        y2 = fma(-ck.W2[k], myL.v[k], y2);
      }
      fw.y1 = y1;
      fw.y2 = y2;
    }
#pragma unroll 1
    for (int g = 0; g < SG; ++g) {
      Grp<K> cur;
      read_group(sc * SG + g, cur);
#pragma unroll
      for (int u = 0; u < G; ++u) {
        const int j = (sc * SG + g) * G + u;
        double a2, a1, e, c1, c2, b, pn, qn, yn, wn[K];
        coeffs(cur, u, j, a2, a1, e, c1, c2, b);
        elim_row<K, false>(fw, a2, a1, e, c1, c2, b, pn, qn, yn, wn, bad);
        slot(AP, j) = pn;
        if (K == 2) slot(AQ, j) = qn;
        slot(AY, j) = yn;
      }
    }
#pragma unroll 4
    for (int jj = S - 1; jj >= 0; --jj) {
      const int j = sc * S + jj;
      double x = fma(-slot(AP, j), xn1, slot(AY, j));
      if (K == 2) x = fma(-slot(AQ, j), xn2, x);
      slot(AY, j) = x;
      xn2 = xn1;
      xn1 = x;
    }
  }
  BX_ST(4);
  __syncthreads();
  // coalesced copy-out of x
#pragma unroll 4
  for (int q = t; q < R / 2; q += T) {
    const int row = seg0 + 2 * q;
    if (row >= n) break;
    const double2 v = *reinterpret_cast<const double2 *>(in + (NA - 1) * R + 2 * phys<M>(q));
    if (row + 1 < n) {
      *reinterpret_cast<double2 *>(xp + sb + row) = v;
    } else {
      xp[sb + row] = v.x;
    }
  }

  // ---------------- flags / counters ------------------------------------------
  const bool any_bad = __syncthreads_or(bad);
  if (K == 2 && nzpart) {
    nzc = __reduce_add_sync(0xffffffffu, nzc);
    if (lane == 0) wlr[warp] = (double)nzc;  // wlr is free again
    __syncthreads();
  }
  if (t == 0) {
    flags[s * csize + crank] = any_bad ? 1 : 0;
    if (K == 2 && nzpart) {
      int tot = 0;
      for (int w = 0; w < W; ++w) tot += (int)wlr[w];
      nzpart[s * csize + crank] = tot;
    }
  }
  if (csize > 1) asm volatile("barrier.cluster.wait.aligned;" ::: "memory");  // no peer reads us any more
#ifdef BX_SEG_TRACE
  if (t == 0 && blockIdx.x < 65536u) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_seg_trace[blockIdx.x][5] = clock64();
    g_seg_trace[blockIdx.x][6] = smid;
  }
#endif
}

template <int K, int W, int M>
static int launch(const double *c2, const double *c1, const double *e, const double *f1,
                  const double *f2, const double *b, double *x, int32_t *flags, int32_t *nzpart,
                  int64_t batch, int64_t n, int64_t ld, int csize, cudaStream_t stream) {
  const size_t smem = Layout<K, W, M>::bytes;
  auto kern = seg_kernel<K, W, M>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_set = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(batch * csize));
  cfg.blockDim = dim3(W * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = csize;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t err = cudaLaunchKernelEx(&cfg, kern, c2, c1, e, f1, f2, b, x, flags, nzpart,
                                             (int)n, ld, csize);
  if (err != cudaSuccess) {
    bxh::set_error("segment solver launch: %s", cudaGetErrorString(err));
    return BX_ERR_CUDA;
  }
  return BX_OK;
}

static bool aligned16(const void *p) { return p == nullptr || ((uintptr_t)p & 15u) == 0; }

// Segment shapes (rows R = 32 W M per CTA, C = ceil(n / R) CTAs per cluster,
// C <= 8).  BX_SEG_CFG (developer knob, benchmarking only) forces one.
template <int K>
static int dispatch(const double *c2, const double *c1, const double *e, const double *f1,
                    const double *f2, const double *b, double *x, int32_t *flags, int32_t *nzpart,
                    int64_t batch, int64_t n, int64_t ld, cudaStream_t stream, int *csize_out) {
  static int forced = -2;
  if (forced == -2) {
    const char *env = getenv("BX_SEG_CFG");
    forced = env ? atoi(env) : -1;
  }
  int W = 2, M = 16;  // default: 1024-row segments
  switch (forced) {
    case 1: W = 1; M = 16; break;
    case 2: W = 2; M = 16; break;
    case 3: W = 4; M = 16; break;
    case 4: W = 1; M = 32; break;
    case 5: W = 2; M = 32; break;
    default:
      if (n <= 512) { W = 1; M = 16; }
      else if (n <= 1024) { W = 2; M = 16; }
      break;
  }
  int R = 32 * W * M;
  int C = (int)((n + R - 1) / R);
  if (C > 8 && forced < 0) {  // long systems: bigger segments
    W = 4; M = 16; R = 2048;
    C = (int)((n + R - 1) / R);
    if (C > 8) { W = 4; M = 32; R = 4096; C = (int)((n + R - 1) / R); }
  }
  if (C > 8) return BX_ERR_UNSUPPORTED;
  *csize_out = C;
#define BX_L(W_, M_) \
  if (W == W_ && M == M_) return launch<K, W_, M_>(c2, c1, e, f1, f2, b, x, flags, nzpart, batch, n, ld, C, stream)
  BX_L(1, 16);
  BX_L(2, 16);
  BX_L(4, 16);
  BX_L(1, 32);
  BX_L(2, 32);
  BX_L(4, 32);
#undef BX_L
  return BX_ERR_UNSUPPORTED;
}

}  // namespace seg

// Segment path applicability: system-major, 16-byte aligned rows (ld even),
// n <= 32768 (8 segments of 4096 rows).
bool seg_applicable(const double *const *ptrs, int nptr, int64_t n, int64_t ld, int layout) {
  if (layout != BX_LAYOUT_SYSTEM_MAJOR || ld % 2 != 0 || n > 32768 || n < 4) return false;
  for (int i = 0; i < nptr; ++i)
    if (!seg::aligned16(ptrs[i])) return false;
  return true;
}

int seg_solve(int K, const double *c2, const double *c1, const double *e, const double *f1,
              const double *f2, const double *b, double *x, int32_t *flags, int32_t *nzpart,
              int64_t batch, int64_t n, int64_t ld, cudaStream_t stream, int *csize) {
  if (K == 1)
    return seg::dispatch<1>(nullptr, c1, e, f1, nullptr, b, x, flags, nullptr, batch, n, ld, stream, csize);
  return seg::dispatch<2>(c2, c1, e, f1, f2, b, x, flags, nzpart, batch, n, ld, stream, csize);
}

}  // namespace bx
