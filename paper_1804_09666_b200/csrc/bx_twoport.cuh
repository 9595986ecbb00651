// Two-port algebra shared by the partitioned direct solvers
// (bx_direct_part.cu, bx_direct_pers.cu): a chunk of consecutive rows of a
// banded system of half-bandwidth K is summarised by its first K unknowns F
// and last K unknowns E as affine functions of the K unknowns just left (L)
// and right (R) of it; adjacent chunks merge by eliminating their interface.
#pragma once
#include "bx_common.cuh"

namespace bx {
namespace part {

// 1/a to ~1 ulp: MUFU seed + two Newton steps (tolerance path only)
__device__ __forceinline__ double rcp(double a) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a));
  double e = fma(-a, r, 1.0);
  r = fma(r, e, r);
  e = fma(-a, r, 1.0);
  return fma(r, e, r);
}

template <int K>
struct Vec {
  double v[K];
};
template <int K>
struct Mat {
  double m[K][K];
};

template <int K>
__device__ __forceinline__ Vec<K> mv(const Mat<K> &a, const Vec<K> &x) {
  Vec<K> r;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < K; ++j) s = fma(a.m[i][j], x.v[j], s);
    r.v[i] = s;
  }
  return r;
}
template <int K>
__device__ __forceinline__ Mat<K> mm(const Mat<K> &a, const Mat<K> &b) {
  Mat<K> r;
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int j = 0; j < K; ++j) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < K; ++k) s = fma(a.m[i][k], b.m[k][j], s);
      r.m[i][j] = s;
    }
  return r;
}
template <int K>
__device__ __forceinline__ Vec<K> vadd(const Vec<K> &a, const Vec<K> &b) {
  Vec<K> r;
#pragma unroll
  for (int i = 0; i < K; ++i) r.v[i] = a.v[i] + b.v[i];
  return r;
}
template <int K>
__device__ __forceinline__ Mat<K> madd(const Mat<K> &a, const Mat<K> &b) {
  Mat<K> r;
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int j = 0; j < K; ++j) r.m[i][j] = a.m[i][j] + b.m[i][j];
  return r;
}
// (I - P)^{-1}; returns false if singular
template <int K>
__device__ __forceinline__ bool inv_i_minus(const Mat<K> &p, Mat<K> &out) {
  if (K == 1) {
    const double d = 1.0 - p.m[0][0];
    out.m[0][0] = rcp(d);
    return d != 0.0;
  } else {
    const double a = 1.0 - p.m[0][0], b = -p.m[0][1], c = -p.m[1][0], d = 1.0 - p.m[1][1];
    const double det = a * d - b * c;
    const double r = rcp(det);
    out.m[0][0] = d * r;
    out.m[0][1] = -b * r;
    out.m[1][0] = -c * r;
    out.m[1][1] = a * r;
    return det != 0.0;
  }
}

// one side (F or E) of a two-port: x = g + A L + B R
template <int K>
struct Port {
  Vec<K> g;
  Mat<K> A, B;
};
template <int K>
struct TwoPort {
  Port<K> F, E;
};
// what the descent needs at a merge node: u (left child's E) and v (right
// child's F) as affine functions of the merged node's L and R
template <int K>
struct MergeInfo {
  Port<K> u, v;
};

template <int K>
__device__ __forceinline__ bool merge(const TwoPort<K> &a, const TwoPort<K> &b, TwoPort<K> &out,
                                      MergeInfo<K> &info) {
  Mat<K> S;
  const bool ok = inv_i_minus<K>(mm<K>(a.E.B, b.F.A), S);
  // u = S (gAE + BAE gBF) + S AAE L + S BAE BBF R
  info.u.g = mv<K>(S, vadd<K>(a.E.g, mv<K>(a.E.B, b.F.g)));
  info.u.A = mm<K>(S, a.E.A);
  info.u.B = mm<K>(S, mm<K>(a.E.B, b.F.B));
  // v = gBF + ABF u + BBF R
  info.v.g = vadd<K>(b.F.g, mv<K>(b.F.A, info.u.g));
  info.v.A = mm<K>(b.F.A, info.u.A);
  info.v.B = madd<K>(mm<K>(b.F.A, info.u.B), b.F.B);
  // merged F = A.F with its R replaced by v ; merged E = B.E with L replaced by u
  out.F.g = vadd<K>(a.F.g, mv<K>(a.F.B, info.v.g));
  out.F.A = madd<K>(a.F.A, mm<K>(a.F.B, info.v.A));
  out.F.B = mm<K>(a.F.B, info.v.B);
  out.E.g = vadd<K>(b.E.g, mv<K>(b.E.A, info.u.g));
  out.E.A = mm<K>(b.E.A, info.u.A);
  out.E.B = madd<K>(mm<K>(b.E.A, info.u.B), b.E.B);
  return ok;
}

// The two halves of merge(), for two warps working one merge together:
//   merge_u(a.E, b.F, b.E): S = (I - aE.B bF.A)^-1, u (the left child's E as a
//     function of the merged L, R) and the merged node's E;
//   merge_v(a.E, b.F, a.F): T = (I - bF.A aE.B)^-1, v (the right child's F)
//     and the merged node's F -- the mirror image, same cost (78 FP64 ops
//     each for K=2 against 130 for the whole merge).
template <int K>
__device__ __forceinline__ bool merge_u(const Port<K> &aE, const Port<K> &bF, const Port<K> &bE,
                                        Port<K> &u, Port<K> &outE) {
  Mat<K> S;
  const bool ok = inv_i_minus<K>(mm<K>(aE.B, bF.A), S);
  u.g = mv<K>(S, vadd<K>(aE.g, mv<K>(aE.B, bF.g)));
  u.A = mm<K>(S, aE.A);
  u.B = mm<K>(S, mm<K>(aE.B, bF.B));
  outE.g = vadd<K>(bE.g, mv<K>(bE.A, u.g));
  outE.A = mm<K>(bE.A, u.A);
  outE.B = madd<K>(mm<K>(bE.A, u.B), bE.B);
  return ok;
}
template <int K>
__device__ __forceinline__ bool merge_v(const Port<K> &aE, const Port<K> &bF, const Port<K> &aF,
                                        Port<K> &v, Port<K> &outF) {
  Mat<K> Tm;
  const bool ok = inv_i_minus<K>(mm<K>(bF.A, aE.B), Tm);
  v.g = mv<K>(Tm, vadd<K>(bF.g, mv<K>(bF.A, aE.g)));
  v.A = mm<K>(Tm, mm<K>(bF.A, aE.A));
  v.B = mm<K>(Tm, bF.B);
  outF.g = vadd<K>(aF.g, mv<K>(aF.B, v.g));
  outF.A = madd<K>(aF.A, mm<K>(aF.B, v.A));
  outF.B = mm<K>(aF.B, v.B);
  return ok;
}

// one Port of a merge info (component offset c0: 0 = u, NP/2 = v), SoA
template <int K, int T>
__device__ __forceinline__ void store_port(double *base, int c0, int node, const Port<K> &p) {
  const double *v = reinterpret_cast<const double *>(&p);
#pragma unroll
  for (int c = 0; c < (int)(sizeof(Port<K>) / 8); ++c) base[(c0 + c) * T + node] = v[c];
}

template <int K>
__device__ __forceinline__ Vec<K> apply(const Port<K> &p, const Vec<K> &L, const Vec<K> &R) {
  return vadd<K>(p.g, vadd<K>(mv<K>(p.A, L), mv<K>(p.B, R)));
}

// merge info in shared memory, structure-of-arrays: component c of node k at
// base[c * T + k] (consecutive nodes -> consecutive banks)
template <int K, int T>
__device__ __forceinline__ void store_info(double *base, int node, const MergeInfo<K> &mi) {
  const double *v = reinterpret_cast<const double *>(&mi);
#pragma unroll
  for (int c = 0; c < (int)(sizeof(MergeInfo<K>) / 8); ++c) base[c * T + node] = v[c];
}
template <int K, int T>
__device__ __forceinline__ MergeInfo<K> load_info(const double *base, int node) {
  MergeInfo<K> mi;
  double *v = reinterpret_cast<double *>(&mi);
#pragma unroll
  for (int c = 0; c < (int)(sizeof(MergeInfo<K>) / 8); ++c) v[c] = base[c * T + node];
  return mi;
}

__device__ __forceinline__ unsigned smem_addr(const void *p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

// 32-byte vector global accesses (LDG.E.ENL2.256 / STG.E.ENL2.256 on sm_100a);
// streaming: no L1 allocation for data that is touched once
__device__ __forceinline__ void ld4(const double *p, double *o) {
  asm("ld.global.nc.L1::no_allocate.v4.f64 {%0, %1, %2, %3}, [%4];"
      : "=d"(o[0]), "=d"(o[1]), "=d"(o[2]), "=d"(o[3])
      : "l"(p));
}
__device__ __forceinline__ void st4(double *p, const double *v) {
  asm volatile("st.global.L1::no_allocate.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(v[0]),
               "d"(v[1]), "d"(v[2]), "d"(v[3])
               : "memory");
}

template <int K>
__device__ __forceinline__ TwoPort<K> shfl_down_port(const TwoPort<K> &p, int delta) {
  TwoPort<K> r;
  const double *src = reinterpret_cast<const double *>(&p);
  double *dst = reinterpret_cast<double *>(&r);
#pragma unroll
  for (int i = 0; i < (int)(sizeof(TwoPort<K>) / 8); ++i)
    dst[i] = __shfl_down_sync(0xffffffffu, src[i], delta);
  return r;
}
template <int K>
__device__ __forceinline__ Vec<K> shfl_up_vec(const Vec<K> &v, int delta) {
  Vec<K> r;
#pragma unroll
  for (int i = 0; i < K; ++i) r.v[i] = __shfl_up_sync(0xffffffffu, v.v[i], delta);
  return r;
}

}  // namespace part
}  // namespace bx
