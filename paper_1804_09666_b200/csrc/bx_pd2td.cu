// Pentadiagonal -> tridiagonal Gaussian reduction (pd_to_td) and the
// reduce-then-Thomas solve (solve_pd2td_ntdm), reference operation order.
//
//   pd_to_td          direct.py:116-165
//   solve_pd2td_ntdm  direct.py:168-177 (NTDM = bx_direct_seq.cu, bit-exact)
//
// One thread per system (the reduction is a pair of scalar recurrences):
//   pass 1, rows i = 2..n-1 ascending: a nonzero sub2 entry A[i,i-2] is
//     eliminated with row i-1 (pivot A[i-1,i-2], already final), touching
//     A[i,i-1], A[i,i], A[i,i+1] (only if A[i-1,i+1] != 0) and rhs_i;
//   pass 2, rows i = n-3..0 descending: a nonzero sup2 entry A[i,i+2] is
//     eliminated with row i+1 (pivot A[i+1,i+2], final), touching A[i,i],
//     A[i,i+1] and rhs_i.
// Every operation is one IEEE rounding (bx::mul/sub/dvd) in the reference's
// order, so the reduced system and the Thomas solution are bit-identical to
// bandix 0.1.0.  Zero tests are exact (is_zero on floats).  Operation counts
// (muls, subs, divs) are accumulated per system as the reference's
// CounterBox does.
#include "bx_common.cuh"
#include "bx_kernels.h"

namespace bx {

constexpr int kRedThreads = 32;

template <class Lay>
__global__ void __launch_bounds__(kRedThreads)
pd2td_kernel(const double *__restrict__ c, const double *__restrict__ d,
             const double *__restrict__ e, const double *__restrict__ f,
             const double *__restrict__ g, const double *__restrict__ b, double *__restrict__ td,
             double *__restrict__ te, double *__restrict__ tf, double *__restrict__ tr,
             int64_t *ops, int32_t *status, int32_t *index, int64_t batch, int64_t n, Lay in,
             Lay out) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= batch) return;
  int64_t muls = 0, subs = 0, divs = 0;
  // ---- pass 1 (direct.py:134-152): carried row i-1 after its own step
  double dp = 0.0, ep = 0.0, fp = 0.0, rp = 0.0, gp = 0.0;  // A[i-1,i-2], A[i-1,i-1], A[i-1,i], rhs, A[i-1,i+1]
  for (int64_t i = 0; i < n; ++i) {
    double di = i >= 1 ? ldg(d + in(i, s)) : 0.0;
    double ei = ldg(e + in(i, s));
    double fi = i <= n - 2 ? ldg(f + in(i, s)) : 0.0;
    double ri = ldg(b + in(i, s));
    const double gi = i <= n - 3 ? ldg(g + in(i, s)) : 0.0;
    if (i >= 2) {
      const double ci = ldg(c + in(i, s));
      if (ci != 0.0) {
        if (dp == 0.0) {  // ReductionPivotZero(i)
          set_status(status, index, s, BX_STATUS_REDUCTION_PIVOT, (int32_t)i);
          if (ops) { ops[3 * s] = muls; ops[3 * s + 1] = subs; ops[3 * s + 2] = divs; }
          return;
        }
        const double m = dvd(ci, dp);
        di = sub(di, mul(m, ep));
        ei = sub(ei, mul(m, fp));
        divs += 1; muls += 2; subs += 2;
        if (gp != 0.0) {  // gi_above = g[i-1] (i-1 <= n-3)
          fi = sub(fi, mul(m, gp));
          muls += 1; subs += 1;
        }
        ri = sub(ri, mul(m, rp));
        muls += 1; subs += 1;
      }
    }
    td[out(i, s)] = di;
    te[out(i, s)] = ei;
    tf[out(i, s)] = fi;
    tr[out(i, s)] = ri;
    dp = di; ep = ei; fp = fi; rp = ri; gp = gi;
  }
  // ---- pass 2 (direct.py:153-164): carried row i+1 after its own step
  // row n-1 / n-2 are never modified by pass 2; start the carry from them
  double dn = n >= 2 ? td[out(n - 1, s)] : 0.0;           // A[i+1,i]
  double en = n >= 2 ? te[out(n - 1, s)] : 0.0;           // A[i+1,i+1]
  double fn = n >= 2 ? tf[out(n - 1, s)] : 0.0;           // A[i+1,i+2]
  double rn = n >= 2 ? tr[out(n - 1, s)] : 0.0;
  if (n >= 3) {
    dn = td[out(n - 2, s)]; en = te[out(n - 2, s)]; fn = tf[out(n - 2, s)]; rn = tr[out(n - 2, s)];
  }
  for (int64_t i = n - 3; i >= 0; --i) {
    const double di = td[out(i, s)];
    double ei = te[out(i, s)], fi = tf[out(i, s)], ri = tr[out(i, s)];
    const double gi = ldg(g + in(i, s));
    if (gi != 0.0) {
      if (fn == 0.0) {  // ReductionPivotZero(i)
        set_status(status, index, s, BX_STATUS_REDUCTION_PIVOT, (int32_t)i);
        if (ops) { ops[3 * s] = muls; ops[3 * s + 1] = subs; ops[3 * s + 2] = divs; }
        return;
      }
      const double m = dvd(gi, fn);
      ei = sub(ei, mul(m, dn));
      fi = sub(fi, mul(m, en));
      ri = sub(ri, mul(m, rn));
      divs += 1; muls += 3; subs += 3;
      te[out(i, s)] = ei;
      tf[out(i, s)] = fi;
      tr[out(i, s)] = ri;
    }
    dn = di; en = ei; fn = fi; rn = ri;
  }
  if (ops) { ops[3 * s] = muls; ops[3 * s + 1] = subs; ops[3 * s + 2] = divs; }
  set_status(status, index, s, BX_STATUS_OK, -1);
}

// final status = reduction failure, else the Thomas solve's; x of failed
// reductions is NaN; x copied from the compact temp into the caller's layout
template <class Lay>
__global__ void pd2td_finish_kernel(const double *__restrict__ xt, double *__restrict__ x,
                                    const int32_t *rst, const int32_t *rix, const int32_t *nst,
                                    const int32_t *nix, int32_t *status, int32_t *index,
                                    int64_t batch, int64_t n, Lay tmp, Lay out) {
  const int64_t total = batch * n;
  const double nan = __longlong_as_double(0x7ff8000000000000LL);
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total;
       k += (int64_t)gridDim.x * blockDim.x) {
    // k enumerates (i, s) with s fastest for the interleaved tmp, i fastest otherwise
    int64_t i, s;
    if (tmp(1, 0) == 1) { s = k / n; i = k % n; } else { i = k / batch; s = k % batch; }
    const bool red_ok = rst[s] == BX_STATUS_OK;
    x[out(i, s)] = red_ok ? xt[tmp(i, s)] : nan;
    if (i == 0) {
      if (status) status[s] = red_ok ? nst[s] : rst[s];
      if (index) index[s] = red_ok ? nix[s] : rix[s];
    }
  }
}

static unsigned red_grid(int64_t batch) { return (unsigned)((batch + kRedThreads - 1) / kRedThreads); }

int pd2td(const double *c, const double *d, const double *e, const double *f, const double *g,
          const double *b, double *td, double *te, double *tf, double *tr, int64_t *ops,
          int32_t *st, int32_t *ix, int64_t batch, int64_t n, int64_t ld, int64_t ld_out,
          int layout, cudaStream_t stream) {
  if (layout == BX_LAYOUT_INTERLEAVED)
    pd2td_kernel<<<red_grid(batch), kRedThreads, 0, stream>>>(c, d, e, f, g, b, td, te, tf, tr, ops,
                                                              st, ix, batch, n, Interleaved{ld},
                                                              Interleaved{ld_out});
  else
    pd2td_kernel<<<red_grid(batch), kRedThreads, 0, stream>>>(c, d, e, f, g, b, td, te, tf, tr, ops,
                                                              st, ix, batch, n, SystemMajor{ld},
                                                              SystemMajor{ld_out});
  return BX_OK;
}

size_t pd2td_workspace_bytes(int64_t batch, int64_t n) {
  // reduced system (4 arrays) + NTDM scratch + x temp (compact), 4 status/index arrays
  return sizeof(double) * 6 * (size_t)batch * (size_t)n + sizeof(int32_t) * 4 * (size_t)batch + 256;
}

int pd2td_ntdm(const double *c, const double *d, const double *e, const double *f,
               const double *g, const double *b, double *x, int64_t *ops, int32_t *st,
               int32_t *ix, int64_t batch, int64_t n, int64_t ld, int layout, void *ws,
               cudaStream_t stream) {
  const size_t plane = (size_t)batch * (size_t)n;
  double *base = (double *)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
  double *td = base, *te = base + plane, *tf = base + 2 * plane, *tr = base + 3 * plane;
  double *scr = base + 4 * plane, *xt = base + 5 * plane;
  int32_t *rst = (int32_t *)(base + 6 * plane), *rix = rst + batch, *nst = rix + batch,
          *nix = nst + batch;
  const int64_t ldc = layout == BX_LAYOUT_INTERLEAVED ? batch : n;  // compact
  pd2td(c, d, e, f, g, b, td, te, tf, tr, ops, rst, rix, batch, n, ld, ldc, layout, stream);
  ntdm_seq(td, te, tf, tr, xt, scr, nst, nix, batch, n, ldc, layout, stream);
  const int64_t total = batch * n;
  const unsigned grid = (unsigned)(total / 256 + 1 < 8192 ? total / 256 + 1 : 8192);
  if (layout == BX_LAYOUT_INTERLEAVED)
    pd2td_finish_kernel<<<grid, 256, 0, stream>>>(xt, x, rst, rix, nst, nix, st, ix, batch, n,
                                                  Interleaved{ldc}, Interleaved{ld});
  else
    pd2td_finish_kernel<<<grid, 256, 0, stream>>>(xt, x, rst, rix, nst, nix, st, ix, batch, n,
                                                  SystemMajor{ldc}, SystemMajor{ld});
  return BX_OK;
}

}  // namespace bx
