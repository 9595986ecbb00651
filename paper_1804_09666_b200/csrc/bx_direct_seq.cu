// Sequential (reference-operation-order) direct solvers: NTDM, NPDM, MNPDM.
//
// One thread owns one system and walks its rows exactly in the order of the
// reference's scalar loops, with one IEEE rounding per operation (bx::mul/
// sub/dvd), so the results are bit-identical to bandix 0.1.0:
//   ntdm  : tri_factor_recip + tri_solve_recip      (_elim.py:90-122)
//   npdm  : penta_factor + penta_forward + backward (_elim.py:30-87)
//   mnpdm : mnpdm_sweep                             (_elim.py:125-190)
// The forward-substitution value y_i is produced in the same loop as the
// pivot of row i; that changes no operand of any operation, only the
// interleaving of independent ones, so bit parity is kept.
//
// Memory: intermediates of the forward sweep (reciprocal pivots / pivots and
// the U superdiagonal) go to an interleaved scratch; y is staged in x and
// overwritten by the back substitution.  Loads are software-pipelined in
// chunks of U rows so a thread keeps 4-6 x U independent loads in flight
// (the recurrence itself is latency-bound).
#include "bx_common.cuh"

namespace bx {

constexpr int kSeqThreads = 32;  // one warp per CTA: spread few systems over all SMs
constexpr int U = 8;             // rows per prefetch chunk

template <class Lay>
__device__ __forceinline__ void fill_nan(double *x, int64_t n, int64_t s, Lay lay) {
  const double nan = __longlong_as_double(0x7ff8000000000000LL);
  for (int64_t i = 0; i < n; ++i) x[lay(i, s)] = nan;
}

// ----------------------------------------------------------------------------
// NTDM
// ----------------------------------------------------------------------------
// one system (s) with its scratch column w of a Scratch{ws}: the kernel body
template <class Lay>
__device__ __forceinline__ void ntdm_one(const double *__restrict__ d, const double *__restrict__ e,
                                         const double *__restrict__ f, const double *__restrict__ b,
                                         double *__restrict__ x, double *__restrict__ recw,
                                         int32_t *status, int32_t *index, int64_t n, Lay lay,
                                         int64_t s, const Scratch ws, int64_t w) {

  // ---- factor + forward substitution (rows 0..n-1) ----
  double cd[U], ce[U], cf[U], cb[U];   // current chunk: d_i, e_i, f_{i-1}, b_i
  double nd[U], ne[U], nf[U], nb[U];   // next chunk
  auto load = [&](int64_t base, double *D, double *E, double *F, double *Bv) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u;
      if (i < n) {
        D[u] = i >= 1 ? ldg(d + lay(i, s)) : 0.0;
        E[u] = ldg(e + lay(i, s));
        F[u] = i >= 1 ? ldg(f + lay(i - 1, s)) : 0.0;
        Bv[u] = ldg(b + lay(i, s));
      }
    }
  };
  load(0, cd, ce, cf, cb);
  double rprev = 0.0, yprev = 0.0;
  for (int64_t base = 0; base < n; base += U) {
    if (base + U < n) load(base + U, nd, ne, nf, nb);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u;
      if (i < n) {
        double mi, yi;
        if (i == 0) {
          mi = ce[u];                                   // _elim.py:101
          yi = cb[u];                                   // _elim.py:116
        } else {
          const double li = mul(cd[u], rprev);          // _elim.py:104
          mi = sub(ce[u], mul(li, cf[u]));              // _elim.py:105
          yi = sub(cb[u], mul(li, yprev));              // _elim.py:117
        }
        if (mi == 0.0) {                                // ZeroPivot(i), _elim.py:26-27
          set_status(status, index, s, BX_STATUS_ZERO_PIVOT, (int32_t)i);
          fill_nan(x, n, s, lay);
          return;
        }
        rprev = dvd(1.0, mi);                           // _elim.py:108
        yprev = yi;
        recw[ws(i, w)] = rprev;
        x[lay(i, s)] = yi;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) { cd[u] = nd[u]; ce[u] = ne[u]; cf[u] = nf[u]; cb[u] = nb[u]; }
  }

  // ---- back substitution (rows n-1..0), _elim.py:118-121 ----
  double xnext = mul(yprev, rprev);
  x[lay(n - 1, s)] = xnext;
  double cy[U], cr[U], cc[U], ny[U], nr[U], nc[U];
  auto loadb = [&](int64_t top, double *Y, double *R, double *C) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = top - u;
      if (i >= 0) {
        Y[u] = x[lay(i, s)];
        R[u] = recw[ws(i, w)];
        C[u] = ldg(f + lay(i, s));
      }
    }
  };
  loadb(n - 2, cy, cr, cc);
  for (int64_t top = n - 2; top >= 0; top -= U) {
    if (top - U >= 0) loadb(top - U, ny, nr, nc);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = top - u;
      if (i >= 0) {
        xnext = mul(sub(cy[u], mul(cc[u], xnext)), cr[u]);
        x[lay(i, s)] = xnext;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) { cy[u] = ny[u]; cr[u] = nr[u]; cc[u] = nc[u]; }
  }
  set_status(status, index, s, BX_STATUS_OK, -1);
}

// flags == nullptr: one thread per system, scratch column = system.
// flags != nullptr (re-solve of systems a partitioned kernel flagged): `slots`
// one-warp CTAs walk the batch 32 systems at a time; a flagged system is
// solved by its lane with the CTA's scratch column (Scratch{slots}); every
// other system gets status OK / -1.
__device__ __forceinline__ bool flagged(const int32_t *flags, int64_t s, int fs) {
  bool f = false;
  for (int r = 0; r < fs; ++r) f |= flags[s * fs + r] != 0;
  return f;
}

template <class Lay>
__global__ void __launch_bounds__(kSeqThreads)
ntdm_seq_kernel(const double *__restrict__ d, const double *__restrict__ e,
                const double *__restrict__ f, const double *__restrict__ b,
                double *__restrict__ x, double *__restrict__ recw, int32_t *status,
                int32_t *index, int64_t batch, int64_t n, Lay lay, const int32_t *flags,
                int64_t slots, int fs) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (!flags) {
    if (t < batch) ntdm_one(d, e, f, b, x, recw, status, index, n, lay, t, Scratch{batch}, t);
    return;
  }
  // re-solve mode: one warp per scratch slot (CTA), lanes check 32 systems'
  // flags at a time; flagged ones are solved one after another by their lane.
  // Launched with programmatic stream serialization: resident early, held
  // here until the partitioned kernels before it have completed.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int slot = blockIdx.x, lane = threadIdx.x;
  for (int64_t s0 = (int64_t)slot * 32; s0 < batch; s0 += slots * 32) {
    const int64_t s = s0 + lane;
    const bool fl = s < batch && flagged(flags, s, fs);
    if (s < batch && !fl) set_status(status, index, s, BX_STATUS_OK, -1);
    unsigned todo = __ballot_sync(0xffffffffu, fl);
    while (todo) {
      const int l = __ffs(todo) - 1;
      todo &= todo - 1;
      if (lane == l) ntdm_one(d, e, f, b, x, recw, status, index, n, lay, s, Scratch{slots}, slot);
      __syncwarp();
    }
  }
}

// ----------------------------------------------------------------------------
// NPDM (and MNPDM: kMod = true)
// ----------------------------------------------------------------------------
// Forward sweep state (row-aligned names of _elim.py): piv = mu (NPDM) or
// rec = 1/mu (MNPDM); phi = U(i,i+1); psi = U(i,i+2) = sup2[i].
template <bool kMod, class Lay>
__device__ __forceinline__ void penta_one(const double *__restrict__ c, const double *__restrict__ d,
                                          const double *__restrict__ e, const double *__restrict__ f,
                                          const double *__restrict__ g, const double *__restrict__ b,
                                          double *__restrict__ x, double *__restrict__ pivw,
                                          double *__restrict__ phiw, int32_t *status,
                                          int32_t *index, int64_t *nz_out, int64_t n, Lay lay,
                                          int64_t s, const Scratch ws, int64_t w) {

  double cc[U], cd[U], ce[U], cf[U], cg[U], cb[U];
  double nc[U], nd[U], ne[U], nf[U], ng[U], nb[U];
  // row i needs c_i, d_i, e_i, f_i, b_i and psi_{i-1} = g_{i-1}, psi_{i-2} = g_{i-2}
  // (carried in registers); g_i is loaded for i <= n-3.
  auto load = [&](int64_t base, double *C, double *D, double *E, double *F, double *G,
                  double *Bv) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u;
      if (i < n) {
        C[u] = i >= 2 ? ldg(c + lay(i, s)) : 0.0;
        D[u] = i >= 1 ? ldg(d + lay(i, s)) : 0.0;
        E[u] = ldg(e + lay(i, s));
        F[u] = i <= n - 2 ? ldg(f + lay(i, s)) : 0.0;
        G[u] = i <= n - 3 ? ldg(g + lay(i, s)) : 0.0;
        Bv[u] = ldg(b + lay(i, s));
      }
    }
  };
  load(0, cc, cd, ce, cf, cg, cb);
  // carried state: pivot (mu or rec), phi, psi, y for rows i-1 and i-2
  double p1 = 0.0, p2 = 0.0, ph1 = 0.0, ph2 = 0.0, ps1 = 0.0, ps2 = 0.0, y1 = 0.0, y2 = 0.0;
  int64_t nz = 0;
  for (int64_t base = 0; base < n; base += U) {
    if (base + U < n) load(base + U, nc, nd, ne, nf, ng, nb);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u;
      if (i < n) {
        double mi, phi, yi;
        if (i == 0) {
          mi = ce[u];                                            // _elim.py:44 / 146
          phi = cf[u];
          yi = cb[u];
        } else if (i == 1) {
          // NPDM: l1 = d/mu0 (_elim.py:47); MNPDM: l1 = d*rec0 (_elim.py:150)
          const double l1 = kMod ? mul(cd[u], p1) : dvd(cd[u], p1);
          mi = sub(ce[u], mul(l1, ph1));
          phi = sub(cf[u], mul(l1, ps1));                        // _elim.py:50 / 155
          yi = sub(cb[u], mul(l1, y1));                          // _elim.py:69 / 179
        } else if (!kMod) {
          const double l2 = dvd(cc[u], p2);                      // _elim.py:54
          const double l1 = dvd(sub(cd[u], mul(l2, ph2)), p1);   // _elim.py:55
          mi = sub(sub(ce[u], mul(l2, ps2)), mul(l1, ph1));      // _elim.py:56
          phi = i <= n - 2 ? sub(cf[u], mul(l1, ps1)) : 0.0;     // _elim.py:60
          yi = sub(sub(cb[u], mul(l1, y1)), mul(l2, y2));        // _elim.py:72
        } else {
          const bool has2 = cc[u] != 0.0;                        // _elim.py:160-167
          nz += has2;
          const double l2 = mul(cc[u], p2);
          const double t = has2 ? sub(cd[u], mul(l2, ph2)) : cd[u];
          const double l1 = mul(t, p1);
          double m = sub(ce[u], mul(l1, ph1));                   // _elim.py:169
          if (has2) m = sub(m, mul(l2, ps2));                    // _elim.py:170-171
          mi = m;
          phi = i <= n - 2 ? sub(cf[u], mul(l1, ps1)) : 0.0;     // _elim.py:174
          double yv = sub(cb[u], mul(l1, y1));                   // _elim.py:181
          if (has2) yv = sub(yv, mul(l2, y2));                   // _elim.py:182-183
          yi = yv;
        }
        if (mi == 0.0) {
          set_status(status, index, s, BX_STATUS_ZERO_PIVOT, (int32_t)i);
          if (nz_out) nz_out[s] = nz;
          fill_nan(x, n, s, lay);
          return;
        }
        const double piv = kMod ? dvd(1.0, mi) : mi;             // rec (MNPDM) or mu
        pivw[ws(i, w)] = piv;
        phiw[ws(i, w)] = phi;
        x[lay(i, s)] = yi;
        p2 = p1; p1 = piv;
        ph2 = ph1; ph1 = phi;
        ps2 = ps1; ps1 = cg[u];
        y2 = y1; y1 = yi;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      cc[u] = nc[u]; cd[u] = nd[u]; ce[u] = ne[u]; cf[u] = nf[u]; cg[u] = ng[u]; cb[u] = nb[u];
    }
  }
  if (nz_out) nz_out[s] = nz;

  // ---- back substitution, _elim.py:83-86 (NPDM) / 185-189 (MNPDM) ----
  // x_{n-1} = y/mu ; x_{n-2} = (y - phi x_{n-1})/mu ; x_i = ((y - phi x1) - psi x2)/mu
  auto fin = [&](double num, double piv) { return kMod ? mul(num, piv) : dvd(num, piv); };
  double x1 = fin(y1, p1);
  x[lay(n - 1, s)] = x1;
  double x2 = x1;
  x1 = fin(sub(y2, mul(ph2, x1)), p2);
  x[lay(n - 2, s)] = x1;
  double cy[U], cp[U], cph[U], cps[U], ny[U], np_[U], nph[U], nps[U];
  auto loadb = [&](int64_t top, double *Y, double *P, double *PH, double *PS) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = top - u;
      if (i >= 0) {
        Y[u] = x[lay(i, s)];
        P[u] = pivw[ws(i, w)];
        PH[u] = phiw[ws(i, w)];
        PS[u] = ldg(g + lay(i, s));
      }
    }
  };
  if (n >= 3) loadb(n - 3, cy, cp, cph, cps);
  for (int64_t top = n - 3; top >= 0; top -= U) {
    if (top - U >= 0) loadb(top - U, ny, np_, nph, nps);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = top - u;
      if (i >= 0) {
        const double xi = fin(sub(sub(cy[u], mul(cph[u], x1)), mul(cps[u], x2)), cp[u]);
        x[lay(i, s)] = xi;
        x2 = x1; x1 = xi;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) { cy[u] = ny[u]; cp[u] = np_[u]; cph[u] = nph[u]; cps[u] = nps[u]; }
  }
  set_status(status, index, s, BX_STATUS_OK, -1);
}

template <bool kMod, class Lay>
__global__ void __launch_bounds__(kSeqThreads)
penta_seq_kernel(const double *__restrict__ c, const double *__restrict__ d,
                 const double *__restrict__ e, const double *__restrict__ f,
                 const double *__restrict__ g, const double *__restrict__ b,
                 double *__restrict__ x, double *__restrict__ pivw, double *__restrict__ phiw,
                 int32_t *status, int32_t *index, int64_t *nz_out, int64_t batch, int64_t n,
                 Lay lay, const int32_t *flags, int64_t slots, int fs, const int32_t *nzpart) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (!flags) {
    if (t < batch)
      penta_one<kMod>(c, d, e, f, g, b, x, pivw, phiw, status, index, nz_out, n, lay, t,
                      Scratch{batch}, t);
    return;
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");  // (see ntdm_seq_kernel)
  const int slot = blockIdx.x, lane = threadIdx.x;
  for (int64_t s0 = (int64_t)slot * 32; s0 < batch; s0 += slots * 32) {
    const int64_t s = s0 + lane;
    const bool fl = s < batch && flagged(flags, s, fs);
    if (s < batch && !fl) {
      set_status(status, index, s, BX_STATUS_OK, -1);
      if (nz_out && nzpart) {
        int64_t nz = 0;
        for (int r = 0; r < fs; ++r) nz += nzpart[s * fs + r];
        nz_out[s] = nz;
      }
    }
    unsigned todo = __ballot_sync(0xffffffffu, fl);
    while (todo) {
      const int l = __ffs(todo) - 1;
      todo &= todo - 1;
      if (lane == l)
        penta_one<kMod>(c, d, e, f, g, b, x, pivw, phiw, status, index, nz_out, n, lay, s,
                        Scratch{slots}, slot);
      __syncwarp();
    }
  }
}

// ----------------------------------------------------------------------------
// report residual ||b - A x||_inf, row-fused order of core.penta_matvec /
// tri_matvec (core.py:249-256, 279-284) then residual/inf_norm (303-321)
// ----------------------------------------------------------------------------
template <class Lay>
__global__ void __launch_bounds__(kSeqThreads)
residual_inf_kernel(int bw, const double *__restrict__ c, const double *__restrict__ d,
                    const double *__restrict__ e, const double *__restrict__ f,
                    const double *__restrict__ g, const double *__restrict__ x,
                    const double *__restrict__ b, double *__restrict__ out, int64_t batch,
                    int64_t n, Lay lay) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= batch) return;
  double xm2 = 0.0, xm1 = 0.0;
  double x0 = ldg(x + lay(0, s));
  double xp1 = n > 1 ? ldg(x + lay(1, s)) : 0.0;
  double xp2 = n > 2 ? ldg(x + lay(2, s)) : 0.0;
  double best = 0.0;
  bool has_nan = false;
  for (int64_t i = 0; i < n; ++i) {
    double acc = mul(ldg(e + lay(i, s)), x0);
    if (i >= 1) acc = add(acc, mul(ldg(d + lay(i, s)), xm1));
    if (i <= n - 2) acc = add(acc, mul(ldg(f + lay(i, s)), xp1));
    if (bw == 2) {
      if (i >= 2) acc = add(acc, mul(ldg(c + lay(i, s)), xm2));
      if (i <= n - 3) acc = add(acc, mul(ldg(g + lay(i, s)), xp2));
    }
    const double r = fabs(sub(ldg(b + lay(i, s)), acc));
    has_nan |= (r != r);
    best = r > best ? r : best;
    xm2 = xm1; xm1 = x0; x0 = xp1; xp1 = xp2;
    xp2 = (i + 3 < n) ? ldg(x + lay(i + 3, s)) : 0.0;
  }
  out[s] = has_nan ? __longlong_as_double(0x7ff8000000000000LL) : best;
}

// ----------------------------------------------------------------------------
// host launchers
// ----------------------------------------------------------------------------
static inline dim3 seq_grid(int64_t batch) {
  return dim3((unsigned)((batch + kSeqThreads - 1) / kSeqThreads));
}

template <class Lay>
static void launch_ntdm(const double *d, const double *e, const double *f, const double *b,
                        double *x, double *ws, int32_t *st, int32_t *ix, int64_t batch,
                        int64_t n, Lay lay, cudaStream_t stream) {
  ntdm_seq_kernel<Lay><<<seq_grid(batch), kSeqThreads, 0, stream>>>(d, e, f, b, x, ws, st, ix,
                                                                     batch, n, lay, nullptr, 0, 1);
}

template <bool kMod, class Lay>
static void launch_penta(const double *c, const double *d, const double *e, const double *f,
                         const double *g, const double *b, double *x, double *ws, int32_t *st,
                         int32_t *ix, int64_t *nz, int64_t batch, int64_t n, Lay lay,
                         cudaStream_t stream) {
  penta_seq_kernel<kMod, Lay><<<seq_grid(batch), kSeqThreads, 0, stream>>>(
      c, d, e, f, g, b, x, ws, ws + batch * n, st, ix, nz, batch, n, lay, nullptr, 0, 1, nullptr);
}

void ntdm_seq(const double *d, const double *e, const double *f, const double *b, double *x,
              double *ws, int32_t *st, int32_t *ix, int64_t batch, int64_t n, int64_t ld,
              int layout, cudaStream_t stream) {
  if (layout == BX_LAYOUT_INTERLEAVED)
    launch_ntdm(d, e, f, b, x, ws, st, ix, batch, n, Interleaved{ld}, stream);
  else
    launch_ntdm(d, e, f, b, x, ws, st, ix, batch, n, SystemMajor{ld}, stream);
}

void penta_seq(bool mod, const double *c, const double *d, const double *e, const double *f,
               const double *g, const double *b, double *x, double *ws, int32_t *st,
               int32_t *ix, int64_t *nz, int64_t batch, int64_t n, int64_t ld, int layout,
               cudaStream_t stream) {
  if (layout == BX_LAYOUT_INTERLEAVED) {
    if (mod) launch_penta<true>(c, d, e, f, g, b, x, ws, st, ix, nz, batch, n, Interleaved{ld}, stream);
    else launch_penta<false>(c, d, e, f, g, b, x, ws, st, ix, nz, batch, n, Interleaved{ld}, stream);
  } else {
    if (mod) launch_penta<true>(c, d, e, f, g, b, x, ws, st, ix, nz, batch, n, SystemMajor{ld}, stream);
    else launch_penta<false>(c, d, e, f, g, b, x, ws, st, ix, nz, batch, n, SystemMajor{ld}, stream);
  }
}

// Re-solve, in the reference's operation order, the systems a partitioned
// kernel flagged (flags[s] != 0), and write status / index of every system
// (OK / -1 for the unflagged ones).  Scratch: fixup_scratch_doubles(...).
constexpr int64_t kFixSlots = 128;
size_t fixup_scratch_doubles(int kind, int64_t n) { return (size_t)(kind == 0 ? 1 : 2) * kFixSlots * n; }

// launch on `stream` with programmatic stream serialization (the kernel
// calls griddepcontrol.wait before it touches its predecessors' results)
template <class... KA, class... A>
static void launch_dependent(void (*kern)(KA...), dim3 grid, dim3 block, cudaStream_t stream,
                             A... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, static_cast<KA>(args)...);
}

void direct_fixup(int kind, const double *c, const double *d, const double *e, const double *f,
                  const double *g, const double *b, double *x, double *scratch,
                  const int32_t *flags, int fs, const int32_t *nzpart, int32_t *st, int32_t *ix,
                  int64_t *nz, int64_t batch, int64_t n, int64_t ld, int layout,
                  cudaStream_t stream) {
  const dim3 grid((unsigned)kFixSlots), block(kSeqThreads);  // one warp per scratch slot
  if (kind == 0) {
    if (layout == BX_LAYOUT_INTERLEAVED)
      launch_dependent(ntdm_seq_kernel<Interleaved>, grid, block, stream, d, e, f, b, x, scratch, st,
                       ix, batch, n, Interleaved{ld}, flags, kFixSlots, fs);
    else
      launch_dependent(ntdm_seq_kernel<SystemMajor>, grid, block, stream, d, e, f, b, x, scratch, st,
                       ix, batch, n, SystemMajor{ld}, flags, kFixSlots, fs);
    return;
  }
  double *phiw = scratch + kFixSlots * n;
  if (layout == BX_LAYOUT_INTERLEAVED) {
    if (kind == 2)
      launch_dependent(penta_seq_kernel<true, Interleaved>, grid, block, stream, c, d, e, f, g, b, x,
                       scratch, phiw, st, ix, nz, batch, n, Interleaved{ld}, flags, kFixSlots, fs, nzpart);
    else
      launch_dependent(penta_seq_kernel<false, Interleaved>, grid, block, stream, c, d, e, f, g, b, x,
                       scratch, phiw, st, ix, nz, batch, n, Interleaved{ld}, flags, kFixSlots, fs, nzpart);
  } else {
    if (kind == 2)
      launch_dependent(penta_seq_kernel<true, SystemMajor>, grid, block, stream, c, d, e, f, g, b, x,
                       scratch, phiw, st, ix, nz, batch, n, SystemMajor{ld}, flags, kFixSlots, fs, nzpart);
    else
      launch_dependent(penta_seq_kernel<false, SystemMajor>, grid, block, stream, c, d, e, f, g, b, x,
                       scratch, phiw, st, ix, nz, batch, n, SystemMajor{ld}, flags, kFixSlots, fs, nzpart);
  }
}

void residual_inf(int bw, const double *c, const double *d, const double *e, const double *f,
                  const double *g, const double *x, const double *b, double *out, int64_t batch,
                  int64_t n, int64_t ld, int layout, cudaStream_t stream) {
  if (layout == BX_LAYOUT_INTERLEAVED)
    residual_inf_kernel<<<seq_grid(batch), kSeqThreads, 0, stream>>>(bw, c, d, e, f, g, x, b, out,
                                                                     batch, n, Interleaved{ld});
  else
    residual_inf_kernel<<<seq_grid(batch), kSeqThreads, 0, stream>>>(bw, c, d, e, f, g, x, b, out,
                                                                     batch, n, SystemMajor{ld});
}

}  // namespace bx
