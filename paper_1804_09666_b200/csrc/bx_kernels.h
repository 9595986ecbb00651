// Internal launcher declarations shared by the .cu translation units.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <vector>

namespace bx {

// bx_direct_seq.cu
void ntdm_seq(const double *d, const double *e, const double *f, const double *b, double *x,
              double *ws, int32_t *st, int32_t *ix, int64_t batch, int64_t n, int64_t ld,
              int layout, cudaStream_t stream);
void penta_seq(bool mod, const double *c, const double *d, const double *e, const double *f,
               const double *g, const double *b, double *x, double *ws, int32_t *st,
               int32_t *ix, int64_t *nz, int64_t batch, int64_t n, int64_t ld, int layout,
               cudaStream_t stream);
size_t fixup_scratch_doubles(int kind, int64_t n);  // kind 0 NTDM, 1 NPDM, 2 MNPDM
// flags[s*fs + r] != 0 for some r < fs: system s is re-solved in the
// reference order; otherwise status OK / -1 and (nzpart) nz = sum of parts
void direct_fixup(int kind, const double *c, const double *d, const double *e, const double *f,
                  const double *g, const double *b, double *x, double *scratch,
                  const int32_t *flags, int fs, const int32_t *nzpart, int32_t *st, int32_t *ix,
                  int64_t *nz, int64_t batch, int64_t n, int64_t ld, int layout,
                  cudaStream_t stream);
void residual_inf(int bw, const double *c, const double *d, const double *e, const double *f,
                  const double *g, const double *x, const double *b, double *out, int64_t batch,
                  int64_t n, int64_t ld, int layout, cudaStream_t stream);

// bx_direct_seg.cu (system-major, n <= 32768: the default partitioned path);
// flags / nzpart: [batch][*csize] per segment
bool seg_applicable(const double *const *ptrs, int nptr, int64_t n, int64_t ld, int layout);
int seg_solve(int K, const double *c2, const double *c1, const double *e, const double *f1,
              const double *f2, const double *b, double *x, int32_t *flags, int32_t *nzpart,
              int64_t batch, int64_t n, int64_t ld, cudaStream_t stream, int *csize);

// bx_direct_halo.cu: interface-iteration first pass of the partitioned path.
// flags / retry / nzpart: [batch][*csize] int32 words (one per CTA of a
// system's cluster).  Systems whose interface coupling is too strong for the
// fixed sweep count get a nonzero retry word and are solved again by the
// two-port tree kernel (bx_direct_part.cu)
bool halo_enabled();
int halo_solve(int K, const double *c2, const double *c1, const double *e, const double *f1,
               const double *f2, const double *b, double *x, int32_t *flags, int32_t *retry,
               int32_t *nzpart, int64_t batch, int64_t n, int64_t ld, int layout,
               cudaStream_t stream, const int32_t *outer_rows, const double *outer_sub2,
               const double *outer_sup2, int64_t outer_k, int *csize, int32_t *index = nullptr,
               int64_t *nz = nullptr);

// bx_band_ops.cu (reference order, bit-exact building blocks)
void band_matvec(int bw, int64_t m, const double *c, const double *d, const double *e,
                 const double *f, const double *g, const double *x, const double *b, double *y,
                 int64_t batch, int64_t n, int64_t ld, int layout, cudaStream_t stream);
void lu_penta(const double *c, const double *d, const double *e, const double *f, const double *g,
              double *mu, double *l1, double *l2, double *phi, double *psi, int32_t *st,
              int32_t *ix, int64_t batch, int64_t n, int64_t ld, int layout, cudaStream_t stream);
void forward_sub(int64_t m, const double *l1, const double *lm, const double *b, double *y,
                 int64_t batch, int64_t n, int64_t ld, int layout, cudaStream_t stream);
void backward_sub(int64_t m, const double *mu, const double *phi, const double *psi, const double *y,
                  double *x, int32_t *st, int32_t *ix, int64_t batch, int64_t n, int64_t ld,
                  int layout, cudaStream_t stream);

// bx_direct_part.cu
size_t part_workspace_bytes(int bandwidth, int64_t batch, int64_t n);
int outer_compact(const double *sub2, const double *sup2, int32_t *count, int32_t *rows,
                  double *vsub2, double *vsup2, int64_t cap, int64_t batch, int64_t n, int64_t ld,
                  int layout, cudaStream_t stream);
int mnpdm_sparse_part(const int32_t *rows, const double *vsub2, const double *vsup2, int64_t k,
                      const double *d, const double *e, const double *f, const double *b,
                      double *x, int32_t *st, int32_t *ix, int64_t *nz, int64_t batch, int64_t n,
                      int64_t ld, int layout, cudaStream_t stream);
// pd_to_td / solve_pd2td_ntdm (bx_pd2td.cu)
int pd2td(const double *c, const double *d, const double *e, const double *f, const double *g,
          const double *b, double *td, double *te, double *tf, double *tr, int64_t *ops,
          int32_t *st, int32_t *ix, int64_t batch, int64_t n, int64_t ld, int64_t ld_out,
          int layout, cudaStream_t stream);
size_t pd2td_workspace_bytes(int64_t batch, int64_t n);
int pd2td_ntdm(const double *c, const double *d, const double *e, const double *f,
               const double *g, const double *b, double *x, int64_t *ops, int32_t *st,
               int32_t *ix, int64_t batch, int64_t n, int64_t ld, int layout, void *ws,
               cudaStream_t stream);
int ntdm_part(const double *d, const double *e, const double *f, const double *b, double *x,
              double *ws, int32_t *st, int32_t *ix, int64_t batch, int64_t n, int64_t ld,
              int layout, cudaStream_t stream);
int penta_part(bool mod, const double *c, const double *d, const double *e, const double *f,
               const double *g, const double *b, double *x, double *ws, int32_t *st,
               int32_t *ix, int64_t *nz, int64_t batch, int64_t n, int64_t ld, int layout,
               cudaStream_t stream);

// bx_sip.cu
size_t sip_workspace_bytes(int64_t batch, int64_t n);
int sip_seq(const double *a2, const double *a1, const double *e, const double *c1,
            const double *c2, const double *b, const double *tol, double *x, double *best_x,
            int64_t *iters, double *res, double *best_res, int32_t *st, int32_t *ix,
            double *hist, double *ws, int64_t batch, int64_t n, int64_t m, double alpha,
            int64_t max_iter, int use_x0, int64_t ld, int layout, int factor_only,
            cudaStream_t stream);
int sip_export(double *ws, int64_t batch, int64_t n, double *const *outs12, int64_t ld,
               int layout, cudaStream_t stream);

// bx_sip_wave.cu
size_t sip_wave_workspace_bytes(int64_t batch, int64_t n, int64_t m);
bool sip_is_grid(const double *a1, const double *c1, int64_t batch, int64_t n, int64_t m,
                 int64_t ld, int layout, void *scratch, cudaStream_t stream);
int sip_wave(const double *a2, const double *a1, const double *e, const double *c1,
             const double *c2, const double *b, const double *tol, double *x, double *best_x,
             int64_t *iters, double *res, double *best_res, int32_t *st, int32_t *ix,
             double *hist, double *ws, int64_t batch, int64_t n, int64_t m, double alpha,
             int64_t max_iter, int use_x0, int64_t ld, int layout, cudaStream_t stream, double *nat = nullptr,
             int32_t *setup_ok = nullptr);

// bx_sip_scan.cu (BX_ALGO_SCAN: row-scan sweeps in correction form, tolerance parity)
bool sip_scan_applicable(int64_t n, int64_t m);
size_t sip_scan_workspace_bytes(int64_t batch, int64_t n, int64_t m);
int sip_scan(const double *a2, const double *a1, const double *e, const double *c1,
             const double *c2, const double *b, const double *tol, double *x, double *best_x,
             int64_t *iters, double *res, double *best_res, int32_t *st, int32_t *ix,
             double *hist, double *ws, int64_t batch, int64_t n, int64_t m, double alpha,
             int64_t max_iter, int use_x0, int64_t ld, int layout, cudaStream_t stream);

// bx_exact.cu (kind 1 = STDM, 2 = SPDM)
size_t exact_workspace_bytes(int kind, int64_t batch, int64_t n);
int exact_solve(int kind, const double *c, const double *d, const double *e, const double *f,
                const double *g, const double *b, double *x, int32_t *st, int32_t *ix,
                int32_t *subs, double *ws, int64_t batch, int64_t n, int64_t ld, int layout,
                cudaStream_t stream);

int det_band(int kind, const double *c, const double *d, const double *e, const double *f,
             const double *g, double *mant, int64_t *expo, int32_t *st, int32_t *ix,
             int32_t *subs, int64_t batch, int64_t n, int64_t ld, int layout,
             cudaStream_t stream);

// bx_rcond.cu (kind 1 = tridiagonal, 2 = pentadiagonal)
size_t rcond_workspace_bytes(int kind, int64_t batch, int64_t n);
int rcond_band(int kind, const double *c, const double *d, const double *e, const double *f,
               const double *g, double *rcond, int32_t *st, int32_t *ix, double *ws,
               int64_t batch, int64_t n, int64_t ld, int layout, cudaStream_t stream);

// bx_hb.cu / bx_hb_host.cu
size_t hb_dense_bytes(int64_t batch, int64_t n);
int64_t hb_padded(int64_t n);
int hb_gemm(double *Xa, double *Xb, const int *parity, const double *P, const int *active_list,
            int nactive, int64_t n, int64_t batch, cudaStream_t stream);
int hb_residual(const double *Xa, const double *Xb, const int *parity, double *P, const double *l1,
                const double *l2, const double *mu, const double *phi, const double *psi,
                const int *active_list, int nactive, unsigned long long *rbits, int64_t n,
                int64_t m, int64_t batch, cudaStream_t stream);
int hb_init(double *X, const double *mu, int64_t n, int64_t batch, int32_t *zero_diag,
            cudaStream_t stream);
int hb_apply(const double *Xa, const double *Xb, const int *parity, const double *v, double *y,
             const int *act, int nact, int64_t n, int64_t batch, int upper, cudaStream_t stream);
size_t hb_total_workspace_bytes(int64_t batch, int64_t n);
int sip_hb(const double *a2, const double *a1, const double *e, const double *c1,
           const double *c2, const double *b, const double *tol, double *x, double *best_x,
           int64_t *iterations, double *residual, double *best_residual, int32_t *status,
           int32_t *index, double *history, int64_t *inv_iterations, double *inv_residual,
           int64_t batch, int64_t n, int64_t m, double alpha, int64_t max_iter,
           int64_t max_inv_iter, int use_x0, int64_t ld, int layout, void *workspace,
           cudaStream_t st, bool invert_only, double *xl, double *xu);

// bx_hb_dense.cu (hb_invert_dense on a caller's dense matrices)
size_t hb_dense_invert_workspace_bytes(int64_t batch, int64_t n);
int hb_dense_invert(const double *M, int64_t n, int64_t ldm, int64_t mstride, int64_t batch,
                    const double *tol, int64_t max_iter, double *X, int64_t ldx, int64_t xstride,
                    int64_t *iterations, double *residual, double *history, int32_t *status,
                    int32_t *index, void *ws, cudaStream_t st);

// bx_hb_band.cu (banded HB, inverse.py:122-195)
size_t hb_band_bytes(int64_t batch, int64_t n, int64_t cap);
int hb_band_invert_round(const double *fac, double *X, double *Xn, double *P, double *Best,
                         int *dact, int *dzero, unsigned long long *rbits,
                         const std::vector<int> &act0, const double *tol_f, int64_t batch,
                         int64_t n, int64_t cap, int64_t w, int64_t max_iter, int64_t *iters,
                         double *resid, int *status, int *zero_row,
                         std::vector<std::vector<double>> *hist, cudaStream_t st);
int hb_band_true_residual(const double *fac, const double *X, int *dact, unsigned long long *rbits,
                          const std::vector<int> &act, int64_t batch, int64_t n, int64_t cap,
                          int64_t w, double *out, cudaStream_t st);
int hb_band_apply(const double *X, const int64_t *wf, const double *v, double *out, const int *act,
                  int nact, int64_t batch, int64_t n, int64_t cap, int upper, cudaStream_t st);
int hb_band_factor_planes(const double *mu, const double *l1, const double *l2, const double *phi,
                          const double *psi, double *fac, int64_t batch, int64_t n, int64_t ld,
                          int layout, cudaStream_t st);
int hb_band_invert(const double *mu, const double *l1, const double *l2, const double *phi,
                   const double *psi, int side, int64_t w, const double *tol, int64_t max_iter,
                   double *xdiags, int64_t *iterations, double *residual, double *history,
                   int32_t *status, int32_t *index, int64_t batch, int64_t n, int64_t ld,
                   int layout, void *workspace, cudaStream_t st);
size_t hb_band_invert_workspace_bytes(int64_t batch, int64_t n, int64_t w);
size_t sip_hb_band_workspace_bytes(int64_t batch, int64_t n, int64_t cap);
int sip_hb_band(const double *a2, const double *a1, const double *e, const double *c1,
                const double *c2, const double *b, const double *tol, double *x, double *best_x,
                int64_t *iterations, double *residual, double *best_residual, int32_t *status,
                int32_t *index, double *history, int64_t w, int64_t cap, int64_t *w_used,
                int64_t *inv_iterations, double *inv_residual, double *inv_true_residual,
                int64_t batch, int64_t n, int64_t max_iter, int64_t max_inv_iter, int use_x0,
                int64_t ld, int layout, void *workspace, cudaStream_t st);

// bx_layout.cu
int transpose(const double *src, double *dst, int64_t rows, int64_t cols, int64_t lds,
              int64_t ldd, int64_t nbatch, int64_t bss, int64_t bsd, cudaStream_t stream);

// workspace of the non-direct solvers (bx_api.cu dispatch)
size_t other_workspace_bytes(int solver, int64_t batch, int64_t n);

}  // namespace bx
