// extern "C" entry points of libbandix_b200.so (declared in include/bandix_b200.h).
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include "bx_common.cuh"
#include "bx_kernels.h"

namespace bxh {
static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
}

int check_launch(const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return BX_ERR_CUDA;
  }
  return BX_OK;
}
}  // namespace bxh

using bxh::set_error;

static int check_common(const char *fn, int64_t batch, int64_t n, int64_t nmin, int64_t ld,
                        int32_t layout) {
  if (batch < 0) { set_error("%s: batch must be >= 0", fn); return BX_ERR_ARG; }
  if (n < nmin) { set_error("%s: n=%lld below the minimum %lld", fn, (long long)n, (long long)nmin); return BX_ERR_ARG; }
  if (layout == BX_LAYOUT_INTERLEAVED) {
    if (ld < batch) { set_error("%s: interleaved ld=%lld < batch=%lld", fn, (long long)ld, (long long)batch); return BX_ERR_ARG; }
  } else if (layout == BX_LAYOUT_SYSTEM_MAJOR) {
    if (ld < n) { set_error("%s: system-major ld=%lld < n=%lld", fn, (long long)ld, (long long)n); return BX_ERR_ARG; }
  } else {
    set_error("%s: unknown layout %d", fn, layout);
    return BX_ERR_ARG;
  }
  return BX_OK;
}

#define BX_REQUIRE(cond, ...)            \
  do {                                   \
    if (!(cond)) {                       \
      set_error(__VA_ARGS__);            \
      return BX_ERR_ARG;                 \
    }                                    \
  } while (0)

extern "C" {

/* Workspace of the SIP solver for a given stride (the wavefront planes depend
 * on m); max of the sequential and wavefront requirements. */
size_t bx_sip_workspace_bytes(int64_t batch, int64_t n, int64_t m) {
  const size_t a = bx::sip_workspace_bytes(batch, n), b = bx::sip_wave_workspace_bytes(batch, n, m);
  const size_t c = bx::sip_scan_workspace_bytes(batch, n, m);
  return a > b ? (a > c ? a : c) : (b > c ? b : c);
}

const char *bx_version(void) { return "bandix_b200 0.1.0 (sm_100a)"; }
const char *bx_last_error(void) { return bxh::g_err; }

size_t bx_workspace_bytes(int32_t solver, int64_t batch, int64_t n, int32_t layout, int32_t algo) {
  (void)layout;
  const size_t rows = (size_t)batch * (size_t)n * sizeof(double);
  switch (solver) {
    case BX_SOLVER_NTDM:
      return algo == BX_ALGO_SEQUENTIAL ? rows : bx::part_workspace_bytes(1, batch, n);
    case BX_SOLVER_NPDM:
    case BX_SOLVER_MNPDM:
      return algo == BX_ALGO_SEQUENTIAL ? 2 * rows : bx::part_workspace_bytes(2, batch, n);
    case BX_SOLVER_SIP:
      return algo == BX_ALGO_SEQUENTIAL ? bx::sip_workspace_bytes(batch, n) : 0;
    case BX_SOLVER_PD2TD:
      return bx::pd2td_workspace_bytes(batch, n);
    default:
      return bx::other_workspace_bytes(solver, batch, n);
  }
}

int bx_ntdm_f64(const double *sub1, const double *main, const double *sup1, const double *rhs,
                double *x, int32_t *status, int32_t *index, int64_t batch, int64_t n, int64_t ld,
                int32_t layout, int32_t algo, void *workspace, size_t workspace_bytes,
                void *stream) {
  int rc = check_common("bx_ntdm_f64", batch, n, 2, ld, layout);
  if (rc) return rc;
  if (batch == 0) return BX_OK;
  BX_REQUIRE(sub1 && main && sup1 && rhs && x, "bx_ntdm_f64: null array pointer");
  const size_t need = bx_workspace_bytes(BX_SOLVER_NTDM, batch, n, layout, algo);
  if (workspace_bytes < need || (need && !workspace)) {
    set_error("bx_ntdm_f64: workspace %zu bytes < required %zu", workspace_bytes, need);
    return BX_ERR_WORKSPACE;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (algo == BX_ALGO_SEQUENTIAL) {
    bx::ntdm_seq(sub1, main, sup1, rhs, x, (double *)workspace, status, index, batch, n, ld,
                 layout, st);
  } else if (algo == BX_ALGO_PARTITIONED) {
    rc = bx::ntdm_part(sub1, main, sup1, rhs, x, (double *)workspace, status, index, batch, n,
                       ld, layout, st);
    if (rc) return rc;
  } else {
    set_error("bx_ntdm_f64: unknown algo %d", algo);
    return BX_ERR_ARG;
  }
  return bxh::check_launch("bx_ntdm_f64");
}

static int penta_common(const char *fn, bool mod, const double *sub2, const double *sub1,
                        const double *main, const double *sup1, const double *sup2,
                        const double *rhs, double *x, int32_t *status, int32_t *index,
                        int64_t *nz, int64_t batch, int64_t n, int64_t ld, int32_t layout,
                        int32_t algo, void *workspace, size_t workspace_bytes, void *stream) {
  int rc = check_common(fn, batch, n, 3, ld, layout);
  if (rc) return rc;
  if (batch == 0) return BX_OK;
  BX_REQUIRE(sub2 && sub1 && main && sup1 && sup2 && rhs && x, "%s: null array pointer", fn);
  const size_t need = bx_workspace_bytes(mod ? BX_SOLVER_MNPDM : BX_SOLVER_NPDM, batch, n, layout, algo);
  if (workspace_bytes < need || (need && !workspace)) {
    set_error("%s: workspace %zu bytes < required %zu", fn, workspace_bytes, need);
    return BX_ERR_WORKSPACE;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (algo == BX_ALGO_SEQUENTIAL) {
    bx::penta_seq(mod, sub2, sub1, main, sup1, sup2, rhs, x, (double *)workspace, status, index,
                  nz, batch, n, ld, layout, st);
  } else if (algo == BX_ALGO_PARTITIONED) {
    rc = bx::penta_part(mod, sub2, sub1, main, sup1, sup2, rhs, x, (double *)workspace, status,
                        index, nz, batch, n, ld, layout, st);
    if (rc) return rc;
  } else {
    set_error("%s: unknown algo %d", fn, algo);
    return BX_ERR_ARG;
  }
  return bxh::check_launch(fn);
}

int bx_npdm_f64(const double *sub2, const double *sub1, const double *main, const double *sup1,
                const double *sup2, const double *rhs, double *x, int32_t *status, int32_t *index,
                int64_t batch, int64_t n, int64_t ld, int32_t layout, int32_t algo,
                void *workspace, size_t workspace_bytes, void *stream) {
  return penta_common("bx_npdm_f64", false, sub2, sub1, main, sup1, sup2, rhs, x, status, index,
                      nullptr, batch, n, ld, layout, algo, workspace, workspace_bytes, stream);
}

int bx_mnpdm_f64(const double *sub2, const double *sub1, const double *main, const double *sup1,
                 const double *sup2, const double *rhs, double *x, int32_t *status,
                 int32_t *index, int64_t *nz_sub2, int64_t batch, int64_t n, int64_t ld,
                 int32_t layout, int32_t algo, void *workspace, size_t workspace_bytes,
                 void *stream) {
  return penta_common("bx_mnpdm_f64", true, sub2, sub1, main, sup1, sup2, rhs, x, status, index,
                      nz_sub2, batch, n, ld, layout, algo, workspace, workspace_bytes, stream);
}

int bx_pd2td_f64(const double *sub2, const double *sub1, const double *main, const double *sup1,
                 const double *sup2, const double *rhs, double *t_sub1, double *t_main,
                 double *t_sup1, double *t_rhs, int64_t *ops, int32_t *status, int32_t *index,
                 int64_t batch, int64_t n, int64_t ld, int64_t ld_out, int32_t layout,
                 void *stream) {
  int rc = check_common("bx_pd2td_f64", batch, n, 3, ld, layout);
  if (rc) return rc;
  rc = check_common("bx_pd2td_f64 (out)", batch, n, 3, ld_out, layout);
  if (rc) return rc;
  if (batch == 0) return BX_OK;
  BX_REQUIRE(sub2 && sub1 && main && sup1 && sup2 && rhs && t_sub1 && t_main && t_sup1 && t_rhs,
             "bx_pd2td_f64: null array pointer");
  bx::pd2td(sub2, sub1, main, sup1, sup2, rhs, t_sub1, t_main, t_sup1, t_rhs, ops, status, index,
            batch, n, ld, ld_out, layout, (cudaStream_t)stream);
  return bxh::check_launch("bx_pd2td_f64");
}

int bx_pd2td_ntdm_f64(const double *sub2, const double *sub1, const double *main,
                      const double *sup1, const double *sup2, const double *rhs, double *x,
                      int64_t *ops, int32_t *status, int32_t *index, int64_t batch, int64_t n,
                      int64_t ld, int32_t layout, void *workspace, size_t workspace_bytes,
                      void *stream) {
  int rc = check_common("bx_pd2td_ntdm_f64", batch, n, 3, ld, layout);
  if (rc) return rc;
  if (batch == 0) return BX_OK;
  BX_REQUIRE(sub2 && sub1 && main && sup1 && sup2 && rhs && x, "bx_pd2td_ntdm_f64: null array pointer");
  const size_t need = bx::pd2td_workspace_bytes(batch, n);
  if (workspace_bytes < need || !workspace) {
    set_error("bx_pd2td_ntdm_f64: workspace %zu bytes < required %zu", workspace_bytes, need);
    return BX_ERR_WORKSPACE;
  }
  bx::pd2td_ntdm(sub2, sub1, main, sup1, sup2, rhs, x, ops, status, index, batch, n, ld, layout,
                 workspace, (cudaStream_t)stream);
  return bxh::check_launch("bx_pd2td_ntdm_f64");
}

/* ---- band building blocks (bx_band_ops.cu) ------------------------------ */
int bx_band_matvec_f64(int32_t bandwidth, int64_t m, const double *subm, const double *sub1,
                       const double *main, const double *sup1, const double *supm, const double *x,
                       const double *rhs, double *y, int64_t batch, int64_t n, int64_t ld,
                       int32_t layout, void *stream) {
  BX_REQUIRE(bandwidth == 1 || bandwidth == 2, "bx_band_matvec_f64: bandwidth must be 1 or 2");
  BX_REQUIRE(bandwidth == 1 || m >= 2, "bx_band_matvec_f64: outer stride m must be >= 2");
  int rc = check_common("bx_band_matvec_f64", batch, n, bandwidth == 1 ? 2 : m + 1, ld, layout);
  if (rc) return rc;
  if (batch == 0) return BX_OK;
  BX_REQUIRE(sub1 && main && sup1 && x && y, "bx_band_matvec_f64: null pointer");
  BX_REQUIRE(bandwidth == 1 || (subm && supm), "bx_band_matvec_f64: null outer diagonal");
  bx::band_matvec(bandwidth, m, subm, sub1, main, sup1, supm, x, rhs, y, batch, n, ld, layout,
                  (cudaStream_t)stream);
  return bxh::check_launch("bx_band_matvec_f64");
}

int bx_lu_penta_f64(const double *sub2, const double *sub1, const double *main, const double *sup1,
                    const double *sup2, double *mu, double *l1, double *l2, double *phi, double *psi,
                    int32_t *status, int32_t *index, int64_t batch, int64_t n, int64_t ld,
                    int32_t layout, void *stream) {
  int rc = check_common("bx_lu_penta_f64", batch, n, 3, ld, layout);
  if (rc) return rc;
  if (batch == 0) return BX_OK;
  BX_REQUIRE(sub2 && sub1 && main && sup1 && sup2 && mu && l1 && l2 && phi && psi,
             "bx_lu_penta_f64: null pointer");
  bx::lu_penta(sub2, sub1, main, sup1, sup2, mu, l1, l2, phi, psi, status, index, batch, n, ld,
               layout, (cudaStream_t)stream);
  return bxh::check_launch("bx_lu_penta_f64");
}

int bx_forward_sub_f64(int64_t m, const double *l1, const double *lm, const double *rhs, double *y,
                       int64_t batch, int64_t n, int64_t ld, int32_t layout, void *stream) {
  BX_REQUIRE(m >= 2, "bx_forward_sub_f64: outer stride m must be >= 2");
  int rc = check_common("bx_forward_sub_f64", batch, n, 2, ld, layout);
  if (rc) return rc;
  if (batch == 0) return BX_OK;
  BX_REQUIRE(l1 && lm && rhs && y, "bx_forward_sub_f64: null pointer");
  bx::forward_sub(m, l1, lm, rhs, y, batch, n, ld, layout, (cudaStream_t)stream);
  return bxh::check_launch("bx_forward_sub_f64");
}

int bx_backward_sub_f64(int64_t m, const double *mu, const double *phi, const double *psi,
                        const double *y, double *x, int32_t *status, int32_t *index, int64_t batch,
                        int64_t n, int64_t ld, int32_t layout, void *stream) {
  BX_REQUIRE(m >= 2, "bx_backward_sub_f64: outer stride m must be >= 2");
  int rc = check_common("bx_backward_sub_f64", batch, n, 2, ld, layout);
  if (rc) return rc;
  if (batch == 0) return BX_OK;
  BX_REQUIRE(mu && phi && psi && y && x, "bx_backward_sub_f64: null pointer");
  bx::backward_sub(m, mu, phi, psi, y, x, status, index, batch, n, ld, layout, (cudaStream_t)stream);
  return bxh::check_launch("bx_backward_sub_f64");
}

size_t bx_hb_invert_dense_workspace_bytes(int64_t batch, int64_t n) {
  return bx::hb_dense_invert_workspace_bytes(batch, n);
}

int bx_hb_invert_dense_f64(const double *m, int64_t n, int64_t ldm, int64_t m_stride, int64_t batch,
                           const double *tol, int64_t max_iter, double *x, int64_t ldx,
                           int64_t x_stride, int64_t *iterations, double *residual,
                           double *history, int32_t *status, int32_t *index, void *workspace,
                           size_t workspace_bytes, void *stream) {
  BX_REQUIRE(n >= 1 && batch >= 0 && max_iter >= 0, "bx_hb_invert_dense_f64: bad sizes");
  BX_REQUIRE(ldm >= n && ldx >= n && m_stride >= n * ldm && (x == nullptr || x_stride >= n * ldx),
             "bx_hb_invert_dense_f64: bad leading dimensions");
  if (batch == 0) return BX_OK;
  BX_REQUIRE(m && tol, "bx_hb_invert_dense_f64: null pointer");
  const size_t need = bx::hb_dense_invert_workspace_bytes(batch, n);
  if (workspace_bytes < need || !workspace) {
    set_error("bx_hb_invert_dense_f64: workspace %zu bytes < required %zu", workspace_bytes, need);
    return BX_ERR_WORKSPACE;
  }
  return bx::hb_dense_invert(m, n, ldm, m_stride, batch, tol, max_iter, x, ldx, x_stride, iterations,
                             residual, history, status, index, workspace, (cudaStream_t)stream);
}

int bx_residual_inf_f64(int32_t bandwidth, const double *sub2, const double *sub1,
                        const double *main, const double *sup1, const double *sup2,
                        const double *x, const double *rhs, double *res_inf, int64_t batch,
                        int64_t n, int64_t ld, int32_t layout, void *stream) {
  BX_REQUIRE(bandwidth == 1 || bandwidth == 2, "bx_residual_inf_f64: bandwidth must be 1 or 2");
  int rc = check_common("bx_residual_inf_f64", batch, n, bandwidth == 1 ? 2 : 3, ld, layout);
  if (rc) return rc;
  if (batch == 0) return BX_OK;
  BX_REQUIRE(sub1 && main && sup1 && x && rhs && res_inf, "bx_residual_inf_f64: null pointer");
  BX_REQUIRE(bandwidth == 1 || (sub2 && sup2), "bx_residual_inf_f64: null sub2/sup2");
  bx::residual_inf(bandwidth, sub2, sub1, main, sup1, sup2, x, rhs, res_inf, batch, n, ld, layout,
                   (cudaStream_t)stream);
  return bxh::check_launch("bx_residual_inf_f64");
}

static int exact_common(const char *fn, int kind, const double *c, const double *d,
                        const double *e, const double *f, const double *g, const double *b,
                        double *x, int32_t *status, int32_t *index, int32_t *subs, int64_t batch,
                        int64_t n, int64_t ld, int32_t layout, void *workspace,
                        size_t workspace_bytes, void *stream) {
  int rc = check_common(fn, batch, n, kind == 1 ? 2 : 3, ld, layout);
  if (rc) return rc;
  if (batch == 0) return BX_OK;
  BX_REQUIRE(d && e && f && b && x && (kind == 1 || (c && g)), "%s: null array pointer", fn);
  const size_t need = bx::exact_workspace_bytes(kind, batch, n);
  if (workspace_bytes < need || !workspace) {
    set_error("%s: workspace %zu bytes < required %zu", fn, workspace_bytes, need);
    return BX_ERR_WORKSPACE;
  }
  bx::exact_solve(kind, c, d, e, f, g, b, x, status, index, subs, (double *)workspace, batch, n,
                  ld, layout, (cudaStream_t)stream);
  return bxh::check_launch(fn);
}

int bx_stdm_f64(const double *sub1, const double *main, const double *sup1, const double *rhs,
                double *x, int32_t *status, int32_t *index, int32_t *substitutions,
                int64_t batch, int64_t n, int64_t ld, int32_t layout, void *workspace,
                size_t workspace_bytes, void *stream) {
  return exact_common("bx_stdm_f64", 1, nullptr, sub1, main, sup1, nullptr, rhs, x, status, index,
                      substitutions, batch, n, ld, layout, workspace, workspace_bytes, stream);
}

int bx_spdm_f64(const double *sub2, const double *sub1, const double *main, const double *sup1,
                const double *sup2, const double *rhs, double *x, int32_t *status,
                int32_t *index, int32_t *substitutions, int64_t batch, int64_t n, int64_t ld,
                int32_t layout, void *workspace, size_t workspace_bytes, void *stream) {
  return exact_common("bx_spdm_f64", 2, sub2, sub1, main, sup1, sup2, rhs, x, status, index,
                      substitutions, batch, n, ld, layout, workspace, workspace_bytes, stream);
}

int bx_det_band_f64(int32_t bandwidth, const double *sub2, const double *sub1, const double *main,
                    const double *sup1, const double *sup2, double *mantissa, int64_t *exponent,
                    int32_t *status, int32_t *index, int32_t *substitutions, int64_t batch,
                    int64_t n, int64_t ld, int32_t layout, void *stream) {
  BX_REQUIRE(bandwidth == 1 || bandwidth == 2, "bx_det_band_f64: bandwidth must be 1 or 2");
  int rc = check_common("bx_det_band_f64", batch, n, bandwidth == 1 ? 2 : 3, ld, layout);
  if (rc) return rc;
  if (batch == 0) return BX_OK;
  BX_REQUIRE(sub1 && main && sup1 && mantissa && exponent && (bandwidth == 1 || (sub2 && sup2)),
             "bx_det_band_f64: null array pointer");
  bx::det_band(bandwidth, sub2, sub1, main, sup1, sup2, mantissa, exponent, status, index,
               substitutions, batch, n, ld, layout, (cudaStream_t)stream);
  return bxh::check_launch("bx_det_band_f64");
}

int bx_outer_compact_f64(const double *sub2, const double *sup2, int32_t *count, int32_t *rows,
                         double *vals_sub2, double *vals_sup2, int64_t capacity, int64_t batch,
                         int64_t n, int64_t ld, int32_t layout, void *stream) {
  const char *fn = "bx_outer_compact_f64";
  int rc = check_common(fn, batch, n, 3, ld, layout);
  if (rc) return rc;
  BX_REQUIRE(capacity >= 0, "%s: capacity must be >= 0", fn);
  if (batch == 0) return BX_OK;
  BX_REQUIRE(sub2 && sup2 && count && (capacity == 0 || (rows && vals_sub2 && vals_sup2)),
             "%s: null pointer", fn);
  bx::outer_compact(sub2, sup2, count, rows, vals_sub2, vals_sup2, capacity, batch, n, ld, layout,
                    (cudaStream_t)stream);
  return bxh::check_launch(fn);
}

int bx_mnpdm_sparse_f64(const int32_t *outer_rows, const double *outer_sub2,
                        const double *outer_sup2, int64_t outer_k, const double *sub1,
                        const double *main, const double *sup1, const double *rhs, double *x,
                        int32_t *status, int32_t *index, int64_t *nz_sub2, int64_t batch,
                        int64_t n, int64_t ld, int32_t layout, void *stream) {
  const char *fn = "bx_mnpdm_sparse_f64";
  int rc = check_common(fn, batch, n, 3, ld, layout);
  if (rc) return rc;
  BX_REQUIRE(outer_k >= 0, "%s: outer_k must be >= 0", fn);
  if (batch == 0) return BX_OK;
  BX_REQUIRE(sub1 && main && sup1 && rhs && x && (outer_k == 0 || (outer_rows && outer_sub2 && outer_sup2)),
             "%s: null pointer", fn);
  rc = bx::mnpdm_sparse_part(outer_rows, outer_sub2, outer_sup2, outer_k, sub1, main, sup1, rhs, x,
                             status, index, nz_sub2, batch, n, ld, layout, (cudaStream_t)stream);
  if (rc) return rc;
  return bxh::check_launch(fn);
}

size_t bx_rcond_workspace_bytes(int32_t bandwidth, int64_t batch, int64_t n) {
  return bx::rcond_workspace_bytes(bandwidth == 1 ? 1 : 2, batch, n);
}

int bx_rcond_band_f64(int32_t bandwidth, const double *sub2, const double *sub1,
                      const double *main, const double *sup1, const double *sup2, double *rcond,
                      int32_t *status, int32_t *index, int64_t batch, int64_t n, int64_t ld,
                      int32_t layout, void *workspace, size_t workspace_bytes, void *stream) {
  const char *fn = "bx_rcond_band_f64";
  BX_REQUIRE(bandwidth == 1 || bandwidth == 2, "%s: bandwidth must be 1 or 2", fn);
  int rc = check_common(fn, batch, n, bandwidth == 1 ? 2 : 3, ld, layout);
  if (rc) return rc;
  if (batch == 0) return BX_OK;
  BX_REQUIRE(sub1 && main && sup1 && rcond && (bandwidth == 1 || (sub2 && sup2)),
             "%s: null array pointer", fn);
  const size_t need = bx::rcond_workspace_bytes(bandwidth, batch, n);
  if (workspace_bytes < need || !workspace) {
    set_error("%s: workspace %zu bytes < required %zu", fn, workspace_bytes, need);
    return BX_ERR_WORKSPACE;
  }
  bx::rcond_band(bandwidth, sub2, sub1, main, sup1, sup2, rcond, status, index,
                 (double *)workspace, batch, n, ld, layout, (cudaStream_t)stream);
  return bxh::check_launch(fn);
}

static int check_sip_args(const char *fn, int64_t batch, int64_t n, int64_t m, double alpha,
                          int64_t ld, int32_t layout) {
  int rc = check_common(fn, batch, n, 3, ld, layout);
  if (rc) return rc;
  BX_REQUIRE(m >= 2 && m < n, "%s: outer offset m=%lld must satisfy 2 <= m < n", fn, (long long)m);
  BX_REQUIRE(m >= 3 || alpha == 0.0, "%s: Stone's alpha needs m >= 3 (m = 2 is the reference ILU(0))", fn);
  BX_REQUIRE(alpha == alpha, "%s: alpha is NaN", fn);
  return BX_OK;
}

int bx_ilu0_f64(const double *subm, const double *sub1, const double *main, const double *sup1,
                const double *supm, double *mu, double *l1, double *l2, double *phi, double *psi,
                double *k_subm, double *k_sub1, double *k_main, double *k_sup1, double *k_supm,
                double *k_subq, double *k_supq, int32_t *status, int32_t *index, int64_t batch,
                int64_t n, int64_t m, double alpha, int64_t ld, int32_t layout, void *workspace,
                size_t workspace_bytes, void *stream) {
  int rc = check_sip_args("bx_ilu0_f64", batch, n, m, alpha, ld, layout);
  if (rc) return rc;
  if (batch == 0) return BX_OK;
  BX_REQUIRE(subm && sub1 && main && sup1 && supm, "bx_ilu0_f64: null matrix pointer");
  const size_t need = bx::sip_workspace_bytes(batch, n);
  if (workspace_bytes < need || !workspace) {
    set_error("bx_ilu0_f64: workspace %zu bytes < required %zu", workspace_bytes, need);
    return BX_ERR_WORKSPACE;
  }
  cudaStream_t st = (cudaStream_t)stream;
  bx::sip_seq(subm, sub1, main, sup1, supm, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
              nullptr, status, index, nullptr, (double *)workspace, batch, n, m, alpha, 0, 0, ld,
              layout, 1, st);
  rc = bxh::check_launch("bx_ilu0_f64");
  if (rc) return rc;
  double *outs[12] = {mu, l1, l2, phi, psi, k_subm, k_sub1, k_main, k_sup1, k_supm, k_subq, k_supq};
  rc = bx::sip_export((double *)workspace, batch, n, outs, ld, layout, st);
  if (rc) return rc;
  return bxh::check_launch("bx_ilu0_f64 export");
}

int bx_sip_f64(const double *subm, const double *sub1, const double *main, const double *sup1,
               const double *supm, const double *rhs, const double *tol, double *x,
               double *best_x, int64_t *iterations, double *residual, double *best_residual,
               int32_t *status, int32_t *index, double *history, int64_t batch, int64_t n,
               int64_t m, double alpha, int64_t max_iter, int32_t use_x0, int64_t ld,
               int32_t layout, int32_t algo, void *workspace, size_t workspace_bytes,
               void *stream) {
  int rc = check_sip_args("bx_sip_f64", batch, n, m, alpha, ld, layout);
  if (rc) return rc;
  BX_REQUIRE(max_iter >= 1, "bx_sip_f64: max_iter must be at least 1");
  if (batch == 0) return BX_OK;
  BX_REQUIRE(subm && sub1 && main && sup1 && supm && rhs && tol && x,
             "bx_sip_f64: null array pointer");
  cudaStream_t st = (cudaStream_t)stream;
  if (algo == BX_ALGO_AUTO) {
    BX_REQUIRE(workspace && workspace_bytes >= 4, "bx_sip_f64: workspace required");
    algo = bx::sip_is_grid(sub1, sup1, batch, n, m, ld, layout, workspace, st)
               ? BX_ALGO_WAVEFRONT
               : BX_ALGO_SEQUENTIAL;
  }
  if (algo != BX_ALGO_SEQUENTIAL && algo != BX_ALGO_WAVEFRONT && algo != BX_ALGO_SCAN) {
    set_error("bx_sip_f64: unknown algo %d", algo);
    return BX_ERR_ARG;
  }
  const size_t need = algo == BX_ALGO_WAVEFRONT ? bx::sip_wave_workspace_bytes(batch, n, m)
                      : algo == BX_ALGO_SCAN    ? bx::sip_scan_workspace_bytes(batch, n, m)
                                                : bx::sip_workspace_bytes(batch, n);
  if (algo == BX_ALGO_SCAN && need == 0) {
    set_error("bx_sip_f64: BX_ALGO_SCAN needs a grid width m that is a multiple of 32 in [32, 512] "
              "and n %% m == 0 (n=%lld, m=%lld)", (long long)n, (long long)m);
    return BX_ERR_UNSUPPORTED;
  }
  if (workspace_bytes < need || !workspace) {
    set_error("bx_sip_f64: workspace %zu bytes < required %zu", workspace_bytes, need);
    return BX_ERR_WORKSPACE;
  }
  if (algo == BX_ALGO_SEQUENTIAL) {
    bx::sip_seq(subm, sub1, main, sup1, supm, rhs, tol, x, best_x, iterations, residual,
                best_residual, status, index, history, (double *)workspace, batch, n, m, alpha,
                max_iter, use_x0, ld, layout, 0, st);
  } else if (algo == BX_ALGO_SCAN) {
    rc = bx::sip_scan(subm, sub1, main, sup1, supm, rhs, tol, x, best_x, iterations, residual,
                      best_residual, status, index, history, (double *)workspace, batch, n, m,
                      alpha, max_iter, use_x0, ld, layout, st);
    if (rc) return rc;
  } else {
    rc = bx::sip_wave(subm, sub1, main, sup1, supm, rhs, tol, x, best_x, iterations, residual,
                      best_residual, status, index, history, (double *)workspace, batch, n, m,
                      alpha, max_iter, use_x0, ld, layout, st);
    if (rc) return rc;
  }
  return bxh::check_launch("bx_sip_f64");
}

int bx_transpose_f64(const double *src, double *dst, int64_t rows, int64_t cols, int64_t ld_src,
                     int64_t ld_dst, int64_t nbatch, int64_t batch_stride_src,
                     int64_t batch_stride_dst, void *stream) {
  BX_REQUIRE(rows >= 0 && cols >= 0 && nbatch >= 0, "bx_transpose_f64: negative extent");
  if (rows == 0 || cols == 0 || nbatch == 0) return BX_OK;
  BX_REQUIRE(src && dst, "bx_transpose_f64: null pointer");
  BX_REQUIRE(ld_src >= cols && ld_dst >= rows, "bx_transpose_f64: leading dimension too small");
  BX_REQUIRE(rows / 32 < 65535 && nbatch < 65535, "bx_transpose_f64: extent too large");
  bx::transpose(src, dst, rows, cols, ld_src, ld_dst, nbatch, batch_stride_src, batch_stride_dst,
                (cudaStream_t)stream);
  return bxh::check_launch("bx_transpose_f64");
}

size_t bx_hb_workspace_bytes(int64_t batch, int64_t n) {
  return bx::hb_total_workspace_bytes(batch, n);
}

int bx_hb_invert_f64(const double *subm, const double *sub1, const double *main,
                     const double *sup1, const double *supm, const double *tol, double *x_lower,
                     double *x_upper, int64_t *inv_iterations, double *inv_residual,
                     int32_t *status, int32_t *index, int64_t batch, int64_t n, int64_t m,
                     double alpha, int64_t max_iter, int64_t ld, int32_t layout, void *workspace,
                     size_t workspace_bytes, void *stream) {
  int rc = check_sip_args("bx_hb_invert_f64", batch, n, m, alpha, ld, layout);
  if (rc) return rc;
  if (batch == 0) return BX_OK;
  BX_REQUIRE(subm && sub1 && main && sup1 && supm && tol, "bx_hb_invert_f64: null pointer");
  BX_REQUIRE(max_iter >= 0, "bx_hb_invert_f64: max_iter must be >= 0");
  const size_t need = bx::hb_total_workspace_bytes(batch, n);
  if (workspace_bytes < need || !workspace) {
    set_error("bx_hb_invert_f64: workspace %zu bytes < required %zu", workspace_bytes, need);
    return BX_ERR_WORKSPACE;
  }
  return bx::sip_hb(subm, sub1, main, sup1, supm, nullptr, tol, nullptr, nullptr, nullptr, nullptr,
                    nullptr, status, index, nullptr, inv_iterations, inv_residual, batch, n, m,
                    alpha, 0, max_iter, 0, ld, layout, workspace, (cudaStream_t)stream, true,
                    x_lower, x_upper);
}

int bx_sip_hb_f64(const double *subm, const double *sub1, const double *main, const double *sup1,
                  const double *supm, const double *rhs, const double *tol, double *x,
                  double *best_x, int64_t *iterations, double *residual, double *best_residual,
                  int32_t *status, int32_t *index, double *history, int64_t *inv_iterations,
                  double *inv_residual, int64_t batch, int64_t n, int64_t m, double alpha,
                  int64_t max_iter, int64_t max_inv_iter, int32_t use_x0, int64_t ld,
                  int32_t layout, void *workspace, size_t workspace_bytes, void *stream) {
  int rc = check_sip_args("bx_sip_hb_f64", batch, n, m, alpha, ld, layout);
  if (rc) return rc;
  BX_REQUIRE(max_iter >= 1, "bx_sip_hb_f64: max_iter must be at least 1");
  if (batch == 0) return BX_OK;
  BX_REQUIRE(subm && sub1 && main && sup1 && supm && rhs && tol && x,
             "bx_sip_hb_f64: null array pointer");
  const size_t need = bx::hb_total_workspace_bytes(batch, n);
  if (workspace_bytes < need || !workspace) {
    set_error("bx_sip_hb_f64: workspace %zu bytes < required %zu", workspace_bytes, need);
    return BX_ERR_WORKSPACE;
  }
  return bx::sip_hb(subm, sub1, main, sup1, supm, rhs, tol, x, best_x, iterations, residual,
                    best_residual, status, index, history, inv_iterations, inv_residual, batch, n,
                    m, alpha, max_iter, max_inv_iter, use_x0, ld, layout, workspace,
                    (cudaStream_t)stream, false, nullptr, nullptr);
}

size_t bx_hb_banded_workspace_bytes(int64_t batch, int64_t n, int64_t w_cap) {
  return bx::sip_hb_band_workspace_bytes(batch, n, w_cap);
}

int bx_hb_invert_banded_f64(const double *mu, const double *l1, const double *l2,
                            const double *phi, const double *psi, int32_t side, int64_t w,
                            const double *tol, int64_t max_iter, double *x_diags,
                            int64_t *iterations, double *residual, double *history,
                            int32_t *status, int32_t *index, int64_t batch, int64_t n, int64_t ld,
                            int32_t layout, void *workspace, size_t workspace_bytes,
                            void *stream) {
  const char *fn = "bx_hb_invert_banded_f64";
  int rc = check_common(fn, batch, n, 3, ld, layout);
  if (rc) return rc;
  BX_REQUIRE(side == 0 || side == 1, "%s: side must be 0 (lower) or 1 (upper)", fn);
  BX_REQUIRE(w >= 2, "%s: banded inversion needs bandwidth w >= 2 (inverse.py:160-161)", fn);
  BX_REQUIRE(w <= n - 1, "%s: bandwidth w=%lld exceeds n-1", fn, (long long)w);
  BX_REQUIRE(max_iter >= 0, "%s: max_iter must be >= 0", fn);
  if (batch == 0) return BX_OK;
  BX_REQUIRE(tol && (side == 0 ? (l1 && l2) : (mu && phi && psi)), "%s: null pointer", fn);
  const size_t need = bx::hb_band_invert_workspace_bytes(batch, n, w);
  if (workspace_bytes < need || !workspace) {
    set_error("%s: workspace %zu bytes < required %zu", fn, workspace_bytes, need);
    return BX_ERR_WORKSPACE;
  }
  return bx::hb_band_invert(mu, l1, l2, phi, psi, side, w, tol, max_iter, x_diags, iterations,
                            residual, history, status, index, batch, n, ld, layout, workspace,
                            (cudaStream_t)stream);
}

int bx_sip_hb_banded_f64(const double *sub2, const double *sub1, const double *main,
                         const double *sup1, const double *sup2, const double *rhs,
                         const double *tol, double *x, double *best_x, int64_t *iterations,
                         double *residual, double *best_residual, int32_t *status,
                         int32_t *index, double *history, int64_t hb_bandwidth, int64_t w_cap,
                         int64_t *w_used, int64_t *inv_iterations, double *inv_residual,
                         double *inv_true_residual, int64_t batch, int64_t n, int64_t max_iter,
                         int64_t max_inv_iter, int32_t use_x0, int64_t ld, int32_t layout,
                         void *workspace, size_t workspace_bytes, void *stream) {
  const char *fn = "bx_sip_hb_banded_f64";
  int rc = check_sip_args(fn, batch, n, 2, 0.0, ld, layout);
  if (rc) return rc;
  BX_REQUIRE(max_iter >= 1, "%s: max_iter must be at least 1", fn);
  BX_REQUIRE(hb_bandwidth == 0 || hb_bandwidth >= 2, "%s: hb_bandwidth must be 0 (auto) or >= 2", fn);
  BX_REQUIRE(hb_bandwidth <= n - 1, "%s: hb_bandwidth exceeds n-1", fn);
  BX_REQUIRE(w_cap >= 2 && w_cap >= hb_bandwidth, "%s: w_cap must be >= max(2, hb_bandwidth)", fn);
  if (batch == 0) return BX_OK;
  BX_REQUIRE(sub2 && sub1 && main && sup1 && sup2 && rhs && tol && x, "%s: null array pointer", fn);
  const size_t need = bx::sip_hb_band_workspace_bytes(batch, n, w_cap);
  if (workspace_bytes < need || !workspace) {
    set_error("%s: workspace %zu bytes < required %zu", fn, workspace_bytes, need);
    return BX_ERR_WORKSPACE;
  }
  return bx::sip_hb_band(sub2, sub1, main, sup1, sup2, rhs, tol, x, best_x, iterations, residual,
                         best_residual, status, index, history, hb_bandwidth, w_cap, w_used,
                         inv_iterations, inv_residual, inv_true_residual, batch, n, max_iter,
                         max_inv_iter, use_x0, ld, layout, workspace, (cudaStream_t)stream);
}

}  // extern "C"
