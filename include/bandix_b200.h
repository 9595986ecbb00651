/*
 * bandix_b200 -- C ABI of the B200-native batched band-SLAE solvers.
 *
 * This is the drop-in boundary for the hot path of the reference package
 * bandix 0.1.0 (/root/reference/pkg/src/bandix).  The reference is pure
 * Python and has no FFI of its own; each entry point below replaces one
 * reference solver function, batched over a system index, and is what a
 * ctypes / cffi binding of the reference would call (INTEGRATION.md shows
 * the binding).  No torch types cross this boundary: plain device pointers,
 * sizes and a cudaStream_t passed as void*.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - All arrays are DEVICE pointers to IEEE binary64 (or int32 for status).
 *  - A band system of order n is stored by diagonals, ROW-ALIGNED: every
 *    diagonal array has n rows and row i holds the coefficient of equation
 *    i (sub2[i] = A[i,i-2], sub1[i] = A[i,i-1], main[i] = A[i,i],
 *    sup1[i] = A[i,i+1], sup2[i] = A[i,i+2]).  The reference stores the same
 *    entries unpadded (core.py:117-164: sub2[i-2], sub1[i-1], ...); slots that
 *    fall outside the matrix (sub2 rows 0-1, sub1 row 0, sup1 row n-1,
 *    sup2 rows n-2..n-1) are NEVER read.
 *  - layout = BX_LAYOUT_INTERLEAVED: element (row i, system s) at p[i*ld + s]
 *    (system index fastest, ld >= batch).  BX_LAYOUT_SYSTEM_MAJOR: at
 *    p[s*ld + i] (ld >= n).  One ld applies to every array of the call.
 *  - status[s] / index[s] (int32, may be NULL): per-system outcome, the
 *    batched form of the reference's exceptions (errors.py): BX_STATUS_*
 *    below; index is the failing row (ZeroPivot.index) or -1.
 *  - Return value: BX_OK, or an argument / launch error (bx_last_error()
 *    gives the message).  Numerical outcomes never fail the call.
 *  - Calls are stream-ordered and asynchronous (exceptions, stated at their
 *    declarations: the Hotelling-Bodewig entry points drive their iteration
 *    from the host and synchronise the stream); they do not allocate on the
 *    hot path -- scratch comes from a caller-provided workspace of at least
 *    bx_workspace_bytes(...) bytes.  Reentrant on distinct buffers/streams.
 */
#ifndef BANDIX_B200_H
#define BANDIX_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* return codes */
#define BX_OK 0
#define BX_ERR_ARG 1
#define BX_ERR_CUDA 2
#define BX_ERR_WORKSPACE 3
#define BX_ERR_UNSUPPORTED 4

/* per-system status (errors.py:29-102) */
#define BX_STATUS_OK 0
#define BX_STATUS_ZERO_PIVOT 1      /* ZeroPivot(index)            errors.py:29-34 */
#define BX_STATUS_SINGULAR 2        /* SingularMatrix              errors.py:45-46 */
#define BX_STATUS_MAX_ITER 3        /* MaxIterationsExceeded       errors.py:49-59 */
#define BX_STATUS_DIVERGED 4        /* Diverged                    errors.py:62-70 */
#define BX_STATUS_ZERO_DIAG 5       /* ZeroDiagonal(index)         errors.py:73-78 */
#define BX_STATUS_WINDOW_OVERFLOW 6 /* fp64 symbolic window exceeded (no reference twin) */
#define BX_STATUS_NOT_GRID 7        /* wavefront SIP given a system whose +-1 couplings cross grid rows */
#define BX_STATUS_REDUCTION_PIVOT 8 /* ReductionPivotZero(index)   errors.py:37-42 */
#define BX_STATUS_STAGNATED 9       /* Stagnated(best report)      errors.py:81-93 */

/* layouts */
#define BX_LAYOUT_INTERLEAVED 0
#define BX_LAYOUT_SYSTEM_MAJOR 1

/* algorithms for the direct solvers */
#define BX_ALGO_SEQUENTIAL 0   /* reference operation order, bit-identical results */
/* On-chip partitioned elimination, tolerance parity (<= 1e-10 relative).  Two
 * passes chosen per system on the device: chunk two-ports coupled by a fixed
 * number of block-Jacobi sweeps over the chunk interfaces (exact to rounding
 * when the measured interface coupling is below 2^-13, i.e. for diagonally
 * dominant systems), then the two-port tree for the systems that fail that
 * test (exact for any nonsingular reduced system).  Systems with a zero or
 * non-finite pivot of this elimination order are re-solved in the reference
 * order, so their x / status / index are the reference's. */
#define BX_ALGO_PARTITIONED 1

/* solver ids for bx_workspace_bytes */
#define BX_SOLVER_NTDM 0
#define BX_SOLVER_NPDM 1
#define BX_SOLVER_MNPDM 2
#define BX_SOLVER_STDM 3
#define BX_SOLVER_SPDM 4
#define BX_SOLVER_SIP 5
#define BX_SOLVER_HB 6
#define BX_SOLVER_PD2TD 7          /* bx_pd2td_ntdm_f64 */

const char *bx_version(void);
const char *bx_last_error(void);

/* Bytes of scratch the given solver needs (0 is a valid answer). */
size_t bx_workspace_bytes(int32_t solver, int64_t batch, int64_t n, int32_t layout,
                          int32_t algo);

/* ---- direct solvers ----------------------------------------------------- */

/* Thomas with reciprocal pivots.  Replaces solve_ntdm (direct.py:103-113):
 * tri_factor_recip + tri_solve_recip (_elim.py:90-122).  n >= 2. */
int bx_ntdm_f64(const double *sub1, const double *main, const double *sup1,
                const double *rhs, double *x, int32_t *status, int32_t *index,
                int64_t batch, int64_t n, int64_t ld, int32_t layout, int32_t algo,
                void *workspace, size_t workspace_bytes, void *stream);

/* Banded Doolittle LU + substitutions.  Replaces solve_npdm
 * (direct.py:73-81): penta_factor/penta_forward/penta_backward
 * (_elim.py:30-87).  n >= 3. */
int bx_npdm_f64(const double *sub2, const double *sub1, const double *main,
                const double *sup1, const double *sup2, const double *rhs, double *x,
                int32_t *status, int32_t *index, int64_t batch, int64_t n, int64_t ld,
                int32_t layout, int32_t algo, void *workspace, size_t workspace_bytes,
                void *stream);

/* Sparsity-aware reciprocal-pivot PD solve.  Replaces solve_mnpdm
 * (direct.py:84-100): mnpdm_sweep (_elim.py:125-190).  nz_sub2 (int64 per
 * system, may be NULL) receives the structurally nonzero sub2 count that the
 * reference's op counter uses (direct.py:98-99). */
int bx_mnpdm_f64(const double *sub2, const double *sub1, const double *main,
                 const double *sup1, const double *sup2, const double *rhs, double *x,
                 int32_t *status, int32_t *index, int64_t *nz_sub2, int64_t batch, int64_t n,
                 int64_t ld, int32_t layout, int32_t algo, void *workspace,
                 size_t workspace_bytes, void *stream);

/* MNPDM with sparse outer diagonals -- the case MNPDM exists for (_elim.py:
 * 125-190 skips the eliminations where sub2 == 0; the paper's K outer
 * nonzeros).  bx_outer_compact_f64 lists, per system and in row order, the
 * rows whose sub2 (i >= 2) or sup2 (i <= n-3) is nonzero: count[batch]
 * always; with capacity > 0 also rows[batch][capacity] (-1 pads) and the
 * two values at those rows.  bx_mnpdm_sparse_f64 then solves from sub1 /
 * main / sup1 / rhs plus that list (partitioned algorithm, 40 B/row of
 * compulsory traffic instead of 56): x, status, index and nz_sub2 (may be
 * NULL) as bx_mnpdm_f64. */
int bx_outer_compact_f64(const double *sub2, const double *sup2, int32_t *count, int32_t *rows,
                         double *vals_sub2, double *vals_sup2, int64_t capacity, int64_t batch,
                         int64_t n, int64_t ld, int32_t layout, void *stream);
int bx_mnpdm_sparse_f64(const int32_t *outer_rows, const double *outer_sub2,
                        const double *outer_sup2, int64_t outer_k, const double *sub1,
                        const double *main, const double *sup1, const double *rhs, double *x,
                        int32_t *status, int32_t *index, int64_t *nz_sub2, int64_t batch,
                        int64_t n, int64_t ld, int32_t layout, void *stream);

/* pd_to_td (direct.py:116-165): Gaussian reduction of pentadiagonal systems
 * to tridiagonal ones in the reference's operation order (bit-identical).
 * Inputs as bx_npdm_f64 (layout/ld); outputs t_sub1/t_main/t_sup1/t_rhs are
 * row-aligned in the same layout with leading dimension ld_out.  ops
 * (3*batch int64, may be NULL): (muls, subs, divs) of each system's reduction
 * (the reference's CounterBox).  status BX_STATUS_REDUCTION_PIVOT with index =
 * the row whose elimination met a zero pivot (ReductionPivotZero(i)). */
int bx_pd2td_f64(const double *sub2, const double *sub1, const double *main,
                 const double *sup1, const double *sup2, const double *rhs, double *t_sub1,
                 double *t_main, double *t_sup1, double *t_rhs, int64_t *ops, int32_t *status,
                 int32_t *index, int64_t batch, int64_t n, int64_t ld, int64_t ld_out,
                 int32_t layout, void *stream);

/* solve_pd2td_ntdm (direct.py:168-177): pd_to_td, then the reference NTDM
 * (bx_ntdm_f64, sequential) on the reduced system; x in the input layout.
 * ops as bx_pd2td_f64 (reduction only; the Thomas part is 9N-7 closed form).
 * status: REDUCTION_PIVOT from the reduction, else ZERO_PIVOT from NTDM.
 * Workspace: bx_workspace_bytes(BX_SOLVER_PD2TD, batch, n, layout, 0). */
int bx_pd2td_ntdm_f64(const double *sub2, const double *sub1, const double *main,
                      const double *sup1, const double *sup2, const double *rhs, double *x,
                      int64_t *ops, int32_t *status, int32_t *index, int64_t batch, int64_t n,
                      int64_t ld, int32_t layout, void *workspace, size_t workspace_bytes,
                      void *stream);

/* ---- band building blocks (reference operation order, bit-identical) ------ */
/* y = A x (rhs == NULL) or y = rhs - A x for a band of bandwidth 1 (subm/supm
 * unused, may be NULL) or a five-point band with outer offset m (m = 2: the
 * pentadiagonal).  Replaces penta_matvec / tri_matvec / residual
 * (core.py:243-314; the float branch's array-sweep order main, sub1, sup1,
 * sub2, sup2).  One thread per element. */
int bx_band_matvec_f64(int32_t bandwidth, int64_t m, const double *subm, const double *sub1,
                       const double *main, const double *sup1, const double *supm, const double *x,
                       const double *rhs, double *y, int64_t batch, int64_t n, int64_t ld,
                       int32_t layout, void *stream);

/* lu_penta (direct.py:42-63 -> penta_factor, _elim.py:30-62): banded Doolittle
 * factors, row-aligned in the call's layout: mu (U main), l1 = L(i,i-1),
 * l2 = L(i,i-2), phi = U(i,i+1), psi = U(i,i+2); structurally absent slots
 * are 0.  status ZERO_PIVOT with index = the first zero pivot (ZeroPivot(i);
 * the factors are then not usable).  n >= 3. */
int bx_lu_penta_f64(const double *sub2, const double *sub1, const double *main, const double *sup1,
                    const double *sup2, double *mu, double *l1, double *l2, double *phi, double *psi,
                    int32_t *status, int32_t *index, int64_t batch, int64_t n, int64_t ld,
                    int32_t layout, void *stream);

/* forward_sub (iterative.py:127-137 -> penta_forward): L y = rhs with unit
 * diagonal, l1 at offset -1 and lm at offset -m (m = 2: lu_penta / ilu0
 * factors of the pentadiagonal; m >= 3: grid ILU(0) factors).  y may alias
 * rhs. */
int bx_forward_sub_f64(int64_t m, const double *l1, const double *lm, const double *rhs, double *y,
                       int64_t batch, int64_t n, int64_t ld, int32_t layout, void *stream);

/* backward_sub (iterative.py:140-149 -> penta_backward): U x = y with pivots
 * mu, phi at +1, psi at +m.  A zero pivot anywhere gives status ZERO_PIVOT
 * with index = the first one (checked before any division) and x = NaN. */
int bx_backward_sub_f64(int64_t m, const double *mu, const double *phi, const double *psi,
                        const double *y, double *x, int32_t *status, int32_t *index, int64_t batch,
                        int64_t n, int64_t ld, int32_t layout, void *stream);

/* ||b - A x||_inf per system, the report residual of _finish_report
 * (direct.py:66-70 -> core.py:243-321), in the reference's row-fused
 * operation order.  bandwidth 1 (tridiagonal: sub2/sup2 ignored, may be
 * NULL) or 2 (pentadiagonal). */
int bx_residual_inf_f64(int32_t bandwidth, const double *sub2, const double *sub1,
                        const double *main, const double *sup1, const double *sup2,
                        const double *x, const double *rhs, double *res_inf, int64_t batch,
                        int64_t n, int64_t ld, int32_t layout, void *stream);

/* dst[b][c][r] = src[b][r][c] (r < rows, c < cols): converts between the
 * interleaved and system-major storages (and feeds the ADI y-sweep the
 * x-sweep output).  Strides in elements; smem-tiled, both sides coalesced. */
int bx_transpose_f64(const double *src, double *dst, int64_t rows, int64_t cols, int64_t ld_src,
                     int64_t ld_dst, int64_t nbatch, int64_t batch_stride_src,
                     int64_t batch_stride_dst, void *stream);

/* ---- symbolic solvers ----------------------------------------------------- */
/* STDM / SPDM: exact-zero pivots are replaced by the indeterminate t and the
 * solution is the limit t -> 0, as exact_solve_stdm / exact_solve_spdm
 * (exact.py:278-307).  The reference works over exact rationals; here the
 * rational functions are truncated Laurent series in t with binary64
 * coefficients.  Inputs are binary64 (the reference requires exact
 * input and rejects floats, exact.py:232-236; a float is an exact rational).
 * substitutions[s] (may be NULL) = ExactSolveResult.pivot_substitutions.
 * status: OK, SINGULAR (exact_det_band == 0 -> SingularMatrix) or
 * WINDOW_OVERFLOW (the fixed series window could not hold the expansion). */
int bx_stdm_f64(const double *sub1, const double *main, const double *sup1, const double *rhs,
                double *x, int32_t *status, int32_t *index, int32_t *substitutions,
                int64_t batch, int64_t n, int64_t ld, int32_t layout, void *workspace,
                size_t workspace_bytes, void *stream);
int bx_spdm_f64(const double *sub2, const double *sub1, const double *main, const double *sup1,
                const double *sup2, const double *rhs, double *x, int32_t *status,
                int32_t *index, int32_t *substitutions, int64_t batch, int64_t n, int64_t ld,
                int32_t layout, void *workspace, size_t workspace_bytes, void *stream);

/* exact_det_band (exact.py:254-275): the determinant as the product of the
 * same t-substituted pivots at t -> 0 (zero exactly when the substituted
 * pivots' orders sum to > 0 -- the reference's nonsingularity gate).  One
 * thread per system, bandwidth 1 (sub2/sup2 unused, may be NULL) or 2.
 * det[s] = mantissa[s] * 2^exponent[s], |mantissa| in [0.5, 1) or 0, so that
 * no product of n pivots overflows.  substitutions (may be NULL) as
 * bx_stdm_f64; status OK or WINDOW_OVERFLOW (mantissa NaN). */
int bx_det_band_f64(int32_t bandwidth, const double *sub2, const double *sub1, const double *main,
                    const double *sup1, const double *sup2, double *mantissa, int64_t *exponent,
                    int32_t *status, int32_t *index, int32_t *substitutions, int64_t batch,
                    int64_t n, int64_t ld, int32_t layout, void *stream);

/* Reciprocal condition estimate in the 1-norm, LAPACK's convention
 * (dgtcon / dgbcon, norm '1'): rcond = 1 / (||A||_1 est ||A^-1||_1), A = P L U
 * with partial pivoting, est by Hager-Higham (dlacn2).  The condition gate
 * of SURVEY 8f row f1 (no reference twin: the reference's exact solvers need
 * none; SURVEY H7 asks config-3 errors to be read against it).  rcond = 0 and
 * status SINGULAR (index = first zero pivot column) for an exactly singular
 * U.  Workspace: bx_rcond_workspace_bytes(bandwidth, batch, n). */
size_t bx_rcond_workspace_bytes(int32_t bandwidth, int64_t batch, int64_t n);
int bx_rcond_band_f64(int32_t bandwidth, const double *sub2, const double *sub1,
                      const double *main, const double *sup1, const double *sup2, double *rcond,
                      int32_t *status, int32_t *index, int64_t batch, int64_t n, int64_t ld,
                      int32_t layout, void *workspace, size_t workspace_bytes, void *stream);

/* ---- ILU(0) / SIP -------------------------------------------------------- */
/* Stride-m five-point band: subm[i] = A[i,i-m], sub1[i] = A[i,i-1], main[i],
 * sup1[i] = A[i,i+1], supm[i] = A[i,i+m] (row-aligned, n rows each).  m = 2
 * is the reference's pentadiagonal (offsets -2..+2) bit-for-bit; m >= 3 is
 * the grid generalisation and admits Stone's alpha.  */

/* Pattern-restricted ILU(0) and defect K = L U - A.  Replaces ilu0_penta
 * (iterative.py:62-124) and defect_matrix (186-200).  Every output is a
 * row-aligned array in the call's layout and may be NULL: factors mu (U
 * main), l1 (L(i,i-1)), l2 (L(i,i-m)), phi (U(i,i+1)), psi (U(i,i+m)); defect
 * diagonals at offsets -m, -1, 0, +1, +m, -(m-1), +(m-1) (the last two are
 * zero for m = 2).  Stream-ordered; no allocation. */
int bx_ilu0_f64(const double *subm, const double *sub1, const double *main, const double *sup1,
                const double *supm, double *mu, double *l1, double *l2, double *phi, double *psi,
                double *k_subm, double *k_sub1, double *k_main, double *k_sup1, double *k_supm,
                double *k_subq, double *k_supq, int32_t *status, int32_t *index, int64_t batch,
                int64_t n, int64_t m, double alpha, int64_t ld, int32_t layout, void *workspace,
                size_t workspace_bytes, void *stream);

/* Stone's strongly implicit procedure (Algorithm 1).  Replaces sip_solve
 * (iterative.py:255-308).  tol[batch]: absolute thresholds on ||b - A x||_inf
 * (the loop runs while r >= tol).  x: in = initial guess when use_x0 (else
 * zeros), out = final iterate.  Optional (NULL-able): best_x (the best iterate,
 * as MaxIterationsExceeded.best), iterations, residual, best_residual, history
 * ([batch][max_iter], r after each iteration).  status: OK, ZERO_PIVOT(index),
 * MAX_ITER, DIVERGED (r > 1e6 r0), NOT_GRID (wavefront only).  algo:
 * BX_ALGO_SEQUENTIAL (one thread per system, any band), BX_ALGO_WAVEFRONT
 * (grid-structured systems, n % m == 0, m <= 512: one CTA per system walks the
 * grid's anti-diagonals) or BX_ALGO_AUTO. */
#define BX_ALGO_WAVEFRONT 2
size_t bx_sip_workspace_bytes(int64_t batch, int64_t n, int64_t m);
#define BX_ALGO_AUTO 3  /* wavefront when every system is grid-structured, else sequential (syncs) */
/* Throughput path for grid-structured systems (m a multiple of 32, m <= 512):
 * the same iteration in correction form, x += (LU)^-1 (b - A x), every grid
 * row's recurrence solved by a parallel scan.  Not bit-identical to the
 * reference: iteration counts agree to +-1 and the final residual is below
 * the tolerance (the north-star SIP contract). */
#define BX_ALGO_SCAN 4
int bx_sip_f64(const double *subm, const double *sub1, const double *main, const double *sup1,
               const double *supm, const double *rhs, const double *tol, double *x,
               double *best_x, int64_t *iterations, double *residual, double *best_residual,
               int32_t *status, int32_t *index, double *history, int64_t batch, int64_t n,
               int64_t m, double alpha, int64_t max_iter, int32_t use_x0, int64_t ld,
               int32_t layout, int32_t algo, void *workspace, size_t workspace_bytes,
               void *stream);

/* ---- Hotelling-Bodewig ----------------------------------------------------- */
/* Dense Newton-Schulz inversion X <- X (2I - M X) from X0 = diag(1/m_ii) of the
 * ILU(0)/Stone factors L (unit lower) and U (upper) of every system, stopping
 * when ||I - M X||_inf < tol[s] (hb_invert_dense, inverse.py:94-119, on
 * dense_lower_factor / dense_upper_factor, 72-87).  X X P runs on the FP64
 * tensor cores (mma.sync ... f64, DMMA) over the triangle only.  x_lower /
 * x_upper (may be NULL): [batch][n][n] row-major.  inv_iterations /
 * inv_residual: [2*batch] (L of system s at s, U at batch+s).  status[s]: OK,
 * ZERO_PIVOT (ILU), ZERO_DIAG(index) or MAX_ITER (index -2: the inversion).
 * Host-driven iteration: synchronises the stream. */
size_t bx_hb_workspace_bytes(int64_t batch, int64_t n);
int bx_hb_invert_f64(const double *subm, const double *sub1, const double *main,
                     const double *sup1, const double *supm, const double *tol, double *x_lower,
                     double *x_upper, int64_t *inv_iterations, double *inv_residual,
                     int32_t *status, int32_t *index, int64_t batch, int64_t n, int64_t m,
                     double alpha, int64_t max_iter, int64_t ld, int32_t layout, void *workspace,
                     size_t workspace_bytes, void *stream);

/* hb_invert_dense(m, tol, max_iter) (inverse.py:94-119) on the caller's dense
 * square matrices: m[s] at m + s*m_stride, row i at +i*ldm (row-major).
 * X0 = diag(1/m_ii); P = M X, r = ||I - P||_inf, stop when r < tol[s], else
 * X <- X (2I - P); both products are DMMA GEMMs (agreement with the
 * reference's BLAS products to rounding; counts and statuses are the
 * reference's).  x (may be NULL): the returned inverse (the converged iterate;
 * after max_iter the once-more-updated one, as MaxIterationsExceeded.best).
 * status: OK, ZERO_DIAG(index = first zero m_ii), MAX_ITER.  iterations,
 * residual (the last r), history ([batch][max_iter+1], NaN padded) may be
 * NULL.  Host-driven loop: synchronises the stream.  Workspace:
 * bx_hb_invert_dense_workspace_bytes(batch, n). */
size_t bx_hb_invert_dense_workspace_bytes(int64_t batch, int64_t n);
int bx_hb_invert_dense_f64(const double *m, int64_t n, int64_t ldm, int64_t m_stride, int64_t batch,
                           const double *tol, int64_t max_iter, double *x, int64_t ldx,
                           int64_t x_stride, int64_t *iterations, double *residual,
                           double *history, int32_t *status, int32_t *index, void *workspace,
                           size_t workspace_bytes, void *stream);

/* SIP with the substitutions replaced by the HB inverses (sip_hb_solve,
 * mode="dense", inverse.py:205-302): same contract as bx_sip_f64 plus the
 * inversion counters.  The inversion tolerance is tol[s], as in the reference
 * (inverse.py:235-236); max_inv_iter = 200 there.  Synchronises the stream. */
int bx_sip_hb_f64(const double *subm, const double *sub1, const double *main, const double *sup1,
                  const double *supm, const double *rhs, const double *tol, double *x,
                  double *best_x, int64_t *iterations, double *residual, double *best_residual,
                  int32_t *status, int32_t *index, double *history, int64_t *inv_iterations,
                  double *inv_residual, int64_t batch, int64_t n, int64_t m, double alpha,
                  int64_t max_iter, int64_t max_inv_iter, int32_t use_x0, int64_t ld,
                  int32_t layout, void *workspace, size_t workspace_bytes, void *stream);

/* ---- banded Hotelling-Bodewig (the reference's array implementation) ------ */
/* Workspace (bytes) of both banded entry points for bandwidths up to w_cap. */
size_t bx_hb_banded_workspace_bytes(int64_t batch, int64_t n, int64_t w_cap);

/* hb_invert_banded(factors, side, w, tol, max_iter) (inverse.py:148-195) on
 * one triangular ILU(0) factor per system, bit-for-bit the reference's
 * band-truncated iteration (_band_mul_tri order, inverse.py:122-137).
 * Factor diagonals row-aligned in the call's layout: side 0 = unit-lower L
 * (l1, l2 used), side 1 = upper U (mu, phi, psi used).  tol[batch].
 * x_diags (batch, w+1, n): diagonal r of X at [s][r][k], k < n-r (lower:
 * entry (k+r, k), upper: (k, k+r)).  status: OK, STAGNATED (x = best
 * approximation, iterations/residual of it), MAX_ITER (x = best, residual
 * = last), ZERO_DIAG (index = first zero row of U).  history (may be NULL):
 * [batch][max_iter+1] band residuals, NaN-padded. */
int bx_hb_invert_banded_f64(const double *mu, const double *l1, const double *l2,
                            const double *phi, const double *psi, int32_t side, int64_t w,
                            const double *tol, int64_t max_iter, double *x_diags,
                            int64_t *iterations, double *residual, double *history,
                            int32_t *status, int32_t *index, int64_t batch, int64_t n, int64_t ld,
                            int32_t layout, void *workspace, size_t workspace_bytes, void *stream);

/* sip_hb_solve(mode="banded") (inverse.py:205-302, pentadiagonal, m = 2).
 * hb_bandwidth >= 2: the reference's explicit width (a stagnated inverse
 * is accepted).  hb_bandwidth = 0: auto width 2, 4, 8, ... <= w_cap; a width
 * is accepted once the TRUE residual ||I - M X||_inf is below tol (the
 * reference widens on stagnation of the truncated iteration only, which
 * never triggers -- SURVEY D8).  w_used / inv_iterations / inv_residual /
 * inv_true_residual: [2*batch] (L factors, then U), may be NULL.  Other
 * arguments and outputs as bx_sip_hb_f64. */
int bx_sip_hb_banded_f64(const double *sub2, const double *sub1, const double *main,
                         const double *sup1, const double *sup2, const double *rhs,
                         const double *tol, double *x, double *best_x, int64_t *iterations,
                         double *residual, double *best_residual, int32_t *status,
                         int32_t *index, double *history, int64_t hb_bandwidth, int64_t w_cap,
                         int64_t *w_used, int64_t *inv_iterations, double *inv_residual,
                         double *inv_true_residual, int64_t batch, int64_t n, int64_t max_iter,
                         int64_t max_inv_iter, int32_t use_x0, int64_t ld, int32_t layout,
                         void *workspace, size_t workspace_bytes, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* BANDIX_B200_H */
