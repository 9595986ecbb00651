/*
 * C restatement of the reference's direct and iterative solvers.
 * TEST INFRASTRUCTURE / CPU BASELINE ONLY (see oracle/__init__.py).
 *
 * Same operation order as bandix 0.1.0 (one IEEE rounding per operation;
 * compiled with -ffp-contract=off so no FMA is formed), batched over systems
 * with OpenMP.  Arrays are ROW-ALIGNED and SYSTEM-MAJOR: system s, row i at
 * p[s*ld + i] (the C ABI's BX_LAYOUT_SYSTEM_MAJOR).  Pinned bit-for-bit to
 * the numpy restatement / reference golden vectors by tests/test_oracle_c.py.
 *
 *   ox_ntdm   : tri_factor_recip + tri_solve_recip  (_elim.py:90-122)
 *   ox_npdm   : penta_factor + forward + backward   (_elim.py:30-87)
 *   ox_mnpdm  : mnpdm_sweep                         (_elim.py:125-190)
 *   ox_sip    : ilu0_penta/defect/sip_solve with stride m and Stone alpha
 *               (iterative.py:62-308; m=2, alpha=0 is the reference)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ST_OK 0
#define ST_ZERO_PIVOT 1
#define ST_MAX_ITER 3
#define ST_DIVERGED 4

int ox_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* the host threads of the timed sections (a launcher may export OMP_NUM_THREADS=1) */
void ox_set_threads(int n) {
#ifdef _OPENMP
  omp_set_num_threads(n);
#else
  (void)n;
#endif
}

static void nan_fill(double *x, int64_t n) {
  for (int64_t i = 0; i < n; ++i) x[i] = NAN;
}

void ox_ntdm(const double *d, const double *e, const double *f, const double *b, double *x,
             int32_t *status, int32_t *index, int64_t batch, int64_t n, int64_t ld) {
#pragma omp parallel
  {
    double *rec = (double *)malloc(sizeof(double) * (size_t)n);
#pragma omp for schedule(static)
    for (int64_t s = 0; s < batch; ++s) {
      const double *D = d + s * ld, *E = e + s * ld, *F = f + s * ld, *B = b + s * ld;
      double *X = x + s * ld;
      int32_t st = ST_OK, ix = -1;
      if (E[0] == 0.0) { st = ST_ZERO_PIVOT; ix = 0; }
      else {
        rec[0] = 1.0 / E[0];
        X[0] = B[0];
        for (int64_t i = 1; i < n; ++i) {
          const double li = D[i] * rec[i - 1];
          const double mi = E[i] - li * F[i - 1];
          if (mi == 0.0) { st = ST_ZERO_PIVOT; ix = (int32_t)i; break; }
          rec[i] = 1.0 / mi;
          X[i] = B[i] - li * X[i - 1];
        }
      }
      if (st == ST_OK) {
        double xn = X[n - 1] * rec[n - 1];
        X[n - 1] = xn;
        for (int64_t i = n - 2; i >= 0; --i) {
          xn = (X[i] - F[i] * xn) * rec[i];
          X[i] = xn;
        }
      } else {
        nan_fill(X, n);
      }
      if (status) status[s] = st;
      if (index) index[s] = ix;
    }
    free(rec);
  }
}

/* mod = 0: NPDM (divide by mu); mod = 1: MNPDM (reciprocal pivots, skip zero sub2) */
void ox_penta(int mod, const double *c, const double *d, const double *e, const double *f,
              const double *g, const double *b, double *x, int32_t *status, int32_t *index,
              int64_t *nzout, int64_t batch, int64_t n, int64_t ld) {
#pragma omp parallel
  {
    double *piv = (double *)malloc(sizeof(double) * (size_t)n);
    double *phi = (double *)malloc(sizeof(double) * (size_t)n);
#pragma omp for schedule(static)
    for (int64_t s = 0; s < batch; ++s) {
      const double *C = c + s * ld, *D = d + s * ld, *E = e + s * ld, *F = f + s * ld,
                   *G = g + s * ld, *B = b + s * ld;
      double *X = x + s * ld;
      int32_t st = ST_OK, ix = -1;
      int64_t nz = 0;
      for (int64_t i = 0; i < n && st == ST_OK; ++i) {
        double mi, ph, yi;
        if (i == 0) {
          mi = E[0]; ph = F[0]; yi = B[0];
        } else if (i == 1) {
          const double l1 = mod ? D[1] * piv[0] : D[1] / piv[0];
          mi = E[1] - l1 * phi[0];
          ph = F[1] - l1 * G[0];
          yi = B[1] - l1 * X[0];
        } else if (!mod) {
          const double l2 = C[i] / piv[i - 2];
          const double l1 = (D[i] - l2 * phi[i - 2]) / piv[i - 1];
          mi = E[i] - l2 * G[i - 2] - l1 * phi[i - 1];
          ph = i <= n - 2 ? F[i] - l1 * G[i - 1] : 0.0;
          yi = B[i] - l1 * X[i - 1] - l2 * X[i - 2];
        } else {
          const int has2 = C[i] != 0.0;
          nz += has2;
          const double l2 = C[i] * piv[i - 2];
          const double t = has2 ? D[i] - l2 * phi[i - 2] : D[i];
          const double l1 = t * piv[i - 1];
          double m = E[i] - l1 * phi[i - 1];
          if (has2) m = m - l2 * G[i - 2];
          mi = m;
          ph = i <= n - 2 ? F[i] - l1 * G[i - 1] : 0.0;
          double y = B[i] - l1 * X[i - 1];
          if (has2) y = y - l2 * X[i - 2];
          yi = y;
        }
        if (mi == 0.0) { st = ST_ZERO_PIVOT; ix = (int32_t)i; break; }
        piv[i] = mod ? 1.0 / mi : mi;
        phi[i] = ph;
        X[i] = yi;
      }
      if (st == ST_OK) {
        double x1 = mod ? X[n - 1] * piv[n - 1] : X[n - 1] / piv[n - 1];
        X[n - 1] = x1;
        double num = X[n - 2] - phi[n - 2] * x1;
        double x0 = mod ? num * piv[n - 2] : num / piv[n - 2];
        X[n - 2] = x0;
        double x2 = x1;
        x1 = x0;
        for (int64_t i = n - 3; i >= 0; --i) {
          num = X[i] - phi[i] * x1 - G[i] * x2;
          const double xi = mod ? num * piv[i] : num / piv[i];
          X[i] = xi;
          x2 = x1;
          x1 = xi;
        }
      } else {
        nan_fill(X, n);
      }
      if (status) status[s] = st;
      if (index) index[s] = ix;
      if (nzout) nzout[s] = nz;
    }
    free(piv);
    free(phi);
  }
}

/* ------------------------------------------------------------------------ */
/* SIP with stride m (row-aligned: lm[i] = A[i,i-m], l1[i] = A[i,i-1],
 * e[i], u1[i] = A[i,i+1], um[i] = A[i,i+m]); tol per system.               */
/* ------------------------------------------------------------------------ */
typedef struct {
  double *mu, *l1, *l2, *phi, *psi;              /* factors, row-aligned */
  double *k[7];                                  /* defect: -m,-1,0,+1,+m,-(m-1),+(m-1) */
} sip_ws;

static int ilu0_1(const double *a2, const double *a1, const double *e, const double *c1,
                  const double *c2, int64_t n, int64_t m, double alpha, sip_ws *w, int32_t *ix) {
  double *mu = w->mu, *L1 = w->l1, *L2 = w->l2, *phi = w->phi, *psi = w->psi;
  for (int64_t i = 0; i < n; ++i) {
    const int has2 = i >= m && a2[i] != 0.0;
    const int has1 = i >= 1 && a1[i] != 0.0;
    double li2 = 0.0, li1 = 0.0, mi;
    if (m == 2) {
      if (has2) li2 = a2[i] / mu[i - 2];
      if (has1) {
        double t = a1[i];
        if (has2) t = t - li2 * phi[i - 2];
        li1 = t / mu[i - 1];
      }
      mi = e[i];
      if (has2) mi = mi - li2 * psi[i - 2];
      if (has1) mi = mi - li1 * phi[i - 1];
      if (i <= n - 2) {
        double fi = c1[i];
        if (fi != 0.0 && has1) fi = fi - li1 * psi[i - 1];
        phi[i] = fi;
      } else {
        phi[i] = 0.0;
      }
      psi[i] = i <= n - 3 ? c2[i] : 0.0;
    } else {
      if (has2) li2 = a2[i] / (alpha == 0.0 ? mu[i - m] : mu[i - m] + alpha * phi[i - m]);
      if (has1) li1 = a1[i] / (alpha == 0.0 ? mu[i - 1] : mu[i - 1] + alpha * psi[i - 1]);
      mi = e[i];
      if (has2) mi = mi - li2 * psi[i - m];
      if (has1) mi = mi - li1 * phi[i - 1];
      if (alpha != 0.0) {
        double comp = 0.0;
        if (has2) comp = comp + li2 * phi[i - m];
        if (has1) comp = comp + li1 * psi[i - 1];
        mi = mi + alpha * comp;
      }
      if (i <= n - 2) {
        double fi = c1[i];
        if (alpha != 0.0 && fi != 0.0 && has2) fi = fi - alpha * (li2 * phi[i - m]);
        phi[i] = fi;
      } else {
        phi[i] = 0.0;
      }
      if (i <= n - m - 1) {
        double gi = c2[i];
        if (alpha != 0.0 && gi != 0.0 && has1) gi = gi - alpha * (li1 * psi[i - 1]);
        psi[i] = gi;
      } else {
        psi[i] = 0.0;
      }
    }
    if (mi == 0.0) { *ix = (int32_t)i; return ST_ZERO_PIVOT; }
    mu[i] = mi;
    L1[i] = has1 ? li1 : 0.0;
    L2[i] = has2 ? li2 : 0.0;
  }
  return ST_OK;
}

static void defect_1(const double *a2, const double *a1, const double *e, const double *c1,
                     const double *c2, int64_t n, int64_t m, sip_ws *w) {
  const double *mu = w->mu, *l1 = w->l1, *l2 = w->l2, *phi = w->phi, *psi = w->psi;
  double **k = w->k;
  for (int64_t i = 0; i < n; ++i) {
    double pm = i >= m ? l2[i] * mu[i - m] : 0.0;
    double p_1 = i >= 1 ? l1[i] * mu[i - 1] : 0.0;
    if (m == 2 && i >= 2) p_1 = p_1 + l2[i] * phi[i - 2];
    double p0 = mu[i];
    if (i >= 1) p0 = p0 + l1[i] * phi[i - 1];
    if (i >= m) p0 = p0 + l2[i] * psi[i - m];
    double p1 = i <= n - 2 ? phi[i] : 0.0;
    if (m == 2 && i >= 1 && i <= n - 2) p1 = p1 + l1[i] * psi[i - 1];
    double pp = i <= n - m - 1 ? psi[i] : 0.0;
    k[0][i] = pm - (i >= m ? a2[i] : 0.0);
    k[1][i] = p_1 - (i >= 1 ? a1[i] : 0.0);
    k[2][i] = p0 - e[i];
    k[3][i] = p1 - (i <= n - 2 ? c1[i] : 0.0);
    k[4][i] = pp - (i <= n - m - 1 ? c2[i] : 0.0);
    if (m != 2) {
      k[5][i] = i >= m ? l2[i] * phi[i - m] : 0.0;
      k[6][i] = (i >= 1 && i <= n - m) ? l1[i] * psi[i - 1] : 0.0;
    }
  }
}

/* acc from 0: main, -1, +1, -m, +m [, -(m-1), +(m-1)] (iterative.py:213-221) */
static void sweep_1(const double *lm, const double *l1, const double *e, const double *u1,
                    const double *um, const double *lq, const double *uq, int64_t n, int64_t m,
                    const double *x, double *out) {
  for (int64_t i = 0; i < n; ++i) {
    double acc = 0.0 + e[i] * x[i];
    if (i >= 1) acc = acc + l1[i] * x[i - 1];
    if (i <= n - 2) acc = acc + u1[i] * x[i + 1];
    if (i >= m) acc = acc + lm[i] * x[i - m];
    if (i + m <= n - 1) acc = acc + um[i] * x[i + m];
    if (lq) {
      const int64_t q = m - 1;
      if (i >= q) acc = acc + lq[i] * x[i - q];
      if (i + q <= n - 1) acc = acc + uq[i] * x[i + q];
    }
    out[i] = acc;
  }
}

void ox_sip(const double *A2, const double *A1, const double *E, const double *C1,
            const double *C2, const double *Bv, const double *tol, double *X, double *best_x,
            int64_t *iters, double *res, double *best_res, int32_t *status, int32_t *index,
            int64_t batch, int64_t n, int64_t ld, int64_t m, double alpha, int64_t max_iter) {
#pragma omp parallel
  {
    sip_ws w;
    double *buf = (double *)calloc((size_t)n * 15, sizeof(double));
    w.mu = buf; w.l1 = buf + n; w.l2 = buf + 2 * n; w.phi = buf + 3 * n; w.psi = buf + 4 * n;
    for (int j = 0; j < 7; ++j) w.k[j] = buf + (5 + j) * n;
    double *nr = buf + 12 * n, *y = buf + 13 * n, *xn = buf + 14 * n;
#pragma omp for schedule(dynamic, 1)
    for (int64_t s = 0; s < batch; ++s) {
      const double *a2 = A2 + s * ld, *a1 = A1 + s * ld, *e = E + s * ld, *c1 = C1 + s * ld,
                   *c2 = C2 + s * ld, *b = Bv + s * ld;
      double *x = X + s * ld, *bx = best_x + s * ld;
      int32_t ix = -1;
      int st = ilu0_1(a2, a1, e, c1, c2, n, m, alpha, &w, &ix);
      int64_t k = 0;
      double r = NAN, bestr = NAN;
      if (st == ST_OK) {
        defect_1(a2, a1, e, c1, c2, n, m, &w);
        const double *kq = m != 2 ? w.k[5] : NULL, *kp = m != 2 ? w.k[6] : NULL;
        for (int64_t i = 0; i < n; ++i) x[i] = 0.0;
        sweep_1(a2, a1, e, c1, c2, NULL, NULL, n, m, x, nr);
        r = 0.0;
        for (int64_t i = 0; i < n; ++i) { double v = fabs(b[i] - nr[i]); r = v > r || v != v ? v : r; }
        const double r0 = r;
        bestr = r;
        memcpy(bx, x, sizeof(double) * (size_t)n);
        while (r >= tol[s]) {
          if (k >= max_iter) { st = ST_MAX_ITER; break; }
          sweep_1(w.k[0], w.k[1], w.k[2], w.k[3], w.k[4], kq, kp, n, m, x, nr);
          for (int64_t i = 0; i < n; ++i) nr[i] = nr[i] + b[i];
          /* forward: y_i = (v_i - l1 y_{i-1}) - l2 y_{i-m} */
          y[0] = nr[0];
          for (int64_t i = 1; i < n; ++i) {
            double t = nr[i] - w.l1[i] * y[i - 1];
            if (i >= m) t = t - w.l2[i] * y[i - m];
            y[i] = t;
          }
          /* backward: x_i = ((y_i - phi x_{i+1}) - psi x_{i+m}) / mu */
          xn[n - 1] = y[n - 1] / w.mu[n - 1];
          for (int64_t i = n - 2; i >= 0; --i) {
            double t = y[i] - w.phi[i] * xn[i + 1];
            if (i + m <= n - 1) t = t - w.psi[i] * xn[i + m];
            xn[i] = t / w.mu[i];
          }
          memcpy(x, xn, sizeof(double) * (size_t)n);
          sweep_1(a2, a1, e, c1, c2, NULL, NULL, n, m, x, nr);
          r = 0.0;
          for (int64_t i = 0; i < n; ++i) { double v = fabs(b[i] - nr[i]); r = v > r || v != v ? v : r; }
          ++k;
          if (r < bestr) { bestr = r; memcpy(bx, x, sizeof(double) * (size_t)n); }
          if (r0 > 0 && r > 1e6 * r0) { st = ST_DIVERGED; break; }
        }
      }
      if (iters) iters[s] = k;
      if (res) res[s] = r;
      if (best_res) best_res[s] = bestr;
      if (status) status[s] = st;
      if (index) index[s] = ix;
    }
    free(buf);
  }
}
