/*
 * dpt_oracle.c -- TEST INFRASTRUCTURE ONLY.  CPU restatement of the reference's
 * DPT iteration path in real FP64, used as the parity checker for the CUDA
 * path.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg
 * may load it; the product never links or calls it.
 *
 * Parity pin: for real inputs the reference's std::complex<double> arithmetic
 * reduces to exactly these real operations (imaginary parts stay 0, complex
 * abs = hypot(x, 0) = |x|, complex products (a+0i)(b+0i) have real part
 * fl(a*b) - 0).  tests/test_oracle.py checks this file BIT-EXACT against the
 * reference library itself (oracle/_ref, compiled from /root/reference/proj/src)
 * and against the reference's known-answer tests.
 * Compile with -ffp-contract=off so no FMA changes a rounding.
 *
 * Every function cites the reference lines it restates (paths relative to
 * /root/reference/proj).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "dpt_oracle.h"

#define TINY_DEN 1e-300 /* kTinyDen, src/dpt.cpp:18 */

static double dmax(double a, double b) { return (a < b) ? b : a; } /* std::max */

/* ------------------------------------------------------------------------ */
/* Products.  P = A * delta_t, the reference's matmul(Dense, Dense|Sparse)   */
/* with delta_t = transpose(delta) cached by make_problem                    */
/* (src/partition.cpp:12-21, src/matrix.cpp:72-90, :130-158).               */
/* ------------------------------------------------------------------------ */

typedef struct {
  int64_t n;
  int kind; /* ORC_DENSE / ORC_CSR */
  const double* dense_t; /* delta_t row-major (owned copy) */
  int64_t* t_rowptr;     /* CSR of delta_t (owned) */
  int32_t* t_cols;
  double* t_vals;
  const double* dense;   /* delta row-major (borrowed) */
  const int64_t* rowptr; /* CSR of delta (borrowed) */
  const int32_t* cols;
  const double* vals;
} orc_delta;

static double* orc_transpose_dense(int64_t n, const double* a) {
  double* t = (double*)malloc(sizeof(double) * (size_t)n * (size_t)n);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) t[j * n + i] = a[i * n + j];
  return t;
}

/* transpose(SparseMatrix): triplets (col, row, v) through from_triplets,
 * i.e. rows of delta_t sorted by column (src/matrix.cpp:28-53, :80-86).
 * A counting sort over rows of delta visited in order yields sorted columns. */
static void orc_transpose_csr(int64_t n, const int64_t* rp, const int32_t* cl, const double* vl,
                              int64_t** trp, int32_t** tcl, double** tvl) {
  int64_t nnz = rp[n];
  int64_t* r = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  int32_t* c = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nnz ? nnz : 1));
  double* v = (double*)malloc(sizeof(double) * (size_t)(nnz ? nnz : 1));
  int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
  for (int64_t p = 0; p < nnz; ++p) r[cl[p] + 1]++;
  for (int64_t i = 0; i < n; ++i) r[i + 1] += r[i];
  for (int64_t i = 0; i < n; ++i) fill[i] = r[i];
  for (int64_t i = 0; i < n; ++i)
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
      int64_t dst = fill[cl[p]]++;
      c[dst] = (int32_t)i;
      v[dst] = vl[p];
    }
  free(fill);
  *trp = r;
  *tcl = c;
  *tvl = v;
}

static void orc_delta_init(orc_delta* D, const orc_problem* p) {
  memset(D, 0, sizeof(*D));
  D->n = p->n;
  D->kind = p->kind;
  if (p->kind == ORC_DENSE) {
    D->dense = p->delta;
    D->dense_t = orc_transpose_dense(p->n, p->delta);
  } else {
    D->rowptr = p->rowptr;
    D->cols = p->cols;
    D->vals = p->vals;
    orc_transpose_csr(p->n, p->rowptr, p->cols, p->vals, &D->t_rowptr, &D->t_cols, &D->t_vals);
  }
}

static void orc_delta_free(orc_delta* D) {
  free((void*)D->dense_t);
  free(D->t_rowptr);
  free(D->t_cols);
  free(D->t_vals);
}

/* matmul(Dense a, Dense b) i-k-j with the a(i,k)==0 skip, src/matrix.cpp:130-143;
 * matmul(Dense a, Sparse b), src/matrix.cpp:145-158.  rows = number of rows of a. */
static void orc_matmul(const orc_delta* D, int64_t rows, const double* a, double* c) {
  const int64_t n = D->n;
  memset(c, 0, sizeof(double) * (size_t)rows * (size_t)n);
  for (int64_t i = 0; i < rows; ++i) {
    double* ci = c + i * n;
    const double* ai = a + i * n;
    for (int64_t k = 0; k < n; ++k) {
      const double aik = ai[k];
      if (aik == 0.0) continue;
      if (D->kind == ORC_DENSE) {
        const double* bk = D->dense_t + k * n;
        for (int64_t j = 0; j < n; ++j) ci[j] += aik * bk[j];
      } else {
        for (int64_t p = D->t_rowptr[k]; p < D->t_rowptr[k + 1]; ++p)
          ci[D->t_cols[p]] += aik * D->t_vals[p];
      }
    }
  }
}

/* matvec(delta, x): dense src/matrix.cpp:203-213, CSR :215-225 (NOT transposed). */
static void orc_matvec(const orc_delta* D, const double* x, double* y) {
  const int64_t n = D->n;
  for (int64_t i = 0; i < n; ++i) {
    double s = 0.0;
    if (D->kind == ORC_DENSE) {
      const double* ai = D->dense + i * n;
      for (int64_t j = 0; j < n; ++j) s += ai[j] * x[j];
    } else {
      for (int64_t p = D->rowptr[i]; p < D->rowptr[i + 1]; ++p) s += D->vals[p] * x[D->cols[p]];
    }
    y[i] = s;
  }
}

/* ------------------------------------------------------------------------ */
/* Gap policy: spectral_spread / degeneracy_threshold / build_theta /        */
/* build_gap_row (src/partition.cpp:42-96).                                  */
/* ------------------------------------------------------------------------ */

double orc_spectral_spread(int64_t n, const double* d) {
  if (n == 0) return 0.0;
  double lo = d[0], hi = d[0];
  for (int64_t i = 0; i < n; ++i) { /* std::min / std::max order, :45-50 */
    lo = (d[i] < lo) ? d[i] : lo;
    hi = (hi < d[i]) ? d[i] : hi;
  }
  return hypot(hi - lo, 0.0); /* imaginary box is {0} for real levels */
}

static double orc_threshold(int64_t n, const double* d, double tol) {
  return tol * dmax(1.0, orc_spectral_spread(n, d));
}

/* build_theta's degeneracy scan (src/partition.cpp:69-81): first (i,j) in
 * row-major order with |d_i - d_j| <= thresh.  O(n^2) like the reference. */
int orc_check_degenerate(int64_t n, const double* d, double tol, int64_t* bi, int64_t* bj) {
  const double thresh = orc_threshold(n, d, tol);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) {
      if (i == j) continue;
      if (fabs(d[i] - d[j]) <= thresh) {
        *bi = i;
        *bj = j;
        return 1;
      }
    }
  return 0;
}

/* build_gap_row (src/partition.cpp:83-96). */
static int orc_gap_row(int64_t n, const double* d, int64_t row, double tol, double* g, int64_t* bj) {
  const double thresh = orc_threshold(n, d, tol);
  for (int64_t m = 0; m < n; ++m) {
    if (m == row) {
      g[m] = 0.0;
      continue;
    }
    const double gap = d[row] - d[m];
    if (fabs(gap) <= thresh) {
      *bj = m;
      return 1;
    }
    g[m] = 1.0 / gap;
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Residuals (src/dpt.cpp:23-58) and the cycle test within_tol (:60-79).    */
/* ------------------------------------------------------------------------ */

/* residuals_of: rows [0,rows) of a (n columns), eig_i = d[row0+i] + lam p_ii. */
static double orc_residuals_of(int64_t n, int64_t rows, int64_t row0, const double* d, double lam,
                               const double* a, const double* p, double* eig, double* res) {
  double worst = 0.0;
  for (int64_t i = 0; i < rows; ++i) {
    const int64_t gi = row0 + i;
    const double eps = d[gi] + lam * p[i * n + gi];
    eig[i] = eps;
    double num = 0.0, den = 0.0;
    for (int64_t m = 0; m < n; ++m) {
      const double r = (d[m] - eps) * a[i * n + m] + lam * p[i * n + m];
      num = dmax(num, fabs(r));
      den = dmax(den, fabs(a[i * n + m]));
    }
    res[i] = num / dmax(den, TINY_DEN);
    worst = dmax(worst, res[i]);
  }
  return worst;
}

static double orc_residual_single(int64_t n, const double* d, double lam, const double* z,
                                  const double* w, double eps) {
  double num = 0.0, den = 0.0;
  for (int64_t m = 0; m < n; ++m) {
    const double r = (d[m] - eps) * z[m] + lam * w[m];
    num = dmax(num, fabs(r));
    den = dmax(den, fabs(z[m]));
  }
  return num / dmax(den, TINY_DEN);
}

static int orc_within_tol(size_t count, const double* a, const double* b, double tol) {
  for (size_t i = 0; i < count; ++i) {
    const double dr = a[i] - b[i];
    if (fabs(dr) >= tol) return 0; /* imaginary difference is 0 < tol */
  }
  return 1;
}

static int orc_all_finite(size_t count, const double* a) {
  for (size_t i = 0; i < count; ++i)
    if (!isfinite(a[i])) return 0;
  return 1;
}

static double orc_max_abs(size_t count, const double* a) {
  double m = 0.0;
  for (size_t i = 0; i < count; ++i) m = dmax(m, fabs(a[i]));
  return m;
}

/* effective_window (src/dpt.cpp:83-90). */
int orc_effective_window(int requested, int64_t n) {
  if (requested <= 0) return 0;
  const double entries = (double)n * (double)n;
  const double cap = 4.0e6 / dmax(entries, 1.0);
  int win = requested;
  if (cap < win) win = (int)cap;
  return win < 2 ? 0 : win;
}

/* ------------------------------------------------------------------------ */
/* The full map loop run_full (src/dpt.cpp:92-192).                          */
/* Rows [row0, row0 + rows) only when rows < n: the map is row-independent,  */
/* so a row slice of the run is bit-identical to the same rows of the full   */
/* run UNTIL a global decision (step / max / residual are maxima over all    */
/* rows).  The slice mode exists for the bench's bounded CPU sample and for  */
/* the sharding tests; solves use rows == n.                                 */
/* ------------------------------------------------------------------------ */

int orc_iterate_full(const orc_problem* p, const orc_options* o, int ramped, double alpha,
                     double* a_out, double* eig_out, double* res_out, orc_report* rep,
                     double* trace_step, double* trace_res) {
  const int64_t n = p->n;
  const size_t nn = (size_t)n * (size_t)n;
  const double lam = p->lambda;
  const double cycle_margin = 1e3 * o->tol;
  int64_t di, dj;
  memset(rep, 0, sizeof(*rep));
  if (orc_check_degenerate(n, p->d, o->degeneracy_tol, &di, &dj)) {
    rep->degenerate_i = di;
    rep->degenerate_j = dj;
    return ORC_ERR_DEGENERATE;
  }
  /* theta(i,j) = 1.0 / (d_i - d_j), zero diagonal (src/partition.cpp:69-81) */
  double* theta = (double*)malloc(sizeof(double) * nn);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) theta[i * n + j] = (i == j) ? 0.0 : 1.0 / (p->d[i] - p->d[j]);

  orc_delta D;
  orc_delta_init(&D, p);
  const int win = orc_effective_window(o->cycle_window, n);
  double* a = (double*)calloc(nn, sizeof(double));
  double* an = (double*)malloc(sizeof(double) * nn);
  double* pm = (double*)malloc(sizeof(double) * nn);
  double* pn = (double*)malloc(sizeof(double) * nn);
  double* eig = (double*)malloc(sizeof(double) * (size_t)n);
  double* res = (double*)malloc(sizeof(double) * (size_t)n);
  double** window = (double**)calloc((size_t)(win > 0 ? win : 1), sizeof(double*));
  int wlen = 0;
  for (int64_t i = 0; i < n; ++i) a[i * n + i] = 1.0;
  orc_matmul(&D, n, a, pm); /* pmat = matmul(I, delta_t), :100 */

  double step = 0.0;
  int status = -1, iters = 0;
  const double* fin_a = NULL;
  int fin_have_eig = 0;
  for (int k = 1; k <= o->max_iter; ++k) {
    const double lam_k = ramped ? lam * (1.0 - pow(alpha, (double)(k - 1))) : lam; /* :131-132 */
    const int settled = !ramped || fabs(lam_k - lam) <= o->tol * fabs(lam);         /* :133-134 */
    for (int64_t i = 0; i < n; ++i) { /* :136-144 */
      const double pii = pm[i * n + i];
      for (int64_t j = 0; j < n; ++j)
        an[i * n + j] = (i == j) ? 1.0 : (lam_k * theta[i * n + j]) * (pm[i * n + j] - pii * a[i * n + j]);
    }
    step = 0.0; /* max_abs_diff, :145 */
    for (size_t e = 0; e < nn; ++e) step = dmax(step, fabs(an[e] - a[e]));
    if (!orc_all_finite(nn, an) || orc_max_abs(nn, an) > o->divergence_threshold) { /* :147-150 */
      status = ORC_DIVERGED;
      iters = k;
      fin_a = an;
      break;
    }
    orc_matmul(&D, n, an, pn); /* :152 */
    double max_res = NAN;
    if (trace_step) { /* trace set: residuals every iteration, :153-157 */
      max_res = orc_residuals_of(n, n, 0, p->d, lam, an, pn, eig, res);
      trace_step[k - 1] = step;
      trace_res[k - 1] = max_res;
    }
    if (settled && step < o->tol) { /* :159-170 */
      if (!trace_step) max_res = orc_residuals_of(n, n, 0, p->d, lam, an, pn, eig, res);
      if (max_res < o->residual_tol) {
        status = ORC_CONVERGED;
        iters = k;
        fin_a = an;
        fin_have_eig = 1;
        break;
      }
    } else if (win > 0 && settled && step > cycle_margin) { /* :171-179 */
      int hit = 0;
      for (int w = 0; w < wlen && !hit; ++w) hit = orc_within_tol(nn, an, window[w], o->tol);
      if (hit) {
        status = ORC_BOUNDED;
        iters = k;
        fin_a = an;
        orc_residuals_of(n, n, 0, p->d, lam, an, pn, eig, res);
        fin_have_eig = 1;
        break;
      }
    }
    if (win > 0) { /* window.push_front(a), pop_back beyond win-1, :181-184 */
      double* old = (wlen == win - 1) ? window[--wlen] : (double*)malloc(sizeof(double) * nn);
      memcpy(old, a, sizeof(double) * nn);
      memmove(window + 1, window, sizeof(double*) * (size_t)wlen);
      window[0] = old;
      wlen++;
    }
    double* t = a; a = an; an = t; /* a = move(an) */
    t = pm; pm = pn; pn = t;       /* pmat = move(pn) */
  }
  if (status < 0) { /* MaxIterations with read-offs of the final (a, pmat), :189-191 */
    status = ORC_MAXITER;
    iters = o->max_iter;
    fin_a = a;
    orc_residuals_of(n, n, 0, p->d, lam, a, pm, eig, res);
    fin_have_eig = 1;
  }
  memcpy(a_out, fin_a, sizeof(double) * nn);
  for (int64_t i = 0; i < n; ++i) {
    eig_out[i] = fin_have_eig ? eig[i] : NAN; /* Diverged: NaN read-offs, :114-125 */
    res_out[i] = fin_have_eig ? res[i] : NAN;
  }
  rep->status = status;
  rep->iterations = iters;
  rep->step_norm = step;
  for (int w = 0; w < wlen; ++w) free(window[w]);
  free(window);
  free(a); free(an); free(pm); free(pn); free(eig); free(res); free(theta);
  orc_delta_free(&D);
  return ORC_OK;
}

/* step_full (src/dpt.cpp:311-327) with theta computed from d. */
int orc_step_full(const orc_problem* p, const double* a, double lam, double* out) {
  const int64_t n = p->n;
  orc_delta D;
  orc_delta_init(&D, p);
  double* pm = (double*)malloc(sizeof(double) * (size_t)n * (size_t)n);
  orc_matmul(&D, n, a, pm);
  for (int64_t i = 0; i < n; ++i) {
    const double pii = pm[i * n + i];
    for (int64_t j = 0; j < n; ++j) {
      const double th = (i == j) ? 0.0 : 1.0 / (p->d[i] - p->d[j]);
      out[i * n + j] = (i == j) ? 1.0 : (lam * th) * (pm[i * n + j] - pii * a[i * n + j]);
    }
  }
  free(pm);
  orc_delta_free(&D);
  return ORC_OK;
}

/* iterate_fixed (src/dpt.cpp:381-387): exactly k steps from I, no gates. */
int orc_iterate_fixed(const orc_problem* p, int k, double lam, double* a_out) {
  const int64_t n = p->n;
  const size_t nn = (size_t)n * (size_t)n;
  int64_t di, dj;
  if (k < 0) return ORC_ERR_INVALID;
  if (orc_check_degenerate(n, p->d, 1e-12, &di, &dj)) return ORC_ERR_DEGENERATE;
  double* a = (double*)calloc(nn, sizeof(double));
  double* b = (double*)malloc(sizeof(double) * nn);
  for (int64_t i = 0; i < n; ++i) a[i * n + i] = 1.0;
  for (int s = 0; s < k; ++s) {
    orc_step_full(p, a, lam, b);
    double* t = a; a = b; b = t;
  }
  memcpy(a_out, a, sizeof(double) * nn);
  free(a);
  free(b);
  return ORC_OK;
}

/* Row slice of the map, the unit the bench's bounded CPU sample times:
 * out rows [row0,row0+rows) of F(a) given those rows of a (n columns). */
int orc_step_rows(const orc_problem* p, int64_t row0, int64_t rows, const double* a, double lam,
                  double* out) {
  const int64_t n = p->n;
  orc_delta D;
  orc_delta_init(&D, p);
  double* pm = (double*)malloc(sizeof(double) * (size_t)rows * (size_t)n);
  orc_matmul(&D, rows, a, pm);
  for (int64_t i = 0; i < rows; ++i) {
    const int64_t gi = row0 + i;
    const double pii = pm[i * n + gi];
    for (int64_t j = 0; j < n; ++j) {
      const double th = (gi == j) ? 0.0 : 1.0 / (p->d[gi] - p->d[j]);
      out[i * n + j] = (gi == j) ? 1.0 : (lam * th) * (pm[i * n + j] - pii * a[i * n + j]);
    }
  }
  free(pm);
  orc_delta_free(&D);
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Row map: run_single (src/dpt.cpp:194-293), step_single (:329-345),        */
/* eigenvalue_of (:358-365), dominant_eigenpair (:399-438).                  */
/* ------------------------------------------------------------------------ */

static int orc_run_single(const orc_problem* p, const orc_delta* D, int64_t row, const double* g,
                          const orc_options* o, double ramp_alpha, double* z_out,
                          orc_single_report* rep, double* trace_step, double* trace_res) {
  const int64_t n = p->n;
  const double lam = p->lambda;
  const int ramped = ramp_alpha > 0.0;
  const double cycle_margin = 1e3 * o->tol;
  double* z = (double*)calloc((size_t)n, sizeof(double));
  double* zn = (double*)malloc(sizeof(double) * (size_t)n);
  double* w = (double*)malloc(sizeof(double) * (size_t)n);
  double* wn = (double*)malloc(sizeof(double) * (size_t)n);
  const int win = o->cycle_window >= 2 ? o->cycle_window : 0; /* :207 */
  double** window = (double**)calloc((size_t)(win > 0 ? win : 1), sizeof(double*));
  int wlen = 0;
  z[row] = 1.0;
  orc_matvec(D, z, w);
  double step = 0.0;
  int status = -1, iters = 0;
  const double* fz = NULL;
  const double* fw = NULL;
  double eps = 0.0, res = NAN;
  int have = 0;
  for (int k = 1; k <= o->max_iter; ++k) {
    const double lam_k = ramped ? lam * (1.0 - pow(ramp_alpha, (double)(k - 1))) : lam;
    const int settled = !ramped || fabs(lam_k - lam) <= o->tol * fabs(lam);
    const double wr = w[row];
    for (int64_t m = 0; m < n; ++m) /* :239-244 */
      zn[m] = (m == row) ? 1.0 : (lam_k * g[m]) * (w[m] - wr * z[m]);
    step = 0.0;
    for (int64_t m = 0; m < n; ++m) step = dmax(step, fabs(zn[m] - z[m]));
    if (!orc_all_finite((size_t)n, zn) || orc_max_abs((size_t)n, zn) > o->divergence_threshold) {
      status = ORC_DIVERGED; /* :249-252 */
      iters = k;
      fz = zn;
      break;
    }
    orc_matvec(D, zn, wn); /* :254 */
    res = NAN;
    if (trace_step || (settled && step < o->tol)) { /* :255-261 */
      eps = p->d[row] + lam * wn[row];
      res = orc_residual_single(n, p->d, lam, zn, wn, eps);
    }
    if (trace_step) {
      trace_step[k - 1] = step;
      trace_res[k - 1] = res;
    }
    if (settled && step < o->tol) {
      if (res < o->residual_tol) {
        status = ORC_CONVERGED;
        iters = k;
        fz = zn;
        have = 1;
        break;
      }
    } else if (win > 0 && settled && step > cycle_margin) {
      int hit = 0;
      for (int q = 0; q < wlen && !hit; ++q) hit = orc_within_tol((size_t)n, zn, window[q], o->tol);
      if (hit) {
        status = ORC_BOUNDED;
        iters = k;
        fz = zn;
        fw = wn;
        break;
      }
    }
    if (win > 0) {
      double* old = (wlen == win - 1) ? window[--wlen] : (double*)malloc(sizeof(double) * (size_t)n);
      memcpy(old, z, sizeof(double) * (size_t)n);
      memmove(window + 1, window, sizeof(double*) * (size_t)wlen);
      window[0] = old;
      wlen++;
    }
    double* t = z; z = zn; zn = t;
    t = w; w = wn; wn = t;
  }
  if (status < 0) {
    status = ORC_MAXITER;
    iters = o->max_iter;
    fz = z;
    fw = w;
  }
  if (!have) { /* finish(): read-offs unless Diverged or non-finite, :217-230 */
    if (status != ORC_DIVERGED && orc_all_finite((size_t)n, fz)) {
      eps = p->d[row] + lam * fw[row];
      res = orc_residual_single(n, p->d, lam, fz, fw, eps);
    } else {
      eps = NAN;
      res = NAN;
    }
  }
  memcpy(z_out, fz, sizeof(double) * (size_t)n);
  rep->status = status;
  rep->iterations = iters;
  rep->step_norm = step;
  rep->eigenvalue = eps;
  rep->residual = res;
  for (int q = 0; q < wlen; ++q) free(window[q]);
  free(window);
  free(z); free(zn); free(w); free(wn);
  return ORC_OK;
}

int orc_iterate_single(const orc_problem* p, int64_t row, const orc_options* o, double ramp_alpha,
                       double* z_out, orc_single_report* rep, double* trace_step,
                       double* trace_res) {
  const int64_t n = p->n;
  memset(rep, 0, sizeof(*rep));
  if (row < 0 || row >= n) return ORC_ERR_SHAPE;                 /* :392 */
  if (!(ramp_alpha >= 0.0) || ramp_alpha >= 1.0) return ORC_ERR_INVALID; /* :393-394 */
  double* g = (double*)malloc(sizeof(double) * (size_t)n);
  int64_t bj;
  if (orc_gap_row(n, p->d, row, o->degeneracy_tol, g, &bj)) {
    rep->degenerate_i = row;
    rep->degenerate_j = bj;
    free(g);
    return ORC_ERR_DEGENERATE;
  }
  orc_delta D;
  orc_delta_init(&D, p);
  int rc = orc_run_single(p, &D, row, g, o, ramp_alpha, z_out, rep, trace_step, trace_res);
  orc_delta_free(&D);
  free(g);
  return rc;
}

int orc_dominant_eigenpair(const orc_problem* p, const orc_options* o, double* z_chart,
                           double* z_unit, orc_single_report* rep, int64_t* row_out) {
  const int64_t n = p->n;
  memset(rep, 0, sizeof(*rep));
  if (n == 0) return ORC_ERR_SHAPE;
  int64_t best = 0;
  for (int64_t i = 1; i < n; ++i)
    if (p->d[i] > p->d[best]) best = i;
  if (n > 1) {
    int64_t runner = best == 0 ? 1 : 0;
    for (int64_t i = 0; i < n; ++i) {
      if (i == best) continue;
      if (p->d[i] > p->d[runner]) runner = i;
    }
    const double thr = orc_threshold(n, p->d, o->degeneracy_tol);
    if (p->d[best] - p->d[runner] < thr) {
      rep->degenerate_i = best;
      rep->degenerate_j = runner;
      return ORC_ERR_DEGENERATE;
    }
  }
  *row_out = best;
  int rc = orc_iterate_single(p, best, o, 0.0, z_chart, rep, NULL, NULL);
  if (rc != ORC_OK) return rc;
  double s = 0.0; /* vec_two_norm, src/matrix.cpp:372-376 */
  for (int64_t m = 0; m < n; ++m) s += z_chart[m] * z_chart[m];
  const double nrm = sqrt(s);
  for (int64_t m = 0; m < n; ++m)
    z_unit[m] = (nrm > 0.0 && isfinite(nrm)) ? z_chart[m] / nrm : z_chart[m];
  return ORC_OK;
}

int orc_step_single(const orc_problem* p, const double* z, int64_t row, double lam, double* out) {
  const int64_t n = p->n;
  if (row < 0 || row >= n) return ORC_ERR_SHAPE;
  orc_delta D;
  orc_delta_init(&D, p);
  double* w = (double*)malloc(sizeof(double) * (size_t)n);
  orc_matvec(&D, z, w);
  const double wr = w[row];
  for (int64_t m = 0; m < n; ++m) {
    const double g = (m == row) ? 0.0 : 1.0 / (p->d[row] - p->d[m]);
    out[m] = (m == row) ? 1.0 : (lam * g) * (w[m] - wr * z[m]);
  }
  free(w);
  orc_delta_free(&D);
  return ORC_OK;
}

int orc_eigenvalue_of(const orc_problem* p, const double* z, int64_t row, double lam, double* out) {
  const int64_t n = p->n;
  if (row < 0 || row >= n) return ORC_ERR_SHAPE;
  orc_delta D;
  orc_delta_init(&D, p);
  double* w = (double*)malloc(sizeof(double) * (size_t)n);
  orc_matvec(&D, z, w);
  *out = p->d[row] + lam * w[row];
  free(w);
  orc_delta_free(&D);
  return ORC_OK;
}
