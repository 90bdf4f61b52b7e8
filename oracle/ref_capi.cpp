// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.  A C shim over the REFERENCE
// library itself (dynspec, compiled from /root/reference/proj/src into
// oracle/_ref by oracle/Makefile), exposing the same orc_* structs as the C
// restatement so tests can run both on identical inputs.  Nothing here is
// product code; the product never links it.
#include <cmath>
#include <complex>
#include <cstring>
#include <vector>

#include "dpt_oracle.h"
#include "dynspec/analysis.hpp"
#include "dynspec/dpt.hpp"
#include "dynspec/matrix_market.hpp"
#include "dynspec/matrix.hpp"
#include "dynspec/partition.hpp"

using namespace dynspec;

namespace {

MatrixVariant to_delta(const orc_problem* p) {
  const std::size_t n = std::size_t(p->n);
  if (p->kind == ORC_DENSE) {
    DenseMatrix m(n, n);
    for (std::size_t i = 0; i < n * n; ++i) m.data()[i] = p->delta[i];
    return m;
  }
  std::vector<SparseMatrix::Triplet> t;
  t.reserve(std::size_t(p->rowptr[n]));
  for (std::size_t i = 0; i < n; ++i)
    for (int64_t q = p->rowptr[i]; q < p->rowptr[i + 1]; ++q)
      t.push_back({i, std::size_t(p->cols[q]), cdouble{p->vals[q], 0.0}});
  return SparseMatrix::from_triplets(n, n, std::move(t));
}

PartitionedProblem to_problem(const orc_problem* p) {
  std::vector<cdouble> d(std::size_t(p->n));
  for (int64_t i = 0; i < p->n; ++i) d[std::size_t(i)] = p->d[i];
  return make_problem(DiagonalMatrix(std::move(d)), to_delta(p), cdouble{p->lambda, 0.0});
}

IterationOptions to_opts(const orc_options* o) {
  IterationOptions r;
  r.tol = o->tol;
  r.residual_tol = o->residual_tol;
  r.max_iter = o->max_iter;
  r.divergence_threshold = o->divergence_threshold;
  r.cycle_window = o->cycle_window;
  r.degeneracy_tol = o->degeneracy_tol;
  return r;
}

void put_dense(const DenseMatrix& a, double* out, double* imag_max) {
  const std::size_t nn = a.rows() * a.cols();
  double im = 0.0;
  for (std::size_t i = 0; i < nn; ++i) {
    out[i] = a.data()[i].real();
    im = std::max(im, std::fabs(a.data()[i].imag()));
  }
  if (imag_max) *imag_max = std::max(*imag_max, im);
}

}  // namespace

extern "C" {

int ref_iterate_full(const orc_problem* p, const orc_options* o, int ramped, double alpha, double* a_out,
                     double* eig_out, double* res_out, orc_report* rep, double* trace_step, double* trace_res,
                     double* imag_max) {
  std::memset(rep, 0, sizeof(*rep));
  try {
    const PartitionedProblem pp = to_problem(p);
    int idx = 0;
    TraceSink sink;
    if (trace_step)
      sink = [&](int k, double s, double r) {
        (void)k;
        trace_step[idx] = s;
        trace_res[idx] = r;
        ++idx;
      };
    const ConvergenceReport r =
        ramped ? iterate_ramped(pp, alpha, to_opts(o), sink) : iterate_full(pp, to_opts(o), sink);
    rep->status = int(r.status);
    rep->iterations = r.iterations;
    rep->step_norm = r.step_norm;
    put_dense(r.state.a, a_out, imag_max);
    for (std::size_t i = 0; i < r.eigenvalues.size(); ++i) {
      eig_out[i] = r.eigenvalues[i].real();
      res_out[i] = r.residuals[i];
      if (imag_max && std::isfinite(r.eigenvalues[i].imag()))
        *imag_max = std::max(*imag_max, std::fabs(r.eigenvalues[i].imag()));
    }
    return ORC_OK;
  } catch (const DegenerateSpectrum& e) {
    rep->degenerate_i = int64_t(e.first());
    rep->degenerate_j = int64_t(e.second());
    return ORC_ERR_DEGENERATE;
  } catch (const ShapeError&) {
    return ORC_ERR_SHAPE;
  } catch (const std::invalid_argument&) {
    return ORC_ERR_INVALID;
  }
}

int ref_iterate_fixed(const orc_problem* p, int k, double lam, double* a_out) {
  try {
    put_dense(iterate_fixed(to_problem(p), k, cdouble{lam, 0.0}), a_out, nullptr);
    return ORC_OK;
  } catch (const DegenerateSpectrum&) {
    return ORC_ERR_DEGENERATE;
  } catch (const std::invalid_argument&) {
    return ORC_ERR_INVALID;
  }
}

int ref_step_full(const orc_problem* p, const double* a, double lam, double* out) {
  const PartitionedProblem pp = to_problem(p);
  const std::size_t n = std::size_t(p->n);
  DenseMatrix am(n, n);
  for (std::size_t i = 0; i < n * n; ++i) am.data()[i] = a[i];
  put_dense(step_full(am, build_theta(pp.d), pp.delta_t, cdouble{lam, 0.0}), out, nullptr);
  return ORC_OK;
}

int ref_iterate_single(const orc_problem* p, int64_t row, const orc_options* o, double ramp_alpha, double* z_out,
                       orc_single_report* rep, double* trace_step, double* trace_res) {
  std::memset(rep, 0, sizeof(*rep));
  try {
    const PartitionedProblem pp = to_problem(p);
    int idx = 0;
    TraceSink sink;
    if (trace_step)
      sink = [&](int, double s, double r) {
        trace_step[idx] = s;
        trace_res[idx] = r;
        ++idx;
      };
    const SingleRowReport r = iterate_single(pp, std::size_t(row), to_opts(o), ramp_alpha, sink);
    rep->status = int(r.status);
    rep->iterations = r.iterations;
    rep->step_norm = r.step_norm;
    rep->eigenvalue = r.eigenvalue.real();
    rep->residual = r.residual;
    for (std::size_t m = 0; m < r.z.size(); ++m) z_out[m] = r.z[m].real();
    return ORC_OK;
  } catch (const DegenerateSpectrum& e) {
    rep->degenerate_i = int64_t(e.first());
    rep->degenerate_j = int64_t(e.second());
    return ORC_ERR_DEGENERATE;
  } catch (const ShapeError&) {
    return ORC_ERR_SHAPE;
  } catch (const std::invalid_argument&) {
    return ORC_ERR_INVALID;
  }
}

int ref_dominant_eigenpair(const orc_problem* p, const orc_options* o, double* z_chart, double* z_unit,
                           orc_single_report* rep, int64_t* row_out) {
  std::memset(rep, 0, sizeof(*rep));
  try {
    const DominantEigenpair r = dominant_eigenpair(to_problem(p), to_opts(o));
    rep->status = int(r.status);
    rep->iterations = r.iterations;
    rep->step_norm = r.step_norm;
    rep->eigenvalue = r.eigenvalue.real();
    rep->residual = r.residual;
    *row_out = int64_t(r.row);
    for (std::size_t m = 0; m < r.z_chart.size(); ++m) {
      z_chart[m] = r.z_chart[m].real();
      z_unit[m] = r.z_unit[m].real();
    }
    return ORC_OK;
  } catch (const DegenerateSpectrum& e) {
    rep->degenerate_i = int64_t(e.first());
    rep->degenerate_j = int64_t(e.second());
    return ORC_ERR_DEGENERATE;
  } catch (const ShapeError&) {
    return ORC_ERR_SHAPE;
  }
}

int ref_step_single(const orc_problem* p, const double* z, int64_t row, double lam, double* out) {
  const PartitionedProblem pp = to_problem(p);
  std::vector<cdouble> zz(std::size_t(p->n));
  for (int64_t m = 0; m < p->n; ++m) zz[std::size_t(m)] = z[m];
  const GapRow g = build_gap_row(pp.d, std::size_t(row));
  const auto r = step_single(zz, g, pp.delta, cdouble{lam, 0.0});
  for (std::size_t m = 0; m < r.size(); ++m) out[m] = r[m].real();
  return ORC_OK;
}

int ref_eigenvalue_of(const orc_problem* p, const double* z, int64_t row, double lam, double* out) {
  const PartitionedProblem pp = to_problem(p);
  std::vector<cdouble> zz(std::size_t(p->n));
  for (int64_t m = 0; m < p->n; ++m) zz[std::size_t(m)] = z[m];
  *out = eigenvalue_of(zz, std::size_t(row), pp.d, pp.delta, cdouble{lam, 0.0}).real();
  return ORC_OK;
}

// build_theta's degeneracy payload (partition.cpp:69-81) from the reference itself.
int ref_check_degenerate(int64_t n, const double* d, double tol, int64_t* i, int64_t* j) {
  std::vector<cdouble> dd(static_cast<std::size_t>(n));
  for (int64_t q = 0; q < n; ++q) dd[std::size_t(q)] = d[q];
  try {
    (void)build_theta(DiagonalMatrix(std::move(dd)), tol);
    return 0;
  } catch (const DegenerateSpectrum& e) {
    *i = int64_t(e.first());
    *j = int64_t(e.second());
    return 1;
  }
}

// The reference's own row-subset cost unit for the bounded CPU baseline:
// P = A_rows * delta_t (matmul, src/matrix.cpp:130-158) plus the map
// (src/dpt.cpp:136-144) for rows [row0, row0 + rows).
int ref_step_rows(const orc_problem* p, int64_t row0, int64_t rows, const double* a, double lam, double* out) {
  const PartitionedProblem pp = to_problem(p);
  const std::size_t n = std::size_t(p->n);
  DenseMatrix am(std::size_t(rows), n);
  for (std::size_t i = 0; i < std::size_t(rows) * n; ++i) am.data()[i] = a[i];
  const DenseMatrix pm = matmul(am, pp.delta_t);
  const cdouble lk{lam, 0.0};
  for (std::size_t i = 0; i < std::size_t(rows); ++i) {
    const std::size_t gi = std::size_t(row0) + i;
    const cdouble pii = pm(i, gi);
    for (std::size_t j = 0; j < n; ++j) {
      const cdouble th = gi == j ? cdouble{} : 1.0 / (pp.d.d[gi] - pp.d.d[j]);
      out[i * n + j] = (gi == j ? cdouble{1.0, 0.0} : lk * th * (pm(i, j) - pii * am(i, j))).real();
    }
  }
  return ORC_OK;
}

}  // extern "C"

// Prepared problem for the bench's reference arm: the one-time make_problem
// (with its delta_t cache) stays outside the timed region, as in the
// reference's own bench (proj/tools/main.cpp:691-762).
extern "C" {

void* ref_prepare(const orc_problem* p) { return new PartitionedProblem(to_problem(p)); }

void ref_release(void* h) { delete static_cast<PartitionedProblem*>(h); }

int ref_prepared_step_rows(void* h, int64_t row0, int64_t rows, const double* a, double lam, double* out) {
  const PartitionedProblem& pp = *static_cast<PartitionedProblem*>(h);
  const std::size_t n = pp.size();
  DenseMatrix am(std::size_t(rows), n);
  for (std::size_t i = 0; i < std::size_t(rows) * n; ++i) am.data()[i] = a[i];
  const DenseMatrix pm = matmul(am, pp.delta_t);
  const cdouble lk{lam, 0.0};
  for (std::size_t i = 0; i < std::size_t(rows); ++i) {
    const std::size_t gi = std::size_t(row0) + i;
    const cdouble pii = pm(i, gi);
    for (std::size_t j = 0; j < n; ++j) {
      const cdouble th = gi == j ? cdouble{} : 1.0 / (pp.d.d[gi] - pp.d.d[j]);
      out[i * n + j] = (gi == j ? cdouble{1.0, 0.0} : lk * th * (pm(i, j) - pii * am(i, j))).real();
    }
  }
  return ORC_OK;
}

}  // extern "C"

// ---- complex inputs: the reference's native std::complex<double> path ------
// Arrays are interleaved (re, im) = std::complex<double> layout.
extern "C" {

typedef struct {
  int64_t n;
  const double* d;  // [2n]
  int kind;
  const double* delta;  // dense [2 n n]
  const int64_t* rowptr;
  const int32_t* cols;
  const double* vals;  // [2 nnz]
  double lam_re, lam_im;
} orc_cproblem;

static PartitionedProblem to_cproblem(const orc_cproblem* p) {
  const std::size_t n = std::size_t(p->n);
  std::vector<cdouble> d(n);
  for (std::size_t i = 0; i < n; ++i) d[i] = cdouble{p->d[2 * i], p->d[2 * i + 1]};
  MatrixVariant delta;
  if (p->kind == ORC_DENSE) {
    DenseMatrix m(n, n);
    for (std::size_t i = 0; i < n * n; ++i) m.data()[i] = cdouble{p->delta[2 * i], p->delta[2 * i + 1]};
    delta = std::move(m);
  } else {
    std::vector<SparseMatrix::Triplet> t;
    for (std::size_t i = 0; i < n; ++i)
      for (int64_t q = p->rowptr[i]; q < p->rowptr[i + 1]; ++q)
        t.push_back({i, std::size_t(p->cols[q]), cdouble{p->vals[2 * q], p->vals[2 * q + 1]}});
    delta = SparseMatrix::from_triplets(n, n, std::move(t));
  }
  return make_problem(DiagonalMatrix(std::move(d)), std::move(delta), cdouble{p->lam_re, p->lam_im});
}

static void put_cdense(const DenseMatrix& a, double* out) {
  for (std::size_t i = 0; i < a.rows() * a.cols(); ++i) {
    out[2 * i] = a.data()[i].real();
    out[2 * i + 1] = a.data()[i].imag();
  }
}

int ref_c_iterate_full(const orc_cproblem* p, const orc_options* o, int ramped, double alpha, double* a_out,
                       double* eig_out, double* res_out, orc_report* rep, double* trace_step, double* trace_res) {
  std::memset(rep, 0, sizeof(*rep));
  try {
    const PartitionedProblem pp = to_cproblem(p);
    int idx = 0;
    TraceSink sink;
    if (trace_step)
      sink = [&](int, double s, double r) {
        trace_step[idx] = s;
        trace_res[idx] = r;
        ++idx;
      };
    const ConvergenceReport r =
        ramped ? iterate_ramped(pp, alpha, to_opts(o), sink) : iterate_full(pp, to_opts(o), sink);
    rep->status = int(r.status);
    rep->iterations = r.iterations;
    rep->step_norm = r.step_norm;
    put_cdense(r.state.a, a_out);
    for (std::size_t i = 0; i < r.eigenvalues.size(); ++i) {
      eig_out[2 * i] = r.eigenvalues[i].real();
      eig_out[2 * i + 1] = r.eigenvalues[i].imag();
      res_out[i] = r.residuals[i];
    }
    return ORC_OK;
  } catch (const DegenerateSpectrum& e) {
    rep->degenerate_i = int64_t(e.first());
    rep->degenerate_j = int64_t(e.second());
    return ORC_ERR_DEGENERATE;
  } catch (const std::invalid_argument&) {
    return ORC_ERR_INVALID;
  }
}

int ref_c_iterate_single(const orc_cproblem* p, int64_t row, const orc_options* o, double ramp_alpha, double* z_out,
                         double* eig2, orc_single_report* rep) {
  std::memset(rep, 0, sizeof(*rep));
  try {
    const SingleRowReport r = iterate_single(to_cproblem(p), std::size_t(row), to_opts(o), ramp_alpha, {});
    rep->status = int(r.status);
    rep->iterations = r.iterations;
    rep->step_norm = r.step_norm;
    rep->residual = r.residual;
    eig2[0] = r.eigenvalue.real();
    eig2[1] = r.eigenvalue.imag();
    for (std::size_t m = 0; m < r.z.size(); ++m) {
      z_out[2 * m] = r.z[m].real();
      z_out[2 * m + 1] = r.z[m].imag();
    }
    return ORC_OK;
  } catch (const DegenerateSpectrum& e) {
    rep->degenerate_i = int64_t(e.first());
    rep->degenerate_j = int64_t(e.second());
    return ORC_ERR_DEGENERATE;
  }
}

int ref_c_dominant(const orc_cproblem* p, const orc_options* o, double* z_chart, double* z_unit, double* eig2,
                   orc_single_report* rep, int64_t* row_out) {
  std::memset(rep, 0, sizeof(*rep));
  try {
    const DominantEigenpair r = dominant_eigenpair(to_cproblem(p), to_opts(o));
    rep->status = int(r.status);
    rep->iterations = r.iterations;
    rep->residual = r.residual;
    *row_out = int64_t(r.row);
    eig2[0] = r.eigenvalue.real();
    eig2[1] = r.eigenvalue.imag();
    for (std::size_t m = 0; m < r.z_chart.size(); ++m) {
      z_chart[2 * m] = r.z_chart[m].real();
      z_chart[2 * m + 1] = r.z_chart[m].imag();
      z_unit[2 * m] = r.z_unit[m].real();
      z_unit[2 * m + 1] = r.z_unit[m].imag();
    }
    return ORC_OK;
  } catch (const DegenerateSpectrum& e) {
    rep->degenerate_i = int64_t(e.first());
    rep->degenerate_j = int64_t(e.second());
    return ORC_ERR_DEGENERATE;
  } catch (const std::invalid_argument&) {  // ShapeError: empty problem (dpt.cpp:402)
    return ORC_ERR_SHAPE;
  }
}

int ref_c_iterate_fixed(const orc_cproblem* p, int k, double lr, double li, double* a_out) {
  put_cdense(iterate_fixed(to_cproblem(p), k, cdouble{lr, li}), a_out);
  return ORC_OK;
}

int ref_c_step_full(const orc_cproblem* p, const double* a, double lr, double li, double* out) {
  const PartitionedProblem pp = to_cproblem(p);
  const std::size_t n = std::size_t(p->n);
  DenseMatrix am(n, n);
  for (std::size_t i = 0; i < n * n; ++i) am.data()[i] = cdouble{a[2 * i], a[2 * i + 1]};
  put_cdense(step_full(am, build_theta(pp.d), pp.delta_t, cdouble{lr, li}), out);
  return ORC_OK;
}

int ref_c_step_single(const orc_cproblem* p, const double* z, int64_t row, double lr, double li, double* out,
                      double* eig2) {
  const PartitionedProblem pp = to_cproblem(p);
  std::vector<cdouble> zz(std::size_t(p->n));
  for (int64_t m = 0; m < p->n; ++m) zz[std::size_t(m)] = cdouble{z[2 * m], z[2 * m + 1]};
  const auto r = step_single(zz, build_gap_row(pp.d, std::size_t(row)), pp.delta, cdouble{lr, li});
  for (std::size_t m = 0; m < r.size(); ++m) {
    out[2 * m] = r[m].real();
    out[2 * m + 1] = r[m].imag();
  }
  const cdouble e = eigenvalue_of(zz, std::size_t(row), pp.d, pp.delta, cdouble{lr, li});
  eig2[0] = e.real();
  eig2[1] = e.imag();
  return ORC_OK;
}

int ref_c_check_degenerate(int64_t n, const double* d, double tol, int64_t* i, int64_t* j) {
  std::vector<cdouble> dd(static_cast<std::size_t>(n));
  for (int64_t q = 0; q < n; ++q) dd[std::size_t(q)] = cdouble{d[2 * q], d[2 * q + 1]};
  try {
    (void)build_theta(DiagonalMatrix(std::move(dd)), tol);
    return 0;
  } catch (const DegenerateSpectrum& e) {
    *i = int64_t(e.first());
    *j = int64_t(e.second());
    return 1;
  }
}

}  // extern "C"

// scan_domain (proj/src/analysis.cpp:68-138) of the reference: classes[cells]
// (CellClass), iterations[cells].  mode 0 Full, 1 SingleRow.
extern "C" int ref_scan_domain(const orc_cproblem* p, double re_min, double re_max, double im_min, double im_max,
                               int64_t res_re, int64_t res_im, int mode, int64_t row, double ramp_alpha,
                               const orc_options* o, int threads, uint8_t* classes, int32_t* iterations,
                               int64_t* deg_i, int64_t* deg_j) {
  try {
    const PartitionedProblem pp = to_cproblem(p);
    ScanGrid g;
    g.re_min = re_min;
    g.re_max = re_max;
    g.im_min = im_min;
    g.im_max = im_max;
    g.res_re = std::size_t(res_re);
    g.res_im = std::size_t(res_im);
    ScanMode m;
    m.kind = mode == 1 ? ScanMode::Kind::SingleRow : ScanMode::Kind::Full;
    m.row = std::size_t(row);
    m.ramp_alpha = ramp_alpha;
    const DomainGrid r = scan_domain(pp, g, m, to_opts(o), unsigned(threads));
    for (std::size_t c = 0; c < r.classes.size(); ++c) {
      classes[c] = uint8_t(r.classes[c]);
      iterations[c] = r.iterations[c];
    }
    return ORC_OK;
  } catch (const DegenerateSpectrum& e) {
    if (deg_i) *deg_i = int64_t(e.first());
    if (deg_j) *deg_j = int64_t(e.second());
    return ORC_ERR_DEGENERATE;
  } catch (const std::invalid_argument&) {
    return ORC_ERR_SHAPE;
  } catch (...) {
    return ORC_ERR_INVALID;
  }
}

// read_matrix_market / write_matrix_market (proj/src/matrix_market.cpp) of the
// reference, for the row-f3 parity tests.  Values are complex interleaved.
struct RefMM {
  MatrixVariant m;
};

extern "C" int ref_mm_read(const char* path, int64_t* rows, int64_t* cols, int* is_sparse, int64_t* nnz, void** handle,
                           char* msg, int msglen) {
  try {
    auto* h = new RefMM{read_matrix_market(path)};
    *handle = h;
    if (const auto* d = std::get_if<DenseMatrix>(&h->m)) {
      *rows = int64_t(d->rows());
      *cols = int64_t(d->cols());
      *is_sparse = 0;
      *nnz = int64_t(d->rows() * d->cols());
    } else {
      const auto& sp = std::get<SparseMatrix>(h->m);
      *rows = int64_t(sp.rows());
      *cols = int64_t(sp.cols());
      *is_sparse = 1;
      *nnz = int64_t(sp.nnz());
    }
    return 0;
  } catch (const IoError& e) {
    std::snprintf(msg, size_t(msglen), "%s", e.what());
    return 10;
  } catch (const std::exception& e) {
    std::snprintf(msg, size_t(msglen), "%s", e.what());
    return 1;
  }
}

extern "C" void ref_mm_get(void* handle, int64_t* rowptr, int64_t* colidx, double* vals) {
  const auto* h = static_cast<RefMM*>(handle);
  if (const auto* d = std::get_if<DenseMatrix>(&h->m)) {
    for (std::size_t q = 0; q < d->rows() * d->cols(); ++q) {
      vals[2 * q] = d->data()[q].real();
      vals[2 * q + 1] = d->data()[q].imag();
    }
    return;
  }
  const auto& sp = std::get<SparseMatrix>(h->m);
  for (std::size_t i = 0; i <= sp.rows(); ++i) rowptr[i] = int64_t(sp.row_offsets()[i]);
  for (std::size_t q = 0; q < sp.nnz(); ++q) {
    colidx[q] = int64_t(sp.col_indices()[q]);
    vals[2 * q] = sp.values()[q].real();
    vals[2 * q + 1] = sp.values()[q].imag();
  }
}

extern "C" void ref_mm_release(void* handle) { delete static_cast<RefMM*>(handle); }

extern "C" int ref_mm_write_dense(const char* path, int64_t rows, int64_t cols, const double* vals) {
  DenseMatrix m(static_cast<std::size_t>(rows), static_cast<std::size_t>(cols));
  for (std::size_t q = 0; q < std::size_t(rows * cols); ++q) m.data()[q] = cdouble{vals[2 * q], vals[2 * q + 1]};
  write_matrix_market(m, path);
  return 0;
}

extern "C" int ref_mm_write_csr(const char* path, int64_t rows, int64_t cols, const int64_t* rowptr,
                                const int64_t* colidx, const double* vals) {
  std::vector<SparseMatrix::Triplet> t;
  for (int64_t i = 0; i < rows; ++i)
    for (int64_t q = rowptr[i]; q < rowptr[i + 1]; ++q)
      t.push_back({std::size_t(i), std::size_t(colidx[q]), cdouble{vals[2 * q], vals[2 * q + 1]}});
  write_matrix_market(SparseMatrix::from_triplets(std::size_t(rows), std::size_t(cols), std::move(t)), path);
  return 0;
}

// homotopy_solve (proj/src/dpt.cpp:505-556) of the reference, complex outputs.
extern "C" int ref_c_homotopy(const orc_cproblem* p, int stages, const orc_options* o, double* a_out, double* eig_out,
                              double* res_out, orc_report* rep) {
  std::memset(rep, 0, sizeof(*rep));
  try {
    const ConvergenceReport r = homotopy_solve(to_cproblem(p), stages, to_opts(o));
    rep->status = int(r.status);
    rep->iterations = r.iterations;
    rep->step_norm = r.step_norm;
    put_cdense(r.state.a, a_out);
    for (std::size_t i = 0; i < r.eigenvalues.size(); ++i) {
      eig_out[2 * i] = r.eigenvalues[i].real();
      eig_out[2 * i + 1] = r.eigenvalues[i].imag();
      res_out[i] = r.residuals[i];
    }
    return ORC_OK;
  } catch (const DegenerateSpectrum& e) {
    rep->degenerate_i = int64_t(e.first());
    rep->degenerate_j = int64_t(e.second());
    return ORC_ERR_DEGENERATE;
  } catch (const std::invalid_argument&) {
    return ORC_ERR_INVALID;
  } catch (...) {
    return 9;
  }
}

// matmul (matrix.cpp:130-143) and solve_linear_multi (matrix.cpp:519-533) of the
// reference on interleaved complex row-major arrays (the device linear algebra's checkers).
namespace {
DenseMatrix get_cdense(const double* a, std::size_t r, std::size_t c) {
  DenseMatrix m(r, c);
  for (std::size_t i = 0; i < r * c; ++i) m.data()[i] = cdouble{a[2 * i], a[2 * i + 1]};
  return m;
}
void put_cdense_rc(const DenseMatrix& m, double* out) {
  for (std::size_t i = 0; i < m.rows() * m.cols(); ++i) {
    out[2 * i] = m.data()[i].real();
    out[2 * i + 1] = m.data()[i].imag();
  }
}
}  // namespace

extern "C" int ref_c_matmul(int64_t m, int64_t k, int64_t n, const double* a, const double* b, double* c) {
  try {
    put_cdense_rc(matmul(get_cdense(a, size_t(m), size_t(k)), get_cdense(b, size_t(k), size_t(n))), c);
    return ORC_OK;
  } catch (...) {
    return 9;
  }
}

extern "C" int ref_c_solve_linear_multi(int64_t n, int64_t nrhs, const double* a, const double* b, double* x) {
  try {
    put_cdense_rc(solve_linear_multi(get_cdense(a, size_t(n), size_t(n)), get_cdense(b, size_t(n), size_t(nrhs))), x);
    return ORC_OK;
  } catch (const std::runtime_error&) {
    return 8;  // "solve_linear: singular matrix"
  } catch (...) {
    return 9;
  }
}
