// dynspec_b200.cpp -- drop-in replacement of the reference's proj/src/dpt.cpp.
//
// Defines every function declared by the reference's public header
// proj/include/dynspec/dpt.hpp (namespace dynspec) with the exact signatures,
// on top of the C ABI of libdpt_b200.so (include/dpt_b200.h).  Build it in
// place of src/dpt.cpp and link libdpt_b200.so; the
// reference's callers -- tools/main.cpp, src/rspt.cpp, src/analysis.cpp, the
// tests -- compile and link unchanged.
//
// Hot path (GPU): step_full, step_single (x2), eigenvalue_of, iterate_full,
// iterate_ramped, iterate_fixed, iterate_single, dominant_eigenpair.
// Small-n analysis helpers (jacobian_single, reduced_jacobian, multipliers)
// and the staged homotopy_solve are host orchestration around them.
//
// Documented deviation: the path is real FP64.  Any nonzero imaginary part in
// d, Delta, lambda or an input iterate throws std::invalid_argument
// ("non-real input ...") instead of being dropped.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <variant>
#include <vector>

#include "dpt_b200.h"
#include "dynspec/dpt.hpp"
#include "dynspec/roots.hpp"

namespace dynspec {

namespace {

// One context per calling thread (the reference's functions are reentrant and
// scan_domain calls them from many threads, proj/src/analysis.cpp:96-135).
struct CtxHolder {
  dpt_ctx* ctx = nullptr;
  ~CtxHolder() {
    if (ctx) dpt_ctx_destroy(ctx);
  }
};

[[noreturn]] void raise(int rc, const dpt_error_info& e) {
  const std::string msg = e.message[0] ? std::string(e.message) : std::string("dpt_b200 error");
  switch (rc) {
    case DPT_ERR_SHAPE:
      throw ShapeError(msg);
    case DPT_ERR_DEGENERATE:
      throw DegenerateSpectrum(msg, std::size_t(e.i), std::size_t(e.j), cdouble{e.ei, 0.0}, cdouble{e.ej, 0.0});
    case DPT_ERR_INVALID_ARG:
    case DPT_ERR_NON_REAL:
      throw std::invalid_argument(msg);
    default:
      throw std::runtime_error(msg);
  }
}

void check(int rc, const dpt_error_info& e) {
  if (rc != DPT_OK) raise(rc, e);
}

dpt_ctx* ctx() {
  thread_local CtxHolder h;
  if (!h.ctx) {
    const char* dev = std::getenv("DPT_DEVICE");
    dpt_error_info e{};
    check(dpt_ctx_create(dev ? std::atoi(dev) : 0, &h.ctx, &e), e);
  }
  return h.ctx;
}

double real_of(cdouble v, const char* what) {
  if (v.imag() != 0.0) throw std::invalid_argument(std::string("non-real input (") + what + "): the B200 path is real FP64");
  return v.real();
}

std::vector<double> real_vec(std::span<const cdouble> v, const char* what) {
  std::vector<double> r(v.size());
  for (std::size_t i = 0; i < v.size(); ++i) r[i] = real_of(v[i], what);
  return r;
}

std::vector<double> real_dense(const DenseMatrix& m, const char* what) {
  const std::size_t nn = m.rows() * m.cols();
  std::vector<double> r(nn);
  for (std::size_t i = 0; i < nn; ++i) r[i] = real_of(m.data()[i], what);
  return r;
}

// Plain-array image of a PartitionedProblem (delta, not delta_t).
struct Problem {
  std::vector<double> d, dense, vals;
  std::vector<int64_t> rowptr;
  std::vector<int32_t> cols;
  dpt_problem c{};
};

void fill_delta(Problem& P, const MatrixVariant& delta, std::size_t n) {
  if (const auto* dm = std::get_if<DenseMatrix>(&delta)) {
    if (dm->rows() != n || dm->cols() != n) throw ShapeError("delta shape does not match diagonal");
    P.dense = real_dense(*dm, "delta");
    P.c.delta_kind = DPT_DELTA_DENSE;
    P.c.delta = P.dense.data();
  } else {
    const auto& s = std::get<SparseMatrix>(delta);
    if (s.rows() != n || s.cols() != n) throw ShapeError("delta shape does not match diagonal");
    if (n >= std::size_t(std::numeric_limits<int32_t>::max())) throw ShapeError("CSR dimension exceeds int32");
    P.rowptr.assign(s.row_offsets().begin(), s.row_offsets().end());
    P.cols.resize(s.nnz());
    for (std::size_t q = 0; q < s.nnz(); ++q) P.cols[q] = int32_t(s.col_indices()[q]);
    P.vals = real_vec(s.values(), "delta");
    P.c.delta_kind = DPT_DELTA_CSR;
    P.c.rowptr = P.rowptr.data();
    P.c.cols = P.cols.data();
    P.c.vals = P.vals.data();
    P.c.nnz = int64_t(s.nnz());
  }
}

std::unique_ptr<Problem> to_c(const DiagonalMatrix& d, const MatrixVariant& delta, cdouble lambda) {
  auto P = std::make_unique<Problem>();
  const std::size_t n = d.size();
  P->d = real_vec(d.d, "d");
  fill_delta(*P, delta, n);
  P->c.n = int64_t(n);
  P->c.d = P->d.data();
  P->c.lambda = real_of(lambda, "lambda");
  P->c.mem = DPT_MEM_HOST;
  return P;
}

std::unique_ptr<Problem> to_c(const PartitionedProblem& p) { return to_c(p.d, p.delta, p.lambda); }

dpt_options to_c(const IterationOptions& o) {
  dpt_options r;
  r.tol = o.tol;
  r.residual_tol = o.residual_tol;
  r.max_iter = o.max_iter;
  r.divergence_threshold = o.divergence_threshold;
  r.cycle_window = o.cycle_window;
  r.degeneracy_tol = o.degeneracy_tol;
  return r;
}

DenseMatrix from_real(const std::vector<double>& a, std::size_t n) {
  DenseMatrix m(n, n);
  for (std::size_t i = 0; i < n * n; ++i) m.data()[i] = cdouble{a[i], 0.0};
  return m;
}

cdouble c_of(double v) {  // NaN read-offs are cdouble{nan, nan} (dpt.cpp:121-124)
  return std::isnan(v) ? cdouble{v, v} : cdouble{v, 0.0};
}

// TraceSink trampoline: an exception thrown by the sink aborts the solve and
// propagates to the caller, as in the reference.
struct TraceBox {
  const TraceSink* sink;
  std::exception_ptr exc;
};

int trace_tramp(int k, double s, double r, void* user) {
  auto* b = static_cast<TraceBox*>(user);
  try {
    (*b->sink)(k, s, r);
    return 0;
  } catch (...) {
    b->exc = std::current_exception();
    return 1;
  }
}

ConvergenceReport full_report(std::size_t n, const std::vector<double>& a, const std::vector<double>& eig,
                              const std::vector<double>& res, const dpt_report& r) {
  ConvergenceReport rep;
  rep.status = ConvergenceStatus(r.status);
  rep.iterations = r.iterations;
  rep.step_norm = r.step_norm;
  rep.eigenvalues.resize(n);
  rep.residuals = res;
  for (std::size_t i = 0; i < n; ++i) rep.eigenvalues[i] = c_of(eig[i]);
  rep.state = EigenIterate{from_real(a, n), r.iterations};
  return rep;
}

ConvergenceReport run_full(const PartitionedProblem& p, const IterationOptions& opts, bool ramped, double alpha,
                           const TraceSink& trace) {
  auto P = to_c(p);
  const std::size_t n = p.size();
  std::vector<double> a(n * n), eig(n), res(n);
  dpt_options o = to_c(opts);
  dpt_report r{};
  dpt_error_info e{};
  TraceBox box{&trace, nullptr};
  dpt_trace_fn fn = trace ? &trace_tramp : nullptr;
  const int rc = ramped ? dpt_iterate_ramped(ctx(), &P->c, alpha, &o, fn, &box, a.data(), eig.data(), res.data(),
                                             DPT_MEM_HOST, &r, &e)
                        : dpt_iterate_full(ctx(), &P->c, &o, fn, &box, a.data(), eig.data(), res.data(),
                                           DPT_MEM_HOST, &r, &e);
  if (rc == DPT_ERR_TRACE && box.exc) std::rethrow_exception(box.exc);
  check(rc, e);
  return full_report(n, a, eig, res, r);
}

std::vector<cdouble> to_complex(const std::vector<double>& v) {
  std::vector<cdouble> r(v.size());
  for (std::size_t i = 0; i < v.size(); ++i) r[i] = cdouble{v[i], 0.0};
  return r;
}

}  // namespace

std::string to_string(ConvergenceStatus s) { return dpt_status_string(int(s)); }

DenseMatrix step_full(const DenseMatrix& a, const GapMatrix& theta, const MatrixVariant& delta_t, cdouble lambda) {
  const std::size_t n = a.rows();
  if (a.cols() != n || theta.theta.rows() != n) throw ShapeError("step_full: dimension mismatch");
  // the C ABI takes Delta; recover it from the cached transpose (no conjugation)
  const MatrixVariant delta = transpose(delta_t);
  DiagonalMatrix zeros(std::vector<cdouble>(n, cdouble{}));  // levels unused with an explicit gap matrix
  auto P = to_c(zeros, delta, lambda);
  const std::vector<double> ar = real_dense(a, "iterate"), g = real_dense(theta.theta, "theta");
  std::vector<double> out(n * n);
  dpt_error_info e{};
  check(dpt_step_full_gap(ctx(), &P->c, ar.data(), g.data(), P->c.lambda, out.data(), DPT_MEM_HOST, &e), e);
  return from_real(out, n);
}

std::vector<cdouble> step_single(std::span<const cdouble> z, const GapRow& gaps, const MatrixVariant& delta,
                                 cdouble lambda) {
  const std::size_t n = z.size();
  if (gaps.inv_gaps.size() != n) throw ShapeError("step_single: dimension mismatch");
  DiagonalMatrix zeros(std::vector<cdouble>(n, cdouble{}));
  auto P = to_c(zeros, delta, lambda);
  const std::vector<double> zr = real_vec(z, "z"), g = real_vec(gaps.inv_gaps, "gap row");
  std::vector<double> out(n);
  dpt_error_info e{};
  check(dpt_step_single_gap(ctx(), &P->c, zr.data(), int64_t(gaps.row), g.data(), P->c.lambda, out.data(),
                            DPT_MEM_HOST, &e),
        e);
  return to_complex(out);
}

std::vector<cdouble> step_single(std::span<const cdouble> z, std::size_t n, const GapMatrix& theta,
                                 const MatrixVariant& delta, cdouble lambda) {
  const std::size_t dim = z.size();
  if (theta.theta.rows() != dim || n >= dim) throw ShapeError("step_single: dimension mismatch");
  GapRow gaps;
  gaps.row = n;
  gaps.inv_gaps.assign(theta.theta.row(n).begin(), theta.theta.row(n).end());
  return step_single(z, gaps, delta, lambda);
}

cdouble eigenvalue_of(std::span<const cdouble> z, std::size_t n, const DiagonalMatrix& d, const MatrixVariant& delta,
                      cdouble lambda) {
  if (z.size() != d.size() || n >= z.size()) throw ShapeError("eigenvalue_of: dimension mismatch");
  auto P = to_c(d, delta, lambda);
  const std::vector<double> zr = real_vec(z, "z");
  double out = 0.0;
  dpt_error_info e{};
  check(dpt_eigenvalue_of(ctx(), &P->c, zr.data(), int64_t(n), P->c.lambda, &out, DPT_MEM_HOST, &e), e);
  return cdouble{out, 0.0};
}

ConvergenceReport iterate_full(const PartitionedProblem& p, const IterationOptions& opts, const TraceSink& trace) {
  return run_full(p, opts, false, 0.0, trace);
}

ConvergenceReport iterate_ramped(const PartitionedProblem& p, double alpha, const IterationOptions& opts,
                                 const TraceSink& trace) {
  if (!(alpha >= 0.0) || alpha >= 1.0) throw std::invalid_argument("iterate_ramped: alpha must lie in [0, 1)");
  return run_full(p, opts, true, alpha, trace);
}

DenseMatrix iterate_fixed(const PartitionedProblem& p, int k, cdouble lambda) {
  if (k < 0) throw std::invalid_argument("iterate_fixed: negative step count");
  auto P = to_c(p);
  const std::size_t n = p.size();
  std::vector<double> a(n * n);
  dpt_report r{};
  dpt_error_info e{};
  check(dpt_iterate_fixed(ctx(), &P->c, k, real_of(lambda, "lambda"), a.data(), DPT_MEM_HOST, &r, &e), e);
  return from_real(a, n);
}

SingleRowReport iterate_single(const PartitionedProblem& p, std::size_t row, const IterationOptions& opts,
                               double ramp_alpha, const TraceSink& trace) {
  if (row >= p.size()) throw ShapeError("iterate_single: row out of range");
  if (!(ramp_alpha >= 0.0) || ramp_alpha >= 1.0)
    throw std::invalid_argument("iterate_single: ramp alpha must lie in [0, 1)");
  auto P = to_c(p);
  std::vector<double> z(p.size());
  dpt_options o = to_c(opts);
  dpt_report r{};
  dpt_error_info e{};
  TraceBox box{&trace, nullptr};
  const int rc = dpt_iterate_single(ctx(), &P->c, int64_t(row), &o, ramp_alpha, trace ? &trace_tramp : nullptr,
                                    &box, z.data(), DPT_MEM_HOST, &r, &e);
  if (rc == DPT_ERR_TRACE && box.exc) std::rethrow_exception(box.exc);
  check(rc, e);
  SingleRowReport rep;
  rep.z = to_complex(z);
  rep.eigenvalue = c_of(r.eigenvalue);
  rep.status = ConvergenceStatus(r.status);
  rep.iterations = r.iterations;
  rep.residual = r.residual;
  rep.step_norm = r.step_norm;
  return rep;
}

DominantEigenpair dominant_eigenpair(const PartitionedProblem& p, const IterationOptions& opts) {
  if (p.size() == 0) throw ShapeError("dominant_eigenpair: empty problem");
  auto P = to_c(p);
  std::vector<double> zc(p.size()), zu(p.size());
  dpt_options o = to_c(opts);
  dpt_report r{};
  dpt_error_info e{};
  check(dpt_dominant_eigenpair(ctx(), &P->c, &o, zc.data(), zu.data(), DPT_MEM_HOST, &r, &e), e);
  DominantEigenpair out;
  out.row = std::size_t(r.row);
  out.z_chart = to_complex(zc);
  out.z_unit = to_complex(zu);
  out.eigenvalue = c_of(r.eigenvalue);
  out.status = ConvergenceStatus(r.status);
  out.iterations = r.iterations;
  out.residual = r.residual;
  out.step_norm = r.step_norm;
  return out;
}

// ---- small-n analysis helpers (dpt.hpp:131-143): host code, n <= 8 in practice --

// (dF_n)^m_k = lambda theta_nm (Delta_mk - delta_mk (Delta z)^n - z^m Delta_nk); row n is zero.
DenseMatrix jacobian_single(std::span<const cdouble> z, std::size_t n, const GapMatrix& theta,
                            const MatrixVariant& delta, cdouble lambda) {
  const std::size_t dim = z.size();
  if (theta.theta.rows() != dim || n >= dim) throw ShapeError("jacobian_single: dimension mismatch");
  const DenseMatrix dd = densify(delta);
  const std::vector<cdouble> w = matvec(delta, z);
  DenseMatrix j(dim, dim);
  for (std::size_t m = 0; m < dim; ++m) {
    if (m == n) continue;
    const cdouble t = lambda * theta.theta(n, m);
    for (std::size_t k = 0; k < dim; ++k) {
      cdouble v = dd(m, k) - z[m] * dd(n, k);
      if (k == m) v -= w[n];
      j(m, k) = t * v;
    }
  }
  return j;
}

DenseMatrix reduced_jacobian(const DenseMatrix& j, std::size_t n) {
  const std::size_t dim = j.rows();
  if (j.cols() != dim || n >= dim || dim == 0) throw ShapeError("reduced_jacobian: dimension mismatch");
  DenseMatrix out(dim - 1, dim - 1);
  for (std::size_t i = 0, oi = 0; i < dim; ++i) {
    if (i == n) continue;
    for (std::size_t k = 0, ok = 0; k < dim; ++k) {
      if (k == n) continue;
      out(oi, ok++) = j(i, k);
    }
    ++oi;
  }
  return out;
}

std::vector<cdouble> multipliers(const DenseMatrix& reduced) {
  if (reduced.rows() != reduced.cols()) throw ShapeError("multipliers: matrix must be square");
  if (reduced.rows() > 8) throw ShapeError("multipliers: dimension capped at 8");
  return eigenvalues_dense_small(reduced);
}

// Staged continuation (dpt.hpp:145-152): stage s solves the problem rebased by
// the composition W of the converged eigenvector bases, M -> W^-1 M W, re-split
// with a zero-diagonal perturbation; each stage's solve runs on the GPU.
ConvergenceReport homotopy_solve(const PartitionedProblem& p, int stages, const IterationOptions& opts) {
  if (stages < 1) throw std::invalid_argument("homotopy_solve: stages must be >= 1");
  const std::size_t n = p.size();
  const DenseMatrix delta = densify(p.delta);
  DenseMatrix w = DenseMatrix::identity(n);
  ConvergenceReport last;
  int total = 0;
  for (int s = 1; s <= stages; ++s) {
    const cdouble lam_s = p.lambda * (double(s) / double(stages));
    DenseMatrix m = delta;
    for (std::size_t q = 0; q < n * n; ++q) m.data()[q] *= lam_s;
    for (std::size_t i = 0; i < n; ++i) m(i, i) += p.d.d[i];
    const PartitionedProblem sub = partition(MatrixVariant{solve_linear_multi(w, matmul(m, w))});
    last = iterate_full(sub, opts);
    total += last.iterations;
    if (last.status != ConvergenceStatus::Converged) break;
    w = matmul(w, transpose(last.state.a));
  }
  DenseMatrix a(n, n);
  for (std::size_t i = 0; i < n; ++i) {
    const cdouble wii = w(i, i);
    if (std::abs(wii) == 0.0) throw std::runtime_error("homotopy_solve: singular stage basis");
    for (std::size_t m = 0; m < n; ++m) a(i, m) = w(m, i) / wii;
  }
  ConvergenceReport rep;
  rep.status = last.status;
  rep.iterations = total;
  rep.step_norm = last.step_norm;
  if (all_finite(a)) {  // read-offs against the ORIGINAL problem, on the GPU
    auto P = to_c(p);
    const std::vector<double> ar = real_dense(a, "iterate");
    std::vector<double> eig(n), res(n);
    dpt_error_info e{};
    check(dpt_readoffs(ctx(), &P->c, ar.data(), eig.data(), res.data(), DPT_MEM_HOST, &e), e);
    rep.eigenvalues.resize(n);
    for (std::size_t i = 0; i < n; ++i) rep.eigenvalues[i] = c_of(eig[i]);
    rep.residuals = res;
  } else {
    const double nan = std::numeric_limits<double>::quiet_NaN();
    rep.eigenvalues.assign(n, cdouble{nan, nan});
    rep.residuals.assign(n, nan);
  }
  rep.state = EigenIterate{std::move(a), total};
  return rep;
}

}  // namespace dynspec
