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
// Arithmetic: problems whose every imaginary part is 0 (d, Delta, lambda and
// the input iterate / gap arrays) run the real FP64 kernels -- the reference's
// std::complex arithmetic keeps imaginary parts exactly 0 there -- and all
// others run the complex FP64 kernels on the caller's interleaved storage.
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
#include "dynspec/analysis.hpp"
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
      throw DegenerateSpectrum(msg, std::size_t(e.i), std::size_t(e.j), cdouble{e.ei, e.ei_im}, cdouble{e.ej, e.ej_im});
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

bool has_imag(const cdouble* v, std::size_t n) {
  for (std::size_t i = 0; i < n; ++i)
    if (v[i].imag() != 0.0) return true;
  return false;
}

bool has_imag(std::span<const cdouble> v) { return has_imag(v.data(), v.size()); }
bool has_imag(const DenseMatrix& m) { return has_imag(m.data(), m.rows() * m.cols()); }

bool has_imag(const MatrixVariant& delta) {
  if (const auto* dm = std::get_if<DenseMatrix>(&delta)) return has_imag(*dm);
  return has_imag(std::get<SparseMatrix>(delta).values());
}

// Real image of a complex array (the real kernels); complex problems pass the
// caller's std::complex<double> storage straight through as interleaved doubles.
std::vector<double> real_part(const cdouble* v, std::size_t n) {
  std::vector<double> r(n);
  for (std::size_t i = 0; i < n; ++i) r[i] = v[i].real();
  return r;
}

const double* dbl(const cdouble* p) { return reinterpret_cast<const double*>(p); }
double* dbl(cdouble* p) { return reinterpret_cast<double*>(p); }

// Plain-array image of a PartitionedProblem (delta, not delta_t).  Real
// problems (every imaginary part 0, including lambda's and the caller's
// iterate / gap arrays) run the real kernels -- the reference's complex
// arithmetic then keeps imaginary parts exactly 0 -- everything else runs the
// complex FP64 path on the caller's interleaved storage, no copy.
struct Problem {
  bool cplx = false;
  std::vector<double> d, dense, vals;
  std::vector<int64_t> rowptr;
  std::vector<int32_t> cols;
  dpt_problem c{};
};

void fill_delta(Problem& P, const MatrixVariant& delta, std::size_t n) {
  if (const auto* dm = std::get_if<DenseMatrix>(&delta)) {
    if (dm->rows() != n || dm->cols() != n) throw ShapeError("delta shape does not match diagonal");
    if (P.cplx) {
      P.c.delta = dbl(dm->data());
    } else {
      P.dense = real_part(dm->data(), n * n);
      P.c.delta = P.dense.data();
    }
    P.c.delta_kind = DPT_DELTA_DENSE;
  } else {
    const auto& s = std::get<SparseMatrix>(delta);
    if (s.rows() != n || s.cols() != n) throw ShapeError("delta shape does not match diagonal");
    if (n >= std::size_t(std::numeric_limits<int32_t>::max())) throw ShapeError("CSR dimension exceeds int32");
    P.rowptr.assign(s.row_offsets().begin(), s.row_offsets().end());
    P.cols.resize(s.nnz());
    for (std::size_t q = 0; q < s.nnz(); ++q) P.cols[q] = int32_t(s.col_indices()[q]);
    if (P.cplx) {
      P.c.vals = dbl(s.values().data());
    } else {
      P.vals = real_part(s.values().data(), s.nnz());
      P.c.vals = P.vals.data();
    }
    P.c.delta_kind = DPT_DELTA_CSR;
    P.c.rowptr = P.rowptr.data();
    P.c.cols = P.cols.data();
    P.c.nnz = int64_t(s.nnz());
  }
}

std::unique_ptr<Problem> to_c(const DiagonalMatrix& d, const MatrixVariant& delta, cdouble lambda,
                              bool force_complex = false) {
  auto P = std::make_unique<Problem>();
  const std::size_t n = d.size();
  P->cplx = force_complex || lambda.imag() != 0.0 || has_imag(d.d) || has_imag(delta);
  if (P->cplx) {
    P->c.d = dbl(d.d.data());
  } else {
    P->d = real_part(d.d.data(), n);
    P->c.d = P->d.data();
  }
  fill_delta(*P, delta, n);
  P->c.n = int64_t(n);
  P->c.lambda = lambda.real();
  P->c.lambda_im = lambda.imag();
  P->c.is_complex = P->cplx ? 1 : 0;
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

cdouble c_of(double v) {  // NaN read-offs are cdouble{nan, nan} (dpt.cpp:121-124)
  return std::isnan(v) ? cdouble{v, v} : cdouble{v, 0.0};
}

// Output of a call: complex problems write interleaved straight into the
// caller-facing std::complex<double> storage; real problems write a real image
// that finish() widens (imaginary parts 0, NaN read-offs {nan, nan}).
struct OutBuf {
  cdouble* dst;
  std::size_t n;
  bool cplx;
  std::vector<double> re;
  OutBuf(cdouble* d, std::size_t count, bool c) : dst(d), n(count), cplx(c) {
    if (!cplx) re.resize(n);
  }
  double* ptr() { return cplx ? dbl(dst) : re.data(); }
  void finish(bool nan_pairs = false) {
    if (cplx) return;
    for (std::size_t i = 0; i < n; ++i) dst[i] = nan_pairs ? c_of(re[i]) : cdouble{re[i], 0.0};
  }
};

// Input array of a call: interleaved view of the caller's storage (complex
// problems) or its real image.
struct InBuf {
  std::vector<double> re;
  const double* p;
  InBuf(const cdouble* v, std::size_t n, bool cplx) {
    if (cplx) {
      p = dbl(v);
    } else {
      re = real_part(v, n);
      p = re.data();
    }
  }
};

cdouble eig_of(const dpt_report& r, bool cplx) {
  return cplx ? cdouble{r.eigenvalue, r.eigenvalue_im} : c_of(r.eigenvalue);
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

ConvergenceReport run_full(const PartitionedProblem& p, const IterationOptions& opts, bool ramped, double alpha,
                           const TraceSink& trace) {
  auto P = to_c(p);
  const std::size_t n = p.size();
  ConvergenceReport rep;
  DenseMatrix a(n, n);
  rep.eigenvalues.resize(n);
  rep.residuals.resize(n);
  OutBuf ab(a.data(), n * n, P->cplx), eb(rep.eigenvalues.data(), n, P->cplx);
  dpt_options o = to_c(opts);
  dpt_report r{};
  dpt_error_info e{};
  TraceBox box{&trace, nullptr};
  dpt_trace_fn fn = trace ? &trace_tramp : nullptr;
  const int rc = ramped ? dpt_iterate_ramped(ctx(), &P->c, alpha, &o, fn, &box, ab.ptr(), eb.ptr(),
                                             rep.residuals.data(), DPT_MEM_HOST, &r, &e)
                        : dpt_iterate_full(ctx(), &P->c, &o, fn, &box, ab.ptr(), eb.ptr(), rep.residuals.data(),
                                           DPT_MEM_HOST, &r, &e);
  if (rc == DPT_ERR_TRACE && box.exc) std::rethrow_exception(box.exc);
  check(rc, e);
  ab.finish();
  eb.finish(true);
  rep.status = ConvergenceStatus(r.status);
  rep.iterations = r.iterations;
  rep.step_norm = r.step_norm;
  rep.state = EigenIterate{std::move(a), r.iterations};
  return rep;
}

}  // namespace

std::string to_string(ConvergenceStatus s) { return dpt_status_string(int(s)); }

DenseMatrix step_full(const DenseMatrix& a, const GapMatrix& theta, const MatrixVariant& delta_t, cdouble lambda) {
  const std::size_t n = a.rows();
  if (a.cols() != n || theta.theta.rows() != n) throw ShapeError("step_full: dimension mismatch");
  DiagonalMatrix zeros(std::vector<cdouble>(n, cdouble{}));  // levels unused with an explicit gap matrix
  // The C ABI takes Delta.  A dense delta_t goes in as is (DPT_DELTA_DENSE_T:
  // transposed on the device); a sparse one is transposed here (no conjugation).
  const bool dense_t = std::holds_alternative<DenseMatrix>(delta_t);
  const MatrixVariant delta = dense_t ? MatrixVariant{} : transpose(delta_t);
  auto P = to_c(zeros, dense_t ? delta_t : delta, lambda, has_imag(a) || has_imag(theta.theta));
  if (dense_t) P->c.delta_kind = DPT_DELTA_DENSE_T;
  const InBuf ab(a.data(), n * n, P->cplx), gb(theta.theta.data(), n * n, P->cplx);
  DenseMatrix out(n, n);
  OutBuf ob(out.data(), n * n, P->cplx);
  dpt_error_info e{};
  check(dpt_step_full_gap_c(ctx(), &P->c, ab.p, gb.p, lambda.real(), lambda.imag(), ob.ptr(), DPT_MEM_HOST, &e), e);
  ob.finish();
  return out;
}

std::vector<cdouble> step_single(std::span<const cdouble> z, const GapRow& gaps, const MatrixVariant& delta,
                                 cdouble lambda) {
  const std::size_t n = z.size();
  if (gaps.inv_gaps.size() != n) throw ShapeError("step_single: dimension mismatch");
  DiagonalMatrix zeros(std::vector<cdouble>(n, cdouble{}));
  auto P = to_c(zeros, delta, lambda, has_imag(z) || has_imag(gaps.inv_gaps));
  const InBuf zb(z.data(), n, P->cplx), gb(gaps.inv_gaps.data(), n, P->cplx);
  std::vector<cdouble> out(n);
  OutBuf ob(out.data(), n, P->cplx);
  dpt_error_info e{};
  check(dpt_step_single_gap_c(ctx(), &P->c, zb.p, int64_t(gaps.row), gb.p, lambda.real(), lambda.imag(), ob.ptr(),
                              DPT_MEM_HOST, &e),
        e);
  ob.finish();
  return out;
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
  auto P = to_c(d, delta, lambda, has_imag(z));
  const InBuf zb(z.data(), z.size(), P->cplx);
  double out[2] = {0.0, 0.0};
  dpt_error_info e{};
  check(dpt_eigenvalue_of_c(ctx(), &P->c, zb.p, int64_t(n), lambda.real(), lambda.imag(), out, DPT_MEM_HOST, &e), e);
  return cdouble{out[0], out[1]};
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
  // lambda overrides p.lambda (dpt.cpp:383-388): the problem is complex if either is
  auto P = to_c(p.d, p.delta, p.lambda, lambda.imag() != 0.0);
  const std::size_t n = p.size();
  DenseMatrix a(n, n);
  OutBuf ab(a.data(), n * n, P->cplx);
  dpt_report r{};
  dpt_error_info e{};
  check(dpt_iterate_fixed_c(ctx(), &P->c, k, lambda.real(), lambda.imag(), ab.ptr(), DPT_MEM_HOST, &r, &e), e);
  ab.finish();
  return a;
}

SingleRowReport iterate_single(const PartitionedProblem& p, std::size_t row, const IterationOptions& opts,
                               double ramp_alpha, const TraceSink& trace) {
  if (row >= p.size()) throw ShapeError("iterate_single: row out of range");
  if (!(ramp_alpha >= 0.0) || ramp_alpha >= 1.0)
    throw std::invalid_argument("iterate_single: ramp alpha must lie in [0, 1)");
  auto P = to_c(p);
  SingleRowReport rep;
  rep.z.resize(p.size());
  OutBuf zb(rep.z.data(), p.size(), P->cplx);
  dpt_options o = to_c(opts);
  dpt_report r{};
  dpt_error_info e{};
  TraceBox box{&trace, nullptr};
  const int rc = dpt_iterate_single(ctx(), &P->c, int64_t(row), &o, ramp_alpha, trace ? &trace_tramp : nullptr,
                                    &box, zb.ptr(), DPT_MEM_HOST, &r, &e);
  if (rc == DPT_ERR_TRACE && box.exc) std::rethrow_exception(box.exc);
  check(rc, e);
  zb.finish();
  rep.eigenvalue = eig_of(r, P->cplx);
  rep.status = ConvergenceStatus(r.status);
  rep.iterations = r.iterations;
  rep.residual = r.residual;
  rep.step_norm = r.step_norm;
  return rep;
}

DominantEigenpair dominant_eigenpair(const PartitionedProblem& p, const IterationOptions& opts) {
  if (p.size() == 0) throw ShapeError("dominant_eigenpair: empty problem");
  auto P = to_c(p);
  DominantEigenpair out;
  out.z_chart.resize(p.size());
  out.z_unit.resize(p.size());
  OutBuf zc(out.z_chart.data(), p.size(), P->cplx), zu(out.z_unit.data(), p.size(), P->cplx);
  dpt_options o = to_c(opts);
  dpt_report r{};
  dpt_error_info e{};
  check(dpt_dominant_eigenpair(ctx(), &P->c, &o, zc.ptr(), zu.ptr(), DPT_MEM_HOST, &r, &e), e);
  zc.finish();
  zu.finish();
  out.row = std::size_t(r.row);
  out.eigenvalue = eig_of(r, P->cplx);
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

// Staged continuation (dpt.hpp:145-152): every stage's basis algebra and solve
// run on the device (dpt_homotopy_solve).
ConvergenceReport homotopy_solve(const PartitionedProblem& p, int stages, const IterationOptions& opts) {
  if (stages < 1) throw std::invalid_argument("homotopy_solve: stages must be >= 1");
  auto P = to_c(p);
  const std::size_t n = p.size();
  ConvergenceReport rep;
  DenseMatrix a(n, n);
  rep.eigenvalues.resize(n);
  rep.residuals.resize(n);
  OutBuf ab(a.data(), n * n, P->cplx), eb(rep.eigenvalues.data(), n, P->cplx);
  const dpt_options o = to_c(opts);
  dpt_report r{};
  dpt_error_info e{};
  check(dpt_homotopy_solve(ctx(), &P->c, stages, &o, ab.ptr(), eb.ptr(), rep.residuals.data(), DPT_MEM_HOST, &r, &e),
        e);
  ab.finish();
  eb.finish(true);
  rep.status = ConvergenceStatus(r.status);
  rep.iterations = r.iterations;
  rep.step_norm = r.step_norm;
  rep.state = EigenIterate{std::move(a), r.iterations};
  return rep;
}

// ---- batched scan_domain (analysis.hpp:63-69, analysis.cpp:68-138) ---------
// Every lambda cell solved on the device in one launch (one warp -- or, for
// n <= 3, one thread -- per cell) in the reference's operation order, so the
// classes and iteration counts equal the reference's.  To use it, compile the
// reference's analysis.cpp with -Dscan_domain=dynspec_reference_scan_domain
// (INTEGRATION.md); its other callers bind this definition unchanged.
DomainGrid scan_domain(const PartitionedProblem& base, const ScanGrid& grid, const ScanMode& mode,
                       const IterationOptions& opts, unsigned /*threads: the device decides*/) {
  if (grid.res_re == 0 || grid.res_im == 0) throw ShapeError("scan_domain: empty grid");
  if (mode.kind == ScanMode::Kind::SingleRow && mode.row >= base.size())
    throw ShapeError("scan_domain: row out of range");
  auto P = to_c(base.d, base.delta, cdouble{0.0, 0.0});  // each cell sets its own lambda
  dpt_scan_grid g{grid.re_min, grid.re_max, grid.im_min, grid.im_max, int64_t(grid.res_re), int64_t(grid.res_im)};
  DomainGrid out;
  out.grid = grid;
  const std::size_t cells = grid.res_re * grid.res_im;
  std::vector<uint8_t> cls(cells);
  out.iterations.assign(cells, 0);
  const dpt_options o = to_c(opts);
  dpt_error_info e{};
  check(dpt_scan_domain(ctx(), &P->c, &g, mode.kind == ScanMode::Kind::SingleRow ? DPT_SCAN_SINGLE_ROW : DPT_SCAN_FULL,
                        int64_t(mode.row), mode.ramp_alpha, &o, cls.data(), out.iterations.data(), &e),
        e);
  out.classes.resize(cells);
  for (std::size_t c = 0; c < cells; ++c) out.classes[c] = CellClass(cls[c]);
  return out;
}

}  // namespace dynspec
