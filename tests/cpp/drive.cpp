// drive.cpp -- integration driver for the drop-in boundary.
//
// Written only against the reference's PUBLIC headers (dynspec/*.hpp) and
// exercising the reference's own callers of the hot path unchanged:
// compare_orders / truncation_agreement (src/rspt.cpp) and scan_domain /
// bifurcation_scan (src/analysis.cpp, multi-threaded), plus every dpt.hpp
// entry point.  tests/cpp/Makefile links it twice:
//   drive_ref   with the reference's src/dpt.cpp       (CPU, the oracle)
//   drive_b200  with paper_2002_12872_b200/shim/dynspec_b200.cpp + libdpt_b200.so
// and tests/test_gpu_shim.py compares the two outputs line by line.
#include <cmath>
#include <complex>
#include <cstdio>
#include <string>
#include <unistd.h>
#include <vector>

#include "dynspec/analysis.hpp"
#include "dynspec/dpt.hpp"
#include "dynspec/matrix_market.hpp"
#include "dynspec/partition.hpp"
#include "dynspec/rspt.hpp"

using namespace dynspec;

static void put(const std::string& key, double v) { std::printf("%s %.17g\n", key.c_str(), v); }

static void put_vec(const std::string& key, const std::vector<cdouble>& v) {
  for (std::size_t i = 0; i < v.size(); ++i) put(key + "[" + std::to_string(i) + "]", v[i].real());
}

static void put_mat(const std::string& key, const DenseMatrix& a) {
  for (std::size_t i = 0; i < a.rows(); ++i)
    for (std::size_t j = 0; j < a.cols(); ++j)
      put(key + "[" + std::to_string(i) + "," + std::to_string(j) + "]", a(i, j).real());
}

static void put_cvec(const std::string& key, const std::vector<cdouble>& v) {
  for (std::size_t i = 0; i < v.size(); ++i) {
    put(key + "[" + std::to_string(i) + "].re", v[i].real());
    put(key + "[" + std::to_string(i) + "].im", v[i].imag());
  }
}

static void put_cmat(const std::string& key, const DenseMatrix& a) {
  for (std::size_t i = 0; i < a.rows(); ++i)
    for (std::size_t j = 0; j < a.cols(); ++j) {
      put(key + "[" + std::to_string(i) + "," + std::to_string(j) + "].re", a(i, j).real());
      put(key + "[" + std::to_string(i) + "," + std::to_string(j) + "].im", a(i, j).imag());
    }
}

static void put_creport(const std::string& key, const ConvergenceReport& r) {
  std::printf("%s.status %s\n", key.c_str(), to_string(r.status).c_str());
  put(key + ".iterations", r.iterations);
  if (r.status != ConvergenceStatus::Diverged) {
    put_cvec(key + ".eig", r.eigenvalues);
    put_cmat(key + ".a", r.state.a);
  }
}

static void put_report(const std::string& key, const ConvergenceReport& r) {
  std::printf("%s.status %s\n", key.c_str(), to_string(r.status).c_str());
  put(key + ".iterations", r.iterations);
  if (r.status != ConvergenceStatus::Diverged) {
    put_vec(key + ".eig", r.eigenvalues);
    put_mat(key + ".a", r.state.a);
  }
}

int main() {
  // 1. iterate_full / ramped / fixed on the reference fixtures
  put_report("two_by_two", iterate_full(build_two_by_two(cdouble{0.3, 0.0})));
  put_report("two_by_two_bounded", iterate_full(build_two_by_two(cdouble{0.88, 0.0})));
  put_report("two_by_two_diverged", iterate_full(build_two_by_two(cdouble{2.0, 0.0})));
  auto ru = build_random_uniform(9, 17);
  ru.lambda = cdouble{0.03, 0.0};
  put_report("random_uniform", iterate_full(ru));
  put_report("random_uniform_ramped", iterate_ramped(ru, 0.5));
  int traced = 0;
  iterate_full(ru, {}, [&](int k, double, double) { traced = k; });
  put("random_uniform.trace_last_k", traced);
  put_mat("random_uniform.fixed3", iterate_fixed(ru, 3, cdouble{0.03, 0.0}));
  auto osc = build_oscillator(24);
  osc.lambda = cdouble{0.5, 0.0};
  put_report("oscillator", iterate_full(osc));

  // 2. one-step maps and read-offs with the reference's own GapMatrix / GapRow
  const GapMatrix theta = build_theta(ru.d);
  DenseMatrix a = DenseMatrix::identity(9);
  for (int k = 0; k < 4; ++k) a = step_full(a, theta, ru.delta_t, ru.lambda);
  put_mat("step_full4", a);
  std::vector<cdouble> z(9, cdouble{});
  z[4] = 1.0;
  for (int k = 0; k < 4; ++k) z = step_single(z, 4, theta, ru.delta, ru.lambda);
  put_vec("step_single4", z);
  put_vec("step_single_gaprow", step_single(z, build_gap_row(ru.d, 4), ru.delta, ru.lambda));
  put("eigenvalue_of", eigenvalue_of(z, 4, ru.d, ru.delta, ru.lambda).real());

  // 3. row map
  const auto sr = iterate_single(ru, 2);
  std::printf("single.status %s\n", to_string(sr.status).c_str());
  put("single.iterations", sr.iterations);
  put("single.eig", sr.eigenvalue.real());
  put_vec("single.z", sr.z);
  const auto er = build_er_perturbed_oscillator(2000, 42, cdouble{0.01, 0.0});
  const auto dom = dominant_eigenpair(er);
  std::printf("dominant.status %s\n", to_string(dom.status).c_str());
  put("dominant.row", double(dom.row));
  put("dominant.iterations", dom.iterations);
  put("dominant.eig", dom.eigenvalue.real());
  put("dominant.z_unit[1999]", dom.z_unit[1999].real());
  put("dominant.z_unit[1990]", dom.z_unit[1990].real());

  // 4. the reference's own callers (src/rspt.cpp, src/analysis.cpp), unchanged
  auto three = build_three_by_three(cdouble{1.0, 0.0});
  const OrderComparison cmp = compare_orders(three, cdouble{0.1, 0.0}, 1e-10);
  put("compare.k_d", cmp.k_d);
  put("compare.k_rs", cmp.k_rs);
  put("compare.d_converged", cmp.d_converged);
  put("compare.rs_converged", cmp.rs_converged);
  put("truncation_agreement", truncation_agreement(three, 4, cdouble{0.05, 0.0}));
  ScanGrid grid;
  grid.re_min = 0.0;
  grid.re_max = 1.2;
  grid.im_min = 0.0;
  grid.im_max = 0.0;
  grid.res_re = 13;
  grid.res_im = 1;
  IterationOptions sopts;
  sopts.max_iter = 400;
  const DomainGrid full = scan_domain(build_two_by_two(cdouble{1.0, 0.0}), grid, {}, sopts, 4);
  for (std::size_t c = 0; c < full.classes.size(); ++c) {
    put("scan_full.class[" + std::to_string(c) + "]", double(int(full.classes[c])));
    put("scan_full.iters[" + std::to_string(c) + "]", full.iterations[c]);
  }
  ScanMode single_mode;
  single_mode.kind = ScanMode::Kind::SingleRow;
  single_mode.row = 1;
  const DomainGrid sg = scan_domain(three, grid, single_mode, sopts, 3);
  for (std::size_t c = 0; c < sg.classes.size(); ++c)
    put("scan_single.class[" + std::to_string(c) + "]", double(int(sg.classes[c])));
  const auto bif = bifurcation_scan(build_two_by_two(cdouble{1.0, 0.0}), 0, 1, 0.8, 0.95, 4, 200, 2);
  for (std::size_t s = 0; s < bif.size(); ++s)
    for (std::size_t v = 0; v < bif[s].values.size(); ++v)
      put("bif[" + std::to_string(s) + "," + std::to_string(v) + "]", bif[s].values[v].real());

  // 5. staged continuation (homotopy_solve, dpt.hpp:145-152)
  put_report("homotopy", homotopy_solve(ru, 3));

  // 6. complex coupling and complex levels (the scans' lambda plane)
  auto rc = build_random_uniform(9, 17);
  rc.lambda = cdouble{0.05, 0.02};
  put_creport("c.random_uniform", iterate_full(rc));
  put_creport("c.random_uniform_ramped", iterate_ramped(rc, 0.5));
  put_cmat("c.fixed3", iterate_fixed(ru, 3, cdouble{0.03, 0.01}));
  DenseMatrix ca = DenseMatrix::identity(9);
  for (int k = 0; k < 4; ++k) ca = step_full(ca, theta, rc.delta_t, rc.lambda);
  put_cmat("c.step_full4", ca);
  std::vector<cdouble> cz(9, cdouble{});
  cz[4] = 1.0;
  for (int k = 0; k < 4; ++k) cz = step_single(cz, 4, theta, rc.delta, rc.lambda);
  put_cvec("c.step_single4", cz);
  const cdouble ce = eigenvalue_of(cz, 4, rc.d, rc.delta, rc.lambda);
  put("c.eigenvalue_of.re", ce.real());
  put("c.eigenvalue_of.im", ce.imag());
  const auto csr_ = iterate_single(rc, 2);
  std::printf("c.single.status %s\n", to_string(csr_.status).c_str());
  put("c.single.iterations", csr_.iterations);
  put("c.single.eig.re", csr_.eigenvalue.real());
  put("c.single.eig.im", csr_.eigenvalue.imag());
  put_cvec("c.single.z", csr_.z);
  const auto cer = build_er_perturbed_oscillator(2000, 42, cdouble{0.01, 0.004});
  const auto cdom = dominant_eigenpair(cer);
  std::printf("c.dominant.status %s\n", to_string(cdom.status).c_str());
  put("c.dominant.row", double(cdom.row));
  put("c.dominant.iterations", cdom.iterations);
  put("c.dominant.eig.re", cdom.eigenvalue.real());
  put("c.dominant.eig.im", cdom.eigenvalue.imag());
  put("c.dominant.z_unit[1999].im", cdom.z_unit[1999].imag());
  ScanGrid cgrid = grid;
  cgrid.im_min = -0.6;
  cgrid.im_max = 0.6;
  cgrid.res_re = 7;
  cgrid.res_im = 5;
  const DomainGrid cfull = scan_domain(build_two_by_two(cdouble{1.0, 0.0}), cgrid, {}, sopts, 4);
  for (std::size_t c = 0; c < cfull.classes.size(); ++c) {
    put("scan_cfull.class[" + std::to_string(c) + "]", double(int(cfull.classes[c])));
    put("scan_cfull.iters[" + std::to_string(c) + "]", cfull.iterations[c]);
  }
  const DomainGrid csg = scan_domain(three, cgrid, single_mode, sopts, 3);
  for (std::size_t c = 0; c < csg.classes.size(); ++c)
    put("scan_csingle.class[" + std::to_string(c) + "]", double(int(csg.classes[c])));
  put_creport("c.homotopy", homotopy_solve(rc, 3));

  // 7. Matrix Market (row f3): the CLI's --file-d / --file-delta flow -- write
  // a problem, read it back, solve; plus a complex dense round trip
  const std::string dir = std::string(std::getenv("TMPDIR") ? std::getenv("TMPDIR") : "/tmp") + "/dpt_drive_" +
                          std::to_string(getpid()) + "_";
  {
    auto er = build_er_perturbed_oscillator(300, 7, cdouble{0.02, 0.0});
    std::vector<SparseMatrix::Triplet> dt;
    for (std::size_t i = 0; i < er.size(); ++i) dt.push_back({i, i, er.d.d[i]});
    write_matrix_market(SparseMatrix::from_triplets(er.size(), er.size(), std::move(dt)), dir + "d.mtx");
    write_matrix_market(er.delta, dir + "delta.mtx");
    const MatrixVariant dm = read_matrix_market(dir + "d.mtx");
    const MatrixVariant delta = read_matrix_market(dir + "delta.mtx");
    const auto& ds = std::get<SparseMatrix>(dm);
    std::vector<cdouble> diag(ds.rows());
    for (std::size_t i = 0; i < ds.rows(); ++i) diag[i] = ds.at(i, i);
    const PartitionedProblem fp = make_problem(DiagonalMatrix{diag}, delta, cdouble{0.02, 0.0});
    put("mm.delta_nnz", double(std::get<SparseMatrix>(delta).nnz()));
    put_report("mm.solve", iterate_full(fp, sopts));
    DenseMatrix cm(4, 3);
    for (std::size_t q = 0; q < 12; ++q) cm.data()[q] = cdouble{0.1 * double(q) - 0.37, 1.0 / (3.0 + double(q))};
    write_matrix_market(cm, dir + "c.mtx");
    put_cmat("mm.complex_round_trip", std::get<DenseMatrix>(read_matrix_market(dir + "c.mtx")));
    try {
      (void)read_matrix_market(dir + "missing.mtx");
    } catch (const IoError& e) {
      std::printf("mm.missing.status IoError\n");
    }
    for (const char* f : {"d.mtx", "delta.mtx", "c.mtx"}) std::remove((dir + f).c_str());
  }
  std::printf("done 1\n");
  return 0;
}
