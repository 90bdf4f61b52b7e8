// matrix_market_b200.cpp -- drop-in replacement of the reference's
// proj/src/matrix_market.cpp (row f3): defines read_matrix_market and the
// three write_matrix_market overloads of dynspec/matrix_market.hpp over the
// C ABI's multithreaded reader / writer (libdpt_b200.so, csrc/mm_io.cpp).
// Results are bit-identical to the reference's; IoError carries the same
// messages.  Build it in place of src/matrix_market.cpp.
#include <cstring>
#include <string>
#include <vector>

#include "dpt_b200.h"
#include "dynspec/matrix_market.hpp"

namespace dynspec {

namespace {

[[noreturn]] void raise_io(int rc, const dpt_error_info& e) {
  const std::string msg = e.message[0] ? std::string(e.message) : std::string("dpt_b200 I/O error");
  if (rc == DPT_ERR_IO) throw IoError(msg);
  throw std::runtime_error(msg);
}

struct MM {
  dpt_mm_matrix m{};
  ~MM() { dpt_mm_free(&m); }
};

bool pure_real(const cdouble* p, std::size_t n) {
  for (std::size_t i = 0; i < n; ++i)
    if (p[i].imag() != 0.0) return false;
  return true;
}

}  // namespace

MatrixVariant read_matrix_market(const std::string& path) {
  MM h;
  dpt_error_info e{};
  const int rc = dpt_mm_read(path.c_str(), 0, &h.m, &e);
  if (rc != DPT_OK) raise_io(rc, e);
  const std::size_t rows = std::size_t(h.m.rows), cols = std::size_t(h.m.cols);
  const bool cf = h.m.is_complex != 0;
  auto val = [&](std::size_t q) { return cf ? cdouble{h.m.vals[2 * q], h.m.vals[2 * q + 1]} : cdouble{h.m.vals[q], 0.0}; };
  if (!h.m.is_sparse) {
    DenseMatrix d(rows, cols);
    for (std::size_t q = 0; q < rows * cols; ++q) d.data()[q] = val(q);
    return d;
  }
  // the C ABI already ran from_triplets' steps; rebuilding through
  // from_triplets on the sorted, duplicate-free entries is the identity
  std::vector<SparseMatrix::Triplet> t;
  t.reserve(std::size_t(h.m.nnz));
  for (std::size_t i = 0; i < rows; ++i)
    for (int64_t q = h.m.rowptr[i]; q < h.m.rowptr[i + 1]; ++q)
      t.push_back({i, std::size_t(h.m.colidx[q]), val(std::size_t(q))});
  return SparseMatrix::from_triplets(rows, cols, std::move(t));
}

void write_matrix_market(const DenseMatrix& m, const std::string& path) {
  const std::size_t n = m.rows() * m.cols();
  const bool cf = !pure_real(m.data(), n);
  std::vector<double> v(cf ? 2 * n : n);
  for (std::size_t q = 0; q < n; ++q) {
    if (cf) {
      v[2 * q] = m.data()[q].real();
      v[2 * q + 1] = m.data()[q].imag();
    } else {
      v[q] = m.data()[q].real();
    }
  }
  dpt_error_info e{};
  const int rc = dpt_mm_write_dense(path.c_str(), int64_t(m.rows()), int64_t(m.cols()), v.data(), cf ? 1 : 0, 0, &e);
  if (rc != DPT_OK) raise_io(rc, e);
}

void write_matrix_market(const SparseMatrix& m, const std::string& path) {
  const std::size_t nnz = m.nnz();
  const bool cf = !pure_real(m.values().data(), nnz);
  std::vector<int64_t> rp(m.row_offsets().begin(), m.row_offsets().end()), ci(m.col_indices().begin(), m.col_indices().end());
  std::vector<double> v(cf ? 2 * nnz : nnz);
  for (std::size_t q = 0; q < nnz; ++q) {
    if (cf) {
      v[2 * q] = m.values()[q].real();
      v[2 * q + 1] = m.values()[q].imag();
    } else {
      v[q] = m.values()[q].real();
    }
  }
  dpt_error_info e{};
  const int rc = dpt_mm_write_csr(path.c_str(), int64_t(m.rows()), int64_t(m.cols()), rp.data(), ci.data(), v.data(),
                                  cf ? 1 : 0, 0, &e);
  if (rc != DPT_OK) raise_io(rc, e);
}

void write_matrix_market(const MatrixVariant& m, const std::string& path) {
  std::visit([&](const auto& mm) { write_matrix_market(mm, path); }, m);
}

}  // namespace dynspec
