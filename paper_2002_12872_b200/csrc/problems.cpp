// Seeded synthetic inputs for the BASELINE.json configs.
//
// These are input generators, not part of the solver: tests, bench.py and the
// oracle harness all feed the SAME host arrays to the reference build and to
// the CUDA path, so parity never depends on this recipe.
//
// The random source restates the reference's Rng (proj/include/dynspec/rng.hpp:12-54):
// splitmix64 with Steele et al. constants, streams derived as seed XOR FNV-1a(tag),
// uniform01 = (u64 >> 11) * 2^-53, uniform_below by rejection.  The reference has
// no normal sampler; normal() below is the SURVEY §8(d) Box-Muller cos branch.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <thread>
#include <vector>

namespace {

struct Rng {
  std::uint64_t s;
  explicit Rng(std::uint64_t seed) : s(seed) {}
  static std::uint64_t fnv1a(const char* tag) {
    std::uint64_t h = 1469598103934665603ull;
    for (const char* c = tag; *c; ++c) {
      h ^= static_cast<unsigned char>(*c);
      h *= 1099511628211ull;
    }
    return h;
  }
  static Rng stream(std::uint64_t seed, const char* tag) { return Rng(seed ^ fnv1a(tag)); }
  std::uint64_t next() {
    s += 0x9E3779B97F4A7C15ull;
    std::uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  double uniform01() { return double(next() >> 11) * 0x1.0p-53; }
  double uniform(double a, double b) { return a + (b - a) * uniform01(); }
  std::uint64_t uniform_below(std::uint64_t n) {
    const std::uint64_t bound = ~std::uint64_t{0} - (~std::uint64_t{0} % n);
    std::uint64_t x;
    do {
      x = next();
    } while (x >= bound);
    return x % n;
  }
  // u1 is drawn before u2 (explicit sequencing; the product's operand order
  // would otherwise be unspecified).
  double normal() {
    const double u1 = uniform01();
    const double u2 = uniform01();
    return std::sqrt(-2.0 * std::log(1.0 - u1)) * std::cos(2.0 * M_PI * u2);
  }
};

}  // namespace

extern "C" {

uint64_t dpt_gen_rng_u64(uint64_t seed, const char* tag, int64_t skip) {
  Rng r = Rng::stream(seed, tag);
  for (int64_t i = 0; i < skip; ++i) r.next();
  return r.next();
}

// theta_i = scale * i  (c1, c3, c5: scale 1; c4: 1/n; companion 4b: 4/n).
void dpt_gen_theta_linear(int64_t n, double scale, double* theta) {
  for (int64_t i = 0; i < n; ++i) theta[i] = scale * double(i);
}

// c2: theta_i i.i.d. Uniform(0, hi) from stream(seed,"theta"), sorted ascending,
// resampled (the stream continues) until every adjacent gap is >= min_gap.
// Returns the number of draws of the whole vector that were needed.
int dpt_gen_theta_uniform_sorted(int64_t n, uint64_t seed, double hi, double min_gap,
                                 double* theta) {
  Rng r = Rng::stream(seed, "theta");
  for (int attempt = 1;; ++attempt) {
    for (int64_t i = 0; i < n; ++i) theta[i] = r.uniform(0.0, hi);
    std::sort(theta, theta + n);
    bool ok = true;
    for (int64_t i = 1; i < n && ok; ++i) ok = (theta[i] - theta[i - 1]) >= min_gap;
    if (ok) return attempt;
    if (attempt > 100000) return -1;
  }
}

// Dense N(0,1) perturbation, drawn row-major from stream(seed, tag).
// symmetric != 0: Delta(i,j) = (X(i,j) + X(j,i)) / 2 off the diagonal (c1, c5).
// Either way the diagonal is zero (drawn, then zeroed: c2).
// splitmix64's k-th output depends only on state0 + (k+1) gamma, so rows are
// drawn in parallel (row i starts at draw 2 i n): the same values as one
// sequential stream.  The symmetrisation pair (i, j), i < j, is read and
// written only by the thread owning row i.
void dpt_gen_dense_normal(int64_t n, uint64_t seed, const char* tag, int symmetric,
                          double* delta) {
  const Rng base = Rng::stream(seed, tag);
  const size_t nn = size_t(n);
  const unsigned hw = std::thread::hardware_concurrency();
  const int T = int(std::max(1u, std::min(hw ? hw : 1u, nn * nn >= (size_t(1) << 22) ? 32u : 1u)));
  auto run = [&](auto&& body) {
    std::vector<std::thread> th;
    for (int t = 1; t < T; ++t) th.emplace_back(body, t);
    body(0);
    for (auto& x : th) x.join();
  };
  run([&](int t) {
    for (size_t i = size_t(t); i < nn; i += size_t(T)) {
      Rng r(base.s + 0x9E3779B97F4A7C15ull * (2 * i * nn));  // skip the 2 i n draws of rows < i
      for (size_t j = 0; j < nn; ++j) delta[i * nn + j] = r.normal();
    }
  });
  if (symmetric) {
    run([&](int t) {
      for (size_t i = size_t(t); i < nn; i += size_t(T))
        for (size_t j = i + 1; j < nn; ++j) {
          const double v = (delta[i * nn + j] + delta[j * nn + i]) / 2.0;
          delta[i * nn + j] = v;
          delta[j * nn + i] = v;
        }
    });
  }
  for (size_t i = 0; i < nn; ++i) delta[i * nn + i] = 0.0;
}

// c3 pattern: for i < j in row-major order, Bernoulli(density) from
// stream(seed,"pattern"); a hit draws v from stream(seed,"delta") and sets
// Delta(i,j) = Delta(j,i) = v.  Two-pass API: call with rowptr only (cols/vals
// null) to size, then again with storage.  CSR columns are sorted (the
// reference's from_triplets order, proj/src/matrix.cpp:28-53).
int64_t dpt_gen_csr_sym_bernoulli(int64_t n, uint64_t seed, double density, int64_t* rowptr,
                                  int32_t* cols, double* vals) {
  Rng pat = Rng::stream(seed, "pattern");
  Rng val = Rng::stream(seed, "delta");
  std::vector<std::vector<std::pair<int32_t, double>>> rows(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = i + 1; j < n; ++j)
      if (pat.uniform01() < density) {
        const double v = val.normal();
        rows[size_t(i)].push_back({int32_t(j), v});
        rows[size_t(j)].push_back({int32_t(i), v});
      }
  int64_t nnz = 0;
  rowptr[0] = 0;
  for (int64_t i = 0; i < n; ++i) {
    auto& r = rows[size_t(i)];
    std::sort(r.begin(), r.end());
    if (cols && vals)
      for (size_t p = 0; p < r.size(); ++p) {
        cols[nnz + int64_t(p)] = r[p].first;
        vals[nnz + int64_t(p)] = r[p].second;
      }
    nnz += int64_t(r.size());
    rowptr[i + 1] = nnz;
  }
  return nnz;
}

// c4 pattern: per row i, uniform_below(n) draws from stream(seed,"cols"),
// rejecting i and duplicates, until per_row distinct columns; each accepted
// column takes the next normal() of stream(seed,"delta").  Output CSR with
// sorted columns; nnz = n * per_row (rowptr, cols, vals preallocated).
int64_t dpt_gen_csr_fixed_per_row(int64_t n, uint64_t seed, int per_row, int64_t* rowptr,
                                  int32_t* cols, double* vals) {
  Rng cr = Rng::stream(seed, "cols");
  Rng vr = Rng::stream(seed, "delta");
  std::vector<std::pair<int32_t, double>> row;
  int64_t nnz = 0;
  rowptr[0] = 0;
  for (int64_t i = 0; i < n; ++i) {
    row.clear();
    while (int(row.size()) < per_row) {
      const int64_t c = int64_t(cr.uniform_below(uint64_t(n)));
      if (c == i) continue;
      bool dup = false;
      for (const auto& e : row) dup |= (e.first == c);
      if (dup) continue;
      row.push_back({int32_t(c), vr.normal()});
    }
    std::sort(row.begin(), row.end());
    for (const auto& e : row) {
      cols[nnz] = e.first;
      vals[nnz] = e.second;
      ++nnz;
    }
    rowptr[i + 1] = nnz;
  }
  return nnz;
}

// Uniform(-scale, scale) dense perturbation from stream(seed, "random-uniform"),
// row-major, diagonal kept: the reference's build_random_uniform fixture
// (proj/src/partition.cpp:133-142) with theta_i = i + 1.
void dpt_gen_random_uniform(int64_t n, uint64_t seed, double* theta, double* delta) {
  Rng r = Rng::stream(seed, "random-uniform");
  for (int64_t i = 0; i < n; ++i) theta[i] = double(i + 1);
  for (int64_t i = 0; i < n * n; ++i) delta[i] = r.uniform(-1.0, 1.0);
}

// The reference's harmonic-oscillator fixture (proj/src/partition.cpp:98-111):
// eps_n = 2n + 1/2, Delta = phi phi^T with the stable ratio recurrence.
void dpt_gen_oscillator(int64_t n, double* theta, double* delta) {
  std::vector<double> phi(static_cast<size_t>(n));
  phi[0] = std::pow(M_PI, -0.25);
  for (int64_t k = 1; k < n; ++k)
    phi[size_t(k)] = -phi[size_t(k - 1)] * std::sqrt((2.0 * double(k) - 1.0) / (2.0 * double(k)));
  for (int64_t k = 0; k < n; ++k) theta[k] = 2.0 * double(k) + 0.5;
  for (int64_t a = 0; a < n; ++a)
    for (int64_t b = 0; b < n; ++b) delta[a * n + b] = phi[size_t(a)] * phi[size_t(b)];
}

}  // extern "C"
