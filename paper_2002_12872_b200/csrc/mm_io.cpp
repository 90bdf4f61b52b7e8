// mm_io.cpp -- Matrix Market ingestion and output, the
// on-disk format of the reference's large problems (`--file-d/--file-delta`,
// `--eigvec`; proj/src/matrix_market.cpp:70-191).
//
// Same results as the reference, bit for bit:
//   * numbers are read with correctly rounded conversions (std::from_chars;
//     strtod in the C locale for the underflow cases), as the reference's
//     istream extraction (libstdc++ num_get -> strtod) does;
//   * coordinate entries are collected in file order (symmetric mirrors right
//     after their entry) and become CSR through from_triplets' exact steps
//     (proj/src/matrix.cpp:28-53): the same std::sort comparator on the same
//     sequence -- so even duplicate sums keep the reference's order -- skipped
//     only when the sequence is already strictly sorted (then the sort is the
//     identity);
//   * output uses the reference's "%.17g" formatting and field choice.
// Differences are in speed only: the file is read in one block and its data
// lines are parsed by several threads (each a contiguous range of lines), and
// output is formatted by several threads into per-range buffers written in
// order.  Error cases raise the reference's IoError messages.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cctype>
#include <charconv>
#include <cmath>
#include <clocale>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <locale.h>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "dpt_b200.h"

namespace {

struct IoFail {
  std::string msg;
};

void set(dpt_error_info* err, int code, const std::string& msg) {
  if (!err) return;
  err->code = code;
  std::snprintf(err->message, sizeof(err->message), "%s", msg.c_str());
}

std::string lower(std::string s) {
  for (auto& c : s) c = char(std::tolower(static_cast<unsigned char>(c)));
  return s;
}

bool is_space(char c) { return std::isspace(static_cast<unsigned char>(c)) != 0; }

// A line [b, e) without its terminator.
struct Line {
  const char* b;
  const char* e;
};

// skip blank lines and '%' comments (matrix_market.cpp:61-68)
bool data_line(const Line& l) {
  const char* p = l.b;
  while (p < l.e && is_space(*p)) ++p;
  return p < l.e && *p != '%';
}

// istream-style extraction on [p, e): skip whitespace, take the longest prefix
// of the type's grammar, fail if it does not convert entirely.
bool get_ll(const char*& p, const char* e, long long& v) {
  while (p < e && is_space(*p)) ++p;
  const char* s = p;
  bool neg = false;
  if (p < e && (*p == '+' || *p == '-')) {
    neg = *p == '-';
    ++p;
  }
  const char* d = p;
  while (p < e && *p >= '0' && *p <= '9') ++p;
  if (p == d) {
    p = s;
    return false;
  }
  unsigned long long u = 0;
  auto r = std::from_chars(d, p, u);
  if (r.ec != std::errc() || u > (neg ? 9223372036854775808ull : 9223372036854775807ull)) return false;
  v = neg ? (long long)(0ull - u) : (long long)u;
  return true;
}

// Size-line extraction as `stream >> v` chains it: at the end of the line the
// value is left alone; a failed conversion stores 0 (C++11 num_get); either
// failure stops the chain (the stream is in a fail state afterwards).
bool get_size(const char*& p, const char* e, long long& v) {
  const char* q = p;
  while (q < e && is_space(*q)) ++q;
  if (q == e) return false;
  if (!get_ll(p, e, v)) {
    v = 0;
    return false;
  }
  return true;
}

locale_t c_locale() {
  static locale_t loc = newlocale(LC_ALL_MASK, "C", (locale_t)0);
  return loc;
}

bool get_double(const char*& p, const char* e, double& v) {
  while (p < e && is_space(*p)) ++p;
  const char* s = p;
  const char* q = p;
  if (q < e && (*q == '+' || *q == '-')) ++q;
  const char* m0 = q;
  while (q < e && *q >= '0' && *q <= '9') ++q;
  bool digits = q > m0;
  if (q < e && *q == '.') {
    ++q;
    const char* f0 = q;
    while (q < e && *q >= '0' && *q <= '9') ++q;
    digits = digits || q > f0;
  }
  if (!digits) return false;
  if (q < e && (*q == 'e' || *q == 'E')) {  // num_get takes the exponent marker and what follows
    ++q;
    if (q < e && (*q == '+' || *q == '-')) ++q;
    const char* x0 = q;
    while (q < e && *q >= '0' && *q <= '9') ++q;
    if (q == x0) return false;  // "1e" / "1e+": strtod stops before 'e' -> num_get fails
  }
  const char* num = s + ((*s == '+') ? 1 : 0);  // from_chars takes no leading '+'
  double x = 0.0;
  auto r = std::from_chars(num, q, x);
  if (r.ptr != q) return false;
  if (r.ec == std::errc::result_out_of_range) {
    // overflow fails like num_get; underflow yields strtod's value
    char buf[512];
    const size_t len = size_t(q - s);
    if (len >= sizeof(buf)) return false;
    std::memcpy(buf, s, len);
    buf[len] = '\0';
    char* end = nullptr;
    x = strtod_l(buf, &end, c_locale());
    if (end != buf + len) return false;
    if (x == HUGE_VAL || x == -HUGE_VAL) return false;
  } else if (r.ec != std::errc()) {
    return false;
  }
  v = x;
  p = q;
  return true;
}

struct Timer {  // DPT_TIMING=1: phase times on stderr
  bool on = std::getenv("DPT_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* w) {
    if (!on) return;
    auto n = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[dpt mm] %-22s %8.1f ms\n", w, std::chrono::duration<double, std::milli>(n - t).count());
    t = n;
  }
};

struct Trip {
  int64_t r, c;
  double re, im;
};

int threads_for(int requested, size_t lines) {
  int t = requested > 0 ? requested : int(std::thread::hardware_concurrency());
  if (t < 1) t = 1;
  if (size_t(t) > lines / 4096 + 1) t = int(lines / 4096 + 1);
  return t;
}

template <class F>
void parallel(int nt, F f) {
  if (nt <= 1) {
    f(0);
    return;
  }
  std::vector<std::thread> pool;
  for (int t = 0; t < nt; ++t) pool.emplace_back(f, t);
  for (auto& th : pool) th.join();
}

}  // namespace

// Uninitialised storage: value-initialising 100s of MB serially cost more
// than the parallel passes that fill it.
template <class T>
struct RawArray {
  std::unique_ptr<T[]> p;
  size_t n = 0;
  void alloc(size_t count) {
    p.reset(new T[count ? count : 1]);
    n = count;
  }
  T* data() { return p.get(); }
  T& operator[](size_t i) { return p[i]; }
};

struct dpt_mm_store {  // owned arrays behind a dpt_mm_matrix
  RawArray<int64_t> rowptr, colidx;
  RawArray<double> vals;
};

extern "C" {

int dpt_mm_read(const char* path, int threads, dpt_mm_matrix* out, dpt_error_info* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (!out) {
    set(err, DPT_ERR_INVALID_ARG, "dpt_mm_read: null output");
    return DPT_ERR_INVALID_ARG;
  }
  std::memset(out, 0, sizeof(*out));
  const std::string p(path ? path : "");
  Timer tm;
  try {
    // one read of the whole file
    RawArray<char> buf;
    size_t bytes = 0;
    {
      std::FILE* f = std::fopen(p.c_str(), "rb");
      if (!f) throw IoFail{p + ": cannot open for reading"};
      std::fseek(f, 0, SEEK_END);
      const long sz = std::ftell(f);
      std::fseek(f, 0, SEEK_SET);
      buf.alloc(sz > 0 ? size_t(sz) : 0);
      if (sz > 0) bytes = std::fread(buf.data(), 1, size_t(sz), f);
      std::fclose(f);
    }
    const char* const B = buf.data();
    const char* const E = B + bytes;
    auto line_end = [E](const char* q) {
      const void* nl = std::memchr(q, '\n', size_t(E - q));
      return nl ? static_cast<const char*>(nl) : E;
    };
    tm.mark("read");
    // getline semantics: '\n' terminates a line; a final unterminated line counts
    if (bytes == 0) throw IoFail{p + ": empty file"};
    const Line first{B, line_end(B)};
    // banner (matrix_market.cpp:29-57)
    bool coordinate = false, complex_field = false, symmetric = false;
    {
      const std::string hl(first.b, first.e);
      std::vector<std::string> tok;
      size_t i = 0;
      while (tok.size() < 5) {
        while (i < hl.size() && is_space(hl[i])) ++i;
        if (i >= hl.size()) break;
        size_t j = i;
        while (j < hl.size() && !is_space(hl[j])) ++j;
        tok.push_back(hl.substr(i, j - i));
        i = j;
      }
      while (tok.size() < 5) tok.push_back("");
      if (lower(tok[0]) != "%%matrixmarket" || lower(tok[1]) != "matrix")
        throw IoFail{p + ": malformed MatrixMarket banner"};
      const std::string fm = lower(tok[2]), fl = lower(tok[3]), sy = lower(tok[4]);
      if (fm == "coordinate")
        coordinate = true;
      else if (fm != "array")
        throw IoFail{p + ": unsupported format '" + tok[2] + "'"};
      if (fl == "complex")
        complex_field = true;
      else if (fl != "real")
        throw IoFail{p + ": unsupported field '" + tok[3] + "'"};
      if (sy == "symmetric")
        symmetric = true;
      else if (sy != "general")
        throw IoFail{p + ": unsupported symmetry '" + tok[4] + "'"};
    }
    // the size line: the first data line after the banner
    const char* q = first.e < E ? first.e + 1 : E;
    Line size_line{nullptr, nullptr};
    while (q < E) {
      const Line l{q, line_end(q)};
      q = l.e < E ? l.e + 1 : E;
      if (data_line(l)) {
        size_line = l;
        break;
      }
    }
    if (!size_line.b) throw IoFail{p + ": missing size line"};
    const char* const D0 = q;  // data region [D0, E)
    const int cx = complex_field ? 2 : 1;

    // Chunks of the data region start at line starts; pass 1 counts each
    // chunk's data lines, so every data line gets its global index.
    const size_t dbytes = size_t(E - D0);
    int nt = threads > 0 ? threads : int(std::thread::hardware_concurrency());
    if (nt < 1) nt = 1;
    if (size_t(nt) > dbytes / (1 << 16) + 1) nt = int(dbytes / (1 << 16) + 1);
    std::vector<const char*> cb(static_cast<size_t>(nt) + 1);
    cb[0] = D0;
    cb[size_t(nt)] = E;
    for (int t = 1; t < nt; ++t) {
      const char* c = D0 + dbytes * size_t(t) / size_t(nt);
      if (c > D0 && c[-1] != '\n') c = line_end(c) < E ? line_end(c) + 1 : E;
      cb[size_t(t)] = std::max(c, cb[size_t(t - 1)]);
    }
    std::vector<size_t> cnt(size_t(nt), 0);
    parallel(nt, [&](int t) {
      size_t c = 0;
      for (const char* l = cb[size_t(t)]; l < cb[size_t(t) + 1];) {
        const Line ln{l, line_end(l)};
        c += data_line(ln) ? 1 : 0;
        l = ln.e < E ? ln.e + 1 : E;
      }
      cnt[size_t(t)] = c;
    });
    std::vector<size_t> first_idx(size_t(nt) + 1, 0);
    for (int t = 0; t < nt; ++t) first_idx[size_t(t) + 1] = first_idx[size_t(t)] + cnt[size_t(t)];
    const size_t ndata = first_idx[size_t(nt)];
    tm.mark("split");
    // the first failing data line in file order, over all threads
    std::vector<size_t> fail_at(static_cast<size_t>(nt), SIZE_MAX);
    std::vector<int> fail_kind(static_cast<size_t>(nt), 0);
    std::vector<std::string> fail_line(static_cast<size_t>(nt));
    auto first_fail = [&](int* kind, std::string* line) {
      size_t best = SIZE_MAX;
      for (int t = 0; t < nt; ++t)
        if (fail_at[size_t(t)] < best) {
          best = fail_at[size_t(t)];
          *kind = fail_kind[size_t(t)];
          *line = fail_line[size_t(t)];
        }
      return best;
    };

    if (coordinate) {
      long long rows = -1, cols = -1, entries = -1;
      {
        const char* z = size_line.b;
        if (get_size(z, size_line.e, rows) && get_size(z, size_line.e, cols)) get_size(z, size_line.e, entries);
      }
      if (rows < 0 || cols < 0 || entries < 0) throw IoFail{p + ": malformed coordinate size line"};
      const size_t ne = size_t(entries);
      const size_t upto = std::min(ne, ndata);  // lines after the last entry are ignored
      // pass 2: parse; per-thread triplets in file order
      std::vector<std::vector<Trip>> part(static_cast<size_t>(nt));
      parallel(nt, [&](int t) {
        size_t g = first_idx[size_t(t)];
        if (g >= upto) return;
        auto& v = part[size_t(t)];
        v.reserve(std::min(upto - g, cnt[size_t(t)]) * (symmetric ? 2 : 1));
        for (const char* l = cb[size_t(t)]; l < cb[size_t(t) + 1] && g < upto;) {
          const Line ln{l, line_end(l)};
          l = ln.e < E ? ln.e + 1 : E;
          if (!data_line(ln)) continue;
          const char* z = ln.b;
          long long i = 0, j = 0;
          double re = 0.0, im = 0.0;
          bool ok = get_ll(z, ln.e, i) && get_ll(z, ln.e, j) && get_double(z, ln.e, re);
          if (ok && complex_field) ok = get_double(z, ln.e, im);
          if (!ok || i < 1 || i > rows || j < 1 || j > cols) {
            fail_at[size_t(t)] = g;
            fail_kind[size_t(t)] = ok ? 2 : 1;
            fail_line[size_t(t)] = std::string(ln.b, ln.e);
            return;
          }
          v.push_back(Trip{i - 1, j - 1, re, im});
          if (symmetric && i != j) v.push_back(Trip{j - 1, i - 1, re, im});
          ++g;
        }
      });
      {
        int kind = 0;
        std::string line;
        if (first_fail(&kind, &line) != SIZE_MAX) {
          if (kind == 1) throw IoFail{p + ": malformed entry line '" + line + "'"};
          throw IoFail{p + ": entry index out of bounds"};
        }
      }
      if (ndata < ne) throw IoFail{p + ": truncated entry list"};
      tm.mark("parse");
      // concatenate in file order (parallel copies)
      std::vector<size_t> off(size_t(nt) + 1, 0);
      for (int t = 0; t < nt; ++t) off[size_t(t) + 1] = off[size_t(t)] + part[size_t(t)].size();
      const size_t nt_total = off[size_t(nt)];
      RawArray<Trip> trips;
      trips.alloc(nt_total);
      parallel(nt, [&](int t) {
        std::copy(part[size_t(t)].begin(), part[size_t(t)].end(), trips.data() + off[size_t(t)]);
        std::vector<Trip>().swap(part[size_t(t)]);
      });
      // strictly increasing (row, col)?  then std::sort would be the identity
      auto less = [](const Trip& x, const Trip& y) { return x.r != y.r ? x.r < y.r : x.c < y.c; };
      std::atomic<bool> sorted{true};
      {
        const int ns = nt_total > (1 << 16) ? nt : 1;
        parallel(ns, [&](int t) {
          const size_t k0 = std::max<size_t>(1, nt_total * size_t(t) / size_t(ns)),
                       k1 = nt_total * size_t(t + 1) / size_t(ns);
          for (size_t k = k0; k < k1; ++k)
            if (!less(trips[k - 1], trips[k])) {
              sorted = false;
              return;
            }
        });
      }
      tm.mark("concat+check");
      auto* st = new dpt_mm_store();
      st->rowptr.alloc(size_t(rows) + 1);
      int64_t* rp = st->rowptr.data();
      if (sorted) {  // from_triplets without duplicates: a parallel copy
        st->colidx.alloc(nt_total);
        st->vals.alloc(nt_total * size_t(cx));
        const int ns = nt_total > (1 << 16) ? nt : 1;
        parallel(ns, [&](int t) {
          const size_t k0 = nt_total * size_t(t) / size_t(ns), k1 = nt_total * size_t(t + 1) / size_t(ns);
          for (size_t k = k0; k < k1; ++k) {
            const Trip& x = trips[k];
            st->colidx[k] = x.c;
            st->vals[k * size_t(cx)] = x.re;
            if (cx == 2) st->vals[k * size_t(cx) + 1] = x.im;
            // rows (prev row, this row] start at k; each boundary has one owner
            const int64_t prev = k == 0 ? -1 : trips[k - 1].r;
            for (int64_t r = prev + 1; r <= x.r; ++r) rp[r] = int64_t(k);
          }
        });
        const int64_t last = nt_total ? trips[nt_total - 1].r : -1;
        for (int64_t r = last + 1; r <= rows; ++r) rp[r] = int64_t(nt_total);
      } else {  // from_triplets (matrix.cpp:28-53) step by step
        std::sort(trips.data(), trips.data() + nt_total, less);
        std::vector<int64_t> ci;
        std::vector<double> vv;
        ci.reserve(nt_total);
        vv.reserve(nt_total * size_t(cx));
        std::fill(rp, rp + rows + 1, int64_t(0));
        for (size_t i = 0; i < nt_total;) {
          size_t j = i + 1;
          double vr = trips[i].re, vi = trips[i].im;
          while (j < nt_total && trips[j].r == trips[i].r && trips[j].c == trips[i].c) {
            vr += trips[j].re;  // complex += adds the parts independently
            vi += trips[j].im;
            ++j;
          }
          ci.push_back(trips[i].c);
          vv.push_back(vr);
          if (cx == 2) vv.push_back(vi);
          ++rp[size_t(trips[i].r) + 1];
          i = j;
        }
        for (long long r = 0; r < rows; ++r) rp[size_t(r) + 1] += rp[size_t(r)];
        st->colidx.alloc(ci.size());
        std::copy(ci.begin(), ci.end(), st->colidx.data());
        st->vals.alloc(vv.size());
        std::copy(vv.begin(), vv.end(), st->vals.data());
      }
      out->rows = rows;
      out->cols = cols;
      out->is_sparse = 1;
      out->is_complex = complex_field ? 1 : 0;
      out->nnz = int64_t(st->colidx.n);
      out->rowptr = st->rowptr.data();
      out->colidx = st->colidx.data();
      out->vals = st->vals.data();
      out->store = st;
      tm.mark("csr");
      return DPT_OK;
    }

    long long rows = -1, cols = -1;
    {
      const char* z = size_line.b;
      if (get_size(z, size_line.e, rows)) get_size(z, size_line.e, cols);
    }
    if (rows < 0 || cols < 0) throw IoFail{p + ": malformed array size line"};
    if (symmetric && rows != cols) throw IoFail{p + ": symmetric array must be square"};
    // column-major values, the lower triangle when symmetric (matrix_market.cpp:124-140);
    // value index k -> (i, j): col_base(j) = sum_{c<j} (rows - (sym ? c : 0))
    auto col_len = [&](long long j) { return size_t(rows - (symmetric ? j : 0)); };
    size_t need = 0;
    for (long long j = 0; j < cols; ++j) need += col_len(j);
    auto* st = new dpt_mm_store();
    st->vals.alloc(size_t(rows) * size_t(cols) * size_t(cx));  // every value is written below
    std::fill(st->vals.data(), st->vals.data() + st->vals.n, 0.0);
    const size_t upto = std::min(need, ndata);
    parallel(nt, [&](int t) {
      size_t g = first_idx[size_t(t)];
      if (g >= upto) return;
      long long j = 0;  // the column holding value g
      size_t base = 0;
      while (j < cols && base + col_len(j) <= g) {
        base += col_len(j);
        ++j;
      }
      long long i = (symmetric ? j : 0) + (long long)(g - base);
      for (const char* l = cb[size_t(t)]; l < cb[size_t(t) + 1] && g < upto;) {
        const Line ln{l, line_end(l)};
        l = ln.e < E ? ln.e + 1 : E;
        if (!data_line(ln)) continue;
        while (i >= rows) {
          ++j;
          i = symmetric ? j : 0;
        }
        const char* z = ln.b;
        double re = 0.0, im = 0.0;
        bool ok = get_double(z, ln.e, re);
        if (ok && complex_field) ok = get_double(z, ln.e, im);
        if (!ok) {
          fail_at[size_t(t)] = g;
          fail_kind[size_t(t)] = 1;
          fail_line[size_t(t)] = std::string(ln.b, ln.e);
          return;
        }
        double* dst = st->vals.data() + (size_t(i) * size_t(cols) + size_t(j)) * size_t(cx);  // row-major out
        dst[0] = re;
        if (cx == 2) dst[1] = im;
        if (symmetric && i != j) {
          double* mir = st->vals.data() + (size_t(j) * size_t(cols) + size_t(i)) * size_t(cx);
          mir[0] = re;
          if (cx == 2) mir[1] = im;
        }
        ++i;
        ++g;
      }
    });
    {
      int kind = 0;
      std::string line;
      if (first_fail(&kind, &line) != SIZE_MAX) {
        delete st;
        throw IoFail{p + ": malformed array value '" + line + "'"};
      }
    }
    if (ndata < need) {
      delete st;
      throw IoFail{p + ": truncated array data"};
    }
    out->rows = rows;
    out->cols = cols;
    out->is_sparse = 0;
    out->is_complex = complex_field ? 1 : 0;
    out->nnz = rows * cols;
    out->vals = st->vals.data();
    out->store = st;
    return DPT_OK;
  } catch (const IoFail& e) {
    set(err, DPT_ERR_IO, e.msg);
    return DPT_ERR_IO;
  } catch (const std::exception& e) {
    set(err, DPT_ERR_IO, p + ": " + e.what());
    return DPT_ERR_IO;
  }
}

void dpt_mm_free(dpt_mm_matrix* m) {
  if (!m) return;
  delete static_cast<dpt_mm_store*>(m->store);
  std::memset(m, 0, sizeof(*m));
}

}  // extern "C"

namespace {

// "%.17g" of v (+ " %.17g" of the imaginary part) and '\n' appended to out.
// std::to_chars(general, 17) is specified as printf's "%.17g" in the C locale
// (same digits, same exponent form), several times faster than snprintf.
void put_g17(std::string& out, double v) {
  char b[48];
  const auto r = std::to_chars(b, b + sizeof(b), v, std::chars_format::general, 17);
  out.append(b, size_t(r.ptr - b));
}

void put_value(std::string& out, double re, double im, bool cf) {
  put_g17(out, re);
  if (cf) {
    out.push_back(' ');
    put_g17(out, im);
  }
  out.push_back('\n');
}

void put_index(std::string& out, size_t v) {
  char b[24];
  const auto r = std::to_chars(b, b + sizeof(b), v);
  out.append(b, size_t(r.ptr - b));
}

int write_chunks(const std::string& path, const std::string& head, size_t units, int threads,
                 const std::function<void(size_t, size_t, std::string&)>& fmt, dpt_error_info* err) {
  std::FILE* f = std::fopen(path.c_str(), "w");
  if (!f) {
    set(err, DPT_ERR_IO, path + ": cannot open for writing");
    return DPT_ERR_IO;
  }
  std::fwrite(head.data(), 1, head.size(), f);
  const int nt = threads_for(threads, units);
  const size_t per = 1 << 16;  // units per batch
  for (size_t b0 = 0; b0 < units; b0 += per * size_t(nt)) {
    std::vector<std::string> bufs(static_cast<size_t>(nt));
    parallel(nt, [&](int t) {
      const size_t s0 = b0 + per * size_t(t), s1 = std::min(units, s0 + per);
      if (s0 < s1) fmt(s0, s1, bufs[size_t(t)]);
    });
    for (auto& s : bufs) std::fwrite(s.data(), 1, s.size(), f);
  }
  std::fclose(f);
  return DPT_OK;
}

}  // namespace

extern "C" {

// write_matrix_market(DenseMatrix) (matrix_market.cpp:170-178): array format,
// column-major, real field when every imaginary part is 0.  vals: row-major,
// interleaved (re, im) when is_complex.
int dpt_mm_write_dense(const char* path, int64_t rows, int64_t cols, const double* vals, int is_complex,
                       int threads, dpt_error_info* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  const int cx = is_complex ? 2 : 1;
  bool cf = false;
  if (is_complex)
    for (int64_t q = 0; q < rows * cols && !cf; ++q) cf = vals[2 * q + 1] != 0.0;
  char head[160];
  std::snprintf(head, sizeof(head), "%%%%MatrixMarket matrix array %s general\n%zu %zu\n", cf ? "complex" : "real",
                size_t(rows), size_t(cols));
  return write_chunks(path ? path : "", head, size_t(rows * cols), threads,
                      [&](size_t s0, size_t s1, std::string& o) {
                        for (size_t u = s0; u < s1; ++u) {  // unit u = column-major position
                          const size_t j = u / size_t(rows), i = u % size_t(rows);
                          const double* v = vals + (i * size_t(cols) + j) * size_t(cx);
                          put_value(o, v[0], cx == 2 ? v[1] : 0.0, cf);
                        }
                      },
                      err);
}

// write_matrix_market(SparseMatrix) (:180-191): coordinate format, row order.
int dpt_mm_write_csr(const char* path, int64_t rows, int64_t cols, const int64_t* rowptr, const int64_t* colidx,
                     const double* vals, int is_complex, int threads, dpt_error_info* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  const int cx = is_complex ? 2 : 1;
  const int64_t nnz = rows > 0 ? rowptr[rows] : 0;
  bool cf = false;
  if (is_complex)
    for (int64_t q = 0; q < nnz && !cf; ++q) cf = vals[2 * q + 1] != 0.0;
  char head[200];
  std::snprintf(head, sizeof(head), "%%%%MatrixMarket matrix coordinate %s general\n%zu %zu %zu\n",
                cf ? "complex" : "real", size_t(rows), size_t(cols), size_t(nnz));
  // units = entries; a binary search finds each entry's row
  return write_chunks(path ? path : "", head, size_t(nnz), threads,
                      [&](size_t s0, size_t s1, std::string& o) {
                        int64_t r = int64_t(std::upper_bound(rowptr, rowptr + rows + 1, int64_t(s0)) - rowptr) - 1;
                        for (size_t q = s0; q < s1; ++q) {
                          while (int64_t(q) >= rowptr[r + 1]) ++r;
                          put_index(o, size_t(r) + 1);
                          o.push_back(' ');
                          put_index(o, size_t(colidx[q]) + 1);
                          o.push_back(' ');
                          put_value(o, vals[q * size_t(cx)], cx == 2 ? vals[q * size_t(cx) + 1] : 0.0, cf);
                        }
                      },
                      err);
}

}  // extern "C"
