// solver.cu -- host driver of the DPT iteration and the C ABI (include/dpt_b200.h).
//
// The reference's loops run_full / run_single (proj/src/dpt.cpp:92-192,
// :194-293) become a stream of device work per iteration:
//     step kernel (K1 dense / K2 CSR / K3 row map)
//  -> fold (K4a)  [-> ncclAllReduce(max) of the stats when sharded]
//  -> decide (K4b, the reference's decision order, dpt_state.h)
//  -> cycle test (only when the window is on)
// Every kernel reads the launch index from the device state, so the host can
// enqueue a CHUNK of iterations without looking at results; launches after a
// terminal decision are no-ops.  The host syncs once per chunk, replays the
// trace log to the TraceSink in k order, and stops.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <exception>
#include <chrono>
#include <condition_variable>
#include <mutex>
#include <complex>
#include <cstring>
#include <set>
#include <cstdio>
#include <map>
#include <unordered_map>
#include <cmath>
#include <limits>
#include <memory>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/dpt_b200.h"
#include "dpt_kernels.h"
#include "dpt_state.h"

// ------------------------------------------------------------- NCCL (dlopen) --
// NCCL is bound at run time so the library loads on a CPU-only host and in a
// process where torch already mapped its own libnccl.so.2.
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef int (*nccl_get_unique_id_fn)(ncclUniqueId*);
typedef int (*nccl_comm_init_rank_fn)(ncclComm_t*, int, ncclUniqueId, int);
typedef int (*nccl_all_reduce_fn)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t);
typedef int (*nccl_all_gather_fn)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t);
typedef int (*nccl_comm_destroy_fn)(ncclComm_t);
struct NcclApi {
  void* h = nullptr;
  nccl_get_unique_id_fn get_unique_id = nullptr;
  nccl_comm_init_rank_fn comm_init_rank = nullptr;
  nccl_all_reduce_fn all_reduce = nullptr;
  nccl_all_gather_fn all_gather = nullptr;
  nccl_comm_destroy_fn comm_destroy = nullptr;
};
static NcclApi* nccl_api() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    api.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (api.h) {
      api.get_unique_id = (nccl_get_unique_id_fn)dlsym(api.h, "ncclGetUniqueId");
      api.comm_init_rank = (nccl_comm_init_rank_fn)dlsym(api.h, "ncclCommInitRank");
      api.all_reduce = (nccl_all_reduce_fn)dlsym(api.h, "ncclAllReduce");
      api.all_gather = (nccl_all_gather_fn)dlsym(api.h, "ncclAllGather");
      api.comm_destroy = (nccl_comm_destroy_fn)dlsym(api.h, "ncclCommDestroy");
    }
  }
  return api.all_reduce ? &api : nullptr;
}
static const int kNcclFloat64 = 8, kNcclMax = 2;

// Test-only stand-in for NCCL when several ranks share ONE device in one
// process (the pool gives one GPU per call): each rank is a dpt_ctx driven by
// its own host thread.  A collective is a host rendezvous at ENQUEUE time plus
// stream-ordered dependencies: every rank records an event after its input is
// produced, all ranks meet, each waits (cudaStreamWaitEvent) on every peer's
// event and reads the peers' buffers with a kernel / device copies, records a
// second event, all meet again, and each waits on every peer's second event
// before it may overwrite its input.  No kernel ever waits on another rank's
// kernel (no spin flags), so the ranks' work may run in any order on the GPU.
constexpr int kMaxLoopbackRanks = 8;

struct LoopbackGroup {
  ~LoopbackGroup() {
    for (cudaEvent_t e : ev_in) cudaEventDestroy(e);
    for (cudaEvent_t e : ev_out) cudaEventDestroy(e);
  }
  int world = 0;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  bool broken = false;
  std::vector<const void*> src;
  std::vector<cudaEvent_t> ev_in, ev_out;
  // Host barrier of the ranks' threads; false (and the group marked broken) on a
  // 120 s timeout or after another rank failed, so no rank hangs forever.
  bool barrier() {
    std::unique_lock<std::mutex> lk(m);
    if (broken) return false;
    const uint64_t g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return true;
    }
    if (!cv.wait_for(lk, std::chrono::seconds(120), [&] { return gen != g || broken; }) || broken) {
      broken = true;
      cv.notify_all();
      return false;
    }
    return true;
  }
  void fail() {
    std::lock_guard<std::mutex> lk(m);
    broken = true;
    cv.notify_all();
  }
};

struct dpt_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int rank = 0, world = 1;
  ncclComm_t comm = nullptr;
  std::shared_ptr<LoopbackGroup> loop;  // test-only loopback communicator (dpt_ctx_set_loopback)
  int64_t launches = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // Caching allocator: device blocks released by a call are kept for the next
  // call on this context (cudaMalloc / cudaFree synchronise and cost ~ms for
  // the 100 MB-scale iterate buffers).  All work of a call is stream-ordered on
  // `stream`, so a recycled block is never touched by stale kernels.
  // Ordered by (size, address): a request takes the smallest fitting size and,
  // among equal sizes, the lowest address -- independent of release order, so
  // an identical call sequence gets identical buffers (cached loop graphs hit).
  std::set<std::pair<size_t, void*>> free_blocks;
  size_t cached = 0;
  // pinned host snapshot buffers, kept across calls
  void* pinned = nullptr;
  size_t pinned_bytes = 0;
  // staging ring for large copies to / from PAGEABLE host memory (stage_copy)
  void* stage[2] = {nullptr, nullptr};
  cudaEvent_t stage_ev[2] = {nullptr, nullptr};
  // Instantiated device-loop graphs (drive_graph), keyed by every parameter
  // the captured launches depend on.  Repeated solves of one problem get the
  // same workspace blocks from the caching allocator, hence the same key, and
  // skip the ~0.45 ms instantiation.
  struct LoopGraph {
    std::vector<unsigned char> key;
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ge = nullptr;
    unsigned long long cond = 0;
    int64_t per_body = 0;
  };
  std::vector<LoopGraph> loop_graphs;  // most recent last, at most kMaxLoopGraphs
  int64_t graph_hits = 0, graph_misses = 0;
};

namespace {
thread_local dpt_ctx* t_ctx = nullptr;  // the context of the API call on this thread (set by Guard)

size_t round_block(size_t bytes) {
  const size_t g = bytes >= (size_t(1) << 20) ? (size_t(2) << 20) : 512;
  return (bytes + g - 1) / g * g;
}

void* ctx_malloc(size_t bytes, cudaError_t* e) {
  dpt_ctx* c = t_ctx;
  bytes = round_block(bytes);
  if (c) {
    auto it = c->free_blocks.lower_bound(std::make_pair(bytes, static_cast<void*>(nullptr)));
    if (it != c->free_blocks.end() && it->first <= bytes + bytes / 4) {
      void* p = it->second;
      c->cached -= it->first;
      c->free_blocks.erase(it);
      *e = cudaSuccess;
      return p;
    }
  }
  void* p = nullptr;
  *e = cudaMalloc(&p, bytes);
  if (*e != cudaSuccess && c && !c->free_blocks.empty()) {  // trim the cache and retry
    cudaGetLastError();
    for (auto& kv : c->free_blocks) cudaFree(kv.second);
    c->free_blocks.clear();
    c->cached = 0;
    *e = cudaMalloc(&p, bytes);
  }
  return p;
}

void ctx_release(void* p, size_t bytes) {
  dpt_ctx* c = t_ctx;
  if (!c) {
    cudaFree(p);
    return;
  }
  bytes = round_block(bytes);
  c->free_blocks.emplace(std::make_pair(bytes, p));
  c->cached += bytes;
  const size_t limit = size_t(48) << 30;  // keep at most 48 GiB cached
  while (c->cached > limit && !c->free_blocks.empty()) {
    auto it = c->free_blocks.begin();
    cudaFree(it->second);
    c->cached -= it->first;
    c->free_blocks.erase(it);
  }
}
}  // namespace

namespace {

using namespace dpt;

struct Fail {
  int code;
};

// NVTX range of one host phase (header-only NVTX v3: a no-op unless a tool
// such as nsys / ncu --nvtx is attached)
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
  Nvtx(const Nvtx&) = delete;
  Nvtx& operator=(const Nvtx&) = delete;
};

void set_err(dpt_error_info* e, int code, const std::string& msg) {
  if (!e) return;
  e->code = code;
  snprintf(e->message, sizeof(e->message), "%s", msg.c_str());
}

bool debug_sync() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DPT_DEBUG_SYNC");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

// CK: check a CUDA call; with DPT_DEBUG_SYNC=1 every launch is also synchronised
// so a device fault is attributed to the kernel that raised it.
#define CK(expr)                                                                        \
  do {                                                                                  \
    cudaError_t _e = (expr);                                                            \
    if (_e == cudaSuccess && debug_sync()) _e = cudaDeviceSynchronize();                \
    if (_e != cudaSuccess) {                                                            \
      set_err(err, DPT_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));   \
      throw Fail{DPT_ERR_CUDA};                                                         \
    }                                                                                   \
  } while (0)

// RAII device buffer
struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
  bool owned = true;  // false: a view of caller-owned device memory (never released)
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() {
    if (p && owned) ctx_release(p, bytes);
  }
  void view(const void* q) {
    p = const_cast<void*>(q);
    owned = false;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// Copy a problem array to the host in stream order: device inputs may have
// been produced by this context's own kernels (e.g. a homotopy stage) on its
// non-blocking stream, which the legacy-stream cudaMemcpy does not wait for.
cudaError_t to_host_ordered(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind) {
  if (bytes == 0) return cudaSuccess;
  if (kind == cudaMemcpyHostToHost) {
    std::memcpy(dst, src, bytes);
    return cudaSuccess;
  }
  cudaStream_t st = t_ctx ? t_ctx->stream : nullptr;
  cudaError_t e = cudaMemcpyAsync(dst, src, bytes, kind, st);
  if (e != cudaSuccess) return e;
  return cudaStreamSynchronize(st);
}

// ------------------------------------------------ staged host copies ----
// Copies between the device and PAGEABLE host memory (numpy arrays, the
// reference's std::vector / DenseMatrix storage) go through the driver's own
// bounce buffers at ~5-8 GB/s.  Large ones are staged here instead: a
// two-buffer pinned ring, the DMA of one chunk overlapping the host memcpy of
// the other, the host side split over several threads (which also spreads the
// first-touch page faults of a fresh destination).  Pinned / registered host
// memory and small copies keep the plain cudaMemcpy*Async.
constexpr size_t kStageBytes = size_t(32) << 20;
constexpr size_t kStageMin = size_t(4) << 20;

bool host_pageable(const void* q) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, q) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

int copy_threads() {
  static const int t = [] {
    const unsigned h = std::thread::hardware_concurrency();
    // measured on the GPU box (16 host threads, profiles/r01f_host_copy_threads.txt): a 537 MB
    // download into fresh pages takes 34.7 / 24.6 / 21.1 / 26.8 ms with 4 / 8 / 12 / 16 threads
    int v = int(std::max(1u, std::min(12u, h * 3 / 4)));
    if (const char* e = std::getenv("DPT_COPY_THREADS")) v = std::max(1, std::min(16, atoi(e)));
    return v;
  }();
  return t;
}

void par_memcpy(void* dst, const void* src, size_t bytes) {
  const int T = bytes >= (size_t(2) << 20) ? copy_threads() : 1;
  if (T == 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
  const size_t per = ((bytes + T - 1) / T + 4095) & ~size_t(4095);
  std::thread th[16];
  int nt = 0;
  for (int t = 1; t < T; ++t) {
    const size_t off = size_t(t) * per;
    if (off >= bytes) break;
    th[nt++] = std::thread(std::memcpy, static_cast<char*>(dst) + off, static_cast<const char*>(src) + off,
                           std::min(per, bytes - off));
  }
  std::memcpy(dst, src, std::min(per, bytes));
  for (int t = 0; t < nt; ++t) th[t].join();
}

cudaError_t stage_ready(dpt_ctx* ctx) {
  for (int b = 0; b < 2; ++b) {
    if (!ctx->stage[b]) {
      cudaError_t e = cudaMallocHost(&ctx->stage[b], kStageBytes);
      if (e != cudaSuccess) return e;
      e = cudaEventCreateWithFlags(&ctx->stage_ev[b], cudaEventDisableTiming);
      if (e != cudaSuccess) return e;
    }
    cudaError_t e = cudaEventSynchronize(ctx->stage_ev[b]);  // a previous staged upload may still read it
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// height rows of width bytes; device rows at pitch dpitch_dev, host rows dense
// (pitch = width).  Chunks are whole rows (or, for one long row, byte ranges).
cudaError_t stage_copy(dpt_ctx* ctx, void* dst, size_t dpitch, const void* src, size_t spitch, size_t width,
                       size_t height, cudaMemcpyKind kind) {
  cudaStream_t st = ctx->stream;
  const bool d2h = kind == cudaMemcpyDeviceToHost;
  const size_t total = width * height;
  static const bool timing = std::getenv("DPT_TIMING") != nullptr;
  const auto t_start = std::chrono::steady_clock::now();
  double t_host = 0.0;  // seconds in host memcpys
  struct Report {
    bool on;
    const std::chrono::steady_clock::time_point& t0;
    const double& th;
    size_t bytes;
    bool d2h;
    ~Report() {
      if (!on) return;
      const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      std::fprintf(stderr, "[dpt] staged %s %8.1f MB %8.1f us (%5.1f GB/s; host memcpy %8.1f us)\n", d2h ? "d2h" : "h2d",
                   bytes / 1e6, s * 1e6, bytes / s / 1e9, th * 1e6);
    }
  } report{timing, t_start, t_host, total, d2h};
  auto timed_memcpy = [&](void* dd, const void* ss, size_t nb) {
    const auto a = std::chrono::steady_clock::now();
    par_memcpy(dd, ss, nb);
    if (timing) t_host += std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count();
  };
  cudaError_t e = stage_ready(ctx);
  if (e != cudaSuccess) return e;
  // chunk geometry: rows per chunk, or bytes per chunk of a single row
  const bool by_rows = height > 1 && width <= kStageBytes;
  const size_t rows_per = by_rows ? kStageBytes / width : 0;
  const size_t nch = by_rows ? (height + rows_per - 1) / rows_per : (total + kStageBytes - 1) / kStageBytes;
  auto dev_op = [&](size_t i) -> cudaError_t {
    void* buf = ctx->stage[i & 1];
    if (by_rows) {
      const size_t r0 = i * rows_per, nr = std::min(rows_per, height - r0);
      if (d2h)
        e = cudaMemcpy2DAsync(buf, width, static_cast<const char*>(src) + r0 * spitch, spitch, width, nr, kind, st);
      else
        e = cudaMemcpy2DAsync(static_cast<char*>(dst) + r0 * dpitch, dpitch, buf, width, width, nr, kind, st);
    } else {
      const size_t o = i * kStageBytes, nb = std::min(kStageBytes, total - o);
      if (d2h)
        e = cudaMemcpyAsync(buf, static_cast<const char*>(src) + o, nb, kind, st);
      else
        e = cudaMemcpyAsync(static_cast<char*>(dst) + o, buf, nb, kind, st);
    }
    if (e != cudaSuccess) return e;
    return cudaEventRecord(ctx->stage_ev[i & 1], st);
  };
  auto host_span = [&](size_t i, size_t* off) -> size_t {  // host byte range of chunk i
    if (by_rows) {
      const size_t r0 = i * rows_per;
      *off = r0 * width;
      return std::min(rows_per, height - r0) * width;
    }
    *off = i * kStageBytes;
    return std::min(kStageBytes, total - *off);
  };
  if (d2h) {
    for (size_t i = 0; i < nch && i < 2; ++i)
      if ((e = dev_op(i)) != cudaSuccess) return e;
    for (size_t i = 0; i < nch; ++i) {
      if ((e = cudaEventSynchronize(ctx->stage_ev[i & 1])) != cudaSuccess) return e;
      size_t off;
      const size_t nb = host_span(i, &off);
      timed_memcpy(static_cast<char*>(dst) + off, ctx->stage[i & 1], nb);
      if (i + 2 < nch && (e = dev_op(i + 2)) != cudaSuccess) return e;
    }
  } else {
    for (size_t i = 0; i < nch; ++i) {
      if (i >= 2 && (e = cudaEventSynchronize(ctx->stage_ev[i & 1])) != cudaSuccess) return e;
      size_t off;
      const size_t nb = host_span(i, &off);
      timed_memcpy(ctx->stage[i & 1], static_cast<const char*>(src) + off, nb);
      if ((e = dev_op(i)) != cudaSuccess) return e;
    }
  }
  return cudaSuccess;
}

// cudaMemcpyAsync / cudaMemcpy2DAsync on the context's stream, staged when the
// host side is large and pageable.  Device-to-host copies return complete.
cudaError_t copy_async(dpt_ctx* ctx, void* dst, const void* src, size_t bytes, cudaMemcpyKind kind) {
  if (bytes == 0) return cudaSuccess;
  if ((kind == cudaMemcpyHostToDevice || kind == cudaMemcpyDeviceToHost) && bytes >= kStageMin &&
      host_pageable(kind == cudaMemcpyHostToDevice ? src : dst))
    return stage_copy(ctx, dst, bytes, src, bytes, bytes, 1, kind);
  return cudaMemcpyAsync(dst, src, bytes, kind, ctx->stream);
}

cudaError_t copy2d_async(dpt_ctx* ctx, void* dst, size_t dpitch, const void* src, size_t spitch, size_t width,
                         size_t height, cudaMemcpyKind kind) {
  if (width == 0 || height == 0) return cudaSuccess;
  const bool host_dense = kind == cudaMemcpyHostToDevice ? spitch == width : dpitch == width;
  if ((kind == cudaMemcpyHostToDevice || kind == cudaMemcpyDeviceToHost) && host_dense &&
      width * height >= kStageMin && host_pageable(kind == cudaMemcpyHostToDevice ? src : dst))
    return stage_copy(ctx, dst, dpitch, src, spitch, width, height, kind);
  return cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, kind, ctx->stream);
}

void dalloc(DBuf& b, size_t bytes, dpt_error_info* err) {
  if (bytes == 0) bytes = 16;
  cudaError_t e;
  b.p = ctx_malloc(bytes, &e);
  b.bytes = bytes;
  if (e != cudaSuccess) {
    set_err(err, DPT_ERR_CUDA, std::string("cudaMalloc(") + std::to_string(bytes) + "): " + cudaGetErrorString(e));
    throw Fail{DPT_ERR_CUDA};
  }
}

// ------------------------------------------------------------ gap policy ----
double spread_of(int64_t n, const double* d) {  // spectral_spread, partition.cpp:42-53
  if (n == 0) return 0.0;
  double lo = d[0], hi = d[0];
  for (int64_t i = 0; i < n; ++i) {
    lo = std::min(lo, d[i]);
    hi = std::max(hi, d[i]);
  }
  return std::hypot(hi - lo, 0.0);
}

double threshold_of(int64_t n, const double* d, double tol) {  // degeneracy_threshold, :57-59
  return tol * std::max(1.0, spread_of(n, d));
}

// build_theta's scan (partition.cpp:69-81) -- the first (i, j) in row-major
// order with |d_i - d_j| <= thresh -- in O(n log n): rounding of d_i - d_j is
// monotone in d_j, so the partners of i form a contiguous run of the sorted
// order around i, and i has a partner iff a sorted neighbour is within thresh.
bool find_degenerate(int64_t n, const double* d, double tol, int64_t* bi, int64_t* bj) {
  if (n < 2) return false;
  const double thresh = threshold_of(n, d, tol);
  std::vector<int64_t> ord(static_cast<size_t>(n));
  std::iota(ord.begin(), ord.end(), int64_t(0));
  std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) {
    const bool na = std::isnan(d[a]), nb = std::isnan(d[b]);
    if (na != nb) return nb;  // NaNs last
    if (na) return a < b;
    return d[a] < d[b];
  });
  std::vector<int64_t> pos(static_cast<size_t>(n));
  for (int64_t q = 0; q < n; ++q) pos[size_t(ord[size_t(q)])] = q;
  auto close = [&](int64_t a, int64_t b) { return std::fabs(d[a] - d[b]) <= thresh; };
  for (int64_t i = 0; i < n; ++i) {
    const int64_t q = pos[size_t(i)];
    const bool has = (q > 0 && close(i, ord[size_t(q - 1)])) || (q + 1 < n && close(i, ord[size_t(q + 1)]));
    if (!has) continue;
    int64_t best = std::numeric_limits<int64_t>::max();
    for (int64_t r = q - 1; r >= 0 && close(i, ord[size_t(r)]); --r) best = std::min(best, ord[size_t(r)]);
    for (int64_t r = q + 1; r < n && close(i, ord[size_t(r)]); ++r) best = std::min(best, ord[size_t(r)]);
    *bi = i;
    *bj = best;
    return true;
  }
  return false;
}

// build_gap_row's check for one chart row (partition.cpp:83-96): first m.
bool find_degenerate_row(int64_t n, const double* d, int64_t row, double tol, int64_t* bj) {
  const double thresh = threshold_of(n, d, tol);
  for (int64_t m = 0; m < n; ++m) {
    if (m == row) continue;
    if (std::fabs(d[row] - d[m]) <= thresh) {
      *bj = m;
      return true;
    }
  }
  return false;
}

// Complex levels (interleaved re, im): the same policies with |z| = hypot.
double spread_of_c(int64_t n, const double* d) {  // bounding box, partition.cpp:42-53
  if (n == 0) return 0.0;
  double rl = d[0], rh = d[0], il = d[1], ih = d[1];
  for (int64_t i = 0; i < n; ++i) {
    rl = std::min(rl, d[2 * i]);
    rh = std::max(rh, d[2 * i]);
    il = std::min(il, d[2 * i + 1]);
    ih = std::max(ih, d[2 * i + 1]);
  }
  return std::hypot(rh - rl, ih - il);
}

double threshold_of_c(int64_t n, const double* d, double tol) { return tol * std::max(1.0, spread_of_c(n, d)); }

// First (i, j) in row-major order with |d_i - d_j| <= thresh, for complex
// levels.  Points closer than thresh sit in neighbouring cells of a grid of
// pitch thresh, so a hash of cells answers "does i have a partner" in O(1);
// O(n^2) fallback when the grid would overflow or thresh is 0.
bool find_degenerate_c(int64_t n, const double* d, double tol, int64_t* bi, int64_t* bj) {
  if (n < 2) return false;
  const double t = threshold_of_c(n, d, tol);
  auto close = [&](int64_t a, int64_t b) { return std::hypot(d[2 * a] - d[2 * b], d[2 * a + 1] - d[2 * b + 1]) <= t; };
  double amax = 0.0;
  for (int64_t i = 0; i < 2 * n; ++i)
    if (std::isfinite(d[i])) amax = std::max(amax, std::fabs(d[i]));
  const bool grid = t > 0.0 && amax / t < 1e15;
  if (!grid) {
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = 0; j < n; ++j)
        if (i != j && close(i, j)) {
          *bi = i;
          *bj = j;
          return true;
        }
    return false;
  }
  std::unordered_map<uint64_t, std::vector<int64_t>> cells;
  auto key = [](int64_t x, int64_t y) { return (uint64_t(x) * 0x9E3779B97F4A7C15ull) ^ uint64_t(y); };
  auto cx = [&](int64_t i) { return int64_t(std::floor(d[2 * i] / t)); };
  auto cy = [&](int64_t i) { return int64_t(std::floor(d[2 * i + 1] / t)); };
  for (int64_t i = 0; i < n; ++i)
    if (std::isfinite(d[2 * i]) && std::isfinite(d[2 * i + 1])) cells[key(cx(i), cy(i))].push_back(i);
  for (int64_t i = 0; i < n; ++i) {
    if (!std::isfinite(d[2 * i]) || !std::isfinite(d[2 * i + 1])) continue;
    int64_t best = std::numeric_limits<int64_t>::max();
    for (int64_t ox = -2; ox <= 2; ++ox)
      for (int64_t oy = -2; oy <= 2; ++oy) {
        auto it = cells.find(key(cx(i) + ox, cy(i) + oy));
        if (it == cells.end()) continue;
        for (int64_t j : it->second)
          if (j != i && close(i, j)) best = std::min(best, j);
      }
    if (best != std::numeric_limits<int64_t>::max()) {
      *bi = i;
      *bj = best;
      return true;
    }
  }
  return false;
}

bool find_degenerate_row_c(int64_t n, const double* d, int64_t row, double tol, int64_t* bj) {
  const double t = threshold_of_c(n, d, tol);
  for (int64_t m = 0; m < n; ++m) {
    if (m == row) continue;
    if (std::hypot(d[2 * row] - d[2 * m], d[2 * row + 1] - d[2 * m + 1]) <= t) {
      *bj = m;
      return true;
    }
  }
  return false;
}

int effective_window(int requested, int64_t n) {  // dpt.cpp:83-90
  if (requested <= 0) return 0;
  const double entries = double(n) * double(n);
  const double cap = 4.0e6 / std::max(entries, 1.0);
  int win = requested;
  if (cap < win) win = int(cap);
  return win < 2 ? 0 : win;
}

void degenerate_error(dpt_error_info* err, int64_t i, int64_t j, const double* d, bool cplx = false) {
  if (err) {
    err->i = i;
    err->j = j;
    err->ei = cplx ? d[2 * i] : d[i];
    err->ej = cplx ? d[2 * j] : d[j];
    err->ei_im = cplx ? d[2 * i + 1] : 0.0;
    err->ej_im = cplx ? d[2 * j + 1] : 0.0;
  }
  set_err(err, DPT_ERR_DEGENERATE,
          "degenerate spectrum: levels " + std::to_string(i) + " and " + std::to_string(j) +
              " coincide within tolerance");
  throw Fail{DPT_ERR_DEGENERATE};
}

// with a communicator (NCCL or the test loopback) the solve is row-sharded
bool sharded(const dpt_ctx* ctx) { return ctx->comm != nullptr || ctx->loop != nullptr; }

// ------------------------------------------------------ device problem ----
struct DevProblem {
  int64_t n = 0, ld = 0, nnz = 0;
  int64_t ncol = 0;  // real columns per iterate row (n, or 2n when complex)
  int64_t ldd = 0;   // leading dimension of the device Delta image
  int cplx = 0;
  double lambda_im = 0.0;
  int kind = DPT_DELTA_DENSE;
  DBuf theta, delta, rowptr, cols, vals;
  DBuf dmap;  // CUtensorMap for dense Delta
  int big = 1;  // dense tile configuration (dense_cfg_for)
  int uniform16 = 0;  // CSR with exactly 16 nonzeros per row (K3 fast path)
  DBuf u16c_cols, u16c_vals;  // complex uniform-16: trip-major copy (complex_steps.cu)
  DBuf s_cols, s_vals, s_off, s_lcol, s_llen, s_pos;  // SELL-32 image (K2)
  DBuf s_perm, s_inv;                                 // column relabelling (bank balance), empty = identity
  DBuf s_cols16, s_lpos, s_ltheta;                    // packed copy for K2's shared-memory kernel (launch_sell_pack)
  int64_t nslices = 0, s_npad = 0;
  int csr_strict = 0;  // every CSR row's columns strictly increase (no repeated pair): launch_csr_init applies
  DevCsr csr() const { return DevCsr{rowptr.as<int64_t>(), cols.as<int32_t>(), vals.as<double>(), nnz}; }
  DevSell sell() const {
    return DevSell{s_cols.as<int32_t>(), s_vals.as<double>(), s_off.as<int64_t>(), s_lcol.as<int32_t>(),
                   s_llen.as<int32_t>(), s_pos.as<int64_t>(), nslices, s_perm.as<int32_t>(), s_inv.as<int32_t>(),
                   s_npad, s_cols16.as<uint16_t>(), s_lpos.as<int32_t>(), s_ltheta.as<double>()};
  }
};

// SELL-32 image of a CSR matrix for K2 (layout and bank-aware schedule:
// csrc/sell_build.cu), built on the device from the CSR already in HBM.
void build_sell_device(DevProblem& dp, cudaStream_t st, dpt_error_info* err) {
  const int64_t n = dp.n;
  const int64_t ns = (n + 31) / 32;
  const int cx = dp.cplx ? 2 : 1;
  const int G = dp.cplx ? 8 : 16;
  const char* sched_env = std::getenv("DPT_SELL_SCHED");
  // 2: free-order bank schedule (default); 1: CSR-order bank schedule; 0: dense packing
  const int sched = (sched_env && sched_env[0] >= '0' && sched_env[0] <= '2') ? sched_env[0] - '0' : 2;
  dalloc(dp.s_lcol, size_t(ns * 32) * 4, err);
  dalloc(dp.s_llen, size_t(ns * 32) * 4, err);
  dalloc(dp.s_pos, size_t(n) * 8 + 8, err);
  dalloc(dp.s_off, size_t(ns + 1) * 8, err);
  CK(cudaMemsetAsync(dp.s_lcol.p, 0xff, size_t(ns * 32) * 4, st));
  CK(cudaMemsetAsync(dp.s_llen.p, 0, size_t(ns * 32) * 4, st));
  CK(launch_sell_perm(dp.rowptr.as<int64_t>(), n, dp.s_lcol.as<int32_t>(), dp.s_llen.as<int32_t>(),
                      dp.s_pos.as<int64_t>(), st));
  // Real problems whose rows are staged in shared memory get their columns
  // relabelled for bank balance (sell_build.cu, relabel_kernel); the staged
  // row then has npad >= n positions, at most what keeps K2's natural R.
  DBuf tot;
  dalloc(tot, 16, err);
  CK(cudaMemsetAsync(tot.p, 0, 16, st));
  CK(launch_csr_order_check(dp.rowptr.as<int64_t>(), dp.cols.as<int32_t>(), n, tot.as<int32_t>() + 3, st));
  const int64_t per_bank = (n + 15) / 16;
  const int64_t cap = std::min<int64_t>(per_bank + 16, csr_staged_cols_max(n) / 16);
  const char* rl_env = std::getenv("DPT_SELL_RELABEL");
  const bool relabel = !dp.cplx && sched == 2 && n >= 64 && cap >= per_bank && !(rl_env && rl_env[0] == '0') &&
                       relabel_smem_bytes(ns) <= size_t(200 * 1024);
  dp.s_npad = n;
  DBuf scratch, bankb;  // released after the synchronize below
  if (relabel) {
    dalloc(scratch, size_t(3 * n + 1 + dp.nnz) * 4, err);
    dalloc(bankb, size_t(n) * 4, err);
    dalloc(dp.s_perm, size_t(n) * 4, err);
    dalloc(dp.s_inv, size_t(16 * cap) * 4, err);
    // Local-search passes of the relabelling (DPT_SELL_PASSES = 1..9).  One pass
    // brings c3's image from 14 384 to 12 500 steps; passes 2 and 3 reach 12 448
    // and 12 440 (K2 1.5734 vs 1.5688 ms per step) at 0.65 ms each -- more than
    // an 18-iteration solve gets back, so the default is one.
    const char* ps_env = std::getenv("DPT_SELL_PASSES");
    const int rl_passes = (ps_env && ps_env[0] >= '1' && ps_env[0] <= '9') ? ps_env[0] - '0' : 1;
    CK(launch_relabel(dp.rowptr.as<int64_t>(), dp.cols.as<int32_t>(), n, dp.nnz, ns, dp.s_pos.as<int64_t>(), int(cap),
                      rl_passes, scratch.as<int32_t>(), bankb.as<int32_t>(), dp.s_perm.as<int32_t>(), dp.s_inv.as<int32_t>(),
                      16 * cap, tot.as<int32_t>() + 2, st));
  }
  CK(launch_sell_widths(dp.rowptr.as<int64_t>(), dp.cols.as<int32_t>(), ns, dp.s_lcol.as<int32_t>(), G, sched,
                        dp.s_perm.as<int32_t>(), dp.s_off.as<int64_t>(), st));
  CK(launch_sell_scan(dp.s_off.as<int64_t>(), ns, tot.as<int64_t>(), st));
  int64_t total = 0;
  int32_t npad = 0;
  CK(cudaMemcpyAsync(&total, tot.p, 8, cudaMemcpyDeviceToHost, st));
  if (relabel) CK(cudaMemcpyAsync(&npad, tot.as<int32_t>() + 2, 4, cudaMemcpyDeviceToHost, st));
  int32_t disorder = 1;
  CK(cudaMemcpyAsync(&disorder, tot.as<int32_t>() + 3, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  dp.csr_strict = disorder == 0 ? 1 : 0;
  if (relabel) dp.s_npad = std::max<int64_t>(npad, n);
  if (std::getenv("DPT_SELL_DEBUG"))
    std::fprintf(stderr, "[dpt] SELL image: n=%lld slices=%lld steps=%lld sched=%d relabel=%d npad=%lld\n",
                 (long long)n, (long long)ns, (long long)(total / 32), sched, int(relabel), (long long)dp.s_npad);
  const int64_t alloc = std::max<int64_t>(total, 1);
  dalloc(dp.s_cols, size_t(alloc) * 4, err);
  dalloc(dp.s_vals, size_t(cx * alloc) * 8, err);
  CK(cudaMemsetAsync(dp.s_cols.p, 0xff, size_t(alloc) * 4, st));
  CK(cudaMemsetAsync(dp.s_vals.p, 0, size_t(cx * alloc) * 8, st));
  CK(launch_sell_fill(dp.rowptr.as<int64_t>(), dp.cols.as<int32_t>(), dp.vals.as<double>(), cx, ns,
                      dp.s_lcol.as<int32_t>(), G, sched, dp.s_perm.as<int32_t>(), dp.s_off.as<int64_t>(),
                      dp.s_cols.as<int32_t>(),
                      dp.s_vals.as<double>(), st));
  if (!dp.cplx && csr_staged_cols_max(n) > 0) {  // real rows that fit shared memory: positions < 65535
    dalloc(dp.s_cols16, size_t(alloc) * 2, err);
    dalloc(dp.s_lpos, size_t(ns * 32) * 4, err);
    dalloc(dp.s_ltheta, size_t(ns * 32) * 8, err);
    CK(launch_sell_pack(dp.s_cols.as<int32_t>(), dp.s_off.as<int64_t>(), ns, dp.s_lcol.as<int32_t>(),
                        dp.s_perm.as<int32_t>(), dp.theta.as<double>(), dp.s_cols16.as<uint16_t>(),
                        dp.s_lpos.as<int32_t>(), dp.s_ltheta.as<double>(), st));
  }
  dp.nslices = ns;
}

// allow_transposed: DPT_DELTA_DENSE_T (the caller passes Delta^T, the
// reference's cached delta_t) is accepted by the single-step entry points only.
void validate(const dpt_problem* p, dpt_error_info* err, bool allow_transposed = false) {
  if (!p || p->n < 0) {
    set_err(err, DPT_ERR_SHAPE, "problem: bad size");
    throw Fail{DPT_ERR_SHAPE};
  }
  if (p->n > 0 && !p->d) {
    set_err(err, DPT_ERR_SHAPE, "problem: missing levels");
    throw Fail{DPT_ERR_SHAPE};
  }
  if (p->delta_kind == DPT_DELTA_DENSE || (p->delta_kind == DPT_DELTA_DENSE_T && allow_transposed)) {
    if (p->n > 0 && !p->delta) {
      set_err(err, DPT_ERR_SHAPE, "problem: missing dense delta");
      throw Fail{DPT_ERR_SHAPE};
    }
  } else if (p->delta_kind == DPT_DELTA_CSR) {
    if (!p->rowptr || (p->nnz > 0 && (!p->cols || !p->vals))) {
      set_err(err, DPT_ERR_SHAPE, "problem: missing CSR arrays");
      throw Fail{DPT_ERR_SHAPE};
    }
  } else {
    set_err(err, DPT_ERR_INVALID_ARG, "problem: unknown delta kind");
    throw Fail{DPT_ERR_INVALID_ARG};
  }
}

void upload(DevProblem& dp, dpt_ctx* ctx, const dpt_problem* p, dpt_error_info* err, bool sell = false) {
  Nvtx nvtx_range("dpt.upload");
  validate(p, err, true);
  const int64_t n = p->n;
  const int cx = p->is_complex ? 2 : 1;  // doubles per scalar
  dp.n = n;
  dp.cplx = p->is_complex ? 1 : 0;
  dp.lambda_im = p->is_complex ? p->lambda_im : 0.0;
  dp.ncol = cx * n;
  dp.ld = (dp.ncol + 1) & ~int64_t(1);
  dp.kind = p->delta_kind == DPT_DELTA_CSR ? DPT_DELTA_CSR : DPT_DELTA_DENSE;  // Delta^T input is transposed below
  const bool dense_t = p->delta_kind == DPT_DELTA_DENSE_T;
  const cudaMemcpyKind k = p->mem == DPT_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  cudaStream_t st = ctx->stream;
  // Device-resident inputs whose layout the kernels take as is are used in
  // place (views); host inputs and re-laid-out arrays are copied.
  const bool dev = p->mem == DPT_MEM_DEVICE;
  auto aligned16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15u) == 0; };
  if (dev && n) {
    dp.theta.view(p->d);
  } else {
    dalloc(dp.theta, size_t(cx * n) * 8, err);
    if (n) CK(copy_async(ctx, dp.theta.p, p->d, size_t(cx * n) * 8, k));
  }
  if (p->delta_kind != DPT_DELTA_CSR) {
    if (dp.cplx || dense_t) {
      // Complex: the real image B (2n x 2n): row 2j = (Re D(j,k), -Im D(j,k))_k,
      // row 2j+1 = (Im D(j,k), Re D(j,k))_k, so the real NT GEMM of the
      // interleaved iterate with B yields (Re P, Im P) pairs.  Delta^T input:
      // transposed on the way.  Both are built on the device (delta_image_kernel)
      // from the caller's array, used in place when device-resident.
      dp.ldd = dp.cplx ? 2 * n : dp.ld;
      dalloc(dp.delta, size_t(dp.cplx ? 2 * n : n) * size_t(dp.ldd) * 8 + 64, err);
      DBuf raw;
      const double* src = p->delta;
      if (!dev && n) {
        dalloc(raw, size_t(cx) * size_t(n) * size_t(n) * 8, err);
        CK(copy_async(ctx, raw.p, p->delta, size_t(cx) * size_t(n) * size_t(n) * 8, k));
        src = raw.as<double>();
      }
      if (n) CK(launch_delta_image(src, n, cx, dense_t ? 1 : 0, dp.delta.as<double>(), dp.ldd, st));
      ctx->launches += 1;
      CK(cudaStreamSynchronize(st));  // raw goes out of scope
    } else if (dev && n && dp.ld == n && aligned16(p->delta)) {
      dp.ldd = dp.ld;
      dp.delta.view(p->delta);  // TMA-ready as is: 16-byte aligned, even leading dimension
    } else {
      dp.ldd = dp.ld;
      dalloc(dp.delta, size_t(n) * size_t(dp.ldd) * 8 + 64, err);
      if (n) {
        if (dp.ldd == n)
          CK(copy_async(ctx, dp.delta.p, p->delta, size_t(n) * size_t(n) * 8, k));
        else
          CK(copy2d_async(ctx, dp.delta.p, size_t(dp.ldd) * 8, p->delta, size_t(n) * 8, size_t(n) * 8, size_t(n), k));
      }
    }
  } else {
    int64_t nnz = p->nnz;
    if (p->mem == DPT_MEM_HOST) {
      nnz = p->rowptr[n];
    } else {
      CK(to_host_ordered(&nnz, p->rowptr + n, 8, cudaMemcpyDeviceToHost));
    }
    dp.nnz = nnz;
    if (dev && nnz && aligned16(p->cols) && aligned16(p->vals) && aligned16(p->rowptr)) {
      dp.rowptr.view(p->rowptr);  // K3 reads int4 / double2 vectors: 16-byte alignment
      dp.cols.view(p->cols);
      dp.vals.view(p->vals);
    } else {
      dalloc(dp.rowptr, size_t(n + 1) * 8, err);
      dalloc(dp.cols, size_t(nnz) * 4, err);
      dalloc(dp.vals, size_t(cx * nnz) * 8, err);
      CK(copy_async(ctx, dp.rowptr.p, p->rowptr, size_t(n + 1) * 8, k));
      if (nnz) {
        CK(copy_async(ctx, dp.cols.p, p->cols, size_t(nnz) * 4, k));
        CK(copy_async(ctx, dp.vals.p, p->vals, size_t(cx * nnz) * 8, k));
      }
    }
    if (sell) {
      build_sell_device(dp, st, err);
    } else if (n > 0 && nnz == 16 * n) {  // K3's uniform-16 fast path, tested on the device
      DBuf bad;
      dalloc(bad, 16, err);
      CK(cudaMemsetAsync(bad.p, 0, 4, st));
      CK(launch_rowptr_uniform(dp.rowptr.as<int64_t>(), n, 16, bad.as<unsigned>(), st));
      unsigned hb = 1;
      CK(cudaMemcpyAsync(&hb, bad.p, 4, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      dp.uniform16 = hb == 0 ? 1 : 0;
      if (dp.uniform16 && dp.cplx) {  // complex: trip-major copy for the per-warp pipeline
        const int64_t trips = (n + 31) / 32;
        dalloc(dp.u16c_cols, size_t(trips) * 512 * 4, err);
        dalloc(dp.u16c_vals, size_t(trips) * 512 * 16, err);
        CK(cudaMemsetAsync(dp.u16c_cols.p, 0, size_t(trips) * 512 * 4, st));
        CK(cudaMemsetAsync(dp.u16c_vals.p, 0, size_t(trips) * 512 * 16, st));
        CK(launch_u16c_build(dp.cols.as<int32_t>(), dp.vals.as<double>(), n, dp.u16c_cols.as<int32_t>(),
                             dp.u16c_vals.as<double>(), st));
      }
    }
  }
}

// ----------------------------------------------------------- workspace ----
struct Work {
  DevSolve s{};
  DBuf initpart;  // launch_csr_init scratch (CSR full map from the identity)
  DBuf slots, dvec, eps, res, rowpart, tilepart, blockpart, stats, state, trace, counter, cyclepart,
      amaps, lam_table, settled_table, sk_ws, sk_cnt;
  int ntiles_step = 0;
  int max_trace = 0;
  dpt_sm_state* h_state = nullptr;  // pinned (the context's cached host buffer)
  double* h_trace = nullptr;        // pinned
};

enum Mode { MODE_DENSE_FULL, MODE_CSR_FULL, MODE_SINGLE };

void make_work(Work& w, dpt_ctx* ctx, DevProblem& dp, Mode mode, int64_t row0, int64_t rows,
               int64_t rows_alloc, int nslots,
               int max_iter, const std::vector<double>* lam_tab, const std::vector<int>* set_tab,
               const dpt_sm_options& so, double lambda, int fixed_mode, dpt_error_info* err) {
  DevSolve& s = w.s;
  std::memset(&s, 0, sizeof(s));  // padding too: the bytes key the cached loop graphs
  s.n = dp.n;
  s.ld = dp.ld;
  s.ncol = dp.ncol;
  s.ldd = dp.ldd;
  s.cplx = dp.cplx;
  s.lambda_im = dp.lambda_im;
  const int cx = dp.cplx ? 2 : 1;
  s.row0 = row0;
  s.rows = rows;
  s.nslots = nslots;
  s.lambda = lambda;
  s.opts = so;
  s.fixed_mode = fixed_mode;
  s.fuse_decide = sharded(ctx) ? 0 : 1;  // with a communicator the stats are max-allreduced first
  int ntiles_aux = 1;
  if (mode == MODE_DENSE_FULL) {
    dp.big = dense_cfg_for(dp.n, rows);
    s.ntn = int((dp.ncol + dense_tile_n(dp.big) - 1) / dense_tile_n(dp.big));
    w.ntiles_step = dense_step_ntiles(rows, s.ntn, dp.big);
    ntiles_aux = dense_init_ntiles(rows, s.ntn, dp.cplx);
  } else if (mode == MODE_CSR_FULL) {
    s.ntn = csr_ntn(dp.n);
    w.ntiles_step = dp.cplx ? csr_cplx_ntiles(rows, dp.n) : csr_step_ntiles(rows, dp.n);
  } else if (dp.cplx) {
    s.ntn = single_cplx_ntiles(dp.n, dp.kind == DPT_DELTA_DENSE, dp.u16c_cols.p != nullptr);
    w.ntiles_step = s.ntn;
  } else {
    const int sm = single_mode(dp.kind == DPT_DELTA_DENSE, dp.uniform16);
    s.ntn = single_ntn(dp.n, sm);
    w.ntiles_step = single_ntiles(dp.n, sm);
  }
  s.ntiles = std::max(w.ntiles_step, ntiles_aux);
  const size_t slot_elems = size_t(std::max<int64_t>(rows_alloc, 1)) * size_t(dp.ld);
  s.slot_elems = int64_t(slot_elems);
  dalloc(w.slots, size_t(nslots) * slot_elems * 8 + 64, err);
  dalloc(w.dvec, size_t(2 * cx) * size_t(rows) * 8, err);
  dalloc(w.eps, size_t(cx) * size_t(std::max<int64_t>(rows_alloc, 1)) * 8, err);
  dalloc(w.res, size_t(std::max<int64_t>(rows_alloc, 1)) * 8, err);
  dalloc(w.rowpart, size_t(4) * size_t(s.ntn) * size_t(rows) * 8, err);
  dalloc(w.tilepart, size_t(s.ntiles) * 4 * 8, err);
  dalloc(w.blockpart, size_t(fold_blocks(rows) + 512) * 8 * 8, err);
  dalloc(w.stats, DPT_NSTATS * 8, err);
  dalloc(w.state, sizeof(dpt_sm_state), err);
  w.max_trace = (max_iter > 0 ? max_iter : 0) + 2;
  dalloc(w.trace, size_t(w.max_trace) * 3 * 8, err);
  dalloc(w.counter, 16, err);
  dalloc(w.cyclepart, size_t(512) * DPT_MAX_WINDOW * 8, err);
  if (mode == MODE_CSR_FULL) dalloc(w.initpart, size_t(rows + 4) * 8, err);
  s.theta = dp.theta.as<double>();
  s.slots = w.slots.as<double>();
  s.dvec[0] = w.dvec.as<double>();
  s.dvec[1] = w.dvec.as<double>() + cx * rows;
  s.eps = w.eps.as<double>();
  s.res = w.res.as<double>();
  s.rowpart = w.rowpart.as<double>();
  s.tilepart = w.tilepart.as<double>();
  s.blockpart = w.blockpart.as<double>();
  s.stats = w.stats.as<double>();
  s.state = w.state.as<dpt_sm_state>();
  s.trace = w.trace.as<double>();
  s.counter = w.counter.as<unsigned int>();
  s.cyclepart = w.cyclepart.as<double>();
  cudaStream_t st = ctx->stream;
  CK(cudaMemsetAsync(w.counter.p, 0, 16, st));
  CK(cudaMemsetAsync(w.state.p, 0, sizeof(dpt_sm_state), st));
  CK(cudaMemsetAsync(w.dvec.p, 0, size_t(2 * cx) * size_t(rows) * 8, st));
  CK(cudaMemsetAsync(w.rowpart.p, 0, size_t(4) * size_t(s.ntn) * size_t(rows) * 8, st));
  std::vector<double> ones(DPT_NSTATS, 1.0);
  CK(cudaMemcpyAsync(w.stats.p, ones.data(), DPT_NSTATS * 8, cudaMemcpyHostToDevice, st));
  if (lam_tab) {
    dalloc(w.lam_table, lam_tab->size() * 8, err);
    CK(cudaMemcpyAsync(w.lam_table.p, lam_tab->data(), lam_tab->size() * 8, cudaMemcpyHostToDevice, st));
    s.lam_table = w.lam_table.as<double>();
  }
  if (set_tab) {
    dalloc(w.settled_table, set_tab->size() * 4, err);
    CK(cudaMemcpyAsync(w.settled_table.p, set_tab->data(), set_tab->size() * 4, cudaMemcpyHostToDevice, st));
    s.settled_table = w.settled_table.as<int>();
  }
  if (mode == MODE_DENSE_FULL && dp.n > 0) {
    // tensor maps: one per ring slot (A) + one for Delta; kept in device memory
    const int box = dense_tile_m(dp.big);
    std::vector<CUtensorMap> maps(static_cast<size_t>(nslots));
    for (int q = 0; q < nslots; ++q) {
      if (make_tmap_rowmajor(&maps[size_t(q)], s.slots + size_t(q) * slot_elems, dp.ncol, rows, dp.ld, box) != 0) {
        set_err(err, DPT_ERR_CUDA, "cuTensorMapEncodeTiled failed for an iterate slot");
        throw Fail{DPT_ERR_CUDA};
      }
    }
    dalloc(w.amaps, sizeof(CUtensorMap) * size_t(nslots), err);
    CK(cudaMemcpyAsync(w.amaps.p, maps.data(), sizeof(CUtensorMap) * size_t(nslots), cudaMemcpyHostToDevice, st));
    // stream-K K1 for the small-tile configuration (dense_step.cu): partial-tile
    // slots per resident CTA and per-tile counters (zero; the kernel re-zeroes)
    const char* sk_env = std::getenv("DPT_DENSE_SK");
    if (dp.big == 0 && dp.cplx && !(sk_env && sk_env[0] == '0')) {  // (used for complex problems)
      const int g = dense_sk_grid(dp.cplx);
      dalloc(w.sk_ws, size_t(g) * 2 * dense_sk_part_doubles() * 8, err);
      dalloc(w.sk_cnt, size_t(std::max(w.ntiles_step, 1)) * 4, err);
      CK(cudaMemsetAsync(w.sk_cnt.p, 0, size_t(std::max(w.ntiles_step, 1)) * 4, st));
      s.sk_ws = w.sk_ws.as<double>();
      s.sk_cnt = w.sk_cnt.as<unsigned>();
    }
    if (!dp.dmap.p) {
      CUtensorMap dm;
      if (make_tmap_rowmajor(&dm, dp.delta.as<double>(), dp.ncol, dp.ncol, dp.ldd, dense_tile_n(dp.big)) != 0) {
        set_err(err, DPT_ERR_CUDA, "cuTensorMapEncodeTiled failed for Delta");
        throw Fail{DPT_ERR_CUDA};
      }
      dalloc(dp.dmap, sizeof(CUtensorMap), err);
      CK(cudaMemcpyAsync(dp.dmap.p, &dm, sizeof(CUtensorMap), cudaMemcpyHostToDevice, st));
    }
  }
  {
    const size_t need = 2 * sizeof(dpt_sm_state) + 64 + size_t(w.max_trace) * 3 * 8;
    if (ctx->pinned_bytes < need) {
      if (ctx->pinned) cudaFreeHost(ctx->pinned);
      ctx->pinned = nullptr;
      ctx->pinned_bytes = 0;
      CK(cudaMallocHost(&ctx->pinned, need));
      ctx->pinned_bytes = need;
    }
    w.h_state = static_cast<dpt_sm_state*>(ctx->pinned);
    w.h_trace = reinterpret_cast<double*>(static_cast<char*>(ctx->pinned) + 2 * sizeof(dpt_sm_state) + 64);
  }
}

// ---- loopback collectives (LoopbackGroup) ----
struct PeerPtrs {
  const double* p[kMaxLoopbackRanks];
};

__global__ void loop_max_kernel(PeerPtrs in, int world, int count, double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  double v = in.p[0][i];
  for (int r = 1; r < world; ++r) v = fmax(v, in.p[r][i]);  // ncclMax of the statistics
  out[i] = v;
}

void loop_meet(dpt_ctx* ctx, dpt_error_info* err) {
  if (!ctx->loop->barrier()) {
    set_err(err, DPT_ERR_NCCL, "loopback collective: a peer rank failed or timed out");
    throw Fail{DPT_ERR_NCCL};
  }
}

// in-place max-allreduce of `count` doubles (count <= 1024)
void loop_allreduce_max(dpt_ctx* ctx, double* buf, int count, dpt_error_info* err) {
  LoopbackGroup& G = *ctx->loop;
  const int r = ctx->rank;
  cudaStream_t st = ctx->stream;
  DBuf tmp;
  dalloc(tmp, size_t(count) * 8, err);
  G.src[r] = buf;
  CK(cudaEventRecord(G.ev_in[r], st));
  loop_meet(ctx, err);
  PeerPtrs pp{};
  for (int q = 0; q < G.world; ++q) {
    if (q != r) CK(cudaStreamWaitEvent(st, G.ev_in[q], 0));
    pp.p[q] = static_cast<const double*>(G.src[q]);
  }
  loop_max_kernel<<<(count + 255) / 256, 256, 0, st>>>(pp, G.world, count, tmp.as<double>());
  CK(cudaGetLastError());
  ctx->launches += 1;
  CK(cudaEventRecord(G.ev_out[r], st));
  loop_meet(ctx, err);
  for (int q = 0; q < G.world; ++q)
    if (q != r) CK(cudaStreamWaitEvent(st, G.ev_out[q], 0));  // every peer has read `buf`
  CK(cudaMemcpyAsync(buf, tmp.p, size_t(count) * 8, cudaMemcpyDeviceToDevice, st));
  loop_meet(ctx, err);  // the exchange slots (src, events) are free again
}

// all-gather of `count` doubles per rank into dst[world * count]
void loop_all_gather(dpt_ctx* ctx, const double* src, double* dst, size_t count, dpt_error_info* err) {
  LoopbackGroup& G = *ctx->loop;
  const int r = ctx->rank;
  cudaStream_t st = ctx->stream;
  G.src[r] = src;
  CK(cudaEventRecord(G.ev_in[r], st));
  loop_meet(ctx, err);
  for (int q = 0; q < G.world; ++q) {
    if (q != r) CK(cudaStreamWaitEvent(st, G.ev_in[q], 0));
    CK(cudaMemcpyAsync(dst + size_t(q) * count, G.src[q], count * 8, cudaMemcpyDeviceToDevice, st));
  }
  CK(cudaEventRecord(G.ev_out[r], st));
  loop_meet(ctx, err);
  for (int q = 0; q < G.world; ++q)
    if (q != r) CK(cudaStreamWaitEvent(st, G.ev_out[q], 0));  // every peer has copied `src`
  loop_meet(ctx, err);
}

// C2 all-gather through NCCL or the loopback group
void comm_all_gather(dpt_ctx* ctx, const double* src, double* dst, size_t count, const char* what,
                     dpt_error_info* err) {
  if (ctx->loop) {
    loop_all_gather(ctx, src, dst, count, err);
    return;
  }
  NcclApi* api = nccl_api();
  if (!api || api->all_gather(src, dst, count, kNcclFloat64, ctx->comm, ctx->stream) != 0) {
    set_err(err, DPT_ERR_NCCL, std::string("ncclAllGather of ") + what + " failed");
    throw Fail{DPT_ERR_NCCL};
  }
}

void allreduce_stats(dpt_ctx* ctx, Work& w, dpt_error_info* err) {
  if (ctx->loop) {
    loop_allreduce_max(ctx, w.s.stats, DPT_NSTATS, err);
    return;
  }
  if (!ctx->comm) return;
  NcclApi* api = nccl_api();
  if (!api || api->all_reduce(w.s.stats, w.s.stats, DPT_NSTATS, kNcclFloat64, kNcclMax, ctx->comm, ctx->stream) != 0) {
    set_err(err, DPT_ERR_NCCL, "ncclAllReduce(max) of the iteration statistics failed");
    throw Fail{DPT_ERR_NCCL};
  }
}

// One iteration's device work after the step kernel.
void post_step(dpt_ctx* ctx, Work& w, int ntiles, int64_t cycle_elems, dpt_error_info* err) {
  CK(launch_fold(w.s, ntiles, ctx->stream));
  ctx->launches += 1;
  if (!w.s.fuse_decide) {  // sharded: cross-rank max of the statistics, then the decision
    allreduce_stats(ctx, w, err);
    CK(launch_decide(w.s, ctx->stream));
    ctx->launches += 1;
  }
  if (w.s.opts.win > 0 && !w.s.fixed_mode) {
    CK(launch_cycle(w.s, cycle_elems, ctx->stream));
    ctx->launches += 1;
  }
}

void step_launch(dpt_ctx* ctx, Work& w, DevProblem& dp, Mode mode, int64_t row, dpt_error_info* err) {
  if (mode == MODE_DENSE_FULL)
    CK(launch_dense_step(w.s, w.amaps.as<CUtensorMap>(), dp.dmap.as<CUtensorMap>(), dp.delta.as<double>(),
                         dp.big, ctx->stream));
  else if (mode == MODE_CSR_FULL && dp.cplx)
    CK(launch_csr_step_cplx(w.s, dp.sell(), ctx->stream));
  else if (mode == MODE_CSR_FULL)
    CK(launch_csr_step(w.s, dp.sell(), ctx->stream));
  else if (dp.cplx)
    CK(launch_single_cplx(w.s, dp.csr(), dp.kind == DPT_DELTA_DENSE ? dp.delta.as<double>() : nullptr,
                          dp.u16c_cols.as<int32_t>(), dp.u16c_vals.as<double>(), row, ctx->stream));
  else
    CK(launch_single_step(w.s, dp.csr(), dp.kind == DPT_DELTA_DENSE ? dp.delta.as<double>() : nullptr, row,
                          single_mode(dp.kind == DPT_DELTA_DENSE, dp.uniform16), ctx->stream));
  ctx->launches += 1;
}

bool graph_loop_enabled() {
  const char* e = std::getenv("DPT_GRAPH_LOOP");
  return !(e && e[0] == '0');
}

void replay_trace(Work& w, int nt, int from, dpt_trace_fn trace, void* user, dpt_error_info* err) {
  if (!trace || nt <= from) return;
  CK(cudaMemcpy(w.h_trace, w.s.trace, size_t(nt) * 3 * 8, cudaMemcpyDeviceToHost));
  for (int q = from; q < nt; ++q)
    if (trace(int(w.h_trace[3 * q]), w.h_trace[3 * q + 1], w.h_trace[3 * q + 2], user) != 0) {
      set_err(err, DPT_ERR_TRACE, "trace sink aborted the iteration");
      throw Fail{DPT_ERR_TRACE};
    }
}

// Device-side iteration loop (single rank): one CUDA graph whose WHILE
// conditional node repeats {step, fold (+decision), cycle}; the decision in
// the fold's last block sets the loop condition, so the loop stops exactly at
// the terminal launch -- no host round trips, no speculative no-op launches.
// The trace log is replayed to the sink afterwards, in k order.
constexpr size_t kMaxLoopGraphs = 8;

template <class T>
void key_add(std::vector<unsigned char>& k, const T& v) {
  const unsigned char* p = reinterpret_cast<const unsigned char*>(&v);
  k.insert(k.end(), p, p + sizeof(T));
}

// Development knobs that select kernels (tuning runs and tests switch them
// between calls in one process): part of the loop-graph key, so a graph
// captured under one selection is never replayed under another.
static const char* const kKernelKnobs[] = {"DPT_U16_VARIANT", "DPT_DENSE_CFG", "DPT_SMALL8", "DPT_CSR_ROWS",
                                           "DPT_SELL_SCHED", "DPT_SELL_RELABEL", "DPT_CPLX_U16", "DPT_DENSE_SK", "DPT_SHARD_EMULATE"};

void key_add_knobs(std::vector<unsigned char>& k) {
  for (const char* name : kKernelKnobs) {
    const char* v = std::getenv(name);
    k.push_back(v ? 1 : 0);
    if (v) k.insert(k.end(), v, v + std::strlen(v) + 1);
  }
}

void drive_graph(dpt_ctx* ctx, Work& w, DevProblem& dp, Mode mode, int64_t row, int total, int issued,
                 int64_t cycle_elems, dpt_trace_fn trace, void* user, dpt_error_info* err) {
  Nvtx nvtx_range("dpt.device_loop");
  cudaStream_t st = ctx->stream;
  struct LoopReset {
    DevSolve* s;
    ~LoopReset() { s->has_loop = 0; }
  } lr{&w.s};
  // every input of the captured launches (step_launch + post_step)
  std::vector<unsigned char> key;
  key_add(key, w.s);
  key_add(key, int(mode));
  key_add(key, row);
  key_add(key, total);
  key_add(key, cycle_elems);
  key_add(key, w.ntiles_step);
  key_add(key, w.amaps.p);
  // every device buffer and scalar of the problem, so no buffer a launch reads
  // can be left out of the key (a cache block handed out again at another
  // address must never replay a graph holding the old one)
  for (const DBuf* b : {&dp.theta, &dp.delta, &dp.rowptr, &dp.cols, &dp.vals, &dp.dmap, &dp.u16c_cols,
                        &dp.u16c_vals, &dp.s_cols, &dp.s_vals, &dp.s_off, &dp.s_lcol, &dp.s_llen, &dp.s_pos,
                        &dp.s_perm, &dp.s_inv, &dp.s_cols16, &dp.s_lpos, &dp.s_ltheta})
    key_add(key, b->p);
  for (int64_t v : {dp.n, dp.ld, dp.nnz, dp.ncol, dp.ldd, dp.nslices, dp.s_npad}) key_add(key, v);
  key_add(key, dp.lambda_im);
  key_add(key, dp.big);
  key_add(key, dp.cplx);
  key_add(key, dp.kind);
  key_add(key, dp.uniform16);
  key_add_knobs(key);
  dpt_ctx::LoopGraph* hit = nullptr;
  for (auto& lg : ctx->loop_graphs)
    if (lg.key == key) hit = &lg;
  static const bool dbg = std::getenv("DPT_GRAPH_DEBUG") != nullptr;
  if (dbg) std::fprintf(stderr, "[dpt] loop graph %s (%zu cached)\n", hit ? "hit" : "miss", ctx->loop_graphs.size());
  ++(hit ? ctx->graph_hits : ctx->graph_misses);
  if (!hit) {
    dpt_ctx::LoopGraph lg;
    lg.key = key;
    CK(cudaGraphCreate(&lg.g, 0));
    struct Drop {  // destroy the half-built graph on failure
      dpt_ctx::LoopGraph* p;
      ~Drop() {
        if (p && p->ge) cudaGraphExecDestroy(p->ge);
        if (p && p->g) cudaGraphDestroy(p->g);
      }
    } drop{&lg};
    cudaGraphConditionalHandle h;
    CK(cudaGraphConditionalHandleCreate(&h, lg.g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    CK(cudaGraphAddNode(&node, lg.g, nullptr, 0, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    w.s.has_loop = 1;
    w.s.loop_total = total;
    w.s.loop_cond = static_cast<unsigned long long>(h);
    const int64_t before = ctx->launches;
    CK(cudaStreamBeginCaptureToGraph(st, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    try {
      step_launch(ctx, w, dp, mode, row, err);
      post_step(ctx, w, w.ntiles_step, cycle_elems, err);
    } catch (...) {
      cudaGraph_t junk;
      cudaStreamEndCapture(st, &junk);
      throw;
    }
    cudaGraph_t captured;
    CK(cudaStreamEndCapture(st, &captured));
    lg.per_body = ctx->launches - before;
    ctx->launches = before;
    lg.cond = static_cast<unsigned long long>(h);
    CK(cudaGraphInstantiate(&lg.ge, lg.g, 0));
    if (ctx->loop_graphs.size() >= kMaxLoopGraphs) {
      auto& old = ctx->loop_graphs.front();
      cudaGraphExecDestroy(old.ge);
      cudaGraphDestroy(old.g);
      ctx->loop_graphs.erase(ctx->loop_graphs.begin());
    }
    ctx->loop_graphs.push_back(lg);
    drop.p = nullptr;
    hit = &ctx->loop_graphs.back();
  }
  const auto t0 = std::chrono::steady_clock::now();
  CK(cudaGraphLaunch(hit->ge, st));
  const auto t1 = std::chrono::steady_clock::now();
  CK(cudaMemcpyAsync(w.h_state, w.s.state, sizeof(dpt_sm_state), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const auto t2 = std::chrono::steady_clock::now();
  if (dbg)
    std::fprintf(stderr, "[dpt] loop graph launch %.1f us, run+sync %.1f us\n",
                 std::chrono::duration<double, std::micro>(t1 - t0).count(),
                 std::chrono::duration<double, std::micro>(t2 - t1).count());
  const int bodies = std::max(1, w.h_state->j - issued);
  ctx->launches += hit->per_body * bodies;
  replay_trace(w, w.h_state->trace_len, 0, trace, user, err);
}

// K2's launch 1 from the identity as three small kernels (sparse_step.cu,
// launch_csr_init): real data, levels-generated gaps, the packed image built,
// strictly increasing columns in every CSR row.  DPT_CSR_INIT=0: K2 as launch 1.
bool csr_init_applies(const DevProblem& dp, const Work& w) {
  static const bool off = [] {
    const char* e = std::getenv("DPT_CSR_INIT");
    return e && e[0] == '0';
  }();
  return !off && !dp.cplx && !w.s.gapmat && dp.s_cols16.p && dp.csr_strict && w.initpart.p;
}

// K3's launch 1 from z_0 = e_row without the gathers (single_u16.cu,
// launch_single_u16_init): the uniform-16 CSR row map on real data with gaps from
// the levels.  DPT_U16_INIT=0: K3 as launch 1.
bool u16_init_applies(const DevProblem& dp, const Work& w) {
  const char* e = std::getenv("DPT_U16_INIT");  // read per call: tests switch it in-process
  const bool off = e && e[0] == '0';
  return !off && !dp.cplx && !w.s.gapmat && dp.kind == DPT_DELTA_CSR && dp.uniform16;
}

// Runs launches 1 .. until the state machine terminates (or `total` launches).
// Launch 1 is the special init (dense) or the generic step from slot 0.
// Chunks are double-buffered: chunk c+1 is enqueued before the host waits for
// chunk c's state snapshot, so the GPU never idles on the host's decision;
// launches queued after a terminal decision are no-ops.
void drive(dpt_ctx* ctx, Work& w, DevProblem& dp, Mode mode, int64_t row, int total, bool first_is_init,
           dpt_trace_fn trace, void* user, dpt_error_info* err) {
  Nvtx nvtx_range("dpt.drive");
  cudaStream_t st = ctx->stream;
  const int64_t cycle_elems = (mode == MODE_SINGLE) ? dp.ncol : w.s.rows * dp.ncol;
  int issued = 0;
  if (first_is_init) {
    CK(launch_dense_init(w.s, dp.delta.as<double>(), dp.big, st));
    ctx->launches += 1;
    post_step(ctx, w, dense_init_ntiles(w.s.rows, w.s.ntn, w.s.cplx), cycle_elems, err);
    issued = 1;
  } else if (mode == MODE_SINGLE && u16_init_applies(dp, w)) {
    // the row map starts from z_0 = e_row (run_single): launch 1 from the columns alone
    CK(launch_single_u16_init(w.s, dp.csr(), row, st));
    ctx->launches += 1;
    post_step(ctx, w, w.ntiles_step, cycle_elems, err);
    issued = 1;
  } else if (mode == MODE_CSR_FULL && csr_init_applies(dp, w)) {
    // CSR solves start from A_0 = I (put_identity): launch 1 without the product
    CK(launch_csr_init(w.s, dp.csr(), dp.sell(), w.initpart.p, st));
    ctx->launches += 3;
    post_step(ctx, w, 1, cycle_elems, err);
    issued = 1;
  }
  // With a TraceSink the host chunk driver runs instead of the device loop: the
  // sink is then called while the solve is in flight (after each chunk, in k
  // order) and a sink that aborts stops the device within one chunk, as the
  // reference's sink -- called inside its loop, dpt.cpp:153-157 -- stops it.
  if (w.s.fuse_decide && issued < total && graph_loop_enabled() && !trace) {
    drive_graph(ctx, w, dp, mode, row, total, issued, cycle_elems, trace, user, err);
    return;
  }
  dpt_sm_state* snap = w.h_state;  // [2] pinned snapshots, one per chunk in flight
  cudaEvent_t ev[2];
  CK(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
  struct EvGuard {
    cudaEvent_t* e;
    ~EvGuard() {
      cudaEventDestroy(e[0]);
      cudaEventDestroy(e[1]);
    }
  } eg{ev};
  int chunk = 4, traced = 0, c = 0;
  bool pending = false;
  auto consume = [&](int slot) {
    CK(cudaEventSynchronize(ev[slot]));
    const dpt_sm_state& h = snap[slot];
    if (trace && h.trace_len > traced) {
      const int nt = h.trace_len;
      CK(cudaMemcpy(w.h_trace, w.s.trace, size_t(nt) * 3 * 8, cudaMemcpyDeviceToHost));
      for (int q = traced; q < nt; ++q) {
        if (trace(int(w.h_trace[3 * q]), w.h_trace[3 * q + 1], w.h_trace[3 * q + 2], user) != 0) {
          set_err(err, DPT_ERR_TRACE, "trace sink aborted the iteration");
          throw Fail{DPT_ERR_TRACE};
        }
      }
      traced = nt;
    }
    return h.done != 0;
  };
  bool done = false;
  while (issued < total && !done) {
    const int todo = std::min(chunk, total - issued);
    for (int k = 0; k < todo; ++k) {
      step_launch(ctx, w, dp, mode, row, err);
      post_step(ctx, w, w.ntiles_step, cycle_elems, err);
    }
    issued += todo;
    const int slot = c & 1;
    CK(cudaMemcpyAsync(&snap[slot], w.s.state, sizeof(dpt_sm_state), cudaMemcpyDeviceToHost, st));
    CK(cudaEventRecord(ev[slot], st));
    if (pending) done = consume(slot ^ 1);
    pending = true;
    ++c;
    chunk = std::min(chunk * 2, trace ? 8 : 64);  // a sink sees every iteration within <= 8 launches
  }
  if (pending && !done) done = consume((c - 1) & 1);
  CK(cudaStreamSynchronize(st));
  *w.h_state = snap[(c - 1) & 1];
  // the final snapshot is authoritative (later chunks were no-ops once done)
  if (!w.h_state->done) {
    CK(cudaMemcpy(w.h_state, w.s.state, sizeof(dpt_sm_state), cudaMemcpyDeviceToHost));
  }
  if (trace && w.h_state->trace_len > traced) {
    const int nt = w.h_state->trace_len;
    CK(cudaMemcpy(w.h_trace, w.s.trace, size_t(nt) * 3 * 8, cudaMemcpyDeviceToHost));
    for (int q = traced; q < nt; ++q)
      if (trace(int(w.h_trace[3 * q]), w.h_trace[3 * q + 1], w.h_trace[3 * q + 2], user) != 0) {
        set_err(err, DPT_ERR_TRACE, "trace sink aborted the iteration");
        throw Fail{DPT_ERR_TRACE};
      }
  }
}

void copy_out(double* dst, const double* src, size_t count, int out_mem, cudaStream_t st, dpt_error_info* err) {
  if (!dst || count == 0) return;
  if (out_mem != DPT_MEM_DEVICE && t_ctx && st == t_ctx->stream) {
    CK(copy_async(t_ctx, dst, src, count * 8, cudaMemcpyDeviceToHost));
    return;
  }
  CK(cudaMemcpyAsync(dst, src, count * 8, out_mem == DPT_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
}

void copy_slot_out(double* dst, const Work& w, const DevProblem& dp, int slot, int out_mem, cudaStream_t st,
                   dpt_error_info* err) {
  if (!dst || dp.n == 0) return;
  const double* src = w.s.slots + size_t(slot) * size_t(w.s.slot_elems);
  const cudaMemcpyKind k = out_mem == DPT_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  if (k == cudaMemcpyDeviceToHost && t_ctx && st == t_ctx->stream) {  // staged when pageable
    CK(copy2d_async(t_ctx, dst, size_t(dp.ncol) * 8, src, size_t(dp.ld) * 8, size_t(dp.ncol) * 8, size_t(w.s.rows), k));
    return;
  }
  if (dp.ld == dp.ncol)
    CK(cudaMemcpyAsync(dst, src, size_t(w.s.rows) * size_t(dp.ncol) * 8, k, st));
  else
    CK(cudaMemcpy2DAsync(dst, size_t(dp.ncol) * 8, src, size_t(dp.ld) * 8, size_t(dp.ncol) * 8, size_t(w.s.rows), k, st));
}

void fill_nan(double* dst, size_t count, int out_mem, cudaStream_t st, dpt_error_info* err) {
  if (!dst || count == 0) return;
  std::vector<double> nan(count, std::numeric_limits<double>::quiet_NaN());
  if (out_mem == DPT_MEM_DEVICE) {
    CK(cudaMemcpyAsync(dst, nan.data(), count * 8, cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
  } else {
    memcpy(dst, nan.data(), count * 8);
  }
}


struct Guard {
  dpt_ctx* ctx;
  dpt_ctx* prev_ctx;
  int old = -1;
  explicit Guard(dpt_ctx* c) : ctx(c), prev_ctx(t_ctx) {
    cudaGetDevice(&old);
    cudaSetDevice(c->device);
    t_ctx = c;
  }
  ~Guard() {
    // a rank leaving a call by an exception releases its loopback peers
    // (they would otherwise wait at the next collective until the timeout)
    if (ctx->loop && std::uncaught_exceptions() > 0) ctx->loop->fail();
    t_ctx = prev_ctx;
    if (old >= 0) cudaSetDevice(old);
  }
};

// Rank r owns rows [r*per, min(n, (r+1)*per)) of A (the paper's columns).
void shard_rows(const dpt_ctx* ctx, int64_t n, int64_t* row0, int64_t* rows) {
  int rank = ctx->rank, world = ctx->world;
  // Development knob: DPT_SHARD_EMULATE=r/w gives a communicator-less context
  // rank r's row shard of a w-way solve, to time and test the per-rank kernels
  // at sharded shapes on one GPU (its decisions see only the local rows).
  if (!sharded(ctx)) {
    if (const char* e = std::getenv("DPT_SHARD_EMULATE")) {
      int r = 0, wv = 1;
      if (std::sscanf(e, "%d/%d", &r, &wv) == 2 && wv > 0 && r >= 0 && r < wv) {
        rank = r;
        world = wv;
      }
    }
  }
  const int64_t per = (n + world - 1) / world;
  *row0 = std::min<int64_t>(n, per * rank);
  *rows = std::min<int64_t>(n, *row0 + per) - *row0;
}

// Upload a caller iterate (rows x n, row-major) into ring slot `slot`.
void put_slot(Work& w, const DevProblem& dp, int slot, const double* a, int mem, cudaStream_t st,
              dpt_error_info* err) {
  double* dst = w.s.slots + size_t(slot) * size_t(w.s.slot_elems);
  const cudaMemcpyKind k = mem == DPT_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  CK(cudaMemsetAsync(dst, 0, size_t(w.s.rows) * size_t(dp.ld) * 8, st));
  if (dp.ld == dp.ncol)
    CK(cudaMemcpyAsync(dst, a, size_t(w.s.rows) * size_t(dp.ncol) * 8, k, st));
  else
    CK(cudaMemcpy2DAsync(dst, size_t(dp.ld) * 8, a, size_t(dp.ncol) * 8, size_t(dp.ncol) * 8, size_t(w.s.rows), k, st));
  CK(cudaStreamSynchronize(st));  // `a` may be pageable host memory owned by the caller
}

// A_0 = I in slot 0 and d_0 = diag(Delta) = P(I)(i,i).
// matrix = false: only d_0 (the CSR launch-1 shortcut never reads A_0, and without
// a cycle window nothing else does: every reported iterate has index >= 1).
void put_identity(dpt_ctx* ctx, Work& w, DevProblem& dp, dpt_error_info* err, bool matrix = true) {
  if (matrix) CK(launch_identity(w.s, ctx->stream));
  DevCsr c = dp.csr();
  if (dp.kind == DPT_DELTA_DENSE)
    CK(launch_set_diag_delta(w.s, dp.delta.as<double>(), nullptr, ctx->stream));
  else
    CK(launch_set_diag_delta(w.s, nullptr, &c, ctx->stream));
  ctx->launches += matrix ? 2 : 1;
}

void gather_rows(dpt_ctx* ctx, const Work& w, const DevProblem& dp, int slot, double* dst, int out_mem,
                 dpt_error_info* err) {
  Nvtx nvtx_range("dpt.gather_rows");
  if (!dst) return;
  cudaStream_t st = ctx->stream;
  if (!sharded(ctx)) {
    copy_slot_out(dst, w, dp, slot, out_mem, st, err);
    return;
  }
  // C2: the final eigenvector gather (one all-gather of the row shards)
  DBuf all;
  dalloc(all, size_t(ctx->world) * size_t(w.s.slot_elems) * 8, err);
  const double* src = w.s.slots + size_t(slot) * size_t(w.s.slot_elems);
  comm_all_gather(ctx, src, all.as<double>(), size_t(w.s.slot_elems), "the iterate shards", err);
  const cudaMemcpyKind k = out_mem == DPT_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  CK(copy2d_async(ctx, dst, size_t(dp.ncol) * 8, all.p, size_t(dp.ld) * 8, size_t(dp.ncol) * 8, size_t(dp.n), k));
  CK(cudaStreamSynchronize(st));
}

void gather_vec(dpt_ctx* ctx, const Work& w, const double* src, double* dst, int out_mem, int64_t n,
                dpt_error_info* err, int width = 1) {
  if (!dst) return;
  cudaStream_t st = ctx->stream;
  const int64_t per = width * (w.s.slot_elems / w.s.ld);
  n *= width;
  DBuf all;
  dalloc(all, size_t(ctx->world) * size_t(per) * 8, err);
  comm_all_gather(ctx, src, all.as<double>(), size_t(per), "the read-offs", err);
  copy_out(dst, all.as<double>(), size_t(n), out_mem, st, err);
  CK(cudaStreamSynchronize(st));
}

dpt_options opts_or_default(const dpt_options* o) {
  dpt_options r;
  if (o)
    r = *o;
  else
    dpt_options_default(&r);
  return r;
}

// Device-side level scans for device-resident levels (levels.cu): the
// single-row entry points' selection and gap-row degeneracy policy without
// copying d to the host.  Return false (caller falls back to the sequential
// host scans) for host levels or when d holds a NaN.
bool dev_levels_scan(dpt_ctx* ctx, const dpt_problem* p, double out[7], dpt_error_info* err) {
  if (p->mem != DPT_MEM_DEVICE || p->n == 0) return false;
  Guard g(ctx);
  cudaStream_t st = ctx->stream;
  const int ns = levels_scratch_doubles();
  DBuf scratch;
  dalloc(scratch, size_t(ns + 16) * 8, err);
  double* base = scratch.as<double>();
  unsigned* counter = reinterpret_cast<unsigned*>(base + ns);
  CK(cudaMemsetAsync(counter, 0, 8, st));
  CK(launch_levels_scan(p->d, p->n, p->is_complex ? 2 : 1, base, counter, base + ns + 2, st));
  CK(cudaMemcpyAsync(out, base + ns + 2, 7 * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return out[6] == 0.0;
}

// (Re, Im) of level i of device-resident levels
void dev_level(dpt_ctx* ctx, const dpt_problem* p, int64_t i, double* re, double* im) {
  const int cx = p->is_complex ? 2 : 1;
  double v[2] = {0.0, 0.0};
  Guard g(ctx);
  if (to_host_ordered(v, p->d + cx * i, size_t(cx) * 8, cudaMemcpyDeviceToHost) != cudaSuccess) throw Fail{DPT_ERR_CUDA};
  *re = v[0];
  *im = cx == 2 ? v[1] : 0.0;
}

// first m != row with |d_row - d_m| <= thresh, or -1
int64_t dev_partner(dpt_ctx* ctx, const dpt_problem* p, int64_t row, double thresh, dpt_error_info* err) {
  Guard g(ctx);
  cudaStream_t st = ctx->stream;
  DBuf f;
  dalloc(f, 16, err);
  CK(cudaMemsetAsync(f.p, 0xff, 8, st));
  CK(launch_levels_partner(p->d, p->n, p->is_complex ? 2 : 1, row, thresh, f.as<unsigned long long>(), st));
  unsigned long long h = ~0ull;
  CK(cudaMemcpyAsync(&h, f.p, 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return h == ~0ull ? -1 : int64_t(h);
}

[[noreturn]] void degenerate_error_dev(dpt_ctx* ctx, const dpt_problem* p, int64_t i, int64_t j, dpt_error_info* err) {
  double v[4];
  dev_level(ctx, p, i, &v[0], &v[1]);
  dev_level(ctx, p, j, &v[2], &v[3]);
  const double d2[4] = {v[0], v[1], v[2], v[3]};
  // degenerate_error indexes interleaved (re, im) pairs when cplx
  const double* dd = d2;
  if (p->is_complex) {
    if (err) {
      err->i = i; err->j = j; err->ei = dd[0]; err->ei_im = dd[1]; err->ej = dd[2]; err->ej_im = dd[3];
    }
  } else if (err) {
    err->i = i; err->j = j; err->ei = dd[0]; err->ej = dd[2]; err->ei_im = 0.0; err->ej_im = 0.0;
  }
  set_err(err, DPT_ERR_DEGENERATE,
          "degenerate spectrum: levels " + std::to_string(i) + " and " + std::to_string(j) +
              " coincide within tolerance");
  throw Fail{DPT_ERR_DEGENERATE};
}

// Host phase timer (DPT_TIMING=1 prints each phase of an API call to stderr).
struct PhaseTimer {
  bool on = std::getenv("DPT_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[dpt] %-24s %9.1f us\n", what, std::chrono::duration<double, std::micro>(now - t).count());
    t = now;
  }
};

std::vector<double> host_levels(const dpt_problem* p, dpt_error_info* err) {
  const size_t cnt = size_t(p->n) * (p->is_complex ? 2 : 1);  // interleaved when complex
  std::vector<double> dh(cnt);
  if (p->n)
    CK(to_host_ordered(dh.data(), p->d, cnt * 8, p->mem == DPT_MEM_DEVICE ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost));
  return dh;
}

// build_theta's degeneracy policy for real or complex levels.
void check_levels(const dpt_problem* p, const std::vector<double>& dh, double tol, dpt_error_info* err) {
  int64_t bi, bj;
  const bool hit = p->is_complex ? find_degenerate_c(p->n, dh.data(), tol, &bi, &bj)
                                 : find_degenerate(p->n, dh.data(), tol, &bi, &bj);
  if (hit) degenerate_error(err, bi, bj, dh.data(), p->is_complex != 0);
}

void fill_report(dpt_ctx* ctx, dpt_report* rep, int status, int iters, double step) {
  if (!rep) return;
  memset(rep, 0, sizeof(*rep));
  rep->status = status;
  rep->iterations = iters;
  rep->step_norm = step;
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
  rep->device_ms = ms;
  rep->launches = int(ctx->launches);
}

// ---------------------------------------------------------------- run_full --
// run_full (dpt.cpp:92-192); fixed_k >= 0 selects iterate_fixed (:381-387).
int run_full(dpt_ctx* ctx, const dpt_problem* p, const dpt_options* opts_in, bool ramped, double alpha,
             int fixed_k, double fixed_lambda, dpt_trace_fn trace, void* user, double* a_out,
             double* eig_out, double* res_out, int out_mem, dpt_report* rep, dpt_error_info* err,
             double fixed_lambda_im = 0.0) {
  Nvtx nvtx_range("dpt.run_full");
  const dpt_options o = opts_or_default(opts_in);
  Guard g(ctx);
  validate(p, err);
  const int64_t n = p->n;
  const bool fixed = fixed_k >= 0;
  if (n > 0 && n < ctx->world) {
    set_err(err, DPT_ERR_SHAPE, "sharded solve needs n >= world size");
    throw Fail{DPT_ERR_SHAPE};
  }
  std::vector<double> dh = host_levels(p, err);
  // iterate_fixed builds theta with the default tolerance (dpt.cpp:383)
  check_levels(p, dh, fixed ? 1e-12 : o.degeneracy_tol, err);
  if (n == 0) {  // run_full on an empty problem (dpt.cpp:92-192): every norm is 0
    int status = DPT_MAX_ITERATIONS, iters = fixed ? fixed_k : std::max(o.max_iter, 0);
    if (!fixed && o.max_iter >= 1 && 0.0 < o.tol && 0.0 < o.residual_tol) {
      status = DPT_CONVERGED;  // k = 1: step 0 < tol, max residual 0 < residual_tol
      iters = 1;
    }
    if (rep) {
      std::memset(rep, 0, sizeof(*rep));
      rep->status = status;
      rep->iterations = iters;
    }
    return DPT_OK;
  }
  DevProblem dp;
  upload(dp, ctx, p, err, p->delta_kind == DPT_DELTA_CSR);
  const int cx = dp.cplx ? 2 : 1;
  if (fixed) dp.lambda_im = fixed_lambda_im;
  const Mode mode = p->delta_kind == DPT_DELTA_DENSE ? MODE_DENSE_FULL : MODE_CSR_FULL;
  const int win = fixed ? 0 : effective_window(o.cycle_window, n);
  const int nslots = win > 0 ? win + 1 : 2;
  int64_t row0, rows;
  shard_rows(ctx, n, &row0, &rows);
  const int64_t per = (n + ctx->world - 1) / ctx->world;
  const int max_iter = fixed ? fixed_k : o.max_iter;
  const int total = fixed ? fixed_k : std::max(max_iter, 0) + 1;  // iterations + the read-off launch
  const double lam = fixed ? fixed_lambda : p->lambda;
  std::vector<double> lam_tab;
  std::vector<int> set_tab;
  if (ramped) {  // lambda_k = lambda (1 - alpha^(k-1)) in complex arithmetic (dpt.cpp:131-134)
    const size_t nk = size_t(total) + 2;
    lam_tab.resize(nk * size_t(cx));
    set_tab.resize(nk);
    const double lim = dp.lambda_im;
    for (size_t k = 0; k < nk; ++k) {
      const double f = k == 0 ? 0.0 : 1.0 - std::pow(alpha, double(int(k) - 1));
      const double lr = lam * f, li = lim * f;
      if (cx == 2) {
        lam_tab[2 * k] = lr;
        lam_tab[2 * k + 1] = li;
      } else {
        lam_tab[k] = lr;
      }
      set_tab[k] = std::hypot(lr - lam, li - lim) <= o.tol * std::hypot(lam, lim) ? 1 : 0;
    }
    set_tab[0] = 1;
  }
  dpt_sm_options so{};
  so.tol = o.tol;
  so.residual_tol = o.residual_tol;
  so.divergence_threshold = o.divergence_threshold;
  so.max_iter = max_iter;
  so.win = win;
  so.have_trace = trace ? 1 : 0;
  Work w;
  make_work(w, ctx, dp, mode, row0, rows, per, nslots, max_iter, ramped ? &lam_tab : nullptr,
            ramped ? &set_tab : nullptr, so, lam, fixed ? 1 : 0, err);
  cudaStream_t st = ctx->stream;
  CK(cudaEventRecord(ctx->ev0, st));
  int final_iter = 0, status = DPT_MAX_ITERATIONS, iters = max_iter, readoffs = 1;
  double step = 0.0;
  const bool dense = mode == MODE_DENSE_FULL;
  if (n == 0) {
    readoffs = 0;
  } else if (fixed) {
    if (fixed_k == 0) {
      put_identity(ctx, w, dp, err);
    } else {
      if (!dense) put_identity(ctx, w, dp, err, !csr_init_applies(dp, w));
      drive(ctx, w, dp, mode, 0, total, dense, nullptr, nullptr, err);
    }
    final_iter = fixed_k;
    readoffs = 0;
  } else if (max_iter <= 0) {
    // the loop never runs: MaxIterations with the read-offs of A_0 = I (dpt.cpp:189-191)
    put_identity(ctx, w, dp, err);
    w.s.fixed_mode = 1;
    step_launch(ctx, w, dp, mode, 0, err);
    post_step(ctx, w, w.ntiles_step, 0, err);
    final_iter = 0;
  } else {
    // A_0 = I (CSR start / window entry); the CSR shortcut without a window needs d_0 only
    if (!dense || win > 0) put_identity(ctx, w, dp, err, dense || win > 0 || !csr_init_applies(dp, w));
    drive(ctx, w, dp, mode, 0, total, dense, trace, user, err);
    if (!w.h_state->done) {
      set_err(err, DPT_ERR_CUDA, "internal: iteration budget consumed without a terminal status");
      throw Fail{DPT_ERR_CUDA};
    }
    status = w.h_state->status;
    iters = w.h_state->iterations;
    final_iter = w.h_state->final_iter;
    readoffs = w.h_state->readoffs;
    step = w.h_state->step_norm;
  }
  CK(cudaEventRecord(ctx->ev1, st));
  if (n > 0) {
    gather_rows(ctx, w, dp, final_iter % nslots, a_out, out_mem, err);
    if (readoffs) {
      if (sharded(ctx)) {
        gather_vec(ctx, w, w.s.eps, eig_out, out_mem, n, err, cx);
        gather_vec(ctx, w, w.s.res, res_out, out_mem, n, err);
      } else {
        copy_out(eig_out, w.s.eps, size_t(cx * n), out_mem, st, err);
        copy_out(res_out, w.s.res, size_t(n), out_mem, st, err);
      }
    } else {
      fill_nan(eig_out, size_t(cx * n), out_mem, st, err);  // cdouble{nan, nan} (dpt.cpp:121-124)
      fill_nan(res_out, size_t(n), out_mem, st, err);
    }
  }
  CK(cudaStreamSynchronize(st));
  fill_report(ctx, rep, status, iters, step);
  return DPT_OK;
}

// step_full (dpt.cpp:311-327): F(a) for a caller iterate; with `gap` the
// caller's GapMatrix (n x n, row-major) replaces theta-generated gaps.  With
// eig_out / res_out the read-offs of `a` itself (residuals_of, dpt.cpp:23-44)
// are returned as well (homotopy_solve's final report).
int run_step_full(dpt_ctx* ctx, const dpt_problem* p, const double* a, const double* gap, double lambda,
                  double* out, int io_mem, double* eig_out, double* res_out, dpt_error_info* err,
                  double lambda_im = 0.0) {
  Nvtx nvtx_range("dpt.step_full");
  Guard g(ctx);
  validate(p, err, true);
  if (sharded(ctx)) {
    set_err(err, DPT_ERR_UNSUPPORTED, "step_full is a single-device call");
    throw Fail{DPT_ERR_UNSUPPORTED};
  }
  const int64_t n = p->n;
  if (n == 0) return DPT_OK;
  DevProblem dp;
  upload(dp, ctx, p, err, p->delta_kind == DPT_DELTA_CSR);
  const Mode mode = p->delta_kind == DPT_DELTA_CSR ? MODE_CSR_FULL : MODE_DENSE_FULL;
  dpt_sm_options so{};
  so.max_iter = 1;
  Work w;
  dp.lambda_im = lambda_im;
  make_work(w, ctx, dp, mode, 0, n, n, 2, 1, nullptr, nullptr, so, lambda, 1, err);
  DBuf gbuf;
  if (gap) {  // caller GapMatrix, row-major n x n (interleaved complex when is_complex)
    dalloc(gbuf, size_t(n) * size_t(dp.ld) * 8, err);
    const cudaMemcpyKind k = io_mem == DPT_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    CK(cudaMemcpy2DAsync(gbuf.p, size_t(dp.ld) * 8, gap, size_t(dp.ncol) * 8, size_t(dp.ncol) * 8, size_t(n), k,
                         ctx->stream));
    w.s.gapmat = gbuf.as<double>();
  }
  put_slot(w, dp, 0, a, io_mem, ctx->stream, err);
  DevCsr c = dp.csr();
  CK(launch_rowdot(w.s, dp.kind == DPT_DELTA_DENSE ? dp.delta.as<double>() : nullptr, dp.kind == DPT_DELTA_CSR ? &c : nullptr, ctx->stream));
  step_launch(ctx, w, dp, mode, 0, err);
  post_step(ctx, w, w.ntiles_step, 0, err);
  if (out) copy_slot_out(out, w, dp, 1, io_mem, ctx->stream, err);
  copy_out(eig_out, w.s.eps, size_t(dp.ncol), io_mem, ctx->stream, err);
  copy_out(res_out, w.s.res, size_t(n), io_mem, ctx->stream, err);
  CK(cudaStreamSynchronize(ctx->stream));
  return DPT_OK;
}

// ---------------------------------------------------------------- run_single --
// run_single (dpt.cpp:194-293) for chart row `row`; fixed >= 0: step_single /
// eigenvalue_of (one launch from the caller's z).
int run_single(dpt_ctx* ctx, const dpt_problem* p, int64_t row, const dpt_options* opts_in, double ramp_alpha,
               dpt_trace_fn trace, void* user, double* z_out, int out_mem, dpt_report* rep,
               const double* z_in, int z_mem, double fixed_lambda, double* eig_fixed, double* z_unit,
               dpt_error_info* err, const double* gap_row = nullptr, double fixed_lambda_im = 0.0) {
  Nvtx nvtx_range("dpt.run_single");
  const dpt_options o = opts_or_default(opts_in);
  Guard g(ctx);
  validate(p, err);
  const int64_t n = p->n;
  const bool fixed = z_in != nullptr;
  const bool ramped = ramp_alpha > 0.0;
  PhaseTimer pt;
  DevProblem dp;
  upload(dp, ctx, p, err);
  pt.mark("single: upload");
  const int cx = dp.cplx ? 2 : 1;
  if (fixed) dp.lambda_im = fixed_lambda_im;
  const int win = fixed ? 0 : (o.cycle_window >= 2 ? std::min(o.cycle_window, DPT_MAX_WINDOW) : 0);  // dpt.cpp:207
  const int nslots = win > 0 ? win + 1 : 2;
  const int max_iter = fixed ? 1 : o.max_iter;
  const int total = fixed ? 1 : std::max(max_iter, 0) + 1;
  const double lam = fixed ? fixed_lambda : p->lambda;
  std::vector<double> lam_tab;
  std::vector<int> set_tab;
  if (ramped && !fixed) {  // dpt.cpp:238-240, complex lambda_k
    const size_t nk = size_t(total) + 2;
    lam_tab.resize(nk * size_t(cx));
    set_tab.resize(nk);
    const double lim = dp.lambda_im;
    for (size_t k = 0; k < nk; ++k) {
      const double f = k == 0 ? 0.0 : 1.0 - std::pow(ramp_alpha, double(int(k) - 1));
      const double lr = lam * f, li = lim * f;
      if (cx == 2) {
        lam_tab[2 * k] = lr;
        lam_tab[2 * k + 1] = li;
      } else {
        lam_tab[k] = lr;
      }
      set_tab[k] = std::hypot(lr - lam, li - lim) <= o.tol * std::hypot(lam, lim) ? 1 : 0;
    }
    set_tab[0] = 1;
  }
  dpt_sm_options so{};
  so.tol = o.tol;
  so.residual_tol = o.residual_tol;
  so.divergence_threshold = o.divergence_threshold;
  so.max_iter = max_iter;
  so.win = win;
  so.have_trace = trace ? 1 : 0;
  Work w;
  make_work(w, ctx, dp, MODE_SINGLE, row, 1, 1, nslots, max_iter, ramped && !fixed ? &lam_tab : nullptr,
            ramped && !fixed ? &set_tab : nullptr, so, lam, fixed ? 1 : 0, err);
  pt.mark("single: make_work");
  cudaStream_t st = ctx->stream;
  CK(cudaEventRecord(ctx->ev0, st));
  int final_iter = 0, status = DPT_MAX_ITERATIONS, iters = max_iter, readoffs = 1;
  double step = 0.0;
  DBuf gbuf;
  if (gap_row) {
    dalloc(gbuf, size_t(cx * n) * 8, err);
    CK(cudaMemcpyAsync(gbuf.p, gap_row, size_t(cx * n) * 8,
                       z_mem == DPT_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
    w.s.gapmat = gbuf.as<double>();
  }
  if (fixed) {
    put_slot(w, dp, 0, z_in, z_mem, st, err);
    step_launch(ctx, w, dp, MODE_SINGLE, row, err);
    post_step(ctx, w, w.ntiles_step, 0, err);
    final_iter = 1;
  } else if (max_iter <= 0) {
    CK(launch_identity(w.s, st));  // z = e_row
    w.s.fixed_mode = 1;
    step_launch(ctx, w, dp, MODE_SINGLE, row, err);
    post_step(ctx, w, w.ntiles_step, 0, err);
    final_iter = 0;
  } else {
    CK(launch_identity(w.s, st));  // z = e_row (rows == 1, row0 == row)
    drive(ctx, w, dp, MODE_SINGLE, row, total, false, trace, user, err);
    pt.mark("single: drive");
    if (!w.h_state->done) {
      set_err(err, DPT_ERR_CUDA, "internal: iteration budget consumed without a terminal status");
      throw Fail{DPT_ERR_CUDA};
    }
    status = w.h_state->status;
    iters = w.h_state->iterations;
    final_iter = w.h_state->final_iter;
    readoffs = w.h_state->readoffs;
    step = w.h_state->step_norm;
  }
  CK(cudaEventRecord(ctx->ev1, st));
  if (n > 0 && z_out) copy_slot_out(z_out, w, dp, final_iter % nslots, out_mem, st, err);
  if (n > 0 && z_unit) {  // dominant_eigenpair's z_unit = z / ||z||_2 (dpt.cpp:432-436); |z|^2 = re^2 + im^2
    DBuf tmp;
    dalloc(tmp, size_t(cx * n) * 8, err);
    DBuf scratch;
    dalloc(scratch, 512 * 8, err);
    CK(launch_unit(w.s.slots + size_t(final_iter % nslots) * size_t(w.s.slot_elems), tmp.as<double>(), cx * n,
                   scratch.as<double>(), w.s.counter + 2, st));
    copy_out(z_unit, tmp.as<double>(), size_t(cx * n), out_mem, st, err);
    CK(cudaStreamSynchronize(st));
  }
  double eigv[2] = {std::numeric_limits<double>::quiet_NaN(), std::numeric_limits<double>::quiet_NaN()};
  double res = std::numeric_limits<double>::quiet_NaN();
  if (readoffs) {
    CK(cudaMemcpyAsync(eigv, w.s.eps, size_t(cx) * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&res, w.s.res, 8, cudaMemcpyDeviceToHost, st));
  }
  CK(cudaStreamSynchronize(st));
  if (cx == 1 && readoffs) eigv[1] = 0.0;
  const double eig = eigv[0];
  if (eig_fixed) {
    eig_fixed[0] = eigv[0];
    if (cx == 2) eig_fixed[1] = eigv[1];
  }
  fill_report(ctx, rep, status, iters, step);
  if (rep) {
    rep->eigenvalue_im = eigv[1];
    rep->eigenvalue = eig;
    rep->residual = res;
    rep->row = row;
  }
  pt.mark("single: outputs");
  return DPT_OK;
}


// ------------------------------------------------------ homotopy_solve ----
// dpt.cpp:505-556 on the device, no libraries.  Per stage s:
// M_s = lam_s Delta + diag(d); R = W^-1 (M_s W) -- the product on the DMMA
// GEMM, the solve as an LU of W with partial pivoting (cluster panels + GEMM
// trailing updates) and blocked triangular solves over the n right-hand sides
// (linalg.cu); partition(R) -> d', Delta' (lambda 1), the DPT solve of that
// problem in the solver's kernels (A_s stays in HBM), W <- W A_s^T.  Then
// a(i, m) = W(m, i) / W(i, i) and the read-offs of a against the original problem.
int run_homotopy(dpt_ctx* ctx, const dpt_problem* p, int stages, const dpt_options* opts_in, double* a_out,
                 double* eig_out, double* res_out, int out_mem, dpt_report* rep, dpt_error_info* err) {
  Nvtx nvtx_range("dpt.homotopy_solve");
  Guard g(ctx);
  validate(p, err);
  if (stages < 1) {
    set_err(err, DPT_ERR_INVALID_ARG, "homotopy_solve: stages must be >= 1");
    return DPT_ERR_INVALID_ARG;
  }
  const dpt_options o = opts_or_default(opts_in);
  const int64_t n = p->n;
  const int cx = p->is_complex ? 2 : 1;
  if (n > lu_max_n(cx)) {
    set_err(err, DPT_ERR_UNSUPPORTED, "homotopy_solve: n exceeds the device LU's cluster panel capacity (" +
                                          std::to_string(lu_max_n(cx)) + ")");
    return DPT_ERR_UNSUPPORTED;
  }
  cudaStream_t st = ctx->stream;
  const int64_t ld = (cx * n + 1) & ~int64_t(1);  // doubles per row, even (TMA strides)
  const size_t mat = size_t(n) * size_t(ld) * 8;  // padded row-major matrix
  const size_t cmat = size_t(cx) * size_t(n) * size_t(n) * 8;  // contiguous (the stage problem / its result)
  const int64_t ldop = 2 * n;  // B-operand rows: n (real) or the 2n x 2n image (complex), 2n >= cx n, even
  const size_t opbytes = size_t(cx * n) * size_t(ldop) * 8;
  const cudaMemcpyKind k = p->mem == DPT_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  DBuf bd, bD, bW, bWn, bM, bMW, bLU, bX, bA, bdl, bDp, bop, bscr, bpiv, bperm, binfo, bflag;
  dalloc(bd, size_t(cx * n) * 8, err);
  dalloc(bD, mat, err);
  dalloc(bW, mat, err);
  dalloc(bWn, mat, err);
  dalloc(bM, mat, err);
  dalloc(bMW, mat, err);
  dalloc(bLU, mat, err);
  dalloc(bX, mat, err);
  dalloc(bA, cmat, err);
  dalloc(bdl, size_t(cx * n) * 8, err);
  dalloc(bDp, cmat, err);
  dalloc(bop, opbytes, err);
  dalloc(bscr, size_t(4) * size_t(n) * 128 * 8 + 4096, err);
  dalloc(bpiv, size_t(n) * 8 + 16, err);
  dalloc(bperm, size_t(n) * 8 + 16, err);
  dalloc(binfo, 16, err);
  dalloc(bflag, 16, err);
  if (n) CK(cudaMemcpyAsync(bd.p, p->d, size_t(cx * n) * 8, k, st));
  if (p->delta_kind == DPT_DELTA_DENSE) {  // densify(p.delta) (dpt.cpp:510)
    if (n) CK(copy2d_async(ctx, bD.p, size_t(ld) * 8, p->delta, size_t(cx * n) * 8, size_t(cx * n) * 8, size_t(n), k));
  } else {
    DevProblem dp;
    upload(dp, ctx, p, err);
    CK(cudaMemsetAsync(bD.p, 0, mat, st));
    CK(launch_hom_densify(dp.rowptr.as<int64_t>(), dp.cols.as<int32_t>(), dp.vals.as<double>(), cx, n, ld,
                          bD.as<double>(), st));
    CK(cudaStreamSynchronize(st));  // dp's buffers go out of scope
  }
  CK(launch_hom_identity(bW.as<double>(), cx, n, ld, st));
  ctx->launches += 1;
  std::vector<int64_t> hpiv(static_cast<size_t>(n)), hperm(static_cast<size_t>(n));
  dpt_report last{};
  int total = 0;
  double* W = bW.as<double>();
  double* Wn = bWn.as<double>();
  for (int s = 1; s <= stages && n > 0; ++s) {
    const double f = double(s) / double(stages);  // lam_s = lambda * (s / stages), complex * double
    const double lr = p->lambda * f, li = (p->is_complex ? p->lambda_im : 0.0) * f;
    CK(launch_hom_stage_matrix(bD.as<double>(), bd.as<double>(), lr, li, cx, n, ld, bM.as<double>(), st));
    // M W: B operand = W^T (real) or its image (complex)
    CK(launch_gemm_bop(cx, true, W, ld / cx, n, n, bop.as<double>(), ldop, st));
    CK(launch_gemm_nt(n, cx * n, cx * n, bM.as<double>(), ld, bop.as<double>(), ldop, 1.0, 0.0, bMW.as<double>(), ld,
                      st));
    ctx->launches += 3;
    // R = W^-1 (M W): LU of a copy of W (lu_factor, matrix.cpp:468-494)
    CK(cudaMemcpyAsync(bLU.p, W, mat, cudaMemcpyDeviceToDevice, st));
    int nl = 0;
    CK(launch_lu_factor(cx, bLU.as<double>(), ld, n, bpiv.as<int64_t>(), binfo.as<int>(), bscr.as<double>(), &nl, st));
    int hinfo = 0;
    CK(cudaMemcpyAsync(&hinfo, binfo.p, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hpiv.data(), bpiv.p, size_t(n) * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    ctx->launches += nl;
    if (hinfo >= 1 && hinfo <= n) {  // lu_factor's exact-zero pivot (matrix.cpp:485)
      set_err(err, DPT_ERR_UNSUPPORTED, "solve_linear: singular matrix");
      throw Fail{DPT_ERR_UNSUPPORTED};
    }
    // lu_solve's b[perm[i]] (matrix.cpp:501): the row permutation of the pivot sequence
    for (int64_t i = 0; i < n; ++i) hperm[size_t(i)] = i;
    for (int64_t i = 0; i < n; ++i) std::swap(hperm[size_t(i)], hperm[size_t(hpiv[size_t(i)])]);
    CK(cudaMemcpyAsync(bperm.p, hperm.data(), size_t(n) * 8, cudaMemcpyHostToDevice, st));
    CK(launch_gather_rows(bMW.as<double>(), ld, bperm.as<int64_t>(), n, ld, bX.as<double>(), st));
    nl = 0;
    CK(launch_lu_solve(cx, bLU.as<double>(), ld, n, bX.as<double>(), ld, n, bscr.as<double>(), &nl, st));
    CK(launch_hom_partition(bX.as<double>(), ld, bdl.as<double>(), bDp.as<double>(), cx, n, st));
    ctx->launches += nl + 2;
    CK(cudaStreamSynchronize(st));  // hperm (host) is rewritten next stage
    dpt_problem sp{};
    sp.n = n;
    sp.d = bdl.as<double>();
    sp.delta_kind = DPT_DELTA_DENSE;
    sp.delta = bDp.as<double>();
    sp.lambda = 1.0;  // partition() sets lambda = 1 (partition.cpp:31)
    sp.mem = DPT_MEM_DEVICE;
    sp.is_complex = p->is_complex;
    sp.lambda_im = 0.0;
    last = dpt_report{};
    const int rc = run_full(ctx, &sp, &o, false, 0.0, -1, 0.0, nullptr, nullptr, bA.as<double>(), nullptr, nullptr,
                            DPT_MEM_DEVICE, &last, err);
    if (rc != DPT_OK) return rc;
    total += last.iterations;
    if (last.status != DPT_CONVERGED) break;
    // W V with V = A_s^T (no conjugation): the NT product against A_s itself
    CK(launch_gemm_bop(cx, false, bA.as<double>(), n, n, n, bop.as<double>(), ldop, st));
    CK(launch_gemm_nt(n, cx * n, cx * n, W, ld, bop.as<double>(), ldop, 1.0, 0.0, Wn, ld, st));
    ctx->launches += 2;
    std::swap(W, Wn);
  }
  // a(i, m) = W(m, i) / W(i, i)
  CK(cudaMemsetAsync(bflag.p, 0, 8, st));
  if (n) {
    CK(launch_hom_normalise(W, ld, bA.as<double>(), cx, n, bflag.as<unsigned>(), st));
    CK(launch_hom_nonfinite(bA.as<double>(), int64_t(cx) * n * n, bflag.as<unsigned>() + 1, st));
    ctx->launches += 2;
  }
  unsigned hf[2] = {0, 0};
  CK(cudaMemcpyAsync(hf, bflag.p, 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (hf[0]) {
    set_err(err, DPT_ERR_UNSUPPORTED, "homotopy_solve: singular stage basis");
    throw Fail{DPT_ERR_UNSUPPORTED};
  }
  if (hf[1] == 0) {  // read-offs against the ORIGINAL problem (dpt.cpp:547-550)
    DBuf be, br;
    dalloc(be, size_t(cx * n) * 8, err);
    dalloc(br, size_t(n) * 8, err);
    const int rc = run_step_full(ctx, p, bA.as<double>(), nullptr, p->lambda, nullptr, DPT_MEM_DEVICE,
                                 be.as<double>(), br.as<double>(), err, p->is_complex ? p->lambda_im : 0.0);
    if (rc != DPT_OK) return rc;
    copy_out(eig_out, be.as<double>(), size_t(cx * n), out_mem, st, err);
    copy_out(res_out, br.as<double>(), size_t(n), out_mem, st, err);
  } else {
    fill_nan(eig_out, size_t(cx * n), out_mem, st, err);
    fill_nan(res_out, size_t(n), out_mem, st, err);
  }
  copy_out(a_out, bA.as<double>(), size_t(cx) * size_t(n) * size_t(n), out_mem, st, err);
  CK(cudaStreamSynchronize(st));
  if (rep) {
    std::memset(rep, 0, sizeof(*rep));
    rep->status = last.status;
    rep->iterations = total;
    rep->step_norm = last.step_norm;
    rep->launches = int(ctx->launches);
  }
  return DPT_OK;
}

}  // namespace

// ================================================================ C ABI ====
#define DPT_API_BEGIN \
  if (err) memset(err, 0, sizeof(*err)); \
  try {
#define DPT_API_END                                                  \
  }                                                                  \
  catch (const Fail& f) {                                            \
    return f.code;                                                   \
  }                                                                  \
  catch (const std::exception& e) {                                  \
    set_err(err, DPT_ERR_CUDA, std::string("exception: ") + e.what()); \
    return DPT_ERR_CUDA;                                             \
  }

extern "C" {

void dpt_options_default(dpt_options* o) {  // IterationOptions defaults, dpt.hpp:22-31
  o->tol = 1e-12;
  o->residual_tol = 1e-10;
  o->max_iter = 10000;
  o->divergence_threshold = 1e8;
  o->cycle_window = 16;
  o->degeneracy_tol = 1e-12;
}

const char* dpt_status_string(int s) {  // to_string, dpt.cpp:297-309
  switch (s) {
    case DPT_CONVERGED:
      return "Converged";
    case DPT_BOUNDED_NON_CONVERGED:
      return "BoundedNonConverged";
    case DPT_DIVERGED:
      return "Diverged";
    case DPT_MAX_ITERATIONS:
      return "MaxIterations";
  }
  return "Unknown";
}

int dpt_abi_version(void) { return DPT_B200_ABI_VERSION; }

int dpt_ctx_create(int device, dpt_ctx** out, dpt_error_info* err) {
  DPT_API_BEGIN
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    set_err(err, DPT_ERR_NO_DEVICE, "no CUDA device visible: the DPT path has no CPU fallback");
    return DPT_ERR_NO_DEVICE;
  }
  if (device < 0 || device >= count) {
    set_err(err, DPT_ERR_INVALID_ARG, "device ordinal out of range");
    return DPT_ERR_INVALID_ARG;
  }
  std::unique_ptr<dpt_ctx> c(new dpt_ctx());
  c->device = device;
  Guard g(c.get());
  CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  CK(cudaEventCreate(&c->ev0));
  CK(cudaEventCreate(&c->ev1));
  *out = c.release();
  return DPT_OK;
  DPT_API_END
}

void dpt_ctx_destroy(dpt_ctx* ctx) {
  if (!ctx) return;
  {
    Guard g(ctx);
    if (ctx->comm && nccl_api() && nccl_api()->comm_destroy) nccl_api()->comm_destroy(ctx->comm);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    for (auto& lg : ctx->loop_graphs) {
      if (lg.ge) cudaGraphExecDestroy(lg.ge);
      if (lg.g) cudaGraphDestroy(lg.g);
    }
    ctx->loop_graphs.clear();
    for (auto& kv : ctx->free_blocks) cudaFree(kv.second);
    ctx->free_blocks.clear();
    if (ctx->pinned) cudaFreeHost(ctx->pinned);
    for (int b = 0; b < 2; ++b) {
      if (ctx->stage_ev[b]) cudaEventSynchronize(ctx->stage_ev[b]), cudaEventDestroy(ctx->stage_ev[b]);
      if (ctx->stage[b]) cudaFreeHost(ctx->stage[b]);
    }
    if (ctx->ev0) cudaEventDestroy(ctx->ev0);
    if (ctx->ev1) cudaEventDestroy(ctx->ev1);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
  }
  delete ctx;
}

int dpt_nccl_unique_id(void* out, size_t bytes, dpt_error_info* err) {
  DPT_API_BEGIN
  NcclApi* api = nccl_api();
  if (!api || bytes < sizeof(ncclUniqueId)) {
    set_err(err, DPT_ERR_NCCL, "libnccl.so.2 not loadable or id buffer too small");
    return DPT_ERR_NCCL;
  }
  ncclUniqueId id;
  if (api->get_unique_id(&id) != 0) {
    set_err(err, DPT_ERR_NCCL, "ncclGetUniqueId failed");
    return DPT_ERR_NCCL;
  }
  memcpy(out, &id, sizeof(id));
  return DPT_OK;
  DPT_API_END
}

int dpt_ctx_set_comm(dpt_ctx* ctx, int rank, int world, const void* id, size_t bytes, dpt_error_info* err) {
  DPT_API_BEGIN
  NcclApi* api = nccl_api();
  if (ctx->comm && api && api->comm_destroy) {
    api->comm_destroy(ctx->comm);
    ctx->comm = nullptr;
  }
  ctx->rank = 0;
  ctx->world = 1;
  if (world <= 1 && !id) return DPT_OK;  // single device, no collectives
  // world == 1 with an id builds a 1-rank communicator: the sharded code path
  // (allreduce between fold and decision, allgather of the result) on one GPU.
  if (!api || bytes < sizeof(ncclUniqueId) || rank < 0 || rank >= world || !id) {
    set_err(err, DPT_ERR_NCCL, "bad communicator arguments or libnccl.so.2 missing");
    return DPT_ERR_NCCL;
  }
  Guard g(ctx);
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  if (api->comm_init_rank(&ctx->comm, world, uid, rank) != 0) {
    ctx->comm = nullptr;
    set_err(err, DPT_ERR_NCCL, "ncclCommInitRank failed");
    return DPT_ERR_NCCL;
  }
  ctx->rank = rank;
  ctx->world = world;
  return DPT_OK;
  DPT_API_END
}

int dpt_ctx_set_loopback(dpt_ctx** ctxs, int world, dpt_error_info* err) {
  DPT_API_BEGIN
  if (!ctxs || world < 1 || world > kMaxLoopbackRanks) {
    set_err(err, DPT_ERR_INVALID_ARG, "loopback group: 1..8 contexts");
    return DPT_ERR_INVALID_ARG;
  }
  for (int r = 0; r < world; ++r)
    if (!ctxs[r] || ctxs[r]->comm || ctxs[r]->device != ctxs[0]->device) {
      set_err(err, DPT_ERR_INVALID_ARG, "loopback group: distinct contexts of one device, no NCCL communicator");
      return DPT_ERR_INVALID_ARG;
    }
  auto g = std::make_shared<LoopbackGroup>();
  g->world = world;
  g->src.assign(size_t(world), nullptr);
  {
    Guard gd(ctxs[0]);
    for (int r = 0; r < world; ++r) {
      cudaEvent_t a, b;
      CK(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
      g->ev_in.push_back(a);
      g->ev_out.push_back(b);
    }
  }
  for (int r = 0; r < world; ++r) {
    ctxs[r]->loop = g;
    ctxs[r]->rank = r;
    ctxs[r]->world = world;
  }
  return DPT_OK;
  DPT_API_END
}

void* dpt_ctx_stream(dpt_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }
int64_t dpt_ctx_launch_count(const dpt_ctx* ctx) { return ctx ? ctx->launches : 0; }

void dpt_ctx_graph_stats(const dpt_ctx* ctx, int64_t* hits, int64_t* misses) {
  if (hits) *hits = ctx ? ctx->graph_hits : 0;
  if (misses) *misses = ctx ? ctx->graph_misses : 0;
}

int dpt_iterate_full(dpt_ctx* ctx, const dpt_problem* p, const dpt_options* opts, dpt_trace_fn trace, void* user,
                     double* a_out, double* eig_out, double* res_out, int out_mem, dpt_report* rep,
                     dpt_error_info* err) {
  DPT_API_BEGIN
  return run_full(ctx, p, opts, false, 0.0, -1, 0.0, trace, user, a_out, eig_out, res_out, out_mem, rep, err);
  DPT_API_END
}

int dpt_iterate_ramped(dpt_ctx* ctx, const dpt_problem* p, double alpha, const dpt_options* opts,
                       dpt_trace_fn trace, void* user, double* a_out, double* eig_out, double* res_out,
                       int out_mem, dpt_report* rep, dpt_error_info* err) {
  DPT_API_BEGIN
  if (!(alpha >= 0.0) || alpha >= 1.0) {  // dpt.cpp:376-377
    set_err(err, DPT_ERR_INVALID_ARG, "iterate_ramped: alpha must lie in [0, 1)");
    return DPT_ERR_INVALID_ARG;
  }
  return run_full(ctx, p, opts, true, alpha, -1, 0.0, trace, user, a_out, eig_out, res_out, out_mem, rep, err);
  DPT_API_END
}

int dpt_iterate_fixed(dpt_ctx* ctx, const dpt_problem* p, int k, double lambda, double* a_out, int out_mem,
                      dpt_report* rep, dpt_error_info* err) {
  DPT_API_BEGIN
  if (k < 0) {  // dpt.cpp:382
    set_err(err, DPT_ERR_INVALID_ARG, "iterate_fixed: negative step count");
    return DPT_ERR_INVALID_ARG;
  }
  return run_full(ctx, p, nullptr, false, 0.0, k, lambda, nullptr, nullptr, a_out, nullptr, nullptr, out_mem, rep,
                  err);
  DPT_API_END
}

int dpt_step_full(dpt_ctx* ctx, const dpt_problem* p, const double* a, double lambda, double* out, int io_mem,
                  dpt_error_info* err) {
  DPT_API_BEGIN
  return run_step_full(ctx, p, a, nullptr, lambda, out, io_mem, nullptr, nullptr, err);
  DPT_API_END
}

int dpt_step_full_gap(dpt_ctx* ctx, const dpt_problem* p, const double* a, const double* gap, double lambda,
                      double* out, int io_mem, dpt_error_info* err) {
  DPT_API_BEGIN
  if (!gap) {
    set_err(err, DPT_ERR_INVALID_ARG, "step_full_gap: missing gap matrix");
    return DPT_ERR_INVALID_ARG;
  }
  return run_step_full(ctx, p, a, gap, lambda, out, io_mem, nullptr, nullptr, err);
  DPT_API_END
}

int dpt_readoffs(dpt_ctx* ctx, const dpt_problem* p, const double* a, double* eig_out, double* res_out,
                 int io_mem, dpt_error_info* err) {
  DPT_API_BEGIN
  return run_step_full(ctx, p, a, nullptr, p ? p->lambda : 0.0, nullptr, io_mem, eig_out, res_out, err,
                       p && p->is_complex ? p->lambda_im : 0.0);
  DPT_API_END
}

int dpt_step_single_gap(dpt_ctx* ctx, const dpt_problem* p, const double* z, int64_t row, const double* gap_row,
                        double lambda, double* out, int io_mem, dpt_error_info* err) {
  DPT_API_BEGIN
  validate(p, err);
  if (row < 0 || row >= p->n || !gap_row) {
    set_err(err, DPT_ERR_SHAPE, "step_single: dimension mismatch");
    return DPT_ERR_SHAPE;
  }
  return run_single(ctx, p, row, nullptr, 0.0, nullptr, nullptr, out, io_mem, nullptr, z, io_mem, lambda, nullptr,
                    nullptr, err, gap_row);
  DPT_API_END
}

int dpt_iterate_single(dpt_ctx* ctx, const dpt_problem* p, int64_t row, const dpt_options* opts,
                       double ramp_alpha, dpt_trace_fn trace, void* user, double* z_out, int out_mem,
                       dpt_report* rep, dpt_error_info* err) {
  DPT_API_BEGIN
  validate(p, err);
  if (row < 0 || row >= p->n) {  // dpt.cpp:392
    set_err(err, DPT_ERR_SHAPE, "iterate_single: row out of range");
    return DPT_ERR_SHAPE;
  }
  if (!(ramp_alpha >= 0.0) || ramp_alpha >= 1.0) {  // dpt.cpp:393-394
    set_err(err, DPT_ERR_INVALID_ARG, "iterate_single: ramp alpha must lie in [0, 1)");
    return DPT_ERR_INVALID_ARG;
  }
  const dpt_options o = opts_or_default(opts);
  double sc[7];
  if (dev_levels_scan(ctx, p, sc, err)) {  // device-resident levels, no NaN
    const double thr = o.degeneracy_tol * std::max(1.0, std::hypot(sc[3] - sc[2], sc[5] - sc[4]));
    const int64_t bj = dev_partner(ctx, p, row, thr, err);
    if (bj >= 0) degenerate_error_dev(ctx, p, row, bj, err);
  } else {
    std::vector<double> dh = host_levels(p, err);
    int64_t bj;
    const bool deg = p->is_complex ? find_degenerate_row_c(p->n, dh.data(), row, o.degeneracy_tol, &bj)
                                   : find_degenerate_row(p->n, dh.data(), row, o.degeneracy_tol, &bj);
    if (deg) degenerate_error(err, row, bj, dh.data(), p->is_complex != 0);
  }
  return run_single(ctx, p, row, &o, ramp_alpha, trace, user, z_out, out_mem, rep, nullptr, 0, 0.0, nullptr,
                    nullptr, err);
  DPT_API_END
}

int dpt_dominant_eigenpair(dpt_ctx* ctx, const dpt_problem* p, const dpt_options* opts, double* z_chart,
                           double* z_unit, int out_mem, dpt_report* rep, dpt_error_info* err) {
  DPT_API_BEGIN
  validate(p, err);
  const int64_t n = p->n;
  if (n == 0) {  // dpt.cpp:402
    set_err(err, DPT_ERR_SHAPE, "dominant_eigenpair: empty problem");
    return DPT_ERR_SHAPE;
  }
  const dpt_options o = opts_or_default(opts);
  PhaseTimer pt;
  double sc[7];
  // Large host-resident levels are scanned on the device too, from a temporary
  // copy (the four host passes cost ~4.4 ms at n = 2^20, the copy + scans
  // ~0.5 ms); the solve below still takes the caller's problem as given.
  Guard keep(ctx);  // the temporary returns to this context's cache
  DBuf dlev;
  dpt_problem pdev;
  const dpt_problem* ps = p;
  if (p->mem == DPT_MEM_HOST && n >= (int64_t(1) << 16)) {
    const size_t bytes = size_t(n) * (p->is_complex ? 16 : 8);
    dalloc(dlev, bytes, err);
    CK(copy_async(ctx, dlev.p, p->d, bytes, cudaMemcpyHostToDevice));
    pdev = *p;
    pdev.d = dlev.as<double>();
    pdev.mem = DPT_MEM_DEVICE;
    ps = &pdev;
  }
  if (dev_levels_scan(ctx, ps, sc, err)) {  // device-resident levels, no NaN: scans on the GPU
    const int64_t best = int64_t(sc[0]);
    if (n > 1) {
      const int64_t runner = int64_t(sc[1]);
      const double spread = std::hypot(sc[3] - sc[2], sc[5] - sc[4]);  // spread_of / spread_of_c
      const double thr = o.degeneracy_tol * std::max(1.0, spread);
      double br, bi, rr, ri;
      dev_level(ctx, ps, best, &br, &bi);
      dev_level(ctx, ps, runner, &rr, &ri);
      if (br - rr < thr) {
        if (err) {
          err->i = best;
          err->j = runner;
          err->ei = br;
          err->ej = rr;
          err->ei_im = bi;
          err->ej_im = ri;
        }
        set_err(err, DPT_ERR_DEGENERATE, "dominant_eigenpair: ambiguous dominant level");
        return DPT_ERR_DEGENERATE;
      }
      const int64_t bj = dev_partner(ctx, ps, best, thr, err);
      if (bj >= 0) degenerate_error_dev(ctx, ps, best, bj, err);
    }
    pt.mark("dominant: device selection");
    return run_single(ctx, p, best, &o, 0.0, nullptr, nullptr, z_chart, out_mem, rep, nullptr, 0, 0.0, nullptr,
                      z_unit, err);
  }
  std::vector<double> dcopy;  // device levels only: host levels are read in place
  if (p->mem != DPT_MEM_HOST) dcopy = host_levels(p, err);
  const double* dl = p->mem == DPT_MEM_HOST ? p->d : dcopy.data();
  pt.mark("dominant: host_levels");
  const int cx = p->is_complex ? 2 : 1;
  auto re = [&](int64_t i) { return dl[size_t(cx * i)]; };
  int64_t best = 0;  // first argmax of Re d (dpt.cpp:404-406)
  for (int64_t i = 1; i < n; ++i)
    if (re(i) > re(best)) best = i;
  if (n > 1) {  // runner-up ambiguity (dpt.cpp:408-419)
    int64_t runner = best == 0 ? 1 : 0;
    for (int64_t i = 0; i < n; ++i) {
      if (i == best) continue;
      if (re(i) > re(runner)) runner = i;
    }
    const double thr = cx == 2 ? threshold_of_c(n, dl, o.degeneracy_tol) : threshold_of(n, dl, o.degeneracy_tol);
    if (re(best) - re(runner) < thr) {
      if (err) {
        err->i = best;
        err->j = runner;
        err->ei = re(best);
        err->ej = re(runner);
        err->ei_im = cx == 2 ? dl[size_t(2 * best + 1)] : 0.0;
        err->ej_im = cx == 2 ? dl[size_t(2 * runner + 1)] : 0.0;
      }
      set_err(err, DPT_ERR_DEGENERATE, "dominant_eigenpair: ambiguous dominant level");
      return DPT_ERR_DEGENERATE;
    }
  }
  int64_t bj;
  const bool deg = cx == 2 ? find_degenerate_row_c(n, dl, best, o.degeneracy_tol, &bj)
                           : find_degenerate_row(n, dl, best, o.degeneracy_tol, &bj);
  if (deg) degenerate_error(err, best, bj, dl, cx == 2);
  pt.mark("dominant: selection");
  return run_single(ctx, p, best, &o, 0.0, nullptr, nullptr, z_chart, out_mem, rep, nullptr, 0, 0.0, nullptr,
                    z_unit, err);
  DPT_API_END
}

int dpt_step_single(dpt_ctx* ctx, const dpt_problem* p, const double* z, int64_t row, double lambda, double* out,
                    int io_mem, dpt_error_info* err) {
  DPT_API_BEGIN
  validate(p, err);
  if (row < 0 || row >= p->n) {
    set_err(err, DPT_ERR_SHAPE, "step_single: dimension mismatch");
    return DPT_ERR_SHAPE;
  }
  return run_single(ctx, p, row, nullptr, 0.0, nullptr, nullptr, out, io_mem, nullptr, z, io_mem, lambda, nullptr,
                    nullptr, err);
  DPT_API_END
}

int dpt_eigenvalue_of(dpt_ctx* ctx, const dpt_problem* p, const double* z, int64_t row, double lambda, double* out,
                      int z_mem, dpt_error_info* err) {
  DPT_API_BEGIN
  validate(p, err);
  if (row < 0 || row >= p->n) {  // dpt.cpp:361-362
    set_err(err, DPT_ERR_SHAPE, "eigenvalue_of: dimension mismatch");
    return DPT_ERR_SHAPE;
  }
  return run_single(ctx, p, row, nullptr, 0.0, nullptr, nullptr, nullptr, z_mem, nullptr, z, z_mem, lambda, out,
                    nullptr, err);
  DPT_API_END
}

int dpt_iterate_fixed_c(dpt_ctx* ctx, const dpt_problem* p, int k, double lambda, double lambda_im, double* a_out,
                        int out_mem, dpt_report* rep, dpt_error_info* err) {
  DPT_API_BEGIN
  if (k < 0) {
    set_err(err, DPT_ERR_INVALID_ARG, "iterate_fixed: negative step count");
    return DPT_ERR_INVALID_ARG;
  }
  return run_full(ctx, p, nullptr, false, 0.0, k, lambda, nullptr, nullptr, a_out, nullptr, nullptr, out_mem, rep,
                  err, lambda_im);
  DPT_API_END
}

int dpt_step_full_gap_c(dpt_ctx* ctx, const dpt_problem* p, const double* a, const double* gap, double lambda,
                        double lambda_im, double* out, int io_mem, dpt_error_info* err) {
  DPT_API_BEGIN
  return run_step_full(ctx, p, a, gap, lambda, out, io_mem, nullptr, nullptr, err, lambda_im);
  DPT_API_END
}

int dpt_step_single_gap_c(dpt_ctx* ctx, const dpt_problem* p, const double* z, int64_t row, const double* gap_row,
                          double lambda, double lambda_im, double* out, int io_mem, dpt_error_info* err) {
  DPT_API_BEGIN
  validate(p, err);
  if (row < 0 || row >= p->n) {
    set_err(err, DPT_ERR_SHAPE, "step_single: dimension mismatch");
    return DPT_ERR_SHAPE;
  }
  return run_single(ctx, p, row, nullptr, 0.0, nullptr, nullptr, out, io_mem, nullptr, z, io_mem, lambda, nullptr,
                    nullptr, err, gap_row, lambda_im);
  DPT_API_END
}

int dpt_eigenvalue_of_c(dpt_ctx* ctx, const dpt_problem* p, const double* z, int64_t row, double lambda,
                        double lambda_im, double* out2, int z_mem, dpt_error_info* err) {
  DPT_API_BEGIN
  validate(p, err);
  if (row < 0 || row >= p->n) {
    set_err(err, DPT_ERR_SHAPE, "eigenvalue_of: dimension mismatch");
    return DPT_ERR_SHAPE;
  }
  return run_single(ctx, p, row, nullptr, 0.0, nullptr, nullptr, nullptr, z_mem, nullptr, z, z_mem, lambda, out2,
                    nullptr, err, nullptr, lambda_im);
  DPT_API_END
}

int dpt_check_degenerate(int64_t n, const double* d, double tol, int64_t* i, int64_t* j) {
  return find_degenerate(n, d, tol, i, j) ? 1 : 0;
}

double dpt_spectral_spread(int64_t n, const double* d) { return spread_of(n, d); }

int dpt_effective_window(int requested, int64_t n) { return effective_window(requested, n); }
int dpt_homotopy_solve(dpt_ctx* ctx, const dpt_problem* p, int stages, const dpt_options* opts, double* a_out,
                       double* eig_out, double* res_out, int out_mem, dpt_report* rep, dpt_error_info* err) {
  DPT_API_BEGIN
  return run_homotopy(ctx, p, stages, opts, a_out, eig_out, res_out, out_mem, rep, err);
  DPT_API_END
}

// ---------------------------------------------- dense linear algebra ----
// matmul(Dense, Dense) (matrix.cpp:130-143) and solve_linear_multi
// (matrix.cpp:519-533) on the device kernels of the homotopy (linalg.cu).
namespace {
void put_padded(dpt_ctx* ctx, DBuf& b, const double* src, int64_t rows, int64_t cols_d, int64_t ld, int mem,
                dpt_error_info* err) {
  dalloc(b, size_t(std::max<int64_t>(rows, 1)) * size_t(ld) * 8, err);
  CK(cudaMemsetAsync(b.p, 0, size_t(std::max<int64_t>(rows, 1)) * size_t(ld) * 8, ctx->stream));
  if (rows && cols_d)
    CK(copy2d_async(ctx, b.p, size_t(ld) * 8, src, size_t(cols_d) * 8, size_t(cols_d) * 8, size_t(rows),
                    mem == DPT_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice));
}
void get_padded(dpt_ctx* ctx, double* dst, const DBuf& b, int64_t rows, int64_t cols_d, int64_t ld, int mem,
                dpt_error_info* err) {
  if (rows && cols_d)
    CK(copy2d_async(ctx, dst, size_t(cols_d) * 8, b.p, size_t(ld) * 8, size_t(cols_d) * 8, size_t(rows),
                    mem == DPT_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost));
  CK(cudaStreamSynchronize(ctx->stream));
}
int64_t even_ld(int64_t v) { return (v + 1) & ~int64_t(1); }
}  // namespace

int dpt_matmul_dense(dpt_ctx* ctx, int64_t m, int64_t k, int64_t n, int is_complex, const double* a, const double* b,
                     double* c, int mem, dpt_error_info* err) {
  DPT_API_BEGIN
  Guard g(ctx);
  if (m < 0 || k < 0 || n < 0) {
    set_err(err, DPT_ERR_SHAPE, "matmul shape mismatch");
    return DPT_ERR_SHAPE;
  }
  const int cx = is_complex ? 2 : 1;
  cudaStream_t st = ctx->stream;
  DBuf ba, bb, bop, bc;
  const int64_t lda = even_ld(cx * k), ldc = even_ld(cx * n), ldop = even_ld(cx * k);
  put_padded(ctx, ba, a, m, cx * k, lda, mem, err);
  put_padded(ctx, bb, b, k, cx * n, even_ld(cx * n), mem, err);
  dalloc(bop, size_t(std::max<int64_t>(cx * n, 1)) * size_t(std::max<int64_t>(ldop, 2)) * 8, err);
  dalloc(bc, size_t(std::max<int64_t>(m, 1)) * size_t(ldc) * 8, err);
  if (k == 0) {
    CK(cudaMemsetAsync(bc.p, 0, size_t(std::max<int64_t>(m, 1)) * size_t(ldc) * 8, st));
  } else if (m && n) {
    CK(launch_gemm_bop(cx, true, bb.as<double>(), even_ld(cx * n) / cx, n, k, bop.as<double>(), ldop, st));
    CK(launch_gemm_nt(m, cx * n, cx * k, ba.as<double>(), lda, bop.as<double>(), ldop, 1.0, 0.0, bc.as<double>(), ldc,
                      st));
    ctx->launches += 2;
  }
  get_padded(ctx, c, bc, m, cx * n, ldc, mem, err);
  return DPT_OK;
  DPT_API_END
}

int dpt_solve_linear_multi(dpt_ctx* ctx, int64_t n, int64_t nrhs, int is_complex, const double* a, const double* b,
                           double* x, int mem, dpt_error_info* err) {
  DPT_API_BEGIN
  Guard g(ctx);
  const int cx = is_complex ? 2 : 1;
  if (n < 0 || nrhs < 0) {
    set_err(err, DPT_ERR_SHAPE, "solve_linear_multi shape mismatch");
    return DPT_ERR_SHAPE;
  }
  if (n > lu_max_n(cx)) {
    set_err(err, DPT_ERR_UNSUPPORTED, "solve_linear_multi: n exceeds the device LU's cluster panel capacity");
    return DPT_ERR_UNSUPPORTED;
  }
  if (n == 0) return DPT_OK;
  cudaStream_t st = ctx->stream;
  const int64_t lda = even_ld(cx * n), ldx = even_ld(cx * std::max<int64_t>(nrhs, 1));
  DBuf ba, bb, bx, bpiv, bperm, binfo, bscr;
  put_padded(ctx, ba, a, n, cx * n, lda, mem, err);
  put_padded(ctx, bb, b, n, cx * nrhs, ldx, mem, err);
  dalloc(bx, size_t(n) * size_t(ldx) * 8, err);
  dalloc(bpiv, size_t(n) * 8, err);
  dalloc(bperm, size_t(n) * 8, err);
  dalloc(binfo, 16, err);
  dalloc(bscr, size_t(4) * size_t(std::max(n, nrhs)) * 128 * 8 + 4096, err);
  int nl = 0;
  CK(launch_lu_factor(cx, ba.as<double>(), lda, n, bpiv.as<int64_t>(), binfo.as<int>(), bscr.as<double>(), &nl, st));
  int hinfo = 0;
  std::vector<int64_t> hpiv(static_cast<size_t>(n)), hperm(static_cast<size_t>(n));
  CK(cudaMemcpyAsync(&hinfo, binfo.p, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(hpiv.data(), bpiv.p, size_t(n) * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (hinfo >= 1 && hinfo <= n) {
    set_err(err, DPT_ERR_UNSUPPORTED, "solve_linear: singular matrix");
    return DPT_ERR_UNSUPPORTED;
  }
  for (int64_t i = 0; i < n; ++i) hperm[size_t(i)] = i;
  for (int64_t i = 0; i < n; ++i) std::swap(hperm[size_t(i)], hperm[size_t(hpiv[size_t(i)])]);
  CK(cudaMemcpyAsync(bperm.p, hperm.data(), size_t(n) * 8, cudaMemcpyHostToDevice, st));
  CK(launch_gather_rows(bb.as<double>(), ldx, bperm.as<int64_t>(), n, ldx, bx.as<double>(), st));
  if (nrhs) CK(launch_lu_solve(cx, ba.as<double>(), lda, n, bx.as<double>(), ldx, nrhs, bscr.as<double>(), &nl, st));
  ctx->launches += nl + 1;
  get_padded(ctx, x, bx, n, cx * nrhs, ldx, mem, err);
  return DPT_OK;
  DPT_API_END
}

// ------------------------------------------------------------ scan_domain ----
// analysis.cpp:68-138.  Cells of the lambda grid are independent solves; small
// problems run batched (scan.cu, one warp per cell, the reference's operation
// order), larger ones cell by cell through the solver.
static double grid_coordinate(double lo, double hi, int64_t res, int64_t i) {  // analysis.cpp:42-46
  if (res == 1) return 0.5 * (lo + hi);
  return lo + (hi - lo) * (double(i) / double(res - 1));
}

int dpt_scan_domain(dpt_ctx* ctx, const dpt_problem* p, const dpt_scan_grid* grid, int mode, int64_t row,
                    double ramp_alpha, const dpt_options* opts, uint8_t* classes, int32_t* iterations,
                    dpt_error_info* err) {
  DPT_API_BEGIN
  Guard g(ctx);
  validate(p, err);
  if (!grid || grid->res_re <= 0 || grid->res_im <= 0) {
    set_err(err, DPT_ERR_SHAPE, "scan_domain: empty grid");
    return DPT_ERR_SHAPE;
  }
  const bool single = mode == DPT_SCAN_SINGLE_ROW;
  const int64_t n = p->n;
  if (single && (row < 0 || row >= n)) {
    set_err(err, DPT_ERR_SHAPE, "scan_domain: row out of range");
    return DPT_ERR_SHAPE;
  }
  if (!(ramp_alpha >= 0.0) || ramp_alpha >= 1.0) {
    set_err(err, DPT_ERR_INVALID_ARG, "scan_domain: ramp alpha must lie in [0, 1)");
    return DPT_ERR_INVALID_ARG;
  }
  const dpt_options o = opts_or_default(opts);
  // the spectrum is validated once up front (analysis.cpp:76-80)
  std::vector<double> dh = host_levels(p, err);
  if (single) {
    int64_t bj;
    const bool deg = p->is_complex ? find_degenerate_row_c(n, dh.data(), row, o.degeneracy_tol, &bj)
                                   : find_degenerate_row(n, dh.data(), row, o.degeneracy_tol, &bj);
    if (deg) degenerate_error(err, row, bj, dh.data(), p->is_complex != 0);
  } else {
    check_levels(p, dh, o.degeneracy_tol, err);
  }
  const int64_t cells = grid->res_re * grid->res_im;
  if (cells == 0 || !classes || !iterations) return DPT_OK;
  // complex host images of the problem (the reference's cdouble data)
  typedef std::complex<double> cd_t;
  std::vector<cd_t> d(static_cast<size_t>(n)), D(static_cast<size_t>(n * n), cd_t(0.0, 0.0));
  for (int64_t i = 0; i < n; ++i) d[size_t(i)] = p->is_complex ? cd_t(dh[size_t(2 * i)], dh[size_t(2 * i + 1)]) : cd_t(dh[size_t(i)], 0.0);
  {
    const cudaMemcpyKind hk = p->mem == DPT_MEM_DEVICE ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost;
    const int cx = p->is_complex ? 2 : 1;
    if (p->delta_kind == DPT_DELTA_DENSE) {
      std::vector<double> raw(size_t(cx * n * n));
      if (n) CK(to_host_ordered(raw.data(), p->delta, raw.size() * 8, hk));
      for (int64_t q = 0; q < n * n; ++q) D[size_t(q)] = cx == 2 ? cd_t(raw[size_t(2 * q)], raw[size_t(2 * q + 1)]) : cd_t(raw[size_t(q)], 0.0);
    } else {
      std::vector<int64_t> rp(size_t(n + 1));
      CK(to_host_ordered(rp.data(), p->rowptr, size_t(n + 1) * 8, hk));
      const int64_t nnz = rp[size_t(n)];
      std::vector<int32_t> cl(static_cast<size_t>(nnz));
      std::vector<double> vl(static_cast<size_t>(cx * nnz));
      if (nnz) {
        CK(to_host_ordered(cl.data(), p->cols, size_t(nnz) * 4, hk));
        CK(to_host_ordered(vl.data(), p->vals, size_t(cx * nnz) * 8, hk));
      }
      for (int64_t i = 0; i < n; ++i)
        for (int64_t q = rp[size_t(i)]; q < rp[size_t(i + 1)]; ++q)
          D[size_t(i * n + cl[size_t(q)])] = cx == 2 ? cd_t(vl[size_t(2 * q)], vl[size_t(2 * q + 1)]) : cd_t(vl[size_t(q)], 0.0);
    }
  }
  std::vector<double> re_at(static_cast<size_t>(grid->res_re)), im_at(static_cast<size_t>(grid->res_im));
  for (int64_t j = 0; j < grid->res_re; ++j) re_at[size_t(j)] = grid_coordinate(grid->re_min, grid->re_max, grid->res_re, j);
  for (int64_t i = 0; i < grid->res_im; ++i) im_at[size_t(i)] = grid_coordinate(grid->im_min, grid->im_max, grid->res_im, i);
  const bool ramped = ramp_alpha > 0.0;
  std::vector<double> ramp;
  if (ramped) {
    ramp.assign(size_t(std::max(o.max_iter, 0)) + 2, 0.0);
    for (int k = 1; k <= o.max_iter; ++k) ramp[size_t(k)] = 1.0 - std::pow(ramp_alpha, double(k - 1));
  }
  cudaStream_t st = ctx->stream;

  if (n <= scan_max_n(single ? 1 : 0)) {
    std::vector<cd_t> tab(static_cast<size_t>(single ? n : n * n), cd_t(0.0, 0.0));
    if (single) {
      for (int64_t m = 0; m < n; ++m)
        if (m != row) tab[size_t(m)] = 1.0 / (d[size_t(row)] - d[size_t(m)]);  // build_gap_row, partition.cpp:83-96
    } else {
      for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < n; ++j)
          if (i != j) tab[size_t(i * n + j)] = 1.0 / (d[size_t(i)] - d[size_t(j)]);  // build_theta, :69-81
    }
    std::vector<cd_t> Dt;
    if (!single) {
      Dt.resize(size_t(n * n));
      for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < n; ++j) Dt[size_t(j * n + i)] = D[size_t(i * n + j)];
    }
    const int win = single ? (o.cycle_window >= 2 ? o.cycle_window : 0) : effective_window(o.cycle_window, n);
    int64_t warps = std::min<int64_t>(cells, 148 * 64);
    const size_t per_warp = size_t(win > 1 ? win - 1 : 0) * size_t(single ? n : n * n) * 16;
    if (per_warp > 0) warps = std::max<int64_t>(1, std::min<int64_t>(warps, int64_t((size_t(1) << 30) / per_warp)));
    {  // n <= 3: one thread per cell, a ring per thread
      ScanArgs probe{};
      probe.n = int(n);
      probe.cells = cells;
      const int64_t tt = scan_tiny_threads(probe);
      if (tt > 0) warps = tt;  // ring sized per thread below (per_warp is per ring owner)
    }
    DBuf bd, bD, bt, bre, bim, bramp, bring, bcls, bit;
    dalloc(bd, size_t(n) * 16, err);
    dalloc(bD, size_t(n * n) * 16, err);
    dalloc(bt, tab.size() * 16, err);
    dalloc(bre, re_at.size() * 8, err);
    dalloc(bim, im_at.size() * 8, err);
    if (ramped) dalloc(bramp, ramp.size() * 8, err);
    dalloc(bring, std::max<size_t>(per_warp * size_t(warps), 16), err);
    dalloc(bcls, size_t(cells), err);
    dalloc(bit, size_t(cells) * 4, err);
    CK(cudaMemcpyAsync(bd.p, d.data(), size_t(n) * 16, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(bD.p, single ? D.data() : Dt.data(), size_t(n * n) * 16, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(bt.p, tab.data(), tab.size() * 16, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(bre.p, re_at.data(), re_at.size() * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(bim.p, im_at.data(), im_at.size() * 8, cudaMemcpyHostToDevice, st));
    if (ramped) CK(cudaMemcpyAsync(bramp.p, ramp.data(), ramp.size() * 8, cudaMemcpyHostToDevice, st));
    ScanArgs a{};
    a.cells = cells;
    a.res_re = grid->res_re;
    a.n = int(n);
    a.single = single ? 1 : 0;
    a.row = int(row);
    a.max_iter = o.max_iter;
    a.win = win;
    a.tol = o.tol;
    a.res_tol = o.residual_tol;
    a.div_thr = o.divergence_threshold;
    a.d = bd.as<double>();
    a.delta = single ? bD.as<double>() : nullptr;
    a.delta_t = single ? nullptr : bD.as<double>();
    a.theta = single ? nullptr : bt.as<double>();
    a.gap_row = single ? bt.as<double>() : nullptr;
    a.re_at = bre.as<double>();
    a.im_at = bim.as<double>();
    a.ramp = ramped ? bramp.as<double>() : nullptr;
    a.ring = bring.as<double>();
    a.classes = bcls.as<uint8_t>();
    a.iterations = bit.as<int32_t>();
    CK(cudaEventRecord(ctx->ev0, st));
    CK(launch_scan(a, int(warps), st));
    ctx->launches += 1;
    CK(cudaEventRecord(ctx->ev1, st));
    CK(cudaMemcpyAsync(classes, bcls.p, size_t(cells), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(iterations, bit.p, size_t(cells) * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return DPT_OK;
  }

  // larger problems: one GPU solve per cell on the complex path
  std::vector<double> dc(size_t(2 * n)), Dc;
  for (int64_t i = 0; i < n; ++i) {
    dc[size_t(2 * i)] = d[size_t(i)].real();
    dc[size_t(2 * i + 1)] = d[size_t(i)].imag();
  }
  Dc.resize(size_t(2 * n * n));
  for (int64_t q = 0; q < n * n; ++q) {
    Dc[size_t(2 * q)] = D[size_t(q)].real();
    Dc[size_t(2 * q + 1)] = D[size_t(q)].imag();
  }
  dpt_problem c{};
  c.n = n;
  c.d = dc.data();
  c.delta_kind = DPT_DELTA_DENSE;
  c.delta = Dc.data();
  c.mem = DPT_MEM_HOST;
  c.is_complex = 1;
  for (int64_t cell = 0; cell < cells; ++cell) {
    c.lambda = re_at[size_t(cell % grid->res_re)];
    c.lambda_im = im_at[size_t(cell / grid->res_re)];
    dpt_report r{};
    int rc;
    if (single)
      rc = run_single(ctx, &c, row, &o, ramp_alpha, nullptr, nullptr, nullptr, DPT_MEM_HOST, &r, nullptr, 0, 0.0,
                      nullptr, nullptr, err);
    else
      rc = run_full(ctx, &c, &o, ramped, ramp_alpha, -1, 0.0, nullptr, nullptr, nullptr, nullptr, nullptr,
                    DPT_MEM_HOST, &r, err);
    if (rc != DPT_OK) return rc;
    classes[cell] = uint8_t(r.status == DPT_CONVERGED ? 0 : (r.status == DPT_DIVERGED ? 2 : 1));
    iterations[cell] = r.iterations;
  }
  return DPT_OK;
  DPT_API_END
}


size_t dpt_sm_state_bytes(void) { return sizeof(dpt_sm_state) + sizeof(dpt_sm_options); }

void dpt_sm_init(void* state, void* opts, const dpt_options* o, int win, int have_trace) {
  memset(state, 0, sizeof(dpt_sm_state));
  dpt_sm_options* so = static_cast<dpt_sm_options*>(opts);
  memset(so, 0, sizeof(*so));
  so->tol = o->tol;
  so->residual_tol = o->residual_tol;
  so->divergence_threshold = o->divergence_threshold;
  so->max_iter = o->max_iter;
  so->win = win;
  so->have_trace = have_trace;
}

void dpt_sm_decide_host(void* state, const void* opts, const double* stats, int j, int settled_prev,
                        int settled_cur, double* trace_out) {
  dpt_sm_decide(static_cast<dpt_sm_state*>(state), static_cast<const dpt_sm_options*>(opts), stats, j,
                settled_prev, settled_cur, trace_out);
}

void dpt_sm_query(const void* state, int* done, int* status, int* iterations, int* final_iter, int* readoffs,
                  int* cycle_pending, double* step_norm) {
  const dpt_sm_state* s = static_cast<const dpt_sm_state*>(state);
  *done = s->done;
  *status = s->status;
  *iterations = s->iterations;
  *final_iter = s->final_iter;
  *readoffs = s->readoffs;
  *cycle_pending = s->cycle_pending;
  *step_norm = s->step_norm;
}

}  // extern "C"

// ============================================================ plans ====
// A plan keeps a problem resident in HBM with its workspace, for repeated
// solves / fixed-step throughput runs (the bench's device-resident `value`).
struct dpt_plan {
  dpt_ctx* ctx = nullptr;
  DevProblem dp;
  Work w;
  Mode mode = MODE_DENSE_FULL;
  int64_t row = 0;
  int nslots = 2;
  int issued = 0;
  cudaEvent_t k0 = nullptr, k1 = nullptr;
  ~dpt_plan() {
    if (k0) cudaEventDestroy(k0);
    if (k1) cudaEventDestroy(k1);
  }
};

extern "C" {

int dpt_plan_create(dpt_ctx* ctx, const dpt_problem* p, int single, int64_t row, double lambda, dpt_plan** out,
                    dpt_error_info* err) {
  DPT_API_BEGIN
  Guard g(ctx);
  validate(p, err);
  std::unique_ptr<dpt_plan> pl(new dpt_plan());
  pl->ctx = ctx;
  upload(pl->dp, ctx, p, err, !single && p->delta_kind == DPT_DELTA_CSR);
  const int64_t n = p->n;
  if (n == 0) {
    set_err(err, DPT_ERR_SHAPE, "plan: empty problem");
    return DPT_ERR_SHAPE;
  }
  pl->mode = single ? MODE_SINGLE : (p->delta_kind == DPT_DELTA_DENSE ? MODE_DENSE_FULL : MODE_CSR_FULL);
  pl->row = row;
  dpt_sm_options so{};
  so.max_iter = 1 << 30;
  if (single) {
    if (row < 0 || row >= n) {
      set_err(err, DPT_ERR_SHAPE, "plan: row out of range");
      return DPT_ERR_SHAPE;
    }
    make_work(pl->w, ctx, pl->dp, MODE_SINGLE, row, 1, 1, 2, 0, nullptr, nullptr, so, lambda, 1, err);
  } else {
    int64_t row0, rows;
    shard_rows(ctx, n, &row0, &rows);
    const int64_t per = (n + ctx->world - 1) / ctx->world;
    make_work(pl->w, ctx, pl->dp, pl->mode, row0, rows, per, 2, 0, nullptr, nullptr, so, lambda, 1, err);
  }
  CK(cudaEventCreate(&pl->k0));
  CK(cudaEventCreate(&pl->k1));
  CK(cudaStreamSynchronize(ctx->stream));
  *out = pl.release();
  return DPT_OK;
  DPT_API_END
}

void dpt_plan_destroy(dpt_plan* pl) {
  if (!pl) return;
  Guard g(pl->ctx);
  delete pl;
}

// Restart from A_0 = I (or e_row) and run launch 1: afterwards the plan holds A_1.
int dpt_plan_begin(dpt_plan* pl, dpt_error_info* err) {
  DPT_API_BEGIN
  Guard g(pl->ctx);
  dpt_ctx* ctx = pl->ctx;
  Work& w = pl->w;
  cudaStream_t st = ctx->stream;
  CK(cudaMemsetAsync(w.s.state, 0, sizeof(dpt_sm_state), st));
  CK(cudaMemsetAsync(w.s.counter, 0, 16, st));
  if (pl->mode == MODE_DENSE_FULL) {
    CK(launch_dense_init(w.s, pl->dp.delta.as<double>(), pl->dp.big, st));
    ctx->launches += 1;
    post_step(ctx, w, dense_init_ntiles(w.s.rows, w.s.ntn, w.s.cplx), 0, err);
  } else {
    if (pl->mode == MODE_SINGLE)
      CK(launch_identity(w.s, st));
    else
      put_identity(ctx, w, pl->dp, err);
    step_launch(ctx, w, pl->dp, pl->mode, pl->row, err);
    post_step(ctx, w, w.ntiles_step, 0, err);
  }
  pl->issued = 1;
  return DPT_OK;
  DPT_API_END
}

// Enqueue k more fixed steps (iterate_fixed semantics: no gates).  With
// kernel_ms != NULL each step kernel is bracketed by CUDA events on the
// context stream and the summed kernel time is returned (synchronises).
int dpt_plan_steps(dpt_plan* pl, int k, double* kernel_ms, dpt_error_info* err) {
  DPT_API_BEGIN
  Guard g(pl->ctx);
  dpt_ctx* ctx = pl->ctx;
  Work& w = pl->w;
  double tot = 0.0;
  for (int i = 0; i < k; ++i) {
    if (kernel_ms) CK(cudaEventRecord(pl->k0, ctx->stream));
    step_launch(ctx, w, pl->dp, pl->mode, pl->row, err);
    if (kernel_ms) CK(cudaEventRecord(pl->k1, ctx->stream));
    post_step(ctx, w, w.ntiles_step, 0, err);
    if (kernel_ms) {
      CK(cudaEventSynchronize(pl->k1));
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, pl->k0, pl->k1));
      tot += ms;
    }
  }
  pl->issued += k;
  if (kernel_ms) *kernel_ms = tot;
  return DPT_OK;
  DPT_API_END
}

// Copy the current iterate (A_issued or z_issued) out.
int dpt_plan_read(dpt_plan* pl, double* out, int out_mem, dpt_error_info* err) {
  DPT_API_BEGIN
  Guard g(pl->ctx);
  if (pl->mode == MODE_SINGLE || !sharded(pl->ctx))
    copy_slot_out(out, pl->w, pl->dp, pl->issued % 2, out_mem, pl->ctx->stream, err);
  else
    gather_rows(pl->ctx, pl->w, pl->dp, pl->issued % 2, out, out_mem, err);
  CK(cudaStreamSynchronize(pl->ctx->stream));
  return DPT_OK;
  DPT_API_END
}

// Statistics of the latest launch (step, max|A|, nonfinite, max residual of the previous iterate).
int dpt_plan_stats(dpt_plan* pl, double* out4, dpt_error_info* err) {
  DPT_API_BEGIN
  Guard g(pl->ctx);
  CK(cudaMemcpyAsync(out4, pl->w.s.stats, 4 * sizeof(double), cudaMemcpyDeviceToHost, pl->ctx->stream));
  CK(cudaStreamSynchronize(pl->ctx->stream));
  return DPT_OK;
  DPT_API_END
}

}  // extern "C"
