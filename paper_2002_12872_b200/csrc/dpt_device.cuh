// dpt_device.cuh -- device-side plumbing shared by the DPT kernels:
// the per-solve device workspace descriptor, PTX wrappers (mbarrier, TMA,
// DMMA) and deterministic warp reductions.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "dpt_state.h"

namespace dpt {

// Function attributes (cudaFuncSetAttribute) are per device, and one process
// may drive several devices (dpt_ctx_create(device)): `mask` holds one bit per
// device ordinal on which the attributes were already set. The bit is set only
// after the attributes, so a concurrent caller can at worst set them twice.
struct DeviceAttrOnce {
  std::atomic<unsigned long long> mask{0};
  template <class F>
  void operator()(F&& set) {
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ull << (dev & 63);
    if (mask.load(std::memory_order_acquire) & bit) return;
    set();
    mask.fetch_or(bit, std::memory_order_release);
  }
};

// Everything a launch needs that may change from iteration to iteration is
// read from device memory (the state / tables below), so one captured CUDA
// graph of K iterations can be replayed unchanged.
struct DevSolve {
  int64_t n;            // global problem size (columns of A, length of theta)
  int64_t row0, rows;   // this rank's row shard [row0, row0 + rows)
  int64_t ld;           // leading dimension (doubles) of A slots: ncol rounded up to even
  int64_t ncol;         // real columns per iterate row: n (real) or 2n (complex, interleaved re/im)
  int64_t ldd;          // leading dimension (doubles) of the device Delta rows
  int cplx;             // complex FP64 (std::complex<double> layout everywhere)
  double lambda_im;     // Im p.lambda (complex problems)
  int nslots;           // ring of iterates A_m in slot m % nslots
  int64_t slot_elems;   // doubles per slot (>= rows * ld; equal on every rank for the gather)
  int ntn;              // column partial blocks per row (rowpart leading dim)
  double lambda;        // p.lambda (read-offs always use it, dpt.cpp:23-44)
  const double* theta;  // [n] unperturbed levels (device)
  const double* gapmat; // optional explicit gap matrix (step_full / step_single with a caller
                        // GapMatrix / GapRow): row-major [rows x ld] (full) or [n] (row map)
  const double* lam_table;  // [max_iter + 2] lambda_k (ramped schedule) or null
  const int* settled_table; // [max_iter + 2] settled(k) or null (=1)
  double* slots;        // nslots * rows * n, row-major per slot (row-local)
  double* dvec[2];      // d_m(i) = P(A_m)(i,i) for local rows, m % 2
  double* eps;          // [rows] read-offs of the latest folded iterate
  double* res;          // [rows]
  double* rowpart;      // [4][rows][ntn] (sum d, max num, max den, sum d im), see rp_index
  double* tilepart;     // [ntiles][4] (max step, max |A|, nonfinite count, spare)
  int ntiles;
  double* blockpart;    // fold partials [fold_blocks][8]
  double* stats;        // [DPT_NSTATS] after (optional) cross-rank max
  dpt_sm_state* state;
  dpt_sm_options opts;
  double* trace;        // [3 * (max_iter + 1)] (k, step, max_res) log
  unsigned int* counter;  // last-block election for the folds
  double* cyclepart;    // [fold_blocks][DPT_MAX_WINDOW]
  int fixed_mode;       // iterate_fixed: no decisions, step every launch
  int fuse_decide;      // single rank: the fold's last block also runs the decision
  double* sk_ws;        // stream-K K1 (small n): per-CTA partial-tile slots, or null
  unsigned* sk_cnt;     // stream-K K1: per-tile part counters
  // device-side iteration loop (CUDA graph WHILE node, solver.cu drive_graph):
  // the fold's decision sets the loop condition; 0 = launched from the host.
  int has_loop;
  int loop_total;                      // last launch index the loop may run
  unsigned long long loop_cond;        // cudaGraphConditionalHandle
};

// Last-block election fences.  __threadfence() is fence.sc.gpu (MEMBAR.SC.GPU),
// measured at 73k-165k cycles for the first one in a kernel on B200
// (tools/probe/latency.cu); the release/acquire pattern only needs acq_rel
// (~800 cycles): writers release their partials before the counter atomic,
// the elected last block acquires them after it.
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

__device__ __forceinline__ int launch_index(const DevSolve& s) { return s.state->j + 1; }

// rowpart layout [4][rows][ntn]: a row's column-block partials are contiguous
// so the fold reads them coalesced.  k: 0 = sum d (re), 1 = max num, 2 = max den,
// 3 = sum d (im, complex problems).
__device__ __forceinline__ size_t rp_index(int k, int64_t row, int tn, int64_t rows, int ntn) {
  return (size_t(k) * size_t(rows) + size_t(row)) * size_t(ntn) + size_t(tn);
}

__device__ __forceinline__ double lam_of(const DevSolve& s, int j) {
  return s.lam_table ? s.lam_table[s.cplx ? 2 * j : j] : s.lambda;
}

// ------------------------------------------------------- complex FP64 ----
// The reference computes in std::complex<double> compiled without FMA
// contraction: products (ac - bd, ad + bc) with separately rounded terms,
// |z| = hypot, and 1/z by Smith's algorithm (libgcc __divdc3, normal range).
struct cd {
  double x, y;
};
__device__ __forceinline__ cd cmake(double x, double y) { return cd{x, y}; }
__device__ __forceinline__ cd cmul(cd a, cd b) {
  return cd{__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)), __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x))};
}
__device__ __forceinline__ cd cadd(cd a, cd b) { return cd{__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y)}; }
__device__ __forceinline__ cd csub(cd a, cd b) { return cd{__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y)}; }
__device__ __forceinline__ double cabs_(cd a) { return hypot(a.x, a.y); }
__device__ __forceinline__ cd crecip(cd z) {  // (1 + 0i) / z
  const double c = z.x, d = z.y;
  if (fabs(c) < fabs(d)) {
    const double ratio = c / d, denom = __dadd_rn(__dmul_rn(c, ratio), d);
    return cd{ratio / denom, -1.0 / denom};
  }
  const double ratio = d / c, denom = __dadd_rn(__dmul_rn(d, ratio), c);
  return cd{1.0 / denom, -ratio / denom};
}
__device__ __forceinline__ cd cdiv(cd x, cd z) {  // x / z, Smith's method (the finite-value path of __divdc3)
  const double a = x.x, b = x.y, c = z.x, d = z.y;
  if (fabs(c) < fabs(d)) {
    const double ratio = c / d, denom = __dadd_rn(__dmul_rn(c, ratio), d);
    return cd{__dadd_rn(__dmul_rn(a, ratio), b) / denom, __dsub_rn(__dmul_rn(b, ratio), a) / denom};
  }
  const double ratio = d / c, denom = __dadd_rn(__dmul_rn(d, ratio), c);
  return cd{__dadd_rn(__dmul_rn(b, ratio), a) / denom, __dsub_rn(b, __dmul_rn(a, ratio)) / denom};
}
__device__ __forceinline__ bool cfinite(cd a) { return isfinite(a.x) && isfinite(a.y); }
__device__ __forceinline__ cd lamc_of(const DevSolve& s, int j) {
  return s.lam_table ? cd{s.lam_table[2 * j], s.lam_table[2 * j + 1]} : cd{s.lambda, s.lambda_im};
}

// ---------------------------------------------------------------- PTX ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

// Consumer release of a stage (WAR handshake before an async-proxy refill):
// mbarrier.arrive is a release at CTA scope, so this lane's preceding shared
// reads are ordered before the producer's acquire (mbar_wait) of the phase.
__device__ __forceinline__ void mbar_arrive_release(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

// Orders the generic-proxy shared accesses made visible to this thread (the
// consumers' reads acquired through the empty barrier) before its subsequent
// async-proxy (cp.async.bulk) writes to shared memory.
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// 2-D TMA tile load (global -> shared), completion on an mbarrier.
__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, uint64_t* bar, int c0,
                                            int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];\n" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// 1-D bulk copy global -> shared (contiguous, 16-byte multiple), completion on an mbarrier.
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(tmap) : "memory");
}

// 16-byte shared-memory load from a 32-bit shared address (LDS.128, not a
// generic LD that must resolve the address space at run time).
__device__ __forceinline__ double2 lds128(uint32_t addr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}

// 8-byte shared-memory load from a 32-bit shared address (LDS.64 with an
// immediate offset; the address is data-dependent at every use, so the load
// cannot move above the barrier that publishes the data).
__device__ __forceinline__ double lds64(uint32_t addr) {
  double v;
  asm("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(addr));
  return v;
}

// D(8x8) += A(8x4, row) * B(4x8, col), FP64 tensor core (SASS DMMA.8x8x4).
// Fragments: a = A[lane>>2][lane&3], b = B[lane&3][lane>>2],
// d = {D[lane>>2][2(lane&3)], D[lane>>2][2(lane&3)+1]}.
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// ------------------------------------------------------- reductions ----
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace dpt
