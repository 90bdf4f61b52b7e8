// levels.cu -- device-side setup scans over the levels d and the CSR row
// pointer, so a solve on device-resident inputs never copies them to the host:
//
//   dominant_eigenpair's selection (proj/src/dpt.cpp:404-419): the first
//   argmax of Re d, the runner-up (first argmax over i != best), and the
//   spectral spread (proj/src/partition.cpp:42-53) for the ambiguity and
//   degeneracy thresholds;
//   build_gap_row's degeneracy scan (partition.cpp:83-96): the first m != row
//   with |d_row - d_m| <= thresh;
//   the uniform-16 CSR test that selects K3's fast path.
//
// Results are exact: max / min are order-independent, ties resolve to the
// lowest index as the reference's sequential scans do, and |d_row - d_m| is
// the same IEEE subtraction (complex: hypot).  Any NaN in d makes the host
// repeat the scan sequentially (the reference's NaN behaviour depends on scan
// order); the kernels only count them.
#include <cuda_runtime.h>
#include <stdint.h>

#include "dpt_device.cuh"
#include "dpt_kernels.h"

namespace dpt {

namespace {

constexpr int kLvThreads = 256;
constexpr int kLvBlocks = 296;

// (value, index) ordered by value desc, then index asc.
struct Top {
  double v;
  int64_t i;
};
__device__ __forceinline__ bool better(const Top& a, const Top& b) {
  return a.i >= 0 && (b.i < 0 || a.v > b.v || (a.v == b.v && a.i < b.i));
}
// merge two top-2 lists (distinct indices within each list)
__device__ __forceinline__ void merge2(Top& t0, Top& t1, const Top& u0, const Top& u1) {
  Top c[4] = {t0, t1, u0, u1};
  Top b0{0.0, -1}, b1{0.0, -1};
  for (int q = 0; q < 4; ++q) {
    if (c[q].i < 0) continue;
    if (better(c[q], b0)) {
      if (b0.i != c[q].i) b1 = b0;
      b0 = c[q];
    } else if (c[q].i != b0.i && better(c[q], b1)) {
      b1 = c[q];
    }
  }
  t0 = b0;
  t1 = b1;
}

// part layout per block: [0] top0.v [1] top0.i [2] top1.v [3] top1.i
//                        [4] lo re [5] hi re [6] lo im [7] hi im [8] nan count
__global__ void __launch_bounds__(kLvThreads) levels_scan_kernel(const double* __restrict__ d, int64_t n, int cx,
                                                                  double* part, unsigned* counter, double* out) {
  Top t0{0.0, -1}, t1{0.0, -1};
  double lr = INFINITY, hr = -INFINITY, li = INFINITY, hi = -INFINITY, nans = 0.0;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const double re = d[cx * i];
    const double im = cx == 2 ? d[cx * i + 1] : 0.0;
    if (isnan(re) || isnan(im)) {
      nans += 1.0;
      continue;
    }
    lr = fmin(lr, re);
    hr = fmax(hr, re);
    li = fmin(li, im);
    hi = fmax(hi, im);
    const Top c{re, i};
    const Top none{0.0, -1};
    merge2(t0, t1, c, none);
  }
  // block merge (the order does not matter: top-2 under a total order, exact
  // min / max, integer-valued counts), result in thread 0
  auto block_merge = [&]() {
    for (int o = 16; o > 0; o >>= 1) {
      Top u0{__shfl_xor_sync(0xffffffffu, t0.v, o), __shfl_xor_sync(0xffffffffu, t0.i, o)};
      Top u1{__shfl_xor_sync(0xffffffffu, t1.v, o), __shfl_xor_sync(0xffffffffu, t1.i, o)};
      merge2(t0, t1, u0, u1);
      lr = fmin(lr, __shfl_xor_sync(0xffffffffu, lr, o));
      hr = fmax(hr, __shfl_xor_sync(0xffffffffu, hr, o));
      li = fmin(li, __shfl_xor_sync(0xffffffffu, li, o));
      hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
      nans += __shfl_xor_sync(0xffffffffu, nans, o);
    }
    __shared__ double sh[kLvThreads / 32][9];
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
      sh[w][0] = t0.v;
      sh[w][1] = double(t0.i);
      sh[w][2] = t1.v;
      sh[w][3] = double(t1.i);
      sh[w][4] = lr;
      sh[w][5] = hr;
      sh[w][6] = li;
      sh[w][7] = hi;
      sh[w][8] = nans;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int q = 1; q < kLvThreads / 32; ++q) {
        merge2(t0, t1, Top{sh[q][0], int64_t(sh[q][1])}, Top{sh[q][2], int64_t(sh[q][3])});
        lr = fmin(lr, sh[q][4]);
        hr = fmax(hr, sh[q][5]);
        li = fmin(li, sh[q][6]);
        hi = fmax(hi, sh[q][7]);
        nans += sh[q][8];
      }
    }
    __syncthreads();
  };
  block_merge();
  __shared__ bool last;
  if (threadIdx.x == 0) {
    double* bp = part + size_t(blockIdx.x) * 9;
    bp[0] = t0.v;
    bp[1] = double(t0.i);
    bp[2] = t1.v;
    bp[3] = double(t1.i);
    bp[4] = lr;
    bp[5] = hr;
    bp[6] = li;
    bp[7] = hi;
    bp[8] = nans;
    fence_acq_rel_gpu();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  // the elected block merges the per-block parts with all its threads (a
  // serial loop over ~300 parts cost ~170 us of dependent L2 round trips)
  if (threadIdx.x == 0) fence_acq_rel_gpu();
  __syncthreads();
  t0 = Top{0.0, -1};
  t1 = Top{0.0, -1};
  lr = INFINITY;
  hr = -INFINITY;
  li = INFINITY;
  hi = -INFINITY;
  nans = 0.0;
  for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x) {
    const double* bp = part + size_t(b) * 9;
    merge2(t0, t1, Top{__ldcg(bp + 0), int64_t(__ldcg(bp + 1))}, Top{__ldcg(bp + 2), int64_t(__ldcg(bp + 3))});
    lr = fmin(lr, __ldcg(bp + 4));
    hr = fmax(hr, __ldcg(bp + 5));
    li = fmin(li, __ldcg(bp + 6));
    hi = fmax(hi, __ldcg(bp + 7));
    nans += __ldcg(bp + 8);
  }
  block_merge();
  if (threadIdx.x != 0) return;
  out[0] = double(t0.i);
  out[1] = double(t1.i);
  out[2] = lr;
  out[3] = hr;
  out[4] = li;
  out[5] = hi;
  out[6] = nans;
  *counter = 0u;
}

// first m != row with |d_row - d_m| <= thresh (complex: hypot of the
// component differences, as std::abs of the complex difference)
__global__ void __launch_bounds__(kLvThreads) levels_partner_kernel(const double* __restrict__ d, int64_t n, int cx,
                                                                     int64_t row, double thresh,
                                                                     unsigned long long* first) {
  const double rr = d[cx * row], ri = cx == 2 ? d[cx * row + 1] : 0.0;
  unsigned long long best = ~0ull;
  for (int64_t m = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; m < n; m += int64_t(gridDim.x) * blockDim.x) {
    if (m == row) continue;
    double g;
    if (cx == 2)
      g = hypot(rr - d[2 * m], ri - d[2 * m + 1]);
    else
      g = fabs(rr - d[m]);
    if (g <= thresh && (unsigned long long)m < best) best = (unsigned long long)m;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long u = __shfl_xor_sync(0xffffffffu, best, o);
    best = u < best ? u : best;
  }
  if ((threadIdx.x & 31) == 0 && best != ~0ull) atomicMin(first, best);
}

__global__ void __launch_bounds__(kLvThreads) rowptr_uniform_kernel(const int64_t* __restrict__ rp, int64_t n,
                                                                     int64_t per, unsigned* bad) {
  unsigned b = 0;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i <= n; i += int64_t(gridDim.x) * blockDim.x)
    b |= rp[i] != per * i ? 1u : 0u;
  b = __reduce_or_sync(0xffffffffu, b);
  if ((threadIdx.x & 31) == 0 && b) atomicOr(bad, 1u);
}

int blocks_for(int64_t n) {
  int64_t b = (n + kLvThreads - 1) / kLvThreads;
  return int(b < 1 ? 1 : (b > kLvBlocks ? kLvBlocks : b));
}

}  // namespace

// scratch: >= kLvBlocks * 9 + 16 doubles; counter zeroed, left zeroed.
// out (device, 7 doubles): best, runner, lo re, hi re, lo im, hi im, nan count.
cudaError_t launch_levels_scan(const double* d, int64_t n, int cx, double* scratch, unsigned* counter, double* out,
                               cudaStream_t st) {
  levels_scan_kernel<<<blocks_for(n), kLvThreads, 0, st>>>(d, n, cx, scratch, counter, out);
  return cudaGetLastError();
}

// first (device, 1 u64): set to ~0 by the caller; the first partner or ~0.
cudaError_t launch_levels_partner(const double* d, int64_t n, int cx, int64_t row, double thresh,
                                  unsigned long long* first, cudaStream_t st) {
  levels_partner_kernel<<<blocks_for(n), kLvThreads, 0, st>>>(d, n, cx, row, thresh, first);
  return cudaGetLastError();
}

// bad (device, 1 u32): zeroed by the caller; nonzero unless rp[i] == per * i for all i <= n.
cudaError_t launch_rowptr_uniform(const int64_t* rp, int64_t n, int64_t per, unsigned* bad, cudaStream_t st) {
  rowptr_uniform_kernel<<<blocks_for(n + 1), kLvThreads, 0, st>>>(rp, n, per, bad);
  return cudaGetLastError();
}

int levels_scratch_doubles() { return kLvBlocks * 9 + 16; }

}  // namespace dpt
