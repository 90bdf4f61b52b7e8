// sell_build.cu -- K2's SELL-32 image of Delta, built on the device from the
// CSR already in HBM (no host round trip of cols / vals).
//
// Layout (consumed by csr_step_kernel / csr_step_cplx_kernel):
//   rows of Delta sorted by length, descending and stable, inside windows of
//   256 rows; 32 consecutive sorted rows form a slice, lane L of slice sl owns
//   row lane_col[32 sl + L]; entry (step q, lane L) of slice sl lives at
//   slice_off[sl] + 32 q + L.  Column -1 / value 0 marks a bubble or padding.
//   Widths are padded to a multiple of kSellPad steps (K2 reads 4 per trip).
//
// Bank-aware schedule: the lanes the shared-memory unit serves together (G = 16
// lanes for 8-byte elements, 8 for 16-byte complex ones) must hit distinct
// banks (col mod G) at every step.  Greedily, in priority order (most entries
// remaining first, then the lower lane), each lane issues its next entry unless
// a higher-priority lane of its group already took that bank this step.  Since
// each lane wants exactly one bank per step, that greedy equals "each bank goes
// to its highest-priority requester" -- a warp computes it with one
// __match_any_sync and a priority compare, one slice per warp.  Every lane
// keeps its row's CSR order, so the FMA chain of each P(i, j) is unchanged by
// the schedule (results are identical for any schedule).
#include <cuda_runtime.h>
#include <stdint.h>

#include "dpt_device.cuh"
#include "dpt_kernels.h"

namespace dpt {

namespace {

constexpr int kWin = 256;
constexpr int kSellPad = 4;

// stable descending rank of each row's length inside its 256-row window
__global__ void __launch_bounds__(kWin) sell_perm_kernel(const int64_t* __restrict__ rp, int64_t n,
                                                         int32_t* lane_col, int32_t* lane_len, int64_t* pos_of) {
  __shared__ int64_t len[kWin];
  const int64_t w0 = int64_t(blockIdx.x) * kWin;
  const int cnt = int(n - w0 < kWin ? n - w0 : kWin);
  const int t = threadIdx.x;
  if (t < cnt) len[t] = rp[w0 + t + 1] - rp[w0 + t];
  __syncthreads();
  if (t < cnt) {
    const int64_t me = len[t];
    int rank = 0;
    for (int q = 0; q < cnt; ++q) rank += (len[q] > me || (len[q] == me && q < t)) ? 1 : 0;
    const int64_t slot = w0 + rank;
    lane_col[slot] = int32_t(w0 + t);
    lane_len[slot] = int32_t(me);
    pos_of[w0 + t] = slot;
  }
}

// One warp per slice.  WRITE = false: count the schedule's steps (padded);
// WRITE = true: emit the entries at slice_off.
template <bool WRITE>
__global__ void sell_sched_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ cl,
                                  const double* __restrict__ vl, int cx, int64_t nslices,
                                  const int32_t* __restrict__ lane_col, int G, int sched, int64_t* width_or_off,
                                  int32_t* s_cols, double* s_vals) {
  const int lane = threadIdx.x & 31;
  const int64_t sl = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (sl >= nslices) return;  // warp-uniform
  const int32_t j = lane_col[sl * 32 + lane];
  const int64_t beg = j >= 0 ? rp[j] : 0;
  const int64_t len = j >= 0 ? rp[j + 1] - beg : 0;
  const int64_t off = WRITE ? width_or_off[sl] : 0;
  int64_t head = 0, step = 0;
  if (!sched) {  // dense packing: entry q at step q
    int64_t w = len;
    for (int o = 16; o > 0; o >>= 1) {
      const int64_t u = __shfl_xor_sync(0xffffffffu, w, o);
      w = u > w ? u : w;
    }
    if (WRITE) {
      for (int64_t q = 0; q < len; ++q) {
        const int64_t dst = off + q * 32 + lane;
        s_cols[dst] = cl[beg + q];
        for (int c = 0; c < cx; ++c) s_vals[cx * dst + c] = vl[cx * (beg + q) + c];
      }
    }
    step = w;
  } else {
    while (__any_sync(0xffffffffu, head < len)) {
      const bool active = head < len;
      const int32_t col = active ? cl[beg + head] : 0;
      const int bank = int(uint32_t(col) % uint32_t(G));
      // active lanes of one group wanting one bank share a key; others are unique
      const int key = active ? (lane / G) * 64 + bank : 4096 + lane;
      const unsigned peers = __match_any_sync(0xffffffffu, key);
      const long long prio = active ? (long long)(len - head) * 32 + (31 - lane) : -1;
      bool win = active;
      for (int q = 0; q < 32; ++q) {
        const long long pq = __shfl_sync(0xffffffffu, prio, q);
        if (((peers >> q) & 1u) && pq > prio) win = false;
      }
      if (win) {
        if (WRITE) {
          const int64_t dst = off + step * 32 + lane;
          s_cols[dst] = col;
          for (int c = 0; c < cx; ++c) s_vals[cx * dst + c] = vl[cx * (beg + head) + c];
        }
        ++head;
      }
      ++step;
    }
  }
  if (!WRITE && lane == 0) width_or_off[sl] = (step + kSellPad - 1) / kSellPad * kSellPad;
}

// exclusive scan of widths (in steps) into entry offsets (x 32), one block
__global__ void __launch_bounds__(1024) sell_scan_kernel(int64_t* w, int64_t ns, int64_t* total) {
  __shared__ int64_t carry;
  __shared__ int64_t buf[1024];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t b0 = 0; b0 < ns; b0 += 1024) {
    const int64_t i = b0 + threadIdx.x;
    const int64_t v = i < ns ? w[i] * 32 : 0;
    buf[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {  // Hillis-Steele inclusive scan
      const int64_t add = threadIdx.x >= o ? buf[threadIdx.x - o] : 0;
      __syncthreads();
      buf[threadIdx.x] += add;
      __syncthreads();
    }
    if (i < ns) w[i] = carry + buf[threadIdx.x] - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry += buf[1023];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    w[ns] = carry;
    *total = carry;
  }
}

}  // namespace

cudaError_t launch_sell_perm(const int64_t* rp, int64_t n, int32_t* lane_col, int32_t* lane_len, int64_t* pos_of,
                             cudaStream_t st) {
  const int64_t wins = (n + kWin - 1) / kWin;
  if (wins > 0) sell_perm_kernel<<<unsigned(wins), kWin, 0, st>>>(rp, n, lane_col, lane_len, pos_of);
  return cudaGetLastError();
}

cudaError_t launch_sell_widths(const int64_t* rp, const int32_t* cl, int64_t nslices, const int32_t* lane_col, int G,
                               int sched, int64_t* widths, cudaStream_t st) {
  const int64_t blocks = (nslices * 32 + 255) / 256;
  if (blocks > 0)
    sell_sched_kernel<false><<<unsigned(blocks), 256, 0, st>>>(rp, cl, nullptr, 1, nslices, lane_col, G, sched,
                                                                widths, nullptr, nullptr);
  return cudaGetLastError();
}

cudaError_t launch_sell_scan(int64_t* widths, int64_t nslices, int64_t* total, cudaStream_t st) {
  sell_scan_kernel<<<1, 1024, 0, st>>>(widths, nslices, total);
  return cudaGetLastError();
}

cudaError_t launch_sell_fill(const int64_t* rp, const int32_t* cl, const double* vl, int cx, int64_t nslices,
                             const int32_t* lane_col, int G, int sched, const int64_t* off, int32_t* s_cols,
                             double* s_vals, cudaStream_t st) {
  const int64_t blocks = (nslices * 32 + 255) / 256;
  if (blocks > 0)
    sell_sched_kernel<true><<<unsigned(blocks), 256, 0, st>>>(rp, cl, vl, cx, nslices, lane_col, G, sched,
                                                               const_cast<int64_t*>(off), s_cols, s_vals);
  return cudaGetLastError();
}

}  // namespace dpt
