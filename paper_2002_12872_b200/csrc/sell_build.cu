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
// Bank-aware schedules: the lanes the shared-memory unit serves together (G =
// 16 lanes for 8-byte elements, 8 for 16-byte complex ones) must hit distinct
// banks (col mod G) at every step; a lane that cannot gets a bubble.
//   sched 2 (default, sell_free_kernel): lanes take their row's entries in any
//     order, bidding for banks each step (see the kernel).
//   sched 1 (sell_sched_kernel): lanes keep CSR order; in priority order (most
//     entries remaining first, then the lower lane) each lane issues its next
//     entry unless a higher-priority lane of its group took that bank -- one
//     __match_any_sync and a priority compare per step.
//   sched 0: dense packing, no schedule (DPT_SELL_SCHED selects; A/B only).
#include <algorithm>
#include <cuda_runtime.h>
#include <stdint.h>

#include "dpt_device.cuh"
#include "dpt_kernels.h"

namespace dpt {

namespace {

constexpr int kWin = 256;
constexpr int kSellPad = 4;
constexpr int kBankStage = 124;  // entries per row whose banks sell_free_kernel stages in shared memory

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

// Free-order bank schedule (sched = 2, the default).  A lane must own its row
// (its output column j), but nothing forces it to take the row's entries in
// CSR order: at each step it may issue ANY remaining entry.  Per step and
// group the lanes bid for banks: every lane without a bank proposes the free
// bank of which it holds the most remaining entries; each contested bank goes
// to the highest-priority bidder (most entries remaining, then the lower
// lane); losers re-bid among the banks still free until nobody can bid.  A
// lane then issues its next entry (CSR order within a bank) of the bank it won.
// Simulated on c3 (n = 8192, 0.5 %): the sum of slice widths drops from 18744
// steps (CSR-order greedy) to 14428, within 1 % of the per-group bound
// max(longest row, busiest bank).  The FMA chain of each P(i, j) runs in the
// schedule's order: deterministic (both passes make the same choices), the
// same for every staging variant R, within rounding of the reference's
// CSR-order sum.  Counts and cursors live in registers (unrolled bank loops).
template <bool WRITE>
__global__ void __launch_bounds__(256)
    sell_free_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ cl, const double* __restrict__ vl,
                     int cx, int64_t nslices, const int32_t* __restrict__ lane_col, int G,
                     const int32_t* __restrict__ perm, int64_t* width_or_off, int32_t* s_cols, double* s_vals) {
  const int lane = threadIdx.x & 31;
  const int64_t sl = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (sl >= nslices) return;  // warp-uniform
  const int32_t j = lane_col[sl * 32 + lane];
  const int64_t beg = j >= 0 ? rp[j] : 0;
  const int len = j >= 0 ? int(rp[j + 1] - beg) : 0;
  const int64_t off = WRITE ? width_or_off[sl] : 0;
  const uint32_t gm = uint32_t(G - 1);  // G is 16 (8-byte) or 8 (16-byte elements)
  // the image holds shared-memory positions: perm[k] when the columns were
  // relabelled for bank balance (sell_relabel_kernel), else k
  auto colpos = [&](int64_t q) -> int32_t { return perm ? perm[cl[q]] : cl[q]; };
  // The bank of every entry of the slice's rows, staged in shared memory by the
  // whole warp (row r's entries loaded by consecutive lanes: coalesced, and the
  // 32 rows' loads are independent).  The schedule below walks a row's entries
  // bank by bank; reading each bank through cl -> perm from global memory made
  // every step a chain of dependent L2 round trips (c3: 0.58 ms per pass).
  // Rows longer than the stage keep the global reads.  Same schedule either way.
  __shared__ uint8_t sbank[8][32][kBankStage + 4];  // [warp][row][entry], padded: conflict-free per-lane reads
  const int wib = (threadIdx.x >> 5) & 7;
  const bool use_stage = __all_sync(0xffffffffu, len <= kBankStage);
  if (use_stage) {
#pragma unroll 8
    for (int r = 0; r < 32; ++r) {  // unrolled: the rows' load chains (cl -> perm) overlap
      const int64_t beg_r = __shfl_sync(0xffffffffu, beg, r);
      const int len_r = __shfl_sync(0xffffffffu, len, r);
      for (int q = lane; q < len_r; q += 32) sbank[wib][r][q] = uint8_t(uint32_t(colpos(beg_r + q)) & gm);
    }
    __syncwarp();
  }
  auto bankof = [&](int q) -> int {
    return use_stage ? int(sbank[wib][lane][q]) : int(uint32_t(colpos(beg + q)) & gm);
  };
  int cnt[16], pos[16];
#pragma unroll
  for (int b = 0; b < 16; ++b) {
    cnt[b] = 0;
    pos[b] = len;
  }
  for (int q = 0; q < len; ++q) {
    const int bk = bankof(q);
#pragma unroll
    for (int b = 0; b < 16; ++b)
      if (b == bk) {
        if (cnt[b] == 0) pos[b] = q;
        ++cnt[b];
      }
  }
  int rem = len;
  int64_t step = 0;
  while (__any_sync(0xffffffffu, rem > 0)) {
    unsigned taken = 0;  // banks won in this step (uniform within a group)
    int mybank = -1;
    while (true) {
      int choice = -1;
      if (rem > 0 && mybank < 0) {
        int best = 0;
#pragma unroll
        for (int b = 0; b < 16; ++b)
          if (!((taken >> b) & 1u) && cnt[b] > best) {
            best = cnt[b];
            choice = b;
          }
      }
      if (!__any_sync(0xffffffffu, choice >= 0)) break;
      // the top bidder of each contested bank: every lane compares its bid with
      // the G - 1 others of its group (xor-shuffles stay inside the aligned
      // group).  Priorities are distinct (the lane is part of them), so exactly
      // one bidder per bank wins.  (__match_any_sync + a masked
      // __reduce_max_sync did the same at ~2000 cycles per round: both
      // serialise over the distinct keys / masks of the warp.)
      const unsigned remc = rem < (1 << 22) ? unsigned(rem) : (1u << 22) - 1u;  // 27-bit priority field
      const unsigned prio = choice >= 0 ? remc * 32u + unsigned(31 - lane) : 0u;
      const unsigned bid = choice >= 0 ? (unsigned(choice) << 27) | prio : 0xffffffffu;
      bool top = choice >= 0;
      for (int o = 1; o < G; ++o) {
        const unsigned other = __shfl_xor_sync(0xffffffffu, bid, o);
        if (other != 0xffffffffu && (other >> 27) == unsigned(choice) && (other & 0x7ffffffu) > prio) top = false;
      }
      unsigned won = 0;
      if (top) {
        mybank = choice;
        won = 1u << choice;
      }
      for (int o = 1; o < G; o <<= 1) won |= __shfl_xor_sync(0xffffffffu, won, o);  // OR over the group
      taken |= won;
    }
    if (mybank >= 0) {
      int q = 0, left = 0;
#pragma unroll
      for (int b = 0; b < 16; ++b)
        if (b == mybank) {
          q = pos[b];
          left = --cnt[b];
        }
      if (WRITE) {
        const int64_t dst = off + step * 32 + lane;
        s_cols[dst] = colpos(beg + q);
        for (int c = 0; c < cx; ++c) s_vals[cx * dst + c] = vl[cx * (beg + q) + c];
      }
      --rem;
      if (left > 0) {
        int q2 = q + 1;
        while (bankof(q2) != mybank) ++q2;
#pragma unroll
        for (int b = 0; b < 16; ++b)
          if (b == mybank) pos[b] = q2;
      }
    }
    ++step;
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


// ---------------------------------------------------------------- relabel ----
// Column relabelling for bank balance (real K2, 16 banks of 8-byte words).
// The bank of column k in K2's staged rows is pos(k) mod 16, where pos is the
// column's shared-memory position -- any permutation works.  With pos(k) = k
// the busiest bank of a 16-row group sets its schedule length (c3: 1.25x the
// longest row); choosing pos so that every group's 16 bank loads are level
// brings that to ~1.05x.  Local search on the group x bank load matrix L
// (groups = 16-lane halves of the SELL slices; column k adds one to L[g][bank]
// for every row j of group g that holds k), minimising sum L^2: batches of 64
// columns, 16 threads per column (one per target bank) evaluate the move
// deltas against the loads before the batch; improving moves are accepted in
// column order up to each bank's capacity (so positions fit the staged row),
// and L is updated with integer atomics -- the result is deterministic.
// Simulated on c3: schedule bound 1.25x -> 1.049x after 3 passes.

// column -> list of groups (CSC of the group map): counts, then fill
__global__ void relabel_count_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ cl, int64_t n,
                                     int32_t* ccount) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t j = w; j < n; j += nw)
    for (int64_t q = rp[j] + lane; q < rp[j + 1]; q += 32) atomicAdd(ccount + cl[q], 1);
}

__global__ void __launch_bounds__(1024) relabel_scan_kernel(const int32_t* cnt, int64_t n, int32_t* start) {
  __shared__ int32_t buf[1024];
  __shared__ int32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t b0 = 0; b0 < n; b0 += 1024) {
    const int64_t i = b0 + threadIdx.x;
    const int32_t v = i < n ? cnt[i] : 0;
    buf[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
      const int32_t add = threadIdx.x >= o ? buf[threadIdx.x - o] : 0;
      __syncthreads();
      buf[threadIdx.x] += add;
      __syncthreads();
    }
    if (i < n) start[i] = carry + buf[threadIdx.x] - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry += buf[1023];
    __syncthreads();
  }
  if (threadIdx.x == 0) start[n] = carry;
}

__global__ void relabel_fill_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ cl, int64_t n,
                                    const int64_t* __restrict__ slot_of, const int32_t* __restrict__ start,
                                    int32_t* cfill, int32_t* cgroups) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t j = w; j < n; j += nw) {
    const int32_t g = int32_t(slot_of[j] >> 4);  // 16-lane group of row j's SELL lane
    for (int64_t q = rp[j] + lane; q < rp[j + 1]; q += 32) {
      const int32_t k = cl[q];
      cgroups[start[k] + atomicAdd(cfill + k, 1)] = g;  // order within a column is irrelevant (integer sums)
    }
  }
}

constexpr int kRelabelBatch = 64;
constexpr int kRelabelStage = 4096;  // group-list entries of a batch staged in shared memory (2 x 16 KB)
// One block.  L lives in shared memory: ng x 16 int32 (the caller checks it fits).
// The group lists of a batch's columns are one contiguous range of cgroups,
// staged in shared memory (double-buffered, see the batch loop); a batch whose
// lists exceed the stage reads them from global memory.  Same arithmetic in
// the same order as the unstaged kernel.
__global__ void __launch_bounds__(1024) relabel_kernel(const int32_t* __restrict__ start,
                                                       const int32_t* __restrict__ cgroups, int64_t n, int ng,
                                                       int cap, int passes, int32_t* bank, int32_t* pos,
                                                       int32_t* inv, int64_t npad_alloc, int32_t* npad_out) {
  extern __shared__ int32_t L[];  // [ng][16]
  __shared__ int32_t size[16];
  __shared__ int32_t prop[kRelabelBatch], acc[kRelabelBatch], oldb[kRelabelBatch];
  __shared__ int32_t stage[2][kRelabelStage];
  __shared__ int32_t sstart[2][kRelabelBatch + 1], sbk[2][kRelabelBatch];
  const int tid = threadIdx.x, c = tid >> 4, t = tid & 15;
  for (int64_t e = tid; e < int64_t(ng) * 16; e += blockDim.x) L[e] = 0;
  if (tid < 16) size[tid] = 0;
  for (int64_t k = tid; k < n; k += blockDim.x) bank[k] = int32_t(k & 15);
  __syncthreads();
  for (int64_t k = tid; k < n; k += blockDim.x) {
    atomicAdd(&size[k & 15], 1);
    for (int32_t q = start[k]; q < start[k + 1]; ++q) atomicAdd(&L[cgroups[q] * 16 + int(k & 15)], 1);
  }
  __syncthreads();
  // Batches run strictly one after another (each sees the loads the previous one
  // left), so a batch's global reads -- its columns' list bounds, banks and
  // group lists -- are a chain of L2 round trips on the critical path.  They
  // are software-pipelined: while batch i is evaluated from shared memory,
  // every thread holds batch i + 1's values in registers (the next lists start
  // where this batch's end, so their address needs no lookup) and parks them in
  // the other buffer before the closing barrier.
  const int64_t nbp = (n + kRelabelBatch - 1) / kRelabelBatch;  // batches per pass
  const int64_t nbt = nbp * passes;
  const bool pipelined = nbp > 1;  // one batch per pass: the next batch re-reads what this one writes
  const int32_t total = start[n];
  if (tid <= kRelabelBatch) sstart[0][tid] = start[tid < n ? tid : n];
  if (tid < kRelabelBatch) sbk[0][tid] = tid < n ? bank[tid] : 0;
  for (int32_t q = tid; q < kRelabelStage && q < total; q += blockDim.x) stage[0][q] = cgroups[q];
  __syncthreads();
  for (int64_t it = 0; it < nbt; ++it) {
    const int cur = int(it & 1);
    const int64_t b0 = (it % nbp) * kRelabelBatch;
    const int64_t k = b0 + c;
    const bool ok = k < n;
    const int32_t q0 = ok ? sstart[cur][c] : 0, q1 = ok ? sstart[cur][c + 1] : 0;
    const int b = ok ? sbk[cur][c] : 0;
    const int64_t kcnt = n - b0 < kRelabelBatch ? n - b0 : kRelabelBatch;
    const int32_t s0 = sstart[cur][0], s1 = sstart[cur][kcnt];  // the batch's lists: cgroups[s0, s1)
    // ---- prefetch of the next batch (registers) ----
    const bool more = it + 1 < nbt;
    const int64_t nb0 = more ? ((it + 1) % nbp) * kRelabelBatch : 0;
    const int32_t ns0 = nb0 == 0 ? 0 : s1;
    int32_t pre[kRelabelStage / 1024];
    int32_t pstart = 0, pbank = 0;
    if (more && pipelined) {
#pragma unroll
      for (int u = 0; u < kRelabelStage / 1024; ++u) {
        const int32_t q = ns0 + tid + u * 1024;
        pre[u] = q < total ? cgroups[q] : 0;
      }
      if (tid <= kRelabelBatch) pstart = start[nb0 + tid < n ? nb0 + tid : n];
      if (tid < kRelabelBatch) pbank = nb0 + tid < n ? bank[nb0 + tid] : 0;
    }
    // ---- evaluate the batch ----
    const bool staged = s1 - s0 <= kRelabelStage;  // block-uniform
    const int32_t* __restrict__ cg = staged ? stage[cur] : cgroups;  // entry q of the lists at cg[q - cofs]
    const int32_t cofs = staged ? s0 : 0;
    int32_t sum = 0;
    for (int32_t q = q0; q < q1; ++q) sum += L[cg[q - cofs] * 16 + t];
    const int32_t sb = __shfl_sync(0xffffffffu, sum, b, 16);
    // move delta of sum L^2 (exact up to repeated groups): 2 (S_t - S_b) + 2 m
    int32_t d = (t == b || !ok || q1 == q0) ? 0 : 2 * (sum - sb) + 2 * (q1 - q0);
    int bt = t;
    for (int o = 8; o > 0; o >>= 1) {  // argmin over the 16 targets, ties -> lower bank
      const int32_t d2 = __shfl_xor_sync(0xffffffffu, d, o, 16);
      const int bt2 = __shfl_xor_sync(0xffffffffu, bt, o, 16);
      if (d2 < d || (d2 == d && bt2 < bt)) {
        d = d2;
        bt = bt2;
      }
    }
    if (t == 0) {
      prop[c] = d < 0 ? bt : -1;
      oldb[c] = b;
    }
    __syncthreads();
    {  // capacity, in column order, against the sizes before the batch: the 16
       // threads of a column count the earlier columns proposing the same bank
      const int a0 = prop[c];
      int ahead = 0;
      for (int c2 = t; c2 < c; c2 += 16) ahead += (a0 >= 0 && prop[c2] == a0) ? 1 : 0;
      for (int o = 8; o > 0; o >>= 1) ahead += __shfl_xor_sync(0xffffffffu, ahead, o, 16);
      if (t == 0) {
        int a = a0;
        if (a >= 0 && size[a] + ahead >= cap) a = -2;
        acc[c] = a;
      }
    }
    __syncthreads();
    const int nb = acc[c];
    if (nb >= 0) {
      for (int32_t q = q0 + t; q < q1; q += 16) {
        const int32_t g = cg[q - cofs];
        atomicSub(&L[g * 16 + oldb[c]], 1);
        atomicAdd(&L[g * 16 + nb], 1);
      }
      if (t == 0) {
        atomicSub(&size[oldb[c]], 1);
        atomicAdd(&size[nb], 1);
        bank[k] = nb;
      }
    }
    if (more && pipelined) {  // park the prefetched batch in the other buffer
#pragma unroll
      for (int u = 0; u < kRelabelStage / 1024; ++u) stage[cur ^ 1][tid + u * 1024] = pre[u];
      if (tid <= kRelabelBatch) sstart[cur ^ 1][tid] = pstart;
      if (tid < kRelabelBatch) sbk[cur ^ 1][tid] = pbank;
    }
    __syncthreads();
    if (more && !pipelined) {  // n <= 64: the same columns again, reloaded after this batch's writes
      if (tid <= kRelabelBatch) sstart[cur ^ 1][tid] = start[tid < n ? tid : n];
      if (tid < kRelabelBatch) sbk[cur ^ 1][tid] = tid < n ? bank[tid] : 0;
      for (int32_t q = tid; q < kRelabelStage && q < total; q += blockDim.x) stage[cur ^ 1][q] = cgroups[q];
      __syncthreads();
    }
  }
  // positions: pos(k) = bank + 16 * (rank of k among its bank's columns), warp b per bank
  const int warp = tid >> 5, lane = tid & 31;
  for (int64_t p = tid; p < npad_alloc; p += blockDim.x) inv[p] = -1;
  __syncthreads();
  if (warp < 16) {
    int32_t base = 0;
    for (int64_t k0 = 0; k0 < n; k0 += 32) {
      const int64_t k = k0 + lane;
      const bool mine = k < n && bank[k] == warp;
      const unsigned m = __ballot_sync(0xffffffffu, mine);
      if (mine) {
        const int32_t p = warp + 16 * (base + __popc(m & ((1u << lane) - 1u)));
        pos[k] = p;
        inv[p] = int32_t(k);
      }
      base += __popc(m);
    }
  }
  __syncthreads();
  if (tid == 0) {
    int32_t mx = 0;
    for (int b = 0; b < 16; ++b) mx = size[b] > mx ? size[b] : mx;
    *npad_out = 16 * mx;
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
                               int sched, const int32_t* perm, int64_t* widths, cudaStream_t st) {
  const int64_t blocks = (nslices * 32 + 255) / 256;
  if (blocks > 0 && sched == 2)
    sell_free_kernel<false><<<unsigned(blocks), 256, 0, st>>>(rp, cl, nullptr, 1, nslices, lane_col, G, perm,
                                                                         widths, nullptr, nullptr);
  else if (blocks > 0)
    sell_sched_kernel<false><<<unsigned(blocks), 256, 0, st>>>(rp, cl, nullptr, 1, nslices, lane_col, G, sched,
                                                                widths, nullptr, nullptr);
  return cudaGetLastError();
}

cudaError_t launch_sell_scan(int64_t* widths, int64_t nslices, int64_t* total, cudaStream_t st) {
  sell_scan_kernel<<<1, 1024, 0, st>>>(widths, nslices, total);
  return cudaGetLastError();
}

cudaError_t launch_sell_fill(const int64_t* rp, const int32_t* cl, const double* vl, int cx, int64_t nslices,
                             const int32_t* lane_col, int G, int sched, const int32_t* perm, const int64_t* off,
                             int32_t* s_cols, double* s_vals, cudaStream_t st) {
  const int64_t blocks = (nslices * 32 + 255) / 256;
  if (blocks > 0 && sched == 2)
    sell_free_kernel<true><<<unsigned(blocks), 256, 0, st>>>(rp, cl, vl, cx, nslices, lane_col, G, perm,
                                                                        const_cast<int64_t*>(off), s_cols, s_vals);
  else if (blocks > 0)
    sell_sched_kernel<true><<<unsigned(blocks), 256, 0, st>>>(rp, cl, vl, cx, nslices, lane_col, G, sched,
                                                               const_cast<int64_t*>(off), s_cols, s_vals);
  return cudaGetLastError();
}

namespace {
// Packed copy for K2's shared-memory kernel: 16-bit positions, four steps of a
// lane adjacent (one 8-byte load per lane per trip instead of four 4-byte
// ones), and the per-lane epilogue constants (the position and level of the
// lane's own column j) in slice order, so the epilogue reads them coalesced
// instead of gathering perm[j] / theta[j].  One warp per slice.
__global__ void __launch_bounds__(256)
    sell_pack_kernel(const int32_t* __restrict__ s_cols, const int64_t* __restrict__ off, int64_t nslices,
                     const int32_t* __restrict__ lane_col, const int32_t* __restrict__ perm,
                     const double* __restrict__ theta, uint16_t* cols16, int32_t* lane_pos, double* lane_theta) {
  const int lane = threadIdx.x & 31;
  const int64_t sl = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (sl >= nslices) return;
  const int32_t j = lane_col[sl * 32 + lane];
  lane_pos[sl * 32 + lane] = j < 0 ? -1 : (perm ? perm[j] : j);
  lane_theta[sl * 32 + lane] = j < 0 ? 0.0 : theta[j];
  const int64_t o = off[sl];
  const int64_t width = (off[sl + 1] - o) >> 5;  // multiple of kSellPad = 4
  uint2* dst = reinterpret_cast<uint2*>(cols16) + (o >> 2) + lane;
  for (int64_t q0 = 0; q0 < width; q0 += 4) {
    uint32_t c[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) c[u] = uint32_t(s_cols[o + (q0 + u) * 32 + lane]) & 0xffffu;  // -1 -> 0xffff
    dst[(q0 >> 2) * 32] = make_uint2(c[0] | (c[1] << 16), c[2] | (c[3] << 16));
  }
}

}  // namespace

// *flag = 1 if some row's columns are not strictly increasing (a repeated or
// out-of-order (row, column) pair): K2 handles both, the launch-1 shortcut
// (launch_csr_init) assumes one entry per pair.
__global__ void csr_order_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ cl, int64_t n, int32_t* flag) {
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += int64_t(gridDim.x) * blockDim.x)
    for (int64_t q = rp[j] + 1; q < rp[j + 1]; ++q)
      if (cl[q] <= cl[q - 1]) *flag = 1;
}

cudaError_t launch_csr_order_check(const int64_t* rp, const int32_t* cl, int64_t n, int32_t* flag, cudaStream_t st) {
  const int64_t b = (n + 255) / 256;
  if (b > 0) csr_order_kernel<<<unsigned(b > 1184 ? 1184 : b), 256, 0, st>>>(rp, cl, n, flag);
  return cudaGetLastError();
}

cudaError_t launch_sell_pack(const int32_t* s_cols, const int64_t* off, int64_t nslices, const int32_t* lane_col,
                             const int32_t* perm, const double* theta, uint16_t* cols16, int32_t* lane_pos,
                             double* lane_theta, cudaStream_t st) {
  const int64_t blocks = (nslices * 32 + 255) / 256;
  if (blocks > 0)
    sell_pack_kernel<<<unsigned(blocks), 256, 0, st>>>(s_cols, off, nslices, lane_col, perm, theta, cols16, lane_pos,
                                                       lane_theta);
  return cudaGetLastError();
}

size_t relabel_smem_bytes(int64_t nslices) { return size_t(2 * nslices) * 16 * 4 + 2 * kRelabelStage * 4 + 2048; }  // dynamic L + static stages

cudaError_t launch_relabel(const int64_t* rp, const int32_t* cl, int64_t n, int64_t nnz, int64_t nslices,
                           const int64_t* slot_of, int cap, int passes, int32_t* scratch, int32_t* bank, int32_t* pos,
                           int32_t* inv, int64_t npad_alloc, int32_t* npad_out, cudaStream_t st) {
  // scratch: ccount[n] | start[n + 1] | cfill[n] | cgroups[nnz]
  int32_t* ccount = scratch;
  int32_t* start = ccount + n;
  int32_t* cfill = start + n + 1;
  int32_t* cgroups = cfill + n;
  cudaMemsetAsync(ccount, 0, size_t(n) * 4, st);
  cudaMemsetAsync(cfill, 0, size_t(n) * 4, st);
  const unsigned blocks = unsigned(std::min<int64_t>((n + 7) / 8, 1184));
  relabel_count_kernel<<<blocks, 256, 0, st>>>(rp, cl, n, ccount);
  relabel_scan_kernel<<<1, 1024, 0, st>>>(ccount, n, start);
  relabel_fill_kernel<<<blocks, 256, 0, st>>>(rp, cl, n, slot_of, start, cfill, cgroups);
  const size_t smem = size_t(2 * nslices) * 16 * 4;  // L only: the stage is static
  static DeviceAttrOnce attr;
  attr([] { cudaFuncSetAttribute(relabel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 188 * 1024); });  // + ~35 KB static
  relabel_kernel<<<1, 1024, smem, st>>>(start, cgroups, n, int(2 * nslices), cap, passes, bank, pos, inv, npad_alloc,
                                        npad_out);
  (void)nnz;
  return cudaGetLastError();
}

}  // namespace dpt
