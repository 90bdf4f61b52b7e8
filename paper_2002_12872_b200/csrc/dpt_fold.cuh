// dpt_fold.cuh -- device-side pieces of K4: deterministic block reductions,
// the row read-off store, the decision (dpt_state.h) and the sample-first
// cycle test.
#pragma once
#include "dpt_device.cuh"

namespace dpt {

__device__ __forceinline__ double block_max(double v, double* sh) {
  v = warp_max(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < int(blockDim.x >> 5); ++i) r = fmax(r, sh[i]);
  return r;  // valid in thread 0
}

__device__ __forceinline__ double block_sum(double v, double* sh) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < int(blockDim.x >> 5); ++i) r += sh[i];
  return r;
}

// Row fold of one row: column-block partials are summed (d) / maxed (num, den)
// by `width` cooperating lanes in a fixed tree, so the result is deterministic.
// Complex problems keep d, eps interleaved (re, im) per row; dim = Im d.
// Returns the row residual (so the caller never reads it back from memory).
__device__ __forceinline__ double fold_row_store(const DevSolve& s, int64_t i, double d, double dim, double num,
                                                 double den, const double* dprev, double* dnext) {
  const double r = num / fmax(den, 1e-300);  // kTinyDen, dpt.cpp:18, :40
  s.res[i] = r;
  if (s.cplx) {  // eps_i = d_i + lambda P(i,i) in complex arithmetic
    const int64_t gi = s.row0 + i;
    const cd e = cadd(cmake(s.theta[2 * gi], s.theta[2 * gi + 1]),
                      cmul(cmake(s.lambda, s.lambda_im), cmake(dprev[2 * i], dprev[2 * i + 1])));
    s.eps[2 * i] = e.x;
    s.eps[2 * i + 1] = e.y;
    dnext[2 * i] = d;
    dnext[2 * i + 1] = dim;
    return r;
  }
  s.eps[i] = __dadd_rn(s.theta[s.row0 + i], __dmul_rn(s.lambda, dprev[i]));
  dnext[i] = d;
  return r;
}

static __device__ void decide_now(const DevSolve& s);

// Sample-first part of the cycle test, run by one block right after the
// decision: if the first entries already differ by >= tol from every window
// entry, within_tol is false for all of them and the cycle kernel has nothing
// to do (exact early-out, dpt.cpp:60-79).
static __device__ void cycle_sample_precheck(const DevSolve& s, const dpt_sm_state& dec) {
  dpt_sm_state* st = s.state;
  if (dec.done || !dec.cycle_pending) return;
  const int j = dec.j;
  int npast = j - 1;
  if (npast > s.opts.win - 1) npast = s.opts.win - 1;
  const int64_t n = s.ncol, ld = s.ld;
  const int64_t elems = s.rows * n;
  const int64_t ns = elems < int64_t(blockDim.x) ? elems : int64_t(blockDim.x);
  const double* cur = s.slots + size_t(j % s.nslots) * size_t(s.slot_elems);
  // All window entries at once, as one bitmask: bit p = "some sample of A_j
  // differs from window entry p by >= tol" (refutes within_tol for p; a NaN
  // difference refutes nothing, like fmax ignoring it).  One load round, one
  // warp OR-reduction, one shared OR.
  const int64_t e = threadIdx.x;
  const bool have = e < ns;
  const int64_t r = have ? e / n : 0, c = have ? e % n : 0;
  const size_t off = size_t(r * ld + c);
  const double cv = have ? cur[off] : 0.0;
  int slot = (j - 2) % s.nslots;  // slot of A_{j-2-p}, stepping back with wrap
  double pv[DPT_MAX_WINDOW];
#pragma unroll
  for (int p = 0; p < DPT_MAX_WINDOW; ++p) {
    const double* past = s.slots + size_t(slot) * size_t(s.slot_elems);
    pv[p] = (have && p < npast) ? __ldcg(past + off) : cv;
    slot = slot == 0 ? s.nslots - 1 : slot - 1;
  }
  unsigned bits = 0u;
#pragma unroll
  for (int p = 0; p < DPT_MAX_WINDOW; ++p) bits |= (fabs(cv - pv[p]) >= s.opts.tol) ? (1u << p) : 0u;
  bits = __reduce_or_sync(0xffffffffu, bits);
  __shared__ unsigned block_bits;
  if (threadIdx.x == 0) block_bits = 0u;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) atomicOr(&block_bits, bits);
  __syncthreads();
  const unsigned need = npast >= 32 ? 0xffffffffu : ((1u << npast) - 1u);
  if (threadIdx.x == 0 && (block_bits & need) == need) {
    st->cycle_pending = 0;  // refuted for every entry: the stats keep "not within"
#pragma unroll
    for (int p = 0; p < DPT_MAX_WINDOW; ++p) s.stats[DPT_STATS_CYCLE0 + p] = 1.0;
  }
}

// The decision on a register copy of the state and statistics: one batch of
// independent loads, the logic, one batch of stores -- instead of a chain of
// dependent global round trips (the fold's single-thread tail is latency-bound).
// `stats4` are this launch's folded maxima (already in registers); the cycle
// flags come from the previous cycle kernel.  Returns the decided state.
static __device__ dpt_sm_state decide_local(const DevSolve& s, const double* stats4) {
  dpt_sm_state* st = s.state;
  dpt_sm_state loc = *st;
  if (loc.done) return loc;
  const int j = loc.j + 1;
  if (s.fixed_mode) {  // iterate_fixed: no gates (dpt.cpp:381-387)
    loc.j = j;
    st->j = j;
    return loc;
  }
  double stl[DPT_NSTATS];
#pragma unroll
  for (int q = 0; q < 4; ++q) stl[q] = stats4 ? stats4[q] : s.stats[q];
#pragma unroll
  for (int q = 4; q < DPT_NSTATS; ++q) stl[q] = s.stats[q];
  const int sp = s.settled_table ? s.settled_table[j - 1] : 1;
  const int sc = s.settled_table ? s.settled_table[j] : 1;
  dpt_sm_decide(&loc, &s.opts, stl, j, sp, sc, s.trace);
  *st = loc;
  return loc;
}

static __device__ void decide_now(const DevSolve& s) { (void)decide_local(s, nullptr); }


}  // namespace dpt
