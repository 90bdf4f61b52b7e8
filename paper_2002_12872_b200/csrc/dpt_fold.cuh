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
__device__ __forceinline__ void fold_row_store(const DevSolve& s, int64_t i, double d, double dim, double num,
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
    return;
  }
  s.eps[i] = __dadd_rn(s.theta[s.row0 + i], __dmul_rn(s.lambda, dprev[i]));
  dnext[i] = d;
}

static __device__ void decide_now(const DevSolve& s);

// Sample-first part of the cycle test, run by one block right after the
// decision: if the first entries already differ by >= tol from every window
// entry, within_tol is false for all of them and the cycle kernel has nothing
// to do (exact early-out, dpt.cpp:60-79).
static __device__ void cycle_sample_precheck(const DevSolve& s, double* sh) {
  dpt_sm_state* st = s.state;
  if (st->done || !st->cycle_pending) return;
  const int j = st->j;
  int npast = j - 1;
  if (npast > s.opts.win - 1) npast = s.opts.win - 1;
  const int64_t n = s.ncol, ld = s.ld;
  const int64_t elems = s.rows * n;
  const int64_t ns = elems < int64_t(blockDim.x) ? elems : int64_t(blockDim.x);
  const double* cur = s.slots + size_t(j % s.nslots) * size_t(s.slot_elems);
  // all window entries at once: one load round, one reduction round
  double m[DPT_MAX_WINDOW];
  const int64_t e = threadIdx.x;
  const bool have = e < ns;
  const int64_t r = have ? e / n : 0, c = have ? e % n : 0;
  const double cv = have ? cur[r * ld + c] : 0.0;
  // branch-free loads (clamped slot index) so all window entries are in flight
  // at once: a guarded load per entry serialised ~1 us of latency per entry
  double pv[DPT_MAX_WINDOW];
#pragma unroll
  for (int p = 0; p < DPT_MAX_WINDOW; ++p) {
    const int pp = p < npast ? p : 0;
    const double* past = s.slots + size_t((j - 2 - pp) % s.nslots) * size_t(s.slot_elems);
    pv[p] = (have && npast > 0) ? __ldcg(past + r * ld + c) : 0.0;
  }
#pragma unroll
  for (int p = 0; p < DPT_MAX_WINDOW; ++p) m[p] = (p < npast && have) ? fabs(cv - pv[p]) : 0.0;
  __shared__ double wm[32][DPT_MAX_WINDOW];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
  for (int p = 0; p < DPT_MAX_WINDOW; ++p) {
    const double v = warp_max(m[p]);
    if (l == 0) wm[w][p] = v;
  }
  __syncthreads();
  int any = 0;
  if (threadIdx.x == 0) {
    for (int p = 0; p < npast; ++p) {
      double v = 0.0;
      for (int ww = 0; ww < int(blockDim.x >> 5); ++ww) v = fmax(v, wm[ww][p]);
      if (v < s.opts.tol) any = 1;
    }
  }
  if (threadIdx.x == 0 && !any) {
    st->cycle_pending = 0;  // refuted for every entry: the stats keep "not within"
    for (int p = 0; p < DPT_MAX_WINDOW; ++p) s.stats[DPT_STATS_CYCLE0 + p] = 1.0;
  }
}

static __device__ void decide_now(const DevSolve& s) {
  dpt_sm_state* st = s.state;
  if (st->done) return;
  const int j = st->j + 1;
  if (s.fixed_mode) {  // iterate_fixed: no gates (dpt.cpp:381-387)
    st->j = j;
    return;
  }
  const int sp = s.settled_table ? s.settled_table[j - 1] : 1;
  const int sc = s.settled_table ? s.settled_table[j] : 1;
  dpt_sm_decide(st, &s.opts, s.stats, j, sp, sc, s.trace);
}


}  // namespace dpt
