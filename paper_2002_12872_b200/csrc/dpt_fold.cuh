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
static __device__ void cycle_sample_precheck(const DevSolve& s, const dpt_sm_state& dec, unsigned* block_bits) {
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
  if (threadIdx.x == 0) *block_bits = 0u;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) atomicOr(block_bits, bits);
  __syncthreads();
  const unsigned need = npast >= 32 ? 0xffffffffu : ((1u << npast) - 1u);
  if (threadIdx.x == 0 && (*block_bits & need) == need) {
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

// The one-row fold (the row map: rows = 1) run by the LAST block of the step
// kernel itself (fold_in_step): the same reductions as fold_kernel's
// block-per-row path and its elected tail -- the row partials of the ntn step
// blocks, the launch maxima, stats[0..3], and on a single rank the decision,
// the loop condition and the cycle pre-check -- without a fold launch.  The
// residual maxima are order-free and rowpart[0] (the row map's d) is 0, so the
// result equals fold_kernel's bit for bit.  `scratch` is shared memory the
// caller no longer uses (>= 4 * warps + 8 doubles + a dpt_sm_state).  Not
// inlined: the step kernel's main loop keeps its registers.
static __device__ __noinline__ void fold_row_map_in_block(const DevSolve& s, int ntn, double* scratch) {
  const int j = launch_index(s);
  const int nw = int(blockDim.x >> 5), lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* dprev = s.dvec[(j - 1) & 1];
  double* dnext = s.dvec[j & 1];
  double d = 0.0, num = 0.0, den = 0.0, a0 = 0.0, a1 = 0.0, a2 = 0.0;
  for (int tn = threadIdx.x; tn < ntn; tn += blockDim.x) {
    d += __ldcg(s.rowpart + rp_index(0, 0, tn, 1, ntn));
    num = fmax(num, __ldcg(s.rowpart + rp_index(1, 0, tn, 1, ntn)));
    den = fmax(den, __ldcg(s.rowpart + rp_index(2, 0, tn, 1, ntn)));
    const double2 t01 = __ldcg(reinterpret_cast<const double2*>(s.tilepart + size_t(tn) * 4));
    a0 = fmax(a0, t01.x);
    a1 = fmax(a1, t01.y);
    a2 += __ldcg(s.tilepart + size_t(tn) * 4 + 2);
  }
  d = warp_sum(d);
  num = warp_max(num);
  den = warp_max(den);
  a0 = warp_max(a0);
  a1 = warp_max(a1);
  a2 = warp_sum(a2);
  double* red = scratch;  // [nw][6]
  if (lane == 0) {
    red[warp * 6 + 0] = d;
    red[warp * 6 + 1] = num;
    red[warp * 6 + 2] = den;
    red[warp * 6 + 3] = a0;
    red[warp * 6 + 4] = a1;
    red[warp * 6 + 5] = a2;
  }
  __syncthreads();
  dpt_sm_state* dec = reinterpret_cast<dpt_sm_state*>(scratch + 6 * nw + 2);
  if (threadIdx.x == 0) {
    double dd = 0.0, nn = 0.0, ee = 0.0, r[4] = {0.0, 0.0, 0.0, 0.0};
    for (int w = 0; w < nw; ++w) {
      dd += red[w * 6 + 0];
      nn = fmax(nn, red[w * 6 + 1]);
      ee = fmax(ee, red[w * 6 + 2]);
      r[0] = fmax(r[0], red[w * 6 + 3]);
      r[1] = fmax(r[1], red[w * 6 + 4]);
      r[2] += red[w * 6 + 5];
    }
    r[3] = fold_row_store(s, 0, dd, 0.0, nn, ee, dprev, dnext);
    s.stats[0] = r[0];
    s.stats[1] = r[1];
    s.stats[2] = r[2];
    s.stats[3] = r[3];
    if (s.fuse_decide) {
      *dec = decide_local(s, r);
      if (s.has_loop && (dec->done || dec->j >= s.loop_total)) cudaGraphSetConditional(s.loop_cond, 0u);
    }
  }
  if (s.fuse_decide) {
    __syncthreads();
    cycle_sample_precheck(s, *dec, reinterpret_cast<unsigned*>(scratch + 6 * nw));
  }
}


}  // namespace dpt
