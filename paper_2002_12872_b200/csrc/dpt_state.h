// dpt_state.h -- the reference's per-iteration decision logic as one function
// shared by the device (the 1-thread decision kernel, K4b) and the host (unit
// tests through dpt_sm_decide in the C-ABI, no GPU needed).
//
// It restates run_full's loop body order (proj/src/dpt.cpp:130-187) under the
// launch <-> iteration lag of SURVEY.md Appendix B: launch j maps A_{j-1} to A_j
// and, from the same GEMM, yields the read-offs of A_{j-1}.  So after launch j
// the decision for reference iteration k = j-1 (trace, convergence, cycle) is
// taken first, then iteration j's divergence test -- exactly the reference's
// order, because the reference finishes iteration j-1 before forming A_j.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define DPT_HD __host__ __device__
#else
#define DPT_HD
#endif

#define DPT_MAX_WINDOW 16       // IterationOptions::cycle_window default and our cap
#define DPT_STATS_CYCLE0 4      // stats[4 .. 4+DPT_MAX_WINDOW): cycle "not within" flags

// Global statistics of one launch after the (cross-rank) max fold.
//  [0] step_j = max|A_j - A_{j-1}|
//  [1] max|A_j|
//  [2] nonfinite count of A_j (> 0 means some entry is not finite)
//  [3] max_res(A_{j-1})        (max over rows of the row residuals)
//  [4+p] 1 if A_{j-1} differs from window entry p by >= tol somewhere, else 0
//        (p = 0 is A_{j-3}, p = 1 is A_{j-4}, ...: the reference's deque order,
//        most recent first; A_0 = I is a real entry)
#define DPT_NSTATS (DPT_STATS_CYCLE0 + DPT_MAX_WINDOW)

typedef struct dpt_sm_options {
  double tol, residual_tol, divergence_threshold;
  int max_iter;
  int win;            // effective window (0 = cycle detection off)
  int have_trace;     // log (k, step, max_res) for every decided iteration
} dpt_sm_options;

typedef struct dpt_sm_state {
  int done;           // 1 once a terminal status is known
  int status;         // ConvergenceStatus (dpt.hpp:13-18): 0 Conv, 1 Bounded, 2 Diverged, 3 MaxIter
  int iterations;     // reported iterations
  int final_iter;     // index m of the iterate A_m the report carries
  int readoffs;       // 1: eps/res buffers hold the read-offs of A_final; 0: NaN (Diverged)
  int j;              // launches whose statistics have been consumed
  int cycle_pending;  // the cycle kernel must test A_j against the window
  int trace_len;      // entries written to the trace log
  double step_norm;   // reported step norm
  double last_step;   // step_j of the latest launch (iteration j's step)
  double pad[2];
} dpt_sm_state;

// Iteration k's "settled" flag: !ramped || |lam_k - lam| <= tol |lam| (dpt.cpp:131-134),
// precomputed on the host with std::pow for parity and passed as a table.

// Consume launch j's statistics.  settled_prev = settled(j-1), settled_cur = settled(j).
// trace_out (optional) receives {k, step, max_res} triples.
DPT_HD static inline void dpt_sm_decide(dpt_sm_state* s, const dpt_sm_options* o, const double* stats,
                                        int j, int settled_prev, int settled_cur,
                                        double* trace_out) {
  if (s->done) return;
  const double cycle_margin = 1e3 * o->tol;
  if (j >= 2) {
    // ---- reference iteration k = j-1, after pn = P(A_k) (dpt.cpp:152-186) ----
    const int k = j - 1;
    const double step_k = s->last_step;
    const double max_res = stats[3];
    if (o->have_trace && trace_out) {
      trace_out[3 * s->trace_len + 0] = (double)k;
      trace_out[3 * s->trace_len + 1] = step_k;
      trace_out[3 * s->trace_len + 2] = max_res;
      s->trace_len++;
    }
    if (settled_prev && step_k < o->tol) {
      if (max_res < o->residual_tol) {
        s->done = 1; s->status = 0; s->iterations = k; s->final_iter = k;
        s->readoffs = 1; s->step_norm = step_k;
        return;
      }
    } else if (o->win > 0 && settled_prev && step_k > cycle_margin) {
      // window holds A_{k-2} .. A_{k-win}, never older than A_0
      int npast = k - 1;
      if (npast > o->win - 1) npast = o->win - 1;
      for (int p = 0; p < npast; ++p) {
        if (stats[DPT_STATS_CYCLE0 + p] == 0.0) {  // within_tol held for this entry
          s->done = 1; s->status = 1; s->iterations = k; s->final_iter = k;
          s->readoffs = 1; s->step_norm = step_k;
          return;
        }
      }
    }
    if (k == o->max_iter) {  // budget exhausted (dpt.cpp:189-191)
      s->done = 1; s->status = 3; s->iterations = o->max_iter; s->final_iter = k;
      s->readoffs = 1; s->step_norm = step_k;
      return;
    }
  }
  s->j = j;
  if (j <= o->max_iter) {
    // ---- reference iteration j: step and divergence (dpt.cpp:145-150) ----
    const double step_j = stats[0];
    s->last_step = step_j;
    if (stats[2] > 0.0 || stats[1] > o->divergence_threshold) {
      s->done = 1; s->status = 2; s->iterations = j; s->final_iter = j;
      s->readoffs = 0; s->step_norm = step_j;
      return;
    }
    // cycle test of A_j happens only on the else-branch of the convergence gate
    s->cycle_pending = (o->win > 0 && !(settled_cur && step_j < o->tol) && settled_cur &&
                        step_j > cycle_margin && j >= 2) ? 1 : 0;  // window non-empty from k = 2 on
  }
}
