// fold.cu -- K4: the tiny deterministic reductions after each step launch,
// the 1-thread decision kernel, and the cycle (revisit) test.
//
// fold:   d_j(i) = sum over column blocks of the step kernel's partials (fixed
//         order => deterministic), eps_i / res_i of A_{j-1} (residuals_of,
//         proj/src/dpt.cpp:23-44), and the launch's global maxima (step,
//         max|A_j|, nonfinite count, max residual) -> stats[0..3].
// decide: runs dpt_sm_decide (dpt_state.h) on the stats (after the optional
//         cross-rank NCCL max) -- the reference's loop body order.
// cycle:  within_tol(A_j, past) for the window (dpt.cpp:60-79, :171-179) with an
//         exact sample-first early-out: a sample element with |diff| >= tol
//         already proves within_tol false for that past iterate.
#include <cuda_runtime.h>
#include <stdint.h>

#include "dpt_device.cuh"
#include "dpt_kernels.h"

namespace dpt {

constexpr int kFoldThreads = 256;
constexpr int kFoldMaxBlocks = 296;  // 2 x 148 SMs

int fold_blocks(int64_t rows) {
  if (rows < 32) return int(rows < 1 ? 1 : rows);  // block per row
  int64_t b = (rows + (kFoldThreads / 32) - 1) / (kFoldThreads / 32);  // warp per row
  if (b > kFoldMaxBlocks) b = kFoldMaxBlocks;
  if (b < 1) b = 1;
  return int(b);
}

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
__device__ __forceinline__ void fold_row_store(const DevSolve& s, int64_t i, double d, double num, double den,
                                               const double* dprev, double* dnext) {
  const double r = num / fmax(den, 1e-300);  // kTinyDen, dpt.cpp:18, :40
  s.eps[i] = __dadd_rn(s.theta[s.row0 + i], __dmul_rn(s.lambda, dprev[i]));
  s.res[i] = r;
  dnext[i] = d;
}

__device__ void decide_now(const DevSolve& s);

// Sample-first part of the cycle test, run by one block right after the
// decision: if the first entries already differ by >= tol from every window
// entry, within_tol is false for all of them and the cycle kernel has nothing
// to do (exact early-out, dpt.cpp:60-79).
__device__ void cycle_sample_precheck(const DevSolve& s, double* sh) {
  dpt_sm_state* st = s.state;
  if (st->done || !st->cycle_pending) return;
  const int j = st->j;
  int npast = j - 1;
  if (npast > s.opts.win - 1) npast = s.opts.win - 1;
  const int64_t n = s.n, ld = s.ld;
  const int64_t elems = s.rows * n;
  const int64_t ns = elems < int64_t(blockDim.x) ? elems : int64_t(blockDim.x);
  const double* cur = s.slots + size_t(j % s.nslots) * size_t(s.slot_elems);
  int any = 0;
  for (int p = 0; p < npast; ++p) {
    const double* past = s.slots + size_t((j - 2 - p) % s.nslots) * size_t(s.slot_elems);
    double m = 0.0;
    const int64_t e = threadIdx.x;
    if (e < ns) {
      const int64_t r = e / n, c = e % n;
      m = fabs(cur[r * ld + c] - past[r * ld + c]);
    }
    m = block_max(m, sh);
    if (threadIdx.x == 0 && m < s.opts.tol) any = 1;
  }
  if (threadIdx.x == 0 && !any) {
    st->cycle_pending = 0;  // refuted for every entry: the stats keep "not within"
    for (int p = 0; p < DPT_MAX_WINDOW; ++p) s.stats[DPT_STATS_CYCLE0 + p] = 1.0;
  }
}

__global__ void __launch_bounds__(kFoldThreads) fold_kernel(DevSolve s, int ntiles_this) {
  if (s.state->done) return;
  const int j = launch_index(s);
  __shared__ double sh[32];
  __shared__ bool last;
  const int64_t rows = s.rows;
  const int ntn = s.ntn;
  const double* dprev = s.dvec[(j - 1) & 1];
  double* dnext = s.dvec[j & 1];
  const int lane = threadIdx.x & 31;
  double rmax = 0.0;
  if (rows >= 32) {
    // warp per row, lanes stride over the column blocks (coalesced: [rows][ntn])
    const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
    for (int64_t i = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); i < rows; i += warps) {
      double d = 0.0, num = 0.0, den = 0.0;
      for (int tn = lane; tn < ntn; tn += 32) {
        d += s.rowpart[rp_index(0, i, tn, rows, ntn)];
        num = fmax(num, s.rowpart[rp_index(1, i, tn, rows, ntn)]);
        den = fmax(den, s.rowpart[rp_index(2, i, tn, rows, ntn)]);
      }
      d = warp_sum(d);
      num = warp_max(num);
      den = warp_max(den);
      if (lane == 0) {
        fold_row_store(s, i, d, num, den, dprev, dnext);
        rmax = fmax(rmax, s.res[i]);
      }
    }
  } else {
    // few rows (the row map has one): block per row, threads over the blocks
    for (int64_t i = blockIdx.x; i < rows; i += gridDim.x) {
      double d = 0.0, num = 0.0, den = 0.0;
      for (int tn = threadIdx.x; tn < ntn; tn += blockDim.x) {
        d += s.rowpart[rp_index(0, i, tn, rows, ntn)];
        num = fmax(num, s.rowpart[rp_index(1, i, tn, rows, ntn)]);
        den = fmax(den, s.rowpart[rp_index(2, i, tn, rows, ntn)]);
      }
      d = block_sum(d, sh);
      num = block_max(num, sh);
      den = block_max(den, sh);
      if (threadIdx.x == 0) {
        fold_row_store(s, i, d, num, den, dprev, dnext);
        rmax = fmax(rmax, s.res[i]);
      }
      __syncthreads();
    }
  }
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < ntiles_this; t += gridDim.x * blockDim.x) {
    a0 = fmax(a0, s.tilepart[size_t(t) * 4 + 0]);
    a1 = fmax(a1, s.tilepart[size_t(t) * 4 + 1]);
    a2 += s.tilepart[size_t(t) * 4 + 2];
  }
  a0 = block_max(a0, sh);
  a1 = block_max(a1, sh);
  a2 = block_sum(a2, sh);
  rmax = block_max(rmax, sh);
  if (threadIdx.x == 0) {
    double* bp = s.blockpart + size_t(blockIdx.x) * 8;
    bp[0] = a0;
    bp[1] = a1;
    bp[2] = a2;
    bp[3] = rmax;
    __threadfence();
    const unsigned prev = atomicAdd(s.counter, 1u);
    last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  if (threadIdx.x == 0) {
    __threadfence();
    double r0 = 0.0, r1 = 0.0, r2 = 0.0, r3 = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) {
      const volatile double* bp = s.blockpart + size_t(b) * 8;
      r0 = fmax(r0, bp[0]);
      r1 = fmax(r1, bp[1]);
      r2 += bp[2];
      r3 = fmax(r3, bp[3]);
    }
    s.stats[0] = r0;
    s.stats[1] = r1;
    s.stats[2] = r2;
    s.stats[3] = r3;
    *s.counter = 0u;
    if (s.fuse_decide) decide_now(s);  // single rank: no cross-rank max in between
  }
  if (s.fuse_decide) {
    __syncthreads();
    cycle_sample_precheck(s, sh);
  }
}

__device__ void decide_now(const DevSolve& s) {
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

__global__ void decide_kernel(DevSolve s) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  decide_now(s);
}

// Tests A_j (slot j % nslots) against A_{j-2-p}, p < npast.
__global__ void __launch_bounds__(kFoldThreads) cycle_kernel(DevSolve s, int64_t elems) {
  const dpt_sm_state* st = s.state;
  __shared__ double sh[32];
  __shared__ bool last;
  __shared__ int cand[DPT_MAX_WINDOW];
  const int j = st->j;
  if (st->done || !st->cycle_pending) {
    if (blockIdx.x == 0 && threadIdx.x < DPT_MAX_WINDOW) s.stats[DPT_STATS_CYCLE0 + threadIdx.x] = 1.0;
    return;
  }
  const int win = s.opts.win;
  int npast = j - 1;
  if (npast > win - 1) npast = win - 1;
  const int64_t n = s.n, ld = s.ld;
  const double tol = s.opts.tol;
  const size_t slot_elems = size_t(s.slot_elems);
  const double* cur = s.slots + size_t(j % s.nslots) * slot_elems;
  // sample: the first min(elems, 1024) entries
  const int64_t nsample = elems < 1024 ? elems : 1024;
  int any = 0;
  for (int p = 0; p < npast; ++p) {
    const double* past = s.slots + size_t((j - 2 - p) % s.nslots) * slot_elems;
    double m = 0.0;
    for (int64_t e = threadIdx.x; e < nsample; e += blockDim.x) {
      const int64_t r = e / n, c = e % n;
      m = fmax(m, fabs(cur[r * ld + c] - past[r * ld + c]));
    }
    m = block_max(m, sh);
    if (threadIdx.x == 0) cand[p] = (m < tol) ? 1 : 0;
    __syncthreads();
    any |= cand[p];
  }
  if (!any) {  // the sample already refutes within_tol for every window entry
    if (blockIdx.x == 0 && threadIdx.x < DPT_MAX_WINDOW) s.stats[DPT_STATS_CYCLE0 + threadIdx.x] = 1.0;
    return;
  }
  for (int p = 0; p < npast; ++p) {
    double m = 0.0;
    if (cand[p]) {
      const double* past = s.slots + size_t((j - 2 - p) % s.nslots) * slot_elems;
      for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < elems;
           e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = e / n, c = e % n;
        m = fmax(m, fabs(cur[r * ld + c] - past[r * ld + c]));
      }
    }
    m = block_max(m, sh);
    if (threadIdx.x == 0) s.cyclepart[size_t(blockIdx.x) * DPT_MAX_WINDOW + p] = m;
  }
  if (threadIdx.x == 0) {
    __threadfence();
    last = (atomicAdd(s.counter, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    for (int p = 0; p < DPT_MAX_WINDOW; ++p) {
      double m = 0.0;
      if (p < npast && cand[p]) {
        for (unsigned b = 0; b < gridDim.x; ++b)
          m = fmax(m, ((volatile double*)s.cyclepart)[size_t(b) * DPT_MAX_WINDOW + p]);
        s.stats[DPT_STATS_CYCLE0 + p] = (m >= tol) ? 1.0 : 0.0;
      } else {
        s.stats[DPT_STATS_CYCLE0 + p] = 1.0;
      }
    }
    *s.counter = 0u;
  }
}

// d_0(i) = P(I)(i,i) = Delta(i,i) (the reference's pmat = matmul(I, delta_t)).
__global__ void set_diag_kernel(DevSolve s, const double* __restrict__ delta, const int64_t* rp,
                                const int32_t* cl, const double* vl) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < s.rows;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t gi = s.row0 + i;
    double v = 0.0;
    if (delta) {
      v = delta[size_t(gi) * size_t(s.ld) + size_t(gi)];
    } else {
      for (int64_t p = rp[gi]; p < rp[gi + 1]; ++p)
        if (cl[p] == gi) v = vl[p];
    }
    s.dvec[0][i] = v;
  }
}

// A_0 = I (local rows) in slot 0; e_row for the row map (rows == 1, row0 = chart row).
__global__ void identity_kernel(DevSolve s) {
  const size_t total = size_t(s.rows) * size_t(s.ld);
  for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += size_t(gridDim.x) * blockDim.x) {
    const int64_t r = int64_t(e / size_t(s.ld)), c = int64_t(e % size_t(s.ld));
    s.slots[e] = (c < s.n && s.row0 + r == c) ? 1.0 : 0.0;
  }
}

// d(i) = sum_k A(i,k) Delta(i,k) for the iterate in slot 0: P(A)(i,i) for a
// caller-supplied iterate (step_full) -- the dense dot or the CSR row dot.
__global__ void rowdot_kernel(DevSolve s, const double* __restrict__ delta, const int64_t* rp,
                              const int32_t* cl, const double* vl) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t i = wid; i < s.rows; i += nw) {
    const int64_t gi = s.row0 + i;
    const double* a = s.slots + size_t(i) * size_t(s.ld);
    double v = 0.0;
    if (delta) {
      for (int64_t k = lane; k < s.n; k += 32) v = __fma_rn(a[k], delta[size_t(gi) * size_t(s.ld) + size_t(k)], v);
      v = warp_sum(v);
    } else if (lane == 0) {
      for (int64_t q = rp[gi]; q < rp[gi + 1]; ++q) v = __fma_rn(vl[q], a[cl[q]], v);
    }
    if (lane == 0) s.dvec[0][i] = v;
  }
}

// z_unit = z / ||z||_2 when the norm is finite and positive, else z
// (dominant_eigenpair, dpt.cpp:432-436; vec_two_norm, matrix.cpp:372-376).
__global__ void __launch_bounds__(1024) unit_kernel(const double* __restrict__ z, double* __restrict__ out, int64_t n) {
  __shared__ double sh[32];
  __shared__ double nrm;
  double v = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) v = __fma_rn(z[i], z[i], v);
  v = block_sum(v, sh);
  if (threadIdx.x == 0) nrm = sqrt(v);
  __syncthreads();
  const double q = nrm;
  const bool ok = q > 0.0 && isfinite(q);
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) out[i] = ok ? z[i] / q : z[i];
}

cudaError_t launch_unit(const double* z, double* out, int64_t n, cudaStream_t st) {
  unit_kernel<<<1, 1024, 0, st>>>(z, out, n);
  return cudaGetLastError();
}

cudaError_t launch_identity(const DevSolve& s, cudaStream_t st) {
  identity_kernel<<<592, 256, 0, st>>>(s);
  return cudaGetLastError();
}

cudaError_t launch_rowdot(const DevSolve& s, const double* delta, const DevCsr* csr, cudaStream_t st) {
  rowdot_kernel<<<296, 256, 0, st>>>(s, delta, csr ? csr->rowptr : nullptr, csr ? csr->cols : nullptr,
                                     csr ? csr->vals : nullptr);
  return cudaGetLastError();
}

cudaError_t launch_fold(const DevSolve& s, int ntiles_this, cudaStream_t st) {
  fold_kernel<<<fold_blocks(s.rows), kFoldThreads, 0, st>>>(s, ntiles_this);
  return cudaGetLastError();
}

cudaError_t launch_decide(const DevSolve& s, cudaStream_t st) {
  decide_kernel<<<1, 32, 0, st>>>(s);
  return cudaGetLastError();
}

cudaError_t launch_cycle(const DevSolve& s, int64_t elems, cudaStream_t st) {
  int64_t b = (elems + kFoldThreads * 8 - 1) / (kFoldThreads * 8);
  if (b > kFoldMaxBlocks) b = kFoldMaxBlocks;
  if (b < 1) b = 1;
  cycle_kernel<<<unsigned(b), kFoldThreads, 0, st>>>(s, elems);
  return cudaGetLastError();
}

cudaError_t launch_set_diag_delta(const DevSolve& s, const double* delta, const DevCsr* csr,
                                  cudaStream_t st) {
  set_diag_kernel<<<fold_blocks(s.rows), kFoldThreads, 0, st>>>(
      s, delta, csr ? csr->rowptr : nullptr, csr ? csr->cols : nullptr, csr ? csr->vals : nullptr);
  return cudaGetLastError();
}

}  // namespace dpt
