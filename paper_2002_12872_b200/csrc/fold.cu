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
#include "dpt_fold.cuh"
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

// Loop condition of the device-side iteration loop.  It starts at 1 for every
// graph launch and keeps its value between iterations, so only the stop is
// written (cudaGraphSetConditional costs ~15 us of kernel tail; every
// iteration paying it tripled the fold).  Every path that can end the loop --
// the decision and the early return of a finished state -- reaches here.
__device__ __forceinline__ void set_loop_condition(const DevSolve& s) {
  if (s.has_loop) {
    const dpt_sm_state* st = s.state;
    if (st->done || st->j >= s.loop_total) cudaGraphSetConditional(s.loop_cond, 0u);
  }
}

__global__ void __launch_bounds__(kFoldThreads) fold_kernel(DevSolve s, int ntiles_this) {
  if (s.state->done) {
    if (blockIdx.x == 0 && threadIdx.x == 0) set_loop_condition(s);
    return;
  }
  const int j = launch_index(s);
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
      double d = 0.0, dim = 0.0, num = 0.0, den = 0.0;
      for (int tn = lane; tn < ntn; tn += 32) {
        d += s.rowpart[rp_index(0, i, tn, rows, ntn)];
        num = fmax(num, s.rowpart[rp_index(1, i, tn, rows, ntn)]);
        den = fmax(den, s.rowpart[rp_index(2, i, tn, rows, ntn)]);
        if (s.cplx) dim += s.rowpart[rp_index(3, i, tn, rows, ntn)];
      }
      d = warp_sum(d);
      dim = warp_sum(dim);
      num = warp_max(num);
      den = warp_max(den);
      if (lane == 0) rmax = fmax(rmax, fold_row_store(s, i, d, dim, num, den, dprev, dnext));
    }
  } else {
    // few rows (the row map has one): block per row, threads over the blocks;
    // the three row folds share one reduction pass (one barrier)
    __shared__ double red3[kFoldThreads / 32][4];
    for (int64_t i = blockIdx.x; i < rows; i += gridDim.x) {
      double d = 0.0, dim = 0.0, num = 0.0, den = 0.0;
      for (int tn = threadIdx.x; tn < ntn; tn += blockDim.x) {
        d += s.rowpart[rp_index(0, i, tn, rows, ntn)];
        num = fmax(num, s.rowpart[rp_index(1, i, tn, rows, ntn)]);
        den = fmax(den, s.rowpart[rp_index(2, i, tn, rows, ntn)]);
        if (s.cplx) dim += s.rowpart[rp_index(3, i, tn, rows, ntn)];
      }
      d = warp_sum(d);
      dim = warp_sum(dim);
      num = warp_max(num);
      den = warp_max(den);
      if (lane == 0) {
        red3[threadIdx.x >> 5][0] = d;
        red3[threadIdx.x >> 5][1] = num;
        red3[threadIdx.x >> 5][2] = den;
        red3[threadIdx.x >> 5][3] = dim;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        double dd = 0.0, nn = 0.0, ee = 0.0, di = 0.0;
        for (int w = 0; w < int(blockDim.x >> 5); ++w) {
          dd += red3[w][0];
          nn = fmax(nn, red3[w][1]);
          ee = fmax(ee, red3[w][2]);
          di += red3[w][3];
        }
        rmax = fmax(rmax, fold_row_store(s, i, dd, di, nn, ee, dprev, dnext));
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
  {  // the four launch maxima in one reduction pass
    __shared__ double red4[kFoldThreads / 32][4];
    a0 = warp_max(a0);
    a1 = warp_max(a1);
    a2 = warp_sum(a2);
    rmax = warp_max(rmax);
    __syncthreads();
    if (lane == 0) {
      red4[threadIdx.x >> 5][0] = a0;
      red4[threadIdx.x >> 5][1] = a1;
      red4[threadIdx.x >> 5][2] = a2;
      red4[threadIdx.x >> 5][3] = rmax;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      a0 = a1 = a2 = rmax = 0.0;
      for (int w = 0; w < int(blockDim.x >> 5); ++w) {
        a0 = fmax(a0, red4[w][0]);
        a1 = fmax(a1, red4[w][1]);
        a2 += red4[w][2];
        rmax = fmax(rmax, red4[w][3]);
      }
    }
  }
  if (threadIdx.x == 0) {
    double* bp = s.blockpart + size_t(blockIdx.x) * 8;
    bp[0] = a0;
    bp[1] = a1;
    bp[2] = a2;
    bp[3] = rmax;
    if (gridDim.x == 1) {
      last = true;  // nothing to elect (the row map's fold is one block)
    } else {
      fence_acq_rel_gpu();
      const unsigned prev = atomicAdd(s.counter, 1u);
      last = (prev == gridDim.x - 1);
    }
  }
  __syncthreads();
  if (!last) return;
  __shared__ dpt_sm_state dec;  // the decided state, for the precheck
  // The elected block folds the per-block maxima with all its threads (a
  // single-thread loop over ~300 blocks was a chain of L2 round trips: c2's
  // fold took 32 us).  Max is order-free and the nonfinite count is an exact
  // integer sum, so the result does not depend on the reduction shape.
  double r[4] = {a0, a1, a2, rmax};  // thread 0: this block's own maxima
  if (gridDim.x > 1) {
    if (threadIdx.x == 0) fence_acq_rel_gpu();  // acquire the other blocks' partials
    __syncthreads();
    r[0] = r[1] = r[2] = r[3] = 0.0;
    for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x) {  // __ldcg: L2, where they landed
      const double2 p01 = __ldcg(reinterpret_cast<const double2*>(s.blockpart + size_t(b) * 8));
      const double2 p23 = __ldcg(reinterpret_cast<const double2*>(s.blockpart + size_t(b) * 8 + 2));
      r[0] = fmax(r[0], p01.x);
      r[1] = fmax(r[1], p01.y);
      r[2] += p23.x;
      r[3] = fmax(r[3], p23.y);
    }
    __shared__ double red5[kFoldThreads / 32][4];
    r[0] = warp_max(r[0]);
    r[1] = warp_max(r[1]);
    r[2] = warp_sum(r[2]);
    r[3] = warp_max(r[3]);
    if (lane == 0) {
      red5[threadIdx.x >> 5][0] = r[0];
      red5[threadIdx.x >> 5][1] = r[1];
      red5[threadIdx.x >> 5][2] = r[2];
      red5[threadIdx.x >> 5][3] = r[3];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      r[0] = r[1] = r[2] = r[3] = 0.0;
      for (int w = 0; w < int(blockDim.x >> 5); ++w) {
        r[0] = fmax(r[0], red5[w][0]);
        r[1] = fmax(r[1], red5[w][1]);
        r[2] += red5[w][2];
        r[3] = fmax(r[3], red5[w][3]);
      }
    }
  }
  if (threadIdx.x == 0) {
    s.stats[0] = r[0];
    s.stats[1] = r[1];
    s.stats[2] = r[2];
    s.stats[3] = r[3];
    *s.counter = 0u;
    if (s.fuse_decide) {  // single rank: no cross-rank max in between
      dec = decide_local(s, r);
      if (s.has_loop && (dec.done || dec.j >= s.loop_total)) cudaGraphSetConditional(s.loop_cond, 0u);
    }
  }
  if (s.fuse_decide) {
    __syncthreads();
    cycle_sample_precheck(s, dec);
  }
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
  const int64_t n = s.ncol, ld = s.ld;
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
    fence_acq_rel_gpu();
    last = (atomicAdd(s.counter, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    fence_acq_rel_gpu();
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
    double v = 0.0, vi = 0.0;
    if (delta) {
      if (s.cplx) {  // B image: Re D(i,i) = B[2i][2i], Im D(i,i) = B[2i+1][2i]
        v = delta[size_t(2 * gi) * size_t(s.ldd) + size_t(2 * gi)];
        vi = delta[size_t(2 * gi + 1) * size_t(s.ldd) + size_t(2 * gi)];
      } else {
        v = delta[size_t(gi) * size_t(s.ldd) + size_t(gi)];
      }
    } else {
      for (int64_t p = rp[gi]; p < rp[gi + 1]; ++p)
        if (cl[p] == gi) {
          v = s.cplx ? vl[2 * p] : vl[p];
          vi = s.cplx ? vl[2 * p + 1] : 0.0;
        }
    }
    if (s.cplx) {
      s.dvec[0][2 * i] = v;
      s.dvec[0][2 * i + 1] = vi;
    } else {
      s.dvec[0][i] = v;
    }
  }
}

// A_0 = I (local rows) in slot 0; e_row for the row map (rows == 1, row0 = chart row).
__global__ void identity_kernel(DevSolve s) {
  const size_t total = size_t(s.rows) * size_t(s.ld);
  for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += size_t(gridDim.x) * blockDim.x) {
    const int64_t r = int64_t(e / size_t(s.ld)), c = int64_t(e % size_t(s.ld));
    s.slots[e] = (c < s.ncol && (s.cplx ? 2 * (s.row0 + r) == c : s.row0 + r == c)) ? 1.0 : 0.0;
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
    double v = 0.0, vi = 0.0;
    if (s.cplx) {
      cd acc = cmake(0.0, 0.0);
      if (delta) {
        const double* brow = delta + size_t(2 * gi) * size_t(s.ldd);  // (Re D(i,k), -Im D(i,k))
        for (int64_t k = lane; k < s.n; k += 32)
          acc = cadd(acc, cmul(cmake(a[2 * k], a[2 * k + 1]), cmake(brow[2 * k], -brow[2 * k + 1])));
        acc.x = warp_sum(acc.x);
        acc.y = warp_sum(acc.y);
      } else if (lane == 0) {
        for (int64_t q = rp[gi]; q < rp[gi + 1]; ++q)
          acc = cadd(acc, cmul(cmake(vl[2 * q], vl[2 * q + 1]), cmake(a[2 * cl[q]], a[2 * cl[q] + 1])));
      }
      v = acc.x;
      vi = acc.y;
    } else if (delta) {
      for (int64_t k = lane; k < s.n; k += 32) v = __fma_rn(a[k], delta[size_t(gi) * size_t(s.ldd) + size_t(k)], v);
      v = warp_sum(v);
    } else if (lane == 0) {
      for (int64_t q = rp[gi]; q < rp[gi + 1]; ++q) v = __fma_rn(vl[q], a[cl[q]], v);
    }
    if (lane == 0) {
      if (s.cplx) {
        s.dvec[0][2 * i] = v;
        s.dvec[0][2 * i + 1] = vi;
      } else {
        s.dvec[0][i] = v;
      }
    }
  }
}

// z_unit = z / ||z||_2 when the norm is finite and positive, else z
// (dominant_eigenpair, dpt.cpp:432-436; vec_two_norm, matrix.cpp:372-376).
// Fixed grid + fixed chunking + last-block combine: deterministic.
constexpr int kUnitBlocks = 296;
__global__ void __launch_bounds__(256) unit_norm_kernel(const double* __restrict__ z, int64_t n, double* part,
                                                         unsigned* counter, double* nrm) {
  __shared__ double sh[32];
  __shared__ bool last;
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t b0 = int64_t(blockIdx.x) * chunk, b1 = b0 + chunk < n ? b0 + chunk : n;
  double v = 0.0;
  for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) v = __fma_rn(z[i], z[i], v);
  v = block_sum(v, sh);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = v;
    fence_acq_rel_gpu();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    fence_acq_rel_gpu();
    double t = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) t += ((volatile double*)part)[b];
    *nrm = sqrt(t);
    *counter = 0u;
  }
}

__global__ void unit_scale_kernel(const double* __restrict__ z, double* __restrict__ out, int64_t n,
                                  const double* nrm) {
  const double q = *nrm;
  const bool ok = q > 0.0 && isfinite(q);
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    out[i] = ok ? z[i] / q : z[i];
}

cudaError_t launch_unit(const double* z, double* out, int64_t n, double* scratch, unsigned* counter,
                        cudaStream_t st) {
  unit_norm_kernel<<<kUnitBlocks, 256, 0, st>>>(z, n, scratch, counter, scratch + kUnitBlocks);
  unit_scale_kernel<<<592, 256, 0, st>>>(z, out, n, scratch + kUnitBlocks);
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
