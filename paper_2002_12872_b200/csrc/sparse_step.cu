// sparse_step.cu -- K2 (CSR full map) and K3 (row map / single vector).
//
// K2 replaces, per reference iteration with a CSR perturbation:
//   pn = matmul(an, delta_t) with Sparse delta_t   proj/src/matrix.cpp:145-158
//   plus the same map / step / divergence / residual work as K1.
// Row form: P(i,j) = sum_{k in row j of Delta} Delta(j,k) A(i,k), a sparse dot
// per output (i, j).  A CTA owns R whole rows of A: it stages them in shared
// memory (the gathers A(i,k) hit smem), streams the CSR of Delta once from L2
// and writes A'(i, :) coalesced.  Because the CTA owns the whole row, P(i,i)
// and the next iterate's d(i) = sum_m Delta(i,m) A'(i,m) are exact dots in CSR
// order (bit-identical to the P(i,i) the next launch forms) -- no lag here.
//
// K3 replaces run_single's body (proj/src/dpt.cpp:233-289):
//   w = matvec(delta, z)                  src/matrix.cpp:215-225 (dense :203-213)
//   zn[m] = m==row ? 1 : lam_k g_m (w[m] - w[row] z[m])   src/dpt.cpp:239-244
//   step, all_finite / vec_inf_norm divergence           src/dpt.cpp:245-252
//   residual_single of z (eps = d_row + lam w[row])      src/dpt.cpp:47-58
// w[row] is needed by every block: each block recomputes the 16-nonzero dot
// redundantly in CSR order (bit-identical everywhere).  HBM-bound: the CSR
// values + columns stream once, z is gathered from L2.
#include <cuda_runtime.h>
#include <stdint.h>

#include "dpt_device.cuh"
#include "dpt_kernels.h"

namespace dpt {

constexpr int kCsrThreads = 512;
constexpr int kCsrSmemBudget = 200 * 1024;

static int csr_rows_per_cta(int64_t n) {
  int64_t r = kCsrSmemBudget / (n * 8);
  if (r > 8) r = 8;
  return int(r);  // 0 => rows gathered from global memory
}

int csr_ntn(int64_t) { return 1; }

int csr_step_ntiles(int64_t rows, int64_t n) {
  const int R = csr_rows_per_cta(n) > 0 ? csr_rows_per_cta(n) : 1;
  return int((rows + R - 1) / R);
}

template <int R>
__global__ void __launch_bounds__(kCsrThreads) csr_step_kernel(DevSolve s, DevCsr D, int use_smem) {
  if (s.state->done) return;
  const int jl = launch_index(s);
  extern __shared__ __align__(16) double sa[];  // [R][n] staged rows of A_{j-1}
  __shared__ double red[kCsrThreads / 32][R][3];
  __shared__ double wred[kCsrThreads / 32][3];
  const int64_t n = s.n, ld = s.ld, rows = s.rows;
  const int64_t il0 = int64_t(blockIdx.x) * R;
  const int nr = int(rows - il0 < R ? rows - il0 : R);
  const int slot_in = (jl - 1) % s.nslots, slot_out = jl % s.nslots;
  const double* a_in = s.slots + size_t(slot_in) * size_t(s.slot_elems);
  double* a_out = s.slots + size_t(slot_out) * size_t(s.slot_elems);
  const double lam_k = lam_of(s, jl), lam = s.lambda;
  const double* d_in = s.dvec[(jl - 1) & 1];

  const double* arow[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int rr = r < nr ? r : 0;
    arow[r] = use_smem ? sa + size_t(r) * size_t(n) : a_in + size_t(il0 + rr) * size_t(ld);
  }
  if (use_smem) {
    for (int r = 0; r < nr; ++r)
      for (int64_t c = threadIdx.x; c < n; c += blockDim.x)
        sa[size_t(r) * size_t(n) + size_t(c)] = a_in[size_t(il0 + r) * size_t(ld) + size_t(c)];
    __syncthreads();
  }
  double ti[R], di[R], epsi[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int64_t gi = s.row0 + il0 + (r < nr ? r : 0);
    ti[r] = s.theta[gi];
    di[r] = d_in[il0 + (r < nr ? r : 0)];
    epsi[r] = __dadd_rn(ti[r], __dmul_rn(lam, di[r]));
  }
  double num[R], den[R];
#pragma unroll
  for (int r = 0; r < R; ++r) num[r] = den[r] = 0.0;
  double t_step = 0.0, t_max = 0.0, t_nonfin = 0.0;

  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
    double p[R];
#pragma unroll
    for (int r = 0; r < R; ++r) p[r] = 0.0;
    const int64_t pb = D.rowptr[j], pe = D.rowptr[j + 1];
    for (int64_t q = pb; q < pe; ++q) {
      const int32_t k = __ldg(D.cols + q);
      const double v = __ldg(D.vals + q);
#pragma unroll
      for (int r = 0; r < R; ++r) p[r] = __fma_rn(v, arow[r][k], p[r]);
    }
    const double tj = s.theta[j];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (r >= nr) break;
      const int64_t gi = s.row0 + il0 + r;
      const double aij = arow[r][j];
      double v;
      if (gi == j) {
        v = 1.0;
      } else {
        const double g = s.gapmat ? s.gapmat[size_t(il0 + r) * size_t(ld) + size_t(j)] : 1.0 / __dsub_rn(ti[r], tj);
        v = __dmul_rn(__dmul_rn(lam_k, g), __dsub_rn(p[r], __dmul_rn(di[r], aij)));
      }
      a_out[size_t(il0 + r) * size_t(ld) + size_t(j)] = v;
      t_step = fmax(t_step, fabs(__dsub_rn(v, aij)));
      t_max = fmax(t_max, fabs(v));
      t_nonfin += isfinite(v) ? 0.0 : 1.0;
      const double rr = __dadd_rn(__dmul_rn(__dsub_rn(tj, epsi[r]), aij), __dmul_rn(lam, p[r]));
      num[r] = fmax(num[r], fabs(rr));
      den[r] = fmax(den[r], fabs(aij));
    }
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const double a = warp_max(num[r]), b = warp_max(den[r]);
    if (l == 0) {
      red[w][r][1] = a;
      red[w][r][2] = b;
    }
  }
  t_step = warp_max(t_step);
  t_max = warp_max(t_max);
  t_nonfin = warp_sum(t_nonfin);
  if (l == 0) {
    wred[w][0] = t_step;
    wred[w][1] = t_max;
    wred[w][2] = t_nonfin;
  }
  __syncthreads();  // also orders this CTA's A' stores before the d' dots below
  // exact d_j(i) = sum_m Delta(i,m) A_j(i,m) in CSR order (= next launch's P(i,i))
  if (w < nr) {
    const int64_t il = il0 + w, gi = s.row0 + il;
    double part = 0.0;
    // lane-serial in CSR order for bit-identity with the sequential dot above
    if (l == 0) {
      for (int64_t q = D.rowptr[gi]; q < D.rowptr[gi + 1]; ++q)
        part = __fma_rn(D.vals[q], a_out[size_t(il) * size_t(ld) + size_t(D.cols[q])], part);
      double nu = 0.0, de = 0.0;
      for (int ww = 0; ww < kCsrThreads / 32; ++ww) {
        nu = fmax(nu, red[ww][w][1]);
        de = fmax(de, red[ww][w][2]);
      }
      s.rowpart[(size_t(0)) * rows + il] = part;
      s.rowpart[(size_t(1)) * rows + il] = nu;
      s.rowpart[(size_t(2)) * rows + il] = de;
    }
  }
  if (threadIdx.x == 0) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    for (int ww = 0; ww < kCsrThreads / 32; ++ww) {
      a0 = fmax(a0, wred[ww][0]);
      a1 = fmax(a1, wred[ww][1]);
      a2 += wred[ww][2];
    }
    double* tp = s.tilepart + size_t(blockIdx.x) * 4;
    tp[0] = a0;
    tp[1] = a1;
    tp[2] = a2;
    tp[3] = 0.0;
  }
}

cudaError_t launch_csr_step(const DevSolve& s, const DevCsr& d, cudaStream_t st) {
  const int Rs = csr_rows_per_cta(s.n);
  const int use_smem = Rs > 0 ? 1 : 0;
  const int R = use_smem ? Rs : 1;
  const unsigned grid = unsigned((s.rows + R - 1) / R);
  const size_t smem = use_smem ? size_t(R) * size_t(s.n) * 8 : 0;
#define DPT_CSR_CASE(RR)                                                                          \
  case RR: {                                                                                      \
    static bool attr = false;                                                                     \
    if (!attr) {                                                                                  \
      cudaFuncSetAttribute(csr_step_kernel<RR>, cudaFuncAttributeMaxDynamicSharedMemorySize,      \
                           kCsrSmemBudget + 1024);                                                \
      attr = true;                                                                                \
    }                                                                                             \
    csr_step_kernel<RR><<<grid, kCsrThreads, smem, st>>>(s, d, use_smem);                         \
    break;                                                                                        \
  }
  switch (R) {
    DPT_CSR_CASE(1)
    DPT_CSR_CASE(2)
    DPT_CSR_CASE(3)
    DPT_CSR_CASE(4)
    DPT_CSR_CASE(5)
    DPT_CSR_CASE(6)
    DPT_CSR_CASE(7)
    DPT_CSR_CASE(8)
    default:
      return cudaErrorInvalidValue;
  }
#undef DPT_CSR_CASE
  return cudaGetLastError();
}

// ------------------------------------------------------------------ K3 ----
constexpr int kSingleThreads = 256;
constexpr int kSingleRowsPerThread = 1;

int single_ntiles(int64_t n) {
  int64_t b = (n + kSingleThreads * kSingleRowsPerThread - 1) / (kSingleThreads * kSingleRowsPerThread);
  return int(b < 1 ? 1 : b);
}
int single_ntn(int64_t n) { return single_ntiles(n); }

// w_row = Delta(row, :) . z, identical order in every block.
__device__ __forceinline__ double row_dot(const DevCsr& D, const double* dense, int64_t n, int64_t ld,
                                          int64_t row, const double* z) {
  double s = 0.0;
  if (dense) {
    for (int64_t c = 0; c < n; ++c) s = __fma_rn(dense[size_t(row) * size_t(ld) + size_t(c)], z[c], s);
  } else {
    for (int64_t q = D.rowptr[row]; q < D.rowptr[row + 1]; ++q) s = __fma_rn(D.vals[q], z[D.cols[q]], s);
  }
  return s;
}

__global__ void __launch_bounds__(kSingleThreads)
    single_step_kernel(DevSolve s, DevCsr D, const double* __restrict__ dense, int64_t row) {
  if (s.state->done) return;
  const int jl = launch_index(s);
  __shared__ double wrow_s;
  __shared__ double red[kSingleThreads / 32][5];
  const int64_t n = s.n, ld = s.ld;
  const double* z = s.slots + size_t((jl - 1) % s.nslots) * size_t(s.slot_elems);
  double* zo = s.slots + size_t(jl % s.nslots) * size_t(s.slot_elems);
  const double lam_k = lam_of(s, jl), lam = s.lambda;
  if (threadIdx.x == 0) {
    wrow_s = row_dot(D, dense, n, ld, row, z);
    if (blockIdx.x == 0) s.dvec[(jl - 1) & 1][0] = wrow_s;  // w[row] of z_{j-1} for the fold's eps
  }
  __syncthreads();
  const double wr = wrow_s;
  const double trow = s.theta[row];
  const double eps = __dadd_rn(trow, __dmul_rn(lam, wr));
  double num = 0.0, den = 0.0, t_step = 0.0, t_max = 0.0, t_nonfin = 0.0;
  const int64_t m = int64_t(blockIdx.x) * kSingleThreads + threadIdx.x;
  if (m < n) {
    double w = 0.0;
    if (dense) {
      const double* dr = dense + size_t(m) * size_t(ld);
      for (int64_t c = 0; c < n; ++c) w = __fma_rn(dr[c], z[c], w);
    } else {
      const int64_t pb = D.rowptr[m], pe = D.rowptr[m + 1];
      for (int64_t q = pb; q < pe; ++q) w = __fma_rn(__ldg(D.vals + q), z[__ldg(D.cols + q)], w);
    }
    const double zm = z[m];
    const double tm = s.theta[m];
    double v;
    if (m == row) {
      v = 1.0;
    } else {
      const double g = s.gapmat ? s.gapmat[m] : 1.0 / __dsub_rn(trow, tm);  // build_gap_row, partition.cpp:83-96
      v = __dmul_rn(__dmul_rn(lam_k, g), __dsub_rn(w, __dmul_rn(wr, zm)));
    }
    zo[m] = v;
    t_step = fabs(__dsub_rn(v, zm));
    t_max = fabs(v);
    t_nonfin = isfinite(v) ? 0.0 : 1.0;
    const double r = __dadd_rn(__dmul_rn(__dsub_rn(tm, eps), zm), __dmul_rn(lam, w));
    num = fabs(r);
    den = fabs(zm);
  }
  num = warp_max(num);
  den = warp_max(den);
  t_step = warp_max(t_step);
  t_max = warp_max(t_max);
  t_nonfin = warp_sum(t_nonfin);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
    red[w][0] = num;
    red[w][1] = den;
    red[w][2] = t_step;
    red[w][3] = t_max;
    red[w][4] = t_nonfin;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a[5] = {0, 0, 0, 0, 0};
    for (int ww = 0; ww < kSingleThreads / 32; ++ww) {
      a[0] = fmax(a[0], red[ww][0]);
      a[1] = fmax(a[1], red[ww][1]);
      a[2] = fmax(a[2], red[ww][2]);
      a[3] = fmax(a[3], red[ww][3]);
      a[4] += red[ww][4];
    }
    const int tn = blockIdx.x, ntn = s.ntn;
    s.rowpart[(size_t(0) * ntn + tn)] = 0.0;
    s.rowpart[(size_t(1) * ntn + tn)] = a[0];
    s.rowpart[(size_t(2) * ntn + tn)] = a[1];
    double* tp = s.tilepart + size_t(tn) * 4;
    tp[0] = a[2];
    tp[1] = a[3];
    tp[2] = a[4];
    tp[3] = 0.0;
  }
}

cudaError_t launch_single_step(const DevSolve& s, const DevCsr& d, const double* dense, int64_t row,
                               const double*, cudaStream_t st) {
  single_step_kernel<<<single_ntiles(s.n), kSingleThreads, 0, st>>>(s, d, dense, row);
  return cudaGetLastError();
}

}  // namespace dpt
