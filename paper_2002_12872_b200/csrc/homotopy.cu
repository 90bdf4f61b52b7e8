// homotopy.cu -- element-wise kernels of the device homotopy_solve
// (proj/src/dpt.cpp:505-556).  The O(n^3) work of a
// stage -- M W, the LU solve W^-1 (M W) and the basis update W V -- runs in
// linalg.cu (DMMA GEMM, cluster LU, blocked triangular solves), each stage's
// DPT solve in the solver's own kernels; these kernels build the stage matrix,
// re-split the rotated matrix and normalise the final basis.  Row-major n x n,
// complex values interleaved (cx = 2) or real (cx = 1).
#include <cuda_runtime.h>
#include <stdint.h>

#include "dpt_device.cuh"
#include "dpt_kernels.h"

namespace dpt {

namespace {

constexpr int kHomThreads = 256;

unsigned grid_for(int64_t count) {
  int64_t b = (count + kHomThreads - 1) / kHomThreads;
  if (b > 148 * 16) b = 148 * 16;
  return unsigned(b < 1 ? 1 : b);
}

// Matrices are row-major n x n elements with a leading dimension of `ld`
// doubles (ld >= cx n, even: the GEMM's TMA rows need 16-byte strides).

// M = lam_s * Delta (every entry, `md[i] *= lam_s`), then M(i,i) += d_i (dpt.cpp:517-523)
__global__ void stage_matrix_kernel(const double* __restrict__ D, const double* __restrict__ d, double lr, double li,
                                    int cx, int64_t n, int64_t ld, double* __restrict__ M) {
  const int64_t nn = n * n;
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < nn; q += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = q / n, j = q % n, o = i * ld + cx * j;
    if (cx == 2) {
      cd v = cmul(cmake(D[o], D[o + 1]), cmake(lr, li));
      if (i == j) v = cadd(v, cmake(d[2 * i], d[2 * i + 1]));
      M[o] = v.x;
      M[o + 1] = v.y;
    } else {
      double v = __dmul_rn(D[o], lr);
      if (i == j) v = __dadd_rn(v, d[i]);
      M[o] = v;
    }
  }
}

// partition (partition.cpp:23-31): d = diag(R), Delta = R with a zero diagonal
// (Dp contiguous: the stage's dense problem)
__global__ void partition_kernel(const double* __restrict__ R, int64_t ld, double* __restrict__ dlev,
                                 double* __restrict__ Dp, int cx, int64_t n) {
  const int64_t nn = n * n;
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < nn; q += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = q / n, j = q % n;
    for (int c = 0; c < cx; ++c) {
      const double v = R[i * ld + cx * j + c];
      Dp[cx * q + c] = i == j ? 0.0 : v;
      if (i == j) dlev[cx * i + c] = v;
    }
  }
}

// a(i, m) = w(m, i) / w(i, i) (dpt.cpp:536-541), a contiguous; singular flags |w(i,i)| == 0
__global__ void normalise_kernel(const double* __restrict__ W, int64_t ld, double* __restrict__ a, int cx, int64_t n,
                                 unsigned* singular) {
  const int64_t nn = n * n;
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < nn; q += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = q / n, m = q % n;
    if (cx == 2) {
      const cd wii = cmake(W[i * ld + 2 * i], W[i * ld + 2 * i + 1]);
      if (cabs_(wii) == 0.0) {
        atomicOr(singular, 1u);
        continue;
      }
      const cd v = cdiv(cmake(W[m * ld + 2 * i], W[m * ld + 2 * i + 1]), wii);
      a[2 * q] = v.x;
      a[2 * q + 1] = v.y;
    } else {
      const double wii = W[i * ld + i];
      if (wii == 0.0) {
        atomicOr(singular, 1u);
        continue;
      }
      a[q] = __ddiv_rn(W[m * ld + i], wii);
    }
  }
}

__global__ void densify_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ cl,
                               const double* __restrict__ vl, int cx, int64_t n, int64_t ld, double* __restrict__ D) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p)
      for (int c = 0; c < cx; ++c) D[i * ld + cx * cl[p] + c] = vl[cx * p + c];
}

__global__ void identity_fill_kernel(double* __restrict__ W, int cx, int64_t n, int64_t ld) {
  const int64_t total = n * ld;
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < total; q += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = q / ld, c = q % ld;
    W[q] = (c == cx * i) ? 1.0 : 0.0;
  }
}

__global__ void nonfinite_kernel(const double* __restrict__ a, int64_t count, unsigned* bad) {
  unsigned b = 0;
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < count; q += int64_t(gridDim.x) * blockDim.x)
    b |= isfinite(a[q]) ? 0u : 1u;
  b = __reduce_or_sync(0xffffffffu, b);
  if ((threadIdx.x & 31) == 0 && b) atomicOr(bad, 1u);
}

}  // namespace

cudaError_t launch_hom_nonfinite(const double* a, int64_t count, unsigned* bad, cudaStream_t st) {
  nonfinite_kernel<<<grid_for(count), kHomThreads, 0, st>>>(a, count, bad);
  return cudaGetLastError();
}

cudaError_t launch_hom_stage_matrix(const double* D, const double* d, double lr, double li, int cx, int64_t n,
                                    int64_t ld, double* M, cudaStream_t st) {
  stage_matrix_kernel<<<grid_for(n * n), kHomThreads, 0, st>>>(D, d, lr, li, cx, n, ld, M);
  return cudaGetLastError();
}
cudaError_t launch_hom_partition(const double* R, int64_t ld, double* dlev, double* Dp, int cx, int64_t n,
                                 cudaStream_t st) {
  partition_kernel<<<grid_for(n * n), kHomThreads, 0, st>>>(R, ld, dlev, Dp, cx, n);
  return cudaGetLastError();
}
cudaError_t launch_hom_normalise(const double* W, int64_t ld, double* a, int cx, int64_t n, unsigned* singular,
                                 cudaStream_t st) {
  normalise_kernel<<<grid_for(n * n), kHomThreads, 0, st>>>(W, ld, a, cx, n, singular);
  return cudaGetLastError();
}
cudaError_t launch_hom_densify(const int64_t* rp, const int32_t* cl, const double* vl, int cx, int64_t n, int64_t ld,
                               double* D, cudaStream_t st) {
  densify_kernel<<<grid_for(n), kHomThreads, 0, st>>>(rp, cl, vl, cx, n, ld, D);
  return cudaGetLastError();
}
cudaError_t launch_hom_identity(double* W, int cx, int64_t n, int64_t ld, cudaStream_t st) {
  identity_fill_kernel<<<grid_for(n * ld), kHomThreads, 0, st>>>(W, cx, n, ld);
  return cudaGetLastError();
}

}  // namespace dpt
