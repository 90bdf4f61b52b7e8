// linalg.cu -- the dense linear algebra of the device homotopy_solve
// (proj/src/dpt.cpp:505-556: matmul(ms, w), solve_linear_multi(w, .),
// matmul(w, v); LU of proj/src/matrix.cpp:468-533) on the device, without
// libraries:
//
//  * gemm_nt: C = alpha A B^T + beta C (row-major FP64) on K1's machinery --
//    TMA (SWIZZLE_128B) staged k-tiles, mbarrier pipeline, DMMA.8x8x4 tiles
//    (dense_mma.cuh) -- with a plain epilogue.  Complex products run as the
//    real GEMM over interleaved (re, im) rows against a real image of B
//    (as K1 does for complex Delta).
//  * LU with partial pivoting, blocked right-looking: each column panel is
//    factored by ONE thread-block cluster of 8 CTAs whose shared memories hold
//    the panel (column-major, conflict-free); per column the CTAs find their
//    local pivot candidates, meet at a cluster barrier, read each other's
//    candidates and the pivot row through distributed shared memory, swap the
//    two rows by DSMEM, meet again, and eliminate their own rows.  The panel's
//    row swaps are then applied to the other columns, U12 = L11^-1 A12 is a
//    small triangular solve, and the trailing update A22 -= L21 U12 is gemm_nt.
//  * the n right-hand sides of R = W^-1 (M W) are permuted by the pivots and
//    solved with blocked forward / backward substitution whose off-diagonal
//    updates are again gemm_nt.
// The reference's rules are kept: the pivot of column k is the FIRST row of
// maximal |a(i,k)| (std::abs, i.e. hypot for complex), an exactly-zero pivot
// is "solve_linear: singular matrix", multipliers are a(i,k) / a(k,k).
#include <cooperative_groups.h>
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "dense_mma.cuh"
#include "dpt_device.cuh"
#include "dpt_kernels.h"

namespace cg = cooperative_groups;

namespace dpt {

namespace {

// ----------------------------------------------------------------- GEMM ----
template <class C>
__global__ void __launch_bounds__(C::THREADS, C::MINB)
    gemm_nt_kernel(const __grid_constant__ CUtensorMap am, const __grid_constant__ CUtensorMap bm, int64_t M,
                   int64_t N, int64_t K, double alpha, double beta, double* __restrict__ Cm, int64_t ldc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + C::STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tm = blockIdx.y, tn = blockIdx.x;
  const int KT = int((K + C::BK - 1) / C::BK);
  if (threadIdx.x == 0) {
    for (int i = 0; i < C::STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], C::NCW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const bool producer = threadIdx.x == 0;
  if (producer) {
    prefetch_tmap(&am);
    prefetch_tmap(&bm);
    const int pre = KT < C::STAGES ? KT : C::STAGES;
    for (int kt = 0; kt < pre; ++kt) {
      mbar_arrive_expect_tx(&full[kt], C::STAGE_BYTES);
      tma_load_2d(sA + kt * C::A_BYTES, &am, &full[kt], kt * C::BK, tm * C::BM);
      tma_load_2d(sB + kt * C::B_BYTES, &bm, &full[kt], kt * C::BK, tn * C::BN);
    }
  }
  const int wm = warp / C::WARPS_N, wn = warp % C::WARPS_N;
  const int t = lane & 3, gq = lane >> 2;
  double acc[C::MB][C::NB][2];
#pragma unroll
  for (int a = 0; a < C::MB; ++a)
#pragma unroll
    for (int b = 0; b < C::NB; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  for (int kt = 0; kt < KT; ++kt) {
    const int st = kt % C::STAGES;
    mbar_wait(&full[st], (kt / C::STAGES) & 1);
    dmma_consume_stage<C>(acc, sA + st * C::A_BYTES, sB + st * C::B_BYTES, wm, wn, t, gq);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
    if (producer && kt + C::STAGES < KT) {
      const int kn = kt + C::STAGES;
      mbar_wait(&empty[st], (kt / C::STAGES) & 1);
      fence_proxy_async_smem();  // the consumers' generic reads of the stage before the async-proxy refill
      mbar_arrive_expect_tx(&full[st], C::STAGE_BYTES);
      tma_load_2d(sA + st * C::A_BYTES, &am, &full[st], kn * C::BK, tm * C::BM);
      tma_load_2d(sB + st * C::B_BYTES, &bm, &full[st], kn * C::BK, tn * C::BN);
    }
    __syncwarp();
  }
#pragma unroll
  for (int a = 0; a < C::MB; ++a) {
    const int64_t i = int64_t(tm) * C::BM + wm * C::WTM + a * 8 + gq;
    if (i >= M) continue;
    double* crow = Cm + i * ldc;
#pragma unroll
    for (int b = 0; b < C::NB; ++b) {
      const int64_t j = int64_t(tn) * C::BN + wn * C::WTN + b * 8 + 2 * t;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        if (j + e >= N) continue;
        double v = __dmul_rn(alpha, acc[a][b][e]);
        if (beta != 0.0) v = __dadd_rn(v, __dmul_rn(beta, crow[j + e]));
        crow[j + e] = v;
      }
    }
  }
}

template <class C>
cudaError_t gemm_cfg(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B, int64_t ldb,
                     double alpha, double beta, double* Cm, int64_t ldc, cudaStream_t st) {
  CUtensorMap am, bm;
  if (make_tmap_rowmajor(&am, A, K, M, lda, C::BM) != 0 || make_tmap_rowmajor(&bm, B, K, N, ldb, C::BN) != 0)
    return cudaErrorInvalidValue;
  static DeviceAttrOnce attr;
  attr([] { cudaFuncSetAttribute(gemm_nt_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM); });
  const dim3 grid(unsigned((N + C::BN - 1) / C::BN), unsigned((M + C::BM - 1) / C::BM));
  gemm_nt_kernel<C><<<grid, C::THREADS, C::SMEM, st>>>(am, bm, M, N, K, alpha, beta, Cm, ldc);
  return cudaGetLastError();
}

// ------------------------------------------------------- element access ----
template <int CX>
__device__ __forceinline__ cd ld_e(const double* p, int64_t idx) {
  if constexpr (CX == 2) {
    const double2 v = *reinterpret_cast<const double2*>(p + 2 * idx);
    return cmake(v.x, v.y);
  } else {
    return cmake(p[idx], 0.0);
  }
}
template <int CX>
__device__ __forceinline__ void st_e(double* p, int64_t idx, cd v) {
  if constexpr (CX == 2) {
    *reinterpret_cast<double2*>(p + 2 * idx) = make_double2(v.x, v.y);
  } else {
    p[idx] = v.x;
  }
}
template <int CX>
__device__ __forceinline__ double mag(cd v) {
  if constexpr (CX == 2) return hypot(v.x, v.y);  // std::abs(complex)
  else return fabs(v.x);
}
template <int CX>
__device__ __forceinline__ cd e_div(cd a, cd b) {
  if constexpr (CX == 2) return cdiv(a, b);
  else return cmake(__ddiv_rn(a.x, b.x), 0.0);
}
template <int CX>
__device__ __forceinline__ cd e_fms(cd a, cd f, cd u) {  // a - f u (no contraction: the reference's order)
  if constexpr (CX == 2) return csub(a, cmul(f, u));
  else return cmake(__dsub_rn(a.x, __dmul_rn(f.x, u.x)), 0.0);
}

// ------------------------------------------------------------ LU panel ----
constexpr int kPanelCluster = 8;
constexpr int kPanelThreads = 512;
constexpr int kPanelMaxNb = 32;

// Rows [kb, n) x columns [kb, kb + nb) of A (element leading dim lde); CTA r of
// the cluster holds panel rows [r R, (r+1) R) in shared memory, element (i, c)
// at element index c * R + i (column-major: a column walk is conflict-free).
// piv[kb + j] = absolute pivot row of column kb + j; *info = min over the
// singular columns (1-based), untouched if none.
template <int CX>
__global__ void __launch_bounds__(kPanelThreads)
    lu_panel_kernel(double* __restrict__ A, int64_t lde, int64_t n, int64_t kb, int nb, int64_t R,
                    int64_t* __restrict__ piv, int* __restrict__ info, int64_t* __restrict__ swmap) {
  cg::cluster_group cl = cg::this_cluster();
  const int rank = int(cl.block_rank());
  extern __shared__ __align__(16) double sp[];
  __shared__ double cand_v;
  __shared__ int64_t cand_i;
  __shared__ double wv[kPanelThreads / 32];
  __shared__ int64_t wi[kPanelThreads / 32];
  __shared__ cd urow[kPanelMaxNb];
  __shared__ int64_t s_p;
  __shared__ int s_sing;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t m = n - kb;
  const int64_t r0 = int64_t(rank) * R;
  const int64_t rc = m - r0 < 0 ? 0 : (m - r0 < R ? m - r0 : R);
  for (int64_t q = tid; q < rc * nb; q += kPanelThreads) {
    const int64_t i = q / nb, c = q % nb;
    st_e<CX>(sp, c * R + i, ld_e<CX>(A, (kb + r0 + i) * lde + kb + c));
  }
  __syncthreads();
  for (int j = 0; j < nb; ++j) {
    // 1. local candidate: first row of maximal magnitude among panel rows >= j
    double best = -1.0;
    int64_t bi = INT64_MAX;
    for (int64_t i = tid; i < rc; i += kPanelThreads) {
      const int64_t pi = r0 + i;
      if (pi < j) continue;
      const double v = mag<CX>(ld_e<CX>(sp, int64_t(j) * R + i));
      if (v > best) best = v, bi = pi;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_down_sync(0xffffffffu, best, o);
      const int64_t oi = __shfl_down_sync(0xffffffffu, bi, o);
      if (ov > best || (ov == best && oi < bi)) best = ov, bi = oi;
    }
    if (lane == 0) wv[warp] = best, wi[warp] = bi;
    __syncthreads();
    if (warp == 0) {  // the block's candidate: one more shuffle tree over the warps' winners
      best = lane < kPanelThreads / 32 ? wv[lane] : -1.0;
      bi = lane < kPanelThreads / 32 ? wi[lane] : INT64_MAX;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_down_sync(0xffffffffu, best, o);
        const int64_t oi = __shfl_down_sync(0xffffffffu, bi, o);
        if (ov > best || (ov == best && oi < bi)) best = ov, bi = oi;
      }
      if (lane == 0) {
        cand_v = best;
        cand_i = bi;
      }
    }
    cl.sync();  // [A] every CTA's candidate is published
    if (warp == 0) {  // lanes read the cluster's candidates in parallel (DSMEM), then one tree
      const int nblk = int(cl.num_blocks());
      double gb = lane < nblk ? *cl.map_shared_rank(&cand_v, lane) : -1.0;
      int64_t gi = lane < nblk ? *cl.map_shared_rank(&cand_i, lane) : INT64_MAX;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_down_sync(0xffffffffu, gb, o);
        const int64_t oi = __shfl_down_sync(0xffffffffu, gi, o);
        if (ov > gb || (ov == gb && oi < gi)) gb = ov, gi = oi;
      }
      if (lane == 0) {
        s_p = gi;
        s_sing = !(gb > 0.0);  // exactly-zero column: lu_factor's singular test (matrix.cpp:485)
        if (s_sing && rank == 0) atomicMin(info, int(kb + j + 1));
        if (rank == 0) piv[kb + j] = kb + (s_sing ? j : gi);
      }
    }
    __syncthreads();
    const int64_t p = s_sing ? j : s_p;
    const int owner_j = int(j / R), owner_p = int(p / R);
    // 2. every CTA reads the pivot row (old row p); the owner of p also reads old row j
    cd oldj = cmake(0.0, 0.0);
    if (tid < nb) {
      const double* sp_p = cl.map_shared_rank(sp, owner_p);
      urow[tid] = ld_e<CX>(sp_p, int64_t(tid) * R + (p - int64_t(owner_p) * R));
      if (rank == owner_p && p != j) {
        const double* sp_j = cl.map_shared_rank(sp, owner_j);
        oldj = ld_e<CX>(sp_j, int64_t(tid) * R + (j - int64_t(owner_j) * R));
      }
    }
    cl.sync();  // [B] all remote reads of this column are done
    if (tid < nb && p != j) {
      if (rank == owner_j) st_e<CX>(sp, int64_t(tid) * R + (j - r0), urow[tid]);
      if (rank == owner_p) st_e<CX>(sp, int64_t(tid) * R + (p - r0), oldj);
    }
    __syncthreads();
    // 3. eliminate this CTA's rows below the pivot
    if (!s_sing) {
      const cd pv = urow[j];
      for (int64_t i = tid; i < rc; i += kPanelThreads) {
        if (r0 + i <= j) continue;
        const cd f = e_div<CX>(ld_e<CX>(sp, int64_t(j) * R + i), pv);
        st_e<CX>(sp, int64_t(j) * R + i, f);
        for (int c = j + 1; c < nb; ++c)
          st_e<CX>(sp, int64_t(c) * R + i, e_fms<CX>(ld_e<CX>(sp, int64_t(c) * R + i), f, urow[c]));
      }
    }
    __syncthreads();
  }
  for (int64_t q = tid; q < rc * nb; q += kPanelThreads) {
    const int64_t i = q / nb, c = q % nb;
    st_e<CX>(A, (kb + r0 + i) * lde + kb + c, ld_e<CX>(sp, c * R + i));
  }
  // The panel's interchanges as one permutation of the touched rows, for the
  // other columns (lu_swap_rest_kernel): swmap = {count, rows[], src[]}.
  // Warp 0 of rank 0 replays the swaps: positions kb .. kb+nb-1 are indexed
  // directly (cur), pivot rows below the panel live in a short list found by
  // one ballot per column.
  __shared__ int64_t cur[kPanelMaxNb], extpos[kPanelMaxNb], extval[kPanelMaxNb];
  if (rank == 0) {
    __syncthreads();  // piv[kb ..] was written by thread 0 of this block
    if (warp == 0) {
      if (lane < nb) cur[lane] = kb + lane;
      int next = 0;
      __syncwarp();
      for (int j = 0; j < nb; ++j) {
        const int64_t p = piv[kb + j];
        if (p < kb + nb) {
          if (lane == 0) {
            const int64_t t = cur[j];
            cur[j] = cur[p - kb];
            cur[p - kb] = t;
          }
        } else {
          const unsigned hit = __ballot_sync(0xffffffffu, lane < next && extpos[lane] == p);
          if (lane == 0) {
            int q = hit ? __ffs(hit) - 1 : next;
            if (!hit) {
              extpos[q] = p;
              extval[q] = p;
            }
            const int64_t t = cur[j];
            cur[j] = extval[q];
            extval[q] = t;
          }
          next += hit ? 0 : 1;
        }
        __syncwarp();
      }
      for (int q = lane; q < nb + next; q += 32) {
        swmap[1 + q] = q < nb ? kb + q : extpos[q - nb];
        swmap[1 + 2 * kPanelMaxNb + q] = q < nb ? cur[q] : extval[q - nb];
      }
      if (lane == 0) swmap[0] = nb + next;
    }
  }
  cl.sync();  // no CTA exits while a peer could still read its shared memory
}

// The panel's row interchanges applied to the columns outside it ([0, kb) and
// [kb + nb, n)): the composite permutation of the touched rows is rebuilt per
// block, the rows read into shared memory, then written to their targets.
constexpr int kSwapThreads = 64;
constexpr int64_t kSwapMapDoubles = 256;  // scratch head holding the panel's swap map (1 + 4 kPanelMaxNb)

template <int CX>
__global__ void __launch_bounds__(kSwapThreads)
    lu_swap_rest_kernel(double* __restrict__ A, int64_t lde, int64_t n, int64_t kb, int nb,
                        const int64_t* __restrict__ swmap) {
  __shared__ int64_t rows[2 * kPanelMaxNb], src[2 * kPanelMaxNb];
  extern __shared__ __align__(16) double buf[];  // [2 nb][kSwapThreads] elements
  const int cnt = int(swmap[0]);
  for (int q = threadIdx.x; q < cnt; q += blockDim.x) {
    rows[q] = swmap[1 + q];
    src[q] = swmap[1 + 2 * kPanelMaxNb + q];
  }
  __syncthreads();
  const int64_t rest = n - nb;  // columns outside the panel
  const int64_t q = int64_t(blockIdx.x) * kSwapThreads + threadIdx.x;
  if (q >= rest) return;
  const int64_t c = q < kb ? q : q + nb;
  for (int k = 0; k < cnt; ++k) st_e<CX>(buf, k * kSwapThreads + threadIdx.x, ld_e<CX>(A, src[k] * lde + c));
  for (int k = 0; k < cnt; ++k) st_e<CX>(A, rows[k] * lde + c, ld_e<CX>(buf, k * kSwapThreads + threadIdx.x));
}

// ---------------------------------------------------- triangular blocks ----
// X (nb rows at B + row0 * lde, columns [0, ncols)) <- T^-1 X, T the nb x nb
// diagonal block of the LU at (row0, row0): unit lower (LOWER) or upper.
// One thread per right-hand-side column, T in shared memory.
constexpr int kTrsmThreads = 128;

template <int CX, int NBT, bool LOWER>
__global__ void __launch_bounds__(kTrsmThreads)
    trsm_block_kernel(const double* __restrict__ LU, int64_t lde, int64_t row0, int nb, double* __restrict__ B,
                      int64_t ldb, int64_t c0, int64_t ncols) {
  __shared__ cd T[NBT * NBT];
  for (int q = threadIdx.x; q < nb * nb; q += kTrsmThreads) {
    const int r = q / nb, c = q % nb;
    T[r * NBT + c] = ld_e<CX>(LU, (row0 + r) * lde + row0 + c);
  }
  __syncthreads();
  const int64_t col = c0 + int64_t(blockIdx.x) * kTrsmThreads + threadIdx.x;
  if (col >= c0 + ncols) return;
  cd x[NBT];
#pragma unroll
  for (int r = 0; r < NBT; ++r)
    if (r < nb) x[r] = ld_e<CX>(B, (row0 + r) * ldb + col);
  if (LOWER) {
#pragma unroll
    for (int r = 0; r < NBT; ++r) {
      if (r >= nb) break;
#pragma unroll
      for (int q = 0; q < r; ++q) x[r] = e_fms<CX>(x[r], T[r * NBT + q], x[q]);  // lu_solve's forward order
    }
  } else {
#pragma unroll
    for (int r = NBT - 1; r >= 0; --r) {
      if (r >= nb) continue;
#pragma unroll
      for (int q = r + 1; q < NBT; ++q)
        if (q < nb) x[r] = e_fms<CX>(x[r], T[r * NBT + q], x[q]);
      x[r] = e_div<CX>(x[r], T[r * NBT + r]);
    }
  }
#pragma unroll
  for (int r = 0; r < NBT; ++r)
    if (r < nb) st_e<CX>(B, (row0 + r) * ldb + col, x[r]);
}

// ------------------------------------------------------ GEMM operands ----
// The B operand of gemm_nt for the product S-based right factor:
//  TRANS: B = S^T where S is rows x cols (elements); else B = S.
//  real: out[j][k] = B(j, k) (N x K); complex: the real image
//  out[2j][2k] = Re B, out[2j][2k+1] = -Im B, out[2j+1][2k] = Im B, out[2j+1][2k+1] = Re B.
template <int CX, bool TRANS>
__global__ void bop_kernel(const double* __restrict__ S, int64_t lds, int64_t N, int64_t K, double* __restrict__ out,
                           int64_t ldo) {
  const int64_t total = N * K;
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < total; q += int64_t(gridDim.x) * blockDim.x) {
    const int64_t j = TRANS ? q % N : q / K, k = TRANS ? q / N : q % K;  // TRANS: coalesced reads of S's rows
    const cd v = TRANS ? ld_e<CX>(S, k * lds + j) : ld_e<CX>(S, j * lds + k);
    if constexpr (CX == 2) {
      *reinterpret_cast<double2*>(out + (2 * j) * ldo + 2 * k) = make_double2(v.x, -v.y);
      *reinterpret_cast<double2*>(out + (2 * j + 1) * ldo + 2 * k) = make_double2(v.y, v.x);
    } else {
      out[j * ldo + k] = v.x;
    }
  }
}

__global__ void gather_rows_kernel(const double* __restrict__ src, int64_t ld, const int64_t* __restrict__ perm,
                                   int64_t n, int64_t width, double* __restrict__ dst) {
  const int64_t total = n * width;
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < total; q += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = q / width, c = q % width;
    dst[i * ld + c] = src[perm[i] * ld + c];
  }
}

unsigned grid_of(int64_t count, int threads) {
  int64_t b = (count + threads - 1) / threads;
  if (b > 148 * 32) b = 148 * 32;
  return unsigned(b < 1 ? 1 : b);
}

int64_t even(int64_t v) { return (v + 1) & ~int64_t(1); }

}  // namespace

// C[M x N] = alpha A[M x K] B[N x K]^T + beta C, row-major doubles (leading
// dims in doubles; A and B 16-byte aligned with even leading dims for TMA).
cudaError_t launch_gemm_nt(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B,
                           int64_t ldb, double alpha, double beta, double* Cm, int64_t ldc, cudaStream_t st) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  if (K <= 0) return cudaErrorInvalidValue;
  if ((lda & 1) || (ldb & 1) || (reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(B) & 15))
    return cudaErrorMisalignedAddress;
  // 128x64 tiles at two CTAs per SM once they fill the GPU, else 64x64
  if (((M + 127) / 128) * ((N + 63) / 64) >= 2 * 148)
    return gemm_cfg<CfgMid>(M, N, K, A, lda, B, ldb, alpha, beta, Cm, ldc, st);
  return gemm_cfg<CfgSmall8>(M, N, K, A, lda, B, ldb, alpha, beta, Cm, ldc, st);
}

// Operand for gemm_nt from S (element leading dim lds): B = S^T (trans) or S,
// N x K elements; out leading dim (doubles) ldo >= cx K, even.
cudaError_t launch_gemm_bop(int cx, bool trans, const double* S, int64_t lds, int64_t N, int64_t K, double* out,
                            int64_t ldo, cudaStream_t st) {
  const unsigned g = grid_of(N * K, 256);
  if (cx == 2)
    trans ? bop_kernel<2, true><<<g, 256, 0, st>>>(S, lds, N, K, out, ldo)
          : bop_kernel<2, false><<<g, 256, 0, st>>>(S, lds, N, K, out, ldo);
  else
    trans ? bop_kernel<1, true><<<g, 256, 0, st>>>(S, lds, N, K, out, ldo)
          : bop_kernel<1, false><<<g, 256, 0, st>>>(S, lds, N, K, out, ldo);
  return cudaGetLastError();
}

// Complex-aware product: C = alpha X Y^T-operand ... in elements.  C (M x N
// elements) = alpha A (M x K elements) * Bop^T + beta C, where Bop was built by
// launch_gemm_bop (N x K real or 2N x 2K image).  Leading dims in doubles.
static cudaError_t gemm_e(int cx, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* Bop,
                          int64_t ldbop, double alpha, double beta, double* Cm, int64_t ldc, cudaStream_t st) {
  return launch_gemm_nt(M, cx * N, cx * K, A, lda, Bop, ldbop, alpha, beta, Cm, ldc, st);
}

// Panel width for the cluster LU: the widest of 32 / 16 / 8 whose panel fits
// the cluster's shared memory (0: none does).
constexpr int64_t kPanelSmem = 200 * 1024;  // per CTA

static int panel_nb(int cx, int64_t n) {
  const int64_t R = (n + kPanelCluster - 1) / kPanelCluster;
  for (int nb = kPanelMaxNb; nb >= 8; nb /= 2)
    if (R * nb * 8 * cx <= kPanelSmem) return nb;
  return 0;
}

// Largest n the cluster panel holds (8-column panels).
int64_t lu_max_n(int cx) { return int64_t(kPanelCluster) * (kPanelSmem / (8 * 8 * cx)); }

template <int CX>
static cudaError_t lu_panel(double* A, int64_t lde, int64_t n, int64_t kb, int nb, int64_t* piv, int* info,
                            int64_t* swmap, cudaStream_t st) {
  const int64_t m = n - kb;
  // always the full cluster: fewer CTAs hold short panels too, but the
  // per-column elimination then runs on fewer SMs (measured slower)
  const int cs = kPanelCluster;
  const int64_t R = (m + cs - 1) / cs;
  const size_t smem = size_t(R) * size_t(nb) * 8 * CX;
  static DeviceAttrOnce attr;
  attr([] {
    cudaFuncSetAttribute(lu_panel_kernel<CX>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kPanelSmem));
  });
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs);
  cfg.blockDim = dim3(kPanelThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, lu_panel_kernel<CX>, A, lde, n, kb, nb, R, piv, info, swmap);
}

template <int CX>
static cudaError_t trsm_block(bool lower, const double* LU, int64_t lde, int64_t row0, int nb, double* B, int64_t ldb,
                              int64_t c0, int64_t ncols, cudaStream_t st) {
  const unsigned g = unsigned((ncols + kTrsmThreads - 1) / kTrsmThreads);
  if (g == 0) return cudaSuccess;
  if (lower)
    trsm_block_kernel<CX, kPanelMaxNb, true><<<g, kTrsmThreads, 0, st>>>(LU, lde, row0, nb, B, ldb, c0, ncols);
  else
    trsm_block_kernel<CX, kPanelMaxNb, false><<<g, kTrsmThreads, 0, st>>>(LU, lde, row0, nb, B, ldb, c0, ncols);
  return cudaGetLastError();
}

#define LA_CK(x)                          \
  do {                                    \
    const cudaError_t e_ = (x);           \
    if (e_ != cudaSuccess) return e_;     \
  } while (0)

// Two-level blocking: panels of nb <= 32 columns (the cluster kernel) inside
// outer blocks of kOuter columns.  Inside an outer block each panel's update
// only reaches the block's own columns (K = nb GEMMs on narrow strips); the
// columns right of the block get ONE update per outer block with K = kOuter,
// where the DMMA GEMM runs near its peak (a K = 32 update is bound by reading
// and writing C).
constexpr int kOuter = 128;

// B operand of the update "rows r0..r0+k of S (k x ncols elements at S, element
// ld lds) times ..." into the scratch operand area; returns its leading dim.
static int64_t bop_of_rows(int cx, const double* S, int64_t lds, int64_t ncols, int k, double* out, cudaStream_t st,
                           cudaError_t* e) {
  const int64_t ldo = even(cx * k);
  *e = launch_gemm_bop(cx, true, S, lds, ncols, k, out, ldo, st);
  return ldo;
}

// In-place LU with partial pivoting of the n x n matrix A (row-major, leading
// dim lda doubles, complex interleaved when cx = 2).  piv[k] = the row swapped
// with row k at step k (absolute); *info = first singular column + 1, or a
// large value.  scratch: >= 4 * n * kOuter + kSwapMapDoubles doubles.
cudaError_t launch_lu_factor(int cx, double* A, int64_t lda, int64_t n, int64_t* piv, int* info, double* scratch,
                             int* launches, cudaStream_t st) {
  const int nb = panel_nb(cx, n);
  if (nb == 0) return cudaErrorInvalidValue;
  const int outer = kOuter / nb * nb;
  const int64_t lde = lda / cx;  // element leading dim
  int64_t* swmap = reinterpret_cast<int64_t*>(scratch);  // {count, rows[64], src[64]}
  double* bop = scratch + kSwapMapDoubles;
  auto at = [&](int64_t r, int64_t c) { return A + (r * lde + c) * cx; };
  cudaError_t e = cudaSuccess;
  LA_CK(cudaMemsetAsync(info, 0x7f, sizeof(int), st));  // INT_MAX-ish: "none"
  for (int64_t ob = 0; ob < n; ob += outer) {
    const int64_t oe = ob + outer < n ? ob + outer : n;  // outer block columns [ob, oe)
    for (int64_t kb = ob; kb < oe; kb += nb) {
      const int w = int(oe - kb < nb ? oe - kb : nb);
      LA_CK(cx == 2 ? lu_panel<2>(A, lde, n, kb, w, piv, info, swmap, st)
                    : lu_panel<1>(A, lde, n, kb, w, piv, info, swmap, st));
      *launches += 1;
      const int64_t rest = n - w;
      if (rest > 0) {  // the panel's interchanges on every other column
        const unsigned g = unsigned((rest + kSwapThreads - 1) / kSwapThreads);
        const size_t sm = size_t(2 * w) * kSwapThreads * 8 * cx;
        static DeviceAttrOnce attr;
        attr([] {
          cudaFuncSetAttribute(lu_swap_rest_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
          cudaFuncSetAttribute(lu_swap_rest_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
        });
        if (cx == 2)
          lu_swap_rest_kernel<2><<<g, kSwapThreads, sm, st>>>(A, lde, n, kb, w, swmap);
        else
          lu_swap_rest_kernel<1><<<g, kSwapThreads, sm, st>>>(A, lde, n, kb, w, swmap);
        LA_CK(cudaGetLastError());
        *launches += 1;
      }
      // inside the outer block: U = L11^-1 A for its remaining columns, then
      // the rows below -= L21 U (K = w)
      const int64_t c0 = kb + w, wc = oe - c0;
      if (wc <= 0) continue;
      LA_CK(cx == 2 ? trsm_block<2>(true, A, lde, kb, w, A, lde, c0, wc, st)
                    : trsm_block<1>(true, A, lde, kb, w, A, lde, c0, wc, st));
      const int64_t ldo = bop_of_rows(cx, at(kb, c0), lde, wc, w, bop, st, &e);
      LA_CK(e);
      LA_CK(gemm_e(cx, n - c0, wc, w, at(c0, kb), lda, bop, ldo, -1.0, 1.0, at(c0, c0), lda, st));
      *launches += 3;
    }
    const int64_t c2 = oe, m2 = n - c2;
    if (m2 <= 0) continue;
    // right of the outer block: U12 = L11^-1 A12 (L11 = the block's unit lower
    // triangle, blocked by the panels), then the trailing A22 -= L21 U12 (K = outer)
    for (int64_t kb = ob; kb < oe; kb += nb) {
      const int w = int(oe - kb < nb ? oe - kb : nb);
      LA_CK(cx == 2 ? trsm_block<2>(true, A, lde, kb, w, A, lde, c2, m2, st)
                    : trsm_block<1>(true, A, lde, kb, w, A, lde, c2, m2, st));
      *launches += 1;
      const int64_t r1 = kb + w;
      if (r1 >= oe) continue;
      const int64_t ldo = bop_of_rows(cx, at(kb, c2), lde, m2, w, bop, st, &e);
      LA_CK(e);
      LA_CK(gemm_e(cx, oe - r1, m2, w, at(r1, kb), lda, bop, ldo, -1.0, 1.0, at(r1, c2), lda, st));
      *launches += 2;
    }
    const int64_t ldo = bop_of_rows(cx, at(ob, c2), lde, m2, int(oe - ob), bop, st, &e);
    LA_CK(e);
    LA_CK(gemm_e(cx, m2, m2, oe - ob, at(c2, ob), lda, bop, ldo, -1.0, 1.0, at(c2, c2), lda, st));
    *launches += 2;
  }
  return cudaSuccess;
}

// X <- U^-1 L^-1 X for the LU in A (after the caller permuted X's rows):
// nrhs columns; 32-row diagonal blocks (one thread per right-hand side),
// off-diagonal updates by gemm_nt -- within an outer block of kOuter rows with
// K = 32, beyond it once per outer block with K = kOuter.
// scratch: >= 4 * nrhs * kOuter doubles.
cudaError_t launch_lu_solve(int cx, const double* A, int64_t lda, int64_t n, double* X, int64_t ldx, int64_t nrhs,
                            double* scratch, int* launches, cudaStream_t st) {
  const int nb = kPanelMaxNb;
  const int64_t lde = lda / cx, ldxe = ldx / cx;
  auto at = [&](int64_t r, int64_t c) { return A + (r * lde + c) * cx; };
  cudaError_t e = cudaSuccess;
  for (int64_t ob = 0; ob < n; ob += kOuter) {  // forward: L Y = X (unit lower)
    const int64_t oe = ob + kOuter < n ? ob + kOuter : n;
    for (int64_t kb = ob; kb < oe; kb += nb) {
      const int w = int(oe - kb < nb ? oe - kb : nb);
      LA_CK(cx == 2 ? trsm_block<2>(true, A, lde, kb, w, X, ldxe, 0, nrhs, st)
                    : trsm_block<1>(true, A, lde, kb, w, X, ldxe, 0, nrhs, st));
      *launches += 1;
      const int64_t r1 = kb + w;
      if (r1 >= oe) continue;
      const int64_t ldo = bop_of_rows(cx, X + kb * ldx, ldxe, nrhs, w, scratch, st, &e);
      LA_CK(e);
      LA_CK(gemm_e(cx, oe - r1, nrhs, w, at(r1, kb), lda, scratch, ldo, -1.0, 1.0, X + r1 * ldx, ldx, st));
      *launches += 2;
    }
    if (oe >= n) continue;
    const int64_t ldo = bop_of_rows(cx, X + ob * ldx, ldxe, nrhs, int(oe - ob), scratch, st, &e);
    LA_CK(e);
    LA_CK(gemm_e(cx, n - oe, nrhs, oe - ob, at(oe, ob), lda, scratch, ldo, -1.0, 1.0, X + oe * ldx, ldx, st));
    *launches += 2;
  }
  const int64_t nob = (n + kOuter - 1) / kOuter;
  for (int64_t o = nob - 1; o >= 0; --o) {  // backward: U R = Y
    const int64_t ob = o * kOuter, oe = ob + kOuter < n ? ob + kOuter : n;
    const int64_t nblk = (oe - ob + nb - 1) / nb;
    for (int64_t b = nblk - 1; b >= 0; --b) {
      const int64_t kb = ob + b * nb;
      const int w = int(oe - kb < nb ? oe - kb : nb);
      LA_CK(cx == 2 ? trsm_block<2>(false, A, lde, kb, w, X, ldxe, 0, nrhs, st)
                    : trsm_block<1>(false, A, lde, kb, w, X, ldxe, 0, nrhs, st));
      *launches += 1;
      if (kb == ob) continue;
      const int64_t ldo = bop_of_rows(cx, X + kb * ldx, ldxe, nrhs, w, scratch, st, &e);
      LA_CK(e);
      LA_CK(gemm_e(cx, kb - ob, nrhs, w, at(ob, kb), lda, scratch, ldo, -1.0, 1.0, X + ob * ldx, ldx, st));
      *launches += 2;
    }
    if (ob == 0) continue;
    const int64_t ldo = bop_of_rows(cx, X + ob * ldx, ldxe, nrhs, int(oe - ob), scratch, st, &e);
    LA_CK(e);
    LA_CK(gemm_e(cx, ob, nrhs, oe - ob, at(0, ob), lda, scratch, ldo, -1.0, 1.0, X, ldx, st));
    *launches += 2;
  }
  return cudaSuccess;
}

cudaError_t launch_gather_rows(const double* src, int64_t ld, const int64_t* perm, int64_t n, int64_t width,
                               double* dst, cudaStream_t st) {
  gather_rows_kernel<<<grid_of(n * width, 256), 256, 0, st>>>(src, ld, perm, n, width, dst);
  return cudaGetLastError();
}

}  // namespace dpt
