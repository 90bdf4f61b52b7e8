// complex_steps.cu -- K2 and K3 for complex FP64 problems (std::complex<double>
// layout: interleaved re, im), the reference's native arithmetic
// (proj/include/dynspec/matrix.hpp:13).  Same data structures and schedule as
// the real kernels in sparse_step.cu; every product / abs / reciprocal follows
// the reference's std::complex semantics (dpt_device.cuh: cmul, cabs_, crecip).
//
//   csr_step_cplx_kernel   K2: full map with a CSR Delta (SELL-32 image with
//                          interleaved complex values), R rows of A per CTA in smem
//   single_cplx_kernel     K3: row map, MODE 1 = CSR thread per row,
//                          MODE 2 = dense Delta (real image B) warp per row
// (The dense full map needs no separate kernel: K1 runs the complex product as
// a real NT GEMM against B = [[Re D, -Im D], [Im D, Re D]], dense_step.cu.)
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "dpt_device.cuh"
#include "dpt_kernels.h"

namespace dpt {

constexpr int kCsrCThreads = 512;
constexpr int kCsrCSmemBudget = 200 * 1024;

static int csr_c_rows_per_cta(int64_t n) {
  int64_t r = kCsrCSmemBudget / (n * 16);
  if (r > 4) r = 4;
  if (const char* e = getenv("DPT_CSR_ROWS")) {  // tests: force fewer staged rows (0 = global gathers)
    const int64_t f = atoi(e);
    if (f >= 0 && f < r) r = f;
  }
  return int(r);
}

int csr_cplx_ntiles(int64_t rows, int64_t n) {
  const int R = csr_c_rows_per_cta(n) > 0 ? csr_c_rows_per_cta(n) : 1;
  return int((rows + R - 1) / R);
}

template <int R>
__global__ void __launch_bounds__(kCsrCThreads) csr_step_cplx_kernel(DevSolve s, DevSell S, int use_smem) {
  if (s.state->done) return;
  const int jl = launch_index(s);
  extern __shared__ __align__(16) double sa[];  // [R][2n] staged rows of A_{j-1}
  __shared__ unsigned long long next_slice;
  __shared__ double red[kCsrCThreads / 32][R][2];
  __shared__ double wred[kCsrCThreads / 32][3];
  const int64_t n = s.n, ld = s.ld, rows = s.rows;
  const int64_t il0 = int64_t(blockIdx.x) * R;
  const int nr = int(rows - il0 < R ? rows - il0 : R);
  const double* a_in = s.slots + size_t((jl - 1) % s.nslots) * size_t(s.slot_elems);
  double* a_out = s.slots + size_t(jl % s.nslots) * size_t(s.slot_elems);
  const cd lamk = lamc_of(s, jl), lamc = cmake(s.lambda, s.lambda_im);
  const double* d_in = s.dvec[(jl - 1) & 1];
  const double* arow[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int rr = r < nr ? r : 0;
    arow[r] = use_smem ? sa + size_t(rr) * size_t(2 * n) : a_in + size_t(il0 + rr) * size_t(ld);
  }
  if (threadIdx.x == 0) next_slice = 0ull;
  if (use_smem) {
    for (int r = 0; r < nr; ++r) {
      const double2* src = reinterpret_cast<const double2*>(a_in + size_t(il0 + r) * size_t(ld));
      double2* dst = reinterpret_cast<double2*>(sa + size_t(r) * size_t(2 * n));
      for (int64_t c = threadIdx.x; c < n; c += blockDim.x) dst[c] = src[c];
    }
  }
  __syncthreads();
  cd ti[R], di[R], epsi[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int rr = r < nr ? r : 0;
    const int64_t gi = s.row0 + il0 + rr;
    ti[r] = cmake(s.theta[2 * gi], s.theta[2 * gi + 1]);
    di[r] = cmake(d_in[2 * (il0 + rr)], d_in[2 * (il0 + rr) + 1]);
    epsi[r] = cadd(ti[r], cmul(lamc, di[r]));
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = kCsrCThreads / 32;
  double num[R], den[R];
#pragma unroll
  for (int r = 0; r < R; ++r) num[r] = den[r] = 0.0;
  double t_step = 0.0, t_max = 0.0, t_nonfin = 0.0;
  while (true) {
    int64_t sl = 0;
    if (lane == 0) sl = atomicAdd(&next_slice, 1);
    sl = __shfl_sync(0xffffffffu, sl, 0);
    if (sl >= S.nslices) break;
    const int64_t t = sl * 32 + lane;
    const int32_t j = S.lane_col[t];
    const int64_t off = S.slice_off[sl];
    const int32_t width = int32_t((S.slice_off[sl + 1] - off) >> 5);
    cd p[R];
#pragma unroll
    for (int r = 0; r < R; ++r) p[r] = cmake(0.0, 0.0);
    for (int32_t q = 0; q < width; ++q) {  // sequential CSR order in this lane; col -1 = bubble
      const int64_t idx = off + int64_t(q) * 32 + lane;
      const int32_t c = __ldg(S.cols + idx);
      if (c < 0) continue;
      const double2 v2 = __ldg(reinterpret_cast<const double2*>(S.vals) + idx);
      const cd v = cmake(v2.x, v2.y);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double2 a2 = *reinterpret_cast<const double2*>(arow[r] + 2 * c);
        p[r] = cadd(p[r], cmul(v, cmake(a2.x, a2.y)));
      }
    }
    if (j >= 0) {
      const cd tj = cmake(s.theta[2 * j], s.theta[2 * j + 1]);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (r >= nr) break;
        const int64_t gi = s.row0 + il0 + r;
        const double2 a2 = *reinterpret_cast<const double2*>(arow[r] + 2 * j);
        const cd aij = cmake(a2.x, a2.y);
        cd v;
        if (gi == j) {
          v = cmake(1.0, 0.0);
        } else {
          const cd g = s.gapmat ? cmake(s.gapmat[size_t(il0 + r) * size_t(ld) + size_t(2 * j)],
                                        s.gapmat[size_t(il0 + r) * size_t(ld) + size_t(2 * j) + 1])
                                : crecip(csub(ti[r], tj));
          v = cmul(cmul(lamk, g), csub(p[r], cmul(di[r], aij)));
        }
        *reinterpret_cast<double2*>(a_out + size_t(il0 + r) * size_t(ld) + size_t(2 * j)) = make_double2(v.x, v.y);
        t_step = fmax(t_step, cabs_(csub(v, aij)));
        t_max = fmax(t_max, cabs_(v));
        t_nonfin += cfinite(v) ? 0.0 : 1.0;
        const cd rr = cadd(cmul(csub(tj, epsi[r]), aij), cmul(lamc, p[r]));
        num[r] = fmax(num[r], cabs_(rr));
        den[r] = fmax(den[r], cabs_(aij));
      }
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const double a = warp_max(num[r]), b = warp_max(den[r]);
    if (lane == 0) {
      red[warp][r][0] = a;
      red[warp][r][1] = b;
    }
  }
  t_step = warp_max(t_step);
  t_max = warp_max(t_max);
  t_nonfin = warp_sum(t_nonfin);
  if (lane == 0) {
    wred[warp][0] = t_step;
    wred[warp][1] = t_max;
    wred[warp][2] = t_nonfin;
  }
  __syncthreads();
  if (warp < nr) {  // lagged diagonal of A': one warp per owned row
    const int r = warp;
    const int64_t il = il0 + r, gi = s.row0 + il;
    const int64_t t = S.pos_of[gi];
    const int L = int(t & 31);
    const int64_t off = S.slice_off[t >> 5];
    const int32_t width = int32_t((S.slice_off[(t >> 5) + 1] - off) >> 5);
    const double* arow_new = a_out + size_t(il) * size_t(ld);
    cd part = cmake(0.0, 0.0);
    for (int32_t q = lane; q < width; q += 32) {
      const int64_t idx = off + int64_t(q) * 32 + L;
      const int32_t c = __ldg(S.cols + idx);
      if (c < 0) continue;
      const double2 v2 = __ldg(reinterpret_cast<const double2*>(S.vals) + idx);
      part = cadd(part, cmul(cmake(v2.x, v2.y), cmake(arow_new[2 * c], arow_new[2 * c + 1])));
    }
    part.x = warp_sum(part.x);
    part.y = warp_sum(part.y);
    if (lane == 0) {
      double nu = 0.0, de = 0.0;
      for (int ww = 0; ww < NW; ++ww) {
        nu = fmax(nu, red[ww][r][0]);
        de = fmax(de, red[ww][r][1]);
      }
      s.rowpart[rp_index(0, il, 0, rows, 1)] = part.x;
      s.rowpart[rp_index(1, il, 0, rows, 1)] = nu;
      s.rowpart[rp_index(2, il, 0, rows, 1)] = de;
      s.rowpart[rp_index(3, il, 0, rows, 1)] = part.y;
    }
  }
  if (threadIdx.x == 0) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    for (int ww = 0; ww < NW; ++ww) {
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

cudaError_t launch_csr_step_cplx(const DevSolve& s, const DevSell& d, cudaStream_t st) {
  const int Rs = csr_c_rows_per_cta(s.n);
  const int use_smem = Rs > 0 ? 1 : 0;
  const int R = use_smem ? Rs : 1;
  const unsigned grid = unsigned((s.rows + R - 1) / R);
  const size_t smem = use_smem ? size_t(R) * size_t(s.n) * 16 : 0;
#define DPT_CSRC_CASE(RR)                                                                         \
  case RR: {                                                                                      \
    static DeviceAttrOnce attr;                                                                   \
    attr([] {                                                                                     \
      cudaFuncSetAttribute(csr_step_cplx_kernel<RR>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                           kCsrCSmemBudget + 1024);                                               \
    });                                                                                           \
    csr_step_cplx_kernel<RR><<<grid, kCsrCThreads, smem, st>>>(s, d, use_smem);                   \
    break;                                                                                        \
  }
  switch (R) {
    DPT_CSRC_CASE(1)
    DPT_CSRC_CASE(2)
    DPT_CSRC_CASE(3)
    DPT_CSRC_CASE(4)
    default:
      return cudaErrorInvalidValue;
  }
#undef DPT_CSRC_CASE
  return cudaGetLastError();
}

// ------------------------------------------------------------- row map ----
constexpr int kSingleCThreads = 256;

// w_m = (Delta z)_m in CSR order (MODE 1, one thread) or strided over a warp
// (MODE 2, dense: Delta(m,k) = (B[2m][2k], -B[2m][2k+1]) in the real image).
template <int MODE>
__device__ __forceinline__ cd row_dot_c(const DevCsr& D, const double* __restrict__ B, int64_t n, int64_t ldd,
                                        int64_t m, const double* __restrict__ z, int lane) {
  cd w = cmake(0.0, 0.0);
  if constexpr (MODE == 1) {
    for (int64_t q = D.rowptr[m]; q < D.rowptr[m + 1]; ++q) {
      const int32_t c = __ldg(D.cols + q);
      w = cadd(w, cmul(cmake(D.vals[2 * q], D.vals[2 * q + 1]), cmake(z[2 * c], z[2 * c + 1])));
    }
  } else {
    const double* br = B + size_t(2 * m) * size_t(ldd);
    for (int64_t c = lane; c < n; c += 32)
      w = cadd(w, cmul(cmake(br[2 * c], -br[2 * c + 1]), cmake(z[2 * c], z[2 * c + 1])));
    w.x = warp_sum(w.x);
    w.y = warp_sum(w.y);
  }
  return w;
}

template <int MODE>
__global__ void __launch_bounds__(kSingleCThreads)
    single_cplx_kernel(DevSolve s, DevCsr D, const double* __restrict__ B, int64_t row) {
  if (s.state->done) return;
  constexpr int G = MODE == 1 ? 1 : 32;
  constexpr int ROWS_PER_ITER = kSingleCThreads / G;
  const int jl = launch_index(s);
  __shared__ double wsh[2];
  __shared__ double red[kSingleCThreads / 32][5];
  const int64_t n = s.n;
  const double* __restrict__ z = s.slots + size_t((jl - 1) % s.nslots) * size_t(s.slot_elems);
  double* __restrict__ zo = s.slots + size_t(jl % s.nslots) * size_t(s.slot_elems);
  const cd lamk = lamc_of(s, jl), lamc = cmake(s.lambda, s.lambda_im);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp == 0) {
    const cd wr = (MODE == 1 && lane != 0) ? cmake(0.0, 0.0) : row_dot_c<MODE>(D, B, n, s.ldd, row, z, lane);
    if (lane == 0) {
      wsh[0] = wr.x;
      wsh[1] = wr.y;
      if (blockIdx.x == 0) {
        s.dvec[(jl - 1) & 1][0] = wr.x;  // w[row] of z_{j-1} for the fold's eps
        s.dvec[(jl - 1) & 1][1] = wr.y;
      }
    }
  }
  __syncthreads();
  const cd wr = cmake(wsh[0], wsh[1]);
  const cd trow = cmake(s.theta[2 * row], s.theta[2 * row + 1]);
  const cd eps = cadd(trow, cmul(lamc, wr));
  double num = 0.0, den = 0.0, t_step = 0.0, t_max = 0.0, t_nonfin = 0.0;
  const int64_t stride = int64_t(gridDim.x) * ROWS_PER_ITER;
  for (int64_t m0 = int64_t(blockIdx.x) * ROWS_PER_ITER; m0 < n; m0 += stride) {
    const int64_t m = m0 + threadIdx.x / G;
    const cd w = row_dot_c<MODE>(D, B, n, s.ldd, m < n ? m : n - 1, z, lane);
    if (m < n && (MODE == 1 || lane == 0)) {
      const cd zm = cmake(z[2 * m], z[2 * m + 1]);
      const cd tm = cmake(s.theta[2 * m], s.theta[2 * m + 1]);
      cd v;
      if (m == row) {
        v = cmake(1.0, 0.0);
      } else {
        const cd g = s.gapmat ? cmake(s.gapmat[2 * m], s.gapmat[2 * m + 1]) : crecip(csub(trow, tm));
        v = cmul(cmul(lamk, g), csub(w, cmul(wr, zm)));
      }
      zo[2 * m] = v.x;
      zo[2 * m + 1] = v.y;
      t_step = fmax(t_step, cabs_(csub(v, zm)));
      t_max = fmax(t_max, cabs_(v));
      t_nonfin += cfinite(v) ? 0.0 : 1.0;
      const cd r = cadd(cmul(csub(tm, eps), zm), cmul(lamc, w));
      num = fmax(num, cabs_(r));
      den = fmax(den, cabs_(zm));
    }
  }
  num = warp_max(num);
  den = warp_max(den);
  t_step = warp_max(t_step);
  t_max = warp_max(t_max);
  t_nonfin = warp_sum(t_nonfin);
  if (lane == 0) {
    red[warp][0] = num;
    red[warp][1] = den;
    red[warp][2] = t_step;
    red[warp][3] = t_max;
    red[warp][4] = t_nonfin;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a[5] = {0, 0, 0, 0, 0};
    for (int ww = 0; ww < kSingleCThreads / 32; ++ww) {
      a[0] = fmax(a[0], red[ww][0]);
      a[1] = fmax(a[1], red[ww][1]);
      a[2] = fmax(a[2], red[ww][2]);
      a[3] = fmax(a[3], red[ww][3]);
      a[4] += red[ww][4];
    }
    const int tn = blockIdx.x, ntn = s.ntn;
    s.rowpart[rp_index(0, 0, tn, 1, ntn)] = 0.0;
    s.rowpart[rp_index(1, 0, tn, 1, ntn)] = a[0];
    s.rowpart[rp_index(2, 0, tn, 1, ntn)] = a[1];
    s.rowpart[rp_index(3, 0, tn, 1, ntn)] = 0.0;
    double* tp = s.tilepart + size_t(tn) * 4;
    tp[0] = a[2];
    tp[1] = a[3];
    tp[2] = a[4];
    tp[3] = 0.0;
  }
}

// ---------------------------------------- complex row map, 16 per row ----
// Complex CSR with exactly 16 nonzeros per row (c4 with complex data): the
// per-warp pipeline of the real K3 (single_u16.cu) over a trip-major copy of
// the CSR built once per problem (u16c_build_kernel): for 32-row trip t,
// columns at cols_t[t][q/4][lane][4] and values at vals_t[t][q][lane] (one
// complex each), so every stage read is a conflict-free 16-byte LDS and lane L
// still owns row 32 t + L with its entries in CSR order q = 0..15 -- the same
// complex products and sums, in the same order, as row_dot_c (bit-identical to
// the general kernel, and to the w[row] each warp evaluates from the CSR).
constexpr int kU16cWarps = 8;  // measured: 10 warps (100 KB of stages) 0.111 ms vs 0.108 ms
constexpr int kU16cTripBytes = 32 * 16 * 4 + 32 * 16 * 16;  // columns 2 KiB + values 8 KiB
static_assert(kU16cTripBytes == 10240, "trip layout");

__global__ void u16c_build_kernel(const int32_t* __restrict__ cols, const double* __restrict__ vals, int64_t n,
                                  int32_t* __restrict__ ct, double* __restrict__ vt) {
  const int64_t total = n * 16;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t m = e >> 4, q = e & 15, t = m >> 5, L = m & 31;
    ct[t * 512 + (q >> 2) * 128 + L * 4 + (q & 3)] = cols[e];
    const int64_t d = t * 512 + q * 32 + L;
    vt[2 * d] = vals[2 * e];
    vt[2 * d + 1] = vals[2 * e + 1];
  }
}

cudaError_t launch_u16c_build(const int32_t* cols, const double* vals, int64_t n, int32_t* ct, double* vt,
                              cudaStream_t st) {
  const int64_t blocks = (n * 16 + 255) / 256;
  u16c_build_kernel<<<unsigned(blocks < 148 * 16 ? (blocks > 0 ? blocks : 1) : 148 * 16), 256, 0, st>>>(cols, vals, n,
                                                                                                     ct, vt);
  return cudaGetLastError();
}

__global__ void __launch_bounds__(kU16cWarps * 32, 1)
    single_cplx_u16w_kernel(DevSolve s, DevCsr D, const int32_t* __restrict__ ct, const double* __restrict__ vt,
                            int64_t row, int64_t ntrips) {
  if (s.state->done) return;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t bar[kU16cWarps];    // full: the trip landed
  __shared__ uint64_t empty[kU16cWarps];  // empty: all 32 lanes hold the trip in registers
  __shared__ double red[kU16cWarps][5];
  const int jl = launch_index(s);
  const int64_t n = s.n;
  const double* __restrict__ z = s.slots + size_t((jl - 1) % s.nslots) * size_t(s.slot_elems);
  double* __restrict__ zo = s.slots + size_t(jl % s.nslots) * size_t(s.slot_elems);
  const cd lamk = lamc_of(s, jl), lamc = cmake(s.lambda, s.lambda_im);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint8_t* stage = smem + size_t(warp) * kU16cTripBytes;
  const int64_t stride = int64_t(gridDim.x) * kU16cWarps;
  int64_t t = int64_t(blockIdx.x) * kU16cWarps + warp;
  auto issue = [&](int64_t trip) {
    const int64_t nr = (n - trip * 32) < 32 ? (n - trip * 32) : 32;
    // a partial last trip is still laid out with 32 lanes (rows >= n absent):
    // copy the whole trip slab the build wrote (cols / vals beyond the rows are
    // never read)
    (void)nr;
    mbar_arrive_expect_tx(&bar[warp], uint32_t(kU16cTripBytes));
    bulk_load(stage, ct + trip * 512, 2048u, &bar[warp]);
    bulk_load(stage + 2048, vt + trip * 1024, 8192u, &bar[warp]);
  };
  if (lane == 0) {
    mbar_init(&bar[warp], 1);
    mbar_init(&empty[warp], 32);
    fence_mbar_init();
    if (t < ntrips) issue(t);
  }
  __syncwarp();
  const cd wr = row_dot_c<1>(D, nullptr, n, 0, row, z, 0);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    s.dvec[(jl - 1) & 1][0] = wr.x;  // w[row] of z_{j-1} for the fold's eps
    s.dvec[(jl - 1) & 1][1] = wr.y;
  }
  const cd trow = cmake(s.theta[2 * row], s.theta[2 * row + 1]);
  const cd eps = cadd(trow, cmul(lamc, wr));
  double num = 0.0, den = 0.0, t_step = 0.0, t_max = 0.0, t_nonfin = 0.0;
  for (int it = 0; t < ntrips; ++it, t += stride) {
    mbar_wait(&bar[warp], uint32_t(it) & 1u);
    const int64_t m = t * 32 + lane;
    int4 c4[4];
    double2 v[16];
    const int4* cs = reinterpret_cast<const int4*>(stage) + lane;
    const double2* vs = reinterpret_cast<const double2*>(stage + 2048) + lane;
#pragma unroll
    for (int k = 0; k < 4; ++k) c4[k] = cs[k * 32];
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = vs[q * 32];
    // WAR handshake (as single_u16w_kernel): release after the reads, lane 0
    // acquires the phase and fences generic -> async proxy before the refill
    mbar_arrive_release(&empty[warp]);
    if (lane == 0 && t + stride < ntrips) {
      mbar_wait(&empty[warp], uint32_t(it) & 1u);
      fence_proxy_async_smem();
      issue(t + stride);
    }
    if (m < n) {
      const cd zm = cmake(z[2 * m], z[2 * m + 1]);
      const cd tm = cmake(s.theta[2 * m], s.theta[2 * m + 1]);
      const int32_t c[16] = {c4[0].x, c4[0].y, c4[0].z, c4[0].w, c4[1].x, c4[1].y, c4[1].z, c4[1].w,
                             c4[2].x, c4[2].y, c4[2].z, c4[2].w, c4[3].x, c4[3].y, c4[3].z, c4[3].w};
      double2 zg[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) zg[q] = *reinterpret_cast<const double2*>(z + 2 * size_t(c[q]));
      cd w = cmake(0.0, 0.0);
#pragma unroll
      for (int q = 0; q < 16; ++q) w = cadd(w, cmul(cmake(v[q].x, v[q].y), cmake(zg[q].x, zg[q].y)));
      cd val;
      if (m == row) {
        val = cmake(1.0, 0.0);
      } else {
        const cd g = s.gapmat ? cmake(s.gapmat[2 * m], s.gapmat[2 * m + 1]) : crecip(csub(trow, tm));
        val = cmul(cmul(lamk, g), csub(w, cmul(wr, zm)));
      }
      zo[2 * m] = val.x;
      zo[2 * m + 1] = val.y;
      t_step = fmax(t_step, cabs_(csub(val, zm)));
      t_max = fmax(t_max, cabs_(val));
      t_nonfin += cfinite(val) ? 0.0 : 1.0;
      const cd r = cadd(cmul(csub(tm, eps), zm), cmul(lamc, w));
      num = fmax(num, cabs_(r));
      den = fmax(den, cabs_(zm));
    }
  }
  num = warp_max(num);
  den = warp_max(den);
  t_step = warp_max(t_step);
  t_max = warp_max(t_max);
  t_nonfin = warp_sum(t_nonfin);
  if (lane == 0) {
    red[warp][0] = num;
    red[warp][1] = den;
    red[warp][2] = t_step;
    red[warp][3] = t_max;
    red[warp][4] = t_nonfin;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a[5] = {0, 0, 0, 0, 0};
    for (int ww = 0; ww < kU16cWarps; ++ww) {
      a[0] = fmax(a[0], red[ww][0]);
      a[1] = fmax(a[1], red[ww][1]);
      a[2] = fmax(a[2], red[ww][2]);
      a[3] = fmax(a[3], red[ww][3]);
      a[4] += red[ww][4];
    }
    const int tn = blockIdx.x, ntn = s.ntn;
    s.rowpart[rp_index(0, 0, tn, 1, ntn)] = 0.0;
    s.rowpart[rp_index(1, 0, tn, 1, ntn)] = a[0];
    s.rowpart[rp_index(2, 0, tn, 1, ntn)] = a[1];
    s.rowpart[rp_index(3, 0, tn, 1, ntn)] = 0.0;
    double* tp = s.tilepart + size_t(tn) * 4;
    tp[0] = a[2];
    tp[1] = a[3];
    tp[2] = a[4];
    tp[3] = 0.0;
  }
}

static bool u16c_enabled() {
  const char* e = getenv("DPT_CPLX_U16");
  return !(e && e[0] == '0');
}

int single_cplx_u16_grid(int64_t n) {
  const int64_t trips = (n + 31) / 32;
  const int64_t blocks = (trips + kU16cWarps - 1) / kU16cWarps;
  return int(blocks < 148 ? (blocks > 0 ? blocks : 1) : 148);
}

int single_cplx_ntiles(int64_t n, int dense, int u16) {
  if (u16 && !dense && u16c_enabled()) return single_cplx_u16_grid(n);
  const int rows_per_iter = kSingleCThreads / (dense ? 32 : 1);
  int64_t b = (n + rows_per_iter - 1) / rows_per_iter;
  if (b > 148 * 8) b = 148 * 8;
  return int(b < 1 ? 1 : b);
}

cudaError_t launch_single_cplx(const DevSolve& s, const DevCsr& d, const double* B, const int32_t* u16c_cols,
                               const double* u16c_vals, int64_t row, cudaStream_t st) {
  if (!B && u16c_cols && u16c_enabled()) {
    constexpr int smem = kU16cWarps * kU16cTripBytes;
    static DeviceAttrOnce attr;
    attr([] { cudaFuncSetAttribute(single_cplx_u16w_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); });
    single_cplx_u16w_kernel<<<single_cplx_u16_grid(s.n), kU16cWarps * 32, smem, st>>>(s, d, u16c_cols, u16c_vals, row,
                                                                                       (s.n + 31) / 32);
    return cudaGetLastError();
  }
  const unsigned grid = unsigned(single_cplx_ntiles(s.n, B != nullptr, 0));
  if (B)
    single_cplx_kernel<2><<<grid, kSingleCThreads, 0, st>>>(s, d, B, row);
  else
    single_cplx_kernel<1><<<grid, kSingleCThreads, 0, st>>>(s, d, B, row);
  return cudaGetLastError();
}

}  // namespace dpt
