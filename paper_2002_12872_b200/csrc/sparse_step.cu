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
#include <stdlib.h>

#include "dpt_device.cuh"
#include "dpt_kernels.h"

namespace dpt {

constexpr int kCsrThreads = 1024;
constexpr int kCsrSmemBudget = 200 * 1024;

constexpr int csr_stride(int R) { return (R & 1) ? R : R + 1; }

// Rows of A staged per CTA from the shared-memory budget (0 = rows too long:
// gathers from global memory).  Independent of DPT_CSR_ROWS, so the SELL image
// (and with it every accumulation order) is the same for every staging variant.
static int csr_rows_natural(int64_t n) {
  int64_t r = kCsrSmemBudget / (n * 8);
  if (r > 8) r = 8;
  if (r >= 2 && (r & 1) == 0 && (r + 1) * n * 8 > kCsrSmemBudget) --r;  // odd stride must fit (csr_stride)
  return int(r);
}

static int csr_rows_per_cta(int64_t n) {
  int r = csr_rows_natural(n);
  if (const char* e = getenv("DPT_CSR_ROWS")) {  // tests: force fewer staged rows (0 = global gathers)
    const int f = atoi(e);
    if (f >= 0 && f < r) r = f;
  }
  if (r >= 2 && (r & 1) == 0 && (r + 1) * n * 8 > kCsrSmemBudget) --r;
  return r;
}

int csr_staged_cols_max(int64_t n) {
  const int r = csr_rows_natural(n);
  return r > 0 ? int(kCsrSmemBudget / (8 * csr_stride(r))) : 0;
}

int csr_ntn(int64_t) { return 1; }

int csr_step_ntiles(int64_t rows, int64_t n) {
  const int R = csr_rows_per_cta(n) > 0 ? csr_rows_per_cta(n) : 1;
  return int((rows + R - 1) / R);
}

// K2 works on a SELL-32 image of Delta built once per problem on the device
// (sell_build.cu, driven by build_sell_device in solver.cu): rows of Delta are
// grouped 32 to a slice (after a by-length sort inside windows of 256 rows, so
// slices have little padding), and entry q of slice lane L is stored at
// slice_off + 32 q + L (values; the shared-memory kernel reads the columns
// from the packed 16-bit copy, four steps per 8-byte load).  A warp takes one
// slice, lane L owns one output column j of P (one row of Delta): every image
// load is coalesced, the dot P(i, j) = sum_q val * A(i, col) accumulates
// sequentially in the schedule's order in one lane (no shuffle trees).  The next launch's diagonal d(i) = P(A')(i,i) is
// formed at the end by one warp per owned row (lagged, like K1).
//
// Shared-memory layout: the R staged rows are interleaved, element (k, r) at
// sa[k * S + r] with an odd stride S = R | 1, so the R gathers of one entry
// share one address computation (immediate offsets) and the bank of (k, r) is
// a bijection of k mod 16 -- the bank-aware SELL schedule (build_sell) then
// makes every half-warp's gathers conflict-free for every r.  Bubble entries
// (col -1, value 0) load nothing and add fma(0, 0, p) = p exactly (p starts at
// +0 and a sum never turns into -0), so the FMA chain needs no guard.
// SMEM = false (rows too long for shared memory) gathers from global instead.
constexpr int kCsrU = 4;  // entries in flight per lane; slice widths are padded to a multiple

template <int R, bool SMEM, int THREADS = kCsrThreads>
__global__ void __launch_bounds__(THREADS) csr_step_kernel(DevSolve s, DevSell S) {
  constexpr int ST = csr_stride(R);
  if (s.state->done) return;
  const int jl = launch_index(s);
  extern __shared__ __align__(16) double sa[];  // [n][ST] staged rows of A_{j-1}
  __shared__ unsigned int next_slice;  // 32-bit: one ATOMS.ADD (a 64-bit shared atomicAdd is a CAS loop)
  __shared__ double red[THREADS / 32][R][2];
  __shared__ double wred[THREADS / 32][3];
  const int64_t n = s.n, ld = s.ld, rows = s.rows;
  const int64_t il0 = int64_t(blockIdx.x) * R;
  const int nr = int(rows - il0 < R ? rows - il0 : R);
  const int slot_in = (jl - 1) % s.nslots, slot_out = jl % s.nslots;
  const double* a_in = s.slots + size_t(slot_in) * size_t(s.slot_elems);
  double* a_out = s.slots + size_t(slot_out) * size_t(s.slot_elems);
  const double lam_k = lam_of(s, jl), lam = s.lambda;
  const double* d_in = s.dvec[(jl - 1) & 1];
  const double* __restrict__ ain = a_in + size_t(il0) * size_t(ld);  // SMEM = false: row r at ain + r * ld

  if (threadIdx.x == 0) next_slice = 0u;
  // Staged rows are indexed by POSITION: the image's columns are positions
  // (S.perm[k] when the columns were relabelled for bank balance, else k).
  const int32_t* __restrict__ perm = S.perm;
  const int32_t* __restrict__ inv = S.inv;
  if constexpr (SMEM) {
    // all R rows of a column chunk are loaded before any is stored: R * kStageU
    // independent loads in flight per thread (the loop is HBM-latency bound).
    // (Filling by position instead -- conflict-free stores, reads through inv --
    // was measured: the relabelled columns of 32 consecutive positions spread
    // over ~12 lines, 17 M more global wavefronts for 8.5 M fewer shared ones.)
    constexpr int kStageU = R <= 3 ? 4 : 2;
    for (int64_t c0 = threadIdx.x; c0 < n; c0 += kStageU * int64_t(blockDim.x)) {
      double v[kStageU][R];
      int64_t p[kStageU];
#pragma unroll
      for (int u = 0; u < kStageU; ++u) {
        const int64_t c = c0 + int64_t(u) * blockDim.x;
        p[u] = c < n ? (perm ? int64_t(__ldg(perm + c)) : c) : -1;
#pragma unroll
        for (int r = 0; r < R; ++r)
          if (c < n && r < nr) v[u][r] = ain[size_t(r) * size_t(ld) + size_t(c)];
      }
#pragma unroll
      for (int u = 0; u < kStageU; ++u)
#pragma unroll
        for (int r = 0; r < R; ++r)
          if (p[u] >= 0 && r < nr) sa[size_t(p[u]) * ST + r] = v[u][r];
    }
  }
  __syncthreads();
  // 32-bit shared address of the staged rows, kept in a register: left to
  // itself ptxas rematerialises it at every gather (S2R SR_CgaCtaId + LEA)
  uint32_t sab = smem_u32(sa);
  asm volatile("mov.u32 %0, %0;" : "+r"(sab));
  auto A = [&](int r, int64_t p) -> double {  // element at position p of staged row r
    if constexpr (SMEM) return lds64(sab + uint32_t(p) * uint32_t(ST * 8) + uint32_t(r * 8));
    else return ain[size_t(r < nr ? r : 0) * size_t(ld) + size_t(inv ? int64_t(__ldg(inv + p)) : p)];
  };
  // per-row constants of the staged rows live in shared memory (registers go
  // to the image prefetch below)
  __shared__ double rowc[3][R];  // theta_i, d_{j-1}(i), eps_i
  if (threadIdx.x < R) {
    const int rr = int(threadIdx.x) < nr ? int(threadIdx.x) : 0;
    const double ti = s.theta[s.row0 + il0 + rr], di = d_in[il0 + rr];
    rowc[0][threadIdx.x] = ti;
    rowc[1][threadIdx.x] = di;
    rowc[2][threadIdx.x] = __dadd_rn(ti, __dmul_rn(lam, di));
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = THREADS / 32;
  double num[R], den[R];
#pragma unroll
  for (int r = 0; r < R; ++r) num[r] = den[r] = 0.0;
  double t_step = 0.0, t_max = 0.0, t_nonfin = 0.0;

  // Slices differ in width (sorted windows), so warps take them dynamically
  // from a shared counter instead of a fixed stride (which pinned the widest
  // slice of every window on the same warps).  The result does not depend on
  // which warp computes a column.
  while (true) {
    int64_t sl = 0;
    if (lane == 0) sl = int64_t(atomicAdd(&next_slice, 1u));
    sl = __shfl_sync(0xffffffffu, sl, 0);
    if (sl >= S.nslices) break;
    const int64_t t = sl * 32 + lane;
    const int32_t j = S.lane_col[t];
    const int64_t off = S.slice_off[sl];
    const int32_t width = int32_t((S.slice_off[sl + 1] - off) >> 5);  // multiple of kCsrU
    const double* __restrict__ sv = S.vals + off + lane;
    double p[R];
#pragma unroll
    for (int r = 0; r < R; ++r) p[r] = 0.0;
    if constexpr (SMEM) {
      // packed image (launch_sell_pack): the four 16-bit positions of a trip in
      // one 8-byte load per lane; 0xffff = bubble
      static_assert(kCsrU == 4, "the packed image holds four steps per trip");
      const uint2* __restrict__ sc16 = reinterpret_cast<const uint2*>(S.cols16) + (off >> 2) + lane;
      for (int32_t q0 = 0; q0 < width; q0 += kCsrU) {
        const uint2 cc = __ldg(sc16 + (q0 >> 2) * 32);
        uint32_t c[kCsrU] = {cc.x & 0xffffu, cc.x >> 16, cc.y & 0xffffu, cc.y >> 16};
        double v[kCsrU];
#pragma unroll
        for (int u = 0; u < kCsrU; ++u) v[u] = __ldg(sv + (q0 + u) * 32);
        double g[kCsrU][R];
#pragma unroll
        for (int u = 0; u < kCsrU; ++u)
#pragma unroll
          for (int r = 0; r < R; ++r) g[u][r] = c[u] != 0xffffu ? A(r, c[u]) : 0.0;  // bubbles issue no load
#pragma unroll
        for (int u = 0; u < kCsrU; ++u)
#pragma unroll
          for (int r = 0; r < R; ++r) p[r] = __fma_rn(v[u], g[u][r], p[r]);
      }
    } else {
      const int32_t* __restrict__ sc = S.cols + off + lane;
      for (int32_t q0 = 0; q0 < width; q0 += kCsrU) {
        int32_t c[kCsrU];
        double v[kCsrU];
#pragma unroll
        for (int u = 0; u < kCsrU; ++u) {
          c[u] = __ldg(sc + (q0 + u) * 32);
          v[u] = __ldg(sv + (q0 + u) * 32);
        }
        double g[kCsrU][R];
#pragma unroll
        for (int u = 0; u < kCsrU; ++u)
#pragma unroll
          for (int r = 0; r < R; ++r) g[u][r] = c[u] >= 0 ? A(r, c[u]) : 0.0;  // bubbles issue no load
#pragma unroll
        for (int u = 0; u < kCsrU; ++u)
#pragma unroll
          for (int r = 0; r < R; ++r) p[r] = __fma_rn(v[u], g[u][r], p[r]);
      }
    }
    if (j >= 0) {
      // the lane's own column: level and position, in slice order when packed
      const double tj = SMEM ? __ldg(S.lane_theta + t) : s.theta[j];
      const int64_t pj = SMEM ? int64_t(__ldg(S.lane_pos + t)) : (perm ? int64_t(__ldg(perm + j)) : j);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (r >= nr) break;
        const int64_t gi = s.row0 + il0 + r;
        const double aij = A(r, pj);
        double val;
        if (gi == j) {
          val = 1.0;
        } else {
          const double gg = s.gapmat ? s.gapmat[size_t(il0 + r) * size_t(ld) + size_t(j)] : 1.0 / __dsub_rn(rowc[0][r], tj);
          val = __dmul_rn(__dmul_rn(lam_k, gg), __dsub_rn(p[r], __dmul_rn(rowc[1][r], aij)));
        }
        a_out[size_t(il0 + r) * size_t(ld) + size_t(j)] = val;
        t_step = fmax(t_step, fabs(__dsub_rn(val, aij)));
        t_max = fmax(t_max, fabs(val));
        t_nonfin += isfinite(val) ? 0.0 : 1.0;
        const double rr = __dadd_rn(__dmul_rn(__dsub_rn(tj, rowc[2][r]), aij), __dmul_rn(lam, p[r]));
        num[r] = fmax(num[r], fabs(rr));
        den[r] = fmax(den[r], fabs(aij));
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
  __syncthreads();  // also orders this CTA's A' stores before the d' dots below
  // d_j(i) = P(A_j)(i,i) for the next launch (lagged diagonal): one warp per
  // row, lanes split the row's SELL entries, fixed shuffle tree (deterministic).
  if (warp < nr) {
    const int r = warp;
    const int64_t il = il0 + r, gi = s.row0 + il;
    const int64_t t = S.pos_of[gi];
    const int L = int(t & 31);
    const int64_t off = S.slice_off[t >> 5];
    const int32_t width = int32_t((S.slice_off[(t >> 5) + 1] - off) >> 5);
    const double* arow_new = a_out + size_t(il) * size_t(ld);
    double part = 0.0;
    for (int32_t q = lane; q < width; q += 32) {
      const int64_t idx = off + int64_t(q) * 32 + L;
      const int32_t c = __ldg(S.cols + idx);
      if (c >= 0) part = __fma_rn(__ldg(S.vals + idx), arow_new[inv ? __ldg(inv + c) : c], part);
    }
    part = warp_sum(part);
    if (lane == 0) {
      double nu = 0.0, de = 0.0;
      for (int ww = 0; ww < NW; ++ww) {
        nu = fmax(nu, red[ww][r][0]);
        de = fmax(de, red[ww][r][1]);
      }
      s.rowpart[rp_index(0, il, 0, rows, 1)] = part;
      s.rowpart[rp_index(1, il, 0, rows, 1)] = nu;
      s.rowpart[rp_index(2, il, 0, rows, 1)] = de;
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

cudaError_t launch_csr_step(const DevSolve& s, const DevSell& d, cudaStream_t st) {
  const int Rs = csr_rows_per_cta(s.n);
  const int use_smem = Rs > 0 ? 1 : 0;
  const int R = use_smem ? Rs : 1;
  const unsigned grid = unsigned((s.rows + R - 1) / R);
  const size_t smem = use_smem ? size_t(csr_stride(R)) * size_t(d.npad > s.n ? d.npad : s.n) * 8 : 0;
  if (!use_smem) {
    csr_step_kernel<1, false><<<grid, kCsrThreads, 0, st>>>(s, d);
    return cudaGetLastError();
  }
  if (!d.cols16 || !d.lane_pos || !d.lane_theta) return cudaErrorInvalidValue;  // the packed image was not built
#define DPT_CSR_CASE(RR)                                                                          \
  case RR: {                                                                                      \
    static DeviceAttrOnce attr;                                                                   \
    attr([] {                                                                                     \
      cudaFuncSetAttribute(csr_step_kernel<RR, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                           kCsrSmemBudget + 1024);                                                \
    });                                                                                           \
    csr_step_kernel<RR, true><<<grid, kCsrThreads, smem, st>>>(s, d);                             \
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

// ------------------------------------------------- K2, launch 1 from A_0 = I ----
// The first application of the map starts from the identity, where the product
// is known: P(I)(i,j) = Delta(j,i).  Running K2 on it costs a full step (c3:
// 1.57 ms of a 30 ms solve) for n^2 outputs of which nnz are not signed zeros
// -- the dense path's launch 1 is an elementwise kernel for the same reason
// (the reference's matmul skips a(i,k) == 0, matrix.cpp:150).  Three small
// kernels produce exactly what K2's launch 1 writes -- A_1, the step / max /
// nonfinite statistics, the residual partials of A_0 and the lagged diagonal
// d_1 -- with K2's own expressions, so every value is bit-identical to K2's:
//   fill     A_1(i,j) = 1 (i = j), else (lam_1 g(i,j)) * (p - d_0(i) A_0(i,j))
//            with p = +0, A_0(i,j) = 0 (a signed zero; NaN if lam_1 g overflows)
//   scatter  one warp per row j of Delta: entry (j,k,v) is P(I)(k,j) = v, i.e.
//            output (k,j); the maxima go through atomicMax on the bit patterns
//            of non-negative doubles (order-preserving; NaNs skipped as fmax
//            skips them) -- maxima do not depend on the order
//   finish   d_1(i) with K2's lane partition over the SELL image, the diagonal
//            column's residual term, rowpart / tilepart in K2's layout
// Not used with an explicit gap matrix, complex data, rows that do not fit
// shared memory, or a CSR with repeated (row, column) pairs (their sum would
// follow the schedule's order).
struct CsrInitScratch {
  unsigned long long* rownum;  // [rows] max |residual term| of the entries of A_0's row i (bit pattern)
  unsigned long long* stats;   // [0] max step, [1] max |A_1| (bit patterns), [2] nonfinite count (may wrap below
                               //     zero transiently: two's complement), [3] spare
};

__device__ __forceinline__ void atomic_max_nonneg(unsigned long long* slot, double v) {
  if (v == v) atomicMax(slot, (unsigned long long)__double_as_longlong(v));  // v >= 0; NaN skipped like fmax
}

__global__ void __launch_bounds__(256) csr_init_fill_kernel(DevSolve s, CsrInitScratch sc) {
  if (s.state->done) return;
  const int jl = launch_index(s);
  double* a_out = s.slots + size_t(jl % s.nslots) * size_t(s.slot_elems);
  const double lam_k = lam_of(s, jl);
  const double* d_in = s.dvec[(jl - 1) & 1];
  unsigned long long bad = 0;
  for (int64_t il = blockIdx.y; il < s.rows; il += gridDim.y) {
    const int64_t gi = s.row0 + il;
    const double ti = s.theta[gi];
    const double z = __dsub_rn(0.0, __dmul_rn(d_in[il], 0.0));  // p - d A_0(i,j) with p = +0, A_0(i,j) = 0
    double* orow = a_out + size_t(il) * size_t(s.ld);
    for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < s.n; j += int64_t(gridDim.x) * blockDim.x) {
      double val = 1.0;
      if (gi != j) {
        val = __dmul_rn(__dmul_rn(lam_k, 1.0 / __dsub_rn(ti, s.theta[j])), z);
        bad += isfinite(val) ? 0 : 1;
      }
      orow[j] = val;
    }
  }
  for (int o = 16; o > 0; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
  if ((threadIdx.x & 31) == 0 && bad) atomicAdd(&sc.stats[2], bad);
}

__global__ void __launch_bounds__(256) csr_init_scatter_kernel(DevSolve s, DevCsr D, CsrInitScratch sc) {
  if (s.state->done) return;
  const int jl = launch_index(s);
  double* a_out = s.slots + size_t(jl % s.nslots) * size_t(s.slot_elems);
  const double lam_k = lam_of(s, jl), lam = s.lambda;
  const double* d_in = s.dvec[(jl - 1) & 1];
  const int lane = threadIdx.x & 31;
  const int64_t wid = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  double t_step = 0.0, t_max = 0.0;
  long long bad = 0;  // nonfinite entries minus the nonfinite fills they replace
  for (int64_t j = wid; j < s.n; j += nw) {
    const double tj = s.theta[j];
    for (int64_t q = D.rowptr[j] + lane; q < D.rowptr[j + 1]; q += 32) {
      const int64_t k = D.cols[q];
      const int64_t il = k - s.row0;
      if (k == j || il < 0 || il >= s.rows) continue;  // the diagonal entry only feeds d_0; other ranks' rows
      const double v = D.vals[q];
      const double tk = s.theta[k], dk = d_in[il];
      const double eps_k = __dadd_rn(tk, __dmul_rn(lam, dk));
      const double t = __dmul_rn(lam_k, 1.0 / __dsub_rn(tk, tj));
      const double dz = __dmul_rn(dk, 0.0);
      const double val = __dmul_rn(t, __dsub_rn(v, dz));
      const double fill = __dmul_rn(t, __dsub_rn(0.0, dz));
      a_out[size_t(il) * size_t(s.ld) + size_t(j)] = val;
      t_step = fmax(t_step, fabs(__dsub_rn(val, 0.0)));
      t_max = fmax(t_max, fabs(val));
      bad += (isfinite(val) ? 0 : 1) - (isfinite(fill) ? 0 : 1);
      const double rr = __dadd_rn(__dmul_rn(__dsub_rn(tj, eps_k), 0.0), __dmul_rn(lam, v));
      atomic_max_nonneg(&sc.rownum[il], fabs(rr));
    }
  }
  t_step = warp_max(t_step);
  t_max = warp_max(t_max);
  for (int o = 16; o > 0; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
  if (lane == 0) {
    atomic_max_nonneg(&sc.stats[0], t_step);
    atomic_max_nonneg(&sc.stats[1], t_max);
    if (bad) atomicAdd(&sc.stats[2], (unsigned long long)bad);
  }
}

__global__ void __launch_bounds__(256) csr_init_finish_kernel(DevSolve s, DevSell S, CsrInitScratch sc) {
  if (s.state->done) return;
  const int jl = launch_index(s);
  const double* a_out = s.slots + size_t(jl % s.nslots) * size_t(s.slot_elems);
  const double lam = s.lambda;
  const double* d_in = s.dvec[(jl - 1) & 1];
  const int32_t* __restrict__ inv = S.inv;
  const int lane = threadIdx.x & 31;
  const int64_t wid = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int64_t rows = s.rows;
  for (int64_t il = wid; il < rows; il += nw) {
    // d_1(i) = P(A_1)(i,i): K2's tail (lanes split the row's SELL entries, one shuffle tree)
    const int64_t gi = s.row0 + il;
    const int64_t t = S.pos_of[gi];
    const int L = int(t & 31);
    const int64_t off = S.slice_off[t >> 5];
    const int32_t width = int32_t((S.slice_off[(t >> 5) + 1] - off) >> 5);
    const double* arow_new = a_out + size_t(il) * size_t(s.ld);
    double part = 0.0;
    for (int32_t q = lane; q < width; q += 32) {
      const int64_t idx = off + int64_t(q) * 32 + L;
      const int32_t c = __ldg(S.cols + idx);
      if (c >= 0) part = __fma_rn(__ldg(S.vals + idx), arow_new[inv ? __ldg(inv + c) : c], part);
    }
    part = warp_sum(part);
    if (lane == 0) {
      // the diagonal column of A_0's row: a_ii = 1, p = P(I)(i,i) = d_0(i)
      const double ti = s.theta[gi], di = d_in[il];
      const double eps_i = __dadd_rn(ti, __dmul_rn(lam, di));
      const double rr = __dadd_rn(__dmul_rn(__dsub_rn(ti, eps_i), 1.0), __dmul_rn(lam, di));
      const double nu = fmax(__longlong_as_double((long long)sc.rownum[il]), fabs(rr));
      s.rowpart[rp_index(0, il, 0, rows, 1)] = part;
      s.rowpart[rp_index(1, il, 0, rows, 1)] = nu;
      s.rowpart[rp_index(2, il, 0, rows, 1)] = 1.0;  // max_j |A_0(i,j)|
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double* tp = s.tilepart;  // one tile: the fold of this launch reads tile 0 only
    tp[0] = __longlong_as_double((long long)sc.stats[0]);
    tp[1] = fmax(__longlong_as_double((long long)sc.stats[1]), 1.0);  // the unit diagonal
    tp[2] = double((long long)sc.stats[2]);
    tp[3] = 0.0;
  }
}

// scratch: (rows + 4) * 8 bytes, zeroed here.  Tiles of the following fold: 1.
cudaError_t launch_csr_init(const DevSolve& s, const DevCsr& c, const DevSell& d, void* scratch, cudaStream_t st) {
  CsrInitScratch sc;
  sc.rownum = static_cast<unsigned long long*>(scratch);
  sc.stats = sc.rownum + s.rows;
  cudaError_t e = cudaMemsetAsync(scratch, 0, size_t(s.rows + 4) * 8, st);
  if (e != cudaSuccess) return e;
  const int64_t cb = (s.n + 1023) / 1024 > 0 ? (s.n + 1023) / 1024 : 1;  // 4 columns per thread
  const dim3 fgrid(unsigned(cb > 64 ? 64 : cb), unsigned(s.rows > 4096 ? 4096 : (s.rows > 0 ? s.rows : 1)));
  csr_init_fill_kernel<<<fgrid, 256, 0, st>>>(s, sc);
  const int64_t wb = (s.n + 7) / 8;
  csr_init_scatter_kernel<<<unsigned(wb > 1184 ? 1184 : (wb > 0 ? wb : 1)), 256, 0, st>>>(s, c, sc);
  const int64_t fb = (s.rows + 7) / 8;
  csr_init_finish_kernel<<<unsigned(fb > 1184 ? 1184 : (fb > 0 ? fb : 1)), 256, 0, st>>>(s, d, sc);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ K3 ----
// Row-dot "groups": G lanes cooperate on one row m of Delta.
//   MODE 0  CSR with exactly 16 nonzeros per row (BASELINE c4): G = 4, each
//           lane loads one int4 of columns + two double2 of values (a warp's
//           column loads are one contiguous 512-byte span), 4 z gathers.
//   MODE 1  general CSR: G = 1, the row in CSR order.
//   MODE 2  dense Delta (GEMV): G = 32, lanes stride the row.
// The lanes of a group combine with xor-shuffles, so every lane ends with the
// bit-identical value; w[row] (needed by every block) is computed by warp 0 of
// each block with the SAME routine, hence equals w[m = row] exactly.
constexpr int kSingleThreads = 256;
constexpr int kSingleMaxBlocks = 148 * 8;

template <int MODE>
struct RowGroup {
  static constexpr int G = MODE == 0 ? 4 : (MODE == 1 ? 1 : 32);
};

__device__ __forceinline__ bool gemv_vec_ok(const double* dense, const double* z, int64_t ld) {
  return ((ld & 1) == 0) && ((reinterpret_cast<uintptr_t>(dense) | reinterpret_cast<uintptr_t>(z)) & 15) == 0;
}

// w[row] for the dense row map, by the whole block: warp q sums columns
// [q n / NW, (q + 1) n / NW) (even boundaries), the warps' sums are added in
// warp order -- one fixed order, the same in every block.  The warp that owns
// row m = row uses this value too, so w[row] is bit-identical everywhere.
template <int NW>
__device__ __forceinline__ double gemv_block_dot(const double* __restrict__ dense, int64_t n, int64_t ld, int64_t row,
                                                 const double* __restrict__ z, double* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* dr = dense + size_t(row) * size_t(ld);
  double w = 0.0;
  if (gemv_vec_ok(dense, z, ld)) {
    const int64_t n2 = n >> 1;
    const int64_t c0 = n2 * warp / NW, c1 = n2 * (warp + 1) / NW;
    const double2* d2 = reinterpret_cast<const double2*>(dr);
    const double2* z2 = reinterpret_cast<const double2*>(z);
    double a0 = 0.0, a1 = 0.0;
    for (int64_t c = c0 + lane; c < c1; c += 32) {
      const double2 x = __ldg(d2 + c), y = z2[c];
      a0 = __fma_rn(x.x, y.x, a0);
      a1 = __fma_rn(x.y, y.y, a1);
    }
    if ((n & 1) && warp == NW - 1 && lane == 0) a0 = __fma_rn(dr[n - 1], z[n - 1], a0);
    w = a0 + a1;
  } else {
    const int64_t c0 = n * warp / NW, c1 = n * (warp + 1) / NW;
    for (int64_t c = c0 + lane; c < c1; c += 32) w = __fma_rn(dr[c], z[c], w);
  }
  w = warp_sum(w);
  if (lane == 0) sh[warp] = w;
  __syncthreads();
  double t = 0.0;
#pragma unroll
  for (int q = 0; q < NW; ++q) t += sh[q];
  return t;
}

// Rows per warp of the dense row map (measured, tools/gemv_time.py): one row
// per warp keeps z in L1 only for small n; from n = 4096 two rows share each z
// load, from 16384 four.
constexpr int64_t kGemvRpw2 = 4096;
constexpr int64_t kGemvRpw4 = 16384;
// RPW rows per warp (dense row map, n large): rows m .. m+RPW-1 stream
// together, 16-byte loads, four columns-chunks per lane in flight per row; per
// row two accumulators (even / odd columns), one fixed order.  The row m = row
// takes the block's w[row] (bit-identical to every block's).
template <int RPW, class F>
__device__ __forceinline__ void gemv_rows_loop(const double* __restrict__ dense, int64_t n, int64_t ld, int64_t row,
                                               double wr, const double* __restrict__ z, int lane, F& finish_row) {
  const int64_t nwarps = int64_t(gridDim.x) * (blockDim.x >> 5);
  const int64_t wid = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t n2 = n >> 1;
  const double2* z2 = reinterpret_cast<const double2*>(z);
  for (int64_t m0 = wid * RPW; m0 < n; m0 += nwarps * RPW) {
    const double2* d2[RPW];
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
      const int64_t m = m0 + r < n ? m0 + r : n - 1;
      d2[r] = reinterpret_cast<const double2*>(dense + size_t(m) * size_t(ld));
    }
    double a0[RPW], a1[RPW];
#pragma unroll
    for (int r = 0; r < RPW; ++r) a0[r] = a1[r] = 0.0;
    int64_t c = lane;
    for (; c + 96 < n2; c += 128) {
      double2 y[4], x[RPW][4];
#pragma unroll
      for (int u = 0; u < 4; ++u) y[u] = z2[c + 32 * u];
#pragma unroll
      for (int r = 0; r < RPW; ++r)
#pragma unroll
        for (int u = 0; u < 4; ++u) x[r][u] = __ldg(d2[r] + c + 32 * u);
#pragma unroll
      for (int r = 0; r < RPW; ++r)
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          a0[r] = __fma_rn(x[r][u].x, y[u].x, a0[r]);
          a1[r] = __fma_rn(x[r][u].y, y[u].y, a1[r]);
        }
    }
    for (; c < n2; c += 32) {
      const double2 y = z2[c];
#pragma unroll
      for (int r = 0; r < RPW; ++r) {
        const double2 x = __ldg(d2[r] + c);
        a0[r] = __fma_rn(x.x, y.x, a0[r]);
        a1[r] = __fma_rn(x.y, y.y, a1[r]);
      }
    }
    if ((n & 1) && lane == 0) {
#pragma unroll
      for (int r = 0; r < RPW; ++r)
        a0[r] = __fma_rn(reinterpret_cast<const double*>(d2[r])[n - 1], z[n - 1], a0[r]);
    }
    double w[RPW];
#pragma unroll
    for (int r = 0; r < RPW; ++r) w[r] = warp_sum(a0[r] + a1[r]);
    if (lane == 0) {
#pragma unroll
      for (int r = 0; r < RPW; ++r)
        if (m0 + r < n) finish_row(m0 + r, m0 + r == row ? wr : w[r]);
    }
  }
}

template <int MODE>
__device__ __forceinline__ double group_row_dot(const DevCsr& D, const double* __restrict__ dense, int64_t n,
                                                int64_t ld, int64_t m, const double* __restrict__ z, int sub) {
  double w = 0.0;
  if constexpr (MODE == 0) {
    const int4 c = __ldg(reinterpret_cast<const int4*>(D.cols + 16 * m) + sub);
    const double2 v0 = __ldg(reinterpret_cast<const double2*>(D.vals + 16 * m) + 2 * sub);
    const double2 v1 = __ldg(reinterpret_cast<const double2*>(D.vals + 16 * m) + 2 * sub + 1);
    const double z0 = z[c.x], z1 = z[c.y], z2 = z[c.z], z3 = z[c.w];
    w = __fma_rn(v0.x, z0, w);
    w = __fma_rn(v0.y, z1, w);
    w = __fma_rn(v1.x, z2, w);
    w = __fma_rn(v1.y, z3, w);
    w += __shfl_xor_sync(0xffffffffu, w, 1);
    w += __shfl_xor_sync(0xffffffffu, w, 2);
  } else if constexpr (MODE == 1) {
    const int64_t pb = D.rowptr[m], pe = D.rowptr[m + 1];
    for (int64_t q = pb; q < pe; ++q) w = __fma_rn(__ldg(D.vals + q), z[__ldg(D.cols + q)], w);
  } else {
    // GEMV row: HBM-bound stream of Delta's row.  16-byte loads, eight per
    // lane in flight, two accumulators (even / odd columns) -- a fixed order.
    const double* dr = dense + size_t(m) * size_t(ld);
    if (gemv_vec_ok(dense, z, ld)) {
      const double2* d2 = reinterpret_cast<const double2*>(dr);
      const double2* z2 = reinterpret_cast<const double2*>(z);
      const int64_t n2 = n >> 1;
      double a0 = 0.0, a1 = 0.0;
      int64_t c = sub;
      for (; c + 224 < n2; c += 256) {
        double2 x[8], y[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) x[u] = __ldg(d2 + c + 32 * u);
#pragma unroll
        for (int u = 0; u < 8; ++u) y[u] = z2[c + 32 * u];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          a0 = __fma_rn(x[u].x, y[u].x, a0);
          a1 = __fma_rn(x[u].y, y[u].y, a1);
        }
      }
      for (; c < n2; c += 32) {
        const double2 x = __ldg(d2 + c), y = z2[c];
        a0 = __fma_rn(x.x, y.x, a0);
        a1 = __fma_rn(x.y, y.y, a1);
      }
      if ((n & 1) && sub == 0) a0 = __fma_rn(dr[n - 1], z[n - 1], a0);
      w = a0 + a1;
    } else {
      for (int64_t c = sub; c < n; c += 32) w = __fma_rn(dr[c], z[c], w);
    }
    w = warp_sum(w);
  }
  return w;
}

template <int MODE>
__global__ void __launch_bounds__(kSingleThreads)
    single_step_kernel(DevSolve s, DevCsr D, const double* __restrict__ dense, int64_t row) {
  if (s.state->done) return;
  constexpr int G = RowGroup<MODE>::G;
  constexpr int ROWS_PER_ITER = kSingleThreads / G;
  const int jl = launch_index(s);
  __shared__ double wrow_s;
  __shared__ double red[kSingleThreads / 32][5];
  const int64_t n = s.n, ld = s.ld;
  const double* __restrict__ z = s.slots + size_t((jl - 1) % s.nslots) * size_t(s.slot_elems);
  double* __restrict__ zo = s.slots + size_t(jl % s.nslots) * size_t(s.slot_elems);
  const double lam_k = lam_of(s, jl), lam = s.lambda;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sub = threadIdx.x % G;
  if constexpr (MODE == 2) {  // the whole block streams row `row` once
    __shared__ double wsh[kSingleThreads / 32];
    const double wr = gemv_block_dot<kSingleThreads / 32>(dense, n, ld, row, z, wsh);
    if (threadIdx.x == 0) {
      wrow_s = wr;
      if (blockIdx.x == 0) s.dvec[(jl - 1) & 1][0] = wr;  // w[row] of z_{j-1} for the fold's eps
    }
  } else if (warp == 0) {  // one code path for the whole warp (the group shuffles name all lanes)
    const double wr = (MODE == 1 && lane != 0) ? 0.0 : group_row_dot<MODE>(D, dense, n, ld, row, z, sub);
    if (lane == 0) {
      wrow_s = wr;
      if (blockIdx.x == 0) s.dvec[(jl - 1) & 1][0] = wr;  // w[row] of z_{j-1} for the fold's eps
    }
  }
  __syncthreads();
  const double wr = wrow_s;
  const double trow = s.theta[row];
  const double eps = __dadd_rn(trow, __dmul_rn(lam, wr));
  double num = 0.0, den = 0.0, t_step = 0.0, t_max = 0.0, t_nonfin = 0.0;
  const int64_t stride = int64_t(gridDim.x) * ROWS_PER_ITER;
  auto finish_row = [&](int64_t m, double w) {
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
    t_step = fmax(t_step, fabs(__dsub_rn(v, zm)));
    t_max = fmax(t_max, fabs(v));
    t_nonfin += isfinite(v) ? 0.0 : 1.0;
    const double r = __dadd_rn(__dmul_rn(__dsub_rn(tm, eps), zm), __dmul_rn(lam, w));
    num = fmax(num, fabs(r));
    den = fmax(den, fabs(zm));
  };
  // UNROLL row groups per trip, in explicit phases (all row loads, then all z
  // gathers, then the FMA chains) so every load of the trip is in flight
  // together -- the step is bound by the L1/L2 sector traffic of the gathers.
  if constexpr (MODE == 0) {
    constexpr int U = 4;
    for (int64_t m0 = int64_t(blockIdx.x) * ROWS_PER_ITER; m0 < n; m0 += U * stride) {
      int4 c[U];
      double2 v0[U], v1[U];
      int64_t mm[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        mm[u] = m0 + u * stride + threadIdx.x / G;
        const int64_t mc = mm[u] < n ? mm[u] : n - 1;
        c[u] = __ldg(reinterpret_cast<const int4*>(D.cols + 16 * mc) + sub);
        v0[u] = __ldg(reinterpret_cast<const double2*>(D.vals + 16 * mc) + 2 * sub);
        v1[u] = __ldg(reinterpret_cast<const double2*>(D.vals + 16 * mc) + 2 * sub + 1);
      }
      double zg[U][4];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        zg[u][0] = z[c[u].x];
        zg[u][1] = z[c[u].y];
        zg[u][2] = z[c[u].z];
        zg[u][3] = z[c[u].w];
      }
      double w[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {  // the same FMA order / shuffle tree as group_row_dot<0>
        double a = 0.0;
        a = __fma_rn(v0[u].x, zg[u][0], a);
        a = __fma_rn(v0[u].y, zg[u][1], a);
        a = __fma_rn(v1[u].x, zg[u][2], a);
        a = __fma_rn(v1[u].y, zg[u][3], a);
        w[u] = a;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) w[u] += __shfl_xor_sync(0xffffffffu, w[u], 1);
#pragma unroll
      for (int u = 0; u < U; ++u) w[u] += __shfl_xor_sync(0xffffffffu, w[u], 2);
      if (sub == 0) {
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (mm[u] < n) finish_row(mm[u], w[u]);
      }
    }
  } else if (MODE == 2 && gemv_vec_ok(dense, z, ld) && n >= kGemvRpw2) {
    // Dense Delta, large n: each warp streams RPW consecutive rows at once, so
    // every z load (from L2 once z outgrows L1) serves RPW rows -- with one row
    // per warp, z's re-reads matched Delta's own traffic (n^2 doubles each).
    if (n >= kGemvRpw4)
      gemv_rows_loop<4>(dense, n, ld, row, wr, z, lane, finish_row);
    else
      gemv_rows_loop<2>(dense, n, ld, row, wr, z, lane, finish_row);
  } else {
    constexpr int U = 2;
    for (int64_t m0 = int64_t(blockIdx.x) * ROWS_PER_ITER; m0 < n; m0 += U * stride) {
      double w[U];
      int64_t mm[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        mm[u] = m0 + u * stride + threadIdx.x / G;
        w[u] = (MODE == 2 && mm[u] == row) ? wr : group_row_dot<MODE>(D, dense, n, ld, mm[u] < n ? mm[u] : n - 1, z, sub);
      }
      if (sub == 0) {
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (mm[u] < n) finish_row(mm[u], w[u]);
      }
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
    for (int ww = 0; ww < kSingleThreads / 32; ++ww) {
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
    double* tp = s.tilepart + size_t(tn) * 4;
    tp[0] = a[2];
    tp[1] = a[3];
    tp[2] = a[4];
    tp[3] = 0.0;
  }
}

int single_mode(int dense, int uniform16) { return dense ? 2 : (uniform16 ? 0 : 1); }

int u16_grid(int64_t n);
cudaError_t launch_single_u16(const DevSolve& s, const DevCsr& d, int64_t row, cudaStream_t st);

int single_ntiles(int64_t n, int mode) {
  if (mode == 0) return u16_grid(n);
  const int rows_per_iter = kSingleThreads / (mode == 1 ? 1 : 32);
  int64_t b = (n + rows_per_iter - 1) / rows_per_iter;
  if (b > kSingleMaxBlocks) b = kSingleMaxBlocks;
  return int(b < 1 ? 1 : b);
}
int single_ntn(int64_t n, int mode) { return single_ntiles(n, mode); }

cudaError_t launch_single_step(const DevSolve& s, const DevCsr& d, const double* dense, int64_t row, int mode,
                               cudaStream_t st) {
  if (mode == 0) return launch_single_u16(s, d, row, st);
  const unsigned grid = unsigned(single_ntiles(s.n, mode));
  if (mode == 1)
    single_step_kernel<1><<<grid, kSingleThreads, 0, st>>>(s, d, dense, row);
  else
    single_step_kernel<2><<<grid, kSingleThreads, 0, st>>>(s, d, dense, row);
  return cudaGetLastError();
}

}  // namespace dpt
