// dense_step.cu -- K1: the dense DPT step as ONE kernel.
//
// Replaces, per reference iteration (paths relative to /root/reference/proj):
//   pn = matmul(an, delta_t)             src/dpt.cpp:152 -> src/matrix.cpp:130-143
//   an = F(a) (map, unit diagonal)       src/dpt.cpp:136-144
//   step = max_abs_diff(an, a)           src/dpt.cpp:145, src/matrix.cpp:356-364
//   all_finite / max_abs (divergence)    src/dpt.cpp:147, src/matrix.cpp:338-384
//   residuals_of (eps_i, row residuals)  src/dpt.cpp:23-44
// in the row form the reference uses: P = A * Delta^T, i.e.
//   P(i,j) = sum_k A(i,k) Delta(j,k)    (both operands K-contiguous, row-major)
//   A'(i,j) = i==j ? 1 : (lam_k / (theta_i - theta_j)) * (P(i,j) - P(i,i) A(i,j)).
// Row i of A evolves independently; rows are sharded across ranks.
//
// GEMM: 128x128 (or 64x64) CTA tile, BK = 16, a 4-stage TMA (SWIZZLE_128B) +
// mbarrier pipeline fed by one producer warp, FP64 tensor cores through
// mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4; tcgen05 has no f64 kind on sm_100a).
// The two k4-steps of a 16-byte chunk are loaded with one LDS.128: the k index
// is permuted identically for both operands, so the product is unchanged.
//
// P(i,i) is needed by every tile of row i but produced by one tile only, so the
// diagonal is LAGGED (SURVEY.md §7 hard part 1): launch j uses d_{j-1}(i) =
// sum_m A_{j-1}(i,m) Delta(i,m) that launch j-1 emitted as per-tile partials
// (folded deterministically by the fold kernel), and emits d_j partials of its
// own output.  Launch j also yields the residual numerator/denominator of
// A_{j-1} (eps_i = theta_i + lambda d_{j-1}(i)), so a reference iteration's
// read-offs cost no extra GEMM (Appendix B).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <type_traits>
#include <stdint.h>
#include <stdlib.h>

#include "dense_mma.cuh"
#include "dpt_device.cuh"
#include "dpt_kernels.h"

namespace dpt {

// The fused DPT epilogue of one output tile (tm, tn): map, step / max /
// nonfinite, residual partials and the lagged diagonal (shared by the
// one-tile-per-CTA kernel and the stream-K kernel).  Called by every consumer
// thread; ends with the tile's partials written.
template <class C, bool CPLX>
__device__ __forceinline__ void dense_epilogue(const DevSolve& s, double (&acc)[C::MB][C::NB][2], int tm, int tn,
                                               int j_launch, int slot_in, int slot_out, const double* __restrict__ delta,
                                               double* red, double* wred, int warp, int lane) {
  const int wm = warp / C::WARPS_N, wn = warp % C::WARPS_N;
  const int t = lane & 3, gq = lane >> 2;
  const int64_t n = s.ncol, rows = s.rows;
  const int ntn = s.ntn;
  const double lam_k = lam_of(s, j_launch);
  const double lam = s.lambda;
  const double* __restrict__ a_in = s.slots + size_t(slot_in) * size_t(s.slot_elems);
  double* __restrict__ a_out = s.slots + size_t(slot_out) * size_t(s.slot_elems);
  const double* __restrict__ d_in = s.dvec[(j_launch - 1) & 1];
  const double* __restrict__ theta = s.theta;

  const int colbase = tn * C::BN + wn * C::WTN + 2 * t;
  double t_step = 0.0, t_max = 0.0, t_nonfin = 0.0;
  if constexpr (CPLX) {
    // complex element j = c / 2 of row i: the fragment pair (c, c+1) = (re, im)
    const cd lamk = lamc_of(s, j_launch);
    const cd lamc = cmake(s.lambda, s.lambda_im);
#pragma unroll
    for (int a = 0; a < C::MB; ++a) {
      const int il = tm * C::BM + wm * C::WTM + a * 8 + gq;
      const bool row_ok = il < rows;
      const int64_t gi = s.row0 + il;
      double num = 0.0, den = 0.0, dre = 0.0, dim = 0.0;
      if (row_ok) {
        const cd ti = cmake(theta[2 * gi], theta[2 * gi + 1]);
        const cd di = cmake(d_in[2 * il], d_in[2 * il + 1]);
        const cd eps_i = cadd(ti, cmul(lamc, di));
        const double* arow = a_in + size_t(il) * size_t(s.ld);
        double* orow = a_out + size_t(il) * size_t(s.ld);
        const double* drow = delta + size_t(2 * gi) * size_t(s.ldd);  // (Re D(i,j), -Im D(i,j)) pairs
#pragma unroll
        for (int b = 0; b < C::NB; ++b) {
          const int c = colbase + b * 8;
          if (c >= n) continue;
          const double2 av2 = *reinterpret_cast<const double2*>(arow + c);
          const double2 dv2 = *reinterpret_cast<const double2*>(drow + c);
          const double2 tc2 = *reinterpret_cast<const double2*>(theta + c);
          const cd av = cmake(av2.x, av2.y), tc = cmake(tc2.x, tc2.y), dij = cmake(dv2.x, -dv2.y);
          const cd p = cmake(acc[a][b][0], acc[a][b][1]);
          cd v;
          if (2 * gi == c) {
            v = cmake(1.0, 0.0);
          } else {
            const cd g = s.gapmat ? cmake(s.gapmat[size_t(il) * size_t(s.ld) + size_t(c)],
                                          s.gapmat[size_t(il) * size_t(s.ld) + size_t(c) + 1])
                                  : crecip(csub(ti, tc));
            v = cmul(cmul(lamk, g), csub(p, cmul(di, av)));
          }
          *reinterpret_cast<double2*>(orow + c) = make_double2(v.x, v.y);
          t_step = fmax(t_step, cabs_(csub(v, av)));
          t_max = fmax(t_max, cabs_(v));
          t_nonfin += cfinite(v) ? 0.0 : 1.0;
          const cd r = cadd(cmul(csub(tc, eps_i), av), cmul(lamc, p));
          num = fmax(num, cabs_(r));
          den = fmax(den, cabs_(av));
          const cd vd = cmul(v, dij);
          dre += vd.x;
          dim += vd.y;
        }
      }
#pragma unroll
      for (int o = 1; o <= 2; o <<= 1) {
        num = fmax(num, __shfl_xor_sync(0xffffffffu, num, o));
        den = fmax(den, __shfl_xor_sync(0xffffffffu, den, o));
        dre += __shfl_xor_sync(0xffffffffu, dre, o);
        dim += __shfl_xor_sync(0xffffffffu, dim, o);
      }
      if (t == 0) {
        const int rt = wm * C::WTM + a * 8 + gq;
        red[(wn * C::BM + rt) * 4 + 0] = dre;
        red[(wn * C::BM + rt) * 4 + 1] = num;
        red[(wn * C::BM + rt) * 4 + 2] = den;
        red[(wn * C::BM + rt) * 4 + 3] = dim;
      }
    }
  } else {
  const double* __restrict__ gap = s.gapmat;
  int n_nonfin = 0;
  // fmax(acc, x) for an accumulator that is never NaN: a NaN x compares false and
  // is skipped, exactly as fmax skips it
  auto max_keep = [](double acc, double x) { return x > acc ? x : acc; };
  // Interior tiles (every row and column pair in range: all tiles when n is a
  // multiple of the tile) run the same code with the range guards compiled out.
  auto elements = [&](auto full_tag) {
  constexpr bool FULL = decltype(full_tag)::value;
#pragma unroll
  for (int a = 0; a < C::MB; ++a) {
    const int il = tm * C::BM + wm * C::WTM + a * 8 + gq;  // local row
    const bool row_ok = FULL || il < rows;
    const int64_t gi = s.row0 + il;
    const int gi32 = int(gi);  // n < 2^31: the diagonal test in 32 bits
    double num = 0.0, den = 0.0, dsum = 0.0;
    if (row_ok) {
      const double ti = theta[gi];
      const double di = d_in[il];
      const double eps_i = __dadd_rn(ti, __dmul_rn(lam, di));
      const double* arow = a_in + size_t(il) * size_t(s.ld);
      double* orow = a_out + size_t(il) * size_t(s.ld);
      const double* drow = delta + size_t(gi) * size_t(s.ldd);
#pragma unroll
      for (int b = 0; b < C::NB; ++b) {
        const int c = colbase + b * 8;
        if (!FULL && c >= n) continue;
        const bool pair = FULL || c + 1 < n;
        double2 av, dv;
        if (pair) {
          av = *reinterpret_cast<const double2*>(arow + c);
          dv = *reinterpret_cast<const double2*>(drow + c);
        } else {
          av = make_double2(arow[c], 0.0);
          dv = make_double2(drow[c], 0.0);
        }
        const double2 tc = pair ? *reinterpret_cast<const double2*>(theta + c) : make_double2(theta[c], 0.0);
        double out[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          if (e == 1 && !pair) continue;
          const double aij = e ? av.y : av.x;
          const double dij = e ? dv.y : dv.x;
          const double p = acc[a][b][e];
          // Branch-free: the off-diagonal value is formed for every element (on the
          // diagonal 1 / 0 = inf, discarded by the select).  The epilogue is bound
          // by instruction issue (per-CTA timestamps on c1: 4.8 us of element work
          // per 64 x 64 tile, 10 us when both CTAs of an SM reach it together; the
          // operands' loads are not what it waits for -- staging them through the
          // TMA pipeline or hoisting them changed nothing), so the divergent
          // diagonal branch, the 64-bit index compare, the library fmax sequences
          // and the FP64 nonfinite counter are replaced by cheaper equivalents.
          const double g = gap ? gap[size_t(il) * size_t(s.ld) + size_t(c + e)]
                               : 1.0 / __dsub_rn(ti, e ? tc.y : tc.x);  // IEEE division = build_theta
          const double voff = __dmul_rn(__dmul_rn(lam_k, g), __dsub_rn(p, __dmul_rn(di, aij)));
          const double v = (gi32 == c + e) ? 1.0 : voff;  // exact unit diagonal (test_dpt.cpp:45-53)
          out[e] = v;
          t_step = max_keep(t_step, fabs(__dsub_rn(v, aij)));
          t_max = max_keep(t_max, fabs(v));
          n_nonfin += isfinite(v) ? 0 : 1;
          const double r = __dadd_rn(__dmul_rn(__dsub_rn(e ? tc.y : tc.x, eps_i), aij), __dmul_rn(lam, p));
          num = max_keep(num, fabs(r));
          den = max_keep(den, fabs(aij));
          dsum = __fma_rn(v, dij, dsum);
        }
        if (pair)
          *reinterpret_cast<double2*>(orow + c) = make_double2(out[0], out[1]);
        else
          orow[c] = out[0];
      }
    }
    // fold the 4 lanes that share this row (t = 0..3); the maxima are never NaN
    num = max_keep(num, __shfl_xor_sync(0xffffffffu, num, 1));
    den = max_keep(den, __shfl_xor_sync(0xffffffffu, den, 1));
    dsum += __shfl_xor_sync(0xffffffffu, dsum, 1);
    num = max_keep(num, __shfl_xor_sync(0xffffffffu, num, 2));
    den = max_keep(den, __shfl_xor_sync(0xffffffffu, den, 2));
    dsum += __shfl_xor_sync(0xffffffffu, dsum, 2);
    if (t == 0) {
      const int rt = wm * C::WTM + a * 8 + gq;  // row within tile
      red[(wn * C::BM + rt) * 4 + 0] = dsum;
      red[(wn * C::BM + rt) * 4 + 1] = num;
      red[(wn * C::BM + rt) * 4 + 2] = den;
      red[(wn * C::BM + rt) * 4 + 3] = 0.0;
    }
  }
  };
  const bool full_tile = int64_t(tm + 1) * C::BM <= rows && int64_t(tn + 1) * C::BN <= n;  // CTA-uniform
  if (full_tile)
    elements(std::true_type{});
  else
    elements(std::false_type{});
  t_nonfin += double(n_nonfin);
  }
  t_step = warp_max(t_step);
  t_max = warp_max(t_max);
  t_nonfin = warp_sum(t_nonfin);
  if (lane == 0) {
    wred[warp * 4 + 0] = t_step;
    wred[warp * 4 + 1] = t_max;
    wred[warp * 4 + 2] = t_nonfin;
  }
  asm volatile("bar.sync 1, %0;\n" ::"r"(C::NCW * 32) : "memory");  // consumers only

  const int ctid = threadIdx.x;
  for (int rt = ctid; rt < C::BM; rt += C::NCW * 32) {
    const int il = tm * C::BM + rt;
    if (il >= rows) continue;
    double ds = 0.0, nu = 0.0, de = 0.0, di = 0.0;
#pragma unroll
    for (int w = 0; w < C::WARPS_N; ++w) {
      ds += red[(w * C::BM + rt) * 4 + 0];
      nu = fmax(nu, red[(w * C::BM + rt) * 4 + 1]);
      de = fmax(de, red[(w * C::BM + rt) * 4 + 2]);
      di += red[(w * C::BM + rt) * 4 + 3];
    }
    s.rowpart[rp_index(0, il, tn, rows, ntn)] = ds;
    s.rowpart[rp_index(1, il, tn, rows, ntn)] = nu;
    s.rowpart[rp_index(2, il, tn, rows, ntn)] = de;
    if (CPLX) s.rowpart[rp_index(3, il, tn, rows, ntn)] = di;
  }
  if (ctid == 0) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    for (int w = 0; w < C::NCW; ++w) {
      a0 = fmax(a0, wred[w * 4 + 0]);
      a1 = fmax(a1, wred[w * 4 + 1]);
      a2 += wred[w * 4 + 2];
    }
    double* tp = s.tilepart + size_t(tm * ntn + tn) * 4;
    tp[0] = a0;
    tp[1] = a1;
    tp[2] = a2;
    tp[3] = 0.0;
  }
}

#ifndef DPT_REFILL_LAG
#define DPT_REFILL_LAG 0
#endif
constexpr int kRefillLag = DPT_REFILL_LAG;  // k-tiles between a stage's consumption and its refill (0 = at once)

template <class C, bool CPLX>
__global__ void __launch_bounds__(C::THREADS, C::MINB)
    dense_step_kernel(DevSolve s, const CUtensorMap* __restrict__ amaps,
                      const CUtensorMap* __restrict__ dmap, const double* __restrict__ delta,
                      int ntm) {
  const int j_launch = launch_index(s);
  if (s.state->done) return;  // a terminal status was reached: no-op launch

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  double* red = reinterpret_cast<double*>(smem + C::STAGES * C::STAGE_BYTES);
  double* wred = red + C::WARPS_N * C::BM * 4;
  uint64_t* full = reinterpret_cast<uint64_t*>(wred + C::NCW * 4);
  uint64_t* empty = full + C::STAGES;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // grouped rasterisation: 8 row blocks share each column block sweep (L2 reuse)
  const int ntn = s.ntn;
  const int bid = blockIdx.x;
  const int group = 8;
  const int per_group = group * ntn;
  const int g = bid / per_group;
  const int first_tm = g * group;
  const int gsize = min(group, ntm - first_tm);
  const int tm = first_tm + (bid % per_group) % gsize;
  const int tn = (bid % per_group) / gsize;

  const int slot_in = (j_launch - 1) % s.nslots;
  const int slot_out = j_launch % s.nslots;
  // real: P = A Delta^T over n columns; complex: the same NT GEMM over the
  // interleaved (re, im) columns against B = [[Re D, -Im D], [Im D, Re D]]
  // (row 2j of B -> Re P(:, j), row 2j+1 -> Im P(:, j)), i.e. K = N = 2n.
  const int64_t n = s.ncol;
  const int KT = int((n + C::BK - 1) / C::BK);

  if (threadIdx.x == 0) {
    for (int i = 0; i < C::STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], C::NCW);
    }
    fence_mbar_init();
  }
  __syncthreads();

  const CUtensorMap* am = amaps + slot_in;
  const bool producer = (threadIdx.x == 0);
  if (producer) {  // prologue: fill the pipeline
    prefetch_tmap(am);
    prefetch_tmap(dmap);
    const int pre = KT < C::STAGES ? KT : C::STAGES;
    for (int kt = 0; kt < pre; ++kt) {
      mbar_arrive_expect_tx(&full[kt], C::STAGE_BYTES);
      tma_load_2d(sA + kt * C::A_BYTES, am, &full[kt], kt * C::BK, tm * C::BM);
      tma_load_2d(sB + kt * C::B_BYTES, dmap, &full[kt], kt * C::BK, tn * C::BN);
    }
  }

  // ------------------------------------------------------ MMA consumers ----
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
    const uint8_t* a_st = sA + st * C::A_BYTES;
    const uint8_t* b_st = sB + st * C::B_BYTES;
    dmma_consume_stage<C>(acc, a_st, b_st, wm, wn, t, gq);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
    // Refill kRefillLag k-tiles after the consumption (compile-time, default 0 =
    // at once).  The producer is lane 0 of consumer warp 0; refilling the stage
    // it has just finished means waiting for the slower warps of this k-tile,
    // while the stage consumed earlier is already free.  Measured, lag 0 / 1 / 2:
    // c2 3.926 / 3.940 / 3.910 ms (3.929 in one of three runs); c5 shards w = 8
    // 241.9 / - / 242.6 ms, w = 4 498.6 / - / 501.1 ms (two pairs each): within
    // half a percent either way, so the simplest order stays.
    if (producer && kt >= kRefillLag && kt - kRefillLag + C::STAGES < KT) {
      const int kc = kt - kRefillLag, sr = kc % C::STAGES;
      const int kn = kc + C::STAGES;
      mbar_wait(&empty[sr], (kc / C::STAGES) & 1);
      fence_proxy_async_smem();  // the consumers' generic reads of the stage before the async-proxy refill
      mbar_arrive_expect_tx(&full[sr], C::STAGE_BYTES);
      tma_load_2d(sA + sr * C::A_BYTES, am, &full[sr], kn * C::BK, tm * C::BM);
      tma_load_2d(sB + sr * C::B_BYTES, dmap, &full[sr], kn * C::BK, tn * C::BN);
    }
    __syncwarp();
  }

  dense_epilogue<C, CPLX>(s, acc, tm, tn, j_launch, slot_in, slot_out, delta, red, wred, warp, lane);
}

// Stream-K variant for small n (cfg 0): with few output tiles per SM (c1:
// 256 tiles on 148 SMs) the SMs holding two tiles set the step time while the
// rest idle.  Here a persistent grid of exactly the resident CTAs splits the
// flat (tile, k-tile) work evenly: CTA c owns units [c T / G, (c+1) T / G).
// A tile whose k-range spans several CTAs is finished by whichever of them
// completes last: every part stores its accumulators to a per-CTA workspace
// slot and bumps the tile's counter; the last one sums the parts in k order
// (deterministic) and runs the epilogue.  Nobody waits, so no co-residency
// assumption is needed.  The TMA pipeline runs across tile boundaries, so the
// next segment's loads overlap the current segment's epilogue.
__device__ __forceinline__ int64_t sk_cta_of(int64_t u, int64_t total, int64_t G) {
  int64_t c = (u * G) / total;  // floor(c T / G) <= u < floor((c + 1) T / G)
  while (c + 1 < G && ((c + 1) * total) / G <= u) ++c;
  while (c > 0 && (c * total) / G > u) --c;
  return c;
}

template <class C, bool CPLX>
__global__ void __launch_bounds__(C::THREADS, C::MINB)
    dense_step_sk_kernel(DevSolve s, const CUtensorMap* __restrict__ amaps,
                         const CUtensorMap* __restrict__ dmap, const double* __restrict__ delta, int ntm) {
  const int j_launch = launch_index(s);
  if (s.state->done) return;

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  double* red = reinterpret_cast<double*>(smem + C::STAGES * C::STAGE_BYTES);
  double* wred = red + C::WARPS_N * C::BM * 4;
  uint64_t* full = reinterpret_cast<uint64_t*>(wred + C::NCW * 4);
  uint64_t* empty = full + C::STAGES;
  __shared__ int sk_last;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntn = s.ntn;
  const int group = 8, per_group = group * ntn;
  auto raster = [&](int64_t q, int& tm, int& tn) {  // the grouped rasterisation of the one-tile kernel
    const int b = int(q);
    const int g = b / per_group, first_tm = g * group, gsize = min(group, ntm - first_tm);
    tm = first_tm + (b % per_group) % gsize;
    tn = (b % per_group) / gsize;
  };
  const int slot_in = (j_launch - 1) % s.nslots;
  const int slot_out = j_launch % s.nslots;
  const int64_t n = s.ncol;
  const int KT = int((n + C::BK - 1) / C::BK);
  const int64_t total = int64_t(ntm) * ntn * KT, G = gridDim.x, cta = blockIdx.x;
  const int64_t u0 = cta * total / G, u1 = (cta + 1) * total / G;

  if (threadIdx.x == 0) {
    for (int i = 0; i < C::STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], C::NCW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const CUtensorMap* am = amaps + slot_in;
  const bool producer = (threadIdx.x == 0);
  auto issue = [&](int64_t v, int st) {
    int tm, tn;
    raster(v / KT, tm, tn);
    const int kt = int(v % KT);
    mbar_arrive_expect_tx(&full[st], C::STAGE_BYTES);
    tma_load_2d(sA + st * C::A_BYTES, am, &full[st], kt * C::BK, tm * C::BM);
    tma_load_2d(sB + st * C::B_BYTES, dmap, &full[st], kt * C::BK, tn * C::BN);
  };
  if (producer) {
    prefetch_tmap(am);
    prefetch_tmap(dmap);
    for (int64_t i = 0; i < C::STAGES && u0 + i < u1; ++i) issue(u0 + i, int(i));
  }

  const int wm = warp / C::WARPS_N, wn = warp % C::WARPS_N;
  const int t = lane & 3, gq = lane >> 2;
  constexpr int PART = C::NCW * C::MB * C::NB * 64;  // doubles per partial tile
  double acc[C::MB][C::NB][2];
  int64_t it = 0;  // units consumed by this CTA (pipeline stage / phase)
  for (int64_t v = u0; v < u1;) {
    const int64_t tile = v / KT;
    const int ka = int(v % KT);
    const int kb = int(min(int64_t(KT), int64_t(ka) + (u1 - v)));
#pragma unroll
    for (int a = 0; a < C::MB; ++a)
#pragma unroll
      for (int b = 0; b < C::NB; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    for (int kt = ka; kt < kb; ++kt, ++it) {
      const int st = int(it % C::STAGES);
      mbar_wait(&full[st], uint32_t((it / C::STAGES) & 1));
      const uint8_t* a_st = sA + st * C::A_BYTES;
      const uint8_t* b_st = sB + st * C::B_BYTES;
      dmma_consume_stage<C>(acc, a_st, b_st, wm, wn, t, gq);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
      if (producer && u0 + it + C::STAGES < u1) {  // refill this stage with the unit STAGES ahead
        mbar_wait(&empty[st], uint32_t((it / C::STAGES) & 1));
        fence_proxy_async_smem();  // the consumers' generic reads of the stage before the async-proxy refill
        issue(u0 + it + C::STAGES, st);
      }
      __syncwarp();
    }
    int tm, tn;
    raster(tile, tm, tn);
    asm volatile("bar.sync 1, %0;\n" ::"r"(C::NCW * 32) : "memory");  // red / wred / flag reuse
    if (ka == 0 && kb == KT) {
      dense_epilogue<C, CPLX>(s, acc, tm, tn, j_launch, slot_in, slot_out, delta, red, wred, warp, lane);
    } else {
      const int which = v == u0 ? 0 : 1;  // a CTA's partial segments are its first and / or last
      double* part = s.sk_ws + (size_t(cta) * 2 + size_t(which)) * size_t(PART);
#pragma unroll
      for (int a = 0; a < C::MB; ++a)
#pragma unroll
        for (int b = 0; b < C::NB; ++b)
          *reinterpret_cast<double2*>(part + ((size_t(warp) * C::MB + a) * C::NB + b) * 64 + 2 * lane) =
              make_double2(acc[a][b][0], acc[a][b][1]);
      const int64_t c_first = sk_cta_of(tile * KT, total, G), c_last = sk_cta_of(tile * KT + KT - 1, total, G);
      asm volatile("bar.sync 1, %0;\n" ::"r"(C::NCW * 32) : "memory");
      if (threadIdx.x == 0) {
        fence_acq_rel_gpu();  // release this part
        const unsigned prev = atomicAdd(s.sk_cnt + tile, 1u);
        sk_last = prev == unsigned(c_last - c_first);
        if (sk_last) fence_acq_rel_gpu();  // acquire the other parts
      }
      asm volatile("bar.sync 1, %0;\n" ::"r"(C::NCW * 32) : "memory");
      if (sk_last) {
        // P = part(c_first) + part(c_first + 1) + ... in k order
#pragma unroll
        for (int a = 0; a < C::MB; ++a)
#pragma unroll
          for (int b = 0; b < C::NB; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
        for (int64_t cc = c_first; cc <= c_last; ++cc) {
          const int w2 = (cc * total) / G < tile * KT ? 1 : 0;
          const double* pp = s.sk_ws + (size_t(cc) * 2 + size_t(w2)) * size_t(PART);
#pragma unroll
          for (int a = 0; a < C::MB; ++a)
#pragma unroll
            for (int b = 0; b < C::NB; ++b) {
              const double2 o = __ldcg(reinterpret_cast<const double2*>(
                  pp + ((size_t(warp) * C::MB + a) * C::NB + b) * 64 + 2 * lane));
              acc[a][b][0] += o.x;
              acc[a][b][1] += o.y;
            }
        }
        if (threadIdx.x == 0) s.sk_cnt[tile] = 0u;  // ready for the next launch
        dense_epilogue<C, CPLX>(s, acc, tm, tn, j_launch, slot_in, slot_out, delta, red, wred, warp, lane);
      }
    }
    v += kb - ka;
  }
}

// Launch 1: A_1 = F(I).  P(I) = I * Delta^T = Delta^T, so for i != j
// A_1(i,j) = (lam_1 theta(i,j)) * Delta(j,i) -- the reference's matmul(I, delta_t)
// zero-skips to exactly this (src/dpt.cpp:100, :136-144).  Elementwise with a
// shared-memory transpose; emits the same partials as the GEMM step.
// Block: 32 rows x BNI columns, 256 threads (32 x 8).
template <int BNI>
__global__ void __launch_bounds__(256) dense_init_kernel(DevSolve s, const double* __restrict__ delta) {
  if (s.state->done) return;
  __shared__ double sT[32][33];
  __shared__ double wr[8][3];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t n = s.n, rows = s.rows;
  const int tn = blockIdx.x;
  const int tmb = blockIdx.y;  // 32-row block (local rows)
  const int64_t il0 = int64_t(tmb) * 32;
  const double lam1 = lam_of(s, 1);
  double* __restrict__ a_out = s.slots + size_t(1 % s.nslots) * size_t(s.slot_elems);
  double dsum[4] = {0.0, 0.0, 0.0, 0.0};
  double t_step = 0.0, t_max = 0.0, t_nonfin = 0.0;
  for (int sub = 0; sub < BNI / 32; ++sub) {
    const int64_t j0 = int64_t(tn) * BNI + sub * 32;
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 4; ++r) {  // sT[jj][ii] = Delta(j0 + jj, gi0 + ii)
      const int64_t jj = j0 + ty + 8 * r;
      const int64_t gi = s.row0 + il0 + tx;
      sT[ty + 8 * r][tx] = (jj < n && il0 + tx < rows) ? delta[size_t(jj) * size_t(s.ldd) + size_t(gi)] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int64_t il = il0 + ty + 8 * r;
      const int64_t gi = s.row0 + il;
      const int64_t c = j0 + tx;
      if (il >= rows || c >= n) continue;
      double v;
      if (gi == c) {
        v = 1.0;
      } else {
        const double g = 1.0 / __dsub_rn(s.theta[gi], s.theta[c]);
        v = __dmul_rn(__dmul_rn(lam1, g), sT[tx][ty + 8 * r]);
      }
      a_out[size_t(il) * size_t(s.ld) + size_t(c)] = v;
      const double prev = (gi == c) ? 1.0 : 0.0;
      t_step = fmax(t_step, fabs(__dsub_rn(v, prev)));
      t_max = fmax(t_max, fabs(v));
      t_nonfin += isfinite(v) ? 0.0 : 1.0;
      dsum[r] = __fma_rn(v, delta[size_t(gi) * size_t(s.ldd) + size_t(c)], dsum[r]);
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const double v = warp_sum(dsum[r]);
    const int64_t il = il0 + ty + 8 * r;
    if (tx == 0 && il < rows) {
      s.rowpart[rp_index(0, il, tn, rows, s.ntn)] = v;
      s.rowpart[rp_index(1, il, tn, rows, s.ntn)] = 0.0;
      s.rowpart[rp_index(2, il, tn, rows, s.ntn)] = 0.0;
    }
  }
  t_step = warp_max(t_step);
  t_max = warp_max(t_max);
  t_nonfin = warp_sum(t_nonfin);
  if (tx == 0) {
    wr[ty][0] = t_step;
    wr[ty][1] = t_max;
    wr[ty][2] = t_nonfin;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    for (int w = 0; w < 8; ++w) {
      a0 = fmax(a0, wr[w][0]);
      a1 = fmax(a1, wr[w][1]);
      a2 += wr[w][2];
    }
    double* tp = s.tilepart + size_t(tmb * gridDim.x + tn) * 4;
    tp[0] = a0;
    tp[1] = a1;
    tp[2] = a2;
    tp[3] = 0.0;
  }
}

// Complex launch 1: A_1(i,j) = (lam_1 g(i,j)) * Delta(j,i) with Delta read from
// the real image B (Re D(j,i) = B[2j][2i], Im D(j,i) = B[2j+1][2i]).  One block
// per (row, BNI/2 complex columns), emitting the same partials as the step.
template <int BNI>
__global__ void __launch_bounds__(BNI / 2) dense_init_cplx_kernel(DevSolve s, const double* __restrict__ B) {
  if (s.state->done) return;
  __shared__ double wr[BNI / 64 > 0 ? BNI / 64 : 1][5];
  const int64_t n = s.n;
  const int tn = blockIdx.x;
  const int64_t il = blockIdx.y, gi = s.row0 + il;
  const int64_t j = int64_t(tn) * (BNI / 2) + threadIdx.x;
  const cd lam1 = lamc_of(s, 1);
  double* __restrict__ a_out = s.slots + size_t(1 % s.nslots) * size_t(s.slot_elems);
  double t_step = 0.0, t_max = 0.0, t_nonfin = 0.0, dre = 0.0, dim = 0.0;
  if (j < n) {
    cd v;
    if (gi == j) {
      v = cmake(1.0, 0.0);
    } else {
      const cd g = crecip(csub(cmake(s.theta[2 * gi], s.theta[2 * gi + 1]), cmake(s.theta[2 * j], s.theta[2 * j + 1])));
      const cd dji = cmake(B[size_t(2 * j) * size_t(s.ldd) + size_t(2 * gi)], B[size_t(2 * j + 1) * size_t(s.ldd) + size_t(2 * gi)]);
      v = cmul(cmul(lam1, g), dji);
    }
    *reinterpret_cast<double2*>(a_out + size_t(il) * size_t(s.ld) + size_t(2 * j)) = make_double2(v.x, v.y);
    t_step = cabs_(csub(v, cmake(gi == j ? 1.0 : 0.0, 0.0)));
    t_max = cabs_(v);
    t_nonfin = cfinite(v) ? 0.0 : 1.0;
    const double2 dij2 = *reinterpret_cast<const double2*>(B + size_t(2 * gi) * size_t(s.ldd) + size_t(2 * j));
    const cd vd = cmul(v, cmake(dij2.x, -dij2.y));
    dre = vd.x;
    dim = vd.y;
  }
  t_step = warp_max(t_step);
  t_max = warp_max(t_max);
  t_nonfin = warp_sum(t_nonfin);
  dre = warp_sum(dre);
  dim = warp_sum(dim);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    wr[w][0] = t_step;
    wr[w][1] = t_max;
    wr[w][2] = t_nonfin;
    wr[w][3] = dre;
    wr[w][4] = dim;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0, a4 = 0.0;
    for (int q = 0; q < int(blockDim.x + 31) / 32; ++q) {
      a0 = fmax(a0, wr[q][0]);
      a1 = fmax(a1, wr[q][1]);
      a2 += wr[q][2];
      a3 += wr[q][3];
      a4 += wr[q][4];
    }
    s.rowpart[rp_index(0, il, tn, s.rows, s.ntn)] = a3;
    s.rowpart[rp_index(1, il, tn, s.rows, s.ntn)] = 0.0;
    s.rowpart[rp_index(2, il, tn, s.rows, s.ntn)] = 0.0;
    s.rowpart[rp_index(3, il, tn, s.rows, s.ntn)] = a4;
    double* tp = s.tilepart + size_t(blockIdx.y * gridDim.x + tn) * 4;
    tp[0] = a0;
    tp[1] = a1;
    tp[2] = a2;
    tp[3] = 0.0;
  }
}

// ------------------------------------------------------------- host side ----

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// Row-major [dim1 x dim0] doubles with leading dimension ld, box [box1 x 16], 128B swizzle.
int make_tmap_rowmajor(CUtensorMap* out, const double* base, int64_t dim0, int64_t dim1, int64_t ld,
                       int box1) {
  auto enc = get_encode();
  if (!enc) return -1;
  cuuint64_t dims[2] = {cuuint64_t(dim0), cuuint64_t(dim1)};
  cuuint64_t strides[1] = {cuuint64_t(ld) * sizeof(double)};
  cuuint32_t box[2] = {16u, cuuint32_t(box1)};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = enc(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box,
                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : int(r);
}

template <class C>
static int tile_n() { return C::BN; }

int dense_tile_n(int cfg) { return cfg == 0 ? CfgSmall::BN : (cfg == 1 ? CfgBig::BN : CfgMid::BN); }
int dense_tile_m(int cfg) { return cfg == 0 ? CfgSmall::BM : (cfg == 1 ? CfgBig::BM : CfgMid::BM); }

// Tile configuration for a problem size: 64x64 below n = 2048 (enough CTAs to
// fill 148 SMs), otherwise 128x64 with two CTAs per SM (c2 n = 4096: 3.93 ms /
// 94.3 % of the DMMA peak vs 4.21 ms / 87.8 % for 128x128 with one CTA per SM,
// whose epilogue leaves the tensor pipe idle) -- unless the 64x64 tiles put
// fewer 64x64 units on the busiest SM: a 1024-row shard of n = 4096 (the 4-way
// sharded c2) has 512 128x64 tiles (4 on some SMs = 8 units) but 1024 64x64
// tiles (7 units): 1.03 vs 1.15 ms per step (profiles/r01e_shard_times.txt).
// DPT_DENSE_CFG=0/1/2 forces a configuration.
int dense_cfg_for(int64_t n, int64_t rows) {
  if (const char* e = getenv("DPT_DENSE_CFG")) {
    const int v = atoi(e);
    return (v == 0 || v == 1 || v == 2) ? v : 2;
  }
  if (n < 2048) return 0;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const int64_t cols = (n + 63) / 64;
  const int64_t t2 = (rows + CfgMid::BM - 1) / CfgMid::BM * cols, t0 = (rows + CfgSmall::BM - 1) / CfgSmall::BM * cols;
  const int64_t u2 = 2 * ((t2 + sms - 1) / sms), u0 = (t0 + sms - 1) / sms;  // 64x64 units on the busiest SM
  return u0 < u2 ? 0 : 2;
}

// Resident CTAs of the stream-K kernel (its persistent grid).
template <class C, bool CPLX>
static int sk_grid() {
  static int g = 0;
  if (!g) {
    cudaFuncSetAttribute(dense_step_sk_kernel<C, CPLX>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    int per_sm = 0, dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dense_step_sk_kernel<C, CPLX>, C::THREADS, C::SMEM);
    g = (per_sm > 0 ? per_sm : 1) * (sms > 0 ? sms : 148);
  }
  return g;
}

int dense_sk_grid(int) { return sk_grid<CfgSmall, true>(); }
size_t dense_sk_part_doubles() { return size_t(CfgSmall::NCW) * CfgSmall::MB * CfgSmall::NB * 64; }

template <class C>
static cudaError_t launch_cfg(const DevSolve& s, const CUtensorMap* amaps, const CUtensorMap* dmap,
                             const double* delta, cudaStream_t st) {
  const int ntm = int((s.rows + C::BM - 1) / C::BM);
  if constexpr (std::is_same<C, CfgSmall>::value) {
    // stream-K (workspace allocated by make_work) where it measured faster:
    // complex small problems (c1 complex: 0.344 vs 0.366 ms); real c1 is faster
    // one tile per CTA (0.088 vs 0.101 ms).  Every CTA must own >= 1 unit, and
    // a few units per CTA keep the part count per tile small.
    const int64_t units = int64_t(ntm) * s.ntn * ((s.ncol + C::BK - 1) / C::BK);
    if (s.sk_ws && s.cplx && units >= 4 * int64_t(sk_grid<C, true>())) {
      dense_step_sk_kernel<C, true><<<sk_grid<C, true>(), C::THREADS, C::SMEM, st>>>(s, amaps, dmap, delta, ntm);
      return cudaGetLastError();
    }
  }
  if (s.cplx) {
    static DeviceAttrOnce attr;
    attr([] { cudaFuncSetAttribute(dense_step_kernel<C, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM); });
    dense_step_kernel<C, true><<<ntm * s.ntn, C::THREADS, C::SMEM, st>>>(s, amaps, dmap, delta, ntm);
  } else {
    static DeviceAttrOnce attr;
    attr([] { cudaFuncSetAttribute(dense_step_kernel<C, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM); });
    dense_step_kernel<C, false><<<ntm * s.ntn, C::THREADS, C::SMEM, st>>>(s, amaps, dmap, delta, ntm);
  }
  return cudaGetLastError();
}

cudaError_t launch_dense_step(const DevSolve& s, const CUtensorMap* amaps, const CUtensorMap* dmap,
                              const double* delta, int cfg, cudaStream_t st) {
  if (cfg == 0) {
    // real problems: 8 warps of 32x16 at 2 CTAs/SM (c1 K1 89.0 vs 91.1 us for
    // 4 warps of 32x32 at 3 CTAs/SM: more independent DMMA chains per
    // scheduler); DPT_SMALL8=0 selects the 4-warp layout
    static const bool small8 = [] {
      const char* e = getenv("DPT_SMALL8");
      return !(e && e[0] == '0');
    }();
    if (small8 && !s.cplx) return launch_cfg<CfgSmall8>(s, amaps, dmap, delta, st);
    return launch_cfg<CfgSmall>(s, amaps, dmap, delta, st);
  }
  if (cfg == 2) return launch_cfg<CfgMid>(s, amaps, dmap, delta, st);
  return launch_cfg<CfgBig>(s, amaps, dmap, delta, st);
}

// K1's dense B operand from the caller's Delta (src, n x n, row-major; complex
// interleaved when cx = 2), optionally given transposed (the reference's
// cached delta_t): real -> dst[j][k] = Delta(j, k) (ld ldd); complex -> the
// 2n x 2n real image (rows 2j, 2j+1 = (Re, -Im), (Im, Re) of Delta(j, k)).
// 32 x 32 tiles through shared memory, so both the transposed reads and the
// writes are coalesced.
__global__ void __launch_bounds__(256) delta_image_kernel(const double* __restrict__ src, int64_t n, int cx,
                                                            int transposed, double* __restrict__ dst, int64_t ldd) {
  __shared__ double2 tile[32][33];
  const int64_t j0 = int64_t(blockIdx.y) * 32, k0 = int64_t(blockIdx.x) * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  for (int r = ty; r < 32; r += 8) {
    // element (j, k) of Delta = src[j][k], or src[k][j] when transposed; stage it at tile[jj][kk]
    const int64_t a = transposed ? k0 + r : j0 + r, b = transposed ? j0 + tx : k0 + tx;  // src row a, col b
    double2 v = make_double2(0.0, 0.0);
    if (a < n && b < n) v = cx == 2 ? reinterpret_cast<const double2*>(src)[a * n + b] : make_double2(src[a * n + b], 0.0);
    if (transposed)
      tile[tx][r] = v;  // src (k0 + r, j0 + tx) = Delta(j0 + tx, k0 + r)
    else
      tile[r][tx] = v;
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int64_t j = j0 + r, kk = k0 + tx;
    if (j >= n || kk >= n) continue;
    const double2 v = tile[r][tx];
    if (cx == 2) {
      *reinterpret_cast<double2*>(dst + (2 * j) * ldd + 2 * kk) = make_double2(v.x, -v.y);
      *reinterpret_cast<double2*>(dst + (2 * j + 1) * ldd + 2 * kk) = make_double2(v.y, v.x);
    } else {
      dst[j * ldd + kk] = v.x;
    }
  }
}

cudaError_t launch_delta_image(const double* src, int64_t n, int cx, int transposed, double* dst, int64_t ldd,
                               cudaStream_t st) {
  const dim3 grid(unsigned((n + 31) / 32), unsigned((n + 31) / 32));
  delta_image_kernel<<<grid, 256, 0, st>>>(src, n, cx, transposed, dst, ldd);
  return cudaGetLastError();
}

int dense_step_ntiles(int64_t rows, int ntn, int cfg) {
  const int bm = dense_tile_m(cfg);
  return int((rows + bm - 1) / bm) * ntn;
}

int dense_init_ntiles(int64_t rows, int ntn, int cplx) {
  return cplx ? int(rows) * ntn : int((rows + 31) / 32) * ntn;
}

cudaError_t launch_dense_init(const DevSolve& s, const double* delta, int cfg, cudaStream_t st) {
  const int bn = dense_tile_n(cfg);
  if (s.cplx) {
    dim3 grid(s.ntn, unsigned(s.rows));
    if (bn == 128)
      dense_init_cplx_kernel<128><<<grid, 64, 0, st>>>(s, delta);
    else
      dense_init_cplx_kernel<64><<<grid, 32, 0, st>>>(s, delta);
    return cudaGetLastError();
  }
  dim3 grid(s.ntn, unsigned((s.rows + 31) / 32));
  if (bn == 128)
    dense_init_kernel<128><<<grid, 256, 0, st>>>(s, delta);
  else
    dense_init_kernel<64><<<grid, 256, 0, st>>>(s, delta);
  return cudaGetLastError();
}

}  // namespace dpt
