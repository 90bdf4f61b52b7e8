// dense_mma.cuh -- the FP64 tensor-core (DMMA) tile machinery shared by K1
// (dense_step.cu, the fused DPT step) and the plain GEMM of the device
// homotopy (linalg.cu): CTA tile configurations and the consumption of one
// TMA-staged k-tile (BK = 16 doubles, SWIZZLE_128B) by the consumer warps.
#pragma once
#include <stdint.h>

#include "dpt_device.cuh"

namespace dpt {

template <int BM_, int BN_, int WARPS_M_, int WARPS_N_, int MINB_ = 1>
struct DenseCfg {
  static constexpr int BM = BM_, BN = BN_, WARPS_M = WARPS_M_, WARPS_N = WARPS_N_, MINB = MINB_;
  static constexpr int BK = 16;  // 16 doubles = 128 B rows = one swizzle span
  static constexpr int STAGES = 4;
  static constexpr int NCW = WARPS_M * WARPS_N;  // consumer warps
  static constexpr int THREADS = NCW * 32;  // lane 0 of warp 0 doubles as the TMA producer
  static constexpr int WTM = BM / WARPS_M, WTN = BN / WARPS_N;
  static constexpr int MB = WTM / 8, NB = WTN / 8;
  static constexpr int A_BYTES = BM * BK * 8, B_BYTES = BN * BK * 8;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int RED_BYTES = WARPS_N * BM * 4 * 8 + NCW * 4 * 8;
  static constexpr int SMEM = STAGES * STAGE_BYTES + RED_BYTES + 2 * STAGES * 8 + 1024;
};

using CfgBig = DenseCfg<128, 128, 2, 4>;      // cfg 1: one CTA per SM
using CfgSmall = DenseCfg<64, 64, 2, 2, 3>;   // cfg 0: n < 2048 (enough CTAs for 148 SMs), 3 CTAs/SM
using CfgSmall8 = DenseCfg<64, 64, 2, 4, 2>;  // cfg 0, real: the same tiles with 8 warps of 32x16
using CfgMid = DenseCfg<128, 64, 4, 2, 2>;    // cfg 2: two CTAs per SM -> one CTA's epilogue
                                              //        overlaps the other's DMMA mainloop

// Byte offset of 16-byte chunk `chunk` of row `r` in a SWIZZLE_128B TMA box
// with 128-byte rows.
__device__ __forceinline__ uint32_t swz(int r, int chunk) {
  return uint32_t(r) * 128u + uint32_t((chunk ^ (r & 7)) << 4);
}

// One BK = 16 k-tile of the staged A (BM x 16) and B (BN x 16) boxes into the
// warp's accumulators acc[a][b][0..1] = C(row wm*WTM + 8a + gq, cols wn*WTN +
// 8b + 2t, +1).  The two k4-steps of a 16-byte chunk come from one LDS.128: the
// k index is permuted identically for both operands, so the sum is unchanged.
template <class C>
__device__ __forceinline__ void dmma_consume_stage(double (&acc)[C::MB][C::NB][2], const uint8_t* a_st,
                                                   const uint8_t* b_st, int wm, int wn, int t, int gq) {
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    // Row r = base + 8x + gq has (r & 7) == gq, so the swizzled chunk offset is
    // the same for every fragment of this lane: per-fragment addresses differ
    // by immediates (x * 1024 bytes).
    const uint32_t cofs = uint32_t(((4 * q + t) ^ gq) << 4) + uint32_t(gq) * 128u;
    const uint32_t pa = smem_u32(a_st) + uint32_t(wm * C::WTM * 128) + cofs;
    const uint32_t pb = smem_u32(b_st) + uint32_t(wn * C::WTN * 128) + cofs;
    // B fragments for both k4-steps of this 16-byte chunk stay live; A
    // fragments stream through (keeps the 64-double accumulator + operands
    // within the register budget).
    double2 bf[C::NB];
#pragma unroll
    for (int b = 0; b < C::NB; ++b) bf[b] = lds128(pb + b * 1024);
#pragma unroll
    for (int a = 0; a < C::MB; ++a) {
      const double2 af = lds128(pa + a * 1024);
#pragma unroll
      for (int b = 0; b < C::NB; ++b) dmma_8x8x4(acc[a][b][0], acc[a][b][1], af.x, bf[b].x);
#pragma unroll
      for (int b = 0; b < C::NB; ++b) dmma_8x8x4(acc[a][b][0], acc[a][b][1], af.y, bf[b].y);
    }
  }
}

}  // namespace dpt
