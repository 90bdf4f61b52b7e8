// single_u16.cu -- K3 for a CSR perturbation with exactly 16 nonzeros per row
// (BASELINE configs[3], c4): the row map step of run_single
// (proj/src/dpt.cpp:233-289) with w = matvec(delta, z) (src/matrix.cpp:215-225).
//
// HBM-bound stream + L2-resident random gathers of z.  A block takes 256 rows
// per trip; their CSR slices are CONTIGUOUS (16 columns + 16 values per row),
// so one thread issues two cp.async.bulk copies (16 KiB of columns, 32 KiB of
// values) into a double-buffered shared-memory stage while the block works on
// the previous trip.  Each thread then owns one row: 16 independent z gathers
// in flight, then the FMA chain in CSR order (bit-identical to the w[row] every
// block recomputes for the map's w[row] term).  Shared reads are rotated per
// lane ((q + lane) mod chunks) so the 64-/128-byte row strides are
// conflict-free.
#include <cuda_runtime.h>
#include <stdint.h>

#include "dpt_device.cuh"
#include "dpt_kernels.h"

namespace dpt {

constexpr int kU16Rows = 256;  // rows (= threads) per trip
constexpr int kU16Stages = 2;
constexpr int kU16ColBytes = kU16Rows * 16 * 4;
constexpr int kU16ValBytes = kU16Rows * 16 * 8;
constexpr int kU16StageBytes = kU16ColBytes + kU16ValBytes;
constexpr int kU16Smem = kU16Stages * kU16StageBytes + 64;

// w_m = sum_q vals[16m + q] * z[cols[16m + q]], q = 0..15 in order.
__device__ __forceinline__ double u16_dot(const int32_t* c, const double* v, const double* __restrict__ z) {
  double zg[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) zg[q] = z[c[q]];
  double w = 0.0;
#pragma unroll
  for (int q = 0; q < 16; ++q) w = __fma_rn(v[q], zg[q], w);
  return w;
}

__global__ void __launch_bounds__(kU16Rows, 2)
    single_u16_kernel(DevSolve s, DevCsr D, int64_t row, int64_t ntrips) {
  if (s.state->done) return;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t bar[kU16Stages];
  __shared__ double wrow_s;
  __shared__ double red[kU16Rows / 32][5];
  const int jl = launch_index(s);
  const int64_t n = s.n;
  const double* __restrict__ z = s.slots + size_t((jl - 1) % s.nslots) * size_t(s.slot_elems);
  double* __restrict__ zo = s.slots + size_t(jl % s.nslots) * size_t(s.slot_elems);
  const double lam_k = lam_of(s, jl), lam = s.lambda;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  if (tid == 0) {
    for (int i = 0; i < kU16Stages; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](int64_t trip, int st) {
    const int64_t r0 = trip * kU16Rows;
    const int64_t nr = (n - r0) < kU16Rows ? (n - r0) : kU16Rows;
    uint8_t* base = smem + st * kU16StageBytes;
    mbar_arrive_expect_tx(&bar[st], uint32_t(nr * 16 * 12));
    bulk_load(base, D.cols + 16 * r0, uint32_t(nr * 16 * 4), &bar[st]);
    bulk_load(base + kU16ColBytes, D.vals + 16 * r0, uint32_t(nr * 16 * 8), &bar[st]);
  };
  int64_t trip = blockIdx.x;
  if (tid == 0 && trip < ntrips) issue(trip, 0);

  if (tid == 0) {  // w[row] of z_{j-1}: same order as the per-row dot
    int32_t c[16];
    double v[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      c[q] = D.cols[16 * row + q];
      v[q] = D.vals[16 * row + q];
    }
    const double wr = u16_dot(c, v, z);
    wrow_s = wr;
    if (blockIdx.x == 0) s.dvec[(jl - 1) & 1][0] = wr;  // for the fold's eps
  }
  __syncthreads();
  const double wr = wrow_s;
  const double trow = s.theta[row];
  const double eps = __dadd_rn(trow, __dmul_rn(lam, wr));
  double num = 0.0, den = 0.0, t_step = 0.0, t_max = 0.0, t_nonfin = 0.0;

  for (int it = 0; trip < ntrips; ++it, trip += gridDim.x) {
    const int st = it & 1;
    const int64_t next = trip + gridDim.x;
    if (tid == 0 && next < ntrips) issue(next, st ^ 1);  // stage st^1 was released by the barrier below
    mbar_wait(&bar[st], (it >> 1) & 1);
    const int64_t m = trip * kU16Rows + tid;
    if (m < n) {
      const uint8_t* base = smem + st * kU16StageBytes;
      const int4* crow = reinterpret_cast<const int4*>(base + size_t(tid) * 64);
      const double2* vrow = reinterpret_cast<const double2*>(base + kU16ColBytes + size_t(tid) * 128);
      int32_t c[16];
      double v[16];
#pragma unroll
      for (int q = 0; q < 4; ++q) {  // rotated chunk order: conflict-free 64-byte row stride
        const int k = (q + lane) & 3;
        const int4 t = crow[k];
        // place into c[4k..4k+3] without dynamic register indexing
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          if (kk == k) {
            c[4 * kk + 0] = t.x;
            c[4 * kk + 1] = t.y;
            c[4 * kk + 2] = t.z;
            c[4 * kk + 3] = t.w;
          }
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int k = (q + lane) & 7;
        const double2 t = vrow[k];
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          if (kk == k) {
            v[2 * kk + 0] = t.x;
            v[2 * kk + 1] = t.y;
          }
      }
      const double w = u16_dot(c, v, z);
      const double zm = z[m];
      const double tm = s.theta[m];
      double val;
      if (m == row) {
        val = 1.0;
      } else {
        const double g = s.gapmat ? s.gapmat[m] : 1.0 / __dsub_rn(trow, tm);  // build_gap_row, partition.cpp:83-96
        val = __dmul_rn(__dmul_rn(lam_k, g), __dsub_rn(w, __dmul_rn(wr, zm)));
      }
      zo[m] = val;
      t_step = fmax(t_step, fabs(__dsub_rn(val, zm)));
      t_max = fmax(t_max, fabs(val));
      t_nonfin += isfinite(val) ? 0.0 : 1.0;
      const double r = __dadd_rn(__dmul_rn(__dsub_rn(tm, eps), zm), __dmul_rn(lam, w));
      num = fmax(num, fabs(r));
      den = fmax(den, fabs(zm));
    }
    __syncthreads();  // every thread is done with stage st before it is refilled
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
  if (tid == 0) {
    double a[5] = {0, 0, 0, 0, 0};
    for (int ww = 0; ww < kU16Rows / 32; ++ww) {
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

int u16_grid(int64_t n) {
  const int64_t trips = (n + kU16Rows - 1) / kU16Rows;
  const int64_t g = 148 * 2;
  return int(trips < g ? (trips < 1 ? 1 : trips) : g);
}

cudaError_t launch_single_u16(const DevSolve& s, const DevCsr& d, int64_t row, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(single_u16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kU16Smem);
    attr = true;
  }
  const int64_t trips = (s.n + kU16Rows - 1) / kU16Rows;
  single_u16_kernel<<<u16_grid(s.n), kU16Rows, kU16Smem, st>>>(s, d, row, trips);
  return cudaGetLastError();
}

}  // namespace dpt
