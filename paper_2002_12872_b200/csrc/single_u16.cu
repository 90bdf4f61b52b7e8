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
#include <stdlib.h>

#include "dpt_device.cuh"
#include "dpt_kernels.h"

namespace dpt {

constexpr int kU16Stages = 2;
template <int ROWS>
struct U16 {
  static constexpr int ColBytes = ROWS * 16 * 4;
  static constexpr int ValBytes = ROWS * 16 * 8;
  static constexpr int StageBytes = ColBytes + ValBytes;
  static constexpr int Smem = kU16Stages * StageBytes + 64;
};

// Canonical order, select-based placement (no lane rotation of the dot).
__device__ __forceinline__ double u16_dot_sel(const int4* crow, const double2* vrow, int lane,
                                              const double* __restrict__ z) {
  int32_t c[16];
  double v[16];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int k = (q + lane) & 3;
    const int4 t = crow[k];
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
  double zg[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) zg[q] = z[c[q]];
  double w = 0.0;
#pragma unroll
  for (int q = 0; q < 16; ++q) w = __fma_rn(v[q], zg[q], w);
  return w;
}

// Row dot in the lane-rotated chunk order used everywhere for this row:
// chunks of 4 columns are visited in the order k = (q + rot / 2) & 3 (rot = the
// row's lane), which makes the shared-memory reads conflict-free.  Every
// evaluation of a given row -- including the w[row] that each block needs --
// uses the same rot, so the value is bit-identical.  Split into the staged
// loads (u16_load_rot) and the gathers + FMA chain (u16_gather_dot) so the
// per-warp pipeline can release its stage between the two.
struct U16Row {
  int4 c[4];
  double2 va[4], vb[4];
};

__device__ __forceinline__ U16Row u16_load_rot(const int4* crow, const double2* vrow, int rot) {
  U16Row r;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    // A quarter-warp (8 lanes) shares one 128-byte wavefront of a 16-byte
    // load.  Lanes l, l^1 have column rows 64 bytes apart, so chunk k = (q +
    // l/2) & 3 puts the 8 lanes on 8 distinct 16-byte slots; values 4k..4k+3
    // are 16-byte chunks 2k, 2k+1 of a 128-byte row, read first-chunk f = l & 1,
    // again 8 distinct slots.  (Rotating by l itself left the column loads
    // 2-way conflicted: 0.5 M extra wavefronts per c4 step.)
    const int k = (q + (rot >> 1)) & 3;
    r.c[q] = crow[k];
    const int f = rot & 1;
    const double2 x0 = vrow[2 * k + f], x1 = vrow[2 * k + (f ^ 1)];
    r.va[q] = f ? x1 : x0;
    r.vb[q] = f ? x0 : x1;
  }
  return r;
}

// Gather through L1 without allocating a line (tuning variant).
__device__ __forceinline__ double ld_na(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

template <bool NA = false>
__device__ __forceinline__ double u16_gather_dot(const U16Row& r, const double* __restrict__ z) {
  double zg[16];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if (NA) {
      zg[4 * q + 0] = ld_na(z + r.c[q].x);
      zg[4 * q + 1] = ld_na(z + r.c[q].y);
      zg[4 * q + 2] = ld_na(z + r.c[q].z);
      zg[4 * q + 3] = ld_na(z + r.c[q].w);
    } else {
      zg[4 * q + 0] = z[r.c[q].x];
      zg[4 * q + 1] = z[r.c[q].y];
      zg[4 * q + 2] = z[r.c[q].z];
      zg[4 * q + 3] = z[r.c[q].w];
    }
  }
  double w = 0.0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    w = __fma_rn(r.va[q].x, zg[4 * q + 0], w);
    w = __fma_rn(r.va[q].y, zg[4 * q + 1], w);
    w = __fma_rn(r.vb[q].x, zg[4 * q + 2], w);
    w = __fma_rn(r.vb[q].y, zg[4 * q + 3], w);
  }
  return w;
}

__device__ __forceinline__ double u16_dot_rot(const int4* crow, const double2* vrow, int rot,
                                              const double* __restrict__ z) {
  return u16_gather_dot(u16_load_rot(crow, vrow, rot), z);
}

template <int ROWS, int MINB, bool ROT>
__global__ void __launch_bounds__(ROWS, MINB)
    single_u16_kernel(DevSolve s, DevCsr D, int64_t row, int64_t ntrips) {
  constexpr int kU16Rows = ROWS;
  constexpr int kU16ColBytes = U16<ROWS>::ColBytes;
  constexpr int kU16StageBytes = U16<ROWS>::StageBytes;
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

  if (tid == 0) {  // w[row] of z_{j-1}, in the rotation of the lane that owns row
    const int4* cr = reinterpret_cast<const int4*>(D.cols + 16 * row);
    const double2* vr = reinterpret_cast<const double2*>(D.vals + 16 * row);
    const double wr = ROT ? u16_dot_rot(cr, vr, int(row & 31), z) : u16_dot_sel(cr, vr, int(row & 31), z);
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
    if (tid == 0 && next < ntrips) {  // stage st^1 was released by the barrier below
      fence_proxy_async_smem();          // its generic reads before the async-proxy refill
      issue(next, st ^ 1);
    }
    mbar_wait(&bar[st], (it >> 1) & 1);
    const int64_t m = trip * kU16Rows + tid;
    if (m < n) {
      const uint8_t* base = smem + st * kU16StageBytes;
      const double zm = z[m];  // issued before the gathers
      const double tm = s.theta[m];
      const int4* cr = reinterpret_cast<const int4*>(base + size_t(tid) * 64);
      const double2* vr = reinterpret_cast<const double2*>(base + kU16ColBytes + size_t(tid) * 128);
      const double w = ROT ? u16_dot_rot(cr, vr, int(m & 31), z) : u16_dot_sel(cr, vr, int(m & 31), z);
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

// Per-warp pipeline variant: each warp streams its own 32-row trips (2 KiB of
// columns + 4 KiB of values per trip, one cp.async.bulk pair issued by lane 0)
// through an S-deep private ring with its own mbarriers, and releases a stage
// as soon as its lanes hold the row in registers (__syncwarp), before the
// gathers.  No block-wide barrier inside the loop: warps drift freely, so the
// L1's random-gather queue stays fed while other warps wait on L2.  Rows are
// the same lane-rotated dots as above (trip = 32 rows, so rot = m & 31 = lane).
template <int W, int S>
struct U16W {
  static constexpr int TripBytes = 32 * 16 * 12;  // 6 KiB
  static constexpr int Smem = W * S * TripBytes;
};

template <int W, int S, int MINB, bool NA = false>
__global__ void __launch_bounds__(W * 32, MINB)
    single_u16w_kernel(DevSolve s, DevCsr D, int64_t row, int64_t ntrips) {
  constexpr int kTrip = U16W<W, S>::TripBytes;
  if (s.state->done) return;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t bar[W][S];    // full: the trip's bulk copies landed
  __shared__ uint64_t empty[W][S];  // empty: all 32 lanes hold the trip in registers
  __shared__ double red[W][5];
  const int jl = launch_index(s);
  const int64_t n = s.n;
  const double* __restrict__ z = s.slots + size_t((jl - 1) % s.nslots) * size_t(s.slot_elems);
  double* __restrict__ zo = s.slots + size_t(jl % s.nslots) * size_t(s.slot_elems);
  const double lam_k = lam_of(s, jl), lam = s.lambda;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint8_t* ring = smem + size_t(warp) * S * kTrip;
  const int64_t stride = int64_t(gridDim.x) * W;
  int64_t t = int64_t(blockIdx.x) * W + warp;

  auto issue = [&](int64_t trip, int st) {
    const int64_t r0 = trip * 32;
    const int64_t nr = (n - r0) < 32 ? (n - r0) : 32;
    uint8_t* base = ring + st * kTrip;
    mbar_arrive_expect_tx(&bar[warp][st], uint32_t(nr * 16 * 12));
    bulk_load(base, D.cols + 16 * r0, uint32_t(nr * 16 * 4), &bar[warp][st]);
    bulk_load(base + 32 * 64, D.vals + 16 * r0, uint32_t(nr * 16 * 8), &bar[warp][st]);
  };
  if (lane == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&bar[warp][i], 1);
      mbar_init(&empty[warp][i], 32);
    }
    fence_mbar_init();
    for (int i = 0; i < S; ++i)
      if (t + i * stride < ntrips) issue(t + i * stride, i);
  }
  __syncwarp();
  // w[row] of z_{j-1} in the rotation of the lane that owns row; every lane
  // evaluates it (uniform addresses: one sector per load) while the first
  // trips are in flight
  const double wr = u16_dot_rot(reinterpret_cast<const int4*>(D.cols + 16 * row),
                                reinterpret_cast<const double2*>(D.vals + 16 * row), int(row & 31), z);
  if (blockIdx.x == 0 && threadIdx.x == 0) s.dvec[(jl - 1) & 1][0] = wr;  // for the fold's eps
  const double trow = s.theta[row];
  const double eps = __dadd_rn(trow, __dmul_rn(lam, wr));
  double num = 0.0, den = 0.0, t_step = 0.0, t_max = 0.0, t_nonfin = 0.0;

  for (int it = 0; t < ntrips; ++it, t += stride) {
    const int st = it % S;
    mbar_wait(&bar[warp][st], uint32_t(it / S) & 1u);
    const int64_t m = t * 32 + lane;
    const uint8_t* base = ring + st * kTrip;
    U16Row rd = {};
    if (m < n)
      rd = u16_load_rot(reinterpret_cast<const int4*>(base + lane * 64),
                        reinterpret_cast<const double2*>(base + 32 * 64 + lane * 128), lane);
    // WAR handshake: every lane releases the stage after its reads; lane 0
    // acquires that phase, then fences generic -> async proxy before the refill
    mbar_arrive_release(&empty[warp][st]);
    if (lane == 0 && t + S * stride < ntrips) {
      mbar_wait(&empty[warp][st], uint32_t(it / S) & 1u);
      fence_proxy_async_smem();
      issue(t + S * stride, st);
    }
    if (m < n) {
      const double zm = z[m];
      const double tm = s.theta[m];
      const double w = u16_gather_dot<NA>(rd, z);
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
    for (int ww = 0; ww < W; ++ww) {
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

// Variant table (DPT_U16_VARIANT selects one for tuning runs).  Measured on c4
// (profiles/r01f_k3_sweep.txt): block-staged trips 98 us (1), 109 us (0); per-warp
// rings with two stages 91-92 us (6, 8, 10), with one stage 83.3-84.9 us (11,
// 16-18; default 16).  Making the column loads bank-conflict-free (rotation by
// lane / 2) removed 0.53 M shared wavefronts per step and left the time
// unchanged.  The binding unit is the L1's sector rate for the gathers, and
// every byte of shared memory taken from it costs in-flight gather capacity:
// forcing the maximum shared carveout slows every variant to ~146 us, as do
// configurations that need > 196 KB.
struct U16Variant {
  int rows, minb, rot;
};
static const U16Variant kU16Var[] = {{256, 2, 0}, {256, 2, 1}, {128, 4, 0}, {128, 4, 1}, {128, 6, 1}, {64, 8, 1},
                                     // per-warp pipelines (rows = 32 * warps per block)
                                     {256, 2, 1}, {192, 3, 1}, {512, 1, 1}, {128, 3, 1}, {160, 3, 1},
                                     {256, 2, 1}, {192, 3, 1}, {160, 4, 1}, {128, 5, 1}, {128, 4, 1},
                                     {512, 1, 1}, {160, 3, 1}, {128, 4, 1},
                                     {256, 2, 1}, {256, 2, 1}};

static int u16_variant() {
  const char* e = getenv("DPT_U16_VARIANT");
  const int v = e ? atoi(e) : 16;  // per-warp pipeline, 16 warps x 1 block per SM, one stage: fastest on B200 (tools/u16_sweep.sh)
  return (v >= 0 && v < int(sizeof(kU16Var) / sizeof(kU16Var[0]))) ? v : 0;
}

int u16_grid(int64_t n) {
  const U16Variant& V = kU16Var[u16_variant()];
  const int64_t trips = (n + V.rows - 1) / V.rows;
  const int64_t g = 148 * V.minb;  // resident blocks
  return int(trips < g ? (trips < 1 ? 1 : trips) : g);
}

template <int W, int S, int MINB, bool NA = false>
static cudaError_t launch_u16w(const DevSolve& s, const DevCsr& d, int64_t row, cudaStream_t st) {
  static DeviceAttrOnce attr;
  attr([] {
    cudaFuncSetAttribute(single_u16w_kernel<W, S, MINB, NA>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         U16W<W, S>::Smem);
    if (getenv("DPT_U16_CARVEOUT"))  // tuning: force the shared-memory carveout (percent)
      cudaFuncSetAttribute(single_u16w_kernel<W, S, MINB, NA>, cudaFuncAttributePreferredSharedMemoryCarveout,
                           atoi(getenv("DPT_U16_CARVEOUT")));
  });
  const int64_t trips = (s.n + 31) / 32;
  single_u16w_kernel<W, S, MINB, NA><<<u16_grid(s.n), W * 32, U16W<W, S>::Smem, st>>>(s, d, row, trips);
  return cudaGetLastError();
}

template <int ROWS, int MINB, bool ROT>
static cudaError_t launch_u16(const DevSolve& s, const DevCsr& d, int64_t row, cudaStream_t st) {
  static DeviceAttrOnce attr;
  attr([] {
    cudaFuncSetAttribute(single_u16_kernel<ROWS, MINB, ROT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         U16<ROWS>::Smem);
  });
  const int64_t trips = (s.n + ROWS - 1) / ROWS;
  single_u16_kernel<ROWS, MINB, ROT><<<u16_grid(s.n), ROWS, U16<ROWS>::Smem, st>>>(s, d, row, trips);
  return cudaGetLastError();
}

// ---------------------------------------------- launch 1 from z_0 = e_row ----
// The row-map solve starts from z_0 = e_row, where w = Delta z_0 is column
// `row` of Delta: w[m] is the entry (m, row) or +0, and no gather is needed to
// know it -- only the row's 16 columns.  This kernel writes what K3's launch 1
// writes (z_1, the step / max / nonfinite and residual partials per block, w[row]
// for the fold's eps) from the columns alone (67 MB instead of 235 MB and 16.8 M
// gathers at c4: ~15 us instead of 83), with K3's own expressions: the FMA
// chain visits the row's entries in K3's order (rotated chunks when the
// variant rotates) and adds v * 1 for a match -- a skipped entry would add
// fma(v, 0, w) = w for every finite v -- so z_1 and every statistic are
// bit-identical to K3's for finite Delta.  One thread per row; the grid and the
// per-block partial layout are K3's (the fold is unchanged).
__device__ __forceinline__ double u16_dot_unit(const int32_t* __restrict__ cols, const double* __restrict__ vals,
                                               int64_t m, int rot, bool rotate, int64_t row) {
  const int4* crow = reinterpret_cast<const int4*>(cols + 16 * m);
  const double* vrow = vals + 16 * m;
  double w = 0.0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int k = rotate ? (q + (rot >> 1)) & 3 : q;
    const int4 c = __ldg(crow + k);
    if (c.x == row) w = __fma_rn(vrow[4 * k + 0], 1.0, w);
    if (c.y == row) w = __fma_rn(vrow[4 * k + 1], 1.0, w);
    if (c.z == row) w = __fma_rn(vrow[4 * k + 2], 1.0, w);
    if (c.w == row) w = __fma_rn(vrow[4 * k + 3], 1.0, w);
  }
  return w;
}

constexpr int kU16InitThreads = 1024;  // one block per SM (the grid is K3's): all the warps it can hold

__global__ void __launch_bounds__(kU16InitThreads)
    single_u16_init_kernel(DevSolve s, DevCsr D, int64_t row, int rotate) {
  if (s.state->done) return;
  __shared__ double red[kU16InitThreads / 32][5];
  const int jl = launch_index(s);
  const int64_t n = s.n;
  double* __restrict__ zo = s.slots + size_t(jl % s.nslots) * size_t(s.slot_elems);
  const double lam_k = lam_of(s, jl), lam = s.lambda;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double wr = u16_dot_unit(D.cols, D.vals, row, int(row & 31), rotate != 0, row);
  if (blockIdx.x == 0 && threadIdx.x == 0) s.dvec[(jl - 1) & 1][0] = wr;  // for the fold's eps
  const double trow = s.theta[row];
  const double eps = __dadd_rn(trow, __dmul_rn(lam, wr));
  double num = 0.0, den = 0.0, t_step = 0.0, t_max = 0.0, t_nonfin = 0.0;
  for (int64_t m = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; m < n; m += int64_t(gridDim.x) * blockDim.x) {
    const double zm = m == row ? 1.0 : 0.0;  // z_0
    const double tm = s.theta[m];
    const double w = u16_dot_unit(D.cols, D.vals, m, int(m & 31), rotate != 0, row);
    double val;
    if (m == row) {
      val = 1.0;
    } else {
      const double g = 1.0 / __dsub_rn(trow, tm);
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
    for (int ww = 0; ww < kU16InitThreads / 32; ++ww) {
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

// Launch 1 of the uniform-16 row map from z_0 = e_row (real data, gaps from the levels).
cudaError_t launch_single_u16_init(const DevSolve& s, const DevCsr& d, int64_t row, cudaStream_t st) {
  single_u16_init_kernel<<<u16_grid(s.n), kU16InitThreads, 0, st>>>(s, d, row, kU16Var[u16_variant()].rot);
  return cudaGetLastError();
}

cudaError_t launch_single_u16(const DevSolve& s, const DevCsr& d, int64_t row, cudaStream_t st) {
  switch (u16_variant()) {
    case 1: return launch_u16<256, 2, true>(s, d, row, st);
    case 2: return launch_u16<128, 4, false>(s, d, row, st);
    case 3: return launch_u16<128, 4, true>(s, d, row, st);
    case 4: return launch_u16<128, 6, true>(s, d, row, st);
    case 5: return launch_u16<64, 8, true>(s, d, row, st);
    case 6: return launch_u16w<8, 2, 2>(s, d, row, st);
    case 7: return launch_u16w<6, 2, 3>(s, d, row, st);
    case 8: return launch_u16w<16, 2, 1>(s, d, row, st);
    case 9: return launch_u16w<4, 3, 3>(s, d, row, st);
    case 10: return launch_u16w<5, 2, 3>(s, d, row, st);
    case 11: return launch_u16w<8, 1, 2>(s, d, row, st);
    case 12: return launch_u16w<6, 1, 3>(s, d, row, st);
    case 13: return launch_u16w<5, 1, 4>(s, d, row, st);
    case 14: return launch_u16w<4, 1, 5>(s, d, row, st);
    case 15: return launch_u16w<4, 2, 4>(s, d, row, st);
    case 16: return launch_u16w<16, 1, 1>(s, d, row, st);
    case 17: return launch_u16w<5, 1, 3>(s, d, row, st);
    case 18: return launch_u16w<4, 1, 4>(s, d, row, st);
    case 19: return launch_u16w<8, 1, 2, true>(s, d, row, st);
    case 20: return launch_u16w<8, 2, 2, true>(s, d, row, st);
    default: return launch_u16<256, 2, false>(s, d, row, st);
  }
}

}  // namespace dpt
