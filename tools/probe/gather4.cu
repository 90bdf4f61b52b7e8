// TMA gather4 vs LDG random-gather throughput probe (the K3 / c4 pattern:
// 2^20 rows x 16 random columns of an L2-resident 8 MB FP64 vector).
// Question: does cp.async.bulk.tensor...tile::gather4 (TMA unit, not the LSU /
// L1 tag stage) serve random 16-byte rows faster than ~1 LDG gather per SM clock?
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

template <int M>
__device__ __forceinline__ double ldz(const double* p) {
  double v;
  if constexpr (M == 0) v = __ldg(p);
  else if constexpr (M == 1) asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
  else if constexpr (M == 2) asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  else v = *p;
  return v;
}
template <int M>
__global__ void ldg_mode(const int* __restrict__ idx, const double* __restrict__ z, double* out, int64_t rows) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r = t; r < rows; r += stride) {
    const int4* ip = reinterpret_cast<const int4*>(idx + r * 16);
    int c[16];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int4 v = __ldg(ip + q);
      c[4 * q] = v.x; c[4 * q + 1] = v.y; c[4 * q + 2] = v.z; c[4 * q + 3] = v.w;
    }
    double g[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) g[q] = ldz<M>(z + c[q]);
    double acc = 0;
#pragma unroll
    for (int q = 0; q < 16; ++q) acc += g[q];
    out[r] = acc;
  }
}
template <int M>
void run_mode(const int* idx, const double* z, double* out, int64_t rows, const char* name) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int bps : {4, 8}) {
    int blocks = 148 * bps;
    float ms;
    ldg_mode<M><<<blocks, 256>>>(idx, z, out, rows);
    cudaEventRecord(e0);
    for (int r = 0; r < 10; ++r) ldg_mode<M><<<blocks, 256>>>(idx, z, out, rows);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 10;
    printf("%-26s blocks/SM %d: %.1f us  %.1f Ggather/s\n", name, bps, ms * 1e3, rows * 16 / ms / 1e6);
  }
}

__global__ void ldg_gather(const int* __restrict__ idx, const double* __restrict__ z, double* out, int64_t rows) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r = t; r < rows; r += stride) {
    const int4* ip = reinterpret_cast<const int4*>(idx + r * 16);
    int c[16];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int4 v = __ldg(ip + q);
      c[4 * q] = v.x; c[4 * q + 1] = v.y; c[4 * q + 2] = v.z; c[4 * q + 3] = v.w;
    }
    double g[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) g[q] = __ldg(z + c[q]);
    double acc = 0;
#pragma unroll
    for (int q = 0; q < 16; ++q) acc += g[q];
    out[r] = acc;
  }
}

// One thread per row: 4 gather4 instructions fetch the 16-byte pairs holding
// its 16 columns into its own 256 B of shared memory; one mbarrier per warp.
template <int ROWB>  // doubles per gathered row (2 = 16 B, 4 = 32 B)
__global__ void __launch_bounds__(256) tma_gather(const __grid_constant__ CUtensorMap zmap, const int* __restrict__ idx,
                                                  double* out, int64_t rows) {
  extern __shared__ __align__(128) double sbuf[];
  __shared__ __align__(8) uint64_t bar[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(&bar[warp])), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncwarp();
  constexpr int SLOT = 16;  // doubles per gather4 destination: TMA wants 128-byte aligned smem
  double* my = sbuf + size_t(threadIdx.x) * 4 * SLOT;
  uint32_t phase = 0;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r0 = blockIdx.x * (int64_t)blockDim.x; r0 < rows; r0 += stride) {
    const int64_t r = r0 + threadIdx.x;
    const int4* ip = reinterpret_cast<const int4*>(idx + r * 16);
    int c[16];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int4 v = __ldg(ip + q);
      c[4 * q] = v.x; c[4 * q + 1] = v.y; c[4 * q + 2] = v.z; c[4 * q + 3] = v.w;
    }
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(&bar[warp])),
                   "r"(32 * 16 * ROWB * 8) : "memory");
    __syncwarp();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
          :
          : "r"(smem_u32(my + q * SLOT)), "l"(&zmap), "r"(smem_u32(&bar[warp])), "r"(0),
            "r"(c[4 * q] / ROWB), "r"(c[4 * q + 1] / ROWB), "r"(c[4 * q + 2] / ROWB), "r"(c[4 * q + 3] / ROWB)
          : "memory");
    }
    // wait
    asm volatile(
        "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(
            smem_u32(&bar[warp])),
        "r"(phase)
        : "memory");
    phase ^= 1;
    double acc = 0;
#pragma unroll
    for (int q = 0; q < 16; ++q) acc += my[(q >> 2) * SLOT + (q & 3) * ROWB + (c[q] % ROWB)];
    out[r] = acc;
    __syncwarp();
  }
}

int main() {
  const int64_t n = 1 << 20, rows = n, nnz = rows * 16;
  int* idx;
  double *z, *out, *ref;
  cudaMalloc(&idx, nnz * 4);
  cudaMalloc(&z, n * 8);
  cudaMalloc(&out, rows * 8);
  cudaMalloc(&ref, rows * 8);
  int* h = (int*)malloc(nnz * 4);
  double* hz = (double*)malloc(n * 8);
  uint64_t s = 88172645463325252ull;
  for (int64_t i = 0; i < nnz; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = (int)(s % n); }
  for (int64_t i = 0; i < n; ++i) hz[i] = double(i % 1000) * 0.5;
  cudaMemcpy(idx, h, nnz * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(z, hz, n * 8, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  for (int bps : {4, 8}) {
    int blocks = 148 * bps;
    ldg_gather<<<blocks, 256>>>(idx, z, ref, rows);
    cudaEventRecord(e0);
    for (int r = 0; r < 10; ++r) ldg_gather<<<blocks, 256>>>(idx, z, ref, rows);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 10;
    printf("ldg  gather blocks/SM %d: %.1f us  %.1f Ggather/s\n", bps, ms * 1e3, nnz / ms / 1e6);
  }
  run_mode<0>(idx, z, out, rows, "ldg (nc)");
  run_mode<1>(idx, z, out, rows, "ld.global.cg");
  run_mode<2>(idx, z, out, rows, "ld.nc.L1::no_allocate");
  run_mode<3>(idx, z, out, rows, "ld (generic)");
  if (getenv("NO_TMA")) return 0;
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
  double* hr = (double*)malloc(rows * 8);
  double* ho = (double*)malloc(rows * 8);
  cudaMemcpy(hr, ref, rows * 8, cudaMemcpyDeviceToHost);
  for (int rb : {2, 4}) {
    CUtensorMap m;
    cuuint64_t dims[2] = {cuuint64_t(rb), cuuint64_t(n / rb)};
    cuuint64_t strides[1] = {cuuint64_t(rb * 8)};
    cuuint32_t box[2] = {cuuint32_t(rb), 1u};
    cuuint32_t es[2] = {1u, 1u};
    CUresult cr = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, z, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) { printf("encode rb=%d failed %d\n", rb, int(cr)); continue; }
    const int smem = 256 * 4 * 16 * 8;
    for (int bps : {1}) {
      if (smem * bps > 220 * 1024) continue;
      int blocks = 148 * bps;
      cudaError_t err;
      if (rb == 2) {
        cudaFuncSetAttribute(tma_gather<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        tma_gather<2><<<blocks, 256, smem>>>(m, idx, out, rows);
        cudaEventRecord(e0);
        for (int r = 0; r < 10; ++r) tma_gather<2><<<blocks, 256, smem>>>(m, idx, out, rows);
      } else {
        cudaFuncSetAttribute(tma_gather<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        tma_gather<4><<<blocks, 256, smem>>>(m, idx, out, rows);
        cudaEventRecord(e0);
        for (int r = 0; r < 10; ++r) tma_gather<4><<<blocks, 256, smem>>>(m, idx, out, rows);
      }
      cudaEventRecord(e1);
      err = cudaEventSynchronize(e1);
      if (err != cudaSuccess) { printf("tma rb=%d err %s\n", rb, cudaGetErrorString(err)); return 1; }
      cudaEventElapsedTime(&ms, e0, e1);
      ms /= 10;
      cudaMemcpy(ho, out, rows * 8, cudaMemcpyDeviceToHost);
      int bad = 0;
      for (int64_t i = 0; i < rows; ++i) bad += ho[i] != hr[i];
      printf("tma gather4 rowbytes %d blocks/SM %d: %.1f us  %.1f Ggather/s  mismatches %d\n", rb * 8, bps, ms * 1e3,
             nnz / ms / 1e6, bad);
    }
  }
  return 0;
}
