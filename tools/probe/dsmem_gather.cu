// (index loads coalesced across the warp: element q of thread t at idx[q NT + t])
// Random FP64 gathers from distributed shared memory (a z-block spread over a
// thread-block cluster) vs from L2.  Question for K3 (c4: 16.7 M random
// gathers of an 8 MB vector per step): can a cluster-resident z block serve
// random gathers faster than the ~1 gather / SM clock the L2 path gives?
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <stdint.h>

namespace cg = cooperative_groups;

constexpr int kPerCta = 24576;  // doubles of the block held by each CTA (192 KB)

template <int CS>
__global__ void __cluster_dims__(CS, 1, 1) __launch_bounds__(512, 1)
    dsmem_gather(const double* __restrict__ zblk, const uint32_t* __restrict__ idx, int64_t per_thread,
                 double* out) {
  extern __shared__ double zs[];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = int(cl.block_rank());
  for (int i = threadIdx.x; i < kPerCta; i += blockDim.x) zs[i] = zblk[size_t(rank) * kPerCta + i];
  cl.sync();
  const uint32_t base = uint32_t(__cvta_generic_to_shared(zs));
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t NT = int64_t(gridDim.x) * blockDim.x;
  const uint32_t* my = idx + t;
  double acc = 0.0;
  for (int64_t q = 0; q < per_thread; q += 16) {
    uint32_t c[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) c[u] = __ldg(my + (q + u) * NT);
    double g[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const uint32_t r = c[u] / kPerCta, o = c[u] % kPerCta;
      uint32_t addr;
      asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(addr) : "r"(base + o * 8u), "r"(r));
      asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(g[u]) : "r"(addr));
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) acc += g[u];
  }
  out[t] = acc;
  cl.sync();
}

__global__ void __launch_bounds__(512, 1) l2_gather(const double* __restrict__ z, const uint32_t* __restrict__ idx,
                                                    int64_t per_thread, double* out) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t NT = int64_t(gridDim.x) * blockDim.x;
  const uint32_t* my = idx + t;
  double acc = 0.0;
  for (int64_t q = 0; q < per_thread; q += 16) {
    uint32_t c[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) c[u] = __ldg(my + (q + u) * NT);
    double g[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) g[u] = __ldg(z + c[u]);
#pragma unroll
    for (int u = 0; u < 16; ++u) acc += g[u];
  }
  out[t] = acc;
}

// Local shared memory only (cluster size 1): random gathers from the CTA's own 192 KB.
__global__ void __launch_bounds__(512, 1) smem_gather(const double* __restrict__ zblk, const uint32_t* __restrict__ idx,
                                                      int64_t per_thread, double* out) {
  extern __shared__ double zs[];
  for (int i = threadIdx.x; i < kPerCta; i += blockDim.x) zs[i] = zblk[i];
  __syncthreads();
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t NT = int64_t(gridDim.x) * blockDim.x;
  const uint32_t* my = idx + t;
  double acc = 0.0;
  for (int64_t q = 0; q < per_thread; q += 16) {
    uint32_t c[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) c[u] = __ldg(my + (q + u) * NT) % kPerCta;
    double g[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) g[u] = zs[c[u]];
#pragma unroll
    for (int u = 0; u < 16; ++u) acc += g[u];
  }
  out[t] = acc;
}

int main() {
  const int threads = 512, blocks = 144;  // multiple of 8 and 16
  const int64_t per_thread = 512;
  const int64_t total = int64_t(threads) * blocks * per_thread;
  const int64_t zn = int64_t(16) * kPerCta;
  double *z, *out;
  uint32_t* idx;
  cudaMalloc(&z, zn * 8);
  cudaMalloc(&out, int64_t(threads) * blocks * 8);
  cudaMalloc(&idx, total * 4);
  uint32_t* h = (uint32_t*)malloc(total * 4);
  double* hz = (double*)malloc(zn * 8);
  for (int64_t i = 0; i < zn; ++i) hz[i] = double(i % 977);
  cudaMemcpy(z, hz, zn * 8, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto fill = [&](int64_t range) {
    uint64_t s = 88172645463325252ull;
    for (int64_t i = 0; i < total; ++i) {
      s ^= s << 13; s ^= s >> 7; s ^= s << 17;
      h[i] = uint32_t(s % uint64_t(range));
    }
    cudaMemcpy(idx, h, total * 4, cudaMemcpyHostToDevice);
  };
  auto report = [&](const char* name, float ms) {
    printf("%-34s %8.1f us  %7.1f Ggather/s  (%.2f per SM clock @1.9 GHz, %d CTAs)\n", name, ms * 1e3,
           total / ms / 1e6, total / (ms * 1e-3) / (blocks * 1.9e9), blocks);
  };
  float ms;
  const int smem = kPerCta * 8;
  // L2 reference: 8 MB vector (the c4 z)
  {
    const int64_t big = 1 << 20;
    double* zb;
    cudaMalloc(&zb, big * 8);
    cudaMemset(zb, 0, big * 8);
    fill(big);
    l2_gather<<<blocks, threads>>>(zb, idx, per_thread, out);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) l2_gather<<<blocks, threads>>>(zb, idx, per_thread, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    report("L2 gather (8 MB vector)", ms / 5);
  }
  {
    fill(kPerCta);
    cudaFuncSetAttribute(smem_gather, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    smem_gather<<<blocks, threads, smem>>>(z, idx, per_thread, out);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) smem_gather<<<blocks, threads, smem>>>(z, idx, per_thread, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    report("local smem gather (192 KB)", ms / 5);
  }
  {
    fill(8 * kPerCta);
    cudaFuncSetAttribute(dsmem_gather<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    dsmem_gather<8><<<blocks, threads, smem>>>(z, idx, per_thread, out);
    cudaError_t err = cudaDeviceSynchronize();
    if (err != cudaSuccess) { printf("cluster 8: %s\n", cudaGetErrorString(err)); return 1; }
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) dsmem_gather<8><<<blocks, threads, smem>>>(z, idx, per_thread, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    report("DSMEM gather, cluster 8 (1.5 MB)", ms / 5);
  }
  {
    fill(16 * kPerCta);
    cudaFuncSetAttribute(dsmem_gather<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(dsmem_gather<16>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    dsmem_gather<16><<<blocks, threads, smem>>>(z, idx, per_thread, out);
    cudaError_t err = cudaDeviceSynchronize();
    if (err != cudaSuccess) { printf("cluster 16: %s\n", cudaGetErrorString(err)); return 0; }
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) dsmem_gather<16><<<blocks, threads, smem>>>(z, idx, per_thread, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    report("DSMEM gather, cluster 16 (3 MB)", ms / 5);
  }
  return 0;
}
