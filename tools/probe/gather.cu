// Random-gather throughput probe: 16.7M FP64 gathers from an L2-resident 8 MB
// vector (the K3 / c4 pattern), vs a coalesced stream of the same count.
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>
__global__ void gather_k(const int* __restrict__ idx, const double* __restrict__ z, double* out, int64_t m, int per) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  double acc = 0;
  for (int64_t r = t; r < m; r += stride) {
    double g[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) g[q] = z[__ldg(idx + r * 16 + q)];
#pragma unroll
    for (int q = 0; q < 16; ++q) acc += g[q];
  }
  out[t] = acc;
}
__global__ void gather_pre(const int* __restrict__ idx, const double* __restrict__ z, double* out, int64_t total) {
  // idx already in registers: gathers only (idx read coalesced)
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  double acc = 0;
  for (int64_t e = t; e < total; e += stride * 4) {
    int i0 = __ldg(idx + e), i1 = e + stride < total ? __ldg(idx + e + stride) : 0;
    int i2 = e + 2 * stride < total ? __ldg(idx + e + 2 * stride) : 0, i3 = e + 3 * stride < total ? __ldg(idx + e + 3 * stride) : 0;
    acc += z[i0] + z[i1] + z[i2] + z[i3];
  }
  out[t] = acc;
}
__global__ void stream_k(const double* __restrict__ a, double* out, int64_t total) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  double acc = 0;
  for (int64_t e = t; e < total; e += stride) acc += a[e];
  out[t] = acc;
}
int main() {
  const int64_t n = 1 << 20, nnz = n * 16;
  int* idx; double *z, *out, *big;
  cudaMalloc(&idx, nnz * 4); cudaMalloc(&z, n * 8); cudaMalloc(&out, 1 << 26); cudaMalloc(&big, nnz * 8);
  int* h = (int*)malloc(nnz * 4);
  uint64_t s = 88172645463325252ull;
  for (int64_t i = 0; i < nnz; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = (int)(s % n); }
  cudaMemcpy(idx, h, nnz * 4, cudaMemcpyHostToDevice);
  cudaMemset(z, 0, n * 8); cudaMemset(big, 0, nnz * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int bps : {2, 4, 8, 16}) for (int th : {256, 512}) {
    int blocks = 148 * bps; float ms;
    gather_k<<<blocks, th>>>(idx, z, out, n, 16);
    cudaEventRecord(e0); for (int r = 0; r < 5; ++r) gather_k<<<blocks, th>>>(idx, z, out, n, 16); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    printf("row-gather  blocks/SM %2d threads %d: %.1f us  (%.2f Ggather/s, idx stream %.2f TB/s)\n", bps, th, ms * 1e3, nnz / ms / 1e6, nnz * 4 / ms / 1e9);
  }
  for (int bps : {4, 8, 16}) {
    int blocks = 148 * bps; float ms;
    gather_pre<<<blocks, 256>>>(idx, z, out, nnz);
    cudaEventRecord(e0); for (int r = 0; r < 5; ++r) gather_pre<<<blocks, 256>>>(idx, z, out, nnz); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    printf("flat-gather blocks/SM %2d: %.1f us (%.2f Ggather/s)\n", bps, ms * 1e3, nnz / ms / 1e6);
  }
  for (int bps : {4, 8}) {
    int blocks = 148 * bps; float ms;
    cudaEventRecord(e0); for (int r = 0; r < 5; ++r) stream_k<<<blocks, 256>>>(big, out, nnz); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    printf("stream 134MB blocks/SM %d: %.1f us (%.2f TB/s)\n", bps, ms * 1e3, nnz * 8 / ms / 1e9);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
