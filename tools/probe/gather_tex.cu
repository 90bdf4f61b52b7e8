// Random-gather throughput through the TEXTURE path vs LDG: 16.7M FP64 gathers
// from an L2-resident 8 MB vector (the K3 / c4 pattern).  LDG gathers top out at
// ~262 G/s = 0.92 gathers per SM clock (one divergent address per clock through
// the LSU).  Question: do point-sampled 1D texture fetches (tex1Dfetch<int2>
// over linear memory) of the same addresses go faster?
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>
__global__ void gather_ldg(const int* __restrict__ idx, const double* __restrict__ z, double* out, int64_t total) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  double acc = 0;
  for (int64_t e = t; e + 3 * stride < total; e += stride * 4) {
    int i0 = __ldg(idx + e), i1 = __ldg(idx + e + stride), i2 = __ldg(idx + e + 2 * stride), i3 = __ldg(idx + e + 3 * stride);
    acc += z[i0] + z[i1] + z[i2] + z[i3];
  }
  out[t] = acc;
}
__global__ void gather_tex(const int* __restrict__ idx, cudaTextureObject_t tz, double* out, int64_t total) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  double acc = 0;
  for (int64_t e = t; e + 3 * stride < total; e += stride * 4) {
    int i0 = __ldg(idx + e), i1 = __ldg(idx + e + stride), i2 = __ldg(idx + e + 2 * stride), i3 = __ldg(idx + e + 3 * stride);
    int2 a = tex1Dfetch<int2>(tz, i0), b = tex1Dfetch<int2>(tz, i1), c = tex1Dfetch<int2>(tz, i2), d = tex1Dfetch<int2>(tz, i3);
    acc += __hiloint2double(a.y, a.x) + __hiloint2double(b.y, b.x) + __hiloint2double(c.y, c.x) + __hiloint2double(d.y, d.x);
  }
  out[t] = acc;
}
// half of each thread's gathers through LDG, half through TEX (do the two paths add up?)
__global__ void gather_mix(const int* __restrict__ idx, const double* __restrict__ z, cudaTextureObject_t tz, double* out, int64_t total) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  double acc = 0;
  for (int64_t e = t; e + 3 * stride < total; e += stride * 4) {
    int i0 = __ldg(idx + e), i1 = __ldg(idx + e + stride), i2 = __ldg(idx + e + 2 * stride), i3 = __ldg(idx + e + 3 * stride);
    int2 a = tex1Dfetch<int2>(tz, i0), b = tex1Dfetch<int2>(tz, i1);
    acc += __hiloint2double(a.y, a.x) + __hiloint2double(b.y, b.x) + z[i2] + z[i3];
  }
  out[t] = acc;
}
int main() {
  const int64_t n = 1 << 20, nnz = n * 16;
  int* idx; double *z, *out;
  cudaMalloc(&idx, nnz * 4); cudaMalloc(&z, n * 8); cudaMalloc(&out, 1 << 26);
  int* h = (int*)malloc(nnz * 4);
  uint64_t s = 88172645463325252ull;
  for (int64_t i = 0; i < nnz; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = (int)(s % n); }
  cudaMemcpy(idx, h, nnz * 4, cudaMemcpyHostToDevice);
  double* hz = (double*)malloc(n * 8);
  for (int64_t i = 0; i < n; ++i) hz[i] = 1.0 + 1e-6 * double(i);
  cudaMemcpy(z, hz, n * 8, cudaMemcpyHostToDevice);
  cudaResourceDesc rd = {}; rd.resType = cudaResourceTypeLinear; rd.res.linear.devPtr = z;
  rd.res.linear.desc = cudaCreateChannelDesc<int2>(); rd.res.linear.sizeInBytes = n * 8;
  cudaTextureDesc td = {}; td.readMode = cudaReadModeElementType;
  cudaTextureObject_t tz = 0;
  printf("create tex: %s\n", cudaGetErrorString(cudaCreateTextureObject(&tz, &rd, &td, nullptr)));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  double* ho = (double*)malloc(1 << 20);
  for (int bps : {2, 4, 8, 16}) for (int th : {256, 512}) {
    int blocks = 148 * bps; float ms; double s0 = 0, s1 = 0;
    gather_ldg<<<blocks, th>>>(idx, z, out, nnz);
    cudaEventRecord(e0); for (int r = 0; r < 5; ++r) gather_ldg<<<blocks, th>>>(idx, z, out, nnz); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    cudaMemcpy(ho, out, 8 * 1024, cudaMemcpyDeviceToHost); for (int i = 0; i < 1024; ++i) s0 += ho[i];
    printf("ldg  blocks/SM %2d threads %d: %6.1f us  %6.1f Ggather/s\n", bps, th, ms * 1e3, nnz / ms / 1e6);
    gather_tex<<<blocks, th>>>(idx, tz, out, nnz);
    cudaEventRecord(e0); for (int r = 0; r < 5; ++r) gather_tex<<<blocks, th>>>(idx, tz, out, nnz); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    cudaMemcpy(ho, out, 8 * 1024, cudaMemcpyDeviceToHost); for (int i = 0; i < 1024; ++i) s1 += ho[i];
    printf("tex  blocks/SM %2d threads %d: %6.1f us  %6.1f Ggather/s  (sum match %d)\n", bps, th, ms * 1e3, nnz / ms / 1e6, s0 == s1);
    gather_mix<<<blocks, th>>>(idx, z, tz, out, nnz);
    cudaEventRecord(e0); for (int r = 0; r < 5; ++r) gather_mix<<<blocks, th>>>(idx, z, tz, out, nnz); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    printf("mix  blocks/SM %2d threads %d: %6.1f us  %6.1f Ggather/s\n", bps, th, ms * 1e3, nnz / ms / 1e6);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
