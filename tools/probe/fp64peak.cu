// FP64 throughput probe: DFMA vs DMMA (mma.sync m8n8k4 f64) on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__global__ void dmma_kernel(double* out, int iters, double a, double b) {
  double c[8][2];
#pragma unroll
  for (int j = 0; j < 8; ++j) c[j][0] = c[j][1] = threadIdx.x + j;
  double aa = a + threadIdx.x * 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int j = 0; j < 8; ++j) dmma(c[j][0], c[j][1], aa, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__device__ __forceinline__ void dmma16(double (&d)[4], const double (&a)[8], const double (&b)[4]) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                 "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}
__global__ void dmma16_kernel(double* out, int iters, double a, double b) {
  double c[4][4];
  double av[8], bv[4];
#pragma unroll
  for (int j = 0; j < 8; ++j) av[j] = a + threadIdx.x * 1e-9 + j;
#pragma unroll
  for (int j = 0; j < 4; ++j) bv[j] = b + j;
#pragma unroll
  for (int j = 0; j < 4; ++j) for (int q = 0; q < 4; ++q) c[j][q] = threadIdx.x + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) dmma16(c[j], av, bv);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  cudaDeviceProp prop; cudaGetDeviceProperties(&prop, 0);
  printf("device %s SMs %d clock %d kHz\n", prop.name, prop.multiProcessorCount, prop.clockRate);
  double* out; cudaMalloc(&out, 1 << 26);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = prop.multiProcessorCount;
  for (int threads : {256, 512, 1024}) for (int bps : {1, 2, 4}) {
    int blocks = sms * bps; int iters = 4096;
    dfma_kernel<<<blocks, threads>>>(out, 16, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 64 * iters * (double)blocks * threads;
    printf("DFMA  threads %4d blocks/SM %d : %.2f TFLOP/s\n", threads, bps, flops / ms / 1e9);
  }
  for (int threads : {128, 256, 512}) for (int bps : {1, 2, 4}) {
    int blocks = sms * bps; int iters = 1024;
    dmma_kernel<<<blocks, threads>>>(out, 16, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256 * 64 * iters * (double)blocks * (threads / 32);
    printf("DMMA m8n8k4 threads %4d blocks/SM %d : %.2f TFLOP/s\n", threads, bps, flops / ms / 1e9);
  }
  for (int threads : {128, 256, 512}) for (int bps : {1, 2, 4}) {
    int blocks = sms * bps; int iters = 4096;
    dmma16_kernel<<<blocks, threads>>>(out, 16, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    dmma16_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16 * 8 * 16 * 4 * (double)iters * blocks * (threads / 32);
    printf("DMMA m16n8k16 threads %4d blocks/SM %d : %.2f TFLOP/s\n", threads, bps, flops / ms / 1e9);
  }
  cudaError_t err = cudaGetLastError();
  printf("err: %s\n", cudaGetErrorString(err));
  return 0;
}
