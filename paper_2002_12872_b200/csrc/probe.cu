// probe.cu -- the FP64 roofline denominator, measured on the running device:
// a register-resident stream of independent mma.sync.m8n8k4.f64 (SASS
// DMMA.8x8x4) per warp, 4 warps x 2 CTAs per SM (the shape that saturated the
// DMMA pipe in tools/probe/fp64peak.cu).  MEASURED_PEAKS.json carries HBM and
// bf16 only, so bench.py reports the dense step against this number.
#include <cuda_runtime.h>
#include <string.h>

#include "../../include/dpt_b200.h"
#include "dpt_device.cuh"

namespace {
__global__ void dmma_peak_kernel(double* out, int iters) {
  double c[8][2];
#pragma unroll
  for (int j = 0; j < 8; ++j) c[j][0] = c[j][1] = threadIdx.x + j;
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int j = 0; j < 8; ++j) dpt::dmma_8x8x4(c[j][0], c[j][1], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
}  // namespace

extern "C" int dpt_probe_fp64_peak(int device, double* tflops, dpt_error_info* err) {
  if (err) memset(err, 0, sizeof(*err));
  int old = 0;
  cudaGetDevice(&old);
  if (cudaSetDevice(device) != cudaSuccess) {
    cudaGetLastError();
    if (err) err->code = DPT_ERR_NO_DEVICE;
    return DPT_ERR_NO_DEVICE;
  }
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, device);
  const int blocks = prop.multiProcessorCount * 2, threads = 256, iters = 2048;
  double* out = nullptr;
  cudaMalloc(&out, size_t(blocks) * threads * sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dmma_peak_kernel<<<blocks, threads>>>(out, 64);  // warm-up / clock ramp
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    dmma_peak_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const cudaError_t e = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  cudaSetDevice(old);
  if (e != cudaSuccess) {
    if (err) {
      err->code = DPT_ERR_CUDA;
      strncpy(err->message, cudaGetErrorString(e), sizeof(err->message) - 1);
    }
    return DPT_ERR_CUDA;
  }
  const double flops = 2.0 * 256.0 * 64.0 * double(iters) * blocks * (threads / 32);
  *tflops = flops / (double(best) * 1e-3) / 1e12;
  return DPT_OK;
}
