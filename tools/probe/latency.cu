// Latency probe (dev tool): single-thread clock64() timings of the operations
// on the fold kernel's serial tail.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void probe(double* buf, unsigned* ctr, long long* out, int stride) {
  long long t0, t1;
  double acc = 0.0;
  // warm L2 line
  acc += buf[0];
  t0 = clock64();
  acc += *(volatile double*)&buf[0];
  t1 = clock64();
  out[0] = t1 - t0;  // L2-hit (likely) load, volatile
  t0 = clock64();
  acc += __ldcg(&buf[stride * 7]);  // cold line
  asm volatile("" ::: "memory");
  t1 = clock64();
  out[1] = t1 - t0 + (acc == 12345.0);
  t0 = clock64();
  __threadfence();
  t1 = clock64();
  out[2] = t1 - t0;
  buf[1] = acc;
  t0 = clock64();
  __threadfence();
  t1 = clock64();
  out[3] = t1 - t0;  // fence after a store
  t0 = clock64();
  unsigned v = atomicAdd(ctr, 1u);
  t1 = clock64();
  out[4] = t1 - t0 + (v == 777u);
  buf[2] = acc;
  t0 = clock64();
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
  t1 = clock64();
  out[5] = t1 - t0;  // acq_rel fence after a store
  t0 = clock64();
  unsigned w;
  asm volatile("atom.add.release.gpu.u32 %0, [%1], 1;" : "=r"(w) : "l"(ctr) : "memory");
  t1 = clock64();
  out[6] = t1 - t0 + (w == 777u);
  // 10 dependent L2 loads (pointer chase through buf as indices)
  t0 = clock64();
  long long idx = 0;
  for (int i = 0; i < 10; ++i) idx = (long long)__ldcg(&buf[16 + idx]);
  t1 = clock64();
  out[7] = (t1 - t0) / 10 + (idx == 777);
}

int main() {
  double* buf;
  unsigned* ctr;
  long long* out;
  cudaMalloc(&buf, 1 << 26);
  cudaMemset(buf, 0, 1 << 26);
  cudaMalloc(&ctr, 4);
  cudaMemset(ctr, 0, 4);
  cudaMallocManaged(&out, 8 * 8);
  for (int rep = 0; rep < 3; ++rep) {
    probe<<<1, 1>>>(buf, ctr, out, 1 << 20);
    cudaDeviceSynchronize();
    printf("cycles: volatile_ld %lld cold_ldcg %lld fence %lld fence_after_st %lld atomicAdd %lld "
           "fence_acq_rel %lld atom_release %lld dep_L2_ld %lld\n",
           out[0], out[1], out[2], out[3], out[4], out[5], out[6], out[7]);
  }
  // launch latency of back-to-back empty-ish kernels
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int i = 0; i < 100; ++i) probe<<<1, 1>>>(buf, ctr, out, 1 << 20);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("probe kernel back-to-back: %.2f us each\n", ms * 10.0f);
  return 0;
}
