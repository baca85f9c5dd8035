// FP64 peak microbenchmarks for the roofline denominator:
//  - DFMA pipe: independent FMA chains, 1024 threads/SM-worth of blocks
//  - DMMA: mma.sync.aligned.m8n8k4.row.col.f64 (the FP64 tensor path available on sm_100a)
#include <cuda_runtime.h>
#include <stdint.h>

__global__ void k_dfma(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void k_dmma(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[8][2];
  for (int q = 0; q < 8; ++q) c[q][0] = c[q][1] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int q = 0; q < 8; ++q)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[q][0]), "+d"(c[q][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int q = 0; q < 8; ++q) s += c[q][0] + c[q][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

extern "C" int fp64_peak(double* dfma_tflops, double* dmma_tflops) {
  int dev, sms;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out;
  const int blocks = sms * 8, threads = 256;
  cudaMalloc(&out, sizeof(double) * blocks * threads);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  const int it1 = 4000;
  k_dfma<<<blocks, threads>>>(out, 10, 0.999999, 1e-7);
  cudaEventRecord(e0);
  k_dfma<<<blocks, threads>>>(out, it1, 0.999999, 1e-7);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  *dfma_tflops = 2.0 * 8 * 16 * (double)it1 * blocks * threads / (ms * 1e-3) / 1e12;
  const int it2 = 4000;
  k_dmma<<<blocks, threads>>>(out, 10);
  cudaEventRecord(e0);
  k_dmma<<<blocks, threads>>>(out, it2);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  // one m8n8k4 per warp = 2*8*8*4 = 512 flops
  *dmma_tflops = 512.0 * 8 * (double)it2 * (blocks * threads / 32) / (ms * 1e-3) / 1e12;
  cudaFree(out);
  return (int)cudaGetLastError();
}
