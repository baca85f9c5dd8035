// FP64 / shuffle / barrier dependent-latency micro-benchmark (tools only): cycles per operation.
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_1402_5056_b200/csrc tools/lat_bench.cu
#include <cstdio>
#include "devla.cuh"
using namespace h2;
#define R8(s) s s s s s s s s
__global__ void k(double* out, long long* cyc, double x0) {
  double x = x0 + threadIdx.x; float f = x0;
  long long c[12]; int n = 0;
  c[n++] = clock64();
  for (int i = 0; i < 100; ++i) { R8(x = fma(x, 0.999999, 1e-7);) }
  c[n++] = clock64();
  for (int i = 0; i < 100; ++i) { R8(f = fmaf(f, 0.9999f, 1e-3f);) }
  c[n++] = clock64();
  for (int i = 0; i < 100; ++i) { R8(x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31);) }
  c[n++] = clock64();
  for (int i = 0; i < 100; ++i) { R8(x = 1.0 / x;) }
  c[n++] = clock64();
  for (int i = 0; i < 100; ++i) { R8(x = la::fast_rcp(x);) }
  c[n++] = clock64();
  for (int i = 0; i < 100; ++i) { R8(x = rsqrt(x);) }
  c[n++] = clock64();
  for (int i = 0; i < 100; ++i) { R8(x = sqrt(x);) }
  c[n++] = clock64();
  for (int i = 0; i < 100; ++i) { R8(x = la::fast_rsqrt(x);) }
  c[n++] = clock64();
  volatile __shared__ double s[64];
  s[threadIdx.x] = x;
  for (int i = 0; i < 100; ++i) { R8(x = s[(threadIdx.x + (int)x) & 31];) }
  c[n++] = clock64();
  for (int i = 0; i < 100; ++i) { R8(__syncthreads();) }
  c[n++] = clock64();
  out[threadIdx.x] = x + f;
  if (threadIdx.x == 0) for (int i = 0; i + 1 < n; ++i) cyc[i] = c[i + 1] - c[i];
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8 * 256); cudaMalloc(&c, 8 * 16);
  const char* nm[] = {"dfma", "ffma", "shfl.f64", "ddiv", "fast_rcp", "rsqrt", "sqrt", "fast_rsqrt", "lds.f64", "bar.sync"};
  for (int nt : {32, 256}) {
    for (int r = 0; r < 2; ++r) k<<<1, nt>>>(o, c, 1.5);
    long long h[16]; cudaMemcpy(h, c, 128, cudaMemcpyDeviceToHost);
    printf("threads %d:", nt);
    for (int i = 0; i < 10; ++i) printf(" %s %.1f", nm[i], h[i] / 800.0);
    printf("\n");
  }
}
