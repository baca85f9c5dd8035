// Micro-benchmark of the leaf-tile triangular solve item (tools only): cycles of one it_trsm call
// (32 x 32 lower tile, 32 right-hand sides, rowwise RLT and columnwise LLN) in a single CTA.
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_1402_5056_b200/csrc tools/trsm_bench.cu
#include <cstdio>
#include <vector>

#include "h2_arith.cuh"
#include "items_arith.cuh"

using namespace h2;

__global__ void kb(MatDev M, double* B, int mode, long long* cyc) {
  extern __shared__ double sm[];
  long long c0 = clock64();
  ar::it_trsm(M, 0, 32, mode, B, 32, 32, Dim{nullptr, 32}, 0, 1, sm);
  __syncthreads();
  long long c1 = clock64();
  if (threadIdx.x == 0) cyc[0] = c1 - c0;
}

int main() {
  std::vector<double> T(32 * 32, 0.0), B(32 * 32);
  for (int j = 0; j < 32; ++j)
    for (int i = j; i < 32; ++i) T[i + 32 * j] = (i == j) ? 4.0 : 0.01 * ((i * 7 + j * 3) % 11);
  for (auto& b : B) b = 1.0;
  MatDev M{};
  double *dT, *dB;
  long long* dc;
  cudaMalloc(&dT, 8 * 1024);
  cudaMalloc(&dB, 8 * 1024);
  cudaMalloc(&dc, 8);
  cudaMemcpy(dT, T.data(), 8 * 1024, cudaMemcpyHostToDevice);
  M.N = dT;
  M.lmax = 32;
  cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  for (int mode : {RLT, LLN, LLT}) {
    for (int r = 0; r < 3; ++r) {
      cudaMemcpy(dB, B.data(), 8 * 1024, cudaMemcpyHostToDevice);
      kb<<<1, 256, 100000>>>(M, dB, mode, dc);
    }
    long long c;
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    printf("mode %d: %lld cycles (%s)\n", mode, c, cudaGetErrorString(cudaGetLastError()));
  }
}
