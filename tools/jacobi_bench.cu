// Micro-benchmark of the small-SVD building blocks of U4 (tools only, not part of the library):
// clock64 cycles of cta_qr_R, cta_jacobi and warp_jacobi_R on a random m x K matrix, one CTA.
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_1402_5056_b200/csrc tools/jacobi_bench.cu
#include <cstdio>
#include <cstdlib>

#include "devla.cuh"

using namespace h2;
constexpr int LD = 97;

__global__ void kb(const double* Ain, int m, int K, long long* cyc, double* sig_out, int mode) {
  extern __shared__ double sm[];
  double* A = sm;
  double* J = A + LD * 96;
  double* sig = J + LD * 96;
  int* order = (int*)(sig + 96);
  int* scr = order + 96;
  for (int e = threadIdx.x; e < m * K; e += blockDim.x) A[(e % m) + (e / m) * LD] = Ain[e];
  __syncthreads();
  long long c0 = clock64();
  if (mode == 0 || mode == 3) {
    la::cta_qr_R(A, LD, m, K, sig, (double*)order);
  }
  if (mode == 3) {  // W = R^T (K x K) in J
    const int pr = m < K ? m : K;
    for (int e = threadIdx.x; e < K * K; e += blockDim.x) {
      const int i = e % K, j = e / K;
      J[i + j * LD] = (j < pr && j <= i) ? A[j + i * LD] : 0.0;
    }
    __syncthreads();
  }
  long long c1 = clock64();
  int sw = 0;
  const int pr = m < K ? m : K;
  if (mode == 0) {
    if (K <= 8) sw = la::warp_jacobi<8, true>(A, LD, pr, K, J, LD, sig, order, scr);
    else sw = la::warp_jacobi<16, true>(A, LD, pr, K, J, LD, sig, order, scr);
  } else if (mode == 3) {
    if (K <= 8) sw = la::warp_jacobi<8, false>(J, LD, K, K, A, LD, sig, order, scr);
    else sw = la::warp_jacobi<16, false>(J, LD, K, K, A, LD, sig, order, scr);
  } else if (mode == 2) {
    if (m <= 16) sw = la::warp_jacobi<16, false>(A, LD, m, K, J, LD, sig, order, scr);
    else sw = la::warp_jacobi<32, false>(A, LD, m, K, J, LD, sig, order, scr);
  } else {
    sw = la::cta_jacobi(A, LD, m, K, sig, order, scr);
  }
  long long c2 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = c1 - c0;
    cyc[1] = c2 - c1;
    cyc[2] = sw;
  }
  for (int j = threadIdx.x; j < K; j += blockDim.x) sig_out[j] = sig[order[j]];
}

int main(int argc, char** argv) {
  const int m = argc > 1 ? atoi(argv[1]) : 20, K = argc > 2 ? atoi(argv[2]) : 6;
  double* h = (double*)malloc(sizeof(double) * m * K);
  srand(1);
  for (int i = 0; i < m * K; ++i) h[i] = rand() / (double)RAND_MAX - 0.5;
  double *d, *s;
  long long* c;
  cudaMalloc(&d, sizeof(double) * m * K);
  cudaMalloc(&s, sizeof(double) * 96);
  cudaMalloc(&c, sizeof(long long) * 4);
  cudaMemcpy(d, h, sizeof(double) * m * K, cudaMemcpyHostToDevice);
  const int smem = (2 * LD * 96 + 96) * 8 + 200 * 4;
  cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int mode = 0; mode < 4; ++mode) {
    for (int rep = 0; rep < 3; ++rep) kb<<<1, 256, smem>>>(d, m, K, c, s, mode);
    long long hc[4];
    double hs[96];
    cudaMemcpy(hc, c, sizeof(hc), cudaMemcpyDeviceToHost);
    cudaMemcpy(hs, s, sizeof(double) * K, cudaMemcpyDeviceToHost);
    printf("%s m=%d K=%d qr=%lld jacobi=%lld sweeps=%lld sig0=%.15g sigK=%.15g err=%s\n",
           mode == 3 ? "qr+jac(R^T)" : mode == 2 ? "warp_direct" : mode ? "cta_jacobi " : "qr+warp_jac", m, K, hc[0], hc[1], hc[2], hs[0], hs[K - 1],
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
