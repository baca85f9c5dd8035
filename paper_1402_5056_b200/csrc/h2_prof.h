// Optional per-kernel profiling (bench/test hook, off by default).
// When enabled, every library launch is bracketed by cudaEventRecord on its own stream, and the
// kernels add their ALGORITHMIC flops / bytes (fixed formulas) to device counters.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace h2 {

enum KernelId {
  K_EXT_LEAF = 0,
  K_EXT_LEVEL,
  K_W_PATH,
  K_W_LEVEL,
  K_SVD_LEAF,
  K_SVD_LEVEL,
  K_COUPLE,
  K_INSTALL,
  K_RCACHE,
  K_MV,
  K_SOLVE,
  K_AR_EXPAND,
  K_AR_GEMM,
  K_AR_HMUL,
  K_AR_TILE,
  K_AR_TSQR,
  K_AR_TEMP,
  K_AR_MISC,
  K_COUNT
};

extern const char* const kKernelNames[K_COUNT];

// device counters: prof[2*kid] = flops, prof[2*kid+1] = bytes; nullptr when profiling is off
double* prof_dev();
void prof_begin(int kid, cudaStream_t st);
void prof_end(int kid, cudaStream_t st);
extern double g_host_wait_s;  // accumulated host wait in exec_flush (h2_profile_debug out[15])
void count_launch(int n);  // library kernel-launch counter (h2_launch_count)

// Householder QR of an m x n matrix: 2 m n^2 - 2/3 n^3 (m >= n), SURVEY §8(d)
__host__ __device__ inline double hh_flops(int m, int n) {
  if (m <= 0 || n <= 0) return 0.0;
  const double a = m >= n ? m : n, b = m >= n ? n : m;
  return 2.0 * a * b * b - 2.0 / 3.0 * b * b * b;
}
// SVD of an m x n matrix (U and Sigma): 4 m n^2 + 8 n^3 (m >= n), SURVEY §8(d)
__host__ __device__ inline double svd_flops(int m, int n) {
  if (m <= 0 || n <= 0) return 0.0;
  const double a = m >= n ? m : n, b = m >= n ? n : m;
  return 4.0 * a * b * b + 8.0 * b * b * b;
}

}  // namespace h2

#define H2_LAUNCH(KID, ST, ...)        \
  do {                                 \
    ::h2::count_launch(1);             \
    ::h2::prof_begin((KID), (ST));     \
    __VA_ARGS__;                       \
    ::h2::prof_end((KID), (ST));       \
  } while (0)
