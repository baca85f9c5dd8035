// Per-kernel profiling hook (see h2_prof.h).  Not used unless h2_profile_enable(1) is called.
#include "h2_prof.h"

#include <cuda_runtime.h>

#include <cstring>
#include <string>
#include <vector>

#include "h2_internal.h"

namespace h2 {

const char* const kKernelNames[K_COUNT] = {
    "k_upd_ext_leaf", "k_upd_ext_level", "k_upd_weights_path", "k_upd_weights_level", "k_upd_svd_leaf",
    "k_upd_svd_level", "k_upd_couple", "k_upd_install", "k_upd_rcache_path", "k_matvec", "k_solve_sweep",
    "ar_expand", "ar_gemm", "ar_hmul", "ar_tile", "ar_tsqr", "ar_temp_core", "ar_misc"};

namespace {
struct State {
  bool on = false;
  double* d = nullptr;
  std::vector<cudaEvent_t> ev[K_COUNT];
  size_t used[K_COUNT] = {};
};
State g;
}  // namespace

double* prof_dev() { return g.on ? g.d : nullptr; }

static long long g_launches = 0;
double g_host_wait_s = 0.0;
void count_launch(int n) { g_launches += n; }

static cudaEvent_t next_event(int kid) {
  if (g.used[kid] == g.ev[kid].size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    g.ev[kid].push_back(e);
  }
  return g.ev[kid][g.used[kid]++];
}

void prof_begin(int kid, cudaStream_t st) {
  if (g.on) cudaEventRecord(next_event(kid), st);
}

void prof_end(int kid, cudaStream_t st) {
  if (g.on) cudaEventRecord(next_event(kid), st);
}

}  // namespace h2

using namespace h2;

extern "C" h2_status h2_profile_enable(int32_t on) {
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    set_error(std::string("h2_profile_enable: ") + cudaGetErrorString(e));
    return H2_ERR_CUDA;
  }
  if (!g.d) {
    e = cudaMalloc(&g.d, sizeof(double) * (4 * K_COUNT + 32 + 2 * 64));
    if (e != cudaSuccess) {
      set_error("h2_profile_enable: cudaMalloc failed");
      return H2_ERR_NOMEM;
    }
  }
  cudaMemset(g.d, 0, sizeof(double) * (4 * K_COUNT + 32 + 2 * 64));
  for (int k = 0; k < K_COUNT; ++k) g.used[k] = 0;
  g.on = on != 0;
  return H2_OK;
}

extern "C" h2_status h2_profile_read(char* names, int64_t* launches, double* ms_total, double* flops, double* bytes,
                                     int32_t* count) {
  if (count) *count = K_COUNT;
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    set_error(std::string("h2_profile_read: ") + cudaGetErrorString(e));
    return H2_ERR_CUDA;
  }
  double acc[4 * K_COUNT] = {};
  if (g.d) cudaMemcpy(acc, g.d, sizeof(acc), cudaMemcpyDeviceToHost);
  for (int k = 0; k < K_COUNT; ++k) {
    if (names) {
      std::strncpy(names + 32 * k, kKernelNames[k], 31);
      names[32 * k + 31] = 0;
    }
    const size_t pairs = g.used[k] / 2;
    double tot = 0;
    for (size_t i = 0; i < pairs; ++i) {
      float ms = 0;
      cudaEventElapsedTime(&ms, g.ev[k][2 * i], g.ev[k][2 * i + 1]);
      tot += ms;
    }
    // + ops run inside the device executor (timed on the device: op start to its barrier)
    tot += acc[2 * K_COUNT + 2 * k] / 1e6;
    if (launches) launches[k] = (int64_t)pairs + (int64_t)acc[2 * K_COUNT + 2 * k + 1];
    if (ms_total) ms_total[k] = tot;
    if (flops) flops[k] = acc[2 * k];
    if (bytes) bytes[k] = acc[2 * k + 1];
  }
  return H2_OK;
}

extern "C" h2_status h2_profile_debug(double out[16]) {
  if (!out) {
    set_error("h2_profile_debug: NULL argument");
    return H2_ERR_ARG;
  }
  for (int i = 0; i < 16; ++i) out[i] = 0.0;
  if (!g.d) return H2_OK;
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaMemcpy(out, g.d + 4 * K_COUNT, 16 * sizeof(double), cudaMemcpyDeviceToHost);
  out[15] = g_host_wait_s;  // host seconds spent waiting for a free op buffer (executor back-pressure)
  if (e != cudaSuccess) {
    set_error(std::string("h2_profile_debug: ") + cudaGetErrorString(e));
    return H2_ERR_CUDA;
  }
  return H2_OK;
}

extern "C" h2_status h2_profile_ops(double* ns, double* count, int32_t cap, int32_t* nops) {
  if (!ns || !count || cap < 0) {
    set_error("h2_profile_ops: NULL argument");
    return H2_ERR_ARG;
  }
  if (nops) *nops = 64;
  double acc[2 * 64] = {};
  if (g.d) {
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaMemcpy(acc, g.d + 4 * K_COUNT + 32, sizeof(acc), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) {
      set_error(std::string("h2_profile_ops: ") + cudaGetErrorString(e));
      return H2_ERR_CUDA;
    }
  }
  for (int i = 0; i < cap && i < 64; ++i) {
    ns[i] = acc[2 * i];
    count[i] = acc[2 * i + 1];
  }
  return H2_OK;
}

extern "C" h2_status h2_launch_count(int64_t* out) {
  if (!out) {
    set_error("h2_launch_count: NULL argument");
    return H2_ERR_ARG;
  }
  *out = (int64_t)g_launches;
  return H2_OK;
}
