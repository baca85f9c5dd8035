// Preconditioned CG with the H^2 factor as preconditioner (reading R12):
// x0 = 0, z = (L L^T)^{-1} r by h2_solve, A applied by h2_matvec, stop at ||r||/||b|| < tol.
// The vector kernels (dot products with a deterministic two-stage reduction, fused axpys) are the
// library's own; the host reads two scalars per iteration.
#include <cuda_runtime.h>

#include <cmath>
#include <string>

#include "h2_internal.h"
#include "h2_prof.h"

namespace h2 {
namespace {

constexpr int PB = 256;
constexpr int PG = 296;  // 2 x 148 SMs

__global__ void k_dot(const double* __restrict__ a, const double* __restrict__ b, int64_t n, double* part) {
  __shared__ double red[PB / 32];
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * PB + threadIdx.x; i < n; i += (int64_t)gridDim.x * PB) s += a[i] * b[i];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < PB / 32; ++w) t += red[w];
    part[blockIdx.x] = t;
  }
}

__global__ void k_sum(const double* part, int np, double* out) {
  __shared__ double red[PB / 32];
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += PB) s += part[i];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < PB / 32; ++w) t += red[w];
    *out = t;
  }
}

// x += a p ; r -= a q     (a = rz / pAp read from device scalars)
__global__ void k_update_xr(double* x, double* r, const double* p, const double* q, const double* rz,
                            const double* pq, int64_t n) {
  const double a = *rz / *pq;
  for (int64_t i = (int64_t)blockIdx.x * PB + threadIdx.x; i < n; i += (int64_t)gridDim.x * PB) {
    x[i] += a * p[i];
    r[i] -= a * q[i];
  }
}

// p = z + (rz_new / rz_old) p
__global__ void k_update_p(double* p, const double* z, const double* rz_new, const double* rz_old, int64_t n) {
  const double b = *rz_new / *rz_old;
  for (int64_t i = (int64_t)blockIdx.x * PB + threadIdx.x; i < n; i += (int64_t)gridDim.x * PB) p[i] = z[i] + b * p[i];
}

__global__ void k_copy(double* d, const double* s, int64_t n, double scale) {
  for (int64_t i = (int64_t)blockIdx.x * PB + threadIdx.x; i < n; i += (int64_t)gridDim.x * PB) d[i] = scale * s[i];
}

}  // namespace
}  // namespace h2

using namespace h2;

extern "C" h2_status h2_pcg(h2_mat A, h2_mat F, const double* b, double* x, double tol, int32_t maxit,
                            int32_t* iters, double* relres, h2_stream stream) {
  if (h2::batch_open()) {
    h2::set_error("h2_pcg: not allowed inside h2_batch_begin/h2_batch_end");
    return H2_ERR_ARG;
  }
  if (!A || !F || !b || !x || !iters) {
    set_error("h2_pcg: NULL argument");
    return H2_ERR_ARG;
  }
  if (A->bt->rt->n != F->bt->rt->n) {
    set_error("h2_pcg: A and F have different sizes");
    return H2_ERR_SHAPE;
  }
  if (!F->factored) {
    set_error("h2_pcg: the preconditioner is not factored");
    return H2_ERR_ARG;
  }
  if (!(tol > 0) || maxit < 1) {
    set_error("h2_pcg: need tol > 0 and maxit >= 1");
    return H2_ERR_ARG;
  }
  const int64_t n = A->bt->rt->n;
  cudaStream_t st = (cudaStream_t)stream;
  double* w = nullptr;  // r, p, q, z, partials, scalars
  cudaError_t e = cudaMallocAsync(&w, sizeof(double) * (4 * n + PG + 8), st);
  if (e != cudaSuccess) {
    set_error("h2_pcg: out of device memory");
    return H2_ERR_NOMEM;
  }
  double *r = w, *p = w + n, *q = w + 2 * n, *z = w + 3 * n, *part = w + 4 * n, *sc = part + PG;
  double* rz = sc;       // r.z
  double* rz_new = sc + 1;
  double* pq = sc + 2;   // p.Ap
  double* rr = sc + 3;   // r.r
  double* bb = sc + 4;   // b.b
  const int g = PG;
  h2_status status = H2_OK;
  auto dot = [&](const double* u, const double* v, double* out) {
    count_launch(2);
    k_dot<<<g, PB, 0, st>>>(u, v, n, part);
    k_sum<<<1, PB, 0, st>>>(part, g, out);
  };
  auto host = [&](const double* d) {
    double h = 0.0;
    cudaMemcpyAsync(&h, d, sizeof(double), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    return h;
  };
  count_launch(1);
  k_copy<<<g, PB, 0, st>>>(x, b, n, 0.0);  // x0 = 0
  count_launch(1);
  k_copy<<<g, PB, 0, st>>>(r, b, n, 1.0);
  dot(b, b, bb);
  const double nb = std::sqrt(host(bb));
  int m = 0;
  double rel = 0.0;
  if (nb == 0.0) {
    *iters = 0;
    if (relres) *relres = 0.0;
    cudaFreeAsync(w, st);
    return H2_OK;
  }
  count_launch(1);
  k_copy<<<g, PB, 0, st>>>(z, r, n, 1.0);
  status = h2_solve(F, z, 1, n, stream);
  if (status != H2_OK) {
    cudaFreeAsync(w, st);
    return status;
  }
  count_launch(1);
  k_copy<<<g, PB, 0, st>>>(p, z, n, 1.0);
  dot(r, z, rz);
  while (m < maxit) {
    status = h2_matvec(A, 0, 1.0, p, 0.0, q, stream);
    if (status != H2_OK) break;
    ++m;
    dot(p, q, pq);
    count_launch(1);
    k_update_xr<<<g, PB, 0, st>>>(x, r, p, q, rz, pq, n);
    dot(r, r, rr);
    rel = std::sqrt(host(rr)) / nb;
    if (!std::isfinite(rel)) {  // NaN / Inf in the factor, the operator or b: never "converges"
      set_error("h2_pcg: non-finite residual at iteration " + std::to_string(m));
      status = H2_ERR_NONFINITE;
      break;
    }
    if (rel < tol) break;
    count_launch(1);
    k_copy<<<g, PB, 0, st>>>(z, r, n, 1.0);
    status = h2_solve(F, z, 1, n, stream);
    if (status != H2_OK) break;
    dot(r, z, rz_new);
    count_launch(1);
    k_update_p<<<g, PB, 0, st>>>(p, z, rz_new, rz, n);
    cudaMemcpyAsync(rz, rz_new, sizeof(double), cudaMemcpyDeviceToDevice, st);
  }
  cudaFreeAsync(w, st);
  *iters = m;
  if (relres) *relres = rel;
  if (status == H2_OK && (e = cudaGetLastError()) != cudaSuccess) {
    set_error(std::string("h2_pcg: ") + cudaGetErrorString(e));
    return H2_ERR_CUDA;
  }
  if (status == H2_OK && !(rel < tol)) {
    set_error("h2_pcg: no convergence in " + std::to_string(m) + " iterations (relres " + std::to_string(rel) + ")");
    return H2_ERR_NOCONV;
  }
  return status;
}
