// Device items of the product / substitution / factorization primitives (SURVEY §8(a) M1-M3,
// F1-F3, S2), executed by the op executor (h2_exec.cu).  Item i = one CTA's share of the op.
#pragma once
#include <cuda_runtime.h>

#include "devla.cuh"
#include "exec.h"

namespace h2 {
namespace ar {

constexpr int NT = NTHREADS;
constexpr int KC = KCAP_MAX;
constexpr int PR = 192;


// ---- basis expansion ---------------------------------------------------------------------------
__device__ void it_expand(const MatDev& M, const DevSide& D, int t, int l0, double* out, int ld, int item_, int nitems_, double* smx_) {
  double* smx = smx_;
  constexpr int LP = KC + 1;
  double* P[2] = {smx, smx + LP * KC};
  const int q = D.leaves[l0 + item_];
  const int kt = D.rank[t];
  int cur = 0;
  int kq = D.rank[q];
  // P = I (kq x kq)
  for (int e = threadIdx.x; e < kq * kq; e += NT) P[0][(e % kq) + (e / kq) * LP] = (e % kq) == (e / kq) ? 1.0 : 0.0;
  int rows = kq, cols = kq;
  __syncthreads();
  for (int a = q; a != t; a = D.parent[a]) {
    const int kp = D.rank[D.parent[a]];
    const double* E = D.tr + (size_t)a * M.rcap * M.rcap;  // k_a x k_p
    for (int e = threadIdx.x; e < rows * kp; e += NT) {
      const int i = e % rows, j = e / rows;
      double acc = 0.0;
      for (int p = 0; p < cols; ++p) acc += P[cur][i + p * LP] * E[p + j * M.rcap];
      P[cur ^ 1][i + j * LP] = acc;
    }
    cols = kp;
    cur ^= 1;
    __syncthreads();
  }
  (void)kt;
  const int m = D.hi[q] - D.lo[q];
  const int off = D.lo[q] - D.lo[t];
  const double* V = D.leafb + (size_t)D.leafidx[q] * M.lmax * M.rcap;
  for (int e = threadIdx.x; e < m * cols; e += NT) {
    const int i = e % m, j = e / m;
    double acc = 0.0;
    for (int p = 0; p < rows; ++p) acc += V[i + p * M.lmax] * P[cur][p + j * LP];
    out[off + i + (size_t)j * ld] = acc;
  }
}

// ---- GEMMs with device dims -------------------------------------------------------------------
__device__ void it_gemm(double* C, int ldc, const double* A, int lda, bool ta, const double* B, int ldb, bool tb,
                       Dim md, Dim nd, Dim kd, double alpha, double beta, int item_, int nitems_, double* smx_) {
  const int m = md.v(), n = nd.v(), kk = kd.v();
  const long long tot = (long long)m * n;
  for (long long e = (long long)item_ * blockDim.x + threadIdx.x; e < tot; e += (long long)nitems_ * blockDim.x) {
    const int i = (int)(e % m), j = (int)(e / m);
    double acc = 0.0;
    for (int q = 0; q < kk; ++q) {
      const double a = ta ? A[q + (size_t)i * lda] : A[i + (size_t)q * lda];
      const double b = tb ? B[j + (size_t)q * ldb] : B[q + (size_t)j * ldb];
      acc += a * b;
    }
    const size_t o = i + (size_t)j * ldc;
    C[o] = beta == 0.0 ? alpha * acc : alpha * acc + beta * C[o];
  }
}

// long inner dimension: partial sums per chunk, then a deterministic fixed-order reduction
__device__ void it_gemm_inner_part(double* part, const double* A, int lda, bool ta, const double* B, int ldb, bool tb,
                                  Dim md, Dim nd, Dim kd, int chunk, int item_, int nitems_, double* smx_) {
  const int m = md.v(), n = nd.v(), kk = kd.v();
  const int q0 = item_ * chunk, q1 = min(kk, q0 + chunk);
  for (int e = threadIdx.x; e < m * n; e += blockDim.x) {
    const int i = e % m, j = e / m;
    double acc = 0.0;
    for (int q = q0; q < q1; ++q) {
      const double a = ta ? A[q + (size_t)i * lda] : A[i + (size_t)q * lda];
      const double b = tb ? B[j + (size_t)q * ldb] : B[q + (size_t)j * ldb];
      acc += a * b;
    }
    part[(size_t)item_ * KC * KC + e] = acc;
  }
}

__device__ void it_gemm_inner_sum(double* C, int ldc, const double* part, int nparts, Dim md, Dim nd, double alpha,
                                 double beta, int item_, int nitems_, double* smx_) {
  const int m = md.v(), n = nd.v();
  for (int e = threadIdx.x; e < m * n; e += blockDim.x) {
    double acc = 0.0;
    for (int p = 0; p < nparts; ++p) acc += part[(size_t)p * KC * KC + e];
    const int i = e % m, j = e / m;
    const size_t o = i + (size_t)j * ldc;
    C[o] = beta == 0.0 ? alpha * acc : alpha * acc + beta * C[o];
  }
}

constexpr int NPART = 64;

// ---- H^2 block times dense --------------------------------------------------------------------
// forward transform over T_b: leaves
// Every output entry of the five phases is one inline function (the per-phase items below).  (A
// fused one-item variant for small subtrees was measured slower -- 15.8 us per product on one CTA
// against ~3.5 us per op spread over the cluster -- and removed.)
__device__ __forceinline__ double hm_fwd_leaf_entry(const MatDev& M, const DevSide& S, int q, int base_lo,
                                                    const double* D, int ldd, int ident, int j, int c) {
  const int rows = S.hi[q] - S.lo[q];
  const double* W = S.leafb + (size_t)S.leafidx[q] * M.lmax * M.rcap;
  const int off = S.lo[q] - base_lo;
  double acc = 0.0;
  if (ident) {  // D = I: column c of D is e_c, W^T e_c = row (c - off) of W
    const int i = c - off;
    if (i >= 0 && i < rows) acc = W[i + j * M.lmax];
  } else {
    for (int i = 0; i < rows; ++i) acc += W[i + j * M.lmax] * D[off + i + (size_t)c * ldd];
  }
  return acc;
}

__device__ __forceinline__ double hm_fwd_level_entry(const MatDev& M, const DevSide& S, const double* xh, int s, int j,
                                                     int c) {
  double acc = 0.0;
  for (int q = 0; q < 2; ++q) {
    const int sq = q ? S.son1[s] : S.son0[s];
    const int kq = S.rank[sq];
    const double* F = S.tr + (size_t)sq * M.rcap * M.rcap;
    const double* xq = xh + (size_t)sq * M.rcap * KC;
    for (int i = 0; i < kq; ++i) acc += F[i + j * M.rcap] * xq[i + c * M.rcap];
  }
  return acc;
}

__device__ __forceinline__ double hm_couple_entry(const MatDev& M, const DevSide& Dd, const DevSide& Ds, int ap, int b,
                                                  int bsz, int trans, const double* xh, int i, int c) {
  double acc = 0.0;
  for (int q = Dd.bptr[ap]; q < Dd.bptr[ap + 1]; ++q) {
    const int slot = Dd.bidx[q];
    const int bp = trans ? M.adm_t[slot] : M.adm_s[slot];
    if (bp < b || bp >= b + bsz) continue;
    const int kb = Ds.rank[bp];
    const double* Sa = M.S + (size_t)slot * M.rcap * M.rcap;
    const double* x = xh + (size_t)bp * M.rcap * KC + c * M.rcap;
    if (!trans)
      for (int j = 0; j < kb; ++j) acc += Sa[i + j * M.rcap] * x[j];
    else
      for (int j = 0; j < kb; ++j) acc += Sa[j + i * M.rcap] * x[j];
  }
  return acc;
}

__device__ __forceinline__ double hm_bwd_level_entry(const MatDev& M, const DevSide& D, const double* yh, int t, int i,
                                                     int c) {
  const int p = D.parent[t], kp = D.rank[p];
  const double* E = D.tr + (size_t)t * M.rcap * M.rcap;
  const double* yp = yh + (size_t)p * M.rcap * KC;
  double acc = yh[(size_t)t * M.rcap * KC + i + c * M.rcap];
  for (int j = 0; j < kp; ++j) acc += E[i + j * M.rcap] * yp[j + c * M.rcap];
  return acc;
}

__device__ __forceinline__ void hm_leaf_entry(const MatDev& M, const DevSide& Dd, const DevSide& Ds, int ap, int a,
                                              int b, int bsz, int trans, const double* D, int ldd, const double* yh,
                                              double* out, int ldo, double alpha, double beta, int ident, int i,
                                              int c) {
  const int ka = Dd.rank[ap];
  const int offo = Dd.lo[ap] - Dd.lo[a];
  const double* V = Dd.leafb + (size_t)Dd.leafidx[ap] * M.lmax * M.rcap;
  const double* y = yh + (size_t)ap * M.rcap * KC;
  const int32_t* np = trans ? M.ntptr : M.nptr;
  const int32_t* ni = trans ? M.ntidx : M.nidx;
  const int32_t* part = trans ? M.in_t : M.in_s;
  double acc = 0.0;
  for (int j = 0; j < ka; ++j) acc += V[i + j * M.lmax] * y[j + c * M.rcap];
  for (int q = np[ap]; q < np[ap + 1]; ++q) {
    const int slot = ni[q];
    const int bp = part[slot];
    if (bp < b || bp >= b + bsz) continue;
    const int rb = Ds.hi[bp] - Ds.lo[bp];
    const double* Na = M.N + (size_t)slot * M.lmax * M.lmax;
    const int offb = Ds.lo[bp] - Ds.lo[b];
    if (ident) {  // D = I: the tile's column (c - offb) (exact: the other terms are zero products)
      const int jj = c - offb;
      if (jj >= 0 && jj < rb) acc += trans ? Na[jj + i * M.lmax] : Na[i + jj * M.lmax];
      continue;
    }
    const double* x = D + offb + (size_t)c * ldd;
    if (!trans)
      for (int j = 0; j < rb; ++j) acc += Na[i + j * M.lmax] * x[j];
    else
      for (int j = 0; j < rb; ++j) acc += Na[j + i * M.lmax] * x[j];
  }
  double* o = out + offo + i + (size_t)c * ldo;
  *o = beta == 0.0 ? alpha * acc : beta * *o + alpha * acc;
}

__device__ void it_hm_fwd_leaf(const MatDev& M, const DevSide& S, int l0, int base_lo, const double* D, int ldd,
                               Dim md, double* xh, int ident, int item_, int nitems_, double* smx_) {
  const int q = S.leaves[l0 + item_];
  const int m = md.v(), kq = S.rank[q];
  double* x = xh + (size_t)q * M.rcap * KC;
  for (int e = threadIdx.x; e < kq * m; e += NT) {
    const int j = e % kq, c = e / kq;
    x[j + c * M.rcap] = hm_fwd_leaf_entry(M, S, q, base_lo, D, ldd, ident, j, c);
  }
}

__device__ void it_hm_fwd_level(const MatDev& M, const DevSide& S, int b0, Dim md, double* xh, int item_, int nitems_, double* smx_) {
  const int s = S.bfs[b0 + item_];
  if (S.son0[s] < 0) return;
  const int m = md.v(), ks = S.rank[s];
  double* x = xh + (size_t)s * M.rcap * KC;
  for (int e = threadIdx.x; e < ks * m; e += NT) {
    const int j = e % ks, c = e / ks;
    x[j + c * M.rcap] = hm_fwd_level_entry(M, S, xh, s, j, c);
  }
}

// couplings: CTA per cluster a' of T_a (dst side): yhat_{a'} = sum_{(a',b') adm, b' in T_b} S_op xhat_{b'}
__device__ void it_hm_couple(const MatDev& M, const DevSide& Dd, const DevSide& Ds, int a, int b, int trans, Dim md,
                             const double* xh, double* yh, int item_, int nitems_, double* smx_) {
  const int ap = a + item_;
  const int m = md.v(), ka = Dd.rank[ap];
  const int bsz = Ds.tsize[b];
  double* y = yh + (size_t)ap * M.rcap * KC;
  for (int e = threadIdx.x; e < ka * m; e += NT) {
    const int i = e % ka, c = e / ka;
    y[i + c * M.rcap] = hm_couple_entry(M, Dd, Ds, ap, b, bsz, trans, xh, i, c);
  }
}

__device__ void it_hm_bwd_level(const MatDev& M, const DevSide& D, int b0, Dim md, double* yh, int item_, int nitems_, double* smx_) {
  const int t = D.bfs[b0 + item_];
  const int m = md.v(), kt = D.rank[t];
  double* y = yh + (size_t)t * M.rcap * KC;
  for (int e = threadIdx.x; e < kt * m; e += NT) {
    const int i = e % kt, c = e / kt;
    y[i + c * M.rcap] = hm_bwd_level_entry(M, D, yh, t, i, c);
  }
}

__device__ void it_hm_leaf(const MatDev& M, const DevSide& Dd, const DevSide& Ds, int l0, int a, int b, int trans,
                           const double* D, int ldd, Dim md, const double* yh, double* out, int ldo, double alpha,
                           double beta, int ident, int item_, int nitems_, double* smx_) {
  const int ap = Dd.leaves[l0 + item_];
  const int m = md.v();
  const int rows = Dd.hi[ap] - Dd.lo[ap];
  const int bsz = Ds.tsize[b];
  for (int e = threadIdx.x; e < rows * m; e += NT) {
    const int i = e % rows, c = e / rows;
    hm_leaf_entry(M, Dd, Ds, ap, a, b, bsz, trans, D, ldd, yh, out, ldo, alpha, beta, ident, i, c);
  }
}

// ---- dense tiles ------------------------------------------------------------------------------
__device__ void it_potrf(const MatDev& M, int slot, int t, int item_, int nitems_, double* smx_) {
  double* T = smx_;
  double* N = M.N + (size_t)slot * M.lmax * M.lmax;
  const int m = M.row.hi[t] - M.row.lo[t];
  const int ld = 65;
  for (int e = threadIdx.x; e < m * m; e += NT) {
    const int i = e % m, j = e / m;
    T[i + j * ld] = i >= j ? N[i + j * M.lmax] : N[j + i * M.lmax];  // symmetric from the lower triangle
  }
  __syncthreads();
  int& bad = *(int*)(smx_ + 64 * 65);
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int j = 0; j < m; ++j) {
    if (threadIdx.x == 0) {
      const double d = T[j + j * ld];
      if (!(d > 0.0)) bad = 1;
      T[j + j * ld] = sqrt(fmax(d, 0.0));
    }
    __syncthreads();
    const double djj = T[j + j * ld];
    for (int i = j + 1 + threadIdx.x; i < m; i += NT) T[i + j * ld] /= djj;
    __syncthreads();
    for (int e = threadIdx.x; e < (m - j - 1) * (m - j - 1); e += NT) {
      const int i = j + 1 + e % (m - j - 1), c = j + 1 + e / (m - j - 1);
      if (i >= c) T[i + c * ld] -= T[i + j * ld] * T[c + j * ld];
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < m * m; e += NT) {
    const int i = e % m, j = e / m;
    N[i + j * M.lmax] = i >= j ? T[i + j * ld] : 0.0;
  }
  if (threadIdx.x == 0 && bad) {
    atomicExch(M.flags + 1, 1);
    atomicExch(M.flags + 2, t);
  }
}

__device__ void it_getrf(const MatDev& M, int slot, int t, int item_, int nitems_, double* smx_) {
  double* T = smx_;
  double& nrm = smx_[64 * 65 + 1];
  int& bad = *(int*)(smx_ + 64 * 65 + 2);
  double* N = M.N + (size_t)slot * M.lmax * M.lmax;
  const int m = M.row.hi[t] - M.row.lo[t];
  const int ld = 65;
  for (int e = threadIdx.x; e < m * m; e += NT) T[(e % m) + (e / m) * ld] = N[(e % m) + (e / m) * M.lmax];
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int e = 0; e < m * m; ++e) s += T[(e % m) + (e / m) * ld] * T[(e % m) + (e / m) * ld];
    nrm = sqrt(s);
    bad = 0;
  }
  __syncthreads();
  for (int j = 0; j < m; ++j) {
    const double p = T[j + j * ld];
    if (threadIdx.x == 0 && !(fabs(p) > 1e-14 * nrm)) bad = 1;
    for (int i = j + 1 + threadIdx.x; i < m; i += NT) T[i + j * ld] /= p;
    __syncthreads();
    for (int e = threadIdx.x; e < (m - j - 1) * (m - j - 1); e += NT) {
      const int i = j + 1 + e % (m - j - 1), c = j + 1 + e / (m - j - 1);
      T[i + c * ld] -= T[i + j * ld] * T[j + c * ld];
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < m * m; e += NT) N[(e % m) + (e / m) * M.lmax] = T[(e % m) + (e / m) * ld];
  if (threadIdx.x == 0 && bad) {
    atomicExch(M.flags + 1, 1);
    atomicExch(M.flags + 2, t);
  }
}

// Inverse of a diagonal leaf tile (Remark 1: "if t is a leaf, we can compute the
// inverse directly"): Gauss-Jordan on [T | I] in shared memory, pivots in the elimination order of
// the no-pivot LU, so the breakdown rule is the leaf LR's (reading own-2: |p| <= 1e-14 ||T||_F).
__device__ void it_tinv(const MatDev& M, int slot, int t, int item_, int nitems_, double* smx_) {
  constexpr int LD = 65;
  double* G = smx_;                  // m x 2m, ld LD
  double* f = G + LD * 128;          // column-j multipliers
  double& nrm = f[64];
  int& bad = *(int*)(f + 65);
  double* N = M.N + (size_t)slot * M.lmax * M.lmax;
  const int m = M.row.hi[t] - M.row.lo[t];
  for (int e = threadIdx.x; e < m * 2 * m; e += NT) {
    const int i = e % m, c = e / m;
    G[i + c * LD] = c < m ? N[i + (size_t)c * M.lmax] : (c - m == i ? 1.0 : 0.0);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int e = 0; e < m * m; ++e) s += G[(e % m) + (e / m) * LD] * G[(e % m) + (e / m) * LD];
    nrm = sqrt(s);
    bad = 0;
  }
  __syncthreads();
  for (int j = 0; j < m; ++j) {
    const double p = G[j + j * LD];
    if (threadIdx.x == 0 && !(fabs(p) > 1e-14 * nrm)) bad = 1;
    for (int i = threadIdx.x; i < m; i += NT) f[i] = G[i + j * LD];
    __syncthreads();
    for (int c = threadIdx.x; c < 2 * m; c += NT) G[j + c * LD] /= p;
    __syncthreads();
    for (int e = threadIdx.x; e < m * 2 * m; e += NT) {
      const int i = e % m, c = e / m;
      if (i != j) G[i + c * LD] -= f[i] * G[j + c * LD];
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < m * m; e += NT) N[(e % m) + (size_t)(e / m) * M.lmax] = G[(e % m) + (e / m + m) * LD];
  if (threadIdx.x == 0 && bad) {
    atomicExch(M.flags + 1, 1);
    atomicExch(M.flags + 2, t);
  }
}

// Triangular solve with a leaf tile (m <= 32), one warp per 4 right-hand sides: lane i holds row
// i of the 4 vectors and the 32 tile entries it needs (loaded once from the tile), every step is
// one scaling, one shuffle broadcast and one FMA per vector (no shared memory, no block barrier).
__device__ __forceinline__ void trsm_warp32(int mode, int m, const double* N, int lmax, double* B, int ldb,
                                            int nvec, int v0, int vstride) {
  const int lane = threadIdx.x & 31;
  const bool rowwise = (mode == RLT || mode == RUN);
  const bool fwd = !(mode == LLT || mode == LUN);
  const bool unit = mode == LLU;
  // lane i needs A[i][j] of the operator applied: L (LLN/LLU/RLT), L^T (LLT), U^T (RUN/LUT), U (LUN)
  const bool byrow = (mode == RLT || mode == LLN || mode == LLU || mode == LUN);
  double r[32];
#pragma unroll
  for (int j = 0; j < 32; ++j)
    r[j] = (lane < m && j < m) ? (byrow ? N[lane + (size_t)j * lmax] : N[j + (size_t)lane * lmax]) : 0.0;
  const double invd = lane < m ? 1.0 / N[lane + (size_t)lane * lmax] : 0.0;
  constexpr int VPW = 4;
  for (int vb = v0; vb < nvec; vb += vstride) {
    double x[VPW];
#pragma unroll
    for (int q = 0; q < VPW; ++q) {
      const int v = vb + q;
      x[q] = (v < nvec && lane < m) ? (rowwise ? B[v + (size_t)lane * ldb] : B[(size_t)v * ldb + lane]) : 0.0;
    }
    if (fwd) {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        if (j < m) {
#pragma unroll
          for (int q = 0; q < VPW; ++q) {
            const double z = __shfl_sync(0xffffffffu, unit ? x[q] : x[q] * invd, j);
            x[q] = lane == j ? z : (lane > j ? x[q] - r[j] * z : x[q]);
          }
        }
      }
    } else {
#pragma unroll
      for (int j = 31; j >= 0; --j) {
        if (j < m) {
#pragma unroll
          for (int q = 0; q < VPW; ++q) {
            const double z = __shfl_sync(0xffffffffu, x[q] * invd, j);
            x[q] = lane == j ? z : (lane < j ? x[q] - r[j] * z : x[q]);
          }
        }
      }
    }
#pragma unroll
    for (int q = 0; q < VPW; ++q) {
      const int v = vb + q;
      if (v < nvec && lane < m) {
        if (rowwise) B[v + (size_t)lane * ldb] = x[q];
        else B[(size_t)v * ldb + lane] = x[q];
      }
    }
  }
}

__device__ void it_trsm(const MatDev& M, int slot, int m, int mode, double* B, int ldb, int brows,
                                             Dim bcols, int item_, int nitems_, double* smx_) {
  const double* N = M.N + (size_t)slot * M.lmax * M.lmax;
  if (m <= 32) {
    const int nv = (mode == RLT || mode == RUN) ? brows : bcols.v();
    const int w = threadIdx.x >> 5;
    trsm_warp32(mode, m, N, M.lmax, B, ldb, nv, item_ * (NT / 8) + w * 4, nitems_ * (NT / 8));
    return;
  }
  double* T = smx_;
  const int ld = 65;
  double* invd = T + 64 * ld;
  for (int e = threadIdx.x; e < m * m; e += NT) T[(e % m) + (e / m) * ld] = N[(e % m) + (e / m) * M.lmax];
  for (int j = threadIdx.x; j < m; j += NT) invd[j] = 1.0 / N[j + (size_t)j * M.lmax];
  __syncthreads();
  const bool rowwise = (mode == RLT || mode == RUN);
  const int nvec = rowwise ? brows : bcols.v();
  for (int v = item_ * NT + threadIdx.x; v < nvec; v += nitems_ * NT) {
    // rowwise: x = row v of B (length m, stride ldb); columnwise: x = column v (length m, stride 1)
    double* x = rowwise ? B + v : B + (size_t)v * ldb;
    const int st = rowwise ? ldb : 1;
    switch (mode) {
      case RLT:  // x L^T = b  <=>  L x^T = b^T  forward
      case LLN:
      case LLU:
        for (int j = 0; j < m; ++j) {
          double acc = x[j * st];
          for (int i = 0; i < j; ++i) acc -= T[j + i * ld] * x[i * st];
          x[j * st] = mode == LLU ? acc : acc * invd[j];
        }
        break;
      case LLT:  // L^T x = b  backward
        for (int j = m - 1; j >= 0; --j) {
          double acc = x[j * st];
          for (int i = j + 1; i < m; ++i) acc -= T[i + j * ld] * x[i * st];
          x[j * st] = acc * invd[j];
        }
        break;
      case RUN:  // x U = b  <=>  U^T x^T = b^T  forward
      case LUT:
        for (int j = 0; j < m; ++j) {
          double acc = x[j * st];
          for (int i = 0; i < j; ++i) acc -= T[i + j * ld] * x[i * st];
          x[j * st] = acc * invd[j];
        }
        break;
      case LUN:  // U x = b  backward
        for (int j = m - 1; j >= 0; --j) {
          double acc = x[j * st];
          for (int i = j + 1; i < m; ++i) acc -= T[j + i * ld] * x[i * st];
          x[j * st] = acc * invd[j];
        }
        break;
    }
  }
}

// ---- tall R-factor by streaming TSQR (one CTA) --------------------------------------------------
__device__ void it_tsqr_r(const double* A, int lda, int rows, Dim Kd, double* R, int ldr, int item_, int nitems_, double* smx_) {
  double* sm = smx_;
  constexpr int PL = PR + 1;
  double* P = sm;  // PR x KC, leading dim PL (odd)
  double* diag = P + PL * KC;
  double* red = diag + KC;
  const int K = Kd.v();
  int r = 0;  // rows currently in the panel
  for (int r0 = 0; r0 < rows;) {
    const int take = min(rows - r0, PR - r);
    for (int e = threadIdx.x; e < take * K; e += NT) {
      const int i = e % take, j = e / take;
      P[r + i + j * PL] = A[r0 + i + (size_t)j * lda];
    }
    r += take;
    r0 += take;
    la::cta_qr_R(P, PL, r, K, diag, red);
    r = min(r, K);
  }
  for (int e = threadIdx.x; e < K * K; e += NT) {
    const int i = e % K, j = e / K;
    R[i + j * ldr] = i < r ? P[i + j * PL] : 0.0;
  }
}

// ---- temporary truncation core ----------------------------------------------------------------
__device__ void it_temp_core(const double* Ra, const double* Rb, int ldr, Dim Kd, double* Ma,
                                                  double* Mb, int ldm, int* rout, double rel, double abs_tol,
                                                  int max_rank, int cap, int* flags, const int* knew, int item_,
                                                  int nitems_, double* smx_) {
  if (knew && *knew == 0) {  // nothing added: the temporary stays exactly as it is (Ma = Mb = I)
    const int K = Kd.v();
    for (int e = threadIdx.x; e < K * K; e += NT) {
      const int i = e % K, j = e / K;
      Ma[i + j * ldm] = i == j ? 1.0 : 0.0;
      Mb[i + j * ldm] = i == j ? 1.0 : 0.0;
    }
    if (threadIdx.x == 0) *rout = K;
    return;
  }
  double* smt = smx_;
  constexpr int LT = KC + 1;
  double* Mm = smt;
  double* M0 = Mm + LT * KC;
  double* U = M0 + LT * KC;
  double* sig = U + LT * KC;
  int* order = (int*)(sig + KC);
  int* scr = order + KC;
  int& clamped = scr[3];
  const int K = Kd.v();
  // M = Ra Rb^T
  for (int e = threadIdx.x; e < K * K; e += NT) {
    const int i = e % K, j = e / K;
    double acc = 0.0;
    for (int q = 0; q < K; ++q) acc += Ra[i + q * ldr] * Rb[j + q * ldr];
    U[j + i * LT] = acc;   // M^T
    M0[i + j * LT] = acc;
  }
  if (threadIdx.x == 0) clamped = 0;
  __syncthreads();
  // SVD of W = R_A^T with M^T = Q_A R_A (same singular values / left vectors, triangular start
  // for the Jacobi sweeps); small K: Jacobi on M directly
  if (K > 8) {
    la::cta_qr_R(U, LT, K, K, sig, (double*)order);
    for (int e = threadIdx.x; e < K * K; e += NT) {
      const int i = e % K, j = e / K;
      Mm[i + j * LT] = U[j + i * LT];
    }
  } else {
    for (int e = threadIdx.x; e < K * K; e += NT) Mm[(e % K) + (e / K) * LT] = M0[(e % K) + (e / K) * LT];
  }
  __syncthreads();
  la::cta_jacobi(Mm, LT, K, K, sig, order, scr);
  const int r = K > 0 ? la::trunc_rank(sig, order, K, rel, abs_tol, max_rank, cap, &clamped) : 0;
  // U_r
  for (int e = threadIdx.x; e < K * r; e += NT) {
    const int i = e % K, q = e / K;
    U[i + q * LT] = Mm[i + order[q] * LT] / sig[order[q]];
  }
  __syncthreads();
  // V_r = M0^T U_r / sigma   (stored in Mm)
  for (int e = threadIdx.x; e < K * r; e += NT) {
    const int i = e % K, q = e / K;
    double acc = 0.0;
    for (int p = 0; p < K; ++p) acc += M0[p + i * LT] * U[p + q * LT];
    Mm[i + q * LT] = acc / sig[order[q]];
  }
  __syncthreads();
  // Ma = Rb^T V_r ; Mb = Ra^T U_r / sigma
  for (int e = threadIdx.x; e < K * r; e += NT) {
    const int i = e % K, q = e / K;
    double a = 0.0, b = 0.0;
    for (int p = 0; p < K; ++p) {
      a += Rb[p + i * ldr] * Mm[p + q * LT];
      b += Ra[p + i * ldr] * U[p + q * LT];
    }
    Ma[i + q * ldm] = a;
    Mb[i + q * ldm] = b / sig[order[q]];
  }
  if (threadIdx.x == 0) {
    *rout = r;
    if (clamped) atomicOr(flags, 1);
  }
}

__device__ void it_copy_cols(double* dst, int ldd, const double* src, int lds, int rows, Dim cols, int item_, int nitems_, double* smx_) {
  const int c = cols.v();
  const long long tot = (long long)rows * c;
  for (long long e = (long long)item_ * blockDim.x + threadIdx.x; e < tot; e += (long long)nitems_ * blockDim.x) {
    const int i = (int)(e % rows), j = (int)(e / rows);
    dst[i + (size_t)j * ldd] = src[i + (size_t)j * lds];
  }
}

__device__ void it_set_int(int* p, Dim v, int item_, int nitems_, double* smx_) {
  if (threadIdx.x == 0) *p = v.v();
}
__device__ void it_gather_cols(double* Bt, const double* x, const int64_t* perm, int n, int nrhs, int64_t ldx, int item_, int nitems_, double* smx_) {
  for (long long e = (long long)item_ * blockDim.x + threadIdx.x; e < (long long)n * nrhs; e += (long long)nitems_ * blockDim.x) {
    const int i = (int)(e % n), c = (int)(e / n);
    Bt[e] = x[perm[i] + c * ldx];
  }
}
__device__ void it_scatter_cols(double* x, const double* Bt, const int64_t* perm, int n, int nrhs, int64_t ldx, int item_, int nitems_, double* smx_) {
  for (long long e = (long long)item_ * blockDim.x + threadIdx.x; e < (long long)n * nrhs; e += (long long)nitems_ * blockDim.x) {
    const int i = (int)(e % n), c = (int)(e / n);
    x[perm[i] + c * ldx] = Bt[e];
  }
}
__device__ void it_rank_if(int* p, const int* a, const int* b, int item_, int nitems_, double* smx_) {
  if (threadIdx.x == 0) *p = (*a > 0 && *b > 0) ? *b : 0;
}
// stack [T (rows x kT), zero-extended N (rows_new at row_off, knew cols)] -> dst (rows x (kT+knew))
__device__ void it_stack(double* dst, int ldd, int rows, const double* T, int ldt, const int* kT, const double* Nw,
                        int ldn, int row_off, int rows_new, Dim knew, int item_, int nitems_, double* smx_) {
  const int kt = kT ? *kT : 0, kn = knew.v();
  const long long tot = (long long)rows * (kt + kn);
  for (long long e = (long long)item_ * blockDim.x + threadIdx.x; e < tot; e += (long long)nitems_ * blockDim.x) {
    const int i = (int)(e % rows), j = (int)(e / rows);
    double v;
    if (j < kt) v = T[i + (size_t)j * ldt];
    else {
      const int ii = i - row_off;
      v = (ii >= 0 && ii < rows_new) ? Nw[ii + (size_t)(j - kt) * ldn] : 0.0;
    }
    dst[i + (size_t)j * ldd] = v;
  }
}
// choose the Case-2 factorisation of C = S^X G S^Y (k1 x k2), reading R23:
// k1 <= k2: A = V^X (Ca = I), B = W^Y C^T (Cb = C^T); else A = V^X C (Ca = C), B = W^Y (Cb = I)
__device__ void it_choose(const double* Cm, int ldc, const int* k1p, const int* k2p, double* Ca, double* Cb, int ldo,
                         int* kout, int item_, int nitems_, double* smx_) {
  const int k1 = *k1p, k2 = *k2p;
  const bool first = k1 <= k2;
  const int kk = first ? k1 : k2;
  for (int e = threadIdx.x; e < KC * KC; e += blockDim.x) {
    const int i = e % KC, j = e / KC;
    if (j < kk) {
      if (i < k1) Ca[i + j * ldo] = first ? (i == j ? 1.0 : 0.0) : Cm[i + j * ldc];
      if (i < k2) Cb[i + j * ldo] = first ? Cm[j + i * ldc] : (i == j ? 1.0 : 0.0);
    }
  }
  if (threadIdx.x == 0) *kout = kk;
}
// Case 2 with both factors admissible (reading R23), fused into one CTA (was up to
// three GEMM ops and a choose op, each behind a cluster barrier): G = W^X_s^T V^Y_s (when the
// bases are passed; ms <= C2_MS, staged in shared memory), T1 = S^X_or G, C = T1 S^Y_or, then the
// factored side as it_choose.  Every sum runs over the inner index in increasing order, exactly
// as it_gemm, so the result is bit-identical to the unfused sequence.
constexpr int C2_MS = 64;
__device__ void it_c2core(const PC2& q, double* sm) {
  constexpr int RC = RCAP_MAX, LD = RC + 1;  // every rank here is a stored rank (<= rank_cap)
  const int kxt = *q.kd[0], kxs = *q.kd[1], kys = *q.kd[2], kyr = *q.kd[3];
  double* Gs = sm;              // kxs x kys (ld LD)
  double* T1 = Gs + LD * RC;    // kxt x kys
  double* Cm = T1 + LD * RC;    // kxt x kyr
  double* Ws = Cm + LD * RC;    // ms x kxs (ld C2_MS)
  double* Vs = Ws + C2_MS * RC; // ms x kys
  const double* G = q.G;
  int ldg = KC;
  if (q.W) {
    const int ms = q.ms;
    for (int e = threadIdx.x; e < ms * kxs; e += NT) Ws[(e % ms) + (e / ms) * C2_MS] = q.W[(e % ms) + (size_t)(e / ms) * ms];
    for (int e = threadIdx.x; e < ms * kys; e += NT) Vs[(e % ms) + (e / ms) * C2_MS] = q.V[(e % ms) + (size_t)(e / ms) * ms];
    __syncthreads();
    for (int e = threadIdx.x; e < kxs * kys; e += NT) {
      const int i = e % kxs, j = e / kxs;
      double acc = 0.0;
      for (int r = 0; r < ms; ++r) acc += Ws[r + i * C2_MS] * Vs[r + j * C2_MS];
      Gs[i + j * LD] = acc;
    }
    __syncthreads();
    G = Gs;
    ldg = LD;
  }
  for (int e = threadIdx.x; e < kxt * kys; e += NT) {
    const int i = e % kxt, j = e / kxt;
    double acc = 0.0;
    for (int r = 0; r < kxs; ++r) acc += (q.tx ? q.Sx[r + (size_t)i * q.ldsx] : q.Sx[i + (size_t)r * q.ldsx]) * G[r + j * ldg];
    T1[i + j * LD] = acc;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < kxt * kyr; e += NT) {
    const int i = e % kxt, j = e / kxt;
    double acc = 0.0;
    for (int r = 0; r < kys; ++r) acc += T1[i + r * LD] * (q.ty ? q.Sy[j + (size_t)r * q.ldsy] : q.Sy[r + (size_t)j * q.ldsy]);
    Cm[i + j * LD] = acc;
  }
  __syncthreads();
  const bool first = kxt <= kyr;
  const int kk = first ? kxt : kyr;
  for (int e = threadIdx.x; e < RC * RC; e += NT) {
    const int i = e % RC, j = e / RC;
    if (j < kk) {
      if (i < kxt) q.Ca[i + j * q.ldo] = first ? (i == j ? 1.0 : 0.0) : Cm[i + j * LD];
      if (i < kyr) q.Cb[i + j * q.ldo] = first ? Cm[j + i * LD] : (i == j ? 1.0 : 0.0);
    }
  }
  if (threadIdx.x == 0) *q.kout = kk;
}

__device__ void it_identity(double* I, int ld, int m, int item_, int nitems_, double* smx_) {
  for (int e = threadIdx.x + item_ * blockDim.x; e < m * m; e += blockDim.x * nitems_)
    I[(e % m) + (e / m) * ld] = (e % m) == (e / m) ? 1.0 : 0.0;
}
__device__ void it_transpose_tile(double* dst, int ldd, const double* src, int lds, int rows, int cols, int item_, int nitems_, double* smx_) {
  for (int e = threadIdx.x + item_ * blockDim.x; e < rows * cols; e += blockDim.x * nitems_) {
    const int i = e % rows, j = e / rows;  // dst (rows x cols) = src^T
    dst[i + j * ldd] = src[j + i * lds];
  }
}
__device__ void it_add_int(int* p, Dim a, Dim b, int item_, int nitems_, double* smx_) {
  if (threadIdx.x == 0) *p = a.v() + b.v();
}

}  // namespace ar
}  // namespace h2

namespace h2 {
namespace ar {
// Case 2 with both factors dense leaf blocks and a low-rank target (reading own-7):
// P = op(X)|_{t x s} op(Y)|_{s x r} (mt x mr), interpolative decomposition by column-pivoted
// Householder QR  P Pi = Q R  (pivot = remaining column of largest norm, first index on ties),
// stopped at the first step j with |R_jj| <= rel |R_00| -> r = j (P = 0 -> r = 0);
// A = P[:, piv[0..r)] (the r pivot columns, exact copies), B^T = [I_r, R_11^{-1} R_12] Pi^T.
// One CTA; groups of S lanes own one column each (as la::cta_qr_R); the remaining-row norms of
// every column are recomputed exactly after each reflection by the owning group.
__device__ void it_dd_compress(const MatDev& MX, const MatDev& MY, int slotx, int transx, int sloty, int transy,
                               int mt, int ms, int mr, double* A, int lda, double* B, int ldb, int* kout, double rel,
                               int item_, int nitems_, double* smx_) {
  constexpr int L = KC + 1;
  constexpr int TL = 65;   // staged tiles (<= 64 x 64)
  double* P = smx_;        // mt x mr (mr <= 64 columns), QR in place
  double* P0 = P + L * 64; // copy of P (original column order)
  double* Xs = P0 + L * 64;  // op(X)|_{t x s}  (mt x ms, ld TL)
  double* Ys = Xs + TL * 64; // op(Y)|_{s x r}  (ms x mr, ld TL)
  double* cn = Ys + TL * 64; // squared norms of the remaining rows, per (current) column
  double* diag = cn + KC;    // R_jj
  double* red = diag + KC;   // [0] = |R_00|, [1] = |a_j|^2
  int* piv = (int*)(red + 8);
  int* ctl = piv + KC;       // [0] = pivot column (-1: stop)
  const double* NX = MX.N + (size_t)slotx * MX.lmax * MX.lmax;
  const double* NY = MY.N + (size_t)sloty * MY.lmax * MY.lmax;
  const int lx = MX.lmax, ly = MY.lmax;
  const int tid = threadIdx.x, m = mt, n = mr;
  // both tiles into shared memory in one load round (the product then reads shared memory only;
  // the same sums in the same order as reading them from global memory)
  for (int e = tid; e < m * ms; e += NT) {
    const int i = e % m, q = e / m;
    Xs[i + q * TL] = transx ? NX[q + i * lx] : NX[i + q * lx];
  }
  for (int e = tid; e < ms * n; e += NT) {
    const int q = e % ms, j = e / ms;
    Ys[q + j * TL] = transy ? NY[j + q * ly] : NY[q + j * ly];
  }
  __syncthreads();
  for (int e = tid; e < m * n; e += NT) {
    const int i = e % m, j = e / m;
    double acc = 0.0;
    for (int q = 0; q < ms; ++q) acc += Xs[i + q * TL] * Ys[q + j * TL];
    P[i + j * L] = acc;
    P0[i + j * L] = acc;
  }
  for (int j = tid; j < n; j += NT) piv[j] = j;
  int npow = 1;
  while (npow < n) npow *= 2;
  int S = NT / npow;
  if (S > 32) S = 32;
  if (S < 1) S = 1;
  const int c = tid / S, sl = tid % S;
  const unsigned gm = la::group_mask(S);
  __syncthreads();
  {
    double part = 0.0;
    if (c < n)
      for (int i = sl; i < m; i += S) part += P[i + c * L] * P[i + c * L];
    for (int o = S / 2; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if (c < n && sl == 0) cn[c] = part;
  }
  __syncthreads();
  const int jmax = m < n ? m : n;
  int r = jmax;
  for (int j = 0; j < jmax; ++j) {
    if (tid == 0) {
      int p = j;
      double best = cn[j];
      for (int q = j + 1; q < n; ++q)
        if (cn[q] > best) {
          best = cn[q];
          p = q;
        }
      const double nrm = sqrt(best);
      if (j == 0) red[0] = nrm;
      if (nrm <= rel * red[0]) {
        ctl[0] = -1;
      } else {
        ctl[0] = p;
        const int tp = piv[j];
        piv[j] = piv[p];
        piv[p] = tp;
        cn[p] = cn[j];
        cn[j] = best;
      }
    }
    __syncthreads();
    const int p = ctl[0];
    if (p < 0) {
      r = j;
      break;
    }
    if (p != j) {
      for (int i = tid; i < m; i += NT) {
        const double tmp = P[i + j * L];
        P[i + j * L] = P[i + p * L];
        P[i + p * L] = tmp;
      }
      __syncthreads();
    }
    double part = 0.0;
    if (c >= j && c < n)
      for (int i = j + sl; i < m; i += S) part += P[i + j * L] * P[i + c * L];
    for (int o = S / 2; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if (c == j && sl == 0) red[1] = part;
    __syncthreads();
    const double nrm2 = red[1];
    const double ajj = P[j + j * L];
    const double nrm = sqrt(nrm2);
    const double alpha = ajj > 0.0 ? -nrm : nrm;
    const double half_vtv = nrm2 - alpha * ajj;
    if (c > j && c < n) {
      const double ajc = P[j + c * L];
      __syncwarp(gm);
      const double f = (part - alpha * ajc) / half_vtv;
      for (int i = j + sl; i < m; i += S) {
        const double vi = (i == j) ? (ajj - alpha) : P[i + j * L];
        P[i + c * L] -= f * vi;
      }
      __syncwarp(gm);
      double q2 = 0.0;
      for (int i = j + 1 + sl; i < m; i += S) q2 += P[i + c * L] * P[i + c * L];
      for (int o = S / 2; o; o >>= 1) q2 += __shfl_xor_sync(gm, q2, o);
      if (sl == 0) cn[c] = q2;
    }
    if (tid == 0) diag[j] = alpha;
    __syncthreads();
  }
  // T = R_11^{-1} R_12 in place of R_12 (one thread per right-hand side column)
  for (int cc = r + tid; cc < n; cc += NT) {
    for (int i = r - 1; i >= 0; --i) {
      double x = P[i + cc * L];
      for (int k = i + 1; k < r; ++k) x -= P[i + k * L] * P[k + cc * L];
      P[i + cc * L] = x / diag[i];
    }
  }
  __syncthreads();
  for (int e = tid; e < m * r; e += NT) {
    const int i = e % m, q = e / m;
    A[i + (size_t)q * lda] = P0[i + piv[q] * L];
  }
  for (int e = tid; e < n * r; e += NT) {
    const int cc = e % n, q = e / n;  // row piv[cc] of B
    B[piv[cc] + (size_t)q * ldb] = cc < r ? (cc == q ? 1.0 : 0.0) : P[q + cc * L];
  }
  if (tid == 0) *kout = r;
}
}  // namespace ar
}  // namespace h2
