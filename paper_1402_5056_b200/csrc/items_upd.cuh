// Device items of the local low-rank update U0-U6, executed by the op executor
// (h2_exec.cu).  Item i of an op is what one CTA of the corresponding phase computes; see the
// phase list in h2_exec.cu.  Generated from the per-phase kernels of round 1 (same arithmetic).
#pragma once
#include <cuda_runtime.h>

#include "devla.cuh"
#include "exec.h"

namespace h2 {
namespace upd {

constexpr int NT = NTHREADS;
constexpr int KC = KCAP_MAX;      // 96
constexpr int RM = KC + 1;        // (odd) leading dim of V~_t / V^_t in the SVD items: max(lmax, 2 rank_cap) <= 96 rows
constexpr int PR = 192;           // TSQR panel rows (>= KC + largest chunk)
constexpr int PRL = PR + 1;       // odd leading dimensions: column-parallel loops hit distinct smem banks
constexpr int LD2 = 2 * KC + 1;   // (odd) leading dim of a stacked pair of KC x KC factors

__device__ __forceinline__ bool inside(const DevSide& D, int t, int root) {
  return t >= root && t < root + D.tsize[root];
}

__device__ double weights_cluster(const MatDev& M, const UpdArgs& a, bool rs, int t, double* sm, int mode);

// ---- U0 + U1/U2 leaves + local weight stacks of the ancestors (all independent) ---------------
__device__ void it_upd_ext_leaf(const MatDev& M, UpdArgs a_, int rl0, int nrl, int cl0, int ncl,
                                                     int in0, int nin, int npA, int npB, int item_, int nitems_, double* smx_) {
  UpdArgs a = a_;
  if (a.kdev) a.k = *a.kdev;
  if (a.k <= 0) return;
  double* sm = smx_;
  const int b = item_;
  if (b >= nrl + ncl + nin) {
    // U3 (part): C_a = R(local stack) for the proper ancestors a of t0 (side A) / s0 (side B)
    const int j = b - (nrl + ncl + nin);
    const bool rs = j < npA;
    const DevSide& D = rs ? M.row : M.col;
    int t = rs ? a.t0 : a.s0;
    const int lev = rs ? j : j - npA;  // ancestor at this level
    for (int up = (rs ? npA : npB) - lev; up > 0; --up) t = D.parent[t];
    const double fl = weights_cluster(M, a, rs, t, sm, 1 /*W_LOCAL*/);
    if (a.prof && threadIdx.x == 0) atomicAdd(a.prof + 2 * K_W_PATH, fl);
    return;
  }
  if (b == 0 && threadIdx.x == 0 && nrl + ncl > 0) atomicAdd(M.flags + 3, 1);  // non-zero-rank update count
  if (b < nrl + ncl) {
    const bool rs = b < nrl;
    const DevSide& D = rs ? M.row : M.col;
    const int t = D.leaves[rs ? rl0 + b : cl0 + b - nrl];
    const int root = rs ? a.t0 : a.s0;
    const double* Xf = rs ? a.X : a.Y;
    const int64_t ldx = rs ? a.ldx : a.ldy;
    const double al = rs ? a.alpha : 1.0;
    const int m = D.hi[t] - D.lo[t], kt = D.rank[t], K = kt + a.k;
    const int lda = M.lmax | 1;
    double* A = sm;                 // lmax x KC
    double* diag = A + lda * KC;    // KC
    double* red = diag + KC;        // 1
    const double* Vb = D.leafb + (size_t)D.leafidx[t] * M.lmax * M.rcap;
    const int off = D.lo[t] - D.lo[root];
    for (int e = threadIdx.x; e < m * K; e += NT) {
      const int i = e % m, j = e / m;
      A[i + j * lda] = j < kt ? Vb[i + (size_t)j * M.lmax] : al * Xf[off + i + (size_t)(j - kt) * ldx];
    }
    __syncthreads();
    la::cta_qr_R(A, lda, m, K, diag, red);
    double* RE = D.re + (size_t)t * M.kcap * M.kcap;
    const int mk = m < K ? m : K;
    for (int e = threadIdx.x; e < K * K; e += NT) {
      const int i = e % K, j = e / K;
      RE[i + j * M.kcap] = i < mk ? A[i + j * lda] : 0.0;
    }
    if (a.prof && threadIdx.x == 0) atomicAdd(a.prof + 2 * K_EXT_LEAF, hh_flops(m, K));
    return;
  }
  // U0: exact nearfield part N_b += alpha X|t Y|s^T for the inadmissible leaves of T_{b0}
  const int slot = in0 + (b - nrl - ncl);
  if (slot >= in0 + nin) return;
  const int t = M.in_t[slot], s = M.in_s[slot];
  const int mt = M.row.hi[t] - M.row.lo[t], ms = M.col.hi[s] - M.col.lo[s];
  const int ot = M.row.lo[t] - M.row.lo[a.t0], os = M.col.lo[s] - M.col.lo[a.s0];
  double* Na = M.N + (size_t)slot * M.lmax * M.lmax;
  for (int e = threadIdx.x; e < mt * ms; e += NT) {
    const int i = e % mt, j = e / mt;
    double acc = 0.0;
    for (int q = 0; q < a.k; ++q) acc += a.X[ot + i + (size_t)q * a.ldx] * a.Y[os + j + (size_t)q * a.ldy];
    Na[i + (size_t)j * M.lmax] += a.alpha * acc;
  }
  if (a.prof && threadIdx.x == 0) atomicAdd(a.prof + 2 * K_EXT_LEAF, 2.0 * mt * ms * a.k);
}

// ---- U2 internal, bottom-up ------------------------------------------------------------------
__device__ void it_upd_ext_level(const MatDev& M, UpdArgs a_, int bA, int nA, int bB, int nB, int item_, int nitems_, double* smx_) {
  UpdArgs a = a_;
  if (a.kdev) a.k = *a.kdev;
  if (a.k <= 0) return;
  double* sm = smx_;
  const bool rs = (int)item_ < nA;
  const DevSide& D = rs ? M.row : M.col;
  const int t = D.bfs[rs ? bA + item_ : bB + item_ - nA];
  if (D.son0[t] < 0) return;
  const int k = a.k, kt = D.rank[t], K = kt + k;
  double* A = sm;              // LD2 x KC
  double* diag = A + LD2 * KC;
  double* red = diag + KC;
  int row0 = 0;
  for (int q = 0; q < 2; ++q) {
    const int c = q ? D.son1[t] : D.son0[t];
    const int kc = D.rank[c], Kc = kc + k;
    const double* RE = D.re + (size_t)c * M.kcap * M.kcap;
    const double* E = D.tr + (size_t)c * M.rcap * M.rcap;  // kc x kt
    // rows row0..row0+Kc-1:  [ RE[:, :kc] E_c , RE[:, kc:kc+k] ]
    for (int e = threadIdx.x; e < Kc * K; e += NT) {
      const int i = e % Kc, j = e / Kc;
      double v;
      if (j < kt) {
        v = 0.0;
        for (int p = i; p < kc; ++p) v += RE[i + p * M.kcap] * E[p + j * M.rcap];  // RE upper triangular
      } else {
        v = RE[i + (kc + j - kt) * M.kcap];
      }
      A[row0 + i + j * LD2] = v;
    }
    row0 += Kc;
  }
  __syncthreads();
  la::cta_qr_R(A, LD2, row0, K, diag, red);
  double* RE = D.re + (size_t)t * M.kcap * M.kcap;
  const int mk = row0 < K ? row0 : K;
  for (int e = threadIdx.x; e < K * K; e += NT) {
    const int i = e % K, j = e / K;
    RE[i + j * M.kcap] = i < mk ? A[i + j * LD2] : 0.0;
  }
  if (a.prof && threadIdx.x == 0) {
    double f = hh_flops(row0, K);
    for (int q = 0; q < 2; ++q) {
      const int c = q ? D.son1[t] : D.son0[t];
      f += (double)(D.rank[c] + k) * D.rank[c] * kt;  // upper-triangular RE times E
    }
    atomicAdd(a.prof + 2 * K_EXT_LEVEL, f);
  }
}

// ---- U3 weights for one cluster t of side A (partner side B) --------------------------------
// mode W_FULL: B~_t = R([local stack; B~_{t+} E~_t^T]) -> bw[t]
// mode W_LOCAL: C_t = R(local stack) -> re[t]   (proper ancestors of t0 only: their re slot is free)
// mode W_CHAIN: B~_t = R([C_t; B~_{t+} E_t^T])   -> bw[t]  (C_t from re[t])
enum { W_FULL = 0, W_LOCAL = 1, W_CHAIN = 2 };

__device__ double weights_cluster(const MatDev& M, const UpdArgs& a, bool rs, int t, double* sm, int mode) {
  const DevSide& A = rs ? M.row : M.col;
  const DevSide& B = rs ? M.col : M.row;
  const int a0 = rs ? a.t0 : a.s0, b0 = rs ? a.s0 : a.t0;
  const int k = a.k;
  const bool in_t = inside(A, t, a0);
  const int kt = A.rank[t];
  const int K = kt + (in_t ? k : 0);
  double* P = sm;                 // PR x KC panel
  double* diag = P + PRL * KC;
  double* red = diag + KC;
  int rows = 0;
  double fl = 0.0;
  auto flush = [&]() {
    if (rows > 0) {
      la::cta_qr_R(P, PRL, rows, K, diag, red);
      fl += hh_flops(rows, K);
      rows = rows < K ? rows : K;
    }
  };
  if (mode == W_CHAIN) {
    la::cta_copy(P, PRL, A.re + (size_t)t * M.kcap * M.kcap, M.kcap, K, K);
    rows = K;
    __syncthreads();
  }
  for (int q = A.bptr[t]; mode != W_CHAIN && q < A.bptr[t + 1]; ++q) {
    const int slot = A.bidx[q];
    const int s = rs ? M.adm_s[slot] : M.adm_t[slot];
    const double* Sa = M.S + (size_t)slot * M.rcap * M.rcap;
    const bool in_s = inside(B, s, b0);
    const int ls = B.rank[s];
    const int rc = in_s ? ls + k : ls;
    if (rc == 0) continue;
    if (rows + rc > PR) flush();
    const double* RB = in_s ? B.re + (size_t)s * M.kcap * M.kcap : B.rc + (size_t)s * M.rcap * M.rcap;
    const int ldR = in_s ? M.kcap : M.rcap;
    for (int e = threadIdx.x; e < rc * K; e += NT) {
      const int i = e % rc, c = e / rc;
      double v = 0.0;
      if (c < kt) {
        // (R_B S~^T)(i,c) = sum_j R_B(i,j) S_or(c,j),   S_or = S (row side) or S^T (column side)
        for (int j = i; j < ls; ++j) v += RB[i + j * ldR] * (rs ? Sa[c + j * M.rcap] : Sa[j + c * M.rcap]);
      } else if (in_s) {
        v = RB[i + (ls + c - kt) * ldR];  // identity block of S~ = diag(S, I)
      }
      P[rows + i + c * PRL] = v;
    }
    fl += (double)rc * ls * kt;  // triangular R_B times S^T
    rows += rc;
    __syncthreads();
  }
  const int p = A.parent[t];
  if (p >= 0 && mode != W_LOCAL) {
    const bool in_p = inside(A, p, a0);
    const int kp = A.rank[p];
    const int Kp = kp + (in_p ? k : 0);
    if (Kp > 0) {
      if (rows + Kp > PR) flush();
      const double* Bp = A.bw + (size_t)p * M.kcap * M.kcap;
      const double* E = A.tr + (size_t)t * M.rcap * M.rcap;  // kt x kp
      for (int e = threadIdx.x; e < Kp * K; e += NT) {
        const int i = e % Kp, c = e / Kp;
        double v = 0.0;
        if (c < kt) {
          for (int j = 0; j < kp; ++j) v += Bp[i + j * M.kcap] * E[c + j * M.rcap];
        } else if (in_p) {
          v = Bp[i + (kp + c - kt) * M.kcap];  // E~_t = diag(E_t, I) inside T_{t0}
        }                                      // E~_{t0} = [E_{t0}; 0]: zero columns
        P[rows + i + c * PRL] = v;
      }
      fl += 2.0 * Kp * kp * kt;
      rows += Kp;
      __syncthreads();
    }
  }
  flush();
  double* Bt = (mode == W_LOCAL ? A.re : A.bw) + (size_t)t * M.kcap * M.kcap;
  for (int e = threadIdx.x; e < K * K; e += NT) {
    const int i = e % K, j = e / K;
    Bt[i + j * M.kcap] = i < rows ? P[i + j * PRL] : 0.0;
  }
  __syncthreads();
  return fl;
}

__device__ void it_upd_weights_path(const MatDev& M, UpdArgs a_, int item_, int nitems_, double* smx_) {
  UpdArgs a = a_;
  if (a.kdev) a.k = *a.kdev;
  if (a.k <= 0) return;
  double* sm = smx_;
  const bool rs = item_ == 0;
  const DevSide& A = rs ? M.row : M.col;
  int path[64];
  int np = 0;
  for (int t = rs ? a.t0 : a.s0; t >= 0 && np < 64; t = A.parent[t]) path[np++] = t;
  double fl = 0.0;
  // proper ancestors: chain on their local stacks (computed in parallel by k_upd_ext_leaf); t0: full
  for (int q = np - 1; q >= 0; --q) fl += weights_cluster(M, a, rs, path[q], sm, q == 0 ? W_FULL : W_CHAIN);
  if (a.prof && threadIdx.x == 0) atomicAdd(a.prof + 2 * K_W_PATH, fl);
}

__device__ void it_upd_weights_level(const MatDev& M, UpdArgs a_, int bA, int nA, int bB, int nB, int item_, int nitems_, double* smx_) {
  UpdArgs a = a_;
  if (a.kdev) a.k = *a.kdev;
  if (a.k <= 0) return;
  double* sm = smx_;
  const bool rs = (int)item_ < nA;
  const DevSide& A = rs ? M.row : M.col;
  const int t = A.bfs[rs ? bA + item_ : bB + item_ - nA];
  const double fl = weights_cluster(M, a, rs, t, sm, W_FULL);
  if (a.prof && threadIdx.x == 0) atomicAdd(a.prof + 2 * K_W_LEVEL, fl);
}

// ---- U4 truncated nested basis --------------------------------------------------------------
// Given V (m x K, ldv) in shared memory and B~_t, compute M = V B~^T, its SVD, the rank, Q and R_t.
__device__ void svd_core(const MatDev& M, const UpdArgs& a, const DevSide& D, int t, double* V, int ldv, int m,
                         int K, double* sm_rest, int kid, double extra_flops) {
  // U4: left singular vectors / values of M = V B~^T (m x K).  K <= m <= 16: one-sided Jacobi
  // on M in registers of one warp.  K <= 32: Householder R of M, then the same on the
  // min(m, K) columns of R^T (length K), U Sigma = M Y Sigma^-1 (see below).  Otherwise: the SVD is taken
  // of W = R_A^T (m x p, p = min(m, K)) where M^T = Q_A R_A (Householder): M = W Q_A^T with Q_A
  // orthonormal, so W has the singular values and left singular vectors of M, fewer columns and
  // a triangular (preconditioned) start for the one-sided Jacobi (CTA version).
  double* Bt = sm_rest;             // KC x KC (ld RM); later W = R_A^T (m x p, ld RM)
  double* Mm = Bt + RM * KC;        // M^T (K x m, ld RM); later Q (m x r, ld RM)
  double* sig = Mm + RM * KC;       // KC
  int* order = (int*)(sig + KC);    // KC ints
  int* scr = order + KC;            // 4 ints
  const double* Bg = D.bw + (size_t)t * M.kcap * M.kcap;
  const long long c0 = clock64();
  la::cta_copy(Bt, RM, Bg, M.kcap, K, K);
  __syncthreads();
  long long c1;
  int p, sweeps;
  double* W = Bt;
  if (K <= m && m <= 16) {  // K columns of length m <= 16 (no QR)
    // M = V B~^T (m x K) in Mm; one-sided Jacobi on M in registers of one warp (lane j owns
    // column j), W = M J = [sigma_j u_j] into Bt (free after the product)
    la::cta_gemm(Mm, RM, V, ldv, false, Bt, RM, true, m, K, K, false);
    __syncthreads();
    c1 = clock64();
    if (m <= 16) sweeps = la::warp_jacobi<16, false>(Mm, RM, m, K, W, RM, sig, order, scr);
    else sweeps = la::warp_jacobi<32, false>(Mm, RM, m, K, W, RM, sig, order, scr);
    p = K;
  } else if (K <= 32) {
    // M = V B~^T (m x K) in Mm; R of M = Q R (Householder, in Bt[:, 0:32)); one-sided Jacobi on
    // the columns of R^T (K x p, p = min(m, K)) in registers of one warp: R^T J = Y with columns
    // y_j = sigma_j v_j (v_j: right singular vectors of R and M), so M y_j / sigma_j = sigma_j u_j
    // is column j of W (Bt[:, 64:96)).  No rotations to accumulate, columns of length K.
    la::cta_gemm(Mm, RM, V, ldv, false, Bt, RM, true, m, K, K, false);
    __syncthreads();
    double* Rw = Bt;
    double* Y = Bt + 32 * RM;
    W = Bt + 64 * RM;
    la::cta_copy(Rw, RM, Mm, RM, m, K);
    __syncthreads();
    la::cta_qr_R(Rw, RM, m, K, sig, (double*)order);
    const int pr = m < K ? m : K;
    for (int e = threadIdx.x; e < K * pr; e += NT) {  // R^T (K x pr) into W's slot as the input
      const int i = e % K, j = e / K;
      W[i + j * RM] = j <= i ? Rw[j + i * RM] : 0.0;
    }
    __syncthreads();
    c1 = clock64();
    if (K <= 8) sweeps = la::warp_jacobi<8, false>(W, RM, K, pr, Y, RM, sig, order, scr);
    else if (K <= 16) sweeps = la::warp_jacobi<16, false>(W, RM, K, pr, Y, RM, sig, order, scr);
    else sweeps = la::warp_jacobi<32, false>(W, RM, K, pr, Y, RM, sig, order, scr);
    for (int e = threadIdx.x; e < m * pr; e += NT) {
      const int i = e % m, j = e / m;
      double acc = 0.0;
      for (int q = 0; q < K; ++q) acc += Mm[i + q * RM] * Y[q + j * RM];
      W[i + j * RM] = sig[j] > 0.0 ? acc / sig[j] : 0.0;
    }
    p = pr;
    __syncthreads();
  } else {
    // M^T = B~ V^T  (K x m)
    la::cta_gemm(Mm, RM, Bt, RM, false, V, ldv, true, K, m, K, false);
    __syncthreads();
    la::cta_qr_R(Mm, RM, K, m, sig, (double*)order);  // R_A in the first min(K, m) rows (sig/order: scratch)
    p = K < m ? K : m;
    for (int e = threadIdx.x; e < m * p; e += NT) {
      const int i = e % m, j = e / m;
      W[i + j * RM] = Mm[j + i * RM];  // W = R_A^T
    }
    __syncthreads();
    c1 = clock64();
    sweeps = la::cta_jacobi(W, RM, m, p, sig, order, scr);
  }
  const long long c2 = clock64();
  int& clamped = scr[2];
  if (threadIdx.x == 0) clamped = 0;
  __syncthreads();
  const int r = la::trunc_rank(sig, order, p, a.rel_tol, a.abs_tol, a.max_rank, M.rcap, &clamped);
  double* Q = Mm;
  // Q(:, q) = W(:, order[q]) / sigma
  for (int e = threadIdx.x; e < m * r; e += NT) {
    const int i = e % m, q = e / m;
    const int j = order[q];
    Q[i + q * RM] = W[i + j * RM] / sig[j];
  }
  __syncthreads();
  double* qn = D.qn + (size_t)t * M.ldq * M.rcap;
  for (int e = threadIdx.x; e < m * r; e += NT) qn[(e % m) + (e / m) * M.ldq] = Q[(e % m) + (e / m) * RM];
  // R_t = Q^T V  (r x K)
  double* rn = D.rn + (size_t)t * M.kcap * M.kcap;
  la::cta_gemm(rn, M.kcap, Q, RM, true, V, ldv, false, r, K, m, false);
  if (threadIdx.x == 0) {
    D.rnew[t] = r;
    if (clamped) atomicOr(M.flags, 1);
    if (a.prof) {
      atomicAdd(a.prof + 2 * kid, extra_flops + 2.0 * m * K * K + svd_flops(m, K) + 2.0 * r * K * m);
      double* dbg = a.prof + 4 * K_COUNT;  // svd phase counters (profiling only)
      atomicAdd(dbg + 0, (double)(c1 - c0));
      atomicAdd(dbg + 1, (double)(c2 - c1));
      atomicAdd(dbg + 2, (double)(clock64() - c2));
      atomicAdd(dbg + 3, 1.0);
      atomicAdd(dbg + 4, (double)K);
      atomicAdd(dbg + 5, (double)m);
      atomicAdd(dbg + 6, (double)sweeps);
    }
  }
}

__device__ void it_upd_svd_leaf(const MatDev& M, UpdArgs a_, int rl0, int nrl, int cl0, int ncl, int item_, int nitems_, double* smx_) {
  UpdArgs a = a_;
  if (a.kdev) a.k = *a.kdev;
  if (a.k <= 0) return;
  double* sm = smx_;
  const bool rs = (int)item_ < nrl;
  const DevSide& D = rs ? M.row : M.col;
  const int t = D.leaves[rs ? rl0 + item_ : cl0 + item_ - nrl];
  const int root = rs ? a.t0 : a.s0;
  const double* Xf = rs ? a.X : a.Y;
  const int64_t ldx = rs ? a.ldx : a.ldy;
  const double al = rs ? a.alpha : 1.0;
  const int m = D.hi[t] - D.lo[t], kt = D.rank[t], K = kt + a.k;
  double* V = sm;  // RM x KC
  const double* Vb = D.leafb + (size_t)D.leafidx[t] * M.lmax * M.rcap;
  const int off = D.lo[t] - D.lo[root];
  for (int e = threadIdx.x; e < m * K; e += NT) {
    const int i = e % m, j = e / m;
    V[i + j * RM] = j < kt ? Vb[i + (size_t)j * M.lmax] : al * Xf[off + i + (size_t)(j - kt) * ldx];
  }
  __syncthreads();
  svd_core(M, a, D, t, V, RM, m, K, V + RM * KC, K_SVD_LEAF, 0.0);
}

__device__ void it_upd_svd_level(const MatDev& M, UpdArgs a_, int bA, int nA, int bB, int nB, int item_, int nitems_, double* smx_) {
  UpdArgs a = a_;
  if (a.kdev) a.k = *a.kdev;
  if (a.k <= 0) return;
  double* sm = smx_;
  const bool rs = (int)item_ < nA;
  const DevSide& D = rs ? M.row : M.col;
  const int t = D.bfs[rs ? bA + item_ : bB + item_ - nA];
  if (D.son0[t] < 0) return;
  const int k = a.k, kt = D.rank[t], K = kt + k;
  double* V = sm;  // RM x KC : V^_t = [R_{t1} E~_{t1}; R_{t2} E~_{t2}]
  int row0 = 0;
  for (int q = 0; q < 2; ++q) {
    const int c = q ? D.son1[t] : D.son0[t];
    const int rc = D.rnew[c], kc = D.rank[c];
    const double* RN = D.rn + (size_t)c * M.kcap * M.kcap;  // rc x (kc + k)
    const double* E = D.tr + (size_t)c * M.rcap * M.rcap;   // kc x kt
    for (int e = threadIdx.x; e < rc * K; e += NT) {
      const int i = e % rc, j = e / rc;
      double v;
      if (j < kt) {
        v = 0.0;
        for (int p = 0; p < kc; ++p) v += RN[i + p * M.kcap] * E[p + j * M.rcap];
      } else {
        v = RN[i + (kc + j - kt) * M.kcap];
      }
      V[row0 + i + j * RM] = v;
    }
    row0 += rc;
  }
  __syncthreads();
  double fv = 0.0;
  for (int q = 0; q < 2; ++q) {
    const int c = q ? D.son1[t] : D.son0[t];
    fv += 2.0 * D.rnew[c] * D.rank[c] * kt;
  }
  svd_core(M, a, D, t, V, RM, row0, K, V + RM * KC, K_SVD_LEVEL, fv);
}

// ---- U5 couplings ------------------------------------------------------------------------------
__device__ void it_upd_couple(const MatDev& M, UpdArgs a_, int nA, int nB, int item_, int nitems_, double* smx_) {
  UpdArgs a = a_;
  if (a.kdev) a.k = *a.kdev;
  if (a.k <= 0) return;
  double* sm = smx_;
  double* T1 = sm;             // KC x KC (ld KC)
  double* Out = T1 + KC * KC;  // KC x KC (ld KC)
  const int k = a.k;
  const bool rs = (int)item_ < nA;
  double fl = 0.0;
  if (rs) {
    const int t = a.t0 + item_;
    const int kt = M.row.rank[t], rt = M.row.rnew[t];
    const double* RNt = M.row.rn + (size_t)t * M.kcap * M.kcap;  // rt x Kt
    for (int q = M.row.bptr[t]; q < M.row.bptr[t + 1]; ++q) {
      const int slot = M.row.bidx[q];
      const int s = M.adm_s[slot];
      double* Sa = M.S + (size_t)slot * M.rcap * M.rcap;  // kt x ls
      const int ls = M.col.rank[s];
      if (inside(M.col, s, a.s0)) {
        const int Ls = ls + k, rsn = M.col.rnew[s];
        const double* RNs = M.col.rn + (size_t)s * M.kcap * M.kcap;  // rsn x Ls
        // T1 = R_t diag(S, I)  (rt x Ls)
        for (int e = threadIdx.x; e < rt * Ls; e += NT) {
          const int i = e % rt, j = e / rt;
          double v;
          if (j < ls) {
            v = 0.0;
            for (int p = 0; p < kt; ++p) v += RNt[i + p * M.kcap] * Sa[p + j * M.rcap];
          } else {
            v = RNt[i + (kt + j - ls) * M.kcap];
          }
          T1[i + j * KC] = v;
        }
        __syncthreads();
        la::cta_gemm(Out, KC, T1, KC, false, RNs, M.kcap, true, rt, rsn, Ls, false);
        __syncthreads();
        la::cta_copy(Sa, M.rcap, Out, KC, rt, rsn);
        fl += 2.0 * rt * kt * ls + 2.0 * rt * Ls * rsn;
      } else {
        // S <- R_t [S; 0] = R_t(:, :kt) S
        la::cta_gemm(Out, KC, RNt, M.kcap, false, Sa, M.rcap, false, rt, ls, kt, false);
        __syncthreads();
        la::cta_copy(Sa, M.rcap, Out, KC, rt, ls);
        fl += 2.0 * rt * kt * ls;
      }
      __syncthreads();
    }
  } else {
    const int s = a.s0 + (item_ - nA);
    const int ls = M.col.rank[s], rsn = M.col.rnew[s];
    const double* RNs = M.col.rn + (size_t)s * M.kcap * M.kcap;  // rsn x (ls + k)
    for (int q = M.col.bptr[s]; q < M.col.bptr[s + 1]; ++q) {
      const int slot = M.col.bidx[q];
      const int t = M.adm_t[slot];
      if (inside(M.row, t, a.t0)) continue;  // handled by the row-side CTA
      double* Sa = M.S + (size_t)slot * M.rcap * M.rcap;
      const int kt = M.row.rank[t];
      // S <- [S, 0] R_s^T = S R_s(:, :ls)^T
      la::cta_gemm(Out, KC, Sa, M.rcap, false, RNs, M.kcap, true, kt, rsn, ls, false);
      __syncthreads();
      la::cta_copy(Sa, M.rcap, Out, KC, kt, rsn);
      fl += 2.0 * kt * ls * rsn;
      __syncthreads();
    }
  }
  if (a.prof && threadIdx.x == 0) atomicAdd(a.prof + 2 * K_COUPLE, fl);
}

// ---- U6 install --------------------------------------------------------------------------------
__device__ void it_upd_install(const MatDev& M, UpdArgs a_, int nA, int nB, int item_, int nitems_, double* smx_) {
  UpdArgs a = a_;
  if (a.kdev) a.k = *a.kdev;
  if (a.k <= 0) return;
  double* sm = smx_;
  const bool rs = (int)item_ < nA;
  const DevSide& D = rs ? M.row : M.col;
  const int root = rs ? a.t0 : a.s0;
  const int t = root + (rs ? item_ : item_ - nA);
  const int r = D.rnew[t];
  const double* qn = D.qn + (size_t)t * M.ldq * M.rcap;
  if (D.son0[t] < 0) {
    const int m = D.hi[t] - D.lo[t];
    double* Vb = D.leafb + (size_t)D.leafidx[t] * M.lmax * M.rcap;
    la::cta_copy(Vb, M.lmax, qn, M.ldq, m, r);
  } else {
    const int c0 = D.son0[t], c1 = D.son1[t];
    const int r0 = D.rnew[c0], r1 = D.rnew[c1];
    la::cta_copy(D.tr + (size_t)c0 * M.rcap * M.rcap, M.rcap, qn, M.ldq, r0, r);
    la::cta_copy(D.tr + (size_t)c1 * M.rcap * M.rcap, M.rcap, qn + r0, M.ldq, r1, r);
  }
  if (t == root && D.parent[t] >= 0) {
    // E_{t0} <- R_{t0} [E_{t0}; 0] = R_{t0}(:, :k_{t0}) E_{t0}
    const int kold = D.rank[t], kp = D.rank[D.parent[t]];
    double* E = D.tr + (size_t)t * M.rcap * M.rcap;
    const double* RN = D.rn + (size_t)t * M.kcap * M.kcap;
    la::cta_gemm(sm, KC, RN, M.kcap, false, E, M.rcap, false, r, kp, kold, false);
    __syncthreads();
    la::cta_copy(E, M.rcap, sm, KC, r, kp);
    if (a.prof && threadIdx.x == 0) atomicAdd(a.prof + 2 * K_INSTALL, 2.0 * r * kold * kp);
  }
  // the new basis is orthonormal: its R-factor is the identity
  double* rc = D.rc + (size_t)t * M.rcap * M.rcap;
  for (int e = threadIdx.x; e < r * r; e += NT) rc[(e % r) + (e / r) * M.rcap] = (e % r) == (e / r) ? 1.0 : 0.0;
  __syncthreads();
  if (threadIdx.x == 0) D.rank[t] = r;
}

// ---- memoised R-factors on pred(t0) ----------------------------------------------------------
__device__ void it_upd_rcache_path(const MatDev& M, UpdArgs a_, int item_, int nitems_, double* smx_) {
  UpdArgs a = a_;
  if (a.kdev) a.k = *a.kdev;
  if (a.k <= 0) return;
  double* sm = smx_;
  const bool rs = item_ == 0;
  const DevSide& D = rs ? M.row : M.col;
  double* A = sm;  // LD2 x KC
  double* diag = A + LD2 * KC;
  double* red = diag + KC;
  for (int t = D.parent[rs ? a.t0 : a.s0]; t >= 0; t = D.parent[t]) {
    const int kt = D.rank[t];
    int row0 = 0;
    for (int q = 0; q < 2; ++q) {
      const int c = q ? D.son1[t] : D.son0[t];
      const int kc = D.rank[c];
      const double* RC = D.rc + (size_t)c * M.rcap * M.rcap;
      const double* E = D.tr + (size_t)c * M.rcap * M.rcap;
      for (int e = threadIdx.x; e < kc * kt; e += NT) {
        const int i = e % kc, j = e / kc;
        double v = 0.0;
        for (int p = i; p < kc; ++p) v += RC[i + p * M.rcap] * E[p + j * M.rcap];
        A[row0 + i + j * LD2] = v;
      }
      row0 += kc;
    }
    __syncthreads();
    if (kt > 0) la::cta_qr_R(A, LD2, row0, kt, diag, red);
    if (a.prof && threadIdx.x == 0) atomicAdd(a.prof + 2 * K_RCACHE, hh_flops(row0, kt) + (double)row0 * row0 * kt);
    double* RC = D.rc + (size_t)t * M.rcap * M.rcap;
    const int mk = row0 < kt ? row0 : kt;
    for (int e = threadIdx.x; e < kt * kt; e += NT) {
      const int i = e % kt, j = e / kt;
      RC[i + j * M.rcap] = i < mk ? A[i + j * LD2] : 0.0;
    }
    __syncthreads();
  }
}

}  // namespace upd
}  // namespace h2
