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

__device__ double weights_cluster(const MatDev& M, const UpdArgs& a, bool rs, int t, double* sm, int mode,
                                  const double* bp_sm = nullptr, int ldbp = 0, const int* fpc = nullptr,
                                  const int* fpk = nullptr, int fL = 0);

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
  if (b == 0 && threadIdx.x == 0 && nrl + ncl > 0) {
    const int idx = atomicAdd(M.flags + 3, 1);  // non-zero-rank update count
    if (M.updlog && idx < (1 << 20)) {
      M.updlog[5 * idx] = a.t0;
      M.updlog[5 * idx + 1] = a.s0;
      M.updlog[5 * idx + 2] = a.k;
      M.updlog[5 * idx + 3] = M.row.rank[a.t0];  // ranks before the update
      M.updlog[5 * idx + 4] = M.col.rank[a.s0];
    }
  }
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
enum { W_FULL = 0, W_LOCAL = 1, W_CHAIN = 2, W_FLAT = 3 };

__device__ double weights_cluster(const MatDev& M, const UpdArgs& a, bool rs, int t, double* sm, int mode,
                                  const double* bp_sm, int ldbp, const int* fpc, const int* fpk, int fL) {
  const DevSide& A = rs ? M.row : M.col;
  const DevSide& B = rs ? M.col : M.row;
  const int a0 = rs ? a.t0 : a.s0, b0 = rs ? a.s0 : a.t0;
  const int k = a.k;
  // independent structure loads first (one memory round trip instead of one per block)
  const int kt = A.rank[t];
  const int p = A.parent[t];
  const int asz = A.tsize[a0], bsz = B.tsize[b0];
  const int qb = mode == W_CHAIN ? 0 : A.bptr[t], qe = mode == W_CHAIN ? 0 : A.bptr[t + 1];
  const int kp = (p >= 0 && mode != W_LOCAL && mode != W_FLAT) ? A.rank[p] : 0;
  const bool in_t = t >= a0 && t < a0 + asz;
  const int K = kt + (in_t ? k : 0);
  double* P = sm;                 // PR x KC panel
  double* diag = P + PRL * KC;
  double* red = diag + KC;
  // block descriptors of one batch of the block row (shared memory, after the panel)
  constexpr int NBD = 128;
  int* d_slot = reinterpret_cast<int*>(red + 8);
  int* d_s = d_slot + NBD;
  int* d_ls = d_s + NBD;
  int* d_rc = d_ls + NBD;
  int* d_off = d_rc + NBD;
  int* rowblk = d_off + NBD;      // PR: panel row -> descriptor
  double* d_nrm = reinterpret_cast<double*>(rowblk + PR);  // NBD: ||G~_b||_F (blockwise weighting)
  // blockwise (reading own-10): R-factor of this cluster's own (extended) basis
  const double* RVo = in_t ? A.re + (size_t)t * M.kcap * M.kcap : A.rc + (size_t)t * M.rcap * M.rcap;
  const int ldRV = in_t ? M.kcap : M.rcap;
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
  // local stack: R_{W,s} S~_b^T for the blocks b = (t, s) of row(t), in block order, flushed
  // (QR -> its R-factor) before a block that does not fit the panel -- the same flush points and
  // sums as one block at a time, but every block of a segment is filled in one parallel pass
  for (int base = qb; base < qe; base += NBD) {
    const int cnt = qe - base < NBD ? qe - base : NBD;
    for (int j = threadIdx.x; j < cnt; j += NT) {
      const int slot = A.bidx[base + j];
      const int s = rs ? M.adm_s[slot] : M.adm_t[slot];
      const bool in_s = s >= b0 && s < b0 + bsz;
      const int ls = B.rank[s];
      d_slot[j] = slot;
      d_s[j] = s;
      d_ls[j] = ls;
      d_rc[j] = in_s ? ls + k : ls;  // k > 0: in_s <=> rc > ls
    }
    __syncthreads();
    int j = 0;
    while (j < cnt) {
      // the segment [j, je): blocks that fit after `rows` (identical walk on every thread)
      int je = j, r = rows;
      while (je < cnt && (d_rc[je] == 0 || r + d_rc[je] <= PR)) {
        if (threadIdx.x == 0) {
          d_off[je] = r;
          fl += (double)d_rc[je] * d_ls[je] * kt;  // triangular R_B times S^T
        }
        r += d_rc[je];
        ++je;
      }
      __syncthreads();  // d_off
      for (int b = j + (int)threadIdx.x; b < je; b += NT)
        for (int i = 0; i < d_rc[b]; ++i) rowblk[d_off[b] + i] = b;
      __syncthreads();
      const int nr = r - rows;
      for (int e = threadIdx.x; e < nr * K; e += NT) {
        const int rr = rows + e % nr, c = e / nr;
        const int b = rowblk[rr];
        const int i = rr - d_off[b];
        const int ls = d_ls[b], s = d_s[b];
        const bool in_s = d_rc[b] > ls;
        const double* Sa = M.S + (size_t)d_slot[b] * M.rcap * M.rcap;
        const double* RB = in_s ? B.re + (size_t)s * M.kcap * M.kcap : B.rc + (size_t)s * M.rcap * M.rcap;
        const int ldR = in_s ? M.kcap : M.rcap;
        double v = 0.0;
        if (c < kt) {
          // (R_B S~^T)(i,c) = sum_j R_B(i,j) S_or(c,j),   S_or = S (row side) or S^T (column side)
          for (int jj = i; jj < ls; ++jj) v += RB[i + jj * ldR] * (rs ? Sa[c + jj * M.rcap] : Sa[jj + c * M.rcap]);
        } else if (in_s) {
          v = RB[i + (ls + c - kt) * ldR];  // identity block of S~ = diag(S, I)
        }
        P[rr + c * PRL] = v;
      }
      __syncthreads();
      if (a.blockwise) {
        // every block's rows carry the weight 1 / ||G~_b||_F,  G~_b^T = (R_B S~^T) R_V^T
        // (d_rc[b] x K; R_V upper triangular).  One warp per block, fixed summation order.
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        for (int b = j + warp; b < je; b += NT / 32) {
          const int nrb = d_rc[b], ob = d_off[b];
          double sq = 0.0;
          for (int e = lane; e < nrb * K; e += 32) {
            const int i = e % nrb, cp = e / nrb;
            double g = 0.0;
            for (int c = cp; c < K; ++c) g += P[ob + i + c * PRL] * RVo[cp + (size_t)c * ldRV];
            sq += g * g;
          }
          for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
          if (lane == 0) d_nrm[b] = sqrt(sq);
        }
        fl += (double)nr * K * K;
        __syncthreads();
        for (int e = threadIdx.x; e < nr * K; e += NT) {
          const int rr = rows + e % nr, c = e / nr;
          const double nb = d_nrm[rowblk[rr]];
          P[rr + c * PRL] = nb > 0.0 ? P[rr + c * PRL] / nb : 0.0;  // a zero block adds nothing
        }
        __syncthreads();
      }
      rows = r;
      j = je;
      if (j < cnt) flush();  // block j does not fit: compress first
    }
  }
  if (mode == W_FLAT) {
    // the ancestors' local stacks, each carried down to t by its transfer chain:
    // rows C_a G_a^T (G_a = E_t E_{t+} ... : k_t x k_a in bw[a], C_a in re[a]), zero on the k
    // extension columns (E~_{t0} = [E_{t0}; 0]); same R-factor as the level-by-level chain
    // B~_t = R([C_t; B~_{t+} E~_t^T]) (left orthogonal factors drop out), one QR instead of one per level
    int l = fL - 1;
    while (l >= 0) {
      int r = rows, le = l;
      while (le >= 0 && r + fpk[le] <= PR) r += fpk[le--];
      if (le == l) {  // the next block does not fit: compress first
        flush();
        continue;
      }
      const int nr = r - rows;
      for (int e = threadIdx.x; e < nr * K; e += NT) {
        const int rr = e % nr, c = e / nr;
        int b = l, off = 0;
        while (rr >= off + fpk[b]) off += fpk[b--];
        const int i = rr - off, kb = fpk[b];
        double v = 0.0;
        if (c < kt) {
          const double* C = A.re + (size_t)fpc[b] * M.kcap * M.kcap;
          const double* G = A.bw + (size_t)fpc[b] * M.kcap * M.kcap;
          for (int j = 0; j < kb; ++j) v += C[i + j * M.kcap] * G[c + j * M.kcap];
          fl += 2.0 * kb;
        }
        P[rows + rr + c * PRL] = v;
      }
      __syncthreads();
      rows = r;
      l = le;
    }
  }
  if (kp >= 0 && p >= 0 && mode != W_LOCAL && mode != W_FLAT) {
    const bool in_p = p >= a0 && p < a0 + asz;
    const int Kp = kp + (in_p ? k : 0);
    if (Kp > 0) {
      if (rows + Kp > PR) flush();
      // B~_{t+}: from global, or from shared memory when the caller chained it there
      const double* Bp = bp_sm ? bp_sm : A.bw + (size_t)p * M.kcap * M.kcap;
      const int ldb = bp_sm ? ldbp : M.kcap;
      const double* E = A.tr + (size_t)t * M.rcap * M.rcap;  // kt x kp
      for (int e = threadIdx.x; e < Kp * K; e += NT) {
        const int i = e % Kp, c = e / Kp;
        double v = 0.0;
        if (c < kt) {
          for (int j = 0; j < kp; ++j) v += Bp[i + j * ldb] * E[c + j * M.rcap];
        } else if (in_p) {
          v = Bp[i + (kp + c - kt) * ldb];  // E~_t = diag(E_t, I) inside T_{t0}
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

// cp.async (8-byte) global -> shared copies: the operands of the next chain level load while the
// current level computes
__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// U3 along pred(t0): B~_{t0} = R([local stack of t0; B~_{t0+} E~_{t0}^T]) with
// B~_t = R([C_t; B~_{t+} E_t^T]) down the path (C_t = R-factor of t's local stack, computed in
// parallel by the ext_leaf op into re[t]).  Unrolled, B~_{t0} is the R-factor of the local stack of
// t0 stacked over C_a G_a^T for every proper ancestor a, G_a = E_{t0} E_{t0+} ... (the transfer chain
// from t0 up to a): the same matrix up to left orthogonal factors, hence the same R-factor (rows up
// to sign), with ONE QR instead of one QR per level.  The path comes from the leaf-ancestor table,
// the ranks and the path's transfer matrices are loaded in one round each.
__device__ void it_upd_weights_path(const MatDev& M, UpdArgs a_, int l0r, int l0c, int Lr, int Lc, int item_,
                                    double* smx_) {
  UpdArgs a = a_;
  if (a.kdev) a.k = *a.kdev;
  if (a.k <= 0) return;
  const bool rs = item_ == 0;
  const DevSide& A = rs ? M.row : M.col;
  const int L = rs ? Lr : Lc;                  // level of t0: path = anc[0..L]
  const int32_t* anc = A.anc + (size_t)(rs ? l0r : l0c) * A.ancw;
  constexpr int RC = RCAP_MAX, LB = RC + 1;
  // shared memory: [weights panel + descriptors | 1024 spare | G ping-pong (2 LB x RC) | path ints]
  constexpr int GOFF = (PR + 1) * KC + KC + 8 + 1024;
  int* pc = reinterpret_cast<int*>(smx_ + GOFF + 2 * LB * RC);  // path clusters (64)
  int* pk = pc + 64;                                             // their ranks (64)
  for (int l = threadIdx.x; l <= L; l += NT) pc[l] = anc[l];
  __syncthreads();
  for (int l = threadIdx.x; l <= L; l += NT) pk[l] = A.rank[pc[l]];
  __syncthreads();
  double fl = 0.0;
  // transfer chains G_l = E_{t0} E_{a_{L-1}} ... E_{a_{l+1}} (k_{t0} x k_l) for the proper ancestors
  // a_l, bottom-up, into bw[a_l] (free: a proper ancestor's B~ is not needed, see W_FLAT); the E
  // matrices of the whole path are staged in shared memory in one load round first
  if (L > 0) {
    double* stage = smx_;                       // (the weights panel, not used yet)
    double* Gb[2] = {smx_ + GOFF, smx_ + GOFF + LB * RC};
    int* eo = pk + 64;                           // staging offset of E_{a_l}, l = 1..L
    if (threadIdx.x == 0) {
      int o = 0;
      for (int l = 1; l <= L; ++l) {
        eo[l] = o;
        o += pk[l] * pk[l - 1];
      }
      eo[0] = o;  // total
    }
    __syncthreads();
    const bool staged = eo[0] <= (PR + 1) * KC;
    if (staged) {
      for (int l = 1; l <= L; ++l) {
        const int kl = pk[l], kq = pk[l - 1];
        const double* E = A.tr + (size_t)pc[l] * M.rcap * M.rcap;
        for (int e = threadIdx.x; e < kl * kq; e += NT) stage[eo[l] + e] = E[(e % kl) + (e / kl) * M.rcap];
      }
      __syncthreads();
    }
    auto Eel = [&](int l, int i, int j) -> double {  // E_{a_l}(i, j)
      return staged ? stage[eo[l] + i + j * pk[l]] : A.tr[(size_t)pc[l] * M.rcap * M.rcap + i + j * M.rcap];
    };
    const int kt0 = pk[L];
    int cur = 0;
    for (int l = L - 1; l >= 0; --l) {
      const int kl = pk[l], kn = pk[l + 1];
      double* Gn = Gb[cur];
      double* Gg = A.bw + (size_t)pc[l] * M.kcap * M.kcap;
      for (int e = threadIdx.x; e < kt0 * kl; e += NT) {
        const int i = e % kt0, j = e / kt0;
        double v;
        if (l == L - 1) {
          v = Eel(L, i, j);  // G_{L-1} = E_{t0}
        } else {
          v = 0.0;
          for (int q = 0; q < kn; ++q) v += Gb[cur ^ 1][i + q * LB] * Eel(l + 1, q, j);
        }
        Gn[i + j * LB] = v;
        Gg[i + j * M.kcap] = v;
      }
      fl += 2.0 * kt0 * kn * kl;
      cur ^= 1;
      __syncthreads();
    }
  }
  // t0: its full local stack + every ancestor's local stack carried down (one TSQR)
  fl += weights_cluster(M, a, rs, pc[L], smx_, W_FLAT, nullptr, 0, pc, pk, L);
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
                         int K, double* sm_rest, int kid, double extra_flops, const double* RV = nullptr) {
  // RV (leaves): R-factor of V itself (V = Q_V R_V, computed by the extension op, ld kcap): then
  // M = Q_V (R_V B~^T) and N = R_V B~^T (min(m,K) x K, a product of two triangles) replaces the
  // Householder QR of M on the K <= 32 path -- the same singular values and right singular vectors
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
  const int path = (K <= m && m <= 16) ? 0 : (K <= 32 ? 1 : 2);  // profiling: which SVD variant
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
    const int pr = m < K ? m : K;
    if (RV) {
      // N^T = B~ R_V^T (K x pr): N^T(i, j) = sum_q R_V(j, q) B~(i, q), both upper triangular
      for (int e = threadIdx.x; e < K * pr; e += NT) {
        const int i = e % K, j = e / K;
        double v = 0.0;
        for (int q = (i > j ? i : j); q < K; ++q) v += RV[j + (size_t)q * M.kcap] * Bt[i + q * RM];
        W[i + j * RM] = v;
      }
      __syncthreads();
    } else {
      la::cta_copy(Rw, RM, Mm, RM, m, K);
      __syncthreads();
      la::cta_qr_R(Rw, RM, m, K, sig, (double*)order);
      for (int e = threadIdx.x; e < K * pr; e += NT) {  // R^T (K x pr) into W's slot as the input
        const int i = e % K, j = e / K;
        W[i + j * RM] = j <= i ? Rw[j + i * RM] : 0.0;
      }
      __syncthreads();
    }
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
  // blockwise: an absolute threshold eps^ = rel_tol on the block-relative weighted matrix
  const int r = a.blockwise
                    ? la::trunc_rank(sig, order, p, 0.0, fmax(a.rel_tol, a.abs_tol), a.max_rank, M.rcap, &clamped)
                    : la::trunc_rank(sig, order, p, a.rel_tol, a.abs_tol, a.max_rank, M.rcap, &clamped);
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
      atomicAdd(dbg + 7 + path, 1.0);                        // calls per variant
      atomicAdd(dbg + 10 + path, (double)(clock64() - c0));  // cycles per variant
      if (kid == K_SVD_LEAF) atomicAdd(dbg + 13, 1.0);
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
  svd_core(M, a, D, t, V, RM, m, K, V + RM * KC, K_SVD_LEAF, 0.0, D.re + (size_t)t * M.kcap * M.kcap);
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
__device__ __forceinline__ int seg_find(const int* cum, int nb, int e) {  // last b with cum[b] <= e
  int lo = 0, hi = nb - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (cum[mid] <= e) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// U5: every admissible block of row(t), t in T_{t0}, gets S <- R_t S~ R_s^T (s in
// T_{s0}) or R_t [S; 0]; every block of col(s), s in T_{s0}, with its row outside T_{t0} gets
// [S, 0] R_s^T.  The blocks of one cluster are independent: their descriptors are loaded at once and
// all blocks of a segment (as many as fit the shared-memory budget) are multiplied in the same
// parallel passes -- the same sums, in the same order, as one block at a time.
__device__ void it_upd_couple(const MatDev& M, UpdArgs a_, int nA, int nB, int item_, int nitems_, double* smx_) {
  UpdArgs a = a_;
  if (a.kdev) a.k = *a.kdev;
  if (a.k <= 0) return;
  const int k = a.k;
  const bool rs = (int)item_ < nA;
  constexpr int NBD = 128;
  constexpr int BUDGET = 24000;  // doubles of per-block scratch per segment
  double* buf = smx_;
  int* d_slot = reinterpret_cast<int*>(smx_ + BUDGET);
  int* d_p = d_slot + NBD;    // partner cluster
  int* d_kp = d_p + NBD;      // partner's old rank (l_s, or k_t on the column side)
  int* d_rn = d_kp + NBD;     // partner's new rank (in_s only), -1: partner outside (no column change)
  int* d_t1 = d_rn + NBD;     // scratch offset of T1 (in_s) / -1
  int* d_out = d_t1 + NBD;    // scratch offset of Out
  int* cumA = d_out + NBD;    // cumulative T1 entries
  int* cumB = cumA + NBD;     // cumulative Out entries
  int* sc = cumB + NBD;       // [0]: segment end, [1]: T1 total, [2]: Out total
  double fl = 0.0;
  const DevSide& Dm = rs ? M.row : M.col;
  const int c = rs ? a.t0 + item_ : a.s0 + (item_ - nA);  // this item's cluster
  const int kc = Dm.rank[c], rcn = Dm.rnew[c];
  const double* RNc = Dm.rn + (size_t)c * M.kcap * M.kcap;  // rcn x (kc + k)
  const int qb = Dm.bptr[c], qe = Dm.bptr[c + 1];
  const int osz = rs ? M.col.tsize[a.s0] : M.row.tsize[a.t0];
  for (int base = qb; base < qe; base += NBD) {
    const int cnt = qe - base < NBD ? qe - base : NBD;
    for (int j = threadIdx.x; j < cnt; j += NT) {
      const int slot = Dm.bidx[base + j];
      const int p = rs ? M.adm_s[slot] : M.adm_t[slot];
      const bool in_o = rs ? (p >= a.s0 && p < a.s0 + osz) : (p >= a.t0 && p < a.t0 + osz);
      d_slot[j] = slot;
      d_p[j] = p;
      d_kp[j] = rs ? M.col.rank[p] : M.row.rank[p];
      d_rn[j] = rs ? (in_o ? M.col.rnew[p] : -1) : (in_o ? -2 : -1);  // column side: -2 = handled by the row CTA
    }
    __syncthreads();
    int j = 0;
    while (j < cnt) {
      if (threadIdx.x == 0) {  // pack a segment of blocks into the scratch budget
        int used = 0, je = j, na = 0, nbo = 0;
        for (; je < cnt; ++je) {
          const int kp = d_kp[je], rn = d_rn[je];
          int t1 = 0, ou = 0;
          if (rs) {
            if (rn >= 0) {
              t1 = rcn * (kp + k);
              ou = rcn * rn;
            } else {
              ou = rcn * kp;
            }
          } else if (rn == -1) {
            ou = kp * rcn;
          }
          if (used + t1 + ou > BUDGET && je > j) break;
          cumA[je - j] = na;
          cumB[je - j] = nbo;
          d_t1[je] = t1 ? used : -1;
          d_out[je] = used + t1;
          used += t1 + ou;
          na += t1;
          nbo += ou;
        }
        sc[0] = je;
        sc[1] = na;
        sc[2] = nbo;
      }
      __syncthreads();
      const int je = sc[0], na = sc[1], nbo = sc[2], nb = je - j;
      // pass A (row side, partner inside T_{s0}): T1 = R_t diag(S, I)  (rt x (l_s + k), ld rt)
      for (int e = threadIdx.x; e < na; e += NT) {
        const int b = j + seg_find(cumA, nb, e);
        const int x = e - cumA[b - j];
        const int ls = d_kp[b], i = x % rcn, jj = x / rcn;
        const double* Sa = M.S + (size_t)d_slot[b] * M.rcap * M.rcap;
        double v;
        if (jj < ls) {
          v = 0.0;
          for (int p = 0; p < kc; ++p) v += RNc[i + p * M.kcap] * Sa[p + jj * M.rcap];
        } else {
          v = RNc[i + (kc + jj - ls) * M.kcap];
        }
        buf[d_t1[b] + x] = v;
      }
      __syncthreads();
      // pass B: the new couplings into the scratch
      for (int e = threadIdx.x; e < nbo; e += NT) {
        const int b = j + seg_find(cumB, nb, e);
        const int x = e - cumB[b - j];
        const double* Sa = M.S + (size_t)d_slot[b] * M.rcap * M.rcap;
        const int kp = d_kp[b], rn = d_rn[b];
        double acc = 0.0;
        if (rs && rn >= 0) {  // T1 R_s^T  (rt x rsn), inner l_s + k
          const double* RNs = M.col.rn + (size_t)d_p[b] * M.kcap * M.kcap;
          const double* T1 = buf + d_t1[b];
          const int i = x % rcn, jj = x / rcn, Ls = kp + k;
          for (int q = 0; q < Ls; ++q) acc += T1[i + q * rcn] * RNs[jj + q * M.kcap];
        } else if (rs) {  // R_t(:, :kt) S  (rt x ls), inner kt
          const int i = x % rcn, jj = x / rcn;
          for (int q = 0; q < kc; ++q) acc += RNc[i + q * M.kcap] * Sa[q + jj * M.rcap];
        } else {  // S R_s(:, :ls)^T  (kt x rsn), inner ls
          const int i = x % kp, jj = x / kp;
          for (int q = 0; q < kc; ++q) acc += Sa[i + q * M.rcap] * RNc[jj + q * M.kcap];
        }
        buf[d_out[b] + x] = acc;
      }
      __syncthreads();
      // pass C: write back (every read of the old couplings is done)
      for (int e = threadIdx.x; e < nbo; e += NT) {
        const int b = j + seg_find(cumB, nb, e);
        const int x = e - cumB[b - j];
        double* Sa = M.S + (size_t)d_slot[b] * M.rcap * M.rcap;
        const int rows = rs ? rcn : d_kp[b];
        Sa[(x % rows) + (x / rows) * M.rcap] = buf[d_out[b] + x];
      }
      if (threadIdx.x == 0 && a.prof) {
        for (int b = j; b < je; ++b) {
          const int kp = d_kp[b], rn = d_rn[b];
          if (rs && rn >= 0) fl += 2.0 * rcn * kc * kp + 2.0 * rcn * (kp + k) * rn;
          else if (rs) fl += 2.0 * rcn * kc * kp;
          else if (rn == -1) fl += 2.0 * kp * kc * rcn;
        }
      }
      __syncthreads();
      j = je;
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
// rc[a] = R-factor of the nested basis V_a (Alg. 16 recursion, reading R7) for every proper ancestor
// a = a_l of t0 (path a_0 = root ... a_L = t0, s_j = the sibling of a_j).  Unrolled down the path:
//   V_a ~ [ rc[a_L] E_{a_L} T_L ; rc[s_L] E_{s_L} T_L ; ... ; rc[s_{l+1}] E_{s_{l+1}} T_{l+1} ]
// (up to left orthogonal factors), T_{l+1} = I, T_{j+1} = E_{a_j} T_j the transfer chain from a_j up
// to a.  So every ancestor is one independent item -- a chain of small products and ONE QR --
// instead of a sequential chain of QRs from the father of t0 to the root.
__device__ void it_upd_rcache_path(const MatDev& M, UpdArgs a_, int l0r, int l0c, int Lr, int Lc, int item_,
                                   double* smx_) {
  UpdArgs a = a_;
  if (a.kdev) a.k = *a.kdev;
  if (a.k <= 0) return;
  const bool rs = item_ < Lr;
  const DevSide& D = rs ? M.row : M.col;
  const int L = rs ? Lr : Lc;
  const int l = rs ? item_ : item_ - Lr;  // this item's ancestor level
  const int32_t* anc = D.anc + (size_t)(rs ? l0r : l0c) * D.ancw;
  constexpr int RC = RCAP_MAX, LB = RC + 1;
  double* P = smx_;                        // panel (PR x RC, ld PRL)
  double* diag = P + PRL * RC;
  double* T[2] = {diag + KC, diag + KC + LB * RC};  // transfer chain ping-pong (k_j x k_l)
  double* U = T[1] + LB * RC;              // E_s T (k_s x k_l)
  int* pc = reinterpret_cast<int*>(U + LB * RC);  // path a_0..a_L
  int* pk = pc + 64;                       // ranks
  int* ps = pk + 64;                       // sibling s_j of a_j (j >= 1)
  int* psk = ps + 64;                      // its rank
  for (int j = threadIdx.x; j <= L; j += NT) pc[j] = anc[j];
  __syncthreads();
  for (int j = threadIdx.x; j <= L; j += NT) {
    pk[j] = D.rank[pc[j]];
    if (j > 0) {
      const int par = pc[j - 1];
      const int s0 = D.son0[par], s1 = D.son1[par];
      ps[j] = s0 == pc[j] ? s1 : s0;
    }
  }
  __syncthreads();
  for (int j = threadIdx.x + 1; j <= L; j += NT) psk[j] = D.rank[ps[j]];
  __syncthreads();
  const int kl = pk[l];
  int rows = 0;
  double fl = 0.0;
  // T_{l+1} = I (k_l x k_l)
  for (int e = threadIdx.x; e < kl * kl; e += NT) T[0][(e % kl) + (e / kl) * LB] = (e % kl) == (e / kl) ? 1.0 : 0.0;
  __syncthreads();
  int cur = 0;
  auto append = [&](const double* R, int kr, const double* E, int kp) {
    // rows rc (kr x kr, upper triangular, ld rcap) * E (kr x kp, ld rcap) * T (kp x kl)
    if (kr == 0 || kl == 0) return;
    for (int e = threadIdx.x; e < kr * kl; e += NT) {  // U = E T
      const int i = e % kr, c = e / kr;
      double v = 0.0;
      for (int q = 0; q < kp; ++q) v += E[i + q * M.rcap] * T[cur][q + c * LB];
      U[i + c * LB] = v;
    }
    __syncthreads();
    if (rows + kr > PR) {
      la::cta_qr_R(P, PRL, rows, kl, diag, diag);
      fl += hh_flops(rows, kl);
      rows = rows < kl ? rows : kl;
    }
    for (int e = threadIdx.x; e < kr * kl; e += NT) {  // rows rc U
      const int i = e % kr, c = e / kr;
      double v = 0.0;
      for (int q = i; q < kr; ++q) v += R[i + q * M.rcap] * U[q + c * LB];
      P[rows + i + c * PRL] = v;
    }
    fl += 2.0 * kr * kp * kl + (double)kr * kr * kl;
    rows += kr;
    __syncthreads();
  };
  for (int j = l + 1; j <= L; ++j) {
    // the sibling of a_j, carried up to a_l
    append(D.rc + (size_t)ps[j] * M.rcap * M.rcap, psk[j], D.tr + (size_t)ps[j] * M.rcap * M.rcap, pk[j - 1]);
    if (j == L) {  // t0 itself (its R was installed by the previous op)
      append(D.rc + (size_t)pc[L] * M.rcap * M.rcap, pk[L], D.tr + (size_t)pc[L] * M.rcap * M.rcap, pk[L - 1]);
    } else {       // T_{j+1} = E_{a_j} T_j  (k_j x k_l)
      const int kj = pk[j], kq = pk[j - 1];
      const double* E = D.tr + (size_t)pc[j] * M.rcap * M.rcap;
      for (int e = threadIdx.x; e < kj * kl; e += NT) {
        const int i = e % kj, c = e / kj;
        double v = 0.0;
        for (int q = 0; q < kq; ++q) v += E[i + q * M.rcap] * T[cur][q + c * LB];
        T[cur ^ 1][i + c * LB] = v;
      }
      fl += 2.0 * kj * kq * kl;
      cur ^= 1;
      __syncthreads();
    }
  }
  if (rows > 0 && kl > 0) {
    la::cta_qr_R(P, PRL, rows, kl, diag, diag);
    fl += hh_flops(rows, kl);
  }
  double* RCg = D.rc + (size_t)pc[l] * M.rcap * M.rcap;
  const int mk = rows < kl ? rows : kl;
  for (int e = threadIdx.x; e < kl * kl; e += NT) {
    const int i = e % kl, j = e / kl;
    RCg[i + j * M.rcap] = i < mk ? P[i + j * PRL] : 0.0;
  }
  if (a.prof && threadIdx.x == 0) atomicAdd(a.prof + 2 * K_RCACHE, fl);
}

}  // namespace upd
}  // namespace h2
