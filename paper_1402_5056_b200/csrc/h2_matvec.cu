// H^2 matrix-vector product y = alpha op(Z) x + beta y ([BO10 Thm 3.42]).
//
//   forward transform   xhat_s = W_s^T x|s (leaves),  xhat_s = sum_{s'} F_{s'}^T xhat_{s'}   bottom-up
//   couplings           yhat_t = sum_{s in row(t)} S_(t,s) xhat_s                              one warp / cluster
//   backward transform  yhat_{t'} += E_{t'} yhat_t  top-down; leaves y|t = V_t yhat_t
//   nearfield           y|t += sum_{b=(t,s) inadmissible} N_b x|s                            fused in the leaf pass
//
// Bytes are dominated by the nearfield tiles: the leaf pass is written for HBM
// bandwidth (coalesced column reads of the column-major tiles, several loads in flight per lane).
#include <cuda_runtime.h>

#include "h2_internal.h"

namespace h2 {
namespace {

__global__ void k_gather(const double* __restrict__ x, const int64_t* __restrict__ perm, double* __restrict__ xt,
                         int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) xt[i] = x[perm[i]];
}

// One warp per leaf cluster of the source basis: xhat_s = W_s^T x|s.
__global__ void k_fwd_leaf(const int32_t* __restrict__ leaves, int nleaves, const int32_t* __restrict__ lo,
                           const int32_t* __restrict__ hi, const int32_t* __restrict__ leafidx,
                           const int32_t* __restrict__ rank, const double* __restrict__ leafb, int lmax, int rcap,
                           const double* __restrict__ xt, double* __restrict__ xh) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= nleaves) return;
  const int s = leaves[w];
  const int m = hi[s] - lo[s];
  const int k = rank[s];
  const double* Wb = leafb + (size_t)leafidx[s] * lmax * rcap;
  const double x0 = lane < m ? xt[lo[s] + lane] : 0.0;
  const double x1 = lane + 32 < m ? xt[lo[s] + lane + 32] : 0.0;
  double mine = 0.0;
  for (int j = 0; j < k; ++j) {
    double p = 0.0;
    if (lane < m) p = Wb[lane + (size_t)j * lmax] * x0;
    if (lane + 32 < m) p += Wb[lane + 32 + (size_t)j * lmax] * x1;
#pragma unroll
    for (int o = 16; o; o >>= 1) p += __shfl_xor_sync(0xffffffffu, p, o);
    if (lane == (j & 31)) mine = p;
    if ((j & 31) == 31 || j == k - 1) {
      const int base = j & ~31;
      if (base + lane <= j) xh[(size_t)s * rcap + base + lane] = mine;
    }
  }
}

// Internal clusters of one level: xhat_s = F_{s1}^T xhat_{s1} + F_{s2}^T xhat_{s2}; thread per entry.
__global__ void k_fwd_level(const int32_t* __restrict__ list, int count, const int32_t* __restrict__ son0,
                            const int32_t* __restrict__ son1, const int32_t* __restrict__ rank,
                            const double* __restrict__ tr, int rcap, double* __restrict__ xh) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  const int c = idx / rcap, j = idx % rcap;
  if (c >= count) return;
  const int s = list[c];
  if (son0[s] < 0) return;
  if (j >= rank[s]) return;
  double acc = 0.0;
  for (int q = 0; q < 2; ++q) {
    const int sq = q ? son1[s] : son0[s];
    const int kq = rank[sq];
    const double* F = tr + (size_t)sq * rcap * rcap;
    for (int i = 0; i < kq; ++i) acc += F[i + (size_t)j * rcap] * xh[(size_t)sq * rcap + i];
  }
  xh[(size_t)s * rcap + j] = acc;
}

// Couplings: one warp per destination cluster.  Non-transposed: yhat_t = sum S_b xhat_s over row(t).
// Transposed: yhat_s = sum S_b^T xhat_t over col(s).
__global__ void k_couple(int ndst, const int32_t* __restrict__ bptr, const int32_t* __restrict__ bidx,
                         const int32_t* __restrict__ partner, const int32_t* __restrict__ rank_dst,
                         const int32_t* __restrict__ rank_src, const double* __restrict__ S, int rcap, int transpose,
                         const double* __restrict__ xh_src, double* __restrict__ yh_dst) {
  const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= ndst) return;
  const int kt = rank_dst[t];
  for (int i0 = 0; i0 < kt; i0 += 32) {
    const int i = i0 + lane;
    double acc = 0.0;
    for (int q = bptr[t]; q < bptr[t + 1]; ++q) {
      const int a = bidx[q];
      const int s = partner[a];
      const int ks = rank_src[s];
      const double* Sa = S + (size_t)a * rcap * rcap;
      const double* xs = xh_src + (size_t)s * rcap;
      if (i < kt) {
        if (!transpose)
          for (int j = 0; j < ks; ++j) acc += Sa[i + (size_t)j * rcap] * xs[j];
        else
          for (int j = 0; j < ks; ++j) acc += Sa[j + (size_t)i * rcap] * xs[j];
      }
    }
    if (i < kt) yh_dst[(size_t)t * rcap + i] = acc;
  }
}

// Backward transform for one level (L >= 1): yhat_t += E_t yhat_parent; thread per entry.
__global__ void k_bwd_level(const int32_t* __restrict__ list, int count, const int32_t* __restrict__ parent,
                            const int32_t* __restrict__ rank, const double* __restrict__ tr, int rcap,
                            double* __restrict__ yh) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  const int c = idx / rcap, i = idx % rcap;
  if (c >= count) return;
  const int t = list[c];
  const int p = parent[t];
  const int kt = rank[t], kp = rank[p];
  if (i >= kt) return;
  const double* E = tr + (size_t)t * rcap * rcap;
  double acc = yh[(size_t)t * rcap + i];
  for (int j = 0; j < kp; ++j) acc += E[i + (size_t)j * rcap] * yh[(size_t)p * rcap + j];
  yh[(size_t)t * rcap + i] = acc;
}

// Leaf pass, one warp per destination leaf: y|t = V_t yhat_t + sum_b N_b x|s, then scatter to the
// original order with alpha/beta.  Tiles are column-major (lane = row): every column load is coalesced.
__global__ void __launch_bounds__(256) k_leaf_out(
    const int32_t* __restrict__ leaves, int nleaves, const int32_t* __restrict__ lo_d,
    const int32_t* __restrict__ hi_d, const int32_t* __restrict__ leafidx_d, const int32_t* __restrict__ rank_d,
    const double* __restrict__ leafb_d, const int32_t* __restrict__ nptr, const int32_t* __restrict__ nidx,
    const int32_t* __restrict__ npartner, const int32_t* __restrict__ lo_s, const int32_t* __restrict__ hi_s,
    const double* __restrict__ N, int lmax, int rcap, int transpose, const double* __restrict__ yh,
    const double* __restrict__ xt, const int64_t* __restrict__ perm_d, double alpha, double beta,
    double* __restrict__ y, double* __restrict__ prof) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= nleaves) return;
  const int t = leaves[w];
  const int m = hi_d[t] - lo_d[t];
  const int kt = rank_d[t];
  const double* Vb = leafb_d + (size_t)leafidx_d[t] * lmax * rcap;
  const double* yht = yh + (size_t)t * rcap;
  double a0 = 0.0, a1 = 0.0;
  for (int j = 0; j < kt; ++j) {
    const double c = yht[j];
    if (lane < m) a0 += Vb[lane + (size_t)j * lmax] * c;
    if (lane + 32 < m) a1 += Vb[lane + 32 + (size_t)j * lmax] * c;
  }
  for (int q = nptr[t]; q < nptr[t + 1]; ++q) {
    const int a = nidx[q];
    const int s = npartner[a];
    const int ms = hi_s[s] - lo_s[s];
    const double* Na = N + (size_t)a * lmax * lmax;
    const double* xs = xt + lo_s[s];
    if (!transpose) {
      int j = 0;
      for (; j + 4 <= ms; j += 4) {
        const double x0 = xs[j], x1 = xs[j + 1], x2 = xs[j + 2], x3 = xs[j + 3];
        if (lane < m) {
          const double* col = Na + lane + (size_t)j * lmax;
          a0 += col[0] * x0 + col[lmax] * x1 + col[2 * lmax] * x2 + col[3 * lmax] * x3;
        }
        if (lane + 32 < m) {
          const double* col = Na + lane + 32 + (size_t)j * lmax;
          a1 += col[0] * x0 + col[lmax] * x1 + col[2 * lmax] * x2 + col[3 * lmax] * x3;
        }
      }
      for (; j < ms; ++j) {
        const double xj = xs[j];
        if (lane < m) a0 += Na[lane + (size_t)j * lmax] * xj;
        if (lane + 32 < m) a1 += Na[lane + 32 + (size_t)j * lmax] * xj;
      }
    } else {  // y|t += N_a^T x|s : row `lane` of N_a^T is column `lane` of N_a
      for (int i = 0; i < ms; ++i) {
        const double xi = xs[i];
        if (lane < m) a0 += Na[i + (size_t)lane * lmax] * xi;
        if (lane + 32 < m) a1 += Na[i + (size_t)(lane + 32) * lmax] * xi;
      }
    }
  }
  if (prof && lane == 0) {
    // algorithmic bytes: leaf basis m x k_t, every nearfield tile, x|t (read once), y|t written (+read)
    double bytes = 8.0 * ((double)m * kt + m * (beta == 0.0 ? 1 : 2) + m);
    for (int q = nptr[t]; q < nptr[t + 1]; ++q) {
      const int s = npartner[nidx[q]];
      bytes += 8.0 * m * (hi_s[s] - lo_s[s]);
    }
    atomicAdd(prof + 2 * K_MV_LEAF_OUT + 1, bytes);
    atomicAdd(prof + 2 * K_MV_LEAF_OUT, 2.0 * bytes / 8.0);
  }
  if (lane < m) {
    const int64_t o = perm_d[lo_d[t] + lane];
    y[o] = beta == 0.0 ? alpha * a0 : alpha * a0 + beta * y[o];
  }
  if (lane + 32 < m) {
    const int64_t o = perm_d[lo_d[t] + lane + 32];
    y[o] = beta == 0.0 ? alpha * a1 : alpha * a1 + beta * y[o];
  }
}

inline int cdiv(long long a, long long b) { return (int)((a + b - 1) / b); }

}  // namespace

cudaError_t launch_matvec(const h2_mat_* Z, int transpose, double alpha, const double* x, double beta, double* y,
                          cudaStream_t st) {
  const MatDev& M = Z->d;
  const DevSide& src = transpose ? M.row : M.col;  // basis applied to x
  const DevSide& dst = transpose ? M.col : M.row;  // basis producing y
  const h2_tree_* Ts = src.tree;
  const h2_tree_* Td = dst.tree;
  const int64_t n = Ts->n;
  double* prof = prof_dev();
  H2_LAUNCH(K_MV_GATHER, st, k_gather<<<cdiv(n, 256), 256, 0, st>>>(x, src.perm, M.xt, n));
  // forward transform: leaves (all levels), then internal clusters deepest level first
  H2_LAUNCH(K_MV_FWD_LEAF, st,
            k_fwd_leaf<<<cdiv((long long)src.nleaves * 32, 256), 256, 0, st>>>(
                src.leaves, src.nleaves, src.lo, src.hi, src.leafidx, src.rank, src.leafb, M.lmax, M.rcap, M.xt,
                src.xh));
  for (int L = Ts->depth - 1; L >= 0; --L) {
    const int b = Ts->level_ptr[L], e = Ts->level_ptr[L + 1];
    if (e > b)
      H2_LAUNCH(K_MV_FWD_LEVEL, st,
                k_fwd_level<<<cdiv((long long)(e - b) * M.rcap, 256), 256, 0, st>>>(
                    src.bfs + b, e - b, src.son0, src.son1, src.rank, src.tr, M.rcap, src.xh));
  }
  // couplings
  H2_LAUNCH(K_MV_COUPLE, st,
            k_couple<<<cdiv((long long)Td->nclusters * 32, 256), 256, 0, st>>>(
                Td->nclusters, dst.bptr, dst.bidx, transpose ? M.adm_t : M.adm_s, dst.rank, src.rank, M.S, M.rcap,
                transpose, src.xh, dst.xh));
  // backward transform
  for (int L = 1; L <= Td->depth; ++L) {
    const int b = Td->level_ptr[L], e = Td->level_ptr[L + 1];
    if (e > b)
      H2_LAUNCH(K_MV_BWD_LEVEL, st,
                k_bwd_level<<<cdiv((long long)(e - b) * M.rcap, 256), 256, 0, st>>>(
                    dst.bfs + b, e - b, dst.parent, dst.rank, dst.tr, M.rcap, dst.xh));
  }
  // leaves + nearfield + scatter
  const int32_t* np = transpose ? M.ntptr : M.nptr;
  const int32_t* ni = transpose ? M.ntidx : M.nidx;
  const int32_t* npart = transpose ? M.in_t : M.in_s;
  H2_LAUNCH(K_MV_LEAF_OUT, st,
            k_leaf_out<<<cdiv((long long)dst.nleaves * 32, 256), 256, 0, st>>>(
                dst.leaves, dst.nleaves, dst.lo, dst.hi, dst.leafidx, dst.rank, dst.leafb, np, ni, npart, src.lo,
                src.hi, M.N, M.lmax, M.rcap, transpose, dst.xh, M.xt, dst.perm, alpha, beta, y, prof));
  return cudaGetLastError();
}

}  // namespace h2
