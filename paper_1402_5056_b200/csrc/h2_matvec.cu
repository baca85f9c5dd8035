// H^2 matrix-vector product y = alpha op(Z) x + beta y ([BO10 Thm 3.42]).
//
//   forward transform   xhat_s = W_s^T x|s (leaves),  xhat_s = sum_{s'} F_{s'}^T xhat_{s'}   bottom-up
//   couplings           yhat_t = sum_{s in row(t)} S_(t,s) xhat_s
//   backward transform  yhat_{t'} += E_{t'} yhat_t  top-down; leaves y|t = V_t yhat_t
//   nearfield           y|t += sum_{b=(t,s) inadmissible} N_b x|s
//
// Four launches on two streams (nearfield || forward transform + couplings, then the walk), no
// grid-wide barrier, no spin-waits; a matrix whose bases all have rank 0 launches the nearfield only:
//   k_matvec_near  warp per destination leaf: y|t = alpha sum_b N_b x|s + beta y|t (streams the
//                  tiles, the bulk of the bytes) -- on a second stream, concurrently with:
//   k_matvec_fwd   warp per source leaf: forward transform, then climb: the second of two siblings
//                  to finish (arrival counter) computes the father, up to the root.  No waits.
//   k_matvec_couple  warp per destination cluster: yc_t = sum_b S_b xhat_s.
//   k_matvec_walk    warp per destination leaf: yhat along its ancestor path, root first
//                    (yhat_c = yc_c + E_c yhat_father), then y|t += alpha V_t yhat_t; the path
//                    prefix shared by a block's 8 leaves is walked once (shared memory).  No
//                    level-by-level chain of launches or flags.
// The arrival counters are reset by their last user.  Bytes are dominated by the nearfield tiles
// (SURVEY §8(d)): lanes own rows, a 32-column panel is 32 coalesced 256 B streaming loads in flight.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <unordered_map>

#include "h2_internal.h"

namespace h2 {
namespace {

struct MvArgs {
  // source side (the basis applied to x)
  const int32_t *s_leaves, *s_lo, *s_hi, *s_leafidx, *s_rank, *s_parent, *s_son0, *s_son1;
  const int64_t* s_perm;
  const double *s_leafb, *s_tr;
  double* s_xh;
  int32_t* s_arrive;
  int s_nleaves;
  // destination side (the basis producing y)
  const int32_t *d_bfs, *d_leaves, *d_lo, *d_hi, *d_leafidx, *d_rank, *d_parent, *d_son0, *d_bptr, *d_bidx;
  const int64_t* d_perm;
  const double *d_leafb, *d_tr;
  double* d_xh;
  const int32_t* d_anc;
  int d_ancw;
  int d_nclusters, d_nleaves;
  // blocks
  const int32_t* partner;  // admissible slot -> source cluster
  const double* S;
  const int32_t *nptr, *nidx, *npartner;
  const double* N;
  int lmax, rcap, transpose;
  const double* x;
  double* y;
  double alpha, beta;
  int* sync;  // fused kernel: [0] forward done, [1] warps done with the couplings, [2] blocks exited
  // subtree schedule (DevSide::mv_*): source side (forward) and destination side (backward)
  const int32_t *s_roots, *s_top, *s_top_lptr, *s_tsize, *s_level;
  int s_top_nlev;
  int32_t* s_cnt;
  const int32_t *d_roots, *d_top, *d_top_lptr, *d_tsize, *d_level, *d_son1;
  int d_top_nlev;
  int32_t* d_cnt;
};

constexpr unsigned FULL = 0xffffffffu;

// ---- forward transform of one source leaf, then the climb ---------------------------------------
__device__ void mv_up(const MvArgs& a, int s, int lane) {
  const int rcap = a.rcap, lmax = a.lmax;
  {
    const int lo = a.s_lo[s], m = a.s_hi[s] - lo, k = a.s_rank[s];
    if (k > 0) {
      const double x0 = lane < m ? a.x[a.s_perm[lo + lane]] : 0.0;
      const double x1 = lane + 32 < m ? a.x[a.s_perm[lo + lane + 32]] : 0.0;
      const double* W = a.s_leafb + (size_t)a.s_leafidx[s] * lmax * rcap;
      double mine0 = 0.0, mine1 = 0.0;
      for (int j = 0; j < k; ++j) {
        double p = 0.0;
        if (lane < m) p = W[lane + (size_t)j * lmax] * x0;
        if (lane + 32 < m) p += W[lane + 32 + (size_t)j * lmax] * x1;
#pragma unroll
        for (int o = 16; o; o >>= 1) p += __shfl_xor_sync(FULL, p, o);
        if (lane == (j & 31)) {
          if (j < 32) mine0 = p;
          else mine1 = p;
        }
      }
      if (lane < k) a.s_xh[(size_t)s * rcap + lane] = mine0;
      if (lane + 32 < k) a.s_xh[(size_t)s * rcap + lane + 32] = mine1;
    }
  }
  for (;;) {
    const int p = a.s_parent[s];
    if (p < 0) {  // s is the root: every forward coefficient is final (fused kernel: release them)
      if (a.sync) {
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicExch(a.sync, 1);
      }
      return;
    }
    // the father's structure and transfer matrices are static: fetch them (ranks into registers,
    // the F columns of this lane into L1) before the arrival handshake, so the climb step after it
    // waits only for the sibling's coefficients
    const int kp = a.s_rank[p];
    const int sc0 = a.s_son0[p], sc1 = a.s_son1[p];
    const int sk0 = a.s_rank[sc0], sk1 = a.s_rank[sc1];
    for (int j = lane; j < kp; j += 32)
      for (int q = 0; q < 2; ++q) {
        const double* F = a.s_tr + (size_t)(q ? sc1 : sc0) * rcap * rcap + (size_t)j * rcap;
        const int kc = q ? sk1 : sk0;
        for (int i = 0; i < kc; i += 16) asm volatile("prefetch.global.L1 [%0];" ::"l"(F + i));
      }
    __threadfence();
    __syncwarp();
    int old = 0;
    if (lane == 0) old = atomicAdd(a.s_arrive + p, 1);
    old = __shfl_sync(FULL, old, 0);
    if (old == 0) return;  // first of the two sons: the sibling finishes the father
    if (lane == 0) a.s_arrive[p] = 0;
    __threadfence();
    for (int j = lane; j < kp; j += 32) {
      double acc = 0.0;
      for (int q = 0; q < 2; ++q) {
        const int c = q ? sc1 : sc0;
        const int kc = q ? sk1 : sk0;
        const double* F = a.s_tr + (size_t)c * rcap * rcap;
        const double* xc = a.s_xh + (size_t)c * rcap;
        for (int i = 0; i < kc; ++i) acc += F[i + (size_t)j * rcap] * __ldcg(xc + i);
      }
      a.s_xh[(size_t)p * rcap + j] = acc;
    }
    s = p;
  }
}

// ---- nearfield rows of a destination leaf: (a0, a1) += sum_b N_b x|s ----------------------------
__device__ __forceinline__ void mv_near(const MvArgs& a, int t, int m, int lane, double& a0, double& a1) {
  const int lmax = a.lmax;
  for (int q = a.nptr[t]; q < a.nptr[t + 1]; ++q) {
    const int slot = a.nidx[q];
    const int s = a.npartner[slot];
    const int los = a.s_lo[s], ms = a.s_hi[s] - los;
    const double xs0 = lane < ms ? a.x[a.s_perm[los + lane]] : 0.0;
    const double xs1 = lane + 32 < ms ? a.x[a.s_perm[los + lane + 32]] : 0.0;
    const double* Na = a.N + (size_t)slot * lmax * lmax;
    if (!a.transpose) {
      for (int j0 = 0; j0 < ms; j0 += 16) {
        const int jn = ms - j0 < 16 ? ms - j0 : 16;
        const double xsrc = j0 >= 32 ? xs1 : xs0;
        const int jl = j0 & 31;
        const double* Nj = Na + (size_t)j0 * lmax;
        if (jn == 16) {  // 16-column panel in flight: 16 coalesced 256 B loads per row set
          for (int r0 = 0; r0 < m; r0 += 32) {
            double v[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = r0 + lane < m ? __ldcs(Nj + r0 + lane + (size_t)j * lmax) : 0.0;
            double acc = 0.0;
#pragma unroll
            for (int j = 0; j < 16; ++j) acc += v[j] * __shfl_sync(FULL, xsrc, jl + j);
            if (r0) a1 += acc;
            else a0 += acc;
          }
        } else {
          for (int j = 0; j < jn; ++j) {
            const double xj = __shfl_sync(FULL, xsrc, jl + j);
            if (lane < m) a0 += __ldcs(Nj + lane + (size_t)j * lmax) * xj;
            if (lane + 32 < m) a1 += __ldcs(Nj + lane + 32 + (size_t)j * lmax) * xj;
          }
        }
      }
    } else {  // y|t += N_b^T x|s: row `lane` of N_b^T is column `lane` of N_b
      const int i1 = ms < 32 ? ms : 32;
#pragma unroll 8
      for (int i = 0; i < i1; ++i) {
        const double xi = __shfl_sync(FULL, xs0, i);
        if (lane < m) a0 += __ldg(Na + i + (size_t)lane * lmax) * xi;
        if (lane + 32 < m) a1 += __ldg(Na + i + (size_t)(lane + 32) * lmax) * xi;
      }
#pragma unroll 8
      for (int i = 32; i < ms; ++i) {
        const double xi = __shfl_sync(FULL, xs1, i - 32);
        if (lane < m) a0 += __ldg(Na + i + (size_t)lane * lmax) * xi;
        if (lane + 32 < m) a1 += __ldg(Na + i + (size_t)(lane + 32) * lmax) * xi;
      }
    }
  }
}

// ---- nearfield of one destination leaf: y|t = alpha sum_b N_b x|s + beta y|t ----------------------
__device__ void mv_leaf_near(const MvArgs& a, int t, int lane) {
  const int lo = a.d_lo[t], m = a.d_hi[t] - lo;
  double a0 = 0.0, a1 = 0.0;
  mv_near(a, t, m, lane, a0, a1);
  if (lane < m) {
    const int64_t o = a.d_perm[lo + lane];
    a.y[o] = a.beta == 0.0 ? a.alpha * a0 : a.alpha * a0 + a.beta * a.y[o];
  }
  if (lane + 32 < m) {
    const int64_t o = a.d_perm[lo + lane + 32];
    a.y[o] = a.beta == 0.0 ? a.alpha * a1 : a.alpha * a1 + a.beta * a.y[o];
  }
}

// ---- couplings of one destination cluster: yc_t = sum_{b in row(t)} S_b xhat_s --------------------
// Lane = block: each lane forms the whole k_t-vector S_b xhat_s of one block of row(t) in
// registers (all its loads independent: k_t x k_s of them in flight per lane, 32 blocks per warp),
// then the warp sums the lanes with a fixed butterfly (deterministic).  KT = k_t rounded up to a
// register-array bucket.
template <int KT>
__device__ __forceinline__ void mv_couple_kt(const MvArgs& a, int t, int kt, int i0, int lane) {
  const int rcap = a.rcap;
  double acc[KT];
#pragma unroll
  for (int i = 0; i < KT; ++i) acc[i] = 0.0;
  const int qb = a.d_bptr[t], qe = a.d_bptr[t + 1];
  for (int q = qb + lane; q - lane < qe; q += 32) {
    if (q < qe) {
      const int slot = a.d_bidx[q];
      const int s = a.partner[slot];
      const int ks = a.s_rank[s];
      const double* Sa = a.S + (size_t)slot * rcap * rcap;
      const double* xs = a.s_xh + (size_t)s * rcap;
      if (!a.transpose) {  // rows i0.. of S_b: column j contiguous
#pragma unroll 4
        for (int j = 0; j < ks; ++j) {
          const double xj = __ldcg(xs + j);
          const double* Sj = Sa + (size_t)j * rcap + i0;
#pragma unroll
          for (int i = 0; i < KT; ++i)
            if (i0 + i < kt) acc[i] = fma(Sj[i], xj, acc[i]);
        }
      } else {  // S_b^T: row i of S^T = column i of S, contiguous
#pragma unroll
        for (int i = 0; i < KT; ++i) {
          if (i0 + i < kt) {
            const double* Si = Sa + (size_t)(i0 + i) * rcap;
            double v = 0.0;
#pragma unroll 4
            for (int j = 0; j < ks; ++j) v = fma(Si[j], __ldcg(xs + j), v);
            acc[i] += v;
          }
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < KT; ++i) {
    if (i0 + i < kt) {
      double v = acc[i];
#pragma unroll
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
      if (lane == i) a.d_xh[(size_t)t * rcap + i0 + i] = v;
    }
  }
}

__device__ void mv_couple(const MvArgs& a, int t, int lane) {
  const int kt = a.d_rank[t];
  if (kt == 0) return;
  if (kt <= 8) mv_couple_kt<8>(a, t, kt, 0, lane);
  else if (kt <= 16) mv_couple_kt<16>(a, t, kt, 0, lane);
  else {
    for (int i0 = 0; i0 < kt; i0 += 32) mv_couple_kt<32>(a, t, kt, i0, lane);
  }
}

// ---- backward transform along the path root -> leaf t, then y|t += alpha V_t yhat_t ---------------
// yhat_c = yc_c + E_c yhat_{father(c)} level by level along the leaf's ancestor row (lane L holds the
// cluster of level L).  The 8 leaves of a block are consecutive in DFS order, so their paths share
// a prefix (the common ancestors of the first and the last leaf): warp 0 walks it once and leaves
// yhat of the deepest common ancestor in shared memory, then every warp walks its own remainder.
// No cross-block synchronisation.
__device__ __forceinline__ void walk_levels(const MvArgs& a, int c0, int c1, int k0, int k1, int Lb, int Le,
                                            int lane, double& y0, double& y1, int& kprev) {
  const int rcap = a.rcap;
  for (int L = Lb; L < Le; ++L) {
    const int c = __shfl_sync(FULL, L < 32 ? c0 : c1, L & 31);
    const int kc = __shfl_sync(FULL, L < 32 ? k0 : k1, L & 31);
    const double* yc = a.d_xh + (size_t)c * rcap;
    double n0 = lane < kc ? __ldcg(yc + lane) : 0.0;
    double n1 = lane + 32 < kc ? __ldcg(yc + lane + 32) : 0.0;
    if (kprev > 0 && kc > 0) {
      const double* E = a.d_tr + (size_t)c * rcap * rcap;
#pragma unroll 4
      for (int j = 0; j < kprev; ++j) {
        const double yj = __shfl_sync(FULL, j < 32 ? y0 : y1, j & 31);
        if (lane < kc) n0 += E[lane + (size_t)j * rcap] * yj;
        if (lane + 32 < kc) n1 += E[lane + 32 + (size_t)j * rcap] * yj;
      }
    }
    y0 = n0;
    y1 = n1;
    kprev = kc;
  }
}

__device__ void mv_walk(const MvArgs& a, int lane, int group) {
  __shared__ double ysh[64];
  __shared__ int sh[2];  // common prefix length, rank at its end
  const int rcap = a.rcap, lmax = a.lmax, aw = a.d_ancw;
  const int warp = threadIdx.x >> 5;
  const int lf = group * 8, ll = min(lf + 8, a.d_nleaves) - 1;  // first / last leaf ordinal
  if (warp == 0) {
    const int32_t* pf = a.d_anc + (size_t)lf * aw;
    const int32_t* pl = a.d_anc + (size_t)ll * aw;
    const int f0 = lane < aw ? pf[lane] : -2, f1 = lane + 32 < aw ? pf[lane + 32] : -2;
    const int l0 = lane < aw ? pl[lane] : -3, l1 = lane + 32 < aw ? pl[lane + 32] : -3;
    const unsigned d0 = __ballot_sync(FULL, f0 != l0 || f0 < 0), d1 = __ballot_sync(FULL, f1 != l1 || f1 < 0);
    const int Lc = d0 ? __ffs(d0) - 1 : (d1 ? 32 + __ffs(d1) - 1 : 64);  // first differing level
    const int k0 = f0 >= 0 ? a.d_rank[f0] : 0, k1 = f1 >= 0 ? a.d_rank[f1] : 0;
    double y0 = 0.0, y1 = 0.0;
    int kprev = 0;
    walk_levels(a, f0, f1, k0, k1, 0, Lc, lane, y0, y1, kprev);
    if (lane < kprev) ysh[lane] = y0;
    if (lane + 32 < kprev) ysh[lane + 32] = y1;
    if (lane == 0) {
      sh[0] = Lc;
      sh[1] = kprev;
    }
  }
  __syncthreads();
  const int li = lf + warp;
  if (li >= a.d_nleaves) return;
  const int Lc = sh[0];
  int kprev = sh[1];
  double y0 = lane < kprev ? ysh[lane] : 0.0, y1 = lane + 32 < kprev ? ysh[lane + 32] : 0.0;
  const int32_t* path = a.d_anc + (size_t)li * aw;
  const int c0 = lane < aw ? path[lane] : -1;
  const int c1 = lane + 32 < aw ? path[lane + 32] : -1;
  const int nl = __popc(__ballot_sync(FULL, c0 >= 0)) + __popc(__ballot_sync(FULL, c1 >= 0));  // path length
  const int k0 = c0 >= 0 ? a.d_rank[c0] : 0, k1 = c1 >= 0 ? a.d_rank[c1] : 0;
  walk_levels(a, c0, c1, k0, k1, Lc, nl, lane, y0, y1, kprev);
  const int t = __shfl_sync(FULL, (nl - 1) < 32 ? c0 : c1, (nl - 1) & 31);
  const int kt = kprev;
  if (kt == 0) return;
  const int lo = a.d_lo[t], m = a.d_hi[t] - lo;
  const double* V = a.d_leafb + (size_t)a.d_leafidx[t] * lmax * rcap;
  double a0 = 0.0, a1 = 0.0;
  for (int j = 0; j < kt; ++j) {
    const double yj = __shfl_sync(FULL, j < 32 ? y0 : y1, j & 31);
    if (lane < m) a0 += V[lane + (size_t)j * lmax] * yj;
    if (lane + 32 < m) a1 += V[lane + 32 + (size_t)j * lmax] * yj;
  }
  // y was written by another warp (nearfield phase, maybe on another SM in the fused kernel): read
  // it through L2, never from a possibly stale L1 line
  if (lane < m) {
    double* yo = a.y + a.d_perm[lo + lane];
    *yo = __ldcg(yo) + a.alpha * a0;
  }
  if (lane + 32 < m) {
    double* yo = a.y + a.d_perm[lo + lane + 32];
    *yo = __ldcg(yo) + a.alpha * a1;
  }
}

__global__ void __launch_bounds__(256, 4) k_matvec_near(const __grid_constant__ MvArgs a) {
  const int w = (int)(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5));
  if (w < a.d_nleaves) mv_leaf_near(a, a.d_leaves[w], threadIdx.x & 31);
}

__global__ void __launch_bounds__(256) k_matvec_fwd(const __grid_constant__ MvArgs a) {
  const int w = (int)(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5));
  if (w < a.s_nleaves) mv_up(a, a.s_leaves[w], threadIdx.x & 31);
}

__global__ void __launch_bounds__(256, 2) k_matvec_couple(const __grid_constant__ MvArgs a) {
  const int w = (int)(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5));
  if (w < a.d_nclusters) mv_couple(a, w, threadIdx.x & 31);
}

__global__ void __launch_bounds__(256) k_matvec_walk(const __grid_constant__ MvArgs a) {
  mv_walk(a, threadIdx.x & 31, blockIdx.x);
}

// ---- far field by subtrees (default path) ------------------------------------------------------
// The forward transform runs one CTA (32 warps) per maximal subtree with <= 64 leaves: its levels
// bottom-up with block barriers, no atomics; the last CTA to finish (arrival counter) computes the
// clusters above the subtrees level by level.  The couplings run lane-per-block (above); the last
// CTA of that launch carries the backward transform down through the top clusters; then one CTA
// per subtree carries it down to its leaves and adds alpha V_t yhat_t to y.  So the latency chain
// is ~2 x (64-leaf subtree depth + top depth) block-barrier levels instead of ~2 x 13 dependent
// global round trips with atomics per level (climb, ancestor walks).
constexpr int SUBT = 512;  // threads of a subtree CTA (16 warps; leaves room for nearfield CTAs on the SM)

struct SubList {  // the clusters of one subtree bucketed by level below its root
  int nlev;
  int cnt[64];
  int ptr[65];
  int cl[2 * MV_SUB_LEAVES];
};

__device__ void build_sublist(const int32_t* level, const int32_t* tsize, int root, SubList& L) {
  const int n = tsize[root], l0 = level[root];
  if (threadIdx.x < 64) L.cnt[threadIdx.x] = 0;
  __syncthreads();
  int rel = -1, slot = 0;
  if ((int)threadIdx.x < n) {
    rel = level[root + threadIdx.x] - l0;
    slot = atomicAdd(&L.cnt[rel], 1);  // order inside a level is irrelevant (independent clusters)
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0, nl = 0;
    for (int l = 0; l < 64; ++l) {
      L.ptr[l] = acc;
      acc += L.cnt[l];
      if (L.cnt[l]) nl = l + 1;
    }
    L.ptr[64] = acc;
    L.nlev = nl;
  }
  __syncthreads();
  if (rel >= 0) L.cl[L.ptr[rel] + slot] = root + threadIdx.x;
  __syncthreads();
}

// xhat_s for one source cluster by one warp: a leaf from x, an internal cluster from its sons
__device__ __forceinline__ void fwd_cluster(const MvArgs& a, int s, int lane) {
  const int rcap = a.rcap, lmax = a.lmax;
  const int k = a.s_rank[s];
  if (k == 0) return;
  if (a.s_son0[s] < 0) {
    const int lo = a.s_lo[s], m = a.s_hi[s] - lo;
    const double x0 = lane < m ? a.x[a.s_perm[lo + lane]] : 0.0;
    const double x1 = lane + 32 < m ? a.x[a.s_perm[lo + lane + 32]] : 0.0;
    const double* W = a.s_leafb + (size_t)a.s_leafidx[s] * lmax * rcap;
    double mine0 = 0.0, mine1 = 0.0;
    for (int j = 0; j < k; ++j) {
      double p = 0.0;
      if (lane < m) p = W[lane + (size_t)j * lmax] * x0;
      if (lane + 32 < m) p += W[lane + 32 + (size_t)j * lmax] * x1;
#pragma unroll
      for (int o = 16; o; o >>= 1) p += __shfl_xor_sync(FULL, p, o);
      if (lane == (j & 31)) {
        if (j < 32) mine0 = p;
        else mine1 = p;
      }
    }
    if (lane < k) a.s_xh[(size_t)s * rcap + lane] = mine0;
    if (lane + 32 < k) a.s_xh[(size_t)s * rcap + lane + 32] = mine1;
    return;
  }
  const int sc0 = a.s_son0[s], sc1 = a.s_son1[s];
  const int sk0 = a.s_rank[sc0], sk1 = a.s_rank[sc1];
  for (int j = lane; j < k; j += 32) {
    double acc = 0.0;
    for (int q = 0; q < 2; ++q) {
      const int c = q ? sc1 : sc0;
      const int kc = q ? sk1 : sk0;
      const double* F = a.s_tr + (size_t)c * rcap * rcap;
      const double* xc = a.s_xh + (size_t)c * rcap;
      for (int i = 0; i < kc; ++i) acc += F[i + (size_t)j * rcap] * __ldcg(xc + i);
    }
    a.s_xh[(size_t)s * rcap + j] = acc;
  }
}

// yhat_c = yc_c + E_c yhat_{father(c)} in place (the father is final), one warp
__device__ __forceinline__ void bwd_cluster(const MvArgs& a, int c, int lane) {
  const int rcap = a.rcap;
  const int p = a.d_parent[c];
  const int kc = a.d_rank[c];
  if (p < 0 || kc == 0) return;
  const int kp = a.d_rank[p];
  const double* E = a.d_tr + (size_t)c * rcap * rcap;
  const double* yp = a.d_xh + (size_t)p * rcap;
  double* yc = a.d_xh + (size_t)c * rcap;
  double n0 = lane < kc ? __ldcg(yc + lane) : 0.0;
  double n1 = lane + 32 < kc ? __ldcg(yc + lane + 32) : 0.0;
  for (int j = 0; j < kp; ++j) {
    const double yj = __ldcg(yp + j);
    if (lane < kc) n0 += E[lane + (size_t)j * rcap] * yj;
    if (lane + 32 < kc) n1 += E[lane + 32 + (size_t)j * rcap] * yj;
  }
  if (lane < kc) yc[lane] = n0;
  if (lane + 32 < kc) yc[lane + 32] = n1;
}

__global__ void __launch_bounds__(SUBT, 2) k_mv_fwd_sub(const __grid_constant__ MvArgs a) {
  __shared__ SubList L;
  __shared__ int last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = SUBT / 32;
  build_sublist(a.s_level, a.s_tsize, a.s_roots[blockIdx.x], L);
  for (int l = L.nlev - 1; l >= 0; --l) {
    for (int i = L.ptr[l] + warp; i < L.ptr[l + 1]; i += nw) fwd_cluster(a, L.cl[i], lane);
    __syncthreads();
  }
  // the last subtree to finish computes the clusters above the subtrees, bottom-up
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(a.s_cnt, 1) == (int)gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int l = a.s_top_nlev - 1; l >= 0; --l) {
    for (int i = a.s_top_lptr[l] + warp; i < a.s_top_lptr[l + 1]; i += nw) fwd_cluster(a, a.s_top[i], lane);
    __syncthreads();
  }
  if (threadIdx.x == 0) a.s_cnt[0] = 0;
}

// couplings (lane per block), then the last CTA carries yhat down through the top clusters
__global__ void __launch_bounds__(256, 2) k_mv_couple_top(const __grid_constant__ MvArgs a) {
  __shared__ int last;
  const int lane = threadIdx.x & 31;
  const int w = (int)(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5));
  if (w < a.d_nclusters) mv_couple(a, w, lane);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(a.d_cnt, 1) == (int)gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int l = 1; l < a.d_top_nlev; ++l) {  // the root (level 0) keeps its coupling sum
    for (int i = a.d_top_lptr[l] + warp; i < a.d_top_lptr[l + 1]; i += nw) bwd_cluster(a, a.d_top[i], lane);
    __syncthreads();
  }
  if (threadIdx.x == 0) a.d_cnt[0] = 0;
}

// backward transform inside one destination subtree (root first), then y|t += alpha V_t yhat_t
__global__ void __launch_bounds__(SUBT, 2) k_mv_bwd_sub(const __grid_constant__ MvArgs a) {
  __shared__ SubList L;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = SUBT / 32;
  build_sublist(a.d_level, a.d_tsize, a.d_roots[blockIdx.x], L);
  for (int l = 0; l < L.nlev; ++l) {
    for (int i = L.ptr[l] + warp; i < L.ptr[l + 1]; i += nw) bwd_cluster(a, L.cl[i], lane);
    __syncthreads();
  }
  const int rcap = a.rcap, lmax = a.lmax;
  for (int i = warp; i < L.ptr[L.nlev]; i += nw) {
    const int t = L.cl[i];
    if (a.d_son0[t] >= 0) continue;
    const int kt = a.d_rank[t];
    if (kt == 0) continue;
    const int lo = a.d_lo[t], m = a.d_hi[t] - lo;
    const double* V = a.d_leafb + (size_t)a.d_leafidx[t] * lmax * rcap;
    const double* yh = a.d_xh + (size_t)t * rcap;
    double a0 = 0.0, a1 = 0.0;
    for (int j = 0; j < kt; ++j) {
      const double yj = yh[j];
      if (lane < m) a0 += V[lane + (size_t)j * lmax] * yj;
      if (lane + 32 < m) a1 += V[lane + 32 + (size_t)j * lmax] * yj;
    }
    if (lane < m) {
      double* yo = a.y + a.d_perm[lo + lane];
      *yo = *yo + a.alpha * a0;
    }
    if (lane + 32 < m) {
      double* yo = a.y + a.d_perm[lo + lane + 32];
      *yo = *yo + a.alpha * a1;
    }
  }
}

// ---- the whole far + near field in ONE persistent (cooperative) launch --------------------------
// Every warp: (A) forward transform of its source leaves with the climb (the warp completing the
// root publishes sync[0]); (B) the nearfield of its destination leaves, y = alpha N x + beta y --
// the bulk of the bytes streams while the climb's latency chain finishes elsewhere; (C) once the
// forward coefficients are final, the couplings of its destination clusters (sync[1] counts the
// warps done); (D) once every coupling is in, each CTA walks its groups of 8 leaves and adds
// alpha V_t yhat_t.  The CTAs are co-resident (cooperative launch), so the two spin-waits cannot
// deadlock; the last CTA to leave resets the counters for the next product.
__device__ __forceinline__ void spin_until(const int* p, int v) {
  while (*(volatile const int*)p < v) __nanosleep(64);
  __threadfence();
}

__global__ void __launch_bounds__(256, 2) k_matvec_fused(const __grid_constant__ MvArgs a) {
  const int lane = threadIdx.x & 31;
  const int nw = (int)(gridDim.x * (blockDim.x >> 5));
  const int w0 = (int)(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5));
  for (int w = w0; w < a.s_nleaves; w += nw) mv_up(a, a.s_leaves[w], lane);
  for (int w = w0; w < a.d_nleaves; w += nw) mv_leaf_near(a, a.d_leaves[w], lane);
  spin_until(a.sync, 1);
  for (int w = w0; w < a.d_nclusters; w += nw) mv_couple(a, w, lane);
  __threadfence();
  __syncwarp();
  if (lane == 0) atomicAdd(a.sync + 1, 1);
  spin_until(a.sync + 1, nw);
  const int ngroups = (a.d_nleaves + 7) / 8;
  for (int g = blockIdx.x; g < ngroups; g += gridDim.x) {
    mv_walk(a, lane, g);
    __syncthreads();  // the shared path prefix of the next group
  }
  __syncthreads();
  if (threadIdx.x == 0 && atomicAdd(a.sync + 2, 1) == (int)gridDim.x - 1) {
    a.sync[0] = 0;
    a.sync[1] = 0;
    a.sync[2] = 0;
    __threadfence();
  }
}

inline int cdiv(long long a, long long b) { return (int)((a + b - 1) / b); }

}  // namespace

cudaError_t launch_matvec(const h2_mat_* Z, int transpose, double alpha, const double* x, double beta, double* y,
                          cudaStream_t st) {
  const MatDev& M = Z->d;
  const DevSide& src = transpose ? M.row : M.col;  // basis applied to x
  const DevSide& dst = transpose ? M.col : M.row;  // basis producing y
  MvArgs a;
  a.s_leaves = src.leaves;
  a.s_lo = src.lo;
  a.s_hi = src.hi;
  a.s_leafidx = src.leafidx;
  a.s_rank = src.rank;
  a.s_parent = src.parent;
  a.s_son0 = src.son0;
  a.s_son1 = src.son1;
  a.s_perm = src.perm;
  a.s_leafb = src.leafb;
  a.s_tr = src.tr;
  a.s_xh = src.xh;
  a.s_arrive = src.mvsync;
  a.s_nleaves = src.nleaves;
  a.d_bfs = dst.bfs;
  a.d_leaves = dst.leaves;
  a.d_nleaves = dst.nleaves;
  a.d_lo = dst.lo;
  a.d_hi = dst.hi;
  a.d_leafidx = dst.leafidx;
  a.d_rank = dst.rank;
  a.d_parent = dst.parent;
  a.d_son0 = dst.son0;
  a.d_bptr = dst.bptr;
  a.d_bidx = dst.bidx;
  a.d_perm = dst.perm;
  a.d_leafb = dst.leafb;
  a.d_tr = dst.tr;
  a.d_xh = dst.xh;
  a.d_anc = dst.anc;
  a.d_ancw = dst.ancw;
  a.d_nclusters = dst.nclusters;
  a.partner = transpose ? M.adm_t : M.adm_s;
  a.S = M.S;
  a.nptr = transpose ? M.ntptr : M.nptr;
  a.nidx = transpose ? M.ntidx : M.nidx;
  a.npartner = transpose ? M.in_t : M.in_s;
  a.N = M.N;
  a.lmax = M.lmax;
  a.rcap = M.rcap;
  a.transpose = transpose;
  a.x = x;
  a.y = y;
  a.alpha = alpha;
  a.beta = beta;
  a.s_roots = src.mv_roots;
  a.s_top = src.mv_top;
  a.s_top_lptr = src.mv_top_lptr;
  a.s_top_nlev = src.mv_top_nlev;
  a.s_tsize = src.tsize;
  a.s_level = src.level;
  a.s_cnt = src.mv_cnt;
  a.d_roots = dst.mv_roots;
  a.d_top = dst.mv_top;
  a.d_top_lptr = dst.mv_top_lptr;
  a.d_top_nlev = dst.mv_top_nlev;
  a.d_tsize = dst.tsize;
  a.d_level = dst.level;
  a.d_son1 = dst.son1;
  a.d_cnt = dst.mv_cnt;
  // the far field contributes only if some row and some column basis may have a non-zero rank
  const bool far = std::find(Z->nzr.begin(), Z->nzr.end(), 1) != Z->nzr.end() &&
                   std::find(Z->nzc.begin(), Z->nzc.end(), 1) != Z->nzc.end();
  a.sync = nullptr;
  if (!far) {
    H2_LAUNCH(K_MV, st, k_matvec_near<<<cdiv(dst.nleaves, 8), 256, 0, st>>>(a));
    return cudaGetLastError();
  }
  // one cooperative launch (k_matvec_fused) only on request (H2_MV_FUSED=1): measured 334 us for
  // the C2 factor L against 167 us for the four-launch path below -- a persistent grid of 2 CTAs
  // per SM serialises the latency-bound climb / coupling / walk work that the separate launches
  // spread over 8-16k warps
  static const bool fused_on = getenv("H2_MV_FUSED") && atoi(getenv("H2_MV_FUSED")) != 0;
  static int fused_grid = -1;
  static std::unordered_map<cudaStream_t, int*> syncs;  // counters per stream (products on one stream are ordered)
  cudaError_t e;
  if (fused_on && fused_grid < 0) {
    int dev = 0, nsm = 0, per = 0, coop = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_matvec_fused, 256, 0);
    fused_grid = coop ? nsm * std::min(per, 2) : 0;
    cudaGetLastError();
  }
  if (fused_on && fused_grid > 0) {
    int*& sync = syncs[st];
    if (!sync) {
      if ((e = cudaMalloc(&sync, 4 * sizeof(int)))) return e;
      if ((e = cudaMemset(sync, 0, 4 * sizeof(int)))) return e;
    }
    a.sync = sync;
    void* args[] = {(void*)&a};
    H2_LAUNCH(K_MV, st, e = cudaLaunchCooperativeKernel((const void*)k_matvec_fused, dim3(fused_grid), dim3(256), args, 0, st));
    if (e) return e;
    return cudaGetLastError();
  }
  a.sync = nullptr;
  // the nearfield stream (the bulk of the bytes) runs on a second stream, concurrently with the
  // forward transform and the couplings; the backward walk adds V_t yhat_t after both
  static cudaStream_t s2 = nullptr;
  static cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  if (!s2) {
    // the nearfield stream gets the higher priority: it is the bandwidth-bound critical path, the
    // far-field kernels fill the SMs around it
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if ((e = cudaStreamCreateWithPriority(&s2, cudaStreamNonBlocking, hi))) return e;
    if ((e = cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming))) return e;
    if ((e = cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming))) return e;
  }
  static const bool walk_path = getenv("H2_MV_WALK") && atoi(getenv("H2_MV_WALK")) != 0;  // round-1 path (A/B)
  // timing diagnostics (tools): H2_MV_PART=1 far field only, 2 nearfield only (y is then incomplete)
  static const int part = getenv("H2_MV_PART") ? atoi(getenv("H2_MV_PART")) : 0;
  if (part == 1 || part == 3 || part == 4) {  // 3: forward only, 4: forward + couplings
    H2_LAUNCH(K_MV, st, k_mv_fwd_sub<<<src.n_mv_roots, SUBT, 0, st>>>(a));
    if (part != 3) H2_LAUNCH(K_MV, st, k_mv_couple_top<<<cdiv(dst.nclusters, 8), 256, 0, st>>>(a));
    if (part == 1) H2_LAUNCH(K_MV, st, k_mv_bwd_sub<<<dst.n_mv_roots, SUBT, 0, st>>>(a));
    return cudaGetLastError();
  }
  if (part == 2) {
    H2_LAUNCH(K_MV, st, k_matvec_near<<<cdiv(dst.nleaves, 8), 256, 0, st>>>(a));
    return cudaGetLastError();
  }
  if ((e = cudaEventRecord(ev_fork, st))) return e;
  if ((e = cudaStreamWaitEvent(s2, ev_fork, 0))) return e;
  H2_LAUNCH(K_MV, s2, k_matvec_near<<<cdiv(dst.nleaves, 8), 256, 0, s2>>>(a));
  if ((e = cudaEventRecord(ev_join, s2))) return e;
  if (walk_path) {
    H2_LAUNCH(K_MV, st, k_matvec_fwd<<<cdiv(src.nleaves, 8), 256, 0, st>>>(a));
    H2_LAUNCH(K_MV, st, k_matvec_couple<<<cdiv(dst.nclusters, 8), 256, 0, st>>>(a));
    if ((e = cudaStreamWaitEvent(st, ev_join, 0))) return e;
    H2_LAUNCH(K_MV, st, k_matvec_walk<<<cdiv(dst.nleaves, 8), 256, 0, st>>>(a));
    return cudaGetLastError();
  }
  H2_LAUNCH(K_MV, st, k_mv_fwd_sub<<<src.n_mv_roots, SUBT, 0, st>>>(a));
  H2_LAUNCH(K_MV, st, k_mv_couple_top<<<cdiv(dst.nclusters, 8), 256, 0, st>>>(a));
  if ((e = cudaStreamWaitEvent(st, ev_join, 0))) return e;
  H2_LAUNCH(K_MV, st, k_mv_bwd_sub<<<dst.n_mv_roots, SUBT, 0, st>>>(a));
  return cudaGetLastError();
}

}  // namespace h2
