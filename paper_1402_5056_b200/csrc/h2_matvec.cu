// H^2 matrix-vector product y = alpha op(Z) x + beta y ([BO10 Thm 3.42]).
//
//   forward transform   xhat_s = W_s^T x|s (leaves),  xhat_s = sum_{s'} F_{s'}^T xhat_{s'}   bottom-up
//   couplings           yhat_t = sum_{s in row(t)} S_(t,s) xhat_s
//   backward transform  yhat_{t'} += E_{t'} yhat_t  top-down; leaves y|t = V_t yhat_t
//   nearfield           y|t += sum_{b=(t,s) inadmissible} N_b x|s
//
// Two streams: the nearfield kernel (the bulk of the bytes: warp per destination leaf, lanes own
// rows, 16-column panels of coalesced 256 B streaming loads) runs on a second, high-priority
// stream concurrently with the far-field chain
//   k_mv_leaf_fwd -> k_mv_fwd_sub -> k_mv_couple_top -> k_mv_bwd_sub -> [join] -> k_mv_leaf_bwd
// described below; a matrix whose bases all have rank 0 launches the nearfield kernel only.
// No grid-wide barrier, no spin-waits; the arrival counters are reset by their last user.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
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
  // subtree schedule (DevSide::mv_*): source side (forward) and destination side (backward)
  const int32_t *s_roots, *s_top, *s_top_lptr, *s_tsize, *s_level;
  int s_top_nlev;
  int32_t* s_cnt;
  const int32_t *d_roots, *d_top, *d_top_lptr, *d_tsize, *d_level, *d_son1;
  int d_top_nlev;
  int32_t* d_cnt;
  // packed copies at the current ranks (MvPack): couplings (slot -> offset), transfers per side
  const double* Sp;
  const int64_t* Soff;
  const double *s_Tp, *d_Tp;
  const int64_t *s_Toff, *d_Toff;
  int s_nroots;              // CTAs of k_mv_fwd_sub (subtrees of the source side)
  unsigned s_epoch;          // products run on this source side so far + 1: the forward counters never reset
  int same_tree;             // rows and columns share the cluster tree (levels comparable)
  int sub_tb;                // doubles of staged transfers per subtree CTA (shared memory budget)
  const MvPack::Desc* desc;  // blocks of the destination clusters in d_bidx order
  unsigned long long* dbg;  // H2_MV_DBG: globaltimer stamps of the far-field phases (diagnostic)
};

__device__ __forceinline__ void stamp(const MvArgs& a, int i) {
  if (a.dbg && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.dbg[i] = t;
  }
}

constexpr unsigned FULL = 0xffffffffu;

// Programmatic dependent launch (the far-field chain): a kernel launched with the attribute may
// start while its predecessor in the stream still runs; pdl_wait() blocks until the predecessor
// has completed and its memory is visible, pdl_trigger() lets the successor start launching.
// Everything before pdl_wait() must not read what the predecessor writes.
// Far-field operands (leaf bases, packed transfers and couplings: ~90 MB at C2) are loaded with the
// L2 evict_last priority, the nearfield tiles (~340 MB per product) stream with evict_first
// (__ldcs): across consecutive products of the same matrix the far field then stays resident in
// the 126 MB L2 and its dependent round trips hit L2 instead of queueing behind the nearfield
// stream in DRAM.  H2_MV_NOHINT=1 (compile-time -DH2_MV_NOHINT) disables the hint for A/B runs.
__device__ __forceinline__ unsigned long long el_policy() {
  unsigned long long pol = 0;
#ifndef H2_MV_NOHINT
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
#endif
  return pol;
}
__device__ __forceinline__ double ld_el(const double* p, unsigned long long pol) {
#ifdef H2_MV_NOHINT
  return *p;
#else
  double v;
  asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
#endif
}

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---- nearfield rows of a destination leaf: (a0, a1) += sum_b N_b x|s ----------------------------
template <bool TR>
__device__ __forceinline__ void mv_near(const MvArgs& a, int t, int m, int lane, double& a0, double& a1) {
  const int lmax = a.lmax;
  for (int q = a.nptr[t]; q < a.nptr[t + 1]; ++q) {
    const int slot = a.nidx[q];
    const int s = a.npartner[slot];
    const int los = a.s_lo[s], ms = a.s_hi[s] - los;
    const double xs0 = lane < ms ? a.x[a.s_perm[los + lane]] : 0.0;
    const double xs1 = lane + 32 < ms ? a.x[a.s_perm[los + lane + 32]] : 0.0;
    const double* Na = a.N + (size_t)slot * lmax * lmax;
    if (!TR) {
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
      // (a coalesced variant -- lanes own the rows of N_b, 16-column panels, column sums by
      // recursive halving -- measured slower: 435 us against 318-359 us for the C2 operator)
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
template <bool TR>
__device__ __forceinline__ void mv_leaf_near(const MvArgs& a, int t, int lane) {
  const int lo = a.d_lo[t], m = a.d_hi[t] - lo;
  double a0 = 0.0, a1 = 0.0;
  mv_near<TR>(a, t, m, lane, a0, a1);
  const int c = lane;
  if (c < m) {
    const int64_t o = a.d_perm[lo + c];
    a.y[o] = a.beta == 0.0 ? a.alpha * a0 : a.alpha * a0 + a.beta * a.y[o];
  }
  if (c + 32 < m) {
    const int64_t o = a.d_perm[lo + c + 32];
    a.y[o] = a.beta == 0.0 ? a.alpha * a1 : a.alpha * a1 + a.beta * a.y[o];
  }
}

__global__ void __launch_bounds__(256, 4) k_matvec_near(const __grid_constant__ MvArgs a) {
  // grid-stride over the destination leaves (the default grid has one warp per leaf; a grid of
  // fewer CTAs per SM, H2_MV_NEARGRID, measured slower: 90 us against 66 us at 2 CTAs per SM)
  const int nw = (int)(gridDim.x * (blockDim.x >> 5));
  for (int w = (int)(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)); w < a.d_nleaves; w += nw)
    mv_leaf_near<false>(a, a.d_leaves[w], threadIdx.x & 31);
}
// Nearfield with shared-memory staging (32-point leaves, no transpose): a persistent grid of ONE
// small CTA per SM (NEAR_W warps, 16 KB of shared memory per warp); every warp streams the tiles
// of its destination leaves through a two-slot ring with cp.async (an 8 KB tile = 16 16-byte
// copies per lane), so NEAR_W x 16 KB are in flight per SM without holding registers or SM slots:
// the far-field kernels could stay co-resident on every SM instead of waiting for nearfield CTAs
// to retire (the register-panel kernel above needs 4 CTAs x 8 warps per SM and fills the register
// file).  Measured slower (see the launcher) and therefore off by default: an experiment kept
// for the next step (a deeper ring fed by bulk copies).  The slots' padding is zero and x_j = 0 beyond |s|,
// so a tile is always multiplied as 32 x 32.
constexpr int NEAR_W = 4;
__global__ void __launch_bounds__(NEAR_W * 32, 1) k_matvec_near_s(const __grid_constant__ MvArgs a) {
  extern __shared__ __align__(16) double nsm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* ring = nsm + (size_t)warp * 2048;
  const unsigned rbase = (unsigned)__cvta_generic_to_shared(ring);
  const int nwarps = (int)gridDim.x * NEAR_W;
  for (int w = (int)blockIdx.x * NEAR_W + warp; w < a.d_nleaves; w += nwarps) {
    const int t = a.d_leaves[w];
    const int lo = a.d_lo[t], m = a.d_hi[t] - lo;
    const int qb = a.nptr[t], qe = a.nptr[t + 1];
    auto issue = [&](int q, int buf) {
      const double* src = a.N + (size_t)a.nidx[q] * 1024;
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int e = (u * 32 + lane) * 2;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(rbase + (unsigned)(buf * 1024 + e) * 8u), "l"(src + e));
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    auto loadx = [&](int q) -> double {
      const int s = a.npartner[a.nidx[q]];
      const int los = a.s_lo[s], ms = a.s_hi[s] - los;
      return lane < ms ? a.x[a.s_perm[los + lane]] : 0.0;
    };
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0, xcur = 0.0, xnext = 0.0;
    if (qb < qe) {
      issue(qb, 0);
      xcur = loadx(qb);
    }
    for (int q = qb; q < qe; ++q) {
      const int buf = (q - qb) & 1;
      if (q + 1 < qe) {
        issue(q + 1, buf ^ 1);
        xnext = loadx(q + 1);
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      __syncwarp();
      const double* T = ring + buf * 1024 + lane;
#pragma unroll
      for (int j = 0; j < 32; j += 4) {
        acc0 = fma(T[(j + 0) * 32], __shfl_sync(FULL, xcur, j + 0), acc0);
        acc1 = fma(T[(j + 1) * 32], __shfl_sync(FULL, xcur, j + 1), acc1);
        acc2 = fma(T[(j + 2) * 32], __shfl_sync(FULL, xcur, j + 2), acc2);
        acc3 = fma(T[(j + 3) * 32], __shfl_sync(FULL, xcur, j + 3), acc3);
      }
      __syncwarp();  // every lane is done with this slot before it is refilled
      xcur = xnext;
    }
    if (lane < m) {
      const double r = (acc0 + acc1) + (acc2 + acc3);
      const int64_t o = a.d_perm[lo + lane];
      a.y[o] = a.beta == 0.0 ? a.alpha * r : a.alpha * r + a.beta * a.y[o];
    }
  }
}

// the transposed product as its own kernel (its own register allocation)
__global__ void __launch_bounds__(256, 2) k_matvec_near_t(const __grid_constant__ MvArgs a) {
  const int nw = (int)(gridDim.x * (blockDim.x >> 5));
  for (int w = (int)(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)); w < a.d_nleaves; w += nw)
    mv_leaf_near<true>(a, a.d_leaves[w], threadIdx.x & 31);
}


// ---- far field -----------------------------------------------------------------------------------
// Packed copies (MvPack, built once per matrix version by k_mv_pack): the couplings S_b (k_t x k_s,
// ld k_t) and the transfer matrices (k_c x k_parent, ld k_c) stored contiguously at their current
// ranks, so the far-field kernels read exactly the algorithmic bytes in coalesced bursts instead
// of k-long column pieces of rank_cap^2 slots.
//
//   k_mv_leaf_fwd    warp per source leaf: xhat_s = W_s^T x|s                    (wide: the leaf bases
//                    are the bulk of the forward transform's bytes)
//   k_mv_fwd_sub     one CTA per maximal subtree of <= 64 leaves: the subtree's xhat (a contiguous
//                    range of cluster ids) and its packed transfer matrices are staged in shared
//                    memory, the internal levels run bottom-up from shared memory with block
//                    barriers; the last CTA to finish computes the clusters above the subtrees
//   k_mv_couple_top  warp per destination cluster: yc_t = sum_b S_b xhat_s from the packed
//                    couplings (lanes = (row, column group), fixed reduction order); the last CTA
//                    carries yhat down through the clusters above the subtrees
//   k_mv_bwd_sub     one CTA per destination subtree: yhat top-down in shared memory
//   k_mv_leaf_bwd    warp per destination leaf: y|t += alpha V_t yhat_t         (wide, after the
//                    nearfield kernel on the second stream has written y)
constexpr int SUBT = 512;        // threads of a subtree CTA
constexpr int SUB_NC = 2 * MV_SUB_LEAVES;  // clusters of a subtree (<= 2 * 64 - 1)
constexpr int SUB_SMEM = 220 * 1024;  // dynamic shared memory of a subtree CTA: coefficient rows + staged transfers

struct SubList {  // the clusters of one subtree bucketed by level below its root
  int nlev;
  int cnt[64];
  int ptr[65];
  int cl[SUB_NC];
  // structure of cluster root + i (contiguous ids: one coalesced load round), so that the level
  // loops read shared memory only
  int rk[SUB_NC], s0[SUB_NC], s1[SUB_NC], par[SUB_NC];
  long long to[SUB_NC];
};

__device__ void build_sublist(const int32_t* level, const int32_t* tsize, int root, SubList& L, const int32_t* rank,
                              const int32_t* son0, const int32_t* son1, const int32_t* parent, const int64_t* Toff) {
  const int n = tsize[root], l0 = level[root];
  if (threadIdx.x < 64) L.cnt[threadIdx.x] = 0;
  __syncthreads();
  int rel = -1, slot = 0;
  if ((int)threadIdx.x < n) {
    const int c = root + threadIdx.x;
    L.rk[threadIdx.x] = rank[c];
    L.s0[threadIdx.x] = son0[c];
    L.s1[threadIdx.x] = son1[c];
    L.par[threadIdx.x] = parent[c];
    L.to[threadIdx.x] = Toff[c];
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

// xhat_s = W_s^T x|s for one source leaf by one warp
__device__ __forceinline__ void fwd_leaf(const MvArgs& a, int s, int lane) {
  const int rcap = a.rcap, lmax = a.lmax;
  const int k = a.s_rank[s];
  if (k == 0) return;
  const int lo = a.s_lo[s], m = a.s_hi[s] - lo;
  const double x0 = lane < m ? a.x[a.s_perm[lo + lane]] : 0.0;
  const double x1 = lane + 32 < m ? a.x[a.s_perm[lo + lane + 32]] : 0.0;
  const double* W = a.s_leafb + (size_t)a.s_leafidx[s] * lmax * rcap;
  double mine0 = 0.0, mine1 = 0.0;
  const unsigned long long pol = el_policy();
  constexpr int CB = 8;
  for (int j0 = 0; j0 < k; j0 += CB) {  // 8 columns per round: their loads and butterflies overlap
    double p[CB];
#pragma unroll
    for (int u = 0; u < CB; ++u) {
      const int j = j0 + u;
      p[u] = 0.0;
      if (j < k) {
        if (lane < m) p[u] = ld_el(W + lane + (size_t)j * lmax, pol) * x0;
        if (lane + 32 < m) p[u] += ld_el(W + lane + 32 + (size_t)j * lmax, pol) * x1;
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
#pragma unroll
      for (int u = 0; u < CB; ++u) p[u] += __shfl_xor_sync(FULL, p[u], o);
    }
#pragma unroll
    for (int u = 0; u < CB; ++u) {
      const int j = j0 + u;
      if (j < k && lane == (j & 31)) {
        if (j < 32) mine0 = p[u];
        else mine1 = p[u];
      }
    }
  }
  if (lane < k) a.s_xh[(size_t)s * rcap + lane] = mine0;
  if (lane + 32 < k) a.s_xh[(size_t)s * rcap + lane + 32] = mine1;
}

// xhat_s = sum over the sons c of F_c^T xhat_c (F_c^T: k_s x k_c, packed transposed, ld k_s) by one warp, inside
// a subtree: i = s - root; the sons of a binary preorder tree are i + 1 and the cluster after the
// first son's subtree (L.s0 holds son0, son1 = father's other son: found via the parent array)
__device__ __forceinline__ void fwd_internal(const SubList& L, int i, int i0, int i1, int lane, double* xs, int rcap,
                                             const double* tp, int64_t tb) {
  const int k = L.rk[i];
  if (k == 0) return;
  const int sk0 = L.rk[i0], sk1 = L.rk[i1];
  const double* F0 = tp + (L.to[i0] - tb);
  const double* F1 = tp + (L.to[i1] - tb);
  const double* x0 = xs + (size_t)i0 * rcap;
  const double* x1 = xs + (size_t)i1 * rcap;
  for (int j = lane; j < k; j += 32) {  // F^T stored k x k_c (ld k): lanes read consecutive words
    double acc = 0.0;
    for (int q = 0; q < sk0; ++q) acc += F0[j + (size_t)q * k] * x0[q];
    for (int q = 0; q < sk1; ++q) acc += F1[j + (size_t)q * k] * x1[q];
    xs[(size_t)i * rcap + j] = acc;
  }
}

// yhat_c = yc_c + E_c yhat_father (E_c: k_c x k_p, packed, ld k_c), in place, one warp
__device__ __forceinline__ void bwd_cluster(const SubList& L, int i, int ip, int lane, double* ys, int rcap,
                                            const double* tp, int64_t tb) {
  const int kc = L.rk[i];
  if (kc == 0) return;
  const int kp = L.rk[ip];
  const double* E = tp + (L.to[i] - tb);
  double* yc = ys + (size_t)i * rcap;
  const double* yp = ys + (size_t)ip * rcap;
  for (int r = lane; r < kc; r += 32) {
    double v = yc[r];
    for (int j = 0; j < kp; ++j) v += E[r + (size_t)j * kc] * yp[j];
    yc[r] = v;
  }
}

__global__ void __launch_bounds__(256) k_mv_leaf_fwd(const __grid_constant__ MvArgs a) {
  if (blockIdx.x == 0) stamp(a, 0);
  pdl_trigger();
  const int w = (int)(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5));
  if (w < a.s_nleaves) fwd_leaf(a, a.s_leaves[w], threadIdx.x & 31);
}

// Stage the packed transfers of the clusters root+1 .. root+n-1 (contiguous, 16-byte aligned: every
// packed matrix is padded to an even number of doubles) in shared memory with cp.async (16-byte
// copies, all in flight at once, no registers); the caller does other work (the sublist), then
// stage_wait.  `cap`: doubles of shared memory available behind the coefficient rows.
struct StageRegs {
  int64_t tb, len;
  bool ok;
};
__device__ __forceinline__ void stage_load(const double* Tp, const int64_t* Toff, int root, int n, StageRegs& R,
                                           double* tbuf, int cap) {
  R.tb = Toff[root + 1 < root + n ? root + 1 : root];
  R.len = Toff[root + n] - R.tb;
  R.ok = n > 1 && R.len <= cap;
  if (!R.ok) return;
  const double* src = Tp + R.tb;
  const unsigned dst = (unsigned)__cvta_generic_to_shared(tbuf);
  const int nv = (int)(R.len >> 1);  // len is even
#ifdef H2_MV_NOHINT
  for (int e = threadIdx.x; e < nv; e += blockDim.x)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16u * (unsigned)e), "l"(src + 2 * e));
#else
  const unsigned long long pol = el_policy();
  for (int e = threadIdx.x; e < nv; e += blockDim.x)
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(dst + 16u * (unsigned)e),
                 "l"(src + 2 * e), "l"(pol));
#endif
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void stage_store(const StageRegs& R, double*) {
  if (R.ok) asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// the first CTAs of a launch pull the packed transfers of the clusters above the subtrees into L2
// (one cluster each), so that the last CTA's level-by-level pass over them hits L2
__device__ __forceinline__ void prefetch_top(const double* Tp, const int64_t* Toff, const int32_t* top, int ntop) {
  if ((int)blockIdx.x >= ntop) return;
  const int c = top[blockIdx.x];
  const char* b = reinterpret_cast<const char*>(Tp + Toff[c]);
  const int64_t bytes = (Toff[c + 1] - Toff[c]) * 8;
  for (int64_t o = (int64_t)threadIdx.x * 128; o < bytes; o += (int64_t)blockDim.x * 128)
    asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(b + o));
}

__global__ void __launch_bounds__(SUBT, 1) k_mv_fwd_sub(const __grid_constant__ MvArgs a) {
  extern __shared__ __align__(16) double dsm[];
  __shared__ SubList L;
  __shared__ int last;
  const int rcap = a.rcap;
  double* xs = dsm;                       // SUB_NC x rcap: xhat of the subtree's clusters
  double* tbuf = dsm + (size_t)SUB_NC * rcap;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = SUBT / 32;
  const int root = a.s_roots[blockIdx.x], n = a.s_tsize[root];
  if (blockIdx.x == 0) stamp(a, 1);
  unsigned long long t_in = 0, t_st = 0, t_lv = 0;
  if (a.dbg) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_in));
  StageRegs SR;
  stage_load(a.s_Tp, a.s_Toff, root, n, SR, tbuf, a.sub_tb);
  prefetch_top(a.s_Tp, a.s_Toff, a.s_top, a.s_top_lptr[a.s_top_nlev]);
  build_sublist(a.s_level, a.s_tsize, root, L, a.s_rank, a.s_son0, a.s_son1, a.s_parent, a.s_Toff);
  pdl_trigger();
  pdl_wait();  // the leaves' coefficients (k_mv_leaf_fwd)
  if (n > 1) {
    // the leaves' coefficients (k_mv_leaf_fwd) -- the subtree's xhat rows are contiguous in global
    const double* xg = a.s_xh + (size_t)root * rcap;
    for (int i = warp; i < n; i += nw) {
      if (L.s0[i] >= 0) continue;
      const int k = L.rk[i];
      for (int j = lane; j < k; j += 32) xs[(size_t)i * rcap + j] = __ldcg(xg + (size_t)i * rcap + j);
    }
    stage_store(SR, tbuf);
    const bool staged = SR.ok;
    const int64_t tb = staged ? SR.tb : 0;
    const double* tp = staged ? tbuf : a.s_Tp;
    __syncthreads();
    if (a.dbg) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_st));
    for (int l = L.nlev - 2; l >= 0; --l) {
      for (int q = L.ptr[l] + warp; q < L.ptr[l + 1]; q += nw) {
        const int i = L.cl[q] - root;
        if (L.s0[i] >= 0) fwd_internal(L, i, L.s0[i] - root, L.s1[i] - root, lane, xs, rcap, tp, tb);
      }
      __syncthreads();
    }
    if (a.dbg) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_lv));
    // publish the internal clusters' coefficients (the couplings read them from global)
    for (int i = warp; i < n; i += nw) {
      if (L.s0[i] < 0) continue;
      const int k = L.rk[i];
      for (int j = lane; j < k; j += 32) a.s_xh[(size_t)(root + i) * rcap + j] = xs[(size_t)i * rcap + j];
    }
  }
  // the last subtree to finish computes the clusters above the subtrees, bottom-up
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    // [0] counts the published subtrees of all products (never reset): this product's go from
    // (epoch - 1) n_roots to epoch n_roots
    last = (unsigned)atomicAdd(a.s_cnt, 1) == a.s_epoch * (unsigned)gridDim.x - 1u;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (a.dbg && threadIdx.x == 0) {
    a.dbg[2] = t_in;
    a.dbg[3] = t_st;
    a.dbg[4] = t_lv;
  }
  stamp(a, 5);
  // structure of the top clusters into shared memory (reusing the sublist arrays; <= SUB_NC - 1 of
  // them: one per pair of subtrees at most), then the levels read only coefficients and transfers
  const int ntop = a.s_top_lptr[a.s_top_nlev];
  int* t_id = L.cl;      // cluster
  int* t_k = L.rk;       // its rank
  int* t_c0 = L.s0;      // sons
  int* t_c1 = L.s1;
  int* t_k0 = L.par;     // sons' ranks
  int* t_k1 = L.cnt;     // (64 + 65 ints: cnt and ptr are adjacent)
  long long* t_o0 = L.to;
  long long* t_o1 = reinterpret_cast<long long*>(tbuf);
  const bool cached = ntop <= SUB_NC && ntop <= 64 + 65;
  if (cached) {
    for (int i = threadIdx.x; i < ntop; i += SUBT) {
      const int c = a.s_top[i];
      const int c0 = a.s_son0[c], c1 = a.s_son1[c];
      t_id[i] = c;
      t_k[i] = a.s_rank[c];
      t_c0[i] = c0;
      t_c1[i] = c1;
      t_k0[i] = a.s_rank[c0];
      t_k1[i] = a.s_rank[c1];
      t_o0[i] = a.s_Toff[c0];
      t_o1[i] = a.s_Toff[c1];
    }
    __syncthreads();
  }
  const unsigned long long pol = el_policy();
  for (int l = a.s_top_nlev - 1; l >= 0; --l) {
    const int qb = a.s_top_lptr[l], qe = a.s_top_lptr[l + 1];
    for (int i = qb + warp; i < qe; i += nw) {
      int s, k, sc0, sc1, sk0, sk1;
      long long o0, o1;
      if (cached) {
        s = t_id[i], k = t_k[i], sc0 = t_c0[i], sc1 = t_c1[i], sk0 = t_k0[i], sk1 = t_k1[i], o0 = t_o0[i], o1 = t_o1[i];
      } else {
        s = a.s_top[i], k = a.s_rank[s], sc0 = a.s_son0[s], sc1 = a.s_son1[s];
        sk0 = a.s_rank[sc0], sk1 = a.s_rank[sc1], o0 = a.s_Toff[sc0], o1 = a.s_Toff[sc1];
      }
      if (k == 0) continue;
      // sons' coefficients through L2 (written by other CTAs / other warps of this one): one
      // coalesced load per son, then broadcast by shuffles
      const double* F0 = a.s_Tp + o0;
      const double* F1 = a.s_Tp + o1;
      const double* x0 = a.s_xh + (size_t)sc0 * rcap;
      const double* x1 = a.s_xh + (size_t)sc1 * rcap;
      const double xa0 = lane < sk0 ? __ldcg(x0 + lane) : 0.0, xa1 = lane + 32 < sk0 ? __ldcg(x0 + lane + 32) : 0.0;
      const double xb0 = lane < sk1 ? __ldcg(x1 + lane) : 0.0, xb1 = lane + 32 < sk1 ? __ldcg(x1 + lane + 32) : 0.0;
      for (int j0 = 0; j0 < k; j0 += 32) {
        const int j = j0 + lane;
        double acc = 0.0;
        for (int q = 0; q < sk0; ++q) {
          const double xq = __shfl_sync(FULL, q < 32 ? xa0 : xa1, q & 31);
          if (j < k) acc += ld_el(F0 + j + (size_t)q * k, pol) * xq;
        }
        for (int q = 0; q < sk1; ++q) {
          const double xq = __shfl_sync(FULL, q < 32 ? xb0 : xb1, q & 31);
          if (j < k) acc += ld_el(F1 + j + (size_t)q * k, pol) * xq;
        }
        if (j < k) a.s_xh[(size_t)s * rcap + j] = acc;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {  // every forward coefficient is final: [1] = epoch
    __threadfence();
    atomicExch(a.s_cnt + 1, (int)a.s_epoch);
  }
  stamp(a, 6);
}

// ---- couplings of one destination cluster from the packed S --------------------------------------
// Descriptors of up to 32 blocks of row(t) are loaded at once (lane q: slot, offset, partner, its
// rank), then the blocks are walked with shuffles, so the loads of consecutive blocks do not wait
// for one another.  No transpose: lane = (row i, column group g), G = 32 / k_t groups share the
// columns of a block; the groups are summed by a fixed sequence of shuffles.  Transpose: lane =
// output column, each lane walks its contiguous column.
template <bool TR>
__device__ __forceinline__ void mv_couple_packed(const MvArgs& a, int t, int lane) {
  const int rcap = a.rcap;
  const int kt = a.d_rank[t];
  if (kt == 0) return;
  const int qb = a.d_bptr[t], qe = a.d_bptr[t + 1];
  const int G = TR ? 1 : (kt >= 32 ? 1 : 32 / kt);
  const int ig = TR ? lane : (kt >= 32 ? lane : lane % kt);
  const int g = TR ? 0 : (kt >= 32 ? 0 : lane / kt);
  const bool act = TR ? true : g < G;
  const unsigned long long pol = el_policy();
  double acc0 = 0.0, acc1 = 0.0;
  for (int base = qb; base < qe; base += 32) {
    const int cnt = qe - base < 32 ? qe - base : 32;
    int d_s = 0, d_k = 0;
    long long d_off = 0;
    if (lane < cnt) {  // one 16-byte descriptor per block (built with the packed copies)
      const longlong2 dd = __ldg(reinterpret_cast<const longlong2*>(a.desc + base + lane));
      d_off = dd.x;
      d_s = (int)(dd.y & 0xffffffffll);
      d_k = (int)(dd.y >> 32);
      // all blocks of the batch in flight at once: the walk below then hits L2
      const char* pb = reinterpret_cast<const char*>(a.Sp + d_off);
      const int bytes = kt * d_k * 8;
      for (int o = 0; o < bytes; o += 128) asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(pb + o));
    }
    if (!TR) {
      // S_b: k_t x k_s, ld k_t; out[i] += sum_j S[i + j k_t] xhat_s[j].  Group g takes the blocks
      // b = g, g + G, ...: G blocks are in flight per warp (a block's columns are independent loads)
      const int rounds = (cnt + G - 1) / G;
      for (int it = 0; it < rounds; ++it) {
        const int b = it * G + g;
        const bool ok = act && b < cnt;
        const int bb = ok ? b : 0;
        const int s = __shfl_sync(FULL, d_s, bb);
        const int ks = __shfl_sync(FULL, d_k, bb);
        const long long off = __shfl_sync(FULL, d_off, bb);
        if (ok && ks > 0) {
          const double* Sa = a.Sp + off;
          const double* xs = a.s_xh + (size_t)s * rcap;
#pragma unroll 4
          for (int j = 0; j < ks; ++j) {
            const double xj = __ldcg(xs + j);
            if (ig < kt) acc0 = fma(ld_el(Sa + ig + (size_t)j * kt, pol), xj, acc0);
            if (ig + 32 < kt) acc1 = fma(ld_el(Sa + ig + 32 + (size_t)j * kt, pol), xj, acc1);
          }
        }
      }
    } else {
      for (int b = 0; b < cnt; ++b) {
        const int s = __shfl_sync(FULL, d_s, b);
        const int ks = __shfl_sync(FULL, d_k, b);
        const long long off = __shfl_sync(FULL, d_off, b);
        if (ks == 0) continue;
        const double* Sa = a.Sp + off;
        const double* xs = a.s_xh + (size_t)s * rcap;
        // S_b: k_s x k_t (rows = the partner's rank), ld k_s; out[j] += sum_i S[i + j k_s] xhat[i]
        for (int q = 0; q < 2; ++q) {
          const int j = lane + 32 * q;
          if (j < kt) {
            const double* Sj = Sa + (size_t)j * ks;
            double v = 0.0;
            for (int i = 0; i < ks; ++i) v = fma(ld_el(Sj + i, pol), __ldcg(xs + i), v);
            if (q) acc1 += v;
            else acc0 += v;
          }
        }
      }
    }
  }
  if (!TR && G > 1) {  // sum the column groups: lane i collects lanes i + g k_t, g = 1 .. G-1
    double v = acc0;
    for (int gg = 1; gg < G; ++gg) {
      const double o = __shfl_sync(FULL, acc0, (ig + gg * kt) & 31);
      if (g == 0) v += o;
    }
    acc0 = v;
  }
  if (g == 0 || TR) {
    if (ig < kt) a.d_xh[(size_t)t * rcap + ig] = acc0;
    if (ig + 32 < kt) a.d_xh[(size_t)t * rcap + ig + 32] = acc1;
  }
}

// couplings, then the last CTA carries yhat down through the top clusters
__global__ void __launch_bounds__(256, 4) k_mv_couple_top(const __grid_constant__ MvArgs a) {
  __shared__ int last;
  const int lane = threadIdx.x & 31;
  const int w = (int)(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5));
  if (blockIdx.x == 0) stamp(a, 7);
  prefetch_top(a.d_Tp, a.d_Toff, a.d_top, a.d_top_lptr[a.d_top_nlev]);
  pdl_trigger();
  // The forward coefficients: a cluster below the top levels has only partners inside the
  // subtrees, final once every subtree CTA of k_mv_fwd_sub has published ([0] == s_nroots); the
  // others wait for the top pass of its last CTA ([1]).  So the bulk of the couplings overlaps
  // the top forward pass.  (k_mv_fwd_sub's CTAs are all resident before this kernel may start --
  // programmatic launch after their trigger, or a plain launch after their end: no deadlock.)
  if (w < a.d_nclusters) {
    const bool low = a.same_tree && a.d_level[w] >= a.s_top_nlev;
    const volatile int* flag = a.s_cnt + (low ? 0 : 1);
    const unsigned need = low ? a.s_epoch * (unsigned)a.s_nroots : a.s_epoch;
    while ((int)((unsigned)*flag - need) < 0) __nanosleep(200);
    __threadfence();
    if (a.transpose) mv_couple_packed<true>(a, w, lane);
    else mv_couple_packed<false>(a, w, lane);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(a.d_cnt, 1) == (int)gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  stamp(a, 8);
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5, rcap = a.rcap;
  const unsigned long long pol = el_policy();
  for (int l = 1; l < a.d_top_nlev; ++l) {  // the root (level 0) keeps its coupling sum
    for (int i = a.d_top_lptr[l] + warp; i < a.d_top_lptr[l + 1]; i += nw) {
      const int c = a.d_top[i];
      const int p = a.d_parent[c], kc = a.d_rank[c];
      if (p < 0 || kc == 0) continue;
      const int kp = a.d_rank[p];
      const double* E = a.d_Tp + a.d_Toff[c];
      const double* yp = a.d_xh + (size_t)p * rcap;
      double* yc = a.d_xh + (size_t)c * rcap;
      const double yp0 = lane < kp ? __ldcg(yp + lane) : 0.0, yp1 = lane + 32 < kp ? __ldcg(yp + lane + 32) : 0.0;
      for (int r0 = 0; r0 < kc; r0 += 32) {
        const int r = r0 + lane;
        double v = r < kc ? __ldcg(yc + r) : 0.0;
        for (int j = 0; j < kp; ++j) {
          const double yj = __shfl_sync(FULL, j < 32 ? yp0 : yp1, j & 31);
          if (r < kc) v += ld_el(E + r + (size_t)j * kc, pol) * yj;
        }
        if (r < kc) yc[r] = v;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) a.d_cnt[0] = 0;
  stamp(a, 9);
}

// backward transform inside one destination subtree (root first), in shared memory
__global__ void __launch_bounds__(SUBT, 1) k_mv_bwd_sub(const __grid_constant__ MvArgs a) {
  extern __shared__ __align__(16) double dsm[];
  __shared__ SubList L;
  const int rcap = a.rcap;
  double* ys = dsm;  // SUB_NC x rcap: yc / yhat of the subtree's clusters
  double* tbuf = dsm + (size_t)SUB_NC * rcap;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = SUBT / 32;
  const int root = a.d_roots[blockIdx.x], n = a.d_tsize[root];
  if (blockIdx.x == 0) stamp(a, 10);
  StageRegs SR;
  stage_load(a.d_Tp, a.d_Toff, root, n, SR, tbuf, a.sub_tb);
  // the root's father (a top cluster, final in global memory) and the root's own transfer matrix
  const int pr = a.d_parent[root];
  const int kpr = pr >= 0 ? a.d_rank[pr] : 0;
  build_sublist(a.d_level, a.d_tsize, root, L, a.d_rank, a.d_son0, a.d_son1, a.d_parent, a.d_Toff);
  pdl_wait();  // the couplings and the top clusters' yhat (k_mv_couple_top)
  double ypr0 = 0.0, ypr1 = 0.0;
  if (warp == 0 && pr >= 0) {
    const double* yp = a.d_xh + (size_t)pr * rcap;
    ypr0 = lane < kpr ? __ldcg(yp + lane) : 0.0;
    ypr1 = lane + 32 < kpr ? __ldcg(yp + lane + 32) : 0.0;
  }
  double* yg = a.d_xh + (size_t)root * rcap;
  for (int i = warp; i < n; i += nw) {
    const int k = L.rk[i];
    for (int j = lane; j < k; j += 32) ys[(size_t)i * rcap + j] = __ldcg(yg + (size_t)i * rcap + j);
  }
  stage_store(SR, tbuf);
  const bool staged = SR.ok;
  const int64_t tb = staged ? SR.tb : 0;
  const double* tp = staged ? tbuf : a.d_Tp;
  __syncthreads();
  const unsigned long long pol = el_policy();
  if (warp == 0 && pr >= 0) {
    const int kc = L.rk[0];
    const double* E = a.d_Tp + L.to[0];
    for (int r0 = 0; r0 < kc; r0 += 32) {
      const int r = r0 + lane;
      double v = r < kc ? ys[r] : 0.0;
      for (int j = 0; j < kpr; ++j) {
        const double yj = __shfl_sync(FULL, j < 32 ? ypr0 : ypr1, j & 31);
        if (r < kc) v += ld_el(E + r + (size_t)j * kc, pol) * yj;
      }
      if (r < kc) ys[r] = v;
    }
  }
  __syncthreads();
  for (int l = 1; l < L.nlev; ++l) {
    for (int q = L.ptr[l] + warp; q < L.ptr[l + 1]; q += nw) {
      const int i = L.cl[q] - root;
      bwd_cluster(L, i, L.par[i] - root, lane, ys, rcap, tp, tb);
    }
    __syncthreads();
  }
  // the leaves' yhat back to global for k_mv_leaf_bwd
  for (int i = warp; i < n; i += nw) {
    if (L.s0[i] >= 0) continue;
    const int k = L.rk[i];
    for (int j = lane; j < k; j += 32) yg[(size_t)i * rcap + j] = ys[(size_t)i * rcap + j];
  }
  if (blockIdx.x == 0) stamp(a, 11);
}

// y|t += alpha V_t yhat_t, warp per destination leaf
__global__ void __launch_bounds__(256) k_mv_leaf_bwd(const __grid_constant__ MvArgs a) {
  const int w = (int)(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5));
  if (blockIdx.x == 0) stamp(a, 12);
  if (w >= a.d_nleaves) return;
  const int lane = threadIdx.x & 31;
  const int t = a.d_leaves[w];
  const int rcap = a.rcap, lmax = a.lmax;
  const int kt = a.d_rank[t];
  if (kt == 0) return;
  const int lo = a.d_lo[t], m = a.d_hi[t] - lo;
  const double* V = a.d_leafb + (size_t)a.d_leafidx[t] * lmax * rcap;
  const double* yh = a.d_xh + (size_t)t * rcap;
  const double yl0 = lane < kt ? __ldcg(yh + lane) : 0.0;
  const double yl1 = lane + 32 < kt ? __ldcg(yh + lane + 32) : 0.0;
  double a0 = 0.0, a1 = 0.0;
  const unsigned long long pol = el_policy();
#pragma unroll 4
  for (int j = 0; j < kt; ++j) {
    const double yj = __shfl_sync(FULL, j < 32 ? yl0 : yl1, j & 31);
    if (lane < m) a0 += ld_el(V + lane + (size_t)j * lmax, pol) * yj;
    if (lane + 32 < m) a1 += ld_el(V + lane + 32 + (size_t)j * lmax, pol) * yj;
  }
  if (lane < m) {
    double* yo = a.y + a.d_perm[lo + lane];
    *yo = __ldcg(yo) + a.alpha * a0;
  }
  if (lane + 32 < m) {
    double* yo = a.y + a.d_perm[lo + lane + 32];
    *yo = __ldcg(yo) + a.alpha * a1;
  }
}

// ---- packing ------------------------------------------------------------------------------------
struct PackArgs {
  const int32_t *adm_t, *adm_s, *rrank, *crank, *rparent, *cparent;
  const double *S, *rtr, *ctr;
  double *Sp, *rTp, *cTp, *rTpT, *cTpT;
  const int64_t *Soff, *rToff, *cToff;
  int nadm, nr, nc, rcap;
};

__global__ void __launch_bounds__(256) k_mv_pack(const PackArgs p) {
  const int w = (int)(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5));
  const int lane = threadIdx.x & 31;
  const double* src;
  double* dst;
  double* dstT = nullptr;
  int rows, cols;
  if (w < p.nadm) {
    rows = p.rrank[p.adm_t[w]];
    cols = p.crank[p.adm_s[w]];
    src = p.S + (size_t)w * p.rcap * p.rcap;
    dst = p.Sp + p.Soff[w];
  } else if (w < p.nadm + p.nr) {
    const int c = w - p.nadm;
    rows = p.rrank[c];
    cols = p.rparent[c] >= 0 ? p.rrank[p.rparent[c]] : 0;
    src = p.rtr + (size_t)c * p.rcap * p.rcap;
    dst = p.rTp + p.rToff[c];
    dstT = p.rTpT + p.rToff[c];
  } else if (w < p.nadm + p.nr + p.nc) {
    const int c = w - p.nadm - p.nr;
    rows = p.crank[c];
    cols = p.cparent[c] >= 0 ? p.crank[p.cparent[c]] : 0;
    src = p.ctr + (size_t)c * p.rcap * p.rcap;
    dst = p.cTp + p.cToff[c];
    dstT = p.cTpT + p.cToff[c];
  } else {
    return;
  }
  for (int e = lane; e < rows * cols; e += 32) dst[e] = src[(e % rows) + (size_t)(e / rows) * p.rcap];
  if (dstT)  // (cols x rows, ld cols)
    for (int e = lane; e < rows * cols; e += 32) dstT[e] = src[(e / cols) + (size_t)(e % cols) * p.rcap];
}

inline int cdiv(long long a, long long b) { return (int)((a + b - 1) / b); }

}  // namespace

// (Re)build the packed copies of Z's couplings and transfer matrices at its current ranks.  Runs
// once per matrix version (any mutating call bumps h2_mat_::version): ranks to the host (one
// stream synchronisation), offsets by prefix sums, one packing kernel.
static cudaError_t ensure_packed(h2_mat_* Z, cudaStream_t st) {
  MvPack& K = Z->mvpack;
  if (K.version == Z->version) return cudaSuccess;
  const MatDev& M = Z->d;
  cudaError_t e;
  const int nr = M.row.nclusters, nc = M.col.nclusters;
  std::vector<int32_t> kr(nr), kc(nc);
  if ((e = cudaMemcpyAsync(kr.data(), M.row.rank, sizeof(int32_t) * nr, cudaMemcpyDeviceToHost, st))) return e;
  if ((e = cudaMemcpyAsync(kc.data(), M.col.rank, sizeof(int32_t) * nc, cudaMemcpyDeviceToHost, st))) return e;
  if ((e = cudaStreamSynchronize(st))) return e;
  const h2_btree_* B = Z->bt;
  auto even = [](int64_t v) { return (v + 1) & ~int64_t(1); };  // 16-byte aligned packed matrices
  std::vector<int64_t> so(M.nadm + 1, 0), ro(nr + 1, 0), co(nc + 1, 0);
  for (int a = 0; a < M.nadm; ++a) {
    const int b = Z->adm_blk[a];
    so[a + 1] = so[a] + even((int64_t)kr[B->t[b]] * kc[B->s[b]]);
  }
  for (int c = 0; c < nr; ++c) {
    const int p = B->rt->parent[c];
    ro[c + 1] = ro[c] + (p >= 0 ? even((int64_t)kr[c] * kr[p]) : 0);
  }
  for (int c = 0; c < nc; ++c) {
    const int p = B->ct->parent[c];
    co[c + 1] = co[c] + (p >= 0 ? even((int64_t)kc[c] * kc[p]) : 0);
  }
  auto grow = [&](double** p, size_t* cap, size_t need) -> cudaError_t {
    if (*cap >= need && *p) return cudaSuccess;
    if (*p) cudaFree(*p);
    *p = nullptr;
    *cap = need + need / 8 + 1024;
    return cudaMalloc((void**)p, *cap * sizeof(double));
  };
  if ((e = grow(&K.Sp, &K.capS, (size_t)so[M.nadm]))) return e;
  if ((e = grow(&K.Tp[0], &K.capT[0], (size_t)ro[nr]))) return e;
  if ((e = grow(&K.Tp[1], &K.capT[1], (size_t)co[nc]))) return e;
  if ((e = grow(&K.TpT[0], &K.capTT[0], (size_t)ro[nr]))) return e;
  if ((e = grow(&K.TpT[1], &K.capTT[1], (size_t)co[nc]))) return e;
  if (!K.Soff) {
    if ((e = cudaMalloc((void**)&K.desc[0], sizeof(MvPack::Desc) * (M.nadm + 1)))) return e;
    if ((e = cudaMalloc((void**)&K.desc[1], sizeof(MvPack::Desc) * (M.nadm + 1)))) return e;
    if ((e = cudaMalloc((void**)&K.Soff, sizeof(int64_t) * (M.nadm + 1)))) return e;
    if ((e = cudaMalloc((void**)&K.Toff[0], sizeof(int64_t) * (nr + 1)))) return e;
    if ((e = cudaMalloc((void**)&K.Toff[1], sizeof(int64_t) * (nc + 1)))) return e;
  }
  // block descriptors in the order of DevSide::bidx (slots counting-sorted by cluster, setup_side)
  std::vector<MvPack::Desc> dsc[2];
  for (int side = 0; side < 2; ++side) {
    const int ncl = side ? nc : nr;
    std::vector<int32_t> ptr(ncl + 1, 0);
    for (int a = 0; a < M.nadm; ++a) ptr[(side ? B->s[Z->adm_blk[a]] : B->t[Z->adm_blk[a]]) + 1]++;
    for (int c = 0; c < ncl; ++c) ptr[c + 1] += ptr[c];
    dsc[side].resize(M.nadm + 1);
    for (int a = 0; a < M.nadm; ++a) {
      const int b = Z->adm_blk[a];
      const int own = side ? B->s[b] : B->t[b], other = side ? B->t[b] : B->s[b];
      dsc[side][ptr[own]++] = MvPack::Desc{so[a], other, side ? kr[other] : kc[other]};
    }
    if ((e = cudaMemcpyAsync(K.desc[side], dsc[side].data(), sizeof(MvPack::Desc) * M.nadm, cudaMemcpyHostToDevice, st)))
      return e;
  }
  if ((e = cudaMemcpyAsync(K.Soff, so.data(), sizeof(int64_t) * (M.nadm + 1), cudaMemcpyHostToDevice, st))) return e;
  if ((e = cudaMemcpyAsync(K.Toff[0], ro.data(), sizeof(int64_t) * (nr + 1), cudaMemcpyHostToDevice, st))) return e;
  if ((e = cudaMemcpyAsync(K.Toff[1], co.data(), sizeof(int64_t) * (nc + 1), cudaMemcpyHostToDevice, st))) return e;
  PackArgs p;
  p.adm_t = M.adm_t;
  p.adm_s = M.adm_s;
  p.rrank = M.row.rank;
  p.crank = M.col.rank;
  p.rparent = M.row.parent;
  p.cparent = M.col.parent;
  p.S = M.S;
  p.rtr = M.row.tr;
  p.ctr = M.col.tr;
  p.Sp = K.Sp;
  p.rTp = K.Tp[0];
  p.cTp = K.Tp[1];
  p.rTpT = K.TpT[0];
  p.cTpT = K.TpT[1];
  p.Soff = K.Soff;
  p.rToff = K.Toff[0];
  p.cToff = K.Toff[1];
  p.nadm = M.nadm;
  p.nr = nr;
  p.nc = nc;
  p.rcap = M.rcap;
  H2_LAUNCH(K_MV, st, k_mv_pack<<<cdiv((long long)M.nadm + nr + nc, 8), 256, 0, st>>>(p));
  if ((e = cudaStreamSynchronize(st))) return e;  // the host offset vectors go out of scope
  K.version = Z->version;
  return cudaGetLastError();
}

void free_mvpack(h2_mat_* Z) {
  MvPack& K = Z->mvpack;
  for (void* p : {(void*)K.Sp, (void*)K.Tp[0], (void*)K.Tp[1], (void*)K.Soff, (void*)K.Toff[0], (void*)K.Toff[1],
                  (void*)K.desc[0], (void*)K.desc[1], (void*)K.TpT[0], (void*)K.TpT[1]})
    if (p) cudaFree(p);
  K = MvPack();
}

cudaError_t launch_matvec(const h2_mat_* Zc, int transpose, double alpha, const double* x, double beta, double* y,
                          cudaStream_t st) {
  h2_mat_* Z = const_cast<h2_mat_*>(Zc);
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
  a.d_cnt = dst.mv_cnt + 2;  // [0], [1]: this side's forward epoch counters; [2]: the couplings' arrival counter
  a.dbg = nullptr;
  a.desc = nullptr;
  a.Sp = nullptr;
  a.Soff = nullptr;
  a.s_Tp = a.d_Tp = nullptr;
  a.s_Toff = a.d_Toff = nullptr;
  // the far field contributes only if some row and some column basis may have a non-zero rank
  const bool far = std::find(Z->nzr.begin(), Z->nzr.end(), 1) != Z->nzr.end() &&
                   std::find(Z->nzc.begin(), Z->nzc.end(), 1) != Z->nzc.end();
  if (!far) {
    H2_LAUNCH(K_MV, st, (transpose ? k_matvec_near_t : k_matvec_near)<<<cdiv(dst.nleaves, 8), 256, 0, st>>>(a));
    return cudaGetLastError();
  }
  cudaError_t e;
  if ((e = ensure_packed(Z, st))) return e;
  const MvPack& K = Z->mvpack;
  a.Sp = K.Sp;
  a.Soff = K.Soff;
  a.s_Tp = K.TpT[transpose ? 0 : 1];  // the forward transform applies F^T: transposed copies
  a.s_Toff = K.Toff[transpose ? 0 : 1];
  a.d_Tp = K.Tp[transpose ? 1 : 0];
  a.d_Toff = K.Toff[transpose ? 1 : 0];
  a.desc = K.desc[transpose ? 1 : 0];
  // the far-field chain (latency-bound) runs on a high-priority side stream next to the nearfield
  // kernel (the bulk of the bytes) on the caller's stream; the leaf backward transform adds
  // V_t yhat_t after both
  static cudaStream_t s2 = nullptr;
  static cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  static int nsm = 148;
  if (!s2) {
    int lo = 0, hi = 0, dev = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    // H2_MV_PRIO=equal: the far-field stream at the caller's (lowest) priority (A/B)
    const bool equal = getenv("H2_MV_PRIO") && std::string(getenv("H2_MV_PRIO")) == "equal";
    if ((e = cudaStreamCreateWithPriority(&s2, cudaStreamNonBlocking, equal ? lo : hi))) return e;
    if ((e = cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming))) return e;
    if ((e = cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming))) return e;
    if ((e = cudaFuncSetAttribute(k_mv_fwd_sub, cudaFuncAttributeMaxDynamicSharedMemorySize, SUB_SMEM))) return e;
    if ((e = cudaFuncSetAttribute(k_mv_bwd_sub, cudaFuncAttributeMaxDynamicSharedMemorySize, SUB_SMEM))) return e;
    if ((e = cudaFuncSetAttribute(k_matvec_near_s, cudaFuncAttributeMaxDynamicSharedMemorySize, NEAR_W * 16384))) return e;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  const size_t smem = SUB_SMEM;
  a.sub_tb = (int)(SUB_SMEM / sizeof(double)) - SUB_NC * M.rcap;
  a.s_nroots = src.n_mv_roots;
  a.s_epoch = ++const_cast<DevSide&>(src).mv_epoch;
  a.same_tree = Z->bt->rt == Z->bt->ct ? 1 : 0;
  // timing diagnostics (tools): H2_MV_PART=1 far field only, 2 nearfield only, 3 / 4 / 5: the far
  // field up to the forward transform / the couplings / the subtree backward transform (y is then
  // incomplete); H2_MV_NEARGRID: CTAs per SM of the nearfield kernel (default 2)
  static const int part = getenv("H2_MV_PART") ? atoi(getenv("H2_MV_PART")) : 0;
  static const int near_per_sm = getenv("H2_MV_NEARGRID") ? atoi(getenv("H2_MV_NEARGRID")) : 0;
  const int near_grid = near_per_sm > 0 ? std::min(cdiv(dst.nleaves, 8), near_per_sm * nsm) : cdiv(dst.nleaves, 8);
  // the staged nearfield kernel (one small CTA per SM) only on request (H2_MV_NEAR_STAGED=1):
  // measured 101 us alone against 66 us for the register-panel kernel at C2 (4 warps x 2 slots per
  // SM do not cover the load latency; more slots do not fit beside the far field's shared memory)
  static const bool staged_on = getenv("H2_MV_NEAR_STAGED") && atoi(getenv("H2_MV_NEAR_STAGED")) != 0;
  const bool near_staged = staged_on && !transpose && M.lmax == 32;
  if (part == 2) {
    if (near_staged) {
      H2_LAUNCH(K_MV, st, k_matvec_near_s<<<std::min(nsm, cdiv(dst.nleaves, NEAR_W)), NEAR_W * 32, NEAR_W * 16384, st>>>(a));
    } else {
      H2_LAUNCH(K_MV, st, (transpose ? k_matvec_near_t : k_matvec_near)<<<near_grid, 256, 0, st>>>(a));
    }
    return cudaGetLastError();
  }
  static unsigned long long* dbg = nullptr;
  static const bool dbg_on = getenv("H2_MV_DBG") != nullptr;
  if (dbg_on && !dbg) cudaMalloc((void**)&dbg, 16 * sizeof(unsigned long long));
  a.dbg = dbg;
  cudaStream_t sf = part == 0 ? s2 : st;  // the far-field chain
  static const bool near_first = getenv("H2_MV_ORDER") && std::string(getenv("H2_MV_ORDER")) == "near_first";  // A/B
  if (part == 0) {
    if ((e = cudaEventRecord(ev_fork, st))) return e;
    if ((e = cudaStreamWaitEvent(s2, ev_fork, 0))) return e;
    if (near_first) {
      if (near_staged) {
        H2_LAUNCH(K_MV, st, k_matvec_near_s<<<std::min(nsm, cdiv(dst.nleaves, NEAR_W)), NEAR_W * 32, NEAR_W * 16384, st>>>(a));
      } else {
        H2_LAUNCH(K_MV, st, (transpose ? k_matvec_near_t : k_matvec_near)<<<near_grid, 256, 0, st>>>(a));
      }
    }
  }
  // the dependent kernels of the chain are launched programmatically (their prologues -- staging,
  // sublists, prefetches -- overlap the predecessor's tail); H2_MV_NOPDL=1: plain launches (A/B)
  static const bool pdl = !(getenv("H2_MV_NOPDL") && atoi(getenv("H2_MV_NOPDL")) != 0);
  auto launch_dep = [&](auto kern, int grid, int block, size_t sm) -> cudaError_t {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = sf;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, a);
  };
  // a failed launch would leave the forward epoch counters out of step with the host's epoch (the
  // next product's coupling warps would wait forever): start over from zero
  auto fail = [&](cudaError_t err) -> cudaError_t {
    cudaStreamSynchronize(sf);
    cudaMemset(src.mv_cnt, 0, 2 * sizeof(int32_t));
    const_cast<DevSide&>(src).mv_epoch = 0;
    return err;
  };
  H2_LAUNCH(K_MV, sf, k_mv_leaf_fwd<<<cdiv(src.nleaves, 8), 256, 0, sf>>>(a));
  H2_LAUNCH(K_MV, sf, e = launch_dep(k_mv_fwd_sub, src.n_mv_roots, SUBT, smem));
  if (e) return fail(e);
  if (part == 3) return cudaGetLastError();
  H2_LAUNCH(K_MV, sf, e = launch_dep(k_mv_couple_top, cdiv(dst.nclusters, 8), 256, 0));
  if (e) return fail(e);
  if (part == 4) return cudaGetLastError();
  H2_LAUNCH(K_MV, sf, e = launch_dep(k_mv_bwd_sub, dst.n_mv_roots, SUBT, smem));
  if (e) return fail(e);
  if (part == 5) return cudaGetLastError();
  if (part == 0) {
    if ((e = cudaEventRecord(ev_join, s2))) return e;
    if (near_first) {
    } else if (near_staged) {
      H2_LAUNCH(K_MV, st, k_matvec_near_s<<<std::min(nsm, cdiv(dst.nleaves, NEAR_W)), NEAR_W * 32, NEAR_W * 16384, st>>>(a));
    } else {
      H2_LAUNCH(K_MV, st, (transpose ? k_matvec_near_t : k_matvec_near)<<<near_grid, 256, 0, st>>>(a));
    }
    if ((e = cudaStreamWaitEvent(st, ev_join, 0))) return e;
  }
  H2_LAUNCH(K_MV, st, k_mv_leaf_bwd<<<cdiv(dst.nleaves, 8), 256, 0, st>>>(a));
  if (dbg_on) {  // diagnostic: phase stamps of this product, relative to the first kernel's start (us)
    unsigned long long h[16];
    cudaDeviceSynchronize();
    cudaMemcpy(h, dbg, sizeof(h), cudaMemcpyDeviceToHost);
    static int calls = 0;
    if (++calls % 16 == 0) {
      const char* nm[13] = {"leaf_fwd start", "fwd_sub start", "last CTA in", "last CTA staged", "last CTA levels done",
                            "last detected", "top fwd done", "couple start", "couple last detected", "top bwd done",
                            "bwd_sub start", "bwd_sub cta0 end", "leaf_bwd start"};
      fprintf(stderr, "[H2_MV_DBG]");
      for (int i = 0; i < 13; ++i) fprintf(stderr, " %s %.1f;", nm[i], (double)((long long)h[i] - (long long)h[0]) / 1e3);
      fprintf(stderr, "\n");
    }
  }
  return cudaGetLastError();
}

}  // namespace h2
