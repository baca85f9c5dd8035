// H^2 matrix-vector product y = alpha op(Z) x + beta y ([BO10 Thm 3.42]).
//
//   forward transform   xhat_s = W_s^T x|s (leaves),  xhat_s = sum_{s'} F_{s'}^T xhat_{s'}   bottom-up
//   couplings           yhat_t = sum_{s in row(t)} S_(t,s) xhat_s
//   backward transform  yhat_{t'} += E_{t'} yhat_t  top-down; leaves y|t = V_t yhat_t
//   nearfield           y|t += sum_{b=(t,s) inadmissible} N_b x|s
//
// ONE launch, no grid-wide barrier: every warp takes a ticket (atomic counter, so tickets are
// handed out in order and a warp only ever waits on lower tickets, which are resident).
//   tickets [0, #leaves)            forward transform of a source leaf, then climb: the second
//                                   of two siblings to finish (arrival counter) computes the
//                                   father, up to the root, whose completion publishes "xhat done"
//   tickets [#leaves, +#clusters)   destination clusters in level (BFS) order: a leaf first streams
//                                   its nearfield tiles (independent of the transforms), then
//                                   waits for "xhat done" (couplings) and for its father's yhat
//                                   ready flag (backward transform), and writes y|t in original order.
// Ready flags hold the call's epoch (no reset); arrival counters and the ticket counter are reset
// by their last user.  Bytes are dominated by the nearfield tiles: lanes own rows,
// every tile column is one coalesced 256 B load, 8 columns in flight per lane, streaming loads.
#include <cuda_runtime.h>

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
  const int32_t *d_bfs, *d_lo, *d_hi, *d_leafidx, *d_rank, *d_parent, *d_son0, *d_bptr, *d_bidx;
  const int64_t* d_perm;
  const double *d_leafb, *d_tr;
  double* d_xh;
  int32_t* d_ready;
  int d_nclusters;
  // blocks
  const int32_t* partner;  // admissible slot -> source cluster
  const double* S;
  const int32_t *nptr, *nidx, *npartner;
  const double* N;
  int lmax, rcap, transpose, epoch;
  int32_t* ctl;  // [0] ticket counter, [1] "xhat done" (epoch)
  const double* x;
  double* y;
  double alpha, beta;
};

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ int ld_acquire(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int32_t* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// all lanes: wait until *flag == epoch, then every lane has acquired it
__device__ __forceinline__ void wait_epoch(const int32_t* flag, int epoch, int lane) {
  if (lane == 0)
    while (ld_acquire(flag) != epoch) __nanosleep(32);
  __syncwarp();
  (void)ld_acquire(flag);
}

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
    __threadfence();
    __syncwarp();
    if (p < 0) {
      if (lane == 0) st_release(a.ctl + 1, a.epoch);
      return;
    }
    int old = 0;
    if (lane == 0) old = atomicAdd(a.s_arrive + p, 1);
    old = __shfl_sync(FULL, old, 0);
    if (old == 0) return;  // first of the two sons: the sibling finishes the father
    if (lane == 0) a.s_arrive[p] = 0;
    __threadfence();
    const int kp = a.s_rank[p];
    for (int j = lane; j < kp; j += 32) {
      double acc = 0.0;
      for (int q = 0; q < 2; ++q) {
        const int c = q ? a.s_son1[p] : a.s_son0[p];
        const int kc = a.s_rank[c];
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
      const int j1 = ms < 32 ? ms : 32;
#pragma unroll 8
      for (int j = 0; j < j1; ++j) {
        const double xj = __shfl_sync(FULL, xs0, j);
        if (lane < m) a0 += __ldcs(Na + lane + (size_t)j * lmax) * xj;
        if (lane + 32 < m) a1 += __ldcs(Na + lane + 32 + (size_t)j * lmax) * xj;
      }
#pragma unroll 8
      for (int j = 32; j < ms; ++j) {
        const double xj = __shfl_sync(FULL, xs1, j - 32);
        if (lane < m) a0 += __ldcs(Na + lane + (size_t)j * lmax) * xj;
        if (lane + 32 < m) a1 += __ldcs(Na + lane + 32 + (size_t)j * lmax) * xj;
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

// ---- couplings + backward transform of one destination cluster (+ leaf output) ------------------
__device__ void mv_down(const MvArgs& a, int t, int lane) {
  const int rcap = a.rcap, lmax = a.lmax;
  const bool leaf = a.d_son0[t] < 0;
  double a0 = 0.0, a1 = 0.0;
  int lo = 0, m = 0;
  if (leaf) {
    lo = a.d_lo[t];
    m = a.d_hi[t] - lo;
    mv_near(a, t, m, lane, a0, a1);
  }
  const int kt = a.d_rank[t];
  double y0 = 0.0, y1 = 0.0;  // yhat_t rows lane, lane + 32
  const int p = a.d_parent[t];
  const int kp = p >= 0 ? a.d_rank[p] : 0;
  const int qb = a.d_bptr[t], qe = a.d_bptr[t + 1];
  if (kt > 0 && qe > qb) {
    wait_epoch(a.ctl + 1, a.epoch, lane);
    for (int q = qb; q < qe; ++q) {
      const int slot = a.d_bidx[q];
      const int s = a.partner[slot];
      const int ks = a.s_rank[s];
      const double* Sa = a.S + (size_t)slot * rcap * rcap;
      const double* xs = a.s_xh + (size_t)s * rcap;
      if (!a.transpose) {
#pragma unroll 4
        for (int j = 0; j < ks; ++j) {
          const double xj = __ldcg(xs + j);
          if (lane < kt) y0 += Sa[lane + (size_t)j * rcap] * xj;
          if (lane + 32 < kt) y1 += Sa[lane + 32 + (size_t)j * rcap] * xj;
        }
      } else {
#pragma unroll 4
        for (int j = 0; j < ks; ++j) {
          const double xj = __ldcg(xs + j);
          if (lane < kt) y0 += Sa[j + (size_t)lane * rcap] * xj;
          if (lane + 32 < kt) y1 += Sa[j + (size_t)(lane + 32) * rcap] * xj;
        }
      }
    }
  }
  if (kt > 0 && kp > 0) {
    wait_epoch(a.d_ready + p, a.epoch, lane);
    const double* E = a.d_tr + (size_t)t * rcap * rcap;
    const double* yp = a.d_xh + (size_t)p * rcap;
#pragma unroll 4
    for (int j = 0; j < kp; ++j) {
      const double yj = __ldcg(yp + j);
      if (lane < kt) y0 += E[lane + (size_t)j * rcap] * yj;
      if (lane + 32 < kt) y1 += E[lane + 32 + (size_t)j * rcap] * yj;
    }
  }
  if (!leaf) {
    if (lane < kt) a.d_xh[(size_t)t * rcap + lane] = y0;
    if (lane + 32 < kt) a.d_xh[(size_t)t * rcap + lane + 32] = y1;
    __threadfence();
    __syncwarp();
    if (lane == 0) st_release(a.d_ready + t, a.epoch);
    return;
  }
  const double* V = a.d_leafb + (size_t)a.d_leafidx[t] * lmax * rcap;
  for (int j = 0; j < kt; ++j) {
    const double yj = __shfl_sync(FULL, j < 32 ? y0 : y1, j & 31);
    if (lane < m) a0 += V[lane + (size_t)j * lmax] * yj;
    if (lane + 32 < m) a1 += V[lane + 32 + (size_t)j * lmax] * yj;
  }
  if (lane < m) {
    const int64_t o = a.d_perm[lo + lane];
    a.y[o] = a.beta == 0.0 ? a.alpha * a0 : a.alpha * a0 + a.beta * a.y[o];
  }
  if (lane + 32 < m) {
    const int64_t o = a.d_perm[lo + lane + 32];
    a.y[o] = a.beta == 0.0 ? a.alpha * a1 : a.alpha * a1 + a.beta * a.y[o];
  }
}

__global__ void __launch_bounds__(256) k_matvec(const __grid_constant__ MvArgs a) {
  const int lane = threadIdx.x & 31;
  const int total = a.s_nleaves + a.d_nclusters;
  if ((int)(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) >= total) return;  // exactly `total` tickets
  int ticket = 0;
  if (lane == 0) {
    ticket = atomicAdd(a.ctl, 1);
    if (ticket == total - 1) atomicExch(a.ctl, 0);  // every other ticket is already taken
  }
  ticket = __shfl_sync(FULL, ticket, 0);
  if (ticket < a.s_nleaves) mv_up(a, a.s_leaves[ticket], lane);
  else mv_down(a, a.d_bfs[ticket - a.s_nleaves], lane);
}

inline int cdiv(long long a, long long b) { return (int)((a + b - 1) / b); }

}  // namespace

cudaError_t launch_matvec(const h2_mat_* Z, int transpose, double alpha, const double* x, double beta, double* y,
                          cudaStream_t st) {
  const MatDev& M = Z->d;
  const DevSide& src = transpose ? M.row : M.col;  // basis applied to x
  const DevSide& dst = transpose ? M.col : M.row;  // basis producing y
  if (++Z->mv_epoch <= 0) Z->mv_epoch = 1;
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
  a.d_ready = dst.mvsync + dst.nclusters;
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
  a.epoch = Z->mv_epoch;
  a.ctl = dst.mvsync + 2 * dst.nclusters;
  a.x = x;
  a.y = y;
  a.alpha = alpha;
  a.beta = beta;
  const long long total = (long long)src.nleaves + dst.nclusters;
  H2_LAUNCH(K_MV, st, k_matvec<<<cdiv(total, 8), 256, 0, st>>>(a));
  return cudaGetLastError();
}

}  // namespace h2
