// h2_solve: x <- (L L^T)^{-1} x (Cholesky) or x <- (L U)^{-1} x (LR) with the H^2 factor
// (block forward / backward substitution; the factor as PCG
// preconditioner).
//
// The recursion lsolve(t) = lsolve(t1); b|t2 -= L|_{t2 x t1} z|t1; lsolve(t2) is unrolled into one
// sweep over the leaves in processing order (ascending for L, descending for U and L^T), run by a
// single CTA:
//   enter     for every destination cluster whose first leaf (in processing order) this is, top
//             down: yt_c = yh_c + E_c yt_father (yh_c has received every far-field contribution
//             of the blocks (c, s), s solved earlier, at that point);
//   residual  r = b|t - sum over the leaf's off-diagonal nearfield tiles N z|s - V_t yt_t
//             (tiles split over the 8 warps, the diagonal tile staged in shared memory meanwhile);
//   diagonal  z|t = T^{-1} r with the leaf tile (lower, unit lower, upper or lower transposed),
//             one warp per right-hand side, lanes own rows;
//   complete  for every source cluster whose last leaf this is, bottom up: xh_c = W_c^T z|c
//             (leaf) or sum F_c'^T xh_c' (sons), then push: yh_d += S_(d,c) xh_c for the
//             admissible blocks of c whose destination d is processed later (one warp per block).
// The factorization's own substitutions (rfs/lfs with H^2 right-hand sides) keep the recursive
// form of h2_factor.cpp; this sweep serves dense right-hand sides (h2_solve, h2_pcg).
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "h2_internal.h"
#include "h2_prof.h"

namespace h2 {
namespace {

constexpr int SNT = 256;  // one CTA
constexpr int NRC = 8;    // right-hand sides per sweep
constexpr int TLD = 65;   // shared-memory leading dimension of the staged diagonal tile

enum SweepMode { SW_L = 0, SW_U = 1, SW_LT = 2 };

struct SweepArgs {
  SolveSched S;
  int mode, unit, nr, rcap, lmax;
  int64_t n;
  const int32_t *lo, *hi, *parent;
  // source side: forward transform of the solved part; destination side: backward transform
  const int32_t *s_rank, *s_son0, *s_son1, *s_leafidx;
  const double *s_leafb, *s_tr;
  const int32_t *d_rank, *d_leafidx;
  const double *d_leafb, *d_tr;
  const double *Sc, *N;
  double* B;                  // n x nr (ld n), tree order: right-hand side in, solution out
  double* prof;               // profiling: cycles per sweep phase (h2_profile_ops slots 40..44) or null
  double *xh, *yh, *yt;       // [cluster][nr][rcap]
};

constexpr int WLD = 64;    // leading dimension of the staged leaf basis W_t
constexpr size_t SWEEP_SMEM = sizeof(double) * (8 * 64 * NRC + 64 * NRC + 64 * TLD + 64 + WLD * 48 + 48 * NRC);

__global__ void __launch_bounds__(SNT, 1) k_sweep(const __grid_constant__ SweepArgs a) {
  extern __shared__ double smem[];
  double* part = smem;                // [warp][row][rhs]
  double* r = part + 8 * 64 * NRC;    // [rhs][row]
  double* T = r + 64 * NRC;           // diagonal tile, ld TLD
  double* invd = T + 64 * TLD;
  double* Ws = invd + 64;             // W_t of the current leaf (m x k_t, ld WLD), staged during the solve
  double* xs = Ws + WLD * 48;         // xhat of the cluster being completed (k_c x nr), for its pushes
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nr = a.nr, rc = a.rcap, lmax = a.lmax;
  const int64_t n = a.n;
  const bool tr = a.mode == SW_LT;
  long long ph[5] = {0, 0, 0, 0, 0}, c_prev = clock64();
  auto tick = [&](int i) {
    if (a.prof && tid == 0) {
      const long long c = clock64();
      ph[i] += c - c_prev;
      c_prev = c;
    }
  };
  for (int p = 0; p < a.S.nl; ++p) {
    const int t = a.S.order[p];
    const int lo = a.lo[t], m = a.hi[t] - lo;
    // ---- enter: yt_c = yh_c + E_c yt_father, top-down -- by warp 0 alone (a dependent chain of
    // small products, __syncwarp between clusters) while warps 1..7 stage the diagonal tile and
    // take the nearfield tiles: the two are independent
    const int q_en0 = a.S.enter_ptr[p], q_en1 = a.S.enter_ptr[p + 1];
    const bool split = q_en1 > q_en0;
    double b0[NRC], b1[NRC];  // warp 0: b|t, loaded first (consumed after the enter chain)
#pragma unroll
    for (int v = 0; v < NRC; ++v) {
      b0[v] = (warp == 0 && split && v < nr && lane < m) ? a.B[lo + lane + (size_t)v * n] : 0.0;
      b1[v] = (warp == 0 && split && v < nr && lane + 32 < m) ? a.B[lo + lane + 32 + (size_t)v * n] : 0.0;
    }
    if (warp == 0) {
      for (int q = q_en0; q < q_en1; ++q) {
        const int c = a.S.enter[q];
        const int kc = a.d_rank[c];
        const int par = a.parent[c];
        const int kp = par >= 0 ? a.d_rank[par] : 0;
        const double* E = a.d_tr + (size_t)c * rc * rc;
        for (int e = lane; e < kc * nr; e += 32) {
          const int i = e % kc, v = e / kc;
          double acc = a.yh[((size_t)c * nr + v) * rc + i];
          const double* yp = a.yt + ((size_t)par * nr + v) * rc;
          for (int j = 0; j < kp; ++j) acc += E[i + (size_t)j * rc] * yp[j];
          a.yt[((size_t)c * nr + v) * rc + i] = acc;
        }
        __syncwarp();
      }
    }
    // ---- stage the diagonal tile; nearfield partial sums, warp w takes tiles w, w + nw, ...
    const int w0 = split ? 1 : 0, nw = 8 - w0;
    if (tid >= 32 * w0) {
      const int t0 = tid - 32 * w0, nth = SNT - 32 * w0;
      const double* D = a.N + (size_t)a.S.diag[p] * lmax * lmax;
      for (int e = t0; e < m * m; e += nth) T[(e % m) + (e / m) * TLD] = D[(e % m) + (size_t)(e / m) * lmax];
      for (int i = t0; i < m; i += nth) invd[i] = 1.0 / D[i + (size_t)i * lmax];
    }
    double acc0[NRC], acc1[NRC];
#pragma unroll
    for (int v = 0; v < NRC; ++v) acc0[v] = acc1[v] = 0.0;
    if (warp == 0 && split) {
      // the far-field part of the leaf, V_t yt_t (t entered last, just above), minus b|t as warp 0's
      // share of the partial sums: the residual below only adds up shared memory
      const int kt = a.d_rank[t];
      const double* V = a.d_leafb + (size_t)a.d_leafidx[t] * lmax * rc;
#pragma unroll
      for (int v = 0; v < NRC; ++v) {
        acc0[v] = -b0[v];
        acc1[v] = -b1[v];
        if (v < nr) {
          const double* y = a.yt + ((size_t)t * nr + v) * rc;
          for (int j = 0; j < kt; ++j) {
            const double yj = y[j];
            if (lane < m) acc0[v] += V[lane + (size_t)j * lmax] * yj;
            if (lane + 32 < m) acc1[v] += V[lane + 32 + (size_t)j * lmax] * yj;
          }
        }
      }
    }
    for (int q = a.S.near_ptr[p] + warp - w0; warp >= w0 && q < a.S.near_ptr[p + 1]; q += nw) {
      const int slot = a.S.near_slot[q], s = a.S.near_src[q];
      const int los = a.lo[s], ms = a.hi[s] - los;
      const double* Tq = a.N + (size_t)slot * lmax * lmax;
      double z0[NRC], z1[NRC];
#pragma unroll
      for (int v = 0; v < NRC; ++v) {
        z0[v] = (v < nr && lane < ms) ? a.B[los + lane + (size_t)v * n] : 0.0;
        z1[v] = (v < nr && lane + 32 < ms) ? a.B[los + lane + 32 + (size_t)v * n] : 0.0;
      }
      // lane i takes its row of the (transposed) tile into registers, 32 columns at a time, all
      // loads issued before the FMAs
      for (int j0 = 0; j0 < ms; j0 += 32) {
        const int jn = ms - j0 < 32 ? ms - j0 : 32;
        for (int r0 = 0; r0 < m; r0 += 32) {
          const int i = r0 + lane;
          double tv[32];
#pragma unroll
          for (int j = 0; j < 32; ++j)
            tv[j] = (i < m && j < jn) ? (tr ? Tq[j0 + j + (size_t)i * lmax] : Tq[i + (size_t)(j0 + j) * lmax]) : 0.0;
#pragma unroll
          for (int v = 0; v < NRC; ++v) {
            if (v < nr) {
              double acc = 0.0;
#pragma unroll
              for (int j = 0; j < 32; ++j) acc += tv[j] * __shfl_sync(0xffffffffu, j0 ? z1[v] : z0[v], j);
              if (r0) acc1[v] += acc;
              else acc0[v] += acc;
            }
          }
        }
      }
    }
#pragma unroll
    for (int v = 0; v < NRC; ++v) {
      part[(warp * 64 + lane) * NRC + v] = acc0[v];
      part[(warp * 64 + lane + 32) * NRC + v] = acc1[v];
    }
    __syncthreads();
    tick(0);  // enter || diagonal tile + nearfield
    // ---- residual r = b|t - sum part - V_t yt_t
    if (split) {  // -b|t and V_t yt_t are in warp 0's partial sums: shared memory only
      for (int e = tid; e < m * nr; e += SNT) {
        const int i = e % m, v = e / m;
        double acc = 0.0;
        for (int w = 0; w < 8; ++w) acc -= part[(w * 64 + i) * NRC + v];
        r[v * 64 + i] = acc;
      }
    } else {  // (never: every leaf enters at its own step)
      const int kt = a.d_rank[t];
      const double* V = a.d_leafb + (size_t)a.d_leafidx[t] * lmax * rc;
      for (int e = tid; e < m * nr; e += SNT) {
        const int i = e % m, v = e / m;
        double acc = a.B[lo + i + (size_t)v * n];
        for (int w = 0; w < 8; ++w) acc -= part[(w * 64 + i) * NRC + v];
        const double* y = a.yt + ((size_t)t * nr + v) * rc;
        for (int j = 0; j < kt; ++j) acc -= V[i + (size_t)j * lmax] * y[j];
        r[v * 64 + i] = acc;
      }
    }
    __syncthreads();
    tick(1);  // residual
    // ---- diagonal tile solve, warp v = right-hand side v, lanes own rows (lane, lane + 32); the
    // other warps stage the leaf's source basis W_t for the forward transform that follows
    const int kts = a.s_rank[t];
    const bool wst = kts <= 48 && nr < 8;
    if (warp >= nr && wst) {
      const double* W = a.s_leafb + (size_t)a.s_leafidx[t] * lmax * rc;
      for (int e = tid - 32 * nr; e < m * kts; e += SNT - 32 * nr) Ws[(e % m) + (e / m) * WLD] = W[(e % m) + (size_t)(e / m) * lmax];
    }
    if (warp < nr && m <= 32) {  // operator row of this lane in registers: one shuffle + FMA per step
      const bool fwd = a.mode == SW_L, unit = a.unit != 0;
      double av[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) av[j] = (lane < m && j < m) ? (tr ? T[j + lane * TLD] : T[lane + j * TLD]) : 0.0;
      double x = lane < m ? r[warp * 64 + lane] : 0.0;
      const double d = lane < m ? invd[lane] : 0.0;
      if (fwd) {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (j < m) {
            const double z = __shfl_sync(0xffffffffu, unit ? x : x * d, j);
            x = lane == j ? z : (lane > j ? x - av[j] * z : x);
          }
      } else {
#pragma unroll
        for (int j = 31; j >= 0; --j)
          if (j < m) {
            const double z = __shfl_sync(0xffffffffu, x * d, j);
            x = lane == j ? z : (lane < j ? x - av[j] * z : x);
          }
      }
      if (lane < m) r[warp * 64 + lane] = x;
    } else if (warp < nr) {
      double x0 = lane < m ? r[warp * 64 + lane] : 0.0, x1 = lane + 32 < m ? r[warp * 64 + lane + 32] : 0.0;
      const double d0 = lane < m ? invd[lane] : 0.0, d1 = lane + 32 < m ? invd[lane + 32] : 0.0;
      const bool fwd = a.mode == SW_L, unit = a.unit != 0;
      for (int s = 0; s < m; ++s) {
        const int j = fwd ? s : m - 1 - s;
        const double own = j < 32 ? (unit ? x0 : x0 * d0) : (unit ? x1 : x1 * d1);
        const double z = __shfl_sync(0xffffffffu, own, j & 31);
        // A[i][j] of the operator: L / U by rows (T[i + j ld]), L^T by columns (T[j + i ld])
        const double a0 = tr ? T[j + lane * TLD] : T[lane + j * TLD];
        const double a1 = tr ? T[j + (lane + 32) * TLD] : T[lane + 32 + j * TLD];
        const bool pend0 = fwd ? lane > j : lane < j, pend1 = fwd ? lane + 32 > j : lane + 32 < j;
        if (lane == j) x0 = z;
        else if (pend0 && lane < m) x0 -= a0 * z;
        if (lane + 32 == j) x1 = z;
        else if (pend1 && lane + 32 < m) x1 -= a1 * z;
      }
      if (lane < m) r[warp * 64 + lane] = x0;
      if (lane + 32 < m) r[warp * 64 + lane + 32] = x1;
    }
    __syncthreads();
    for (int e = tid; e < m * nr; e += SNT) a.B[lo + (e % m) + (size_t)(e / m) * n] = r[(e / m) * 64 + (e % m)];
    __syncthreads();
    tick(2);  // diagonal solve + store
    // ---- completed source clusters, bottom-up: forward transform, then push into destinations
    for (int q = a.S.done_ptr[p]; q < a.S.done_ptr[p + 1]; ++q) {
      const int c = a.S.done[q];
      const int kc = a.s_rank[c];
      if (kc == 0) continue;  // uniform: every thread reads the same rank
      const bool leaf = a.s_son0[c] < 0;
      for (int e = tid; e < kc * nr; e += SNT) {
        const int j = e % kc, v = e / kc;
        double acc = 0.0;
        if (leaf && wst) {  // c == t, W_t staged in shared memory
          for (int i = 0; i < m; ++i) acc += Ws[i + j * WLD] * r[v * 64 + i];
        } else if (leaf) {
          const double* W = a.s_leafb + (size_t)a.s_leafidx[c] * lmax * rc;
          for (int i = 0; i < m; ++i) acc += W[i + (size_t)j * lmax] * r[v * 64 + i];
        } else {
          for (int h = 0; h < 2; ++h) {
            const int ch = h ? a.s_son1[c] : a.s_son0[c];
            const int kh = a.s_rank[ch];
            const double* F = a.s_tr + (size_t)ch * rc * rc;
            const double* xc = a.xh + ((size_t)ch * nr + v) * rc;
            for (int i = 0; i < kh; ++i) acc += F[i + (size_t)j * rc] * xc[i];
          }
        }
        a.xh[((size_t)c * nr + v) * rc + j] = acc;
        if (kc <= 48) xs[j + v * 48] = acc;
      }
      __syncthreads();
      for (int b = a.S.push_ptr[c] + warp; b < a.S.push_ptr[c + 1]; b += 8) {
        const int slot = a.S.push_slot[b], d = a.S.push_dst[b];
        const int kd = a.d_rank[d];
        const double* Sa = a.Sc + (size_t)slot * rc * rc;
        for (int i = lane; i < kd; i += 32)
          for (int v = 0; v < nr; ++v) {
            const double* x = kc <= 48 ? xs + v * 48 : a.xh + ((size_t)c * nr + v) * rc;
            double acc = 0.0;
            for (int j = 0; j < kc; ++j) acc += (tr ? Sa[j + (size_t)i * rc] : Sa[i + (size_t)j * rc]) * x[j];
            a.yh[((size_t)d * nr + v) * rc + i] += acc;
          }
      }
      __syncthreads();
    }
    tick(3);  // forward transforms + pushes of the completed clusters
  }
  if (a.prof && tid == 0)
    for (int i = 0; i < 4; ++i) {
      atomicAdd(a.prof + 4 * K_COUNT + 32 + 2 * (40 + i), (double)ph[i]);
      atomicAdd(a.prof + 4 * K_COUNT + 32 + 2 * (40 + i) + 1, (double)a.S.nl);
    }
}

__global__ void k_gather_cols(const double* __restrict__ x, int64_t ldx, const int64_t* __restrict__ perm,
                              double* __restrict__ B, int64_t n, int nr) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n * nr) B[e] = x[perm[e % n] + (e / n) * ldx];
}
__global__ void k_scatter_cols(double* __restrict__ x, int64_t ldx, const int64_t* __restrict__ perm,
                               const double* __restrict__ B, int64_t n, int nr) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n * nr) x[perm[e % n] + (e / n) * ldx] = B[e];
}

// ---- host: schedules -----------------------------------------------------------------------------
template <class T>
cudaError_t upload(h2_mat_* Z, T** p, const std::vector<T>& v) {
  *p = nullptr;
  if (v.empty()) return cudaSuccess;
  cudaError_t e = cudaMalloc(p, sizeof(T) * v.size());
  if (e != cudaSuccess) return e;
  Z->allocs.push_back(*p);
  return cudaMemcpy(*p, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice);
}

cudaError_t build_sched(h2_mat_* Z, int mode) {
  SolveSched& S = Z->sched[mode];
  if (S.built) return cudaSuccess;
  const h2_btree_* B = Z->bt;
  const h2_tree_* R = B->rt;
  const int nl = (int)R->leaves.size(), nc = R->nclusters;
  const bool desc = mode != SW_L;
  std::vector<int32_t> order(R->leaves.begin(), R->leaves.end());
  if (desc) std::reverse(order.begin(), order.end());
  std::vector<int32_t> pos(nc, -1);
  for (int p = 0; p < nl; ++p) pos[order[p]] = p;
  // first / last leaf position of every cluster in processing order
  std::vector<int32_t> first(nc, nl), last(nc, -1);
  for (int p = 0; p < nl; ++p)
    for (int c = order[p]; c >= 0; c = R->parent[c]) {
      first[c] = std::min(first[c], p);
      last[c] = std::max(last[c], p);
    }
  auto before = [&](int s, int t) { return first[s] < first[t]; };  // disjoint clusters
  // nearfield: off-diagonal tiles per position, diagonal slot
  std::vector<std::vector<std::pair<int, int>>> near(nl);
  std::vector<int32_t> diag(nl, -1);
  for (size_t a = 0; a < Z->inad_blk.size(); ++a) {
    const int b = Z->inad_blk[a], bt = B->t[b], bs = B->s[b];
    if (bt == bs) {
      diag[pos[bt]] = (int32_t)a;
      continue;
    }
    if (mode == SW_LT) {  // L^T: block (bt, bs) of L acts on row bs, source bt
      if (before(bt, bs)) near[pos[bs]].push_back({(int)a, bt});
    } else {  // L / U: block (bt, bs) acts on row bt, source bs
      if (before(bs, bt)) near[pos[bt]].push_back({(int)a, bs});
    }
  }
  std::vector<int32_t> near_ptr(nl + 1, 0), near_slot, near_src;
  for (int p = 0; p < nl; ++p) {
    for (auto& pr : near[p]) {
      near_slot.push_back(pr.first);
      near_src.push_back(pr.second);
    }
    near_ptr[p + 1] = (int32_t)near_slot.size();
  }
  // enter (top-down) and done (bottom-up) lists
  std::vector<int32_t> enter_ptr(nl + 1, 0), enter, done_ptr(nl + 1, 0), done;
  for (int p = 0; p < nl; ++p) {
    std::vector<int32_t> up;
    for (int c = order[p]; c >= 0 && first[c] == p; c = R->parent[c]) up.push_back(c);
    for (auto it = up.rbegin(); it != up.rend(); ++it) enter.push_back(*it);
    enter_ptr[p + 1] = (int32_t)enter.size();
    for (int c = order[p]; c >= 0 && last[c] == p; c = R->parent[c]) done.push_back(c);
    done_ptr[p + 1] = (int32_t)done.size();
  }
  // push lists: per source cluster c, admissible blocks whose destination is processed later
  std::vector<std::vector<std::pair<int, int>>> push(nc);
  for (size_t a = 0; a < Z->adm_blk.size(); ++a) {
    const int b = Z->adm_blk[a], bt = B->t[b], bs = B->s[b];
    if (mode == SW_LT) {
      if (before(bt, bs)) push[bt].push_back({(int)a, bs});  // source = row cluster, destination = column
    } else {
      if (before(bs, bt)) push[bs].push_back({(int)a, bt});
    }
  }
  std::vector<int32_t> push_ptr(nc + 1, 0), push_slot, push_dst;
  for (int c = 0; c < nc; ++c) {
    for (auto& pr : push[c]) {
      push_slot.push_back(pr.first);
      push_dst.push_back(pr.second);
    }
    push_ptr[c + 1] = (int32_t)push_slot.size();
  }
  cudaError_t e;
  if ((e = upload(Z, &S.order, order)) || (e = upload(Z, &S.diag, diag)) || (e = upload(Z, &S.near_ptr, near_ptr)) ||
      (e = upload(Z, &S.near_slot, near_slot)) || (e = upload(Z, &S.near_src, near_src)) ||
      (e = upload(Z, &S.enter_ptr, enter_ptr)) || (e = upload(Z, &S.enter, enter)) ||
      (e = upload(Z, &S.done_ptr, done_ptr)) || (e = upload(Z, &S.done, done)) ||
      (e = upload(Z, &S.push_ptr, push_ptr)) || (e = upload(Z, &S.push_slot, push_slot)) ||
      (e = upload(Z, &S.push_dst, push_dst)))
    return e;
  S.nl = nl;
  S.built = 1;
  return cudaSuccess;
}

inline int cdiv(long long a, long long b) { return (int)((a + b - 1) / b); }

}  // namespace

cudaError_t solve_factored(h2_mat_* F, double* x, int nrhs, int64_t ldx, cudaStream_t st) {
  const MatDev& M = F->d;
  const h2_tree_* R = F->bt->rt;
  const int64_t n = R->n;
  const bool chol = F->factored == 1;
  static bool attr = false;
  cudaError_t e;
  if (!attr) {
    if ((e = cudaFuncSetAttribute(k_sweep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SWEEP_SMEM))) return e;
    attr = true;
  }
  const int modes[2] = {SW_L, chol ? SW_LT : SW_U};
  for (int mo : modes)
    if ((e = build_sched(F, mo))) return e;
  const int nr_max = std::min(nrhs, NRC);
  const size_t cw = (size_t)R->nclusters * M.rcap * nr_max;
  double* w = nullptr;
  if ((e = cudaMallocAsync(&w, sizeof(double) * ((size_t)n * nr_max + 3 * cw), st))) return e;
  double *Bt = w, *xh = w + (size_t)n * nr_max, *yh = xh + cw, *yt = yh + cw;
  for (int v0 = 0; v0 < nrhs; v0 += NRC) {
    const int nr = std::min(NRC, nrhs - v0);
    H2_LAUNCH(K_SOLVE, st,
              k_gather_cols<<<cdiv(n * nr, 256), 256, 0, st>>>(x + v0 * ldx, ldx, M.row.perm, Bt, n, nr));
    for (int mo : modes) {
      SweepArgs a;
      a.prof = prof_dev();
      a.S = F->sched[mo];
      a.mode = mo;
      a.unit = (mo == SW_L && !chol) ? 1 : 0;
      a.nr = nr;
      a.rcap = M.rcap;
      a.lmax = M.lmax;
      a.n = n;
      a.lo = M.row.lo;
      a.hi = M.row.hi;
      a.parent = M.row.parent;
      const DevSide& src = mo == SW_LT ? M.row : M.col;
      const DevSide& dst = mo == SW_LT ? M.col : M.row;
      a.s_rank = src.rank;
      a.s_son0 = src.son0;
      a.s_son1 = src.son1;
      a.s_leafidx = src.leafidx;
      a.s_leafb = src.leafb;
      a.s_tr = src.tr;
      a.d_rank = dst.rank;
      a.d_leafidx = dst.leafidx;
      a.d_leafb = dst.leafb;
      a.d_tr = dst.tr;
      a.Sc = M.S;
      a.N = M.N;
      a.B = Bt;
      a.xh = xh;
      a.yh = yh;
      a.yt = yt;
      if ((e = cudaMemsetAsync(yh, 0, sizeof(double) * cw, st))) break;
      H2_LAUNCH(K_SOLVE, st, k_sweep<<<1, SNT, SWEEP_SMEM, st>>>(a));
    }
    H2_LAUNCH(K_SOLVE, st,
              k_scatter_cols<<<cdiv(n * nr, 256), 256, 0, st>>>(x + v0 * ldx, ldx, M.row.perm, Bt, n, nr));
  }
  cudaFreeAsync(w, st);
  if (e) return e;
  return cudaGetLastError();
}

}  // namespace h2
