// Host side of the B200 H^2 library: structure (cluster/block trees), device storage, C ABI.
//
// Structure work is exact: integer-valued coordinates give exact box predicates,
// and this file is compiled with -ffp-contract=off.  All FP64 arithmetic of the method runs in
// the CUDA kernels (h2_matvec.cu, h2_update.cu); the host only builds index structures and
// schedules launches.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "exec.h"
#include "h2_internal.h"

using namespace h2;

static thread_local std::string g_last_error;

void h2::set_error(const std::string& msg) { g_last_error = msg; }

extern "C" const char* h2_last_error(void) { return g_last_error.c_str(); }

#define H2_FAIL(code, msg)  \
  do {                      \
    h2::set_error(msg);     \
    return code;            \
  } while (0)
// calls that read or launch on their own must not interleave with an open batch recording
#define H2_NO_BATCH(name)                                                                          \
  do {                                                                                             \
    if (h2::batch_open()) H2_FAIL(H2_ERR_ARG, name ": not allowed inside h2_batch_begin/h2_batch_end"); \
  } while (0)

#define CUDA_TRY(expr)                                                                      \
  do {                                                                                      \
    cudaError_t e_ = (expr);                                                                \
    if (e_ != cudaSuccess) {                                                                \
      h2::set_error(std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " #expr); \
      return e_ == cudaErrorMemoryAllocation ? H2_ERR_NOMEM : H2_ERR_CUDA;                  \
    }                                                                                       \
  } while (0)

// ------------------------------------------------------------------------------------------------
// Cluster tree (binary P:331-332), geometric bisection per SURVEY R2.
// ------------------------------------------------------------------------------------------------
// gptr/gidx: nullptr (geometric bisection) or the symmetrised coupling graph in CSR form ->
// domain-decomposition clustering (DESIGN reading own-11): a DOMAIN
// cluster with more than 2 leaf_size points is bisected geometrically into (left, right), the
// interface gamma = the points of `right` coupled to `left`, dom2 = right minus gamma, and the
// ternary split of [GRKRLE05a] becomes t -> (interior -> (dom1, dom2), gamma): nested dissection
// order.  ddpair[p] marks clusters whose two sons are decoupled domains.
static h2_status build_cluster_tree(const double* pts, int64_t n, int32_t dim, int32_t leaf_size,
                                    const int64_t* gptr, const int32_t* gidx, h2_tree* out) {
  if (!out) H2_FAIL(H2_ERR_ARG, "h2_cluster_tree: out is NULL");
  *out = nullptr;
  if (!pts || n <= 0 || dim < 1 || dim > 3 || leaf_size < 1)
    H2_FAIL(H2_ERR_ARG, "h2_cluster_tree: need pts != NULL, n > 0, 1 <= dim <= 3, leaf_size >= 1");
  for (int64_t i = 0; i < n * dim; ++i)
    if (!std::isfinite(pts[i])) H2_FAIL(H2_ERR_NONFINITE, "h2_cluster_tree: non-finite coordinate");
  h2_tree_* T = new (std::nothrow) h2_tree_();
  if (!T) H2_FAIL(H2_ERR_NOMEM, "h2_cluster_tree: host allocation failed");
  T->n = n;
  T->dim = dim;
  T->leaf = leaf_size;
  T->perm.resize(n);
  std::vector<int64_t> idx(n);
  for (int64_t i = 0; i < n; ++i) idx[i] = i;
  std::vector<char> in_left(gptr ? n : 0, 0);
  enum { DOMAIN = 0, INTERFACE = 1 };

  // presplit: the interior cluster of a DD split (its sons are the two domains, given)
  std::function<int(std::vector<int64_t>&, int64_t, int, int, int, std::vector<int64_t>*, std::vector<int64_t>*)> build =
      [&](std::vector<int64_t>& ids, int64_t start, int par, int lev, int kind, std::vector<int64_t>* pre0,
          std::vector<int64_t>* pre1) -> int {
    int cid = (int)T->lo.size();
    T->ddpair.push_back(0);
    T->lo.push_back((int32_t)start);
    T->hi.push_back((int32_t)(start + (int64_t)ids.size()));
    T->son0.push_back(-1);
    T->son1.push_back(-1);
    T->parent.push_back(par);
    T->level.push_back(lev);
    double bmin[3], bmax[3];
    for (int d = 0; d < dim; ++d) {
      bmin[d] = pts[ids[0] * dim + d];
      bmax[d] = bmin[d];
    }
    for (int64_t q : ids)
      for (int d = 0; d < dim; ++d) {
        bmin[d] = std::min(bmin[d], pts[q * dim + d]);
        bmax[d] = std::max(bmax[d], pts[q * dim + d]);
      }
    for (int d = 0; d < dim; ++d) {
      T->bmin.push_back(bmin[d]);
      T->bmax.push_back(bmax[d]);
    }
    auto make_leaf = [&]() {
      for (size_t i = 0; i < ids.size(); ++i) T->perm[start + (int64_t)i] = ids[i];
      return cid;
    };
    if (pre0) {
      T->ddpair[cid] = 1;
      ids.clear();
      ids.shrink_to_fit();
      const int64_t nl = (int64_t)pre0->size();
      int c0 = build(*pre0, start, cid, lev + 1, DOMAIN, nullptr, nullptr);
      int c1 = build(*pre1, start + nl, cid, lev + 1, DOMAIN, nullptr, nullptr);
      T->son0[cid] = c0;
      T->son1[cid] = c1;
      return cid;
    }
    if ((int64_t)ids.size() <= leaf_size) return make_leaf();
    int ax = 0;
    for (int d = 1; d < dim; ++d)
      if (bmax[d] - bmin[d] > bmax[ax] - bmin[ax]) ax = d;  // strict: lowest axis on ties
    const double twomid = bmin[ax] + bmax[ax];
    std::vector<int64_t> left, right;
    for (int64_t q : ids) (2.0 * pts[q * dim + ax] < twomid ? left : right).push_back(q);
    if (left.empty() || right.empty()) return make_leaf();
    const bool dd = gptr && kind == DOMAIN && (int64_t)ids.size() > 2 * (int64_t)leaf_size;
    ids.clear();
    ids.shrink_to_fit();
    int64_t nl = (int64_t)left.size();
    int c0, c1;
    if (dd) {
      for (int64_t q : left) in_left[q] = 1;
      std::vector<int64_t> gam, d2;
      for (int64_t q : right) {
        bool coupled = false;
        for (int64_t e = gptr[q]; e < gptr[q + 1] && !coupled; ++e) coupled = in_left[gidx[e]] != 0;
        (coupled ? gam : d2).push_back(q);
      }
      for (int64_t q : left) in_left[q] = 0;
      if (gam.empty()) {  // the halves are not coupled at all
        T->ddpair[cid] = 1;
        c0 = build(left, start, cid, lev + 1, DOMAIN, nullptr, nullptr);
        c1 = build(right, start + nl, cid, lev + 1, DOMAIN, nullptr, nullptr);
      } else if (d2.empty() || nl + (int64_t)d2.size() <= leaf_size) {  // no decoupling gained
        c0 = build(left, start, cid, lev + 1, DOMAIN, nullptr, nullptr);
        c1 = build(right, start + nl, cid, lev + 1, d2.empty() ? INTERFACE : DOMAIN, nullptr, nullptr);
      } else {
        right.clear();
        right.shrink_to_fit();
        std::vector<int64_t> inner(left);
        inner.insert(inner.end(), d2.begin(), d2.end());
        const int64_t ni = (int64_t)inner.size();
        c0 = build(inner, start, cid, lev + 1, DOMAIN, &left, &d2);
        c1 = build(gam, start + ni, cid, lev + 1, INTERFACE, nullptr, nullptr);
      }
    } else {
      c0 = build(left, start, cid, lev + 1, kind, nullptr, nullptr);
      c1 = build(right, start + nl, cid, lev + 1, kind, nullptr, nullptr);
    }
    T->son0[cid] = c0;
    T->son1[cid] = c1;
    return cid;
  };
  build(idx, 0, -1, 0, gptr ? DOMAIN : INTERFACE, nullptr, nullptr);
  const int nc = (int)T->lo.size();
  T->nclusters = nc;
  T->depth = *std::max_element(T->level.begin(), T->level.end());
  T->tsize.assign(nc, 1);
  for (int t = nc - 1; t >= 0; --t)
    if (T->son0[t] >= 0) T->tsize[t] = 1 + T->tsize[T->son0[t]] + T->tsize[T->son1[t]];
  // BFS order: sorted by (level, id)
  T->level_ptr.assign(T->depth + 2, 0);
  for (int t = 0; t < nc; ++t) T->level_ptr[T->level[t] + 1]++;
  for (int L = 0; L <= T->depth; ++L) T->level_ptr[L + 1] += T->level_ptr[L];
  T->bfs.assign(nc, 0);
  {
    std::vector<int32_t> fill(T->level_ptr.begin(), T->level_ptr.end() - 1);
    for (int t = 0; t < nc; ++t) T->bfs[fill[T->level[t]]++] = t;
  }
  T->leaf_index.assign(nc, -1);
  for (int t = 0; t < nc; ++t)
    if (T->son0[t] < 0) {
      T->leaf_index[t] = (int32_t)T->leaves.size();
      T->leaves.push_back(t);
    }
  *out = T;
  return H2_OK;
}

extern "C" h2_status h2_cluster_tree(const double* pts, int64_t n, int32_t dim, int32_t leaf_size,
                                     h2_tree* out) {
  return build_cluster_tree(pts, n, dim, leaf_size, nullptr, nullptr, out);
}

extern "C" h2_status h2_cluster_tree_dd(const double* pts, int64_t n, int32_t dim, int32_t leaf_size,
                                        const int64_t* rowptr, const int32_t* colidx, h2_tree* out) {
  if (!out) H2_FAIL(H2_ERR_ARG, "h2_cluster_tree_dd: out is NULL");
  *out = nullptr;
  if (!rowptr || !colidx || n <= 0) H2_FAIL(H2_ERR_ARG, "h2_cluster_tree_dd: need the CSR pattern of the matrix");
  // symmetrised coupling graph (pattern of A + A^T, duplicates harmless)
  std::vector<int64_t> gptr(n + 1, 0);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
      const int32_t j = colidx[e];
      if (j < 0 || j >= n) H2_FAIL(H2_ERR_ARG, "h2_cluster_tree_dd: column index out of range");
      gptr[i + 1]++;
      gptr[j + 1]++;
    }
  for (int64_t i = 0; i < n; ++i) gptr[i + 1] += gptr[i];
  std::vector<int32_t> gidx(gptr[n]);
  std::vector<int64_t> fill(gptr.begin(), gptr.end() - 1);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
      const int32_t j = colidx[e];
      gidx[fill[i]++] = j;
      gidx[fill[j]++] = (int32_t)i;
    }
  return build_cluster_tree(pts, n, dim, leaf_size, gptr.data(), gidx.data(), out);
}

extern "C" h2_status h2_tree_ddpair(h2_tree tree, int8_t* ddpair) {
  if (!tree || !ddpair) H2_FAIL(H2_ERR_ARG, "h2_tree_ddpair: NULL argument");
  for (int t = 0; t < tree->nclusters; ++t) ddpair[t] = (int8_t)tree->ddpair[t];
  return H2_OK;
}

extern "C" h2_status h2_tree_export(h2_tree tree, int64_t* perm, int32_t* lo, int32_t* hi, int32_t* son0,
                                    int32_t* son1, int32_t* level, int32_t* nclusters) {
  if (!tree) H2_FAIL(H2_ERR_ARG, "h2_tree_export: NULL tree");
  const h2_tree_* T = tree;
  if (nclusters) *nclusters = T->nclusters;
  if (perm) std::copy(T->perm.begin(), T->perm.end(), perm);
  if (lo) std::copy(T->lo.begin(), T->lo.end(), lo);
  if (hi) std::copy(T->hi.begin(), T->hi.end(), hi);
  if (son0) std::copy(T->son0.begin(), T->son0.end(), son0);
  if (son1) std::copy(T->son1.begin(), T->son1.end(), son1);
  if (level) std::copy(T->level.begin(), T->level.end(), level);
  return H2_OK;
}

extern "C" void h2_tree_destroy(h2_tree tree) { delete tree; }

// ------------------------------------------------------------------------------------------------
// Block tree (sons+ P:1031-1037), admissibility per SURVEY R1.
// ------------------------------------------------------------------------------------------------
static double diam2(const h2_tree_* T, int t) {
  double s = 0;
  for (int d = 0; d < T->dim; ++d) {
    double e = T->bmax[t * T->dim + d] - T->bmin[t * T->dim + d];
    s += e * e;
  }
  return s;
}

static double dist2(const h2_tree_* R, int t, const h2_tree_* C, int s) {
  double acc = 0;
  for (int d = 0; d < R->dim; ++d) {
    double g = std::max(0.0, std::max(C->bmin[s * C->dim + d] - R->bmax[t * R->dim + d],
                                      R->bmin[t * R->dim + d] - C->bmax[s * C->dim + d]));
    acc += g * g;
  }
  return acc;
}

extern "C" h2_status h2_block_tree(h2_tree rows, h2_tree cols, double eta, h2_btree* out) {
  if (!out) H2_FAIL(H2_ERR_ARG, "h2_block_tree: out is NULL");
  *out = nullptr;
  if (!rows || !cols) H2_FAIL(H2_ERR_ARG, "h2_block_tree: NULL tree");
  if (!(eta > 0) || !std::isfinite(eta)) H2_FAIL(H2_ERR_ARG, "h2_block_tree: eta must be finite and > 0");
  if (rows->dim != cols->dim) H2_FAIL(H2_ERR_ARG, "h2_block_tree: trees of different dimension");
  h2_btree_* B = new (std::nothrow) h2_btree_();
  if (!B) H2_FAIL(H2_ERR_NOMEM, "h2_block_tree: host allocation failed");
  B->rt = rows;
  B->ct = cols;
  B->eta = eta;
  const double eta2 = eta * eta;
  std::function<int(int, int, int)> build = [&](int t, int s, int par) -> int {
    int b = (int)B->t.size();
    B->t.push_back(t);
    B->s.push_back(s);
    B->parent.push_back(par);
    B->sons.push_back({-1, -1, -1, -1});
    B->nsons.push_back(0);
    B->kind.push_back(SUBDIV);
    // the two decoupled domains of a domain-decomposition split form an admissible (zero) block
    // whatever their geometry (reading own-11); needs one tree for rows and columns
    const bool ddzero = rows == cols && t != s && rows->parent[t] >= 0 && rows->parent[t] == cols->parent[s] &&
                        rows->ddpair[rows->parent[t]];
    const double d2 = dist2(rows, t, cols, s);
    if (ddzero || (d2 > 0.0 && std::max(diam2(rows, t), diam2(cols, s)) <= eta2 * d2)) {
      B->kind[b] = ADM;
      return b;
    }
    const bool tl = rows->son0[t] < 0, sl = cols->son0[s] < 0;
    if (tl && sl) {
      B->kind[b] = INADM;
      return b;
    }
    int ts[2], ss[2], nt = 0, ns = 0;
    if (tl) ts[nt++] = t; else { ts[nt++] = rows->son0[t]; ts[nt++] = rows->son1[t]; }
    if (sl) ss[ns++] = s; else { ss[ns++] = cols->son0[s]; ss[ns++] = cols->son1[s]; }
    int q = 0;
    for (int i = 0; i < nt; ++i)
      for (int j = 0; j < ns; ++j) {
        int c = build(ts[i], ss[j], b);
        B->sons[b][q++] = c;
      }
    B->nsons[b] = (int8_t)q;
    return b;
  };
  build(0, 0, -1);
  const int nb = (int)B->t.size();
  B->bsize.assign(nb, 1);
  for (int b = nb - 1; b >= 0; --b)
    for (int q = 0; q < B->nsons[b]; ++q) B->bsize[b] += B->bsize[B->sons[b][q]];
  B->index.reserve(nb * 2);
  std::vector<int> cr(rows->nclusters, 0), cc(cols->nclusters, 0);
  for (int b = 0; b < nb; ++b) {
    B->index[(int64_t)B->t[b] * cols->nclusters + B->s[b]] = b;
    cr[B->t[b]]++;
    cc[B->s[b]]++;
  }
  B->csp = std::max(*std::max_element(cr.begin(), cr.end()), *std::max_element(cc.begin(), cc.end()));
  *out = B;
  return H2_OK;
}

extern "C" h2_status h2_btree_export(h2_btree bt, int32_t* t, int32_t* s, int8_t* kind, int64_t* nblocks,
                                     int32_t* csp) {
  if (!bt) H2_FAIL(H2_ERR_ARG, "h2_btree_export: NULL block tree");
  if (nblocks) *nblocks = (int64_t)bt->t.size();
  if (csp) *csp = bt->csp;
  if (t) std::copy(bt->t.begin(), bt->t.end(), t);
  if (s) std::copy(bt->s.begin(), bt->s.end(), s);
  if (kind) std::copy(bt->kind.begin(), bt->kind.end(), kind);
  return H2_OK;
}

extern "C" void h2_btree_destroy(h2_btree bt) { delete bt; }

// ------------------------------------------------------------------------------------------------
// Device storage
// ------------------------------------------------------------------------------------------------
namespace h2 {
void poison(void* p, size_t bytes) {
  static const bool on = getenv("H2_POISON") && atoi(getenv("H2_POISON")) != 0;
  if (on && p && bytes) cudaMemset(p, 0xFF, bytes);
}
}  // namespace h2

template <class T>
static cudaError_t dalloc(h2_mat_* Z, T** p, size_t count) {
  *p = nullptr;
  if (count == 0) count = 1;
  cudaError_t e = cudaMalloc((void**)p, count * sizeof(T));
  if (e == cudaSuccess) {
    Z->allocs.push_back((void*)*p);
    if (sizeof(T) == 8) h2::poison(*p, count * sizeof(T));
  }
  return e;
}

template <class T>
static cudaError_t dupload(h2_mat_* Z, T** p, const std::vector<T>& v) {
  cudaError_t e = dalloc(Z, p, v.size());
  if (e != cudaSuccess) return e;
  if (!v.empty()) e = cudaMemcpy(*p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
  return e;
}

static void free_mat(h2_mat_* Z) {
  if (!Z) return;
  h2::free_mvpack(Z);
  for (void* p : Z->allocs) cudaFree(p);
  delete Z;
}

extern "C" void h2_mat_destroy(h2_mat Z) { free_mat(Z); }

static h2_status setup_side(h2_mat_* Z, DevSide& D, const h2_tree_* T, bool row_side) {
  const h2_btree_* B = Z->bt;
  const MatDev& M = Z->d;
  D.tree = T;
  D.nclusters = T->nclusters;
  D.nleaves = (int)T->leaves.size();
  CUDA_TRY(dupload(Z, &D.lo, T->lo));
  CUDA_TRY(dupload(Z, &D.hi, T->hi));
  CUDA_TRY(dupload(Z, &D.son0, T->son0));
  CUDA_TRY(dupload(Z, &D.son1, T->son1));
  CUDA_TRY(dupload(Z, &D.parent, T->parent));
  CUDA_TRY(dupload(Z, &D.tsize, T->tsize));
  CUDA_TRY(dupload(Z, &D.leafidx, T->leaf_index));
  CUDA_TRY(dupload(Z, &D.bfs, T->bfs));
  CUDA_TRY(dupload(Z, &D.leaves, T->leaves));
  CUDA_TRY(dupload(Z, &D.level, T->level));
  CUDA_TRY(dupload(Z, &D.perm, T->perm));
  {  // ancestors of every leaf by level (matvec backward transform walks them root -> leaf)
    D.ancw = T->depth + 1;
    std::vector<int32_t> anc((size_t)D.nleaves * D.ancw, -1);
    for (int li = 0; li < D.nleaves; ++li)
      for (int c = T->leaves[li]; c >= 0; c = T->parent[c]) anc[(size_t)li * D.ancw + T->level[c]] = c;
    CUDA_TRY(dupload(Z, &D.anc, anc));
  }
  // admissible stored blocks per cluster (adm slots in DFS order)
  std::vector<int32_t> ptr(T->nclusters + 1, 0), idx;
  for (size_t a = 0; a < Z->adm_blk.size(); ++a) {
    int b = Z->adm_blk[a];
    ptr[(row_side ? B->t[b] : B->s[b]) + 1]++;
  }
  for (int t = 0; t < T->nclusters; ++t) ptr[t + 1] += ptr[t];
  idx.assign(ptr.back(), 0);
  {
    std::vector<int32_t> fill(ptr.begin(), ptr.end() - 1);
    for (size_t a = 0; a < Z->adm_blk.size(); ++a) {
      int b = Z->adm_blk[a];
      idx[fill[row_side ? B->t[b] : B->s[b]]++] = (int32_t)a;
    }
  }
  CUDA_TRY(dupload(Z, &D.bptr, ptr));
  CUDA_TRY(dupload(Z, &D.bidx, idx));
  CUDA_TRY(dalloc(Z, &D.rank, T->nclusters));
  CUDA_TRY(cudaMemset(D.rank, 0, sizeof(int32_t) * T->nclusters));
  const size_t r2 = (size_t)M.rcap * M.rcap;
  CUDA_TRY(dalloc(Z, &D.leafb, (size_t)D.nleaves * M.lmax * M.rcap));
  CUDA_TRY(cudaMemset(D.leafb, 0, sizeof(double) * (size_t)D.nleaves * M.lmax * M.rcap));
  CUDA_TRY(dalloc(Z, &D.tr, (size_t)T->nclusters * r2));
  CUDA_TRY(cudaMemset(D.tr, 0, sizeof(double) * (size_t)T->nclusters * r2));
  CUDA_TRY(dalloc(Z, &D.rc, (size_t)T->nclusters * r2));
  CUDA_TRY(cudaMemset(D.rc, 0, sizeof(double) * (size_t)T->nclusters * r2));
  CUDA_TRY(dalloc(Z, &D.xh, (size_t)T->nclusters * M.rcap));
  CUDA_TRY(dalloc(Z, &D.mvsync, (size_t)T->nclusters));
  CUDA_TRY(cudaMemset(D.mvsync, 0, sizeof(int32_t) * (size_t)T->nclusters));
  {  // matvec schedule: maximal subtrees with <= MV_SUB_LEAVES leaves, and the clusters above them
    std::vector<int32_t> nleaf(T->nclusters, 0);
    for (int c = T->nclusters - 1; c >= 0; --c)
      nleaf[c] = T->son0[c] < 0 ? 1 : nleaf[T->son0[c]] + nleaf[T->son1[c]];
    std::vector<int32_t> roots, top;
    std::vector<std::vector<int32_t>> bylev;
    for (int c = 0; c < T->nclusters; ++c) {
      const int p = T->parent[c];
      if (nleaf[c] <= MV_SUB_LEAVES && (p < 0 || nleaf[p] > MV_SUB_LEAVES)) roots.push_back(c);
      if (nleaf[c] > MV_SUB_LEAVES) {
        if ((int)bylev.size() <= T->level[c]) bylev.resize(T->level[c] + 1);
        bylev[T->level[c]].push_back(c);
      }
    }
    D.h_top_lptr.assign(1, 0);
    for (auto& l : bylev) {
      top.insert(top.end(), l.begin(), l.end());
      D.h_top_lptr.push_back((int32_t)top.size());
    }
    D.n_mv_roots = (int)roots.size();
    D.mv_top_nlev = (int)bylev.size();
    CUDA_TRY(dupload(Z, &D.mv_roots, roots));
    CUDA_TRY(dupload(Z, &D.mv_top, top));
    CUDA_TRY(dupload(Z, &D.mv_top_lptr, D.h_top_lptr));
    CUDA_TRY(dalloc(Z, &D.mv_cnt, 4));
    CUDA_TRY(cudaMemset(D.mv_cnt, 0, 4 * sizeof(int32_t)));
  }
  return H2_OK;
}

static h2_status alloc_update_workspace(h2_mat_* Z, DevSide& D) {
  if (D.re) return H2_OK;
  const MatDev& M = Z->d;
  const size_t nc = D.nclusters, k2 = (size_t)M.kcap * M.kcap;
  CUDA_TRY(dalloc(Z, &D.re, nc * k2));
  CUDA_TRY(dalloc(Z, &D.bw, nc * k2));
  CUDA_TRY(dalloc(Z, &D.rn, nc * k2));
  CUDA_TRY(dalloc(Z, &D.qn, nc * (size_t)M.ldq * M.rcap));
  CUDA_TRY(dalloc(Z, &D.rnew, nc));
  return H2_OK;
}

extern "C" h2_status h2_from_sparse(h2_btree bt, int64_t n, const int64_t* rowptr, const int32_t* colidx,
                                    const double* val, h2_storage storage, int32_t rank_cap,
                                    int32_t update_cap, h2_stream stream, h2_mat* out) {
  if (!out) H2_FAIL(H2_ERR_ARG, "h2_from_sparse: out is NULL");
  *out = nullptr;
  if (!bt) H2_FAIL(H2_ERR_ARG, "h2_from_sparse: NULL block tree");
  const h2_tree_* R = bt->rt;
  const h2_tree_* C = bt->ct;
  if (n != R->n || n != C->n) H2_FAIL(H2_ERR_SHAPE, "h2_from_sparse: n does not match the cluster trees");
  if (!rowptr || (n > 0 && rowptr[n] > 0 && (!colidx || !val)))
    H2_FAIL(H2_ERR_ARG, "h2_from_sparse: NULL CSR array");
  if (storage != H2_FULL && storage != H2_LOWER) H2_FAIL(H2_ERR_ARG, "h2_from_sparse: bad storage");
  if (storage == H2_LOWER && R != C) H2_FAIL(H2_ERR_ARG, "h2_from_sparse: H2_LOWER needs one shared tree");
  if (rank_cap < 1 || rank_cap > RCAP_MAX || update_cap < 0 || rank_cap + update_cap > KCAP_MAX)
    H2_FAIL(H2_ERR_ARG, "h2_from_sparse: need 1 <= rank_cap <= 48, update_cap >= 0, rank_cap + update_cap <= 96");
  int lmax = 0;
  for (int t : R->leaves) lmax = std::max(lmax, R->hi[t] - R->lo[t]);
  for (int t : C->leaves) lmax = std::max(lmax, C->hi[t] - C->lo[t]);
  if (lmax > LMAX_MAX) H2_FAIL(H2_ERR_ARG, "h2_from_sparse: leaf clusters larger than 64 are not supported");
  for (int64_t i = 0; i < n; ++i)
    if (rowptr[i + 1] < rowptr[i]) H2_FAIL(H2_ERR_ARG, "h2_from_sparse: rowptr not monotone");
  const int64_t nnz = rowptr[n] - rowptr[0];
  for (int64_t q = rowptr[0]; q < rowptr[0] + nnz; ++q) {
    if (colidx[q] < 0 || colidx[q] >= n) H2_FAIL(H2_ERR_ARG, "h2_from_sparse: column index out of range");
    if (!std::isfinite(val[q])) H2_FAIL(H2_ERR_NONFINITE, "h2_from_sparse: non-finite value");
  }
  h2_mat_* Z = new (std::nothrow) h2_mat_();
  if (!Z) H2_FAIL(H2_ERR_NOMEM, "h2_from_sparse: host allocation failed");
  Z->bt = bt;
  Z->lower = storage == H2_LOWER;
  MatDev& M = Z->d;
  M.rcap = rank_cap;
  M.ucap = update_cap;
  M.kcap = rank_cap + update_cap;
  M.lmax = lmax;
  M.ldq = std::max(lmax, 2 * rank_cap);
  const int nb = (int)bt->t.size();
  auto stored = [&](int b) { return !Z->lower || R->lo[bt->t[b]] >= C->lo[bt->s[b]]; };
  Z->blk2adm.assign(nb, -1);
  Z->blk2inad.assign(nb, -1);
  Z->inad_range.assign(2 * nb, 0);
  for (int b = 0; b < nb; ++b) {
    if (bt->kind[b] == ADM && stored(b)) {
      Z->blk2adm[b] = (int32_t)Z->adm_blk.size();
      Z->adm_blk.push_back(b);
    } else if (bt->kind[b] == INADM && stored(b)) {
      Z->blk2inad[b] = (int32_t)Z->inad_blk.size();
      Z->inad_blk.push_back(b);
    }
  }
  // [first,last) inadmissible slots inside each block subtree (subtrees are contiguous in DFS order)
  {
    std::vector<int32_t> before(nb + 1, 0);
    for (int b = 0; b < nb; ++b) before[b + 1] = before[b] + (Z->blk2inad[b] >= 0 ? 1 : 0);
    for (int b = 0; b < nb; ++b) {
      Z->inad_range[2 * b] = before[b];
      Z->inad_range[2 * b + 1] = before[b + bt->bsize[b]];
    }
  }
  M.nadm = (int)Z->adm_blk.size();
  M.ninad = (int)Z->inad_blk.size();
  // scatter the CSR into nearfield tiles on the host (tree order), then upload
  std::vector<int64_t> iperm_r(n), iperm_c(n);
  for (int64_t i = 0; i < n; ++i) {
    iperm_r[R->perm[i]] = i;
    iperm_c[C->perm[i]] = i;
  }
  std::vector<int32_t> rleaf(n), cleaf(n);
  for (int t : R->leaves)
    for (int i = R->lo[t]; i < R->hi[t]; ++i) rleaf[i] = t;
  for (int s : C->leaves)
    for (int i = C->lo[s]; i < C->hi[s]; ++i) cleaf[i] = s;
  std::vector<double> tiles((size_t)M.ninad * lmax * lmax, 0.0);
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t q = rowptr[i]; q < rowptr[i + 1]; ++q) {
      const double v = val[q];
      if (v == 0.0) continue;
      const int64_t pi = iperm_r[i], pj = iperm_c[colidx[q]];
      const int t = rleaf[pi], s = cleaf[pj];
      const int b = bt->find(t, s);
      if (b < 0 || bt->kind[b] != INADM) {
        free_mat(Z);
        char msg[200];
        snprintf(msg, sizeof msg, "h2_from_sparse: nonzero (%lld,%lld) lies in an admissible block",
                 (long long)i, (long long)colidx[q]);
        H2_FAIL(H2_ERR_STRUCTURE, msg);
      }
      const int slot = Z->blk2inad[b];
      if (slot < 0) continue;  // upper part of a symmetric matrix in H2_LOWER storage
      tiles[(size_t)slot * lmax * lmax + (pi - R->lo[t]) + (size_t)(pj - C->lo[s]) * lmax] += v;
    }
  }
  h2_status st;
  cudaError_t e;
  std::vector<int32_t> at(M.nadm), as(M.nadm), it(M.ninad), is(M.ninad);
  for (int a = 0; a < M.nadm; ++a) {
    at[a] = bt->t[Z->adm_blk[a]];
    as[a] = bt->s[Z->adm_blk[a]];
  }
  for (int a = 0; a < M.ninad; ++a) {
    it[a] = bt->t[Z->inad_blk[a]];
    is[a] = bt->s[Z->inad_blk[a]];
  }
  // nearfield CSR per row leaf and per column leaf
  std::vector<int32_t> nptr(R->nclusters + 1, 0), nidx(M.ninad), ntptr(C->nclusters + 1, 0), ntidx(M.ninad);
  for (int a = 0; a < M.ninad; ++a) {
    nptr[it[a] + 1]++;
    ntptr[is[a] + 1]++;
  }
  for (int t = 0; t < R->nclusters; ++t) nptr[t + 1] += nptr[t];
  for (int t = 0; t < C->nclusters; ++t) ntptr[t + 1] += ntptr[t];
  {
    std::vector<int32_t> f1(nptr.begin(), nptr.end() - 1), f2(ntptr.begin(), ntptr.end() - 1);
    for (int a = 0; a < M.ninad; ++a) {
      nidx[f1[it[a]]++] = a;
      ntidx[f2[is[a]]++] = a;
    }
  }
#define TRY_ALLOC(expr)        \
  do {                         \
    e = (expr);                \
    if (e != cudaSuccess) {    \
      free_mat(Z);             \
      CUDA_TRY(e);             \
    }                          \
  } while (0)
  TRY_ALLOC(dupload(Z, &M.adm_t, at));
  TRY_ALLOC(dupload(Z, &M.adm_s, as));
  TRY_ALLOC(dupload(Z, &M.in_t, it));
  TRY_ALLOC(dupload(Z, &M.in_s, is));
  TRY_ALLOC(dupload(Z, &M.nptr, nptr));
  TRY_ALLOC(dupload(Z, &M.nidx, nidx));
  TRY_ALLOC(dupload(Z, &M.ntptr, ntptr));
  TRY_ALLOC(dupload(Z, &M.ntidx, ntidx));
  TRY_ALLOC(dupload(Z, &M.N, tiles));
  TRY_ALLOC(dalloc(Z, &M.S, (size_t)M.nadm * M.rcap * M.rcap));
  TRY_ALLOC(cudaMemset(M.S, 0, sizeof(double) * (size_t)M.nadm * M.rcap * M.rcap));
  TRY_ALLOC(dalloc(Z, &M.flags, 4));
  TRY_ALLOC(cudaMemset(M.flags, 0, 4 * sizeof(int32_t)));
  if (getenv("H2_UPD_LOG")) TRY_ALLOC(dalloc(Z, &M.updlog, (size_t)5 << 20));
  TRY_ALLOC(dalloc(Z, &M.xt, n));
  TRY_ALLOC(dalloc(Z, &M.yt, n));
#undef TRY_ALLOC
  Z->nzr.assign(R->nclusters, 0);  // every rank is 0 after h2_from_sparse
  Z->nzc.assign(C->nclusters, 0);
  if ((st = setup_side(Z, M.row, R, true)) != H2_OK) { free_mat(Z); return st; }
  if ((st = setup_side(Z, M.col, C, false)) != H2_OK) { free_mat(Z); return st; }
  e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) { free_mat(Z); CUDA_TRY(e); }
  *out = Z;
  return H2_OK;
}

// ------------------------------------------------------------------------------------------------
// Operations
// ------------------------------------------------------------------------------------------------
extern "C" h2_status h2_matvec(h2_mat Z, int32_t transpose, double alpha, const double* x, double beta,
                               double* y, h2_stream stream) {
  H2_NO_BATCH("h2_matvec");
  if (!Z || !x || !y) H2_FAIL(H2_ERR_ARG, "h2_matvec: NULL argument");
  if (!std::isfinite(alpha) || !std::isfinite(beta)) H2_FAIL(H2_ERR_NONFINITE, "h2_matvec: non-finite scalar");
  CUDA_TRY(launch_matvec(Z, transpose ? 1 : 0, alpha, x, beta, y, (cudaStream_t)stream));
  return H2_OK;
}

extern "C" h2_status h2_lowrank_update(h2_mat Z, int32_t t0, int32_t s0, int32_t k, double alpha,
                                       const double* X, int64_t ldx, const double* Y, int64_t ldy,
                                       const h2_trunc* trunc, h2_stream stream) {
  if (!Z) H2_FAIL(H2_ERR_ARG, "h2_lowrank_update: NULL matrix");
  const h2_btree_* B = Z->bt;
  if (t0 < 0 || t0 >= B->rt->nclusters || s0 < 0 || s0 >= B->ct->nclusters)
    H2_FAIL(H2_ERR_ARG, "h2_lowrank_update: cluster id out of range");
  const int b0 = B->find(t0, s0);
  if (b0 < 0) H2_FAIL(H2_ERR_ARG, "h2_lowrank_update: (t0,s0) is not a block of the block tree");
  if (k < 0 || k > Z->d.ucap) H2_FAIL(H2_ERR_SHAPE, "h2_lowrank_update: k outside [0, update_cap]");
  if (!std::isfinite(alpha)) H2_FAIL(H2_ERR_NONFINITE, "h2_lowrank_update: non-finite alpha");
  if (k > 0 && (!X || !Y)) H2_FAIL(H2_ERR_ARG, "h2_lowrank_update: NULL factor");
  const int mt = B->rt->hi[t0] - B->rt->lo[t0], ms = B->ct->hi[s0] - B->ct->lo[s0];
  if (k > 0 && (ldx < mt || ldy < ms)) H2_FAIL(H2_ERR_SHAPE, "h2_lowrank_update: leading dimension too small");
  h2_trunc tc = trunc ? *trunc : h2_trunc{1e-4, 0.0, 0, 0};
  if (!(tc.rel_tol >= 0) || !(tc.abs_tol >= 0)) H2_FAIL(H2_ERR_ARG, "h2_lowrank_update: negative tolerance");
  if (Z->lower && B->rt->lo[t0] < B->ct->lo[s0])
    H2_FAIL(H2_ERR_ARG, "h2_lowrank_update: target block is not stored in H2_LOWER storage");
  if (h2::batch_open() && h2::exec_ctx()->st != (cudaStream_t)stream)
    H2_FAIL(H2_ERR_ARG, "h2_lowrank_update: inside a batch every update must use the batch's stream");
  if (k == 0) return H2_OK;  // bit-identical
  h2_status st;
  if ((st = alloc_update_workspace(Z, Z->d.row)) != H2_OK) return st;
  if ((st = alloc_update_workspace(Z, Z->d.col)) != H2_OK) return st;
  UpdArgs a;
  a.t0 = t0;
  a.s0 = s0;
  a.k = k;
  a.X = X;
  a.ldx = ldx;
  a.Y = Y;
  a.ldy = ldy;
  a.alpha = alpha;
  a.rel_tol = tc.rel_tol;
  a.abs_tol = tc.abs_tol;
  a.max_rank = tc.max_rank;
  a.blockwise = tc.blockwise != 0;
  a.kdev = nullptr;
  a.prof = nullptr;
  try {
    CUDA_TRY(launch_update(Z, a, (cudaStream_t)stream));
  } catch (const std::exception& ex) {  // recording errors (e.g. too many matrices in one batch)
    H2_FAIL(H2_ERR_ARG, std::string("h2_lowrank_update: ") + ex.what());
  }
  Z->version++;
  if (B->kind[b0] != INADM) {  // the update may give the bases of T_{t0} / T_{s0} a non-zero rank
    for (int q = t0; q < t0 + B->rt->tsize[t0]; ++q) Z->nzr[q] = 1;
    for (int q = s0; q < s0 + B->ct->tsize[s0]; ++q) Z->nzc[q] = 1;
  }
  return H2_OK;
}

// ------------------------------------------------------------------------------------------------
// Inspection
// ------------------------------------------------------------------------------------------------
extern "C" h2_status h2_ranks(h2_mat Z, int32_t* row_rank, int32_t* col_rank) {
  H2_NO_BATCH("h2_ranks");
  if (!Z) H2_FAIL(H2_ERR_ARG, "h2_ranks: NULL matrix");
  CUDA_TRY(cudaDeviceSynchronize());
  if (row_rank)
    CUDA_TRY(cudaMemcpy(row_rank, Z->d.row.rank, sizeof(int32_t) * Z->d.row.nclusters, cudaMemcpyDeviceToHost));
  if (col_rank)
    CUDA_TRY(cudaMemcpy(col_rank, Z->d.col.rank, sizeof(int32_t) * Z->d.col.nclusters, cudaMemcpyDeviceToHost));
  return H2_OK;
}

extern "C" h2_status h2_check_device_flags(h2_mat Z, int32_t* flags) {
  H2_NO_BATCH("h2_check_device_flags");
  if (!Z || !flags) H2_FAIL(H2_ERR_ARG, "h2_check_device_flags: NULL argument");
  CUDA_TRY(cudaDeviceSynchronize());
  int32_t f[3];
  CUDA_TRY(cudaMemcpy(f, Z->d.flags, sizeof(f), cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemset(Z->d.flags, 0, 3 * sizeof(int32_t)));  // flags[3] (update counter) is kept
  if (Z->d.updlog && getenv("H2_UPD_LOG")) {  // diagnostic: the non-zero-rank updates in order, as text
    int32_t cnt = 0;
    CUDA_TRY(cudaMemcpy(&cnt, Z->d.flags + 3, sizeof(cnt), cudaMemcpyDeviceToHost));
    cnt = std::min(cnt, 1 << 20);
    std::vector<int32_t> lg((size_t)5 * cnt);
    CUDA_TRY(cudaMemcpy(lg.data(), Z->d.updlog, sizeof(int32_t) * lg.size(), cudaMemcpyDeviceToHost));
    if (FILE* f = fopen(getenv("H2_UPD_LOG"), "w")) {
      for (int i = 0; i < cnt; ++i)
        fprintf(f, "%d %d %d %d %d\n", lg[5 * i], lg[5 * i + 1], lg[5 * i + 2], lg[5 * i + 3], lg[5 * i + 4]);
      fclose(f);
    }
  }
  flags[0] = f[0] | (f[1] ? 2 : 0);
  if (f[0] & 4) {  // reported first: a dropped contribution usually ends in a leaf breakdown as well
    h2::set_error("a contribution's rank exceeded update_cap and was dropped: the result is invalid; "
                  "rebuild the matrix with a larger update_cap (up to the leaf size)");
    return H2_ERR_NOMEM;
  }
  if (f[1]) {
    char msg[160];
    snprintf(msg, sizeof msg, "dense leaf breakdown (non-positive / tiny pivot) in the diagonal tile of cluster %d", f[2]);
    h2::set_error(msg);
    return H2_ERR_BREAKDOWN;
  }
  return H2_OK;
}

extern "C" h2_status h2_stats(h2_mat Z, int64_t out[4]) {
  H2_NO_BATCH("h2_stats");
  if (!Z || !out) H2_FAIL(H2_ERR_ARG, "h2_stats: NULL argument");
  for (int i = 0; i < 3; ++i) out[i] = Z->stats[i];
  int32_t nz = 0;
  CUDA_TRY(cudaDeviceSynchronize());
  CUDA_TRY(cudaMemcpy(&nz, Z->d.flags + 3, sizeof(int32_t), cudaMemcpyDeviceToHost));
  out[3] = nz;
  return H2_OK;
}

extern "C" h2_status h2_storage_report(h2_mat Z, int64_t scalars[4]) {
  H2_NO_BATCH("h2_storage_report");
  if (!Z || !scalars) H2_FAIL(H2_ERR_ARG, "h2_storage_report: NULL argument");
  const h2_btree_* B = Z->bt;
  std::vector<int32_t> kr(Z->d.row.nclusters), kc(Z->d.col.nclusters);
  h2_status st = h2_ranks(Z, kr.data(), kc.data());
  if (st != H2_OK) return st;
  const h2_tree_* R = B->rt;
  const h2_tree_* C = B->ct;
  int64_t near = 0, leaf = 0, tr = 0, cp = 0;
  for (int b : Z->inad_blk) near += (int64_t)(R->hi[B->t[b]] - R->lo[B->t[b]]) * (C->hi[B->s[b]] - C->lo[B->s[b]]);
  for (int t : R->leaves) leaf += (int64_t)(R->hi[t] - R->lo[t]) * kr[t];
  for (int s : C->leaves) leaf += (int64_t)(C->hi[s] - C->lo[s]) * kc[s];
  for (int t = 1; t < R->nclusters; ++t) tr += (int64_t)kr[t] * kr[R->parent[t]];
  for (int s = 1; s < C->nclusters; ++s) tr += (int64_t)kc[s] * kc[C->parent[s]];
  for (int b : Z->adm_blk) cp += (int64_t)kr[B->t[b]] * kc[B->s[b]];
  scalars[0] = near;
  scalars[1] = leaf;
  scalars[2] = tr;
  scalars[3] = cp;
  return H2_OK;
}

extern "C" h2_status h2_export(h2_mat Z, double* V, double* E, double* W, double* F, double* S, double* N,
                               int64_t sizes[6]) {
  H2_NO_BATCH("h2_export");
  if (!Z || !sizes) H2_FAIL(H2_ERR_ARG, "h2_export: NULL argument");
  const h2_btree_* B = Z->bt;
  const h2_tree_* R = B->rt;
  const h2_tree_* C = B->ct;
  const MatDev& M = Z->d;
  std::vector<int32_t> kr(M.row.nclusters), kc(M.col.nclusters);
  h2_status st = h2_ranks(Z, kr.data(), kc.data());
  if (st != H2_OK) return st;
  const size_t r2 = (size_t)M.rcap * M.rcap;
  std::vector<double> hleafr((size_t)M.row.nleaves * M.lmax * M.rcap), hleafc((size_t)M.col.nleaves * M.lmax * M.rcap);
  std::vector<double> htrr((size_t)R->nclusters * r2), htrc((size_t)C->nclusters * r2);
  std::vector<double> hS((size_t)M.nadm * r2), hN((size_t)M.ninad * M.lmax * M.lmax);
  CUDA_TRY(cudaMemcpy(hleafr.data(), M.row.leafb, hleafr.size() * 8, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(hleafc.data(), M.col.leafb, hleafc.size() * 8, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(htrr.data(), M.row.tr, htrr.size() * 8, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(htrc.data(), M.col.tr, htrc.size() * 8, cudaMemcpyDeviceToHost));
  if (!hS.empty()) CUDA_TRY(cudaMemcpy(hS.data(), M.S, hS.size() * 8, cudaMemcpyDeviceToHost));
  if (!hN.empty()) CUDA_TRY(cudaMemcpy(hN.data(), M.N, hN.size() * 8, cudaMemcpyDeviceToHost));
  int64_t nV = 0, nE = 0, nW = 0, nF = 0, nS = 0, nN = 0;
  auto put = [](double* dst, int64_t& pos, const double* src, int rows, int cols, int ld) {
    for (int j = 0; j < cols; ++j)
      for (int i = 0; i < rows; ++i) {
        if (dst) dst[pos] = src[i + (size_t)j * ld];
        ++pos;
      }
  };
  for (size_t q = 0; q < R->leaves.size(); ++q) {
    int t = R->leaves[q];
    put(V, nV, &hleafr[q * M.lmax * M.rcap], R->hi[t] - R->lo[t], kr[t], M.lmax);
  }
  for (size_t q = 0; q < C->leaves.size(); ++q) {
    int s = C->leaves[q];
    put(W, nW, &hleafc[q * M.lmax * M.rcap], C->hi[s] - C->lo[s], kc[s], M.lmax);
  }
  for (int t = 1; t < R->nclusters; ++t) put(E, nE, &htrr[t * r2], kr[t], kr[R->parent[t]], M.rcap);
  for (int s = 1; s < C->nclusters; ++s) put(F, nF, &htrc[s * r2], kc[s], kc[C->parent[s]], M.rcap);
  for (int a = 0; a < M.nadm; ++a) {
    int b = Z->adm_blk[a];
    put(S, nS, &hS[a * r2], kr[B->t[b]], kc[B->s[b]], M.rcap);
  }
  for (int a = 0; a < M.ninad; ++a) {
    int b = Z->inad_blk[a];
    put(N, nN, &hN[(size_t)a * M.lmax * M.lmax], R->hi[B->t[b]] - R->lo[B->t[b]], C->hi[B->s[b]] - C->lo[B->s[b]],
        M.lmax);
  }
  sizes[0] = nV;
  sizes[1] = nE;
  sizes[2] = nW;
  sizes[3] = nF;
  sizes[4] = nS;
  sizes[5] = nN;
  return H2_OK;
}

// ---- import (test-only, the inverse of h2_export) ---------------------------------------------
namespace {
// R-factor (k x k upper triangle, rows beyond min(rows, k) zero, ld ldr) of the rows x k matrix A
// (column-major, ld lda) by Householder reflections: the memoised R of a nested basis (reading R7)
void host_qr_R(std::vector<double> A, int rows, int k, int lda, double* R, int ldr) {
  const int p = std::min(rows, k);
  for (int j = 0; j < p; ++j) {
    double nrm = 0.0;
    for (int i = j; i < rows; ++i) nrm += A[i + (size_t)j * lda] * A[i + (size_t)j * lda];
    nrm = std::sqrt(nrm);
    if (nrm == 0.0) continue;
    const double a0 = A[j + (size_t)j * lda];
    const double alpha = a0 > 0 ? -nrm : nrm;
    std::vector<double> v(rows - j);
    v[0] = a0 - alpha;
    for (int i = j + 1; i < rows; ++i) v[i - j] = A[i + (size_t)j * lda];
    double vv = 0.0;
    for (double x : v) vv += x * x;
    if (vv == 0.0) continue;
    for (int c = j; c < k; ++c) {
      double d = 0.0;
      for (int i = j; i < rows; ++i) d += v[i - j] * A[i + (size_t)c * lda];
      const double f = 2.0 * d / vv;
      for (int i = j; i < rows; ++i) A[i + (size_t)c * lda] -= f * v[i - j];
    }
  }
  for (int c = 0; c < k; ++c)
    for (int i = 0; i < k; ++i) R[i + (size_t)c * ldr] = (i <= c && i < p) ? A[i + (size_t)c * lda] : 0.0;
}
}  // namespace

extern "C" h2_status h2_import(h2_btree bt, const int32_t* row_rank, const int32_t* col_rank, const double* V,
                               const double* E, const double* W, const double* F, const double* S, const double* N,
                               h2_storage storage, int32_t rank_cap, int32_t update_cap, h2_stream stream,
                               h2_mat* out) {
  if (!out) H2_FAIL(H2_ERR_ARG, "h2_import: out is NULL");
  *out = nullptr;
  if (!bt || !row_rank || !col_rank) H2_FAIL(H2_ERR_ARG, "h2_import: NULL argument");
  const h2_tree_* R = bt->rt;
  const h2_tree_* C = bt->ct;
  for (int t = 0; t < R->nclusters; ++t)
    if (row_rank[t] < 0 || row_rank[t] > rank_cap) H2_FAIL(H2_ERR_SHAPE, "h2_import: row rank outside [0, rank_cap]");
  for (int t = 0; t < C->nclusters; ++t)
    if (col_rank[t] < 0 || col_rank[t] > rank_cap) H2_FAIL(H2_ERR_SHAPE, "h2_import: column rank outside [0, rank_cap]");
  // the rank-0 structure (empty CSR), then the blocks
  std::vector<int64_t> rowptr((size_t)R->n + 1, 0);
  h2_mat Z = nullptr;
  h2_status st = h2_from_sparse(bt, R->n, rowptr.data(), nullptr, nullptr, storage, rank_cap, update_cap, stream, &Z);
  if (st != H2_OK) return st;
  MatDev& M = Z->d;
  const size_t r2 = (size_t)M.rcap * M.rcap;
  int64_t pV = 0, pE = 0, pS = 0, pN = 0;
  auto take = [](const double* src, int64_t& pos, double* dst, int rows, int cols, int ld) {
    for (int j = 0; j < cols; ++j)
      for (int i = 0; i < rows; ++i) dst[i + (size_t)j * ld] = src[pos++];
  };
  for (int side = 0; side < 2; ++side) {
    const h2_tree_* T = side ? C : R;
    const int32_t* k = side ? col_rank : row_rank;
    const double* Lsrc = side ? W : V;
    const double* Tsrc = side ? F : E;
    DevSide& D = side ? M.col : M.row;
    std::vector<double> leafb((size_t)D.nleaves * M.lmax * M.rcap, 0.0), tr((size_t)T->nclusters * r2, 0.0);
    std::vector<double> rc((size_t)T->nclusters * r2, 0.0);
    pV = 0;
    pE = 0;
    for (size_t q = 0; q < T->leaves.size(); ++q) {
      const int t = T->leaves[q];
      if (k[t] && !Lsrc) { h2_mat_destroy(Z); H2_FAIL(H2_ERR_ARG, "h2_import: NULL leaf basis"); }
      take(Lsrc, pV, &leafb[q * M.lmax * M.rcap], T->hi[t] - T->lo[t], k[t], M.lmax);
    }
    for (int t = 1; t < T->nclusters; ++t) {
      if (k[t] * k[T->parent[t]] && !Tsrc) { h2_mat_destroy(Z); H2_FAIL(H2_ERR_ARG, "h2_import: NULL transfers"); }
      take(Tsrc, pE, &tr[(size_t)t * r2], k[t], k[T->parent[t]], M.rcap);
    }
    // memoised R-factors of the nested bases, bottom-up (Alg. 16; reading R7)
    for (int t = T->nclusters - 1; t >= 0; --t) {
      const int kt = k[t];
      if (!kt) continue;
      if (T->son0[t] < 0) {
        const int m = T->hi[t] - T->lo[t];
        const size_t q = (size_t)T->leaf_index[t];
        std::vector<double> A(&leafb[q * M.lmax * M.rcap], &leafb[q * M.lmax * M.rcap] + (size_t)M.lmax * M.rcap);
        host_qr_R(A, m, kt, M.lmax, &rc[(size_t)t * r2], M.rcap);
      } else {
        const int c0 = T->son0[t], c1 = T->son1[t], rows = k[c0] + k[c1];
        std::vector<double> A((size_t)std::max(rows, 1) * kt, 0.0);
        int r0 = 0;
        for (int c : {c0, c1}) {  // R_c E_c  (k_c x k_t)
          for (int j = 0; j < kt; ++j)
            for (int i = 0; i < k[c]; ++i) {
              double v = 0.0;
              for (int p = 0; p < k[c]; ++p) v += rc[(size_t)c * r2 + i + (size_t)p * M.rcap] * tr[(size_t)c * r2 + p + (size_t)j * M.rcap];
              A[r0 + i + (size_t)j * std::max(rows, 1)] = v;
            }
          r0 += k[c];
        }
        host_qr_R(A, rows, kt, std::max(rows, 1), &rc[(size_t)t * r2], M.rcap);
      }
    }
    CUDA_TRY(cudaMemcpy(D.leafb, leafb.data(), leafb.size() * 8, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(D.tr, tr.data(), tr.size() * 8, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(D.rc, rc.data(), rc.size() * 8, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(D.rank, k, sizeof(int32_t) * T->nclusters, cudaMemcpyHostToDevice));
    std::vector<char>& nz = side ? Z->nzc : Z->nzr;
    for (int t = 0; t < T->nclusters; ++t) nz[t] = k[t] != 0;
  }
  if (M.nadm) {
    if (!S) { h2_mat_destroy(Z); H2_FAIL(H2_ERR_ARG, "h2_import: NULL couplings"); }
    std::vector<double> hS((size_t)M.nadm * r2, 0.0);
    for (int a = 0; a < M.nadm; ++a) {
      const int b = Z->adm_blk[a];
      take(S, pS, &hS[a * r2], row_rank[bt->t[b]], col_rank[bt->s[b]], M.rcap);
    }
    CUDA_TRY(cudaMemcpy(M.S, hS.data(), hS.size() * 8, cudaMemcpyHostToDevice));
  }
  if (M.ninad) {
    if (!N) { h2_mat_destroy(Z); H2_FAIL(H2_ERR_ARG, "h2_import: NULL nearfield"); }
    std::vector<double> hN((size_t)M.ninad * M.lmax * M.lmax, 0.0);
    for (int a = 0; a < M.ninad; ++a) {
      const int b = Z->inad_blk[a];
      take(N, pN, &hN[(size_t)a * M.lmax * M.lmax], R->hi[bt->t[b]] - R->lo[bt->t[b]],
           C->hi[bt->s[b]] - C->lo[bt->s[b]], M.lmax);
      for (int64_t e = pN - (int64_t)(R->hi[bt->t[b]] - R->lo[bt->t[b]]) * (C->hi[bt->s[b]] - C->lo[bt->s[b]]); e < pN; ++e)
        if (!std::isfinite(N[e])) { h2_mat_destroy(Z); H2_FAIL(H2_ERR_NONFINITE, "h2_import: non-finite nearfield entry"); }
    }
    CUDA_TRY(cudaMemcpy(M.N, hN.data(), hN.size() * 8, cudaMemcpyHostToDevice));
  }
  *out = Z;
  return H2_OK;
}

// ---- batch recording (include/h2.h) ----------------------------------------------------------
namespace {
thread_local h2::ExecCtx g_batch_ctx;
thread_local bool g_batch_open = false;
}  // namespace

bool h2::batch_open() { return g_batch_open; }

extern "C" h2_status h2_batch_begin(h2_stream stream) {
  if (g_batch_open) H2_FAIL(H2_ERR_ARG, "h2_batch_begin: a batch is already open");
  if (h2::exec_ctx()) H2_FAIL(H2_ERR_ARG, "h2_batch_begin: another recording is active");
  h2::exec_begin(&g_batch_ctx, (cudaStream_t)stream);
  g_batch_open = true;
  return H2_OK;
}

extern "C" h2_status h2_batch_end(void) {
  if (!g_batch_open) H2_FAIL(H2_ERR_ARG, "h2_batch_end: no open batch");
  g_batch_open = false;
  cudaError_t e = h2::exec_end();
  if (e != cudaSuccess) H2_FAIL(H2_ERR_CUDA, std::string("h2_batch_end: ") + cudaGetErrorString(e));
  return H2_OK;
}
