// Host driver of the H^2 product, block substitutions and LR/Cholesky factorization.
//
// The recursion follows PAPER §3/§6 in the paper's order (and call-for-call the same order as the
// oracle, reading R9): the host walks the block tree and the triple tree and only enqueues device
// work on one stream; every rank-dependent shape is consumed from device memory, so nothing is
// copied back until the caller inspects the result.
//   addmul  P:458-509, P:1020-1096 (Case 1 recursion, temporaries P:499-503, Case 2 factors)
//   chol    P:338-390 with R = L^T;  lr  P:338-390 (Doolittle, no pivoting)
//   lfs/rfs P:392-450, P:1165-1245 (admissible leaf: reading R8)
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <string>
#include <vector>

#include "h2_arith.cuh"
#include "h2_internal.h"

using namespace h2;

#define CUDA_TRY(expr)                                                                      \
  do {                                                                                      \
    cudaError_t e_ = (expr);                                                                \
    if (e_ != cudaSuccess) {                                                                \
      h2::set_error(std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " #expr); \
      return e_ == cudaErrorMemoryAllocation ? H2_ERR_NOMEM : H2_ERR_CUDA;                  \
    }                                                                                       \
  } while (0)

namespace {

constexpr int KC = KCAP_MAX;

// ------------------------------------------------------------------------------------------------
// device workspace (bump arena with stack discipline)
// ------------------------------------------------------------------------------------------------
struct Arena {
  double* d = nullptr;
  size_t cap = 0, top = 0;
  int* i = nullptr;
  size_t icap = 0, itop = 0;
  double* alloc(size_t n) {
    n = (n + 31) & ~size_t(31);
    if (top + n > cap) throw std::runtime_error("h2: factorization workspace exhausted");
    double* p = d + top;
    top += n;
    return p;
  }
  int* ialloc(size_t n = 1) {
    n = (n + 7) & ~size_t(7);
    if (itop + n > icap) throw std::runtime_error("h2: factorization int workspace exhausted");
    int* p = i + itop;
    itop += n;
    return p;
  }
};

struct Mark {
  Arena& a;
  size_t t, it;
  explicit Mark(Arena& a_) : a(a_), t(a_.top), it(a_.itop) {}
  ~Mark() {
    a.top = t;
    a.itop = it;
  }
};

// independence group of recorded ops (ExecCtx::group_begin): the caller guarantees that the ops
// recorded inside neither read nor write what another op of the group writes
struct Group {
  ExecCtx* c;
  Group() : c(exec_ctx()) { c->group_begin(); }
  ~Group() { c->group_end(); }
};

// an operand op(Z) of the product
struct HOp {
  h2_mat_* Z;
  bool trans;
  const h2_btree_* bt() const { return Z->bt; }
  int bid(int a, int b) const { return trans ? Z->bt->find(b, a) : Z->bt->find(a, b); }
  int kind(int a, int b) const { return Z->bt->kind[bid(a, b)]; }
  bool stored(int a, int b) const {
    const int x = bid(a, b);
    return Z->bt->kind[x] == SUBDIV || Z->blk2adm[x] >= 0 || Z->blk2inad[x] >= 0;
  }
  const DevSide& rows() const { return trans ? Z->d.col : Z->d.row; }
  const DevSide& cols() const { return trans ? Z->d.row : Z->d.col; }
  HOp t() const { return HOp{Z, !trans}; }
};

struct Temp {
  int ra, rb, ma, mb;
  double* A;
  double* B;
  int* k;
  bool nz;  // some contribution of possibly non-zero rank was added (host-side, symbolic)
};

struct Driver {
  h2_mat_* Z;  // target (in place for the factorizations)
  cudaStream_t st;
  double rel, abs_tol;
  int max_rank;
  int blockwise;  // h2_trunc.blockwise: local updates weight block-relative; temporaries keep the relative rule
  Arena& ar;
  const h2_tree_* T;  // the (shared) cluster tree
  int rcap, lmax;
  double* ident;  // lmax x lmax identity
  long long n_updates = 0, n_dense = 0, n_temps = 0;
  static constexpr size_t NO_SKIP = ~size_t(0);
  size_t pre_skip = NO_SKIP;  // skip region opened by factors() (closed by addmul after the addition)

  // reading own-6 ahead of the work: the contribution's rank and the zero-tile checks are recorded
  // first, then a skip region covers the factor construction and the addition, so a contribution
  // that turns out exactly zero on the device costs no hmul / expansion at all (the addition was
  // skipped before as well: same result)
  void open_pre_skip(int* kdev) { pre_skip = exec_ctx()->begin_skip(kdev); }
  // profiling tag of the skip regions recorded next (h2_profile_ops slots 48 + tag)
  void tag(int v) { exec_ctx()->skip_tag = v; }

  int size(int t) const { return T->hi[t] - T->lo[t]; }
  // Symbolic rank tracking (host): a cluster basis can only have a non-zero rank after an update
  // touched its subtree; a Case-2 factor / substitution whose rank is structurally zero is skipped,
  // exactly where the oracle skips a zero-column factor (the device would run a no-op).
  static bool nzr(const HOp& X, int t) { return X.trans ? X.Z->nzc[t] != 0 : X.Z->nzr[t] != 0; }
  static bool nzc(const HOp& X, int s) { return X.trans ? X.Z->nzr[s] != 0 : X.Z->nzc[s] != 0; }
  void mark_update(int t, int r) {
    for (int q = t; q < t + T->tsize[t]; ++q) Z->nzr[q] = 1;
    for (int q = r; q < r + T->tsize[r]; ++q) Z->nzc[q] = 1;
  }
  bool leaf(int t) const { return T->son0[t] < 0; }
  std::vector<int> sons_plus(int t) const {
    if (leaf(t)) return {t};
    return {T->son0[t], T->son1[t]};
  }
  double* Sptr(h2_mat_* M, int bid) const { return M->d.S + (size_t)M->blk2adm[bid] * M->d.rcap * M->d.rcap; }
  double* Nptr(h2_mat_* M, int bid) const { return M->d.N + (size_t)M->blk2inad[bid] * M->d.lmax * M->d.lmax; }

  // ---- contributions -------------------------------------------------------------------------
  void update(int t, int r, const double* A, int lda, const double* B, int ldb, const int* kdev, double alpha) {
    // a contribution's rank can reach the leaf size (dense x dense, reading own-7): if that may
    // exceed the update capacity, check it on the device (flag 4 of h2_check_device_flags) instead
    // of overrunning the extended-rank workspace
    if (kdev && lmax > Z->d.ucap) rank_check(Z->d, const_cast<int*>(kdev), Z->d.ucap, st);
    UpdArgs a;
    a.t0 = t;
    a.s0 = r;
    a.k = 0;
    a.kdev = kdev;
    a.X = A;
    a.ldx = lda;
    a.Y = B;
    a.ldy = ldb;
    a.alpha = alpha;
    a.rel_tol = rel;
    a.abs_tol = abs_tol;
    a.max_rank = max_rank;
    a.blockwise = blockwise;
    a.prof = nullptr;
    cudaError_t e = launch_update(Z, a, st);
    if (e != cudaSuccess) throw std::runtime_error(std::string("h2 update launch: ") + cudaGetErrorString(e));
    if (Z->bt->kind[Z->bt->find(t, r)] != INADM) mark_update(t, r);
    ++n_updates;
  }

  void temp_add(Temp& Tm, int a, int b, const double* A, int lda, const double* B, int ldb, const int* kdev,
                int kcap, double alpha) {
    Mark mk(ar);
    const int K2 = rcap + kcap;
    double* A2 = ar.alloc((size_t)Tm.ma * K2);
    double* B2 = ar.alloc((size_t)Tm.mb * K2);
    int* K = ar.ialloc();
    // alpha is folded into A: stack [T.A, alpha A]
    double* Aa = const_cast<double*>(A);
    if (alpha != 1.0) {
      Aa = ar.alloc((size_t)size(a) * kcap);
      gemm(Aa, size(a), A, lda, false, ident, lmax, false, dimc(size(a)), dimp(kdev), dimp(kdev), size(a), kcap,
           kcap, alpha, 0.0, st);  // A * (alpha I)
      lda = size(a);
    }
    {
      Group g;  // K = k_T + k_new and the two stacks read the old k_T only
      add_int(K, dimp(Tm.k), dimp(kdev), st);
      stack_cols(A2, Tm.ma, Tm.ma, Tm.A, Tm.ma, Tm.k, Aa, lda, T->lo[a] - T->lo[Tm.ra], size(a), dimp(kdev), K2, st);
      stack_cols(B2, Tm.mb, Tm.mb, Tm.B, Tm.mb, Tm.k, B, ldb, T->lo[b] - T->lo[Tm.rb], size(b), dimp(kdev), K2, st);
    }
    double* Ra = ar.alloc(KC * KC);
    double* Rb = ar.alloc(KC * KC);
    {
      Group g;
      tsqr_r(A2, Tm.ma, Tm.ma, dimp(K), Ra, KC, st);
      tsqr_r(B2, Tm.mb, Tm.mb, dimp(K), Rb, KC, st);
    }
    double* Ma = ar.alloc(KC * KC);
    double* Mb = ar.alloc(KC * KC);
    temp_core(Ra, Rb, KC, dimp(K), Ma, Mb, KC, Tm.k, rel, abs_tol, max_rank, rcap, Z->d.flags, kdev, st);
    {
      Group g;
      gemm(Tm.A, Tm.ma, A2, Tm.ma, false, Ma, KC, false, dimc(Tm.ma), dimp(Tm.k), dimp(K), Tm.ma, rcap, K2, 1.0, 0.0,
           st);
      gemm(Tm.B, Tm.mb, B2, Tm.mb, false, Mb, KC, false, dimc(Tm.mb), dimp(Tm.k), dimp(K), Tm.mb, rcap, K2, 1.0, 0.0,
           st);
    }
  }

  // add alpha A B^T at rows t, cols r of the target (temporary or the H^2 block (t, r) of Z)
  void add(Temp* tgt, int t, int r, const double* A, int lda, const double* B, int ldb, const int* kdev, int kcap,
           double alpha) {
    if (kcap == 0) return;
    if (tgt) {
      tgt->nz = true;
      // a zero device rank leaves the temporary unchanged (own-3): skip the whole truncated addition
      ExecCtx* c = exec_ctx();
      const int old_tag = c->skip_tag;
      c->skip_tag = 2;
      const size_t at = c->begin_skip(kdev);
      c->skip_tag = old_tag;
      temp_add(*tgt, t, r, A, lda, B, ldb, kdev, kcap, alpha);
      c->end_skip(at, exec_big_items());
      return;
    }
    const int b = Z->bt->find(t, r);
    if (Z->bt->kind[b] == INADM) {
      if (Z->blk2inad[b] < 0) return;
      gemm(Nptr(Z, b), lmax, A, lda, false, B, ldb, true, dimc(size(t)), dimc(size(r)), dimp(kdev), size(t), size(r),
           kcap, alpha, 1.0, st);
      ++n_dense;
      return;
    }
    update(t, r, A, lda, B, ldb, kdev, alpha);
  }

  // ---- Case 2 factors (reading R23) -----------------------------------------------
  // returns kcap (0: nothing to add); A: size(t) x k, B: size(r) x k; *kdev set on the device
  int factors(const HOp& X, const HOp& Y, int t, int s, int r, double** A, int* lda, double** B, int* ldb,
              int** kdev, bool dense_target) {
    const int kx = X.kind(t, s), ky = Y.kind(s, r);
    const int bx = X.bid(t, s), by = Y.bid(s, r);
    const int mt = size(t), ms = size(s), mr = size(r);
    *kdev = ar.ialloc();
    if (kx == ADM && ky == ADM) {
      if (X.Z->blk2adm[bx] < 0 || Y.Z->blk2adm[by] < 0) return 0;
      if (!nzr(X, t) || !nzc(Y, r)) return 0;  // min(k^X_t, k^Y_r) = 0
      const DevSide& Xr0 = X.rows();
      const DevSide& Yc0 = Y.cols();
      rank_if(*kdev, Xr0.rank + t, Yc0.rank + r, st);  // 0 iff min(k^X_t, k^Y_r) = 0 (c2core sets the rank)
      tag(3);
      open_pre_skip(*kdev);
      tag(9);
      const DevSide& Xr = X.rows();
      const DevSide& Xc = X.cols();
      const DevSide& Yr = Y.rows();
      const DevSide& Yc = Y.cols();
      double* Vx = ar.alloc((size_t)mt * rcap);
      double* Wy = ar.alloc((size_t)mr * rcap);
      double* Wxs = ar.alloc((size_t)ms * rcap);
      double* Vys = ar.alloc((size_t)ms * rcap);
      {
        Group g;  // four independent basis expansions
        expand_basis(X.Z->d, Xr, t, Vx, mt, st);
        expand_basis(Y.Z->d, Yc, r, Wy, mr, st);
        expand_basis(X.Z->d, Xc, s, Wxs, ms, st);
        expand_basis(Y.Z->d, Yr, s, Vys, ms, st);
      }
      const double* Sx = Sptr(X.Z, bx);
      const double* Sy = Sptr(Y.Z, by);
      double* Ca = ar.alloc(KC * KC);
      double* Cb = ar.alloc(KC * KC);
      // C = S^X (W^X_s^T V^Y_s) S^Y (S^X oriented k^X_t x k^X_s) and the factored side, one op
      if (ms <= case2_core_max_ms()) {
        case2_core(Wxs, Vys, ms, nullptr, Sx, X.Z->d.rcap, X.trans, Sy, Y.Z->d.rcap, Y.trans, Xr.rank + t,
                   Xc.rank + s, Yr.rank + s, Yc.rank + r, Ca, Cb, KC, *kdev, st);
      } else {
        double* G = ar.alloc(KC * KC);  // G = W^X_s^T V^Y_s (long inner dimension: its own op)
        gemm(G, KC, Wxs, ms, true, Vys, ms, false, dimp(Xc.rank + s), dimp(Yr.rank + s), dimc(ms), rcap, rcap, ms,
             1.0, 0.0, st);
        case2_core(nullptr, nullptr, ms, G, Sx, X.Z->d.rcap, X.trans, Sy, Y.Z->d.rcap, Y.trans, Xr.rank + t,
                   Xc.rank + s, Yr.rank + s, Yc.rank + r, Ca, Cb, KC, *kdev, st);
      }
      *A = ar.alloc((size_t)mt * rcap);
      *B = ar.alloc((size_t)mr * rcap);
      {
        Group g;
        gemm(*A, mt, Vx, mt, false, Ca, KC, false, dimc(mt), dimp(*kdev), dimp(Xr.rank + t), mt, rcap, rcap, 1.0, 0.0,
             st);
        gemm(*B, mr, Wy, mr, false, Cb, KC, false, dimc(mr), dimp(*kdev), dimp(Yc.rank + r), mr, rcap, rcap, 1.0, 0.0,
             st);
      }
      *lda = mt;
      *ldb = mr;
      return rcap;
    }
    if (kx == ADM) {
      if (X.Z->blk2adm[bx] < 0) return 0;
      if (!nzr(X, t)) return 0;  // k = k^X_t = 0
      const DevSide& Xr = X.rows();
      const DevSide& Xc = X.cols();
      set_int(*kdev, dimp(Xr.rank + t), st);
      if (ky == INADM && Y.Z->blk2inad[by] >= 0)
        zero_rank_if_zero_tile(Y.Z->d, Y.Z->blk2inad[by], ms * mr, *kdev, st);  // reading own-6
      tag(4);
      open_pre_skip(*kdev);
      tag(10);
      *A = ar.alloc((size_t)mt * rcap);
      double* Wxs = ar.alloc((size_t)ms * rcap);
      {
        Group g;
        expand_basis(X.Z->d, Xr, t, *A, mt, st);
        expand_basis(X.Z->d, Xc, s, Wxs, ms, st);
      }
      double* Dm = ar.alloc((size_t)ms * rcap);
      // D = W^X_s S^X_or^T  (ms x k^X_t)
      gemm(Dm, ms, Wxs, ms, false, Sptr(X.Z, bx), X.Z->d.rcap, !X.trans, dimc(ms), dimp(Xr.rank + t),
           dimp(Xc.rank + s), ms, rcap, rcap, 1.0, 0.0, st);
      *B = ar.alloc((size_t)mr * rcap);
      const HOp Yt = Y.t();
      hmul_dense(Y.Z->d, Yt.trans, r, s, 0, Dm, ms, dimp(Xr.rank + t), rcap, *B, mr, 1.0, 0.0, st);
      *lda = mt;
      *ldb = mr;
      return rcap;
    }
    if (ky == ADM) {
      if (Y.Z->blk2adm[by] < 0) return 0;
      if (!nzc(Y, r)) return 0;  // k = k^Y_r = 0
      const DevSide& Yr = Y.rows();
      const DevSide& Yc = Y.cols();
      set_int(*kdev, dimp(Yc.rank + r), st);
      if (kx == INADM && X.Z->blk2inad[bx] >= 0)
        zero_rank_if_zero_tile(X.Z->d, X.Z->blk2inad[bx], mt * ms, *kdev, st);  // reading own-6
      tag(5);
      open_pre_skip(*kdev);
      tag(11);
      double* Vys = ar.alloc((size_t)ms * rcap);
      *B = ar.alloc((size_t)mr * rcap);
      {
        Group g;
        expand_basis(Y.Z->d, Yr, s, Vys, ms, st);
        expand_basis(Y.Z->d, Yc, r, *B, mr, st);
      }
      double* Dm = ar.alloc((size_t)ms * rcap);
      // D = V^Y_s S^Y_or (ms x k^Y_r)
      gemm(Dm, ms, Vys, ms, false, Sptr(Y.Z, by), Y.Z->d.rcap, Y.trans, dimc(ms), dimp(Yc.rank + r),
           dimp(Yr.rank + s), ms, rcap, rcap, 1.0, 0.0, st);
      *A = ar.alloc((size_t)mt * rcap);
      hmul_dense(X.Z->d, X.trans, t, s, 0, Dm, ms, dimp(Yc.rank + r), rcap, *A, mt, 1.0, 0.0, st);
      *lda = mt;
      *ldb = mr;
      return rcap;
    }
    if (kx == INADM && ky == INADM && !dense_target) {
      // reading own-7: interpolative decomposition of the dense product (a zero tile gives r = 0)
      if (X.Z->blk2inad[bx] < 0 || Y.Z->blk2inad[by] < 0) return 0;
      tag(12);
      const int kc = std::min(mt, mr);
      *A = ar.alloc((size_t)mt * kc);
      *B = ar.alloc((size_t)mr * kc);
      dd_compress(X.Z->d, X.Z->blk2inad[bx], X.trans, Y.Z->d, Y.Z->blk2inad[by], Y.trans, mt, ms, mr, *A, mt, *B,
                  mr, *kdev, 1e-12, st);
      *lda = mt;
      *ldb = mr;
      return kc;
    }
    if (kx == INADM) {
      if (X.Z->blk2inad[bx] < 0) return 0;
      set_int(*kdev, dimc(ms), st);
      zero_rank_if_zero_tile(X.Z->d, X.Z->blk2inad[bx], mt * ms, *kdev, st);  // reading own-6
      if (ky == INADM && Y.Z->blk2inad[by] >= 0) zero_rank_if_zero_tile(Y.Z->d, Y.Z->blk2inad[by], ms * mr, *kdev, st);
      tag(7);
      open_pre_skip(*kdev);
      tag(13);
      *A = ar.alloc((size_t)mt * ms);
      if (X.trans) transpose_tile(*A, mt, Nptr(X.Z, bx), lmax, mt, ms, st);
      else copy_cols(*A, mt, Nptr(X.Z, bx), lmax, mt, dimc(ms), ms, st);
      *B = ar.alloc((size_t)mr * ms);
      const HOp Yt = Y.t();
      hmul_dense(Y.Z->d, Yt.trans, r, s, 1 /* D = I */, ident, lmax, dimc(ms), ms, *B, mr, 1.0, 0.0, st);
      *lda = mt;
      *ldb = mr;
      return ms;
    }
    // ky == INADM
    if (Y.Z->blk2inad[by] < 0) return 0;
    set_int(*kdev, dimc(mr), st);
    zero_rank_if_zero_tile(Y.Z->d, Y.Z->blk2inad[by], ms * mr, *kdev, st);  // reading own-6
    tag(8);
    open_pre_skip(*kdev);
    tag(14);
    double* Ny = ar.alloc((size_t)ms * mr);
    if (Y.trans) transpose_tile(Ny, ms, Nptr(Y.Z, by), lmax, ms, mr, st);
    else copy_cols(Ny, ms, Nptr(Y.Z, by), lmax, ms, dimc(mr), mr, st);
    *A = ar.alloc((size_t)mt * mr);
    hmul_dense(X.Z->d, X.trans, t, s, 0, Ny, ms, dimc(mr), mr, *A, mt, 1.0, 0.0, st);
    *B = ident;
    *lda = mt;
    *ldb = lmax;
    return mr;
  }

  bool target_stored(int t, int r) const {
    if (Z->bt->find(t, r) < 0) return false;
    return !Z->lower || T->lo[t] >= T->lo[r];
  }

  // ---- product: Z|_{t x r} += alpha X|_{t x s} Y|_{s x r} --------------------------------------
  void addmul(double alpha, const HOp& X, const HOp& Y, int t, int s, int r, Temp* tgt) {
    if (!X.stored(t, s) || !Y.stored(s, r)) return;
    const int kx = X.kind(t, s), ky = Y.kind(s, r);
    if (kx == SUBDIV && ky == SUBDIV) {
      const std::vector<int> S2 = sons_plus(s), T2 = sons_plus(t), R2 = sons_plus(r);
      if (!tgt) {
        const int kz = Z->bt->kind[Z->bt->find(t, r)];
        if (kz == ADM) {
          Mark mk(ar);
          std::vector<Temp> temps;
          for (int t2 : T2)
            for (int r2 : R2) {
              Temp tm{t2, r2, size(t2), size(r2), ar.alloc((size_t)size(t2) * rcap), ar.alloc((size_t)size(r2) * rcap),
                      ar.ialloc(), false};
              set_int(tm.k, dimc(0), st);
              temps.push_back(tm);
            }
          n_temps += (long long)temps.size();
          for (int s2 : S2)
            for (size_t i = 0; i < T2.size(); ++i)
              for (size_t j = 0; j < R2.size(); ++j) addmul(alpha, X, Y, T2[i], s2, R2[j], &temps[i * R2.size() + j]);
          // merge: 4 zero-extended local updates into (t, r), order (1,1),(1,2),(2,1),(2,2)
          for (size_t i = 0; i < T2.size(); ++i)
            for (size_t j = 0; j < R2.size(); ++j) {
              const Temp& tm = temps[i * R2.size() + j];
              if (!tm.nz) continue;  // nothing of possibly non-zero rank was added
              Mark mk2(ar);
              double* A = ar.alloc((size_t)size(t) * rcap);
              double* B = ar.alloc((size_t)size(r) * rcap);
              tag(0);
              const size_t pre = exec_ctx()->begin_skip(tm.k);  // a rank-0 temporary adds nothing
              {
                Group g;
                stack_cols(A, size(t), size(t), nullptr, 0, nullptr, tm.A, tm.ma, T->lo[tm.ra] - T->lo[t], tm.ma,
                           dimp(tm.k), rcap, st);
                stack_cols(B, size(r), size(r), nullptr, 0, nullptr, tm.B, tm.mb, T->lo[tm.rb] - T->lo[r], tm.mb,
                           dimp(tm.k), rcap, st);
              }
              tag(1);
              add(nullptr, t, r, A, size(t), B, size(r), tm.k, rcap, 1.0);
              exec_ctx()->end_skip(pre, exec_big_items());
            }
          return;
        }
        for (int s2 : S2)
          for (int t2 : T2)
            for (int r2 : R2)
              if (target_stored(t2, r2)) addmul(alpha, X, Y, t2, s2, r2, nullptr);
        return;
      }
      for (int s2 : S2)
        for (int t2 : T2)
          for (int r2 : R2) addmul(alpha, X, Y, t2, s2, r2, tgt);
      return;
    }
    Mark mk(ar);
    double *A, *B;
    int lda, ldb;
    int* kdev;
    const bool dense_target = !tgt && Z->bt->kind[Z->bt->find(t, r)] == INADM;
    pre_skip = NO_SKIP;
    const int kcap = factors(X, Y, t, s, r, &A, &lda, &B, &ldb, &kdev, dense_target);
    const size_t ps = pre_skip;
    pre_skip = NO_SKIP;
    if (kcap) add(tgt, t, r, A, lda, B, ldb, kdev, kcap, alpha);
    if (ps != NO_SKIP) exec_ctx()->end_skip(ps, exec_big_items());
  }

  // ---- dense-right-hand-side substitutions with the factor (in place on B) ---------------------
  int diag_slot(int t) const { return Z->blk2inad[Z->bt->find(t, t)]; }

  void lsolve(int t, double* B, int ldb, Dim m, int mcap, bool unit) {
    if (leaf(t)) {
      tile_trsm(Z->d, diag_slot(t), size(t), unit ? LLU : LLN, B, ldb, size(t), m, mcap, st);
      return;
    }
    const int t1 = T->son0[t], t2 = T->son1[t], n1 = size(t1);
    lsolve(t1, B, ldb, m, mcap, unit);
    hmul_dense(Z->d, false, t2, t1, 0, B, ldb, m, mcap, B + n1, ldb, -1.0, 1.0, st);
    lsolve(t2, B + n1, ldb, m, mcap, unit);
  }
  void ltsolve(int t, double* B, int ldb, Dim m, int mcap) {
    if (leaf(t)) {
      tile_trsm(Z->d, diag_slot(t), size(t), LLT, B, ldb, size(t), m, mcap, st);
      return;
    }
    const int t1 = T->son0[t], t2 = T->son1[t], n1 = size(t1);
    ltsolve(t2, B + n1, ldb, m, mcap);
    hmul_dense(Z->d, true, t1, t2, 0, B + n1, ldb, m, mcap, B, ldb, -1.0, 1.0, st);
    ltsolve(t1, B, ldb, m, mcap);
  }
  void usolve(int t, double* B, int ldb, Dim m, int mcap) {
    if (leaf(t)) {
      tile_trsm(Z->d, diag_slot(t), size(t), LUN, B, ldb, size(t), m, mcap, st);
      return;
    }
    const int t1 = T->son0[t], t2 = T->son1[t], n1 = size(t1);
    usolve(t2, B + n1, ldb, m, mcap);
    hmul_dense(Z->d, false, t1, t2, 0, B + n1, ldb, m, mcap, B, ldb, -1.0, 1.0, st);
    usolve(t1, B, ldb, m, mcap);
  }
  void utsolve(int t, double* B, int ldb, Dim m, int mcap) {
    if (leaf(t)) {
      tile_trsm(Z->d, diag_slot(t), size(t), LUT, B, ldb, size(t), m, mcap, st);
      return;
    }
    const int t1 = T->son0[t], t2 = T->son1[t], n1 = size(t1);
    utsolve(t1, B, ldb, m, mcap);
    hmul_dense(Z->d, true, t2, t1, 0, B, ldb, m, mcap, B + n1, ldb, -1.0, 1.0, st);
    utsolve(t2, B + n1, ldb, m, mcap);
  }

  // ---- block substitutions in place (reading R8 for admissible leaves) --------------
  void rfs_common(int t, int s, bool chol) {
    const int b = Z->bt->find(t, s);
    const int k = Z->bt->kind[b];
    if (k == INADM) {
      if (Z->blk2inad[b] < 0) return;
      tile_trsm(Z->d, diag_slot(s), size(s), chol ? RLT : RUN, Nptr(Z, b), lmax, size(t), dimc(size(s)), size(s), st);
      return;
    }
    if (k == ADM) {
      if (Z->blk2adm[b] < 0) return;
      if (!Z->nzr[t] || !Z->nzc[s]) return;  // k_t l_s = 0 structurally (oracle: S.size == 0)
      Mark mk(ar);
      const int mt = size(t), ms = size(s);
      int* kdev = ar.ialloc();
      double* Zs = ar.alloc((size_t)ms * rcap);
      double* Vt = ar.alloc((size_t)mt * rcap);
      rank_if(kdev, Z->d.row.rank + t, Z->d.col.rank + s, st);  // rank 0 block -> nothing (oracle: S.size == 0)
      tag(6);
      const size_t pre = exec_ctx()->begin_skip(kdev);  // a rank-0 block needs no solve (reading R8)
      {
        Group g;  // the solves below touch Zs only
        expand_basis(Z->d, Z->d.col, s, Zs, ms, st);
        expand_basis(Z->d, Z->d.row, t, Vt, mt, st);
      }
      if (chol) lsolve(s, Zs, ms, dimp(Z->d.col.rank + s), rcap, false);
      else utsolve(s, Zs, ms, dimp(Z->d.col.rank + s), rcap);
      double* U = ar.alloc((size_t)mt * rcap);
      gemm(U, mt, Vt, mt, false, Sptr(Z, b), Z->d.rcap, false, dimc(mt), dimp(Z->d.col.rank + s),
           dimp(Z->d.row.rank + t), mt, rcap, rcap, 1.0, 0.0, st);
      exec_ctx()->end_skip(pre, exec_big_items());
      zero_fill(Sptr(Z, b), (size_t)Z->d.rcap * Z->d.rcap, st);
      tag(15);
      update(t, s, U, mt, Zs, ms, kdev, 1.0);
      return;
    }
    if (leaf(s)) {
      for (int t2 : sons_plus(t)) rfs_common(t2, s, chol);
      return;
    }
    const int s1 = T->son0[s], s2 = T->son1[s];
    const HOp L{Z, false};
    for (int t2 : sons_plus(t)) {
      rfs_common(t2, s1, chol);
      addmul(-1.0, L, chol ? L.t() : L, t2, s1, s2, nullptr);
      rfs_common(t2, s2, chol);
    }
  }

  void lfs(int t, int s) {
    const int b = Z->bt->find(t, s);
    const int k = Z->bt->kind[b];
    if (k == INADM) {
      if (Z->blk2inad[b] < 0) return;
      tile_trsm(Z->d, diag_slot(t), size(t), LLU, Nptr(Z, b), lmax, size(t), dimc(size(s)), size(s), st);
      return;
    }
    if (k == ADM) {
      if (Z->blk2adm[b] < 0) return;
      if (!Z->nzr[t] || !Z->nzc[s]) return;  // k_t l_s = 0 structurally
      Mark mk(ar);
      const int mt = size(t), ms = size(s);
      int* kdev = ar.ialloc();
      double* Vt = ar.alloc((size_t)mt * rcap);
      double* Ws = ar.alloc((size_t)ms * rcap);
      rank_if(kdev, Z->d.row.rank + t, Z->d.col.rank + s, st);
      tag(6);
      const size_t pre = exec_ctx()->begin_skip(kdev);
      {
        Group g;  // the solve below touches Vt only
        expand_basis(Z->d, Z->d.row, t, Vt, mt, st);
        expand_basis(Z->d, Z->d.col, s, Ws, ms, st);
      }
      lsolve(t, Vt, mt, dimp(Z->d.row.rank + t), rcap, true);
      double* U = ar.alloc((size_t)mt * rcap);
      gemm(U, mt, Vt, mt, false, Sptr(Z, b), Z->d.rcap, false, dimc(mt), dimp(Z->d.col.rank + s),
           dimp(Z->d.row.rank + t), mt, rcap, rcap, 1.0, 0.0, st);
      exec_ctx()->end_skip(pre, exec_big_items());
      zero_fill(Sptr(Z, b), (size_t)Z->d.rcap * Z->d.rcap, st);
      tag(15);
      update(t, s, U, mt, Ws, ms, kdev, 1.0);
      return;
    }
    if (leaf(t)) {
      for (int s2 : sons_plus(s)) lfs(t, s2);
      return;
    }
    const int t1 = T->son0[t], t2 = T->son1[t];
    const HOp L{Z, false};
    for (int s2 : sons_plus(s)) {
      lfs(t1, s2);
      addmul(-1.0, L, L, t2, t1, s2, nullptr);
      lfs(t2, s2);
    }
  }

  void chol(int t) {
    if (leaf(t)) {
      tile_potrf(Z->d, diag_slot(t), t, st);
      return;
    }
    const int t1 = T->son0[t], t2 = T->son1[t];
    chol(t1);
    rfs_common(t2, t1, true);
    const HOp L{Z, false};
    addmul(-1.0, L, L.t(), t2, t1, t2, nullptr);
    chol(t2);
  }

  // ---- approximate inverse (Remark 1) --------------------------
  // Z|_{t x s} <- 0: the couplings of the admissible leaves and the tiles of the inadmissible leaves
  // of the block subtree (contiguous slot ranges); the bases are left as they are
  void zero_block(int t, int s) {
    const h2_btree_* B = Z->bt;
    const int b = B->find(t, s);
    int a0 = -1, a1 = -1;
    for (int q = b; q < b + B->bsize[b]; ++q)
      if (Z->blk2adm[q] >= 0) {
        if (a0 < 0) a0 = Z->blk2adm[q];
        a1 = Z->blk2adm[q];
      }
    const size_t r2 = (size_t)Z->d.rcap * Z->d.rcap, l2 = (size_t)lmax * lmax;
    if (a0 >= 0) zero_fill(Z->d.S + (size_t)a0 * r2, (size_t)(a1 - a0 + 1) * r2, st);
    const int i0 = Z->inad_range[2 * b], i1 = Z->inad_range[2 * b + 1];
    if (i1 > i0) zero_fill(Z->d.N + (size_t)i0 * l2, (size_t)(i1 - i0) * l2, st);
  }
  // in place Z|_{t x t} <- (Z|_{t x t})^{-1}; dT drives the scratch matrix T (zero on entry)
  void inv(int t, Driver& dT) {
    if (leaf(t)) {
      tile_inverse(Z->d, diag_slot(t), t, st);
      return;
    }
    const int t1 = T->son0[t], t2 = T->son1[t];
    const HOp C{Z, false}, W{dT.Z, false};
    inv(t1, dT);
    dT.addmul(1.0, C, C, t1, t1, t2, nullptr);  // B12 = C11 A12      -> T|_{t1 x t2}
    dT.addmul(1.0, C, C, t2, t1, t1, nullptr);  // B21 = A21 C11      -> T|_{t2 x t1}
    addmul(-1.0, C, W, t2, t1, t2, nullptr);    // S = A22 - A21 B12 (P:1382 prints A11: R20)
    inv(t2, dT);                                // C22 = S^{-1}
    zero_block(t1, t2);
    addmul(-1.0, W, C, t1, t2, t2, nullptr);    // C12 = -B12 C22
    zero_block(t2, t1);
    addmul(-1.0, C, W, t2, t2, t1, nullptr);    // C21 = -C22 B21
    addmul(-1.0, C, W, t1, t2, t1, nullptr);    // C11 = C11 - C12 B21
  }

  void lr(int t) {
    if (leaf(t)) {
      tile_getrf(Z->d, diag_slot(t), t, st);
      return;
    }
    const int t1 = T->son0[t], t2 = T->son1[t];
    lr(t1);
    lfs(t1, t2);
    rfs_common(t2, t1, false);
    const HOp L{Z, false};
    addmul(-1.0, L, L, t2, t1, t2, nullptr);
    lr(t2);
  }
};

h2_status ensure_ws(h2_mat_* Z, Arena& ar) {
  MatDev& M = Z->d;
  for (DevSide* D : {&M.row, &M.col}) {
    if (!D->hx) {
      CUDA_TRY(cudaMalloc(&D->hx, sizeof(double) * (size_t)D->nclusters * M.rcap * KC));
      Z->allocs.push_back(D->hx);
      h2::poison(D->hx, sizeof(double) * (size_t)D->nclusters * M.rcap * KC);
      CUDA_TRY(cudaMalloc(&D->hy, sizeof(double) * (size_t)D->nclusters * M.rcap * KC));
      Z->allocs.push_back(D->hy);
      h2::poison(D->hy, sizeof(double) * (size_t)D->nclusters * M.rcap * KC);
    }
  }
  if (!Z->ws) {
    const size_t n = (size_t)Z->bt->rt->n;
    Z->ws_cap = 24 * n * (size_t)KC + ((size_t)1 << 22);
    CUDA_TRY(cudaMalloc(&Z->ws, sizeof(double) * Z->ws_cap));
    Z->allocs.push_back(Z->ws);
    h2::poison(Z->ws, sizeof(double) * Z->ws_cap);
    Z->iws_cap = 1 << 20;
    CUDA_TRY(cudaMalloc(&Z->iws, sizeof(int) * Z->iws_cap));
    Z->allocs.push_back(Z->iws);
  }
  ar.d = Z->ws;
  ar.cap = Z->ws_cap;
  ar.top = 0;
  ar.i = Z->iws;
  ar.icap = Z->iws_cap;
  ar.itop = 0;
  return H2_OK;
}

h2_status run_driver(h2_mat_* Z, const h2_trunc* trunc, h2_stream stream, int what, h2_mat_* X, h2_mat_* Y,
                     double alpha, double* vec, int nrhs, int64_t ldx) {
  if (Z->bt->rt != Z->bt->ct) {
    h2::set_error("factorization/product need one shared cluster tree for rows and columns");
    return H2_ERR_ARG;
  }
  if (Z->d.lmax > 64) {
    h2::set_error("leaf clusters larger than 64 are not supported");
    return H2_ERR_ARG;
  }
  const h2_trunc tc = trunc ? *trunc : h2_trunc{1e-4, 0.0, 0, 0};
  if (what != 3 && what != 4) {  // everything but the solves changes the target (packed matvec copies)
    Z->version++;
    if (what == 5 && X) X->version++;
  }
  Arena ar;
  h2_status s;
  if ((s = ensure_ws(Z, ar)) != H2_OK) return s;
  for (h2_mat_* M : {X, Y})
    if (M && M != Z) {
      Arena dummy;
      if ((s = ensure_ws(M, dummy)) != H2_OK) return s;
    }
  // update workspace of the target(s)
  for (h2_mat_* Tg : {Z, what == 5 ? X : nullptr}) {
    if (!Tg) continue;
    for (DevSide* D : {&Tg->d.row, &Tg->d.col})
      if (!D->re) {
        const size_t nc = D->nclusters, k2 = (size_t)Tg->d.kcap * Tg->d.kcap;
        CUDA_TRY(cudaMalloc(&D->re, 8 * nc * k2));
        Tg->allocs.push_back(D->re);
        h2::poison(D->re, 8 * nc * k2);
        CUDA_TRY(cudaMalloc(&D->bw, 8 * nc * k2));
        Tg->allocs.push_back(D->bw);
        h2::poison(D->bw, 8 * nc * k2);
        CUDA_TRY(cudaMalloc(&D->rn, 8 * nc * k2));
        Tg->allocs.push_back(D->rn);
        h2::poison(D->rn, 8 * nc * k2);
        CUDA_TRY(cudaMalloc(&D->qn, 8 * nc * (size_t)Tg->d.ldq * Tg->d.rcap));
        Tg->allocs.push_back(D->qn);
        h2::poison(D->qn, 8 * nc * (size_t)Tg->d.ldq * Tg->d.rcap);
        CUDA_TRY(cudaMalloc(&D->rnew, 4 * nc));
        Tg->allocs.push_back(D->rnew);
      }
  }
  Arena arT;  // the scratch matrix of the inversion drives its own products
  if (what == 5 && (s = ensure_ws(X, arT)) != H2_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  Driver dr{Z, st, tc.rel_tol, tc.abs_tol, tc.max_rank, tc.blockwise != 0, ar, Z->bt->rt, Z->d.rcap, Z->d.lmax};
  ExecCtx ctx;
  exec_begin(&ctx, st);  // the recursion records ops; the device executor runs them (exec.h)
  try {
    dr.ident = ar.alloc((size_t)Z->d.lmax * Z->d.lmax);
    identity(dr.ident, Z->d.lmax, Z->d.lmax, st);
    if (what == 0) dr.chol(0);
    else if (what == 1) dr.lr(0);
    else if (what == 2) dr.addmul(alpha, HOp{X, false}, HOp{Y, false}, 0, 0, 0, nullptr);
    else if (what == 5) {
      Driver dT{X, st, tc.rel_tol, tc.abs_tol, tc.max_rank, tc.blockwise != 0, arT, X->bt->rt, X->d.rcap, X->d.lmax};
      dT.ident = arT.alloc((size_t)X->d.lmax * X->d.lmax);
      identity(dT.ident, X->d.lmax, X->d.lmax, st);
      dr.inv(0, dT);
      dr.n_updates += dT.n_updates;
      dr.n_dense += dT.n_dense;
      dr.n_temps += dT.n_temps;
    }
    else if (what == 3 || what == 4) {
      // vec: n x nrhs in ORIGINAL order -> tree order, solve, back
      const int n = (int)Z->bt->rt->n;
      double* Bt = ar.alloc((size_t)n * nrhs);
      gather_cols(Bt, vec, Z->d.row.perm, n, nrhs, ldx, st);
      if (what == 3) {
        dr.lsolve(0, Bt, n, dimc(nrhs), nrhs, false);
        dr.ltsolve(0, Bt, n, dimc(nrhs), nrhs);
      } else {
        dr.lsolve(0, Bt, n, dimc(nrhs), nrhs, true);
        dr.usolve(0, Bt, n, dimc(nrhs), nrhs);
      }
      scatter_cols(vec, Bt, Z->d.row.perm, n, nrhs, ldx, st);
    }
  } catch (const std::exception& e) {
    exec_end();
    h2::set_error(e.what());
    return H2_ERR_NOMEM;
  }
  CUDA_TRY(exec_end());
  CUDA_TRY(cudaGetLastError());
  Z->stats[0] += dr.n_updates;
  Z->stats[1] += dr.n_dense;
  Z->stats[2] += dr.n_temps;
  return H2_OK;
}

}  // namespace

extern "C" h2_status h2_lr_factor(h2_mat A, h2_factor_kind kind, const h2_trunc* trunc, h2_stream stream) {
  if (h2::batch_open()) {
    h2::set_error("h2_lr_factor: not allowed inside h2_batch_begin/h2_batch_end");
    return H2_ERR_ARG;
  }
  if (!A) {
    h2::set_error("h2_lr_factor: NULL matrix");
    return H2_ERR_ARG;
  }
  if (kind == H2_CHOLESKY && !A->lower) {
    h2::set_error("h2_lr_factor: Cholesky needs H2_LOWER storage");
    return H2_ERR_ARG;
  }
  if (kind == H2_LR && A->lower) {
    h2::set_error("h2_lr_factor: LR needs H2_FULL storage");
    return H2_ERR_ARG;
  }
  if (A->factored) {
    h2::set_error("h2_lr_factor: matrix is already factored");
    return H2_ERR_ARG;
  }
  h2_status s = run_driver(A, trunc, stream, kind == H2_CHOLESKY ? 0 : 1, nullptr, nullptr, 0.0, nullptr, 0, 0);
  if (s == H2_OK) A->factored = kind == H2_CHOLESKY ? 1 : 2;
  return s;
}

extern "C" h2_status h2_inverse(h2_mat A, const h2_trunc* trunc, h2_stream stream) {
  if (h2::batch_open()) {
    h2::set_error("h2_inverse: not allowed inside h2_batch_begin/h2_batch_end");
    return H2_ERR_ARG;
  }
  if (!A) {
    h2::set_error("h2_inverse: NULL matrix");
    return H2_ERR_ARG;
  }
  if (A->lower || A->factored) {
    h2::set_error("h2_inverse: needs an unfactored H2_FULL matrix");
    return H2_ERR_ARG;
  }
  // scratch matrix T (same trees and capacities, zero): B12 / B21 of every level
  const int64_t n = A->bt->rt->n;
  std::vector<int64_t> rowptr((size_t)n + 1, 0);
  h2_mat T = nullptr;
  h2_status s = h2_from_sparse(A->bt, n, rowptr.data(), nullptr, nullptr, H2_FULL, A->d.rcap, A->d.ucap, stream, &T);
  if (s != H2_OK) return s;
  s = run_driver(A, trunc, stream, 5, T, nullptr, 0.0, nullptr, 0, 0);
  cudaStreamSynchronize((cudaStream_t)stream);  // T's memory is released below
  h2_mat_destroy(T);
  return s;
}

extern "C" h2_status h2_addmul(h2_mat Z, double alpha, h2_mat X, h2_mat Y, const h2_trunc* trunc, h2_stream stream) {
  if (h2::batch_open()) {
    h2::set_error("h2_addmul: not allowed inside h2_batch_begin/h2_batch_end");
    return H2_ERR_ARG;
  }
  if (!Z || !X || !Y) {
    h2::set_error("h2_addmul: NULL matrix");
    return H2_ERR_ARG;
  }
  if (Z->bt->rt != X->bt->rt || Z->bt->rt != Y->bt->rt || Z->bt->ct != X->bt->ct || Z->bt->ct != Y->bt->ct) {
    h2::set_error("h2_addmul: Z, X and Y must share their cluster trees");
    return H2_ERR_ARG;
  }
  if (Z == X || Z == Y) {
    h2::set_error("h2_addmul: Z must not alias X or Y (aliasing happens only inside h2_lr_factor)");
    return H2_ERR_ARG;
  }
  if (X->lower || Y->lower) {
    h2::set_error("h2_addmul: factors in H2_LOWER storage are not supported");
    return H2_ERR_ARG;
  }
  if (!std::isfinite(alpha)) {
    h2::set_error("h2_addmul: non-finite alpha");
    return H2_ERR_NONFINITE;
  }
  if (alpha == 0.0) return H2_OK;
  return run_driver(Z, trunc, stream, 2, X, Y, alpha, nullptr, 0, 0);
}

extern "C" h2_status h2_solve(h2_mat F, double* x, int32_t nrhs, int64_t ldx, h2_stream stream) {
  if (h2::batch_open()) {
    h2::set_error("h2_solve: not allowed inside h2_batch_begin/h2_batch_end");
    return H2_ERR_ARG;
  }
  if (!F || !x) {
    h2::set_error("h2_solve: NULL argument");
    return H2_ERR_ARG;
  }
  if (!F->factored) {
    h2::set_error("h2_solve: matrix is not factored (call h2_lr_factor first)");
    return H2_ERR_ARG;
  }
  if (nrhs < 1 || nrhs > 64 || ldx < F->bt->rt->n) {
    h2::set_error("h2_solve: need 1 <= nrhs <= 64 and ldx >= n");
    return H2_ERR_SHAPE;
  }
  cudaError_t e = h2::solve_factored(F, x, nrhs, ldx, (cudaStream_t)stream);
  if (e != cudaSuccess) {
    h2::set_error(std::string("h2_solve: ") + cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? H2_ERR_NOMEM : H2_ERR_CUDA;
  }
  return H2_OK;
}
