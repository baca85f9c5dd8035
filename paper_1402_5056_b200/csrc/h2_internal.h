// Internal structures of the B200 H^2 library (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <array>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/h2.h"
#include "h2_prof.h"

namespace h2 {

constexpr int KCAP_MAX = 96;  // extended rank capacity (rank_cap + update_cap) handled by the kernels
constexpr int RCAP_MAX = 48;  // stored rank capacity (2 * rank_cap <= KCAP_MAX rows of V^_t)
constexpr int LMAX_MAX = 64;  // largest leaf cluster handled by the kernels
constexpr int NTHREADS = 256; // threads per CTA of the small-matrix kernels
constexpr int MV_SUB_LEAVES = 64;  // leaves per matvec subtree CTA (h2_matvec.cu)

enum { SUBDIV = 0, ADM = 1, INADM = 2 };

}  // namespace h2

struct h2_tree_ {
  int64_t n = 0;
  int dim = 0, leaf = 0;
  int nclusters = 0, depth = 0;
  std::vector<int64_t> perm;
  std::vector<int32_t> lo, hi, son0, son1, parent, level, tsize;
  std::vector<char> ddpair;             // the two sons are decoupled domains (h2_cluster_tree_dd)
  std::vector<double> bmin, bmax;       // nclusters * dim
  std::vector<int32_t> bfs, level_ptr;  // clusters sorted by (level, id); level_ptr[depth+2]
  std::vector<int32_t> leaf_index;      // cluster -> leaf ordinal (or -1)
  std::vector<int32_t> leaves;          // leaf ordinal -> cluster
  bool in_subtree(int t, int root) const { return t >= root && t < root + tsize[root]; }
};

struct h2_btree_ {
  h2_tree_* rt = nullptr;
  h2_tree_* ct = nullptr;
  double eta = 0;
  std::vector<int32_t> t, s, parent, bsize;
  std::vector<int8_t> kind;
  std::vector<std::array<int32_t, 4>> sons;
  std::vector<int8_t> nsons;
  std::unordered_map<int64_t, int32_t> index;  // key t * ct->nclusters + s
  int csp = 0;
  int32_t find(int a, int b) const {
    auto it = index.find((int64_t)a * ct->nclusters + b);
    return it == index.end() ? -1 : it->second;
  }
};

namespace h2 {

// One cluster-basis family (row: V/E, column: W/F) resident on the device.
struct DevSide {
  const h2_tree_* tree = nullptr;
  int nclusters = 0, nleaves = 0;
  // structure
  int32_t *lo = nullptr, *hi = nullptr, *son0 = nullptr, *son1 = nullptr, *parent = nullptr,
          *tsize = nullptr, *leafidx = nullptr, *bfs = nullptr, *level = nullptr, *leaves = nullptr;
  int32_t *bptr = nullptr, *bidx = nullptr;  // admissible stored blocks per cluster (CSR of adm slots)
  int64_t* perm = nullptr;
  // data
  int32_t* rank = nullptr;  // k_t
  double* leafb = nullptr;  // nleaves * lmax * rcap        (V_t, |t| x k_t, ld lmax)
  double* tr = nullptr;     // nclusters * rcap * rcap       (E_t, k_t x k_parent, ld rcap)
  double* rc = nullptr;     // nclusters * rcap * rcap       (R-factor of V_t, k_t x k_t padded, ld rcap)
  // update workspace (indexed by cluster id), ld kcap
  double* re = nullptr;     // R-factor of the extended basis V~_t         (kcap x kcap)
  double* bw = nullptr;     // weight B~_t (square padded)                   (kcap x kcap)
  double* rn = nullptr;     // basis change R_t = Q_t^T V~_t (r_t x K_t)      (kcap x kcap)
  double* qn = nullptr;     // new leaf basis (lmax x rcap) or Qhat_t (2rcap x rcap), ld max(lmax,2rcap)
  int32_t* rnew = nullptr;  // new ranks
  // matvec workspace
  double* xh = nullptr;     // nclusters * rcap coefficients
  int32_t* mvsync = nullptr;  // matvec: nclusters arrival counters (forward-transform climb)
  int32_t* anc = nullptr;     // matvec: per leaf ordinal its ancestors by level (ancw ints, -1 padded)
  int ancw = 0;
  // matvec schedule (h2_matvec.cu): the maximal subtrees with at most MV_SUB_LEAVES leaves, one
  // CTA each, and the clusters above them ("top", by level, root first)
  int32_t* mv_roots = nullptr;
  int n_mv_roots = 0;
  int32_t* mv_top = nullptr;      // top clusters grouped by level, ascending
  int32_t* mv_top_lptr = nullptr; // level l of the top: mv_top[mv_top_lptr[l] .. mv_top_lptr[l+1])
  int mv_top_nlev = 0;
  std::vector<int32_t> h_top_lptr;  // host copy of mv_top_lptr
  int32_t* mv_cnt = nullptr;        // [0] subtrees published, [1] top pass done (epoch counters, never reset); [2] couplings' arrival counter
  unsigned mv_epoch = 0;            // products whose forward transform ran on this side
  double* hx = nullptr;     // H^2-block x dense workspace: nclusters * rcap * 64 (forward coefficients)
  double* hy = nullptr;     // nclusters * rcap * 64 (coupling/backward coefficients)
};

// Everything a device kernel needs for one local update (passed by value).
struct UpdArgs {
  // row side (A) and column side (B) roots and update rank
  int t0, s0, k;
  const double* X;
  int64_t ldx;
  const double* Y;
  int64_t ldy;
  double alpha;
  double rel_tol, abs_tol;
  int max_rank;
  int blockwise;  // h2_trunc.blockwise (reading own-10): block-relative weighting, absolute threshold
  double* prof;  // device flop/byte counters (profiling) or nullptr
  const int* kdev;  // if set, the update rank is read from device memory (internal callers)
};

struct MatDev {
  int rcap, ucap, kcap, lmax, ldq;
  DevSide row, col;
  int nadm, ninad;
  int32_t *adm_t = nullptr, *adm_s = nullptr;
  double* S = nullptr;  // nadm * rcap * rcap (k_t x l_s, ld rcap)
  int32_t *in_t = nullptr, *in_s = nullptr;
  double* N = nullptr;  // ninad * lmax * lmax (|t| x |s|, ld lmax)
  int32_t *nptr = nullptr, *nidx = nullptr;    // inadmissible stored blocks per row leaf (CSR)
  int32_t *ntptr = nullptr, *ntidx = nullptr;  // inadmissible stored blocks per column leaf (CSR)
  int32_t* flags = nullptr;
  int32_t* updlog = nullptr;  // diagnostic (H2_UPD_LOG): (t0, s0, k) of every non-zero-rank local update
  double *xt = nullptr, *yt = nullptr;  // tree-order vectors
};

}  // namespace h2

// Schedule of one sequential block substitution sweep (h2_solve.cu), device arrays, built once.
struct SolveSched {
  int built = 0, nl = 0;
  int32_t *order = nullptr, *diag = nullptr;            // leaf cluster / diagonal tile slot per position
  int32_t *near_ptr = nullptr, *near_slot = nullptr, *near_src = nullptr;  // off-diagonal tiles per position
  int32_t *enter_ptr = nullptr, *enter = nullptr;       // destination clusters entered (top-down)
  int32_t *done_ptr = nullptr, *done = nullptr;         // source clusters completed (bottom-up)
  int32_t *push_ptr = nullptr, *push_slot = nullptr, *push_dst = nullptr;  // per source cluster
};

// Packed copies of the couplings and transfer matrices at the current ranks for the matvec
// (h2_matvec.cu: ensure_packed), valid while version == h2_mat_::version.
struct MvPack {
  double* Sp = nullptr;
  int64_t* Soff = nullptr;                 // nadm + 1
  double* Tp[2] = {nullptr, nullptr};      // row / column side transfers (k_c x k_p, ld k_c)
  double* TpT[2] = {nullptr, nullptr};     // the same matrices transposed (k_p x k_c, ld k_p): forward transform
  int64_t* Toff[2] = {nullptr, nullptr};   // nclusters + 1
  size_t capS = 0, capT[2] = {0, 0}, capTT[2] = {0, 0};
  // per block of row(t) / col(s), in the order of DevSide::bidx: {offset in Sp, partner, partner's rank}
  struct Desc {
    long long off;
    int partner, krank;
  };
  Desc* desc[2] = {nullptr, nullptr};
  long long version = -1;
};

struct h2_mat_ {
  h2_btree_* bt = nullptr;
  long long version = 0;  // bumped by every call that changes ranks, bases or couplings
  MvPack mvpack;
  bool lower = false;
  h2::MatDev d;
  std::vector<int32_t> adm_blk, inad_blk;  // slot -> block id (DFS order)
  std::vector<int32_t> blk2adm, blk2inad;  // block id -> slot or -1
  std::vector<int32_t> inad_range;         // per block: [first,last) inadmissible slot in its subtree
  std::vector<void*> allocs;
  // product / factorization state
  double* ws = nullptr;
  size_t ws_cap = 0;
  int* iws = nullptr;
  size_t iws_cap = 0;
  int factored = 0;              // 0 no, 1 Cholesky, 2 LR
  std::vector<char> nzr, nzc;    // host: cluster rank possibly non-zero (row / column basis)
  long long stats[4] = {0, 0, 0, 0};  // local updates, dense adds, temporaries issued by the driver
  SolveSched sched[3];                 // h2_solve sweeps: L (ascending), U (descending), L^T (descending)
};

namespace h2 {
void set_error(const std::string& msg);
// H2_POISON=1 (diagnostic): fill a fresh FP64 workspace with NaN bytes (0xFF) instead of leaving
// it uninitialised, so that any read of never-written memory shows up as a NaN in the result
void poison(void* p, size_t bytes);
// true while an h2_batch_begin / h2_batch_end recording is open on this thread
bool batch_open();

// launchers (h2_matvec.cu)
void free_mvpack(h2_mat_* Z);
cudaError_t launch_matvec(const h2_mat_* Z, int transpose, double alpha, const double* x, double beta,
                          double* y, cudaStream_t st);
// sequential block substitution (h2_solve.cu): x (original order, n x nrhs, ld ldx) <- F^{-1} x
cudaError_t solve_factored(h2_mat_* F, double* x, int nrhs, int64_t ldx, cudaStream_t st);
// launchers (h2_update.cu)
cudaError_t launch_update(const h2_mat_* Z, const UpdArgs& a, cudaStream_t st);
cudaError_t update_init_attributes();
}  // namespace h2
