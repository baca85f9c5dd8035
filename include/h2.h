/*
 * h2.h — C ABI of the B200-native H^2-matrix hot path (arXiv 1402.5056).
 *
 * Citations: P:n = line n of the paper's text, SURVEY §8 = the build's scope table.
 * All floating point is IEEE double (FP64).  All dense arrays are column-major.
 *
 * Index conventions:
 *   - cluster ids are DFS preorder (root 0, son0 before son1);
 *   - perm[i] is the ORIGINAL index of tree position i;
 *   - low-rank factors X, Y passed to h2_lowrank_update are in TREE order restricted to the
 *     contiguous ranges of t0 / s0;
 *   - vectors passed to h2_matvec / h2_solve are in ORIGINAL order (the library applies perm).
 *
 * Ownership: handles are library-owned and freed by the matching *_destroy.  Host inputs are
 * copied before the call returns.  Device pointers are borrowed for the stream-ordered duration
 * of the call (do not free or overwrite them until the stream has passed the call).  An h2_mat
 * lives in device memory allocated by the library (cudaMalloc) on the current device.
 *
 * Errors: every call validates its arguments before mutating anything and returns an
 * h2_status; h2_last_error() returns a thread-local message for the last non-OK status.
 * Calls on one h2_mat must be ordered on one stream (h2_matvec uses per-matrix device
 * workspace); different matrices are independent.
 */
#ifndef H2_B200_H
#define H2_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct h2_tree_* h2_tree;   /* cluster tree + permutation, immutable      */
typedef struct h2_btree_* h2_btree; /* block tree (rows, cols, eta), immutable   */
typedef struct h2_mat_* h2_mat;     /* H^2 matrix resident on one GPU, mutable    */
typedef void* h2_stream;            /* a cudaStream_t (0 = legacy default stream)             */

typedef enum {
  H2_OK = 0,
  H2_ERR_ARG = 1,       /* invalid argument (e.g. (t0,s0) not a block, n/dim/leaf <= 0)        */
  H2_ERR_SHAPE = 2,     /* shape or rank mismatch, rank above the matrix's capacity             */
  H2_ERR_STRUCTURE = 3, /* a CSR nonzero lands in an admissible block (message names the entry) */
  H2_ERR_NONFINITE = 4, /* NaN/Inf in a host input                                              */
  H2_ERR_BREAKDOWN = 5, /* dense leaf pivot breakdown (message names the cluster and pivot)     */
  H2_ERR_NOMEM = 6,     /* device allocation failed / capacity exceeded                         */
  H2_ERR_CUDA = 7,      /* a CUDA runtime error                                                 */
  H2_ERR_UNSUPPORTED = 8, /* operation not available in this build                              */
  H2_ERR_NOCONV = 9     /* an iteration (h2_pcg) reached maxit without meeting its tolerance    */
} h2_status;

/* TruncationControl (reading SURVEY R5): a cluster keeps
 *   r = #{ sigma_i > max(rel_tol * sigma_1, abs_tol) },  r <= max_rank (max_rank <= 0: unbounded),
 * of the singular values of its weighted basis V~_t B~_t^T. sigma_1 = 0 gives r = 0.
 * blockwise != 0 (DESIGN reading own-10): the paper's "block-relative accuracy
 * eps^" ("weighting factors in the matrices B_{t,s} ... to ensure blockwise relative
 * error bounds"): every block b = (t, s) enters the weight stacks of the local update
 * with the factor 1 / ||R_{V,t} S~_b R_{W,s}^T||_F (the block's Frobenius norm, from the R-factors
 * of the current / extended bases) and a cluster keeps r = #{ sigma_i > max(rel_tol, abs_tol) }
 * -- an ABSOLUTE threshold eps^ = rel_tol on the weighted matrix.  The low-rank temporaries of the
 * product (one block each) keep the relative rule.  (The field occupies what was
 * padding: sizeof(h2_trunc) is unchanged; callers must zero-initialise the struct.) */
typedef struct {
  double rel_tol;
  double abs_tol;
  int32_t max_rank;
  int32_t blockwise;
} h2_trunc;

typedef enum { H2_FULL = 0, H2_LOWER = 1 } h2_storage; /* LOWER: blocks with t-range >= s-range */
typedef enum { H2_LR = 0, H2_CHOLESKY = 1 } h2_factor_kind;

/* ---- structure (host, exact integer/FP predicates) -------------------------------------- */

/* Cluster tree by geometric bisection (binary P:331-332; reading SURVEY R2):
 * tight bounding box, split the longest extent (lowest axis on ties) at its midpoint, points with
 * coord < mid go to son0 (stable), stop at <= leaf_size points.
 * pts: host, n x dim, row-major (point i at pts[i*dim .. i*dim+dim-1]); dim in {1,2,3}. */
h2_status h2_cluster_tree(const double* pts, int64_t n, int32_t dim, int32_t leaf_size, h2_tree* out);

/* Cluster tree by domain-decomposition clustering ("a domain
 * decomposition cluster strategy similar to the one described in [GRKRLE05a]"; the paper gives no
 * details: DESIGN reading own-11).  rowptr/colidx: host CSR pattern of the n x n matrix (taken
 * symmetrically).  A DOMAIN cluster with more than 2 leaf_size points is bisected geometrically
 * as in h2_cluster_tree into (left, right); the interface gamma = the points of `right` coupled
 * to a point of `left`; dom1 = left, dom2 = right minus gamma; the ternary split becomes
 * t -> (interior -> (dom1, dom2), gamma), i.e. the tree order is the nested dissection order.
 * dom1/dom2 are DOMAIN clusters, gamma (an INTERFACE cluster) and small domains are bisected
 * plainly; an empty gamma makes (left, right) itself a decoupled pair; an empty dom2 or an interior
 * of <= leaf_size points gives a plain split.  h2_block_tree with this tree as rows AND columns
 * makes the block of two decoupled domains an admissible leaf: it holds no matrix entry and the
 * LR / Cholesky factorization in tree order creates none (its rank stays 0).
 * h2_tree_ddpair: ddpair[t] = 1 iff the two sons of cluster t are decoupled domains (host, nclusters). */
h2_status h2_cluster_tree_dd(const double* pts, int64_t n, int32_t dim, int32_t leaf_size, const int64_t* rowptr,
                             const int32_t* colidx, h2_tree* out);
h2_status h2_tree_ddpair(h2_tree tree, int8_t* ddpair);

/* Export: perm[n]; lo/hi/son0/son1/level[nclusters] (son = -1 for leaves); any pointer may be
 * NULL.  *nclusters receives the count (call once with NULL arrays to size them). */
h2_status h2_tree_export(h2_tree tree, int64_t* perm, int32_t* lo, int32_t* hi, int32_t* son0,
                         int32_t* son1, int32_t* level, int32_t* nclusters);
void h2_tree_destroy(h2_tree tree);

/* Block tree, sons(b) = sons+(t) x sons+(s) t-son-major; admissible
 * iff dist > 0 and max(diam_t, diam_s) <= eta * dist on tight point boxes (reading SURVEY R1).
 * The handle keeps references to both trees: destroy it before them. */
h2_status h2_block_tree(h2_tree rows, h2_tree cols, double eta, h2_btree* out);

/* Export blocks in DFS preorder: t[], s[], kind[] (0 subdivided, 1 admissible leaf,
 * 2 inadmissible leaf); arrays may be NULL; *nblocks receives the count.  *csp (may be NULL)
 * receives the sparsity constant C_sp. */
h2_status h2_btree_export(h2_btree bt, int32_t* t, int32_t* s, int8_t* kind, int64_t* nblocks,
                          int32_t* csp);
void h2_btree_destroy(h2_btree bt);

/* ---- H^2 matrix on the device ------------------------------------------------------------ */

/* h2_from_sparse: all cluster bases of rank 0, the CSR (host arrays, ORIGINAL
 * order, n x n) scattered into dense nearfield tiles.  A nonzero falling in an
 * admissible block -> H2_ERR_STRUCTURE.  storage = H2_LOWER keeps only blocks whose row range
 * starts at or after the column range (the Cholesky factor layout).
 * rank_cap: capacity of stored ranks per cluster (e.g. 32); update_cap: the largest update rank
 * k a later h2_lowrank_update may pass (rank_cap <= 48, rank_cap + update_cap <= 96). */
h2_status h2_from_sparse(h2_btree bt, int64_t n, const int64_t* rowptr, const int32_t* colidx,
                         const double* val, h2_storage storage, int32_t rank_cap, int32_t update_cap,
                         h2_stream stream, h2_mat* out);

/* Local low-rank update Z|_{t0 x s0} += alpha X Y^T keeping Z globally H^2 (Thm 1):
 * exact nearfield part, basis extension (eq. 4a-c), weights, truncated nested bases
 * (P:769-872), coupling re-projection, transfer fix-up.
 * X: device, |t0| x k, leading dimension ldx >= |t0|; Y: device, |s0| x k, ldy >= |s0|; rows in
 * tree order within t0 / s0.  0 <= k <= update_cap.  (t0,s0) must be a node of the block tree
 * (H2_ERR_ARG otherwise).  An inadmissible-leaf target gets the exact dense add only.
 * Ranks are chosen on the device by *trunc; nothing is copied back to the host. */
h2_status h2_lowrank_update(h2_mat Z, int32_t t0, int32_t s0, int32_t k, double alpha,
                            const double* X, int64_t ldx, const double* Y, int64_t ldy,
                            const h2_trunc* trunc, h2_stream stream);

/* Batch recording (execution only, no change of the arithmetic): between h2_batch_begin(stream)
 * and h2_batch_end(), h2_lowrank_update calls on that stream are recorded into one device op list
 * that the executor runs in chunks (16,384 ops) while recording continues, instead of one executor
 * launch per call; the result is bit-identical to unbatched calls (same ops, same order).  The
 * caller keeps every X / Y alive and unchanged until the stream passes h2_batch_end.  Inside a
 * batch only h2_lowrank_update (same stream) may be called; every other call returns H2_ERR_ARG.
 * One open batch per host thread.  H2_ERR_ARG: nested begin / end without begin; H2_ERR_CUDA. */
h2_status h2_batch_begin(h2_stream stream);
h2_status h2_batch_end(void);

/* y <- alpha op(Z) x + beta y (op = transpose ? Z^T : Z), x/y device vectors in ORIGINAL order
 * (forward transform, couplings, backward transform, nearfield).
 * x and y: device, n doubles each, borrowed until the stream passes the call; y may not alias x.
 * The first product after any call that changed Z (update, product, factorization, inversion)
 * rebuilds Z's packed coupling / transfer copies: it reads the ranks back (one synchronisation of
 * `stream`) and allocates device memory for them (H2_ERR_NOMEM / H2_ERR_CUDA); later products are
 * stream-ordered without host synchronisation.  The far-field part runs on a library-owned side
 * stream, forked from and joined to `stream` inside the call.  Not thread-safe per matrix
 * (the transform coefficients are workspace of Z); different matrices may be used concurrently. */
h2_status h2_matvec(h2_mat Z, int32_t transpose, double alpha, const double* x, double beta, double* y,
                    h2_stream stream);

/* Z <- Z + alpha X Y: recursive product over the triple tree.  Case 1
 * recursion over sons+ in the printed order; an admissible-leaf target receives its
 * sub-products in low-rank temporaries (SVD-truncated) merged by 4 zero-extended local
 * updates; Case 2 builds low-rank factors and performs a local update
 * (or a dense add into an inadmissible target).  X, Y: H2_FULL storage; Z, X, Y share the cluster
 * trees; Z must not alias X or Y.  Truncation of every update and temporary by *trunc. */
h2_status h2_addmul(h2_mat Z, double alpha, h2_mat X, h2_mat Y, const h2_trunc* trunc, h2_stream stream);

/* In-place approximate inverse A <- A^{-1} (Remark 1): block Gauss
 * elimination over the cluster tree, C11 = A11^{-1}, B12 = C11 A12, B21 = A21 C11,
 * S = A22 - A21 B12 (P:1382 prints A11: reading R20), C22 = S^{-1}, C12 = -B12 C22,
 * C21 = -C22 B21, C11 = C11 - C12 B21 -- six h2_addmul-type products per level, truncated by
 * *trunc; a leaf tile is inverted directly (Gauss-Jordan; a pivot |p| <= 1e-14 ||tile||_F is a
 * breakdown, reported by h2_check_device_flags as H2_ERR_BREAKDOWN).  A: unfactored H2_FULL
 * storage, shared row/column tree.  Allocates a scratch matrix of A's structure for B12 / B21 and
 * synchronizes `stream` before releasing it. */
h2_status h2_inverse(h2_mat A, const h2_trunc* trunc, h2_stream stream);

/* In-place factorization:
 *   H2_CHOLESKY: A in H2_LOWER storage, symmetric positive definite; on return the
 *     stored lower triangle holds L (diagonal tiles lower-triangular) with A ~ L L^T;
 *   H2_LR: A in H2_FULL storage; unit-lower L (strict lower part) and R (upper part), no pivoting.
 * Block substitutions P:392-450; an admissible-leaf block X = V S (L^{-1} W)^T is re-entered by
 * S <- 0 and a local update (reading R8).  A non-positive (Cholesky) or |p| <= 1e-14 ||tile||_F
 * (LR) leaf pivot is reported by h2_check_device_flags as H2_ERR_BREAKDOWN (the call itself only
 * enqueues work; the matrix is then partially factored). */
h2_status h2_lr_factor(h2_mat A, h2_factor_kind kind, const h2_trunc* trunc, h2_stream stream);

/* x <- F^{-1} x for a factored matrix: (L L^T)^{-1} x (Cholesky) or (L R)^{-1} x (LR), by H^2
 * forward/backward substitution (the preconditioner of P:1440-1444).  x: device, n x nrhs,
 * column-major with leading dimension ldx >= n, ORIGINAL order; 1 <= nrhs <= 64. */
h2_status h2_solve(h2_mat F, double* x, int32_t nrhs, int64_t ldx, h2_stream stream);

/* Preconditioned CG (reading R12): solves A x = b with the factored F as the
 * preconditioner ((L L^T)^{-1} or (L R)^{-1} via h2_solve), x0 = 0, stops when ||r||/||b|| < tol
 * or after maxit iterations.  b, x: device vectors of length n in ORIGINAL order.  *iters receives
 * the number of A-applications, *relres (may be NULL) the final relative residual.  Synchronizes
 * the stream once per iteration (residual norm).  A non-finite residual (a NaN/Inf in A, F or b)
 * stops the iteration at once with H2_ERR_NONFINITE; maxit iterations without ||r||/||b|| < tol
 * return H2_ERR_NOCONV (*iters / *relres are set in both cases). */
h2_status h2_pcg(h2_mat A, h2_mat F, const double* b, double* x, double tol, int32_t maxit, int32_t* iters,
                 double* relres, h2_stream stream);

/* Number of kernels this library has launched since it was loaded (bench / test hook). */
h2_status h2_launch_count(int64_t* out);

/* Counters of the work the product/factorization driver issued on this matrix:
 * out[0] local low-rank update calls, out[1] dense nearfield adds, out[2] temporaries, out[3] local
 * updates that had a non-zero rank on the device (the oracle's update count; synchronizes). */
h2_status h2_stats(h2_mat Z, int64_t out[4]);

/* ---- inspection (synchronous: these synchronize the given stream) -------------------------- */

/* Row ranks k_t and column ranks l_s per cluster (arrays of nclusters, host). */
h2_status h2_ranks(h2_mat Z, int32_t* row_rank, int32_t* col_rank);

/* Stored scalars at the current ranks: [nearfield, leaf bases, transfers, couplings]. */
h2_status h2_storage_report(h2_mat Z, int64_t scalars[4]);

/* Test hook: copy the whole representation to host buffers (each may be NULL), tight layouts:
 *   V: per leaf cluster in id order |t| x k_t;  E: per non-root cluster k_t x k_parent;
 *   W, F: the same for the column basis;  S: per stored admissible block (DFS order) k_t x l_s;
 *   N: per stored inadmissible block (DFS order) |t| x |s|.   sizes[6] receives the number of
 * doubles of each array (call with NULL buffers first to size them). */
h2_status h2_export(h2_mat Z, double* V, double* E, double* W, double* F, double* S, double* N,
                    int64_t sizes[6]);

/* h2_import (test-only): the inverse of h2_export.  Builds a matrix of block tree
 * bt from host arrays in exactly h2_export's tight layouts: row_rank / col_rank (one int per
 * cluster, <= rank_cap), V / W (leaf bases in leaf order, |t| x k_t), E / F (transfers of clusters
 * 1..nclusters-1, k_t x k_parent), S (couplings of the stored admissible blocks in DFS order,
 * k_t x l_s), N (stored nearfield tiles in DFS order).  The memoised R-factors of the nested bases
 * (reading R7) are recomputed from the imported bases (Alg. 16), so later updates see
 * the same state as on the exporting side.  Arrays may be NULL when they would be empty.  Errors:
 * H2_ERR_SHAPE (rank above rank_cap), H2_ERR_NONFINITE, H2_ERR_ARG, as h2_from_sparse. */
h2_status h2_import(h2_btree bt, const int32_t* row_rank, const int32_t* col_rank, const double* V, const double* E,
                    const double* W, const double* F, const double* S, const double* N, h2_storage storage,
                    int32_t rank_cap, int32_t update_cap, h2_stream stream, h2_mat* out);

/* Device-side status word since the last call (then cleared): bit 0 = a truncation hit a rank above
 * rank_cap (clamped); bit 1 = a dense leaf breakdown (also returned as H2_ERR_BREAKDOWN); bit 2 =
 * a contribution inside h2_addmul / h2_lr_factor / h2_inverse had a rank above update_cap and
 * was dropped (the result is then wrong: re-run with a larger update_cap -- a dense x dense
 * product of leaf tiles can reach rank = leaf size, reading own-7).  Synchronizes the stream. */
h2_status h2_check_device_flags(h2_mat Z, int32_t* flags);

/* Profiling hook (bench/test only; off by default).  h2_profile_enable(1) synchronizes the
 * device, clears the counters and brackets every later library launch with cudaEventRecord on
 * the launch stream; kernels also add their algorithmic flops and bytes (fixed formulas,
 * SURVEY §8(d)) to device counters.  h2_profile_read synchronizes and returns, per kernel kind
 * (*count entries): a 32-byte NUL-terminated name in names[32*i], the number of launches, the
 * summed event time in ms, and the counted flops and bytes.  Any output pointer may be NULL. */
h2_status h2_profile_enable(int32_t on);
h2_status h2_profile_read(char* names, int64_t* launches, double* ms_total, double* flops, double* bytes,
                          int32_t* count);
/* Profiling sub-phase counters of the SVD items (cycles: load+GEMM, Jacobi, output; count; sum K;
 * sum m; sum of Jacobi sweeps), out[16]. */
h2_status h2_profile_debug(double out[16]);
/* Profiling: device-executor time (ns) and count per op code (exec.h OpCode order), cap entries;
 * *nops = number of op-code slots (64). */
h2_status h2_profile_ops(double* ns, double* count, int32_t cap, int32_t* nops);

void h2_mat_destroy(h2_mat Z);
const char* h2_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* H2_B200_H */
