// Device primitives of the H^2 product / substitution / factorization.
// Every shape that depends on a rank lives in device memory (Dim), so the host recursion never
// synchronises on the device.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "exec.h"
#include "h2_internal.h"

namespace h2 {

// ---- emitters (h2_exec.cu): append ops to the current executor context -------------------------------------------------------------------
// out (|t| x k_t, ld) = full nested basis of cluster t of one side (eq. (1))
void expand_basis(const MatDev& M, const DevSide& D, int t, double* out, int ld, cudaStream_t st);
// C (m x n) = alpha op(A) op(B) + beta C, dims on the device (caps on the host for grid sizes)
void gemm(double* C, int ldc, const double* A, int lda, bool ta, const double* B, int ldb, bool tb, Dim m, Dim n,
          Dim k, int mcap, int ncap, int kcap, double alpha, double beta, cudaStream_t st);
// out (|a| x m) = beta out + op(Z)|_{a x b} D,  D: |b| x m  (H^2 block times dense, [BO10 Thm 3.42]);
// b_blk = 1: D is the identity (its products are column selections, exact)
void hmul_dense(const MatDev& M, bool trans, int a, int b, int b_blk, const double* D, int ldd, Dim m, int mcap,
                double* out, int ldo, double alpha, double beta, cudaStream_t st);
// dense tiles (nearfield slots): Cholesky / no-pivot LU in place; breakdown -> flags[1], flags[2] = cluster
void tile_potrf(const MatDev& M, int slot, int t, cudaStream_t st);
void tile_getrf(const MatDev& M, int slot, int t, cudaStream_t st);
// in-place inverse of a diagonal leaf tile (Gauss-Jordan in elimination order; breakdown as getrf)
void tile_inverse(const MatDev& M, int slot, int t, cudaStream_t st);
// triangular solves with a diagonal tile T (m x m, ld lmax):
enum TrsmMode { RLT = 0, LLN, LLU, LLT, RUN, LUN, LUT };
void tile_trsm(const MatDev& M, int slot, int m, int mode, double* B, int ldb, int brows, Dim bcols, int bcolcap,
               cudaStream_t st);
// R-factor (K x K, ld kc) of the tall matrix A (rows x K, K on the device <= 64)
void tsqr_r(const double* A, int lda, int rows, Dim K, double* R, int ldr, cudaStream_t st);
// temporary truncation core: from Ra, Rb (K x K) -> Ma = Rb^T V_r, Mb = Ra^T U_r S_r^-1 (K x r), r -> *rout
void temp_core(const double* Ra, const double* Rb, int ldr, Dim K, double* Ma, double* Mb, int ldm, int* rout,
               double rel, double abs_tol, int max_rank, int cap, int* flags, const int* knew, cudaStream_t st);
// *kdev = 0 if the nearfield tile `slot` is exactly zero (reading own-6)
void zero_rank_if_zero_tile(const MatDev& M, int slot, int count, int* kdev, cudaStream_t st);
// copy a (rows x cols) block with device column count into dst (zero-extended rows are the caller's)
void copy_cols(double* dst, int ldd, const double* src, int lds, int rows, Dim cols, int colcap, cudaStream_t st);
void set_int(int* p, Dim v, cudaStream_t st);
void rank_check(const MatDev& M, int* kdev, int cap, cudaStream_t st);  // *kdev > cap: flag 4, *kdev = 0
void rank_if(int* p, const int* a, const int* b, cudaStream_t st);  // *p = (*a>0 && *b>0) ? *b : 0
void stack_cols(double* dst, int ldd, int rows, const double* T, int ldt, const int* kT, const double* Nw, int ldn,
                int row_off, int rows_new, Dim knew, int colcap, cudaStream_t st);
void choose_case2(const double* Cm, int ldc, const int* k1, const int* k2, double* Ca, double* Cb, int ldo, int* kout,
                  cudaStream_t st);
// Case 2, both factors admissible: C = S^X_or (W^T V) S^Y_or and the factored side (choose_case2),
// one op; W, V (ms x k, ld ms; ms <= case2_core_max_ms()) or G (ld KCAP_MAX) when W == nullptr
void case2_core(const double* W, const double* V, int ms, const double* G, const double* Sx, int ldsx, bool tx,
                const double* Sy, int ldsy, bool ty, const int* kxt, const int* kxs, const int* kys, const int* kyr,
                double* Ca, double* Cb, int ldo, int* kout, cudaStream_t st);
int case2_core_max_ms();
void identity(double* I, int ld, int m, cudaStream_t st);
void transpose_tile(double* dst, int ldd, const double* src, int lds, int rows, int cols, cudaStream_t st);
void add_int(int* p, Dim a, Dim b, cudaStream_t st);
// tree-order <-> original-order for n x nrhs blocks: Bt[i, c] = x[perm[i] + c ldx], x[perm[i] + c ldx] = Bt[i, c]
void gather_cols(double* Bt, const double* x, const int64_t* perm, int n, int nrhs, int64_t ldx, cudaStream_t st);
void scatter_cols(double* x, const double* Bt, const int64_t* perm, int n, int nrhs, int64_t ldx, cudaStream_t st);
// dst[0..count) = 0 (stream-ordered with the recorded ops)
void zero_fill(double* dst, size_t count, cudaStream_t st);
// dense x dense Case-2 factors: A (mt x r), B (mr x r), r -> *kout (see items_arith.cuh it_dd_compress)
void dd_compress(const MatDev& MX, int slotx, bool transx, const MatDev& MY, int sloty, bool transy, int mt, int ms,
                 int mr, double* A, int lda, double* B, int ldb, int* kout, double rel, cudaStream_t st);

}  // namespace h2
