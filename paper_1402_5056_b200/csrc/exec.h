// Device-resident executor of the H^2 arithmetic.
//
// The host recursion (local update, product, substitutions, factorization) does not launch kernels:
// it appends fixed-size op records to a list.  An op is "run item i of kind `code` for i < nitems";
// consecutive ops are separated by a barrier when `barrier` is set.  The list is executed on the
// device by one thread-block cluster (8 CTAs, cluster barriers between dependent ops); an op with
// many items runs as its own full-grid launch.  All shapes that depend on ranks are read from
// device memory by the items, so the list only depends on the block-tree structure.
#pragma once
#include <stdint.h>

#include <cstring>
#include <vector>

#include "h2_internal.h"

namespace h2 {

struct Dim {
  const int* p;
  int c;
#ifdef __CUDACC__
  __device__ __forceinline__ int v() const { return (p ? *p : 0) + c; }
#endif
};
inline Dim dimc(int c) { return Dim{nullptr, c}; }
inline Dim dimp(const int* p, int c = 0) { return Dim{p, c}; }

enum OpCode : int32_t {
  OP_UPD_EXT_LEAF = 0,
  OP_UPD_EXT_LEVEL,
  OP_UPD_W_PATH,
  OP_UPD_W_LEVEL,
  OP_UPD_SVD_LEAF,
  OP_UPD_SVD_LEVEL,
  OP_UPD_COUPLE,
  OP_UPD_INSTALL,
  OP_UPD_RCACHE,
  OP_EXPAND,
  OP_GEMM,
  OP_GEMM_PART,
  OP_GEMM_SUM,
  OP_HM_FWD_LEAF,
  OP_HM_FWD_LEVEL,
  OP_HM_COUPLE,
  OP_HM_BWD_LEVEL,
  OP_HM_LEAF,
  OP_POTRF,
  OP_GETRF,
  OP_TRSM,
  OP_TSQR,
  OP_TEMP,
  OP_COPY_COLS,
  OP_SET_INT,
  OP_ADD_INT,
  OP_RANK_IF,
  OP_STACK,
  OP_CHOOSE,
  OP_IDENTITY,
  OP_TRANSPOSE,
  OP_GATHER,
  OP_SCATTER,
  OP_ZERO,
  OP_DD,
  OP_NZTILE,
  OP_TINV,    // in-place inverse of a diagonal leaf tile (approximate inversion, Remark 1)
  OP_C2CORE,  // Case 2, both factors admissible: [G =] W^T V, C = S^X G S^Y, choose (one CTA)
  OP_SKIPZ,  // all CTAs: if *ip == 0 skip the next `count` ops (a zero-rank local update)
  OP_KCHECK,  // *ip > rows (the update capacity): set the capacity flag and drop the contribution (*ip = 0)
  OP_COUNT
};

// ---- payloads ---------------------------------------------------------------------------------
struct PUpd {
  UpdArgs a;
  int i[8];
};
struct PExpand {
  int side, t, l0, ld;
  double* out;
};
struct PGemm {
  double* C;
  const double* A;
  const double* B;
  int ldc, lda, ldb, ta, tb, chunk;
  Dim m, n, k;
  double alpha, beta;
};
struct PHm {  // all H^2-block x dense items
  int dside, sside, a, b, trans, l0, base_lo, ldd, ldo;
  int ident;  // D is the identity (ld ldd): products with D are column selections
  const double* D;
  double* xh;
  double* yh;
  double* out;
  Dim m;
  double alpha, beta;
};
struct PTile {
  int slot, t, m, mode, ldb, brows;
  double* B;
  Dim bcols;
};
struct PTsqr {
  const double* A;
  double* R;
  int lda, rows, ldr;
  Dim K;
};
struct PTemp {
  const double* Ra;
  const double* Rb;
  double* Ma;
  double* Mb;
  int* rout;
  int* flags;
  const int* knew;  // rank of the contribution being added (0: the temporary is left exactly as is)
  int ldr, ldm, max_rank, cap;
  Dim K;
  double rel, abs_tol;
};
struct PMisc {  // small data-movement ops
  double* dst;
  const double* src;
  const int64_t* perm;
  int* ip;
  const int* ia;
  const int* ib;
  int ldd, lds, rows, cols, row_off, rows_new;
  int64_t ldx;
  Dim d1, d2;
};

struct PDD {  // dense x dense Case-2 factors
  int mx, my, slotx, sloty, transx, transy, mt, ms, mr, lda, ldb;
  double* A;
  double* B;
  int* kout;
  double rel;
};

struct PC2 {  // fused Case-2 core (items_arith.cuh it_c2core)
  const double* W;   // W^X_s (ms x kxs, ld ms) or nullptr: G given
  const double* V;   // V^Y_s (ms x kys, ld ms)
  const double* G;   // G (ld KC) when W == nullptr
  const double* Sx;
  const double* Sy;
  double* Ca;
  double* Cb;
  const int* kd[4];  // kxt, kxs, kys, kyr
  int* kout;
  int ms, ldsx, ldsy, tx, ty, ldo;
};

constexpr int OP_PAYLOAD = 176;
struct alignas(16) OpRec {
  int32_t code;
  int32_t nitems;
  int32_t barrier;  // bit 0: cluster barrier after this op; bit 1: never elide it; bits 8-15: CTA of item 0
  int32_t mat;  // index of the matrix descriptor (0..2) the op uses
  unsigned char p[OP_PAYLOAD];
};
static_assert(sizeof(PUpd) <= OP_PAYLOAD, "payload");
static_assert(sizeof(PGemm) <= OP_PAYLOAD, "payload");
static_assert(sizeof(PHm) <= OP_PAYLOAD, "payload");
static_assert(sizeof(PTemp) <= OP_PAYLOAD, "payload");
static_assert(sizeof(PMisc) <= OP_PAYLOAD, "payload");
static_assert(sizeof(PC2) <= OP_PAYLOAD, "payload");

constexpr int EXEC_MATS = 3;

// ---- host side recording ---------------------------------------------------------------------
size_t default_flush_at();  // 16384 ops; H2_EXEC_FLUSH overrides (tests: frequent chunk boundaries)
struct ExecCtx {
  std::vector<OpRec> ops;
  const MatDev* mats[EXEC_MATS] = {nullptr, nullptr, nullptr};
  cudaStream_t st = 0;
  size_t flush_at = default_flush_at();  // ops are run in chunks while the host keeps recording
  int mat_index(const MatDev& M);
  void maybe_flush();
  int hold = 0;             // > 0 while a skip region is open (no flush inside it)
  int skip_tag = 0;         // origin tag recorded with the next skip op (profiling statistics)
  int group = 0;             // > 0 inside an independence group (group_begin / group_end)
  int group_off = 0;         // CTA of the next grouped op's item 0
  template <class P>
  void emit(int code, int nitems, const MatDev* M, const P& payload, bool barrier = true) {
    if (nitems <= 0) return;
    OpRec r;
    r.code = code;
    r.nitems = nitems;
    if (group > 0) {
      // independent ops of a group: no barrier between them, items spread over the cluster's CTAs
      // (item i of this op runs on CTA (group_off + i) mod CL); group_end places one barrier
      r.barrier = (group_off & 0xff) << 8;
      group_off += nitems;
    } else {
      // two consecutive single-item ops both run on CTA 0 of the cluster, in order: the block
      // barrier after each item orders them, the cluster barrier between them is not needed
      // (a skip op reads its flag on every CTA: the barrier before it stays; a group's closing
      // barrier orders ops on other CTAs and stays too)
      if (nitems == 1 && code != OP_SKIPZ && !ops.empty() && ops.back().nitems == 1 &&
          ops.back().code != OP_SKIPZ && (ops.back().barrier & ~1) == 0)
        ops.back().barrier = 0;
      r.barrier = barrier ? 1 : 0;
    }
    r.mat = M ? mat_index(*M) : 0;
    static_assert(sizeof(P) <= OP_PAYLOAD, "payload");
    std::memcpy(r.p, &payload, sizeof(P));
    ops.push_back(r);
    if (ops.size() >= flush_at && hold == 0) maybe_flush();
  }
  // independence group: the ops recorded between group_begin and group_end neither read what
  // another op of the group writes nor write what another reads or writes (the caller's promise);
  // they run without cluster barriers between them, on different CTAs where possible.
  // A chunk flush inside a group is a kernel boundary (a stronger ordering): still correct.
  void group_begin() {
    ++group;
    group_off = 0;
  }
  void group_end() {
    if (--group == 0 && !ops.empty()) ops.back().barrier |= 3;
  }
  // skip region: the ops recorded between begin_skip and end_skip are skipped on the device when
  // *k == 0 (they must all run inside the cluster executor: end_skip cancels the skip otherwise)
  size_t begin_skip(const int* k);
  void end_skip(size_t at, int big_items);
};

// the recording context of the current thread (set by the public entry points)
ExecCtx* exec_ctx();
void exec_begin(ExecCtx* ctx, cudaStream_t st);
cudaError_t exec_flush();  // runs and clears the recorded ops (stream-ordered)
int exec_big_items();      // ops with more items run as their own full-grid launch
cudaError_t exec_end();    // flush + reset the context pointer

}  // namespace h2
