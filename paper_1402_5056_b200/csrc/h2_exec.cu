// Op executor of the H^2 arithmetic (see exec.h) and the host-side emitters of every op.
//
// k_exec_cluster: one thread-block cluster of CL CTAs walks a segment of the op list; item i of an
//   op runs on CTA (i mod CL); consecutive dependent ops are separated by barrier.cluster
//   (release/acquire at cluster scope orders the global-memory results).  The whole dependent
//   chain of a local update (U0..U6, ~10 phases) or of a Case-2 factor construction therefore
//   costs one op dispatch + one cluster barrier per phase instead of one kernel launch per phase.
// k_exec_big: an op with more than BIG items (large subtrees / big H^2 block products) runs as its
//   own launch over up to all 148 SMs.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <cstring>
#include <stdexcept>
#include <string>

#include "exec.h"
#include "h2_arith.cuh"
#include "items_arith.cuh"
#include "items_upd.cuh"

namespace cg = cooperative_groups;

namespace h2 {
namespace {

constexpr int NT = NTHREADS;
constexpr int CL = 16;    // CTAs of the executor cluster (non-portable size 16; falls back to 8)
constexpr int BIG = 1024;  // ops with more items run as a full-grid launch (64: +5 % at C2)
constexpr int KC = KCAP_MAX;
constexpr int PR = 192;
constexpr int RM = KC + 1;
constexpr size_t SM_EXEC = (size_t)(3 * RM * KC + KC) * 8 + (KC + 8) * 4;  // max over items (SVD items)
static_assert(SM_EXEC >= (size_t)((PR + 1) * KC + KC + 8) * 8 + (5 * 128 + PR) * 4, "smem (weights_cluster panel + block descriptors)");
static_assert(SM_EXEC >= (size_t)((PR + 1) * KC + KC + 8 + 1024 + 2 * (RCAP_MAX + 1) * RCAP_MAX) * 8 + 3 * 64 * 4, "smem (weights path: panel + G chain + path)");
static_assert((5 * 128 + PR) * 4 + 128 * 8 <= 1024 * 8, "weights_cluster descriptors fit the spare area");
static_assert(SM_EXEC >= (size_t)24000 * 8 + 9 * 128 * 4 + 16, "smem (couplings)");
static_assert(SM_EXEC >= (size_t)(2 * (KC + 1) * 64 + 2 * 65 * 64 + 2 * KC + 8) * 8 + 2 * KC * 4 + 64, "smem (dd_compress)");
static_assert(SM_EXEC >= (size_t)((PR + 1) * RCAP_MAX + KC + 3 * (RCAP_MAX + 1) * RCAP_MAX) * 8 + 4 * 64 * 4, "smem (rcache items)");
static_assert(SM_EXEC >= (size_t)(3 * (RCAP_MAX + 1) + 2 * ar::C2_MS) * RCAP_MAX * 8, "smem (it_c2core)");
static_assert(SM_EXEC >= (size_t)(3 * (KC + 1) * KC + KC) * 8 + (KC + 8) * 4 && SM_EXEC >= (size_t)((2 * KC + 1) * KC + KC + 8) * 8, "smem");

struct ExecParams {
  const OpRec* ops;
  int begin, end;
  double* prof;   // profiling counters (h2_prof) or nullptr
  double* gpart;  // partial sums of long-inner-dimension GEMMs
  MatDev mats[EXEC_MATS];
};

__constant__ int c_op_kid[OP_COUNT] = {
    K_EXT_LEAF, K_EXT_LEVEL, K_W_PATH, K_W_LEVEL, K_SVD_LEAF, K_SVD_LEVEL, K_COUPLE, K_INSTALL, K_RCACHE,
    K_AR_EXPAND, K_AR_GEMM, K_AR_GEMM, K_AR_GEMM, K_AR_HMUL, K_AR_HMUL, K_AR_HMUL, K_AR_HMUL, K_AR_HMUL,
    K_AR_TILE, K_AR_TILE, K_AR_TILE, K_AR_TSQR, K_AR_TEMP, K_AR_MISC, K_AR_MISC, K_AR_MISC, K_AR_MISC,
    K_AR_MISC, K_AR_MISC, K_AR_MISC, K_AR_MISC, K_AR_MISC, K_AR_MISC, K_AR_MISC, K_AR_TEMP, K_AR_MISC,
    K_AR_TILE, K_AR_GEMM, K_AR_MISC, K_AR_MISC};

__device__ __forceinline__ const DevSide& side_of(const MatDev& M, int s) { return s ? M.col : M.row; }

__device__ void dispatch(const ExecParams& P, const OpRec& op, int it, int n, double* sm) {
  const MatDev& M = P.mats[op.mat];
  switch (op.code) {
    case OP_UPD_EXT_LEAF: {
      const PUpd& q = *reinterpret_cast<const PUpd*>(op.p);
      upd::it_upd_ext_leaf(M, q.a, q.i[0], q.i[1], q.i[2], q.i[3], q.i[4], q.i[5], q.i[6], q.i[7], it, n, sm);
    } break;
    case OP_UPD_EXT_LEVEL: {
      const PUpd& q = *reinterpret_cast<const PUpd*>(op.p);
      upd::it_upd_ext_level(M, q.a, q.i[0], q.i[1], q.i[2], q.i[3], it, n, sm);
    } break;
    case OP_UPD_W_PATH: {
      const PUpd& q = *reinterpret_cast<const PUpd*>(op.p);
      upd::it_upd_weights_path(M, q.a, q.i[0], q.i[1], q.i[2], q.i[3], it, sm);
    } break;
    case OP_UPD_W_LEVEL: {
      const PUpd& q = *reinterpret_cast<const PUpd*>(op.p);
      upd::it_upd_weights_level(M, q.a, q.i[0], q.i[1], q.i[2], q.i[3], it, n, sm);
    } break;
    case OP_UPD_SVD_LEAF: {
      const PUpd& q = *reinterpret_cast<const PUpd*>(op.p);
      upd::it_upd_svd_leaf(M, q.a, q.i[0], q.i[1], q.i[2], q.i[3], it, n, sm);
    } break;
    case OP_UPD_SVD_LEVEL: {
      const PUpd& q = *reinterpret_cast<const PUpd*>(op.p);
      upd::it_upd_svd_level(M, q.a, q.i[0], q.i[1], q.i[2], q.i[3], it, n, sm);
    } break;
    case OP_UPD_COUPLE: {
      const PUpd& q = *reinterpret_cast<const PUpd*>(op.p);
      upd::it_upd_couple(M, q.a, q.i[0], q.i[1], it, n, sm);
    } break;
    case OP_UPD_INSTALL: {
      const PUpd& q = *reinterpret_cast<const PUpd*>(op.p);
      upd::it_upd_install(M, q.a, q.i[0], q.i[1], it, n, sm);
    } break;
    case OP_UPD_RCACHE: {
      const PUpd& q = *reinterpret_cast<const PUpd*>(op.p);
      upd::it_upd_rcache_path(M, q.a, q.i[0], q.i[1], q.i[2], q.i[3], it, sm);
    } break;
    case OP_EXPAND: {
      const PExpand& q = *reinterpret_cast<const PExpand*>(op.p);
      ar::it_expand(M, side_of(M, q.side), q.t, q.l0, q.out, q.ld, it, n, sm);
    } break;
    case OP_GEMM: {
      const PGemm& q = *reinterpret_cast<const PGemm*>(op.p);
      ar::it_gemm(q.C, q.ldc, q.A, q.lda, q.ta, q.B, q.ldb, q.tb, q.m, q.n, q.k, q.alpha, q.beta, it, n, sm);
    } break;
    case OP_GEMM_PART: {
      const PGemm& q = *reinterpret_cast<const PGemm*>(op.p);
      ar::it_gemm_inner_part(P.gpart, q.A, q.lda, q.ta, q.B, q.ldb, q.tb, q.m, q.n, q.k, q.chunk, it, n, sm);
    } break;
    case OP_GEMM_SUM: {
      const PGemm& q = *reinterpret_cast<const PGemm*>(op.p);
      ar::it_gemm_inner_sum(q.C, q.ldc, P.gpart, q.chunk, q.m, q.n, q.alpha, q.beta, it, n, sm);
    } break;
    case OP_HM_FWD_LEAF: {
      const PHm& q = *reinterpret_cast<const PHm*>(op.p);
      ar::it_hm_fwd_leaf(M, side_of(M, q.sside), q.l0, q.base_lo, q.D, q.ldd, q.m, q.xh, q.ident, it, n, sm);
    } break;
    case OP_HM_FWD_LEVEL: {
      const PHm& q = *reinterpret_cast<const PHm*>(op.p);
      ar::it_hm_fwd_level(M, side_of(M, q.sside), q.l0, q.m, q.xh, it, n, sm);
    } break;
    case OP_HM_COUPLE: {
      const PHm& q = *reinterpret_cast<const PHm*>(op.p);
      ar::it_hm_couple(M, side_of(M, q.dside), side_of(M, q.sside), q.a, q.b, q.trans, q.m, q.xh, q.yh, it, n, sm);
    } break;
    case OP_HM_BWD_LEVEL: {
      const PHm& q = *reinterpret_cast<const PHm*>(op.p);
      ar::it_hm_bwd_level(M, side_of(M, q.dside), q.l0, q.m, q.yh, it, n, sm);
    } break;
    case OP_HM_LEAF: {
      const PHm& q = *reinterpret_cast<const PHm*>(op.p);
      ar::it_hm_leaf(M, side_of(M, q.dside), side_of(M, q.sside), q.l0, q.a, q.b, q.trans, q.D, q.ldd, q.m, q.yh,
                     q.out, q.ldo, q.alpha, q.beta, q.ident, it, n, sm);
    } break;
    case OP_POTRF: {
      const PTile& q = *reinterpret_cast<const PTile*>(op.p);
      ar::it_potrf(M, q.slot, q.t, it, n, sm);
    } break;
    case OP_GETRF: {
      const PTile& q = *reinterpret_cast<const PTile*>(op.p);
      ar::it_getrf(M, q.slot, q.t, it, n, sm);
    } break;
    case OP_TINV: {
      const PTile& q = *reinterpret_cast<const PTile*>(op.p);
      ar::it_tinv(M, q.slot, q.t, it, n, sm);
    } break;
    case OP_TRSM: {
      const PTile& q = *reinterpret_cast<const PTile*>(op.p);
      ar::it_trsm(M, q.slot, q.m, q.mode, q.B, q.ldb, q.brows, q.bcols, it, n, sm);
    } break;
    case OP_TSQR: {
      const PTsqr& q = *reinterpret_cast<const PTsqr*>(op.p);
      ar::it_tsqr_r(q.A, q.lda, q.rows, q.K, q.R, q.ldr, it, n, sm);
    } break;
    case OP_TEMP: {
      const PTemp& q = *reinterpret_cast<const PTemp*>(op.p);
      ar::it_temp_core(q.Ra, q.Rb, q.ldr, q.K, q.Ma, q.Mb, q.ldm, q.rout, q.rel, q.abs_tol, q.max_rank, q.cap, q.flags,
                       q.knew, it, n, sm);
    } break;
    case OP_COPY_COLS: {
      const PMisc& q = *reinterpret_cast<const PMisc*>(op.p);
      ar::it_copy_cols(q.dst, q.ldd, q.src, q.lds, q.rows, q.d1, it, n, sm);
    } break;
    case OP_SET_INT: {
      const PMisc& q = *reinterpret_cast<const PMisc*>(op.p);
      ar::it_set_int(q.ip, q.d1, it, n, sm);
    } break;
    case OP_ADD_INT: {
      const PMisc& q = *reinterpret_cast<const PMisc*>(op.p);
      ar::it_add_int(q.ip, q.d1, q.d2, it, n, sm);
    } break;
    case OP_RANK_IF: {
      const PMisc& q = *reinterpret_cast<const PMisc*>(op.p);
      ar::it_rank_if(q.ip, q.ia, q.ib, it, n, sm);
    } break;
    case OP_STACK: {
      const PMisc& q = *reinterpret_cast<const PMisc*>(op.p);
      ar::it_stack(q.dst, q.ldd, q.rows, q.src, (int)q.ldx, q.ia, reinterpret_cast<const double*>(q.perm), q.lds,
                   q.row_off, q.rows_new, q.d1, it, n, sm);
    } break;
    case OP_CHOOSE: {
      const PMisc& q = *reinterpret_cast<const PMisc*>(op.p);
      ar::it_choose(q.src, q.lds, q.ia, q.ib, q.dst, reinterpret_cast<double*>(const_cast<int64_t*>(q.perm)), q.ldd,
                    q.ip, it, n, sm);
    } break;
    case OP_IDENTITY: {
      const PMisc& q = *reinterpret_cast<const PMisc*>(op.p);
      ar::it_identity(q.dst, q.ldd, q.rows, it, n, sm);
    } break;
    case OP_TRANSPOSE: {
      const PMisc& q = *reinterpret_cast<const PMisc*>(op.p);
      ar::it_transpose_tile(q.dst, q.ldd, q.src, q.lds, q.rows, q.cols, it, n, sm);
    } break;
    case OP_GATHER: {
      const PMisc& q = *reinterpret_cast<const PMisc*>(op.p);
      ar::it_gather_cols(q.dst, q.src, q.perm, q.rows, q.cols, q.ldx, it, n, sm);
    } break;
    case OP_DD: {
      const PDD& q = *reinterpret_cast<const PDD*>(op.p);
      ar::it_dd_compress(P.mats[q.mx], P.mats[q.my], q.slotx, q.transx, q.sloty, q.transy, q.mt, q.ms, q.mr, q.A,
                         q.lda, q.B, q.ldb, q.kout, q.rel, it, n, sm);
    } break;
    case OP_C2CORE: {
      ar::it_c2core(*reinterpret_cast<const PC2*>(op.p), sm);
    } break;
    case OP_NZTILE: {  // *ip = 0 if the nearfield tile is exactly zero (reading own-6)
      const PMisc& q = *reinterpret_cast<const PMisc*>(op.p);
      const double* T = q.src;
      int any = 0;
      for (int e = threadIdx.x; e < q.rows; e += NT) any |= (T[e] != 0.0);
      any = __syncthreads_or(any);
      if (!any && threadIdx.x == 0) *q.ip = 0;
    } break;
    case OP_KCHECK: {  // a contribution whose device rank exceeds the update capacity: flag it, drop it
      const PMisc& q = *reinterpret_cast<const PMisc*>(op.p);
      if (threadIdx.x == 0 && *q.ip > q.rows) {
        atomicOr(M.flags, 4);
        *q.ip = 0;
      }
    } break;
    case OP_ZERO: {
      const PMisc& q = *reinterpret_cast<const PMisc*>(op.p);
      for (long long e = (long long)it * NT + threadIdx.x; e < q.ldx; e += (long long)n * NT) q.dst[e] = 0.0;
    } break;
    case OP_SCATTER: {
      const PMisc& q = *reinterpret_cast<const PMisc*>(op.p);
      ar::it_scatter_cols(q.dst, q.src, q.perm, q.rows, q.cols, q.ldx, it, n, sm);
    } break;
    default:
      break;
  }
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Op records are staged in shared memory: the next record is loaded into registers while the
// current op runs and stored into the other slot before the op's closing barrier, so no op waits
// for an L2 round trip to learn what to do (the cluster barrier's acquire invalidates L1, which
// would otherwise drop a prefetched record).  A skip jumps over the prefetched record: the new next
// record is then fetched directly.
constexpr int REC_VEC = (int)(sizeof(OpRec) / sizeof(uint4));
static_assert(sizeof(OpRec) % sizeof(uint4) == 0 && REC_VEC <= NT, "op record staging");

__device__ __forceinline__ void stage_rec(OpRec* dst, const OpRec* src) {
  if (threadIdx.x < REC_VEC)
    reinterpret_cast<uint4*>(dst)[threadIdx.x] = __ldg(reinterpret_cast<const uint4*>(src) + threadIdx.x);
}

__global__ void __launch_bounds__(NT, 1) k_exec_cluster(const __grid_constant__ ExecParams P) {
  extern __shared__ __align__(16) double sm[];
  __shared__ __align__(16) OpRec srec[2];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank(), nb = (int)cl.num_blocks();
  const bool timing = P.prof && rank == 0 && threadIdx.x == 0;
  int cur = 0;
  if (P.begin < P.end) stage_rec(&srec[0], &P.ops[P.begin]);
  __syncthreads();
  for (int o = P.begin; o < P.end; ++o) {
    const OpRec& op = srec[cur];
    const int n = op.nitems;
    // the next record into registers (it arrives while this op runs)
    const bool pf = threadIdx.x < REC_VEC && o + 1 < P.end;
    uint4 nxt = make_uint4(0, 0, 0, 0);
    if (pf) nxt = __ldg(reinterpret_cast<const uint4*>(&P.ops[o + 1]) + threadIdx.x);
    bool jumped = false;
    if (op.code == OP_SKIPZ) {
      // Every CTA must take the same decision.  The flag was written before the barrier in front
      // of this op; the cluster barrier AFTER the read keeps any later op from overwriting it
      // while a slower CTA has still to read it.  (Without it, a skipped region followed by an op
      // that rewrites the same flag slot -- the workspace arena reuses it for the next
      // contribution's rank -- let a late CTA read the new value and run the region the others
      // skipped: the rare corrupted factorization of VERDICT r01.)
      const PMisc& q = *reinterpret_cast<const PMisc*>(op.p);
      const bool zero = *(volatile const int*)q.ip == 0;
      if (timing) {  // skip statistics per origin tag (h2_profile_ops slots 48 + tag: skipped, seen)
        atomicAdd(P.prof + 4 * K_COUNT + 32 + 2 * (48 + q.rows), zero ? 1.0 : 0.0);
        atomicAdd(P.prof + 4 * K_COUNT + 32 + 2 * (48 + q.rows) + 1, 1.0);
      }
      if (zero && q.cols > 0) {
        o += q.cols;
        jumped = true;
      }
      __syncthreads();  // every thread has read the record before the slot is reused
      if (jumped) {
        if (o + 1 < P.end) stage_rec(&srec[cur ^ 1], &P.ops[o + 1]);
      } else if (pf) {
        reinterpret_cast<uint4*>(&srec[cur ^ 1])[threadIdx.x] = nxt;
      }
      cl.sync();
      cur ^= 1;
      continue;
    }
    unsigned long long t0 = timing ? gtimer() : 0;
    const int off = (op.barrier >> 8) & 0xff;  // item i runs on CTA (off + i) mod nb
    for (int it = ((rank - off) % nb + nb) % nb; it < n; it += nb) {
      dispatch(P, op, it, n, sm);
      __syncthreads();
    }
    const int code = op.code, bar = op.barrier;
    __syncthreads();  // every thread is done with this record before its slot is reused
    if (pf) reinterpret_cast<uint4*>(&srec[cur ^ 1])[threadIdx.x] = nxt;
    // barrier.cluster.arrive (release) / wait (acquire) at cluster scope: this op's global-memory
    // results are visible to every CTA of the cluster afterwards
    if (bar & 1) cl.sync();
    else __syncthreads();
    cur ^= 1;
    if (timing) {
      const int kid = c_op_kid[code];
      const double dt = (double)(gtimer() - t0);
      atomicAdd(P.prof + 2 * K_COUNT + 2 * kid, dt);
      atomicAdd(P.prof + 2 * K_COUNT + 2 * kid + 1, 1.0);
      atomicAdd(P.prof + 4 * K_COUNT + 32 + 2 * code, dt);  // per op code (h2_profile_ops)
      atomicAdd(P.prof + 4 * K_COUNT + 32 + 2 * code + 1, 1.0);
    }
  }
}

__global__ void __launch_bounds__(NT, 1) k_exec_big(const __grid_constant__ ExecParams P, int o) {
  extern __shared__ __align__(16) double sm[];
  const OpRec& op = P.ops[o];
  for (int it = blockIdx.x; it < op.nitems; it += gridDim.x) {
    dispatch(P, op, it, op.nitems, sm);
    __syncthreads();
  }
}

// ---- host: recording context, upload, segmentation ----------------------------------------------
thread_local ExecCtx* g_ctx = nullptr;
bool g_attr = false;
double* g_gpart = nullptr;
OpRec* g_dops = nullptr;
size_t g_dcap = 0;
OpRec* g_hops[2] = {nullptr, nullptr};
size_t g_hcap[2] = {0, 0};
cudaEvent_t g_hev[2] = {nullptr, nullptr};
int g_hbuf = 0;
int g_nsm = 148;
int g_big = getenv("H2_EXEC_BIG") ? atoi(getenv("H2_EXEC_BIG")) : BIG;  // debug override
int g_cl = getenv("H2_EXEC_CL") ? atoi(getenv("H2_EXEC_CL")) : CL;   // executor cluster size

cudaError_t init_exec() {
  if (g_attr) return cudaSuccess;
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(k_exec_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM_EXEC))) return e;
  if (g_cl > 8) {
    // a non-portable cluster size: use it only if the device can place such a cluster
    int ncl = 0;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    cfg.gridDim = dim3(g_cl);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = SM_EXEC;
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = g_cl;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (cudaFuncSetAttribute(k_exec_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess ||
        cudaOccupancyMaxActiveClusters(&ncl, k_exec_cluster, &cfg) != cudaSuccess || ncl < 1)
      g_cl = 8;
    cudaGetLastError();
  }
  if ((e = cudaFuncSetAttribute(k_exec_big, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM_EXEC))) return e;
  if ((e = cudaMalloc(&g_gpart, sizeof(double) * ar::NPART * KC * KC))) return e;
  poison(g_gpart, sizeof(double) * ar::NPART * KC * KC);
  for (int i = 0; i < 2; ++i)
    if ((e = cudaEventCreateWithFlags(&g_hev[i], cudaEventDisableTiming))) return e;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&g_nsm, cudaDevAttrMultiProcessorCount, dev);
  g_attr = true;
  return cudaSuccess;
}

inline int cdiv(long long a, long long b) { return (int)((a + b - 1) / b); }

}  // namespace

int ExecCtx::mat_index(const MatDev& M) {
  for (int i = 0; i < EXEC_MATS; ++i)
    if (mats[i] == &M) return i;
  for (int i = 0; i < EXEC_MATS; ++i)
    if (!mats[i]) {
      mats[i] = &M;
      return i;
    }
  throw std::runtime_error("h2 executor: more than 3 matrices in one op list");
}

void ExecCtx::maybe_flush() {
  cudaError_t e = exec_flush();
  if (e != cudaSuccess) throw std::runtime_error(std::string("h2 executor: ") + cudaGetErrorString(e));
}

size_t default_flush_at() {
  static const size_t v = getenv("H2_EXEC_FLUSH") ? std::max(1, atoi(getenv("H2_EXEC_FLUSH"))) : 16384;
  return v;
}

ExecCtx* exec_ctx() { return g_ctx; }
int exec_big_items() { return g_big; }

size_t ExecCtx::begin_skip(const int* k) {
  PMisc q{};
  q.ip = const_cast<int*>(k);
  q.cols = 0;
  q.rows = skip_tag & 15;  // origin of the region (profiling statistics only)
  ++hold;  // before emit: a flush triggered by this very op would clear the list it indexes
  emit(OP_SKIPZ, 1, nullptr, q);
  return ops.size() - 1;
}

void ExecCtx::end_skip(size_t at, int big_items) {
  --hold;
  int cnt = (int)(ops.size() - at - 1);
  for (size_t i = at + 1; i < ops.size(); ++i)
    if (ops[i].nitems > big_items) cnt = 0;  // a full-grid op cannot be skipped from inside the cluster
  PMisc q;
  std::memcpy(&q, ops[at].p, sizeof(PMisc));
  q.cols = cnt;
  std::memcpy(ops[at].p, &q, sizeof(PMisc));
  if (ops.size() >= flush_at && hold == 0) maybe_flush();
}

void exec_begin(ExecCtx* ctx, cudaStream_t st) {
  ctx->st = st;
  ctx->ops.clear();
  for (int i = 0; i < EXEC_MATS; ++i) ctx->mats[i] = nullptr;  // a reused context starts empty
  ctx->hold = 0;
  ctx->group = 0;
  g_ctx = ctx;
}

cudaError_t exec_flush() {
  ExecCtx* c = g_ctx;
  if (!c || c->ops.empty()) return cudaSuccess;
  static const bool dry = getenv("H2_EXEC_DRYRUN") != nullptr;  // tools: time the host recording alone
  if (dry) {
    static FILE* tf = getenv("H2_EXEC_TRACE") ? fopen(getenv("H2_EXEC_TRACE"), "wb") : nullptr;
    if (tf) {  // (code, nitems, barrier) per op: the op mix of a recording (tools)
      for (const OpRec& r : c->ops) {
        const int32_t rec[3] = {r.code, r.nitems, r.barrier};
        fwrite(rec, sizeof(rec), 1, tf);
      }
      fflush(tf);
    }
    c->ops.clear();
    return cudaSuccess;
  }
  cudaError_t e = init_exec();
  if (e) return e;
  const size_t n = c->ops.size();
  // stage in a pinned buffer (double-buffered), upload, run
  const int hb = g_hbuf;
  g_hbuf ^= 1;
  {
    const auto w0 = std::chrono::steady_clock::now();
    if ((e = cudaEventSynchronize(g_hev[hb]))) return e;
    g_host_wait_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - w0).count();
  }
  if (g_hcap[hb] < n) {
    if (g_hops[hb]) cudaFreeHost(g_hops[hb]);
    g_hcap[hb] = std::max(n, (size_t)16384);
    if ((e = cudaMallocHost(&g_hops[hb], sizeof(OpRec) * g_hcap[hb]))) return e;
  }
  if (g_dcap < n) {
    // the previous executor launches read g_dops: wait for the stream before freeing it
    if (g_dops) {
      cudaStreamSynchronize(c->st);
      cudaFree(g_dops);
    }
    g_dcap = std::max(n, (size_t)16384);
    if ((e = cudaMalloc(&g_dops, sizeof(OpRec) * g_dcap))) return e;
  }
  std::memcpy(g_hops[hb], c->ops.data(), sizeof(OpRec) * n);
  if ((e = cudaMemcpyAsync(g_dops, g_hops[hb], sizeof(OpRec) * n, cudaMemcpyHostToDevice, c->st))) return e;
  if ((e = cudaEventRecord(g_hev[hb], c->st))) return e;
  ExecParams P;
  P.ops = g_dops;
  P.prof = prof_dev();
  P.gpart = g_gpart;
  for (int i = 0; i < EXEC_MATS; ++i) {
    if (c->mats[i]) P.mats[i] = *c->mats[i];
    else std::memset(&P.mats[i], 0, sizeof(MatDev));
  }
  size_t b = 0;
  auto run_cluster = [&](size_t lo, size_t hi) -> cudaError_t {
    if (hi <= lo) return cudaSuccess;
    P.begin = (int)lo;
    P.end = (int)hi;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(g_cl);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = SM_EXEC;
    cfg.stream = c->st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = g_cl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    count_launch(1);
    return cudaLaunchKernelEx(&cfg, k_exec_cluster, P);
  };
  for (size_t i = 0; i < n; ++i) {
    const OpRec& r = c->ops[i];
    if (r.nitems > g_big) {
      if ((e = run_cluster(b, i))) return e;
      const int kid = r.code < 9 ? r.code : K_AR_HMUL;
      prof_begin(kid, c->st);
      count_launch(1);
      k_exec_big<<<std::min(r.nitems, g_nsm), NT, SM_EXEC, c->st>>>(P, (int)i);
      prof_end(kid, c->st);
      if ((e = cudaGetLastError())) return e;
      b = i + 1;
    }
  }
  if ((e = run_cluster(b, n))) return e;
  c->ops.clear();
  return cudaGetLastError();
}

cudaError_t exec_end() {
  cudaError_t e = exec_flush();
  g_ctx = nullptr;
  return e;
}

// ------------------------------------------------------------------------------------------------
// emitters of the local update (U0..U6)
// ------------------------------------------------------------------------------------------------
namespace {

void level_segment(const h2_tree_* T, int root, int L, int* begin, int* count) {
  *begin = 0;
  *count = 0;
  if (L > T->depth || L < T->level[root]) return;
  const int* b = T->bfs.data() + T->level_ptr[L];
  const int* e = T->bfs.data() + T->level_ptr[L + 1];
  const int* lo = std::lower_bound(b, e, root);
  const int* hi = std::lower_bound(b, e, root + T->tsize[root]);
  *begin = (int)(lo - T->bfs.data());
  *count = (int)(hi - lo);
}

void leaf_range(const h2_tree_* T, int root, int* begin, int* count) {
  const auto b = T->leaves.begin(), e = T->leaves.end();
  const auto lo = std::lower_bound(b, e, root);
  const auto hi = std::lower_bound(b, e, root + T->tsize[root]);
  *begin = (int)(lo - b);
  *count = (int)(hi - lo);
}

PUpd pu(const UpdArgs& a, int i0 = 0, int i1 = 0, int i2 = 0, int i3 = 0, int i4 = 0, int i5 = 0, int i6 = 0,
        int i7 = 0) {
  PUpd p;
  p.a = a;
  p.i[0] = i0;
  p.i[1] = i1;
  p.i[2] = i2;
  p.i[3] = i3;
  p.i[4] = i4;
  p.i[5] = i5;
  p.i[6] = i6;
  p.i[7] = i7;
  return p;
}

struct AutoCtx {  // a local recording context when the caller has none
  ExecCtx local;
  bool own;
  explicit AutoCtx(cudaStream_t st) : own(exec_ctx() == nullptr) {
    if (own) exec_begin(&local, st);
  }
  ExecCtx* get() { return exec_ctx(); }
  cudaError_t done() { return own ? exec_end() : cudaSuccess; }
};

}  // namespace

cudaError_t update_init_attributes() { return init_exec(); }

cudaError_t launch_update(const h2_mat_* Z, const UpdArgs& a_in, cudaStream_t st) {
  UpdArgs a = a_in;
  a.prof = prof_dev();
  AutoCtx ac(st);
  ExecCtx* c = ac.get();
  const MatDev& M = Z->d;
  const h2_btree_* B = Z->bt;
  const h2_tree_* R = B->rt;
  const h2_tree_* C = B->ct;
  const int b0 = B->find(a.t0, a.s0);
  const int in0 = Z->inad_range[2 * b0], nin = Z->inad_range[2 * b0 + 1] - in0;
  if (B->kind[b0] == INADM) {  // dense add only
    c->emit(OP_UPD_EXT_LEAF, nin, &M, pu(a, 0, 0, 0, 0, in0, nin, 0, 0));
    return ac.done();
  }
  // a device-determined rank (internal callers) may be zero at run time: skip the whole update
  static const bool no_skip = getenv("H2_NO_SKIP") != nullptr;  // A/B switch (tools)
  const bool skip = a.kdev && !no_skip;
  const size_t skip_at = skip ? c->begin_skip(a.kdev) : 0;
  int rl0, nrl, cl0, ncl;
  leaf_range(R, a.t0, &rl0, &nrl);
  leaf_range(C, a.s0, &cl0, &ncl);
  const int Lr = R->level[a.t0], Lc = C->level[a.s0];
  c->emit(OP_UPD_EXT_LEAF, nrl + ncl + nin + Lr + Lc, &M, pu(a, rl0, nrl, cl0, ncl, in0, nin, Lr, Lc));
  const int Lmax = std::max(R->depth, C->depth), Lmin = std::min(Lr, Lc);
  for (int L = Lmax - 1; L >= Lmin; --L) {  // U2 bottom-up (internal clusters)
    int bA, nA, bB, nB;
    level_segment(R, a.t0, L, &bA, &nA);
    level_segment(C, a.s0, L, &bB, &nB);
    c->emit(OP_UPD_EXT_LEVEL, nA + nB, &M, pu(a, bA, nA, bB, nB));
  }
  c->emit(OP_UPD_W_PATH, 2, &M, pu(a, rl0, cl0, Lr, Lc));  // U3: path root .. t0
  for (int L = Lmin + 1; L <= Lmax; ++L) {  // U3: subtree top-down
    int bA = 0, nA = 0, bB = 0, nB = 0;
    if (L > Lr) level_segment(R, a.t0, L, &bA, &nA);
    if (L > Lc) level_segment(C, a.s0, L, &bB, &nB);
    c->emit(OP_UPD_W_LEVEL, nA + nB, &M, pu(a, bA, nA, bB, nB));
  }
  c->emit(OP_UPD_SVD_LEAF, nrl + ncl, &M, pu(a, rl0, nrl, cl0, ncl));  // U4 bottom-up
  for (int L = Lmax - 1; L >= Lmin; --L) {
    int bA, nA, bB, nB;
    level_segment(R, a.t0, L, &bA, &nA);
    level_segment(C, a.s0, L, &bB, &nB);
    c->emit(OP_UPD_SVD_LEVEL, nA + nB, &M, pu(a, bA, nA, bB, nB));
  }
  const int nA = R->tsize[a.t0], nB = C->tsize[a.s0];
  c->emit(OP_UPD_COUPLE, nA + nB, &M, pu(a, nA, nB));   // U5
  c->emit(OP_UPD_INSTALL, nA + nB, &M, pu(a, nA, nB));  // U6
  c->emit(OP_UPD_RCACHE, Lr + Lc, &M, pu(a, rl0, cl0, Lr, Lc));  // R-factor caches on pred(t0), pred(s0): item per ancestor
  if (skip) c->end_skip(skip_at, g_big);
  return ac.done();
}

// ------------------------------------------------------------------------------------------------
// emitters of the arithmetic primitives (declared in h2_arith.cuh)
// ------------------------------------------------------------------------------------------------
static ExecCtx* ctx_or_throw() {
  ExecCtx* c = exec_ctx();
  if (!c) throw std::runtime_error("h2 executor: no recording context");
  return c;
}

static int side_id(const MatDev& M, const DevSide& D) { return &D == &M.col ? 1 : 0; }

void expand_basis(const MatDev& M, const DevSide& D, int t, double* out, int ld, cudaStream_t) {
  int l0, nl;
  leaf_range(D.tree, t, &l0, &nl);
  ctx_or_throw()->emit(OP_EXPAND, nl, &M, PExpand{side_id(M, D), t, l0, ld, out});
}

void gemm(double* C, int ldc, const double* A, int lda, bool ta, const double* B, int ldb, bool tb, Dim m, Dim n,
          Dim k, int mcap, int ncap, int kcap, double alpha, double beta, cudaStream_t) {
  if (mcap <= 0 || ncap <= 0) return;
  ExecCtx* c = ctx_or_throw();
  PGemm g;
  g.C = C;
  g.A = A;
  g.B = B;
  g.ldc = ldc;
  g.lda = lda;
  g.ldb = ldb;
  g.ta = ta;
  g.tb = tb;
  g.m = m;
  g.n = n;
  g.k = k;
  g.alpha = alpha;
  g.beta = beta;
  if (kcap > 512 && mcap <= KC && ncap <= KC) {
    g.chunk = (kcap + ar::NPART - 1) / ar::NPART;
    c->emit(OP_GEMM_PART, ar::NPART, nullptr, g);
    g.chunk = ar::NPART;  // number of partials to sum
    c->emit(OP_GEMM_SUM, 1, nullptr, g);
    return;
  }
  g.chunk = 0;
  const long long tot = (long long)mcap * ncap;
  c->emit(OP_GEMM, std::max(1, std::min(cdiv(tot, NT), 4 * 148)), nullptr, g);
}

void hmul_dense(const MatDev& M, bool trans, int a, int b, int b_blk, const double* D, int ldd, Dim m, int mcap,
                double* out, int ldo, double alpha, double beta, cudaStream_t) {
  (void)mcap;
  ExecCtx* c = ctx_or_throw();
  const DevSide& Dd = trans ? M.col : M.row;
  const DevSide& Ds = trans ? M.row : M.col;
  const h2_tree_* Td = Dd.tree;
  const h2_tree_* Ts = Ds.tree;
  PHm h;
  h.dside = trans ? 1 : 0;
  h.sside = trans ? 0 : 1;
  h.a = a;
  h.b = b;
  h.trans = trans ? 1 : 0;
  h.D = D;
  h.ldd = ldd;
  h.ldo = ldo;
  h.xh = Ds.hx;
  h.yh = Dd.hy;
  h.out = out;
  h.m = m;
  h.alpha = alpha;
  h.beta = beta;
  h.ident = b_blk;  // 1: D is the identity
  int l0, nl;
  leaf_range(Ts, b, &l0, &nl);
  h.l0 = l0;
  h.base_lo = Ts->lo[b];
  c->emit(OP_HM_FWD_LEAF, nl, &M, h);
  for (int L = Ts->depth - 1; L >= Ts->level[b]; --L) {
    int s0, ns;
    level_segment(Ts, b, L, &s0, &ns);
    h.l0 = s0;
    c->emit(OP_HM_FWD_LEVEL, ns, &M, h);
  }
  c->emit(OP_HM_COUPLE, Td->tsize[a], &M, h);
  for (int L = Td->level[a] + 1; L <= Td->depth; ++L) {
    int s0, ns;
    level_segment(Td, a, L, &s0, &ns);
    h.l0 = s0;
    c->emit(OP_HM_BWD_LEVEL, ns, &M, h);
  }
  int la0, nla;
  leaf_range(Td, a, &la0, &nla);
  h.l0 = la0;
  c->emit(OP_HM_LEAF, nla, &M, h);
}

void tile_potrf(const MatDev& M, int slot, int t, cudaStream_t) {
  ctx_or_throw()->emit(OP_POTRF, 1, &M, PTile{slot, t, 0, 0, 0, 0, nullptr, dimc(0)});
}
void tile_getrf(const MatDev& M, int slot, int t, cudaStream_t) {
  ctx_or_throw()->emit(OP_GETRF, 1, &M, PTile{slot, t, 0, 0, 0, 0, nullptr, dimc(0)});
}
void tile_inverse(const MatDev& M, int slot, int t, cudaStream_t) {
  ctx_or_throw()->emit(OP_TINV, 1, &M, PTile{slot, t, 0, 0, 0, 0, nullptr, dimc(0)});
}
void tile_trsm(const MatDev& M, int slot, int m, int mode, double* B, int ldb, int brows, Dim bcols, int bcolcap,
               cudaStream_t) {
  const bool rowwise = (mode == RLT || mode == RUN);
  const int nvec = rowwise ? brows : bcolcap;
  ctx_or_throw()->emit(OP_TRSM, std::max(1, cdiv(nvec, NT)), &M, PTile{slot, 0, m, mode, ldb, brows, B, bcols});
}
void tsqr_r(const double* A, int lda, int rows, Dim K, double* R, int ldr, cudaStream_t) {
  ctx_or_throw()->emit(OP_TSQR, 1, nullptr, PTsqr{A, R, lda, rows, ldr, K});
}
void temp_core(const double* Ra, const double* Rb, int ldr, Dim K, double* Ma, double* Mb, int ldm, int* rout,
               double rel, double abs_tol, int max_rank, int cap, int* flags, const int* knew, cudaStream_t) {
  ctx_or_throw()->emit(OP_TEMP, 1, nullptr,
                       PTemp{Ra, Rb, Ma, Mb, rout, flags, knew, ldr, ldm, max_rank, cap, K, rel, abs_tol});
}

static PMisc misc() {
  PMisc q;
  std::memset(&q, 0, sizeof(q));
  return q;
}

void copy_cols(double* dst, int ldd, const double* src, int lds, int rows, Dim cols, int colcap, cudaStream_t) {
  const long long tot = (long long)rows * colcap;
  if (tot <= 0) return;
  PMisc q = misc();
  q.dst = dst;
  q.ldd = ldd;
  q.src = src;
  q.lds = lds;
  q.rows = rows;
  q.d1 = cols;
  ctx_or_throw()->emit(OP_COPY_COLS, std::max(1, std::min(cdiv(tot, NT), 4 * 148)), nullptr, q);
}
void set_int(int* p, Dim v, cudaStream_t) {
  PMisc q = misc();
  q.ip = p;
  q.d1 = v;
  ctx_or_throw()->emit(OP_SET_INT, 1, nullptr, q);
}
void add_int(int* p, Dim a, Dim b, cudaStream_t) {
  PMisc q = misc();
  q.ip = p;
  q.d1 = a;
  q.d2 = b;
  ctx_or_throw()->emit(OP_ADD_INT, 1, nullptr, q);
}
void rank_check(const MatDev& M, int* kdev, int cap, cudaStream_t) {
  PMisc q = misc();
  q.ip = kdev;
  q.rows = cap;
  ctx_or_throw()->emit(OP_KCHECK, 1, &M, q);
}
void rank_if(int* p, const int* a, const int* b, cudaStream_t) {
  PMisc q = misc();
  q.ip = p;
  q.ia = a;
  q.ib = b;
  ctx_or_throw()->emit(OP_RANK_IF, 1, nullptr, q);
}
void stack_cols(double* dst, int ldd, int rows, const double* T, int ldt, const int* kT, const double* Nw, int ldn,
                int row_off, int rows_new, Dim knew, int colcap, cudaStream_t) {
  PMisc q = misc();
  q.dst = dst;
  q.ldd = ldd;
  q.rows = rows;
  q.src = T;
  q.ldx = ldt;
  q.ia = kT;
  q.perm = reinterpret_cast<const int64_t*>(Nw);
  q.lds = ldn;
  q.row_off = row_off;
  q.rows_new = rows_new;
  q.d1 = knew;
  const long long tot = (long long)rows * colcap;
  ctx_or_throw()->emit(OP_STACK, std::max(1, std::min(cdiv(tot, NT), 4 * 148)), nullptr, q);
}
void choose_case2(const double* Cm, int ldc, const int* k1, const int* k2, double* Ca, double* Cb, int ldo, int* kout,
                  cudaStream_t) {
  PMisc q = misc();
  q.src = Cm;
  q.lds = ldc;
  q.ia = k1;
  q.ib = k2;
  q.dst = Ca;
  q.perm = reinterpret_cast<const int64_t*>(Cb);
  q.ldd = ldo;
  q.ip = kout;
  ctx_or_throw()->emit(OP_CHOOSE, 1, nullptr, q);
}
void case2_core(const double* W, const double* V, int ms, const double* G, const double* Sx, int ldsx, bool tx,
                const double* Sy, int ldsy, bool ty, const int* kxt, const int* kxs, const int* kys, const int* kyr,
                double* Ca, double* Cb, int ldo, int* kout, cudaStream_t) {
  PC2 q;
  q.W = W;
  q.V = V;
  q.G = G;
  q.Sx = Sx;
  q.Sy = Sy;
  q.Ca = Ca;
  q.Cb = Cb;
  q.kd[0] = kxt;
  q.kd[1] = kxs;
  q.kd[2] = kys;
  q.kd[3] = kyr;
  q.kout = kout;
  q.ms = ms;
  q.ldsx = ldsx;
  q.ldsy = ldsy;
  q.tx = tx ? 1 : 0;
  q.ty = ty ? 1 : 0;
  q.ldo = ldo;
  ctx_or_throw()->emit(OP_C2CORE, 1, nullptr, q);
}
int case2_core_max_ms() { return ar::C2_MS; }
void identity(double* I, int ld, int m, cudaStream_t) {
  PMisc q = misc();
  q.dst = I;
  q.ldd = ld;
  q.rows = m;
  ctx_or_throw()->emit(OP_IDENTITY, std::max(1, cdiv(m * m, NT)), nullptr, q);
}
void transpose_tile(double* dst, int ldd, const double* src, int lds, int rows, int cols, cudaStream_t) {
  PMisc q = misc();
  q.dst = dst;
  q.ldd = ldd;
  q.src = src;
  q.lds = lds;
  q.rows = rows;
  q.cols = cols;
  ctx_or_throw()->emit(OP_TRANSPOSE, std::max(1, cdiv(rows * cols, NT)), nullptr, q);
}
void gather_cols(double* Bt, const double* x, const int64_t* perm, int n, int nrhs, int64_t ldx, cudaStream_t) {
  PMisc q = misc();
  q.dst = Bt;
  q.src = x;
  q.perm = perm;
  q.rows = n;
  q.cols = nrhs;
  q.ldx = ldx;
  ctx_or_throw()->emit(OP_GATHER, std::max(1, std::min(cdiv((long long)n * nrhs, NT), 8 * 148)), nullptr, q);
}
void scatter_cols(double* x, const double* Bt, const int64_t* perm, int n, int nrhs, int64_t ldx, cudaStream_t) {
  PMisc q = misc();
  q.dst = x;
  q.src = Bt;
  q.perm = perm;
  q.rows = n;
  q.cols = nrhs;
  q.ldx = ldx;
  ctx_or_throw()->emit(OP_SCATTER, std::max(1, std::min(cdiv((long long)n * nrhs, NT), 8 * 148)), nullptr, q);
}

}  // namespace h2

namespace h2 {
void zero_fill(double* dst, size_t count, cudaStream_t) {
  PMisc q;
  std::memset(&q, 0, sizeof(q));
  q.dst = dst;
  q.ldx = (int64_t)count;
  ctx_or_throw()->emit(OP_ZERO, std::max(1, std::min(cdiv((long long)count, NT), 4 * 148)), nullptr, q);
}
}  // namespace h2

namespace h2 {
void dd_compress(const MatDev& MX, int slotx, bool transx, const MatDev& MY, int sloty, bool transy, int mt, int ms,
                 int mr, double* A, int lda, double* B, int ldb, int* kout, double rel, cudaStream_t) {
  ExecCtx* c = ctx_or_throw();
  PDD q;
  q.mx = c->mat_index(MX);
  q.my = c->mat_index(MY);
  q.slotx = slotx;
  q.sloty = sloty;
  q.transx = transx ? 1 : 0;
  q.transy = transy ? 1 : 0;
  q.mt = mt;
  q.ms = ms;
  q.mr = mr;
  q.A = A;
  q.lda = lda;
  q.B = B;
  q.ldb = ldb;
  q.kout = kout;
  q.rel = rel;
  c->emit(OP_DD, 1, nullptr, q);
}
}  // namespace h2

namespace h2 {
void zero_rank_if_zero_tile(const MatDev& M, int slot, int count, int* kdev, cudaStream_t) {
  (void)count;
  PMisc q;
  std::memset(&q, 0, sizeof(q));
  q.src = M.N + (size_t)slot * M.lmax * M.lmax;
  q.rows = M.lmax * M.lmax;  // padding of the tile slots is zero
  q.ip = kdev;
  ctx_or_throw()->emit(OP_NZTILE, 1, nullptr, q);
}
}  // namespace h2
