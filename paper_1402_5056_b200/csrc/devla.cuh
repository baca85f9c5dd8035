// CTA-level dense FP64 kernels for the small matrices of the local update.
// One CTA owns one small matrix staged in shared memory; all routines must be called by every
// thread of the block (they contain __syncthreads()).
#pragma once
#include <cuda_runtime.h>
#include <math.h>

namespace h2 {
namespace la {

__device__ __forceinline__ int pow2floor(int x) {
  int p = 1;
  while (p * 2 <= x) p *= 2;
  return p;
}

// 1/x and 1/sqrt(x): the FP64 division and rsqrt of the hardware math library (measured on
// B200: 74 / 68 cycles latency, vs ~200 for a float seed + Newton steps, tools/lat_bench).
__device__ __forceinline__ double fast_rcp(double x) { return 1.0 / x; }
__device__ __forceinline__ double fast_rsqrt(double x) { return rsqrt(x); }

__device__ __forceinline__ unsigned group_mask(int S) {
  if (S >= 32) return 0xffffffffu;
  const int lane = threadIdx.x & 31;
  return ((1u << S) - 1u) << (lane & ~(S - 1));
}

// Warp-level Householder QR (one warp, no block barriers): lanes own rows (row i = lane + 32 q,
// q < ceil(m/32) <= 6), so every dot product is one 5-step butterfly; the Householder vector
// v = a_j[j:] - alpha e_1 stays in registers.  a_c <- a_c - (v^T a_c / (|a_j|^2 - alpha a_jj)) v.
// Leaves R in the upper triangle of the first min(m,n) rows, except the diagonal which is
// written to diag[] (strictly-lower part keeps the reflector data).  m <= 192.
__device__ __forceinline__ double warp_allsum(double p) {
#pragma unroll
  for (int o = 16; o; o >>= 1) p += __shfl_xor_sync(0xffffffffu, p, o);
  return p;
}

static __device__ void warp_qr_R(double* A, int lda, int m, int n, double* diag) {
  const int lane = threadIdx.x & 31;
  const int RP = (m + 31) >> 5;
  const int jmax = m < n ? m : n;
  for (int j = 0; j < jmax; ++j) {
    double v[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      const int i = lane + 32 * q;
      v[q] = (q < RP && i >= j && i < m) ? A[i + j * lda] : 0.0;
    }
    double p = 0.0;
#pragma unroll
    for (int q = 0; q < 6; ++q) p += v[q] * v[q];
    const double nrm2 = warp_allsum(p);
    const double ajj = A[j + j * lda];
    if (!(nrm2 > 0.0)) {
      if (lane == 0) diag[j] = 0.0;
      __syncwarp();
      continue;
    }
    const double nrm = sqrt(nrm2);
    const double alpha = ajj > 0.0 ? -nrm : nrm;
    const double inv_h = 1.0 / (nrm2 - alpha * ajj);
#pragma unroll
    for (int q = 0; q < 6; ++q)
      if (lane + 32 * q == j) v[q] = ajj - alpha;
    int c = j + 1;
    for (; c + 1 < n; c += 2) {
      double p0 = 0.0, p1 = 0.0;
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        if (q < RP) {
          const int i = lane + 32 * q;
          if (i < m) {
            p0 += v[q] * A[i + c * lda];
            p1 += v[q] * A[i + (c + 1) * lda];
          }
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        p0 += __shfl_xor_sync(0xffffffffu, p0, o);
        p1 += __shfl_xor_sync(0xffffffffu, p1, o);
      }
      const double f0 = p0 * inv_h, f1 = p1 * inv_h;
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        if (q < RP) {
          const int i = lane + 32 * q;
          if (i < m && i >= j) {
            A[i + c * lda] -= f0 * v[q];
            A[i + (c + 1) * lda] -= f1 * v[q];
          }
        }
      }
    }
    if (c < n) {
      double p0 = 0.0;
#pragma unroll
      for (int q = 0; q < 6; ++q)
        if (q < RP && lane + 32 * q < m) p0 += v[q] * A[lane + 32 * q + c * lda];
      p0 = warp_allsum(p0);
      const double f0 = p0 * inv_h;
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        const int i = lane + 32 * q;
        if (q < RP && i < m && i >= j) A[i + c * lda] -= f0 * v[q];
      }
    }
    if (lane == 0) diag[j] = alpha;
    __syncwarp();
  }
}

// In-place Householder QR of the m x n column-major matrix A (lda) in shared memory; on return
// the first min(m,n) rows hold R (upper trapezoidal, strictly-lower part zeroed).  Only the
// R-factor is needed by the method ("P_t ... are not computed").
// One reduction per column: all dots d_c = a_j[j:]^T a_c[j:] are formed together (S lanes per
// column, butterfly within the lane group), and with v = a_j[j:] - alpha e_1:
// v^T a_c = d_c - alpha a_jc,  v^T v / 2 = |a_j|^2 - alpha a_jj.
// (A one-warp variant, warp_qr_R above, measured ~2x slower on B200: serial shuffle chains.)
static __device__ void cta_qr_R(double* A, int lda, int m, int n, double* diag, double* red) {
  const int tid = threadIdx.x, nt = blockDim.x;
  int npow = 1;
  while (npow < n) npow *= 2;
  int S = nt / npow;
  if (S > 32) S = 32;
  if (S < 1) S = 1;
  const int c = tid / S, sl = tid % S;
  const unsigned gm = group_mask(S);
  const int jmax = m < n ? m : n;
  __syncthreads();
  for (int j = 0; j < jmax; ++j) {
    double part = 0.0;
    // every active group also forms |a_j|^2 itself (same lanes, same order as column j's own
    // group, hence bit-identical), so no broadcast through shared memory and one barrier per column
    double nj = 0.0;
    if (c >= j && c < n)
      for (int i = j + sl; i < m; i += S) {
        const double aij = A[i + j * lda];
        part += aij * A[i + c * lda];
        nj += aij * aij;
      }
    for (int o = S / 2; o; o >>= 1) {
      part += __shfl_xor_sync(0xffffffffu, part, o);
      nj += __shfl_xor_sync(0xffffffffu, nj, o);
    }
    if (c >= j && c < n) {
      const double nrm2 = nj;
      const double ajj = A[j + j * lda];
      if (nrm2 > 0.0) {
        const double nrm = sqrt(nrm2);
        const double alpha = ajj > 0.0 ? -nrm : nrm;
        const double half_vtv = nrm2 - alpha * ajj;
        if (c > j) {
          const double ajc = A[j + c * lda];
          __syncwarp(gm);
          const double f = (part - alpha * ajc) / half_vtv;
          for (int i = j + sl; i < m; i += S) {
            const double vi = (i == j) ? (ajj - alpha) : A[i + j * lda];
            A[i + c * lda] -= f * vi;
          }
        } else if (sl == 0) {
          diag[j] = alpha;
        }
      } else if (c == j && sl == 0) {
        diag[j] = 0.0;
      }
    }
    __syncthreads();
  }
  for (int e = tid; e < jmax * n; e += nt) {
    const int i = e % jmax, cc = e / jmax;
    if (cc < i) A[i + cc * lda] = 0.0;
    else if (cc == i) A[i + cc * lda] = diag[i];
  }
  __syncthreads();
}

// C (m x n, ldc) = op(A) op(B) (+ C if accumulate); A: m x kk (or kk x m if ta), B: kk x n (or n x kk if tb).
// Any pointers (shared or global).  Every thread of the CTA participates.
static __device__ void cta_gemm(double* C, int ldc, const double* A, int lda, bool ta, const double* B, int ldb, bool tb,
                         int m, int n, int kk, bool accumulate) {
  for (int e = threadIdx.x; e < m * n; e += blockDim.x) {
    const int i = e % m, j = e / m;
    double acc = accumulate ? C[i + j * ldc] : 0.0;
    for (int q = 0; q < kk; ++q) {
      const double a = ta ? A[q + i * lda] : A[i + q * lda];
      const double b = tb ? B[j + q * ldb] : B[q + j * ldb];
      acc += a * b;
    }
    C[i + j * ldc] = acc;
  }
}

__device__ __forceinline__ void cta_fill(double* A, int lda, int m, int n, double v) {
  for (int e = threadIdx.x; e < m * n; e += blockDim.x) A[(e % m) + (e / m) * lda] = v;
}

__device__ __forceinline__ void cta_copy(double* D, int ldd, const double* Sx, int lds, int m, int n) {
  for (int e = threadIdx.x; e < m * n; e += blockDim.x) D[(e % m) + (e / m) * ldd] = Sx[(e % m) + (e / m) * lds];
}

// One-sided (Hestenes) Jacobi SVD of the m x p matrix M (ldm, shared memory): orthogonalises the
// columns by plane rotations until |a_i^T a_j| <= tol sqrt(|a_i|^2 |a_j|^2) for every pair (cyclic
// round-robin ordering, p/2 disjoint pairs per round).  On return column j of M is sigma_j u_j
// (unsorted); sig[j] = |M(:,j)|; order[q] = index of the q-th largest sigma (ties by index).
// scratch: >= 2 ints of shared memory.
static __device__ int cta_jacobi(double* M, int ldm, int m, int p, double* sig, int* order, int* scratch) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int pp = p + (p & 1);
  const int npairs = pp / 2;
  int G = npairs > 0 ? pow2floor(nt / npairs) : 32;
  if (G > 32) G = 32;
  if (G < 1) G = 1;
  const int q = tid / G, g = tid % G;
  // stop when every pair satisfies |a_i^T a_j| <= m eps |a_i| |a_j| (compared in squares)
  const double tol = (m > 8 ? m : 8) * 2.220446049250313e-16;
  const double tol2 = tol * tol;
  const int nr = pp - 1;  // rounds per sweep
  int nsw = 0;
  for (int sweep = 0; sweep < 40 && p > 1; ++sweep) {
    ++nsw;
    if (tid == 0) scratch[0] = 0;
    __syncthreads();
    for (int r = 0; r < nr; ++r) {
      int a = -1, b = -1;
      if (q < npairs) {
        if (q == 0) {
          a = 0;
          b = (r % nr) + 1;
        } else {
          a = ((r + q) % nr) + 1;
          b = ((r - q + nr) % nr) + 1;
        }
        if (a >= p || b >= p) a = b = -1;
      }
      double al = 0.0, be = 0.0, ga = 0.0;
      if (a >= 0)
        for (int i = g; i < m; i += G) {
          const double x = M[i + a * ldm], y = M[i + b * ldm];
          al += x * x;
          be += y * y;
          ga += x * y;
        }
      for (int o = G / 2; o; o >>= 1) {
        al += __shfl_xor_sync(0xffffffffu, al, o);
        be += __shfl_xor_sync(0xffffffffu, be, o);
        ga += __shfl_xor_sync(0xffffffffu, ga, o);
      }
      if (a >= 0 && ga != 0.0 && ga * ga > tol2 * al * be) {
        // tan of the Jacobi angle, t = sign(z) / (|z| + sqrt(1 + z^2)), z = (beta - alpha) / (2 gamma);
        // reciprocals / rsqrt from a float seed + Newton steps in FP64 (full precision, fewer cycles)
        const double zeta = (be - al) * fast_rcp(2.0 * ga);
        double t;
        if (fabs(zeta) > 1e15) t = 0.5 * fast_rcp(zeta);
        else {
          const double w = 1.0 + zeta * zeta;
          t = copysign(fast_rcp(fabs(zeta) + w * fast_rsqrt(w)), zeta);
        }
        const double cs = fast_rsqrt(1.0 + t * t), sn = cs * t;
        for (int i = g; i < m; i += G) {
          const double x = M[i + a * ldm], y = M[i + b * ldm];
          M[i + a * ldm] = cs * x - sn * y;
          M[i + b * ldm] = sn * x + cs * y;
        }
        if (g == 0) scratch[0] = 1;
      }
      __syncthreads();
    }
    const int changed = scratch[0];
    __syncthreads();
    if (!changed) break;
  }
  // column norms
  for (int j = tid; j < p; j += nt) {
    double s = 0.0;
    for (int i = 0; i < m; ++i) s += M[i + j * ldm] * M[i + j * ldm];
    sig[j] = sqrt(s);
  }
  __syncthreads();
  for (int j = tid; j < p; j += nt) {
    int pos = 0;
    const double sj = sig[j];
    for (int i = 0; i < p; ++i) pos += (sig[i] > sj) || (sig[i] == sj && i < j);
    order[pos] = j;
  }
  __syncthreads();
  return nsw;
}

// Keeps the compiler from speculating a division / square root on the unselected operand.
__device__ __forceinline__ double opaque(double x) {
  asm volatile("" : "+d"(x));
  return x;
}

// Jacobi rotation (c, s) that orthogonalises columns x, y with al = |x|^2, be = |y|^2, ga = x.y:
// t = sign(z) / (|z| + sqrt(1 + z^2)), z = (be - al) / (2 ga), written with one division as
// t = sign(d) 2 ga / (|d| + sqrt(d^2 + 4 ga^2)), d = be - al (sign(0) = +1; both forms are the
// same number, the second has one dependent DDIV less per Jacobi round); c = 1/sqrt(1 + t^2),
// s = c t.  Only called with ga != 0.
__device__ __forceinline__ void jacobi_rot(double al, double be, double ga, double* c, double* s) {
  const double d = be - al;
  const double g2 = 2.0 * ga;
  const double t = (d >= 0.0 ? g2 : -g2) / (fabs(d) + sqrt(fma(d, d, g2 * g2)));
  *c = rsqrt(fma(t, t, 1.0));
  *s = *c * t;
}

// One-sided Jacobi on a small matrix A (n x K, n <= NB, K <= 32; smem, ld lda) held in registers
// by one warp: lane j owns column j (and, if ACC, column j of the accumulated rotation J, which
// needs K <= NB).  Rounds pair the columns by the same round-robin tournament as cta_jacobi; the
// two lanes of a pair exchange columns by shuffles and compute the same rotation bit for bit
// (the sums are formed in the same order on both lanes, roles by index), branch-free:
// own' = c own + sgn s other with sgn = -1 on the lower index.  Stops when every pair satisfies
// |a_i^T a_j| <= max(n, 8) eps |a_i| |a_j|.  On return sig[j] = |(A J)(:, j)|, order[] as in
// cta_jacobi, and out (ld ldo) = J (K x K) if ACC, else A J (n x K) = [sigma_j u_j].
// Called by every thread of the CTA (warp 0 computes).
template <int NB, bool ACC>
static __device__ int warp_jacobi(const double* A, int lda, int n, int K, double* out, int ldo, double* sig,
                                  int* order, int* scratch) {
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid < 32) {
    double c[NB], v[ACC ? NB : 1];
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      c[i] = (lane < K && i < n) ? A[i + lane * lda] : 0.0;
      if (ACC) v[i] = (i == lane) ? 1.0 : 0.0;
    }
    const int pp = K + (K & 1), nr = pp - 1;
    const double tol = (n > 8 ? n : 8) * 2.220446049250313e-16;
    const double tol2 = tol * tol;
    int nsw = 0;
    for (int sweep = 0; sweep < 40 && K > 1; ++sweep) {
      ++nsw;
      int rot = 0;
      for (int r = 0; r < nr; ++r) {
        int part;
        if (lane == 0) part = r + 1;
        else {
          const int x = lane - 1;
          int y = 2 * r - x;
          if (y < 0) y += nr;
          if (y >= nr) y -= nr;
          part = (y == x) ? 0 : y + 1;
        }
        if (lane >= pp) part = lane;
        const bool lo = lane < part;
        double xb[NB];
#pragma unroll
        for (int i = 0; i < NB; ++i) xb[i] = __shfl_sync(0xffffffffu, c[i], part);
        double o0 = 0.0, o1 = 0.0, p0 = 0.0, p1 = 0.0, g0 = 0.0, g1 = 0.0;
#pragma unroll
        for (int i = 0; i < NB; i += 2) {
          o0 = fma(c[i], c[i], o0);
          p0 = fma(xb[i], xb[i], p0);
          g0 = fma(c[i], xb[i], g0);
          if (i + 1 < NB) {
            o1 = fma(c[i + 1], c[i + 1], o1);
            p1 = fma(xb[i + 1], xb[i + 1], p1);
            g1 = fma(c[i + 1], xb[i + 1], g1);
          }
        }
        const double own = o0 + o1, oth = p0 + p1, ga = g0 + g1;
        const double al = lo ? own : oth, be = lo ? oth : own;
        const bool doit = lane < K && part < K && ga != 0.0 && ga * ga > tol2 * al * be;
        if (__any_sync(0xffffffffu, doit)) {
          double cs, sn;
          jacobi_rot(opaque(doit ? al : 1.0), opaque(doit ? be : 2.0), opaque(doit ? ga : 1.0), &cs, &sn);
          if (!doit) {
            cs = 1.0;
            sn = 0.0;
          }
          const double ss = lo ? -sn : sn;
          if (ACC) {
            double vb[NB];
#pragma unroll
            for (int i = 0; i < NB; ++i) vb[i] = __shfl_sync(0xffffffffu, v[ACC ? i : 0], part);
#pragma unroll
            for (int i = 0; i < NB; ++i) v[ACC ? i : 0] = fma(cs, v[ACC ? i : 0], ss * vb[i]);
          }
#pragma unroll
          for (int i = 0; i < NB; ++i) c[i] = fma(cs, c[i], ss * xb[i]);
          rot = 1;
        }
      }
      if (!__any_sync(0xffffffffu, rot)) break;
    }
    if (lane < K) {
      double s2 = 0.0;
#pragma unroll
      for (int i = 0; i < NB; ++i) s2 = fma(c[i], c[i], s2);
      sig[lane] = sqrt(s2);
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        if (ACC) {
          if (i < K) out[i + lane * ldo] = v[ACC ? i : 0];
        } else if (i < n) {
          out[i + lane * ldo] = c[i];
        }
      }
    }
    if (lane == 0) scratch[0] = nsw;
  }
  __syncthreads();
  for (int j = tid; j < K; j += blockDim.x) {
    int pos = 0;
    const double sj = sig[j];
    for (int i = 0; i < K; ++i) pos += (sig[i] > sj) || (sig[i] == sj && i < j);
    order[pos] = j;
  }
  const int nsw = scratch[0];
  __syncthreads();
  return nsw;
}

// Rank rule of the truncation: r = #{sigma_q > max(rel sigma_1, abs)}, <= max_rank, <= cap.
__device__ __forceinline__ int trunc_rank(const double* sig, const int* order, int p, double rel, double abs_tol,
                                          int max_rank, int cap, int* clamped) {
  if (p == 0) return 0;
  const double s1 = sig[order[0]];
  if (!(s1 > 0.0)) return 0;
  const double thr = fmax(rel * s1, abs_tol);
  int r = 0;
  for (int q = 0; q < p; ++q) r += sig[order[q]] > thr;
  if (max_rank > 0 && r > max_rank) r = max_rank;
  if (r > cap) {
    r = cap;
    *clamped = 1;
  }
  return r;
}

}  // namespace la
}  // namespace h2
