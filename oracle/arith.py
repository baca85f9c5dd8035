"""ORACLE (test infrastructure only) — H^2 product, substitutions, LR/Cholesky, solves, PCG.

PAPER §3 and §6 in the paper's order and notation:
  addmul   Z|_{t x r} += alpha X|_{t x s} Y|_{s x r}
           Case 1: (t,s), (s,r) subdivided -> recurse over sons+ (s' outermost, then t', r';
                   printed order P:490-497, reading R9); if (t,r) is an admissible leaf the
                   results go to temporaries (low-rank, SVD-truncated addition P:513-517,
                   reading R10) merged by 4 zero-extended local updates
           Case 2: (t,s) or (s,r) a leaf -> low-rank factors (reading R23) ->
                   local update or dense add into an inadmissible target
  chol     chol(t1); rfs(t2,t1); addmul(-1, L21, L21^T) [lower]; chol(t2)
  lr       lr(t1); lfs(t1,t2); rfs(t2,t1); addmul(-1, L21, R12); lr(t2)
  lfs/rfs  block forward substitution L X = Y / X R = Y
           admissible-leaf case (not described in the paper, reading R8): S_b <- 0 and a local
           update with (V_t S_b, L^{-1} W_s) (resp. (L^{-1} V_t S_b, W_s))
  solve    vector forward/backward substitution with the factors (preconditioner of P:1440-1444)
  inv      approximate inverse by block Gauss elimination, six products per level
  pcg      preconditioned CG [HEST52] to ||r||/||b|| < 1e-8 (reading R12)
  power    power iteration for ||I - A~^{-1} A|| (reading R11)

Storage conventions: Cholesky works in place on an H2(lower=True) matrix (block-lower
triangle + full dense diagonal tiles; after chol the diagonal tiles hold L with zero upper part).
LR works in place on a full-storage matrix (strict lower part = unit-lower L, upper part = R).
"""
import numpy as np
from scipy.linalg import solve_triangular, block_diag

from .structure import SUBDIV, ADM, INADM
from .update import Updater, Trunc, qr_R


class BreakdownError(RuntimeError):
    pass


# ---------------------------------------------------------------------------------------------
# operand views
# ---------------------------------------------------------------------------------------------
class Op:
    """op(Z) = Z or Z^T as an operand of the product; blocks addressed by (row cluster, col cluster)
    of op(Z).  Non-stored blocks (lower storage) are zero."""

    def __init__(self, Z, trans=False):
        self.Z, self.trans = Z, trans
        self.bt = Z.bt

    def bid(self, a, b):
        return self.bt.index[(b, a) if self.trans else (a, b)]

    def kind(self, a, b):
        return int(self.bt.kind[self.bid(a, b)])

    def stored(self, a, b):
        b_ = self.bid(a, b)
        return (b_ in self.Z.S) or (b_ in self.Z.N) or self.bt.kind[b_] == SUBDIV

    def row_basis(self, a):
        Z = self.Z
        return Z.full_col_basis(a) if self.trans else Z.full_row_basis(a)

    def col_basis(self, b):
        Z = self.Z
        return Z.full_row_basis(b) if self.trans else Z.full_col_basis(b)

    def coupling(self, a, b):
        b_ = self.bid(a, b)
        if b_ not in self.Z.S:
            return None
        S = self.Z.S[b_]
        return S.T if self.trans else S

    def dense(self, a, b):
        b_ = self.bid(a, b)
        if b_ not in self.Z.N:
            return None
        N = self.Z.N[b_]
        return N.T if self.trans else N

    def mul_dense(self, a, b, D):
        """op(Z)|_{a x b} @ D by recursion over the block tree (H^2 block times dense, [BO10 Thm 3.42])."""
        rt = self.Z.rt
        out = np.zeros((rt.size(a), D.shape[1]))
        k = self.kind(a, b)
        if k == ADM:
            S = self.coupling(a, b)
            if S is not None and S.size:
                out += self.row_basis(a) @ (S @ (self.col_basis(b).T @ D))
        elif k == INADM:
            N = self.dense(a, b)
            if N is not None:
                out += N @ D
        else:
            for a2 in rt.sons_plus(a):
                for b2 in rt.sons_plus(b):
                    if not self.stored(a2, b2):
                        continue
                    lo_a, lo_b = rt.lo[a2] - rt.lo[a], rt.lo[b2] - rt.lo[b]
                    out[lo_a:lo_a + rt.size(a2)] += self.mul_dense(a2, b2, D[lo_b:lo_b + rt.size(b2)])
        return out

    def t(self):
        return Op(self.Z, not self.trans)


# ---------------------------------------------------------------------------------------------
# low-rank temporaries (R10)
# ---------------------------------------------------------------------------------------------
class RkTemp:
    """Low-rank accumulator A B^T over rows(cluster ra) x cols(cluster rb), SVD-truncated addition
     with the rank rule R5 of the matrix's truncation control."""

    def __init__(self, tree, ra, rb, trunc):
        self.tree, self.ra, self.rb, self.trunc = tree, ra, rb, trunc
        self.A = np.zeros((tree.size(ra), 0))
        self.B = np.zeros((tree.size(rb), 0))

    def add(self, a, b, A, B):
        tr = self.tree
        Ae = np.zeros((tr.size(self.ra), A.shape[1]))
        Be = np.zeros((tr.size(self.rb), B.shape[1]))
        oa, ob = tr.lo[a] - tr.lo[self.ra], tr.lo[b] - tr.lo[self.rb]
        Ae[oa:oa + A.shape[0]] = A
        Be[ob:ob + B.shape[0]] = B
        A2 = np.hstack([self.A, Ae])
        B2 = np.hstack([self.B, Be])
        if A2.shape[1] == 0:
            return
        Qa, Ra = np.linalg.qr(A2)
        Qb, Rb = np.linalg.qr(B2)
        U, sig, Vt = np.linalg.svd(Ra @ Rb.T)
        r = self.trunc.rank(sig)
        self.A = Qa @ (U[:, :r] * sig[:r])
        self.B = Qb @ Vt[:r].T


# ---------------------------------------------------------------------------------------------
# the arithmetic driver
# ---------------------------------------------------------------------------------------------
class Arith:
    def __init__(self, Z, trunc: Trunc, lr_unit_lower=False):
        self.Z = Z
        self.trunc = trunc
        self.up = Updater(Z, trunc)
        self.rt = Z.rt
        self.unit_lower = lr_unit_lower  # LR: the diagonal tiles hold unit-lower L and upper R
        self.stats = dict(updates=0, dense_adds=0, temporaries=0, tmp_adds=0)

    # ---- contributions -------------------------------------------------------------------
    def _add(self, target, t, r, A, B):
        """Add A B^T at rows t, cols r of the target (an H^2 block of Z or a temporary)."""
        if A.shape[1] == 0:
            return
        if isinstance(target, RkTemp):
            target.add(t, r, A, B)
            self.stats["tmp_adds"] += 1
            return
        Z, bt = self.Z, self.Z.bt
        b = bt.index[(t, r)]
        if bt.kind[b] == INADM:
            if b in Z.N:
                Z.N[b] += A @ B.T
                self.stats["dense_adds"] += 1
            return
        self.up(t, r, A, B)
        self.stats["updates"] += 1

    def _factors(self, X: Op, Y: Op, t, s, r, dense_target=False):
        """Low-rank factors A, B with X|_{t x s} Y|_{s x r} = A B^T (Case 2; R23)."""
        kx, ky = X.kind(t, s), Y.kind(s, r)
        # reading own-6: a contribution one of whose factors is an exactly zero dense tile adds
        # nothing and is skipped -- in every branch, also when the other factor is admissible (the
        # tiles of the factor that never receive fill stay exactly zero; P:505-509 leaves the
        # construction of the Case-2 factors open)
        if (kx == INADM and X.dense(t, s) is not None and not X.dense(t, s).any()) or \
           (ky == INADM and Y.dense(s, r) is not None and not Y.dense(s, r).any()):
            return np.zeros((self.rt.size(t), 0)), np.zeros((self.rt.size(r), 0))
        if kx == ADM and ky == ADM:
            Sx, Sy = X.coupling(t, s), Y.coupling(s, r)
            Vx, Wy = X.row_basis(t), Y.col_basis(r)
            if Sx is None or Sy is None:
                return np.zeros((Vx.shape[0], 0)), np.zeros((Wy.shape[0], 0))
            Cm = Sx @ (X.col_basis(s).T @ Y.row_basis(s)) @ Sy
            if Cm.shape[0] <= Cm.shape[1]:
                return Vx, Wy @ Cm.T
            return Vx @ Cm, Wy
        if kx == ADM:
            Sx = X.coupling(t, s)
            Vx = X.row_basis(t)
            if Sx is None:
                return np.zeros((Vx.shape[0], 0)), np.zeros((self.rt.size(r), 0))
            B = Y.t().mul_dense(r, s, X.col_basis(s) @ Sx.T)
            return Vx, B
        if ky == ADM:
            Sy = Y.coupling(s, r)
            Wy = Y.col_basis(r)
            if Sy is None:
                return np.zeros((self.rt.size(t), 0)), np.zeros((Wy.shape[0], 0))
            A = X.mul_dense(t, s, Y.row_basis(s) @ Sy)
            return A, Wy
        if kx == INADM and ky == INADM and not dense_target:
            # reading own-7: both factors dense leaf blocks, low-rank target (P:505-509 leaves the factorization
            # open): interpolative decomposition of P = X_ts Y_sr by column-pivoted QR,
            # P Pi = Q R, r = #{|R_kk| > 1e-12 |R_00|}, A = P[:, J] (the r pivot columns),
            # B^T = [I, R_11^{-1} R_12] Pi^T, so that A B^T = P up to |R_rr| <= 1e-12 |R_00|.
            Nx, Ny = X.dense(t, s), Y.dense(s, r)
            if Nx is None or Ny is None:
                return np.zeros((self.rt.size(t), 0)), np.zeros((self.rt.size(r), 0))
            return self._interp_decomp(Nx @ Ny)
        if kx == INADM:
            Nx = X.dense(t, s)
            if Nx is None:
                return np.zeros((self.rt.size(t), 0)), np.zeros((self.rt.size(r), 0))
            B = Y.t().mul_dense(r, s, np.eye(self.rt.size(s)))
            return Nx, B
        # ky == INADM
        Ny = Y.dense(s, r)
        if Ny is None:
            return np.zeros((self.rt.size(t), 0)), np.zeros((self.rt.size(r), 0))
        A = X.mul_dense(t, s, Ny)
        return A, np.eye(self.rt.size(r))

    @staticmethod
    def _interp_decomp(P, rel=1e-12):
        """Interpolative decomposition P ~ A B^T with A = r columns of P (LAPACK dgeqp3 pivots)."""
        from scipy.linalg import qr
        mt, mr = P.shape
        _, R, piv = qr(P, mode="economic", pivoting=True)
        d = np.abs(np.diag(R))
        if d.size == 0 or d[0] == 0.0:
            return np.zeros((mt, 0)), np.zeros((mr, 0))
        small = np.nonzero(d <= rel * d[0])[0]
        r = int(small[0]) if small.size else d.size  # the pivoted QR stops at the first small |R_kk|
        A = P[:, piv[:r]]
        T = solve_triangular(R[:r, :r], R[:r, r:])
        B = np.zeros((mr, r))
        B[piv[:r], :] = np.eye(r)
        B[piv[r:], :] = T.T
        return A, B

    def _target_stored(self, t, r):
        b = self.Z.bt.index.get((t, r))
        if b is None:
            return False
        return (not self.Z.lower) or self.rt.lo[t] >= self.rt.lo[r]

    # ---- product ---------------------------------------------------------------------------
    def addmul(self, alpha, X: Op, Y: Op, t, s, r, target=None):
        """Z|_{t x r} += alpha X|_{t x s} Y|_{s x r}; target None = the H^2 matrix Z itself."""
        rt = self.rt
        if alpha == 0.0 or not (X.stored(t, s) and Y.stored(s, r)):
            return
        kx, ky = X.kind(t, s), Y.kind(s, r)
        if kx == SUBDIV and ky == SUBDIV:
            if target is None:
                kz = int(self.Z.bt.kind[self.Z.bt.index[(t, r)]])
                if kz == ADM:
                    ttr = self.trunc.relative() if self.trunc.blockwise else self.trunc  # one block: relative
                    temps = {(t2, r2): RkTemp(rt, t2, r2, ttr)
                             for t2 in rt.sons_plus(t) for r2 in rt.sons_plus(r)}
                    self.stats["temporaries"] += len(temps)
                    for s2 in rt.sons_plus(s):
                        for t2 in rt.sons_plus(t):
                            for r2 in rt.sons_plus(r):
                                self.addmul(alpha, X, Y, t2, s2, r2, temps[(t2, r2)])
                    # merge: 4 zero-extended local updates into (t, r), order (1,1),(1,2),(2,1),(2,2)
                    for t2 in rt.sons_plus(t):
                        for r2 in rt.sons_plus(r):
                            T = temps[(t2, r2)]
                            if T.A.shape[1] == 0:
                                continue
                            A = np.zeros((rt.size(t), T.A.shape[1]))
                            B = np.zeros((rt.size(r), T.B.shape[1]))
                            A[rt.lo[t2] - rt.lo[t]:rt.hi[t2] - rt.lo[t]] = T.A
                            B[rt.lo[r2] - rt.lo[r]:rt.hi[r2] - rt.lo[r]] = T.B
                            self._add(None, t, r, A, B)
                    return
                for s2 in rt.sons_plus(s):
                    for t2 in rt.sons_plus(t):
                        for r2 in rt.sons_plus(r):
                            if self._target_stored(t2, r2):
                                self.addmul(alpha, X, Y, t2, s2, r2, None)
                return
            for s2 in rt.sons_plus(s):
                for t2 in rt.sons_plus(t):
                    for r2 in rt.sons_plus(r):
                        self.addmul(alpha, X, Y, t2, s2, r2, target)
            return
        dense_target = target is None and self.Z.bt.kind[self.Z.bt.index[(t, r)]] == INADM
        A, B = self._factors(X, Y, t, s, r, dense_target)
        if A.shape[1]:
            self._add(target, t, r, alpha * A, B)

    # ---- substitutions ------------------------------------------------------------------
    def _diag_tile(self, t):
        return self.Z.N[self.Z.bt.index[(t, t)]]

    def lsolve(self, t, B, unit=False):
        """Solve L|_{t x t} X = B (dense B), L = lower part of Z (vector/dense case)."""
        rt = self.rt
        if rt.is_leaf(t):
            return solve_triangular(self._diag_tile(t), B, lower=True, unit_diagonal=unit)
        t1, t2 = rt.sons(t)
        n1 = rt.size(t1)
        X1 = self.lsolve(t1, B[:n1], unit)
        B2 = B[n1:] - Op(self.Z).mul_dense(t2, t1, X1)
        X2 = self.lsolve(t2, B2, unit)
        return np.vstack([X1, X2])

    def ltsolve(self, t, B):
        """Solve L|_{t x t}^T X = B (Cholesky backward substitution)."""
        rt = self.rt
        if rt.is_leaf(t):
            return solve_triangular(self._diag_tile(t).T, B, lower=False)
        t1, t2 = rt.sons(t)
        n1 = rt.size(t1)
        X2 = self.ltsolve(t2, B[n1:])
        B1 = B[:n1] - Op(self.Z, True).mul_dense(t1, t2, X2)
        X1 = self.ltsolve(t1, B1)
        return np.vstack([X1, X2])

    def usolve(self, t, B):
        """Solve R|_{t x t} X = B, R = upper part of Z (LR)."""
        rt = self.rt
        if rt.is_leaf(t):
            return solve_triangular(self._diag_tile(t), B, lower=False)
        t1, t2 = rt.sons(t)
        n1 = rt.size(t1)
        X2 = self.usolve(t2, B[n1:])
        B1 = B[:n1] - Op(self.Z).mul_dense(t1, t2, X2)
        X1 = self.usolve(t1, B1)
        return np.vstack([X1, X2])

    def utsolve(self, t, B):
        """Solve R|_{t x t}^T X = B (forward substitution with R^T, used by rfs in LR)."""
        rt = self.rt
        if rt.is_leaf(t):
            return solve_triangular(self._diag_tile(t).T, B, lower=True)
        t1, t2 = rt.sons(t)
        n1 = rt.size(t1)
        X1 = self.utsolve(t1, B[:n1])
        B2 = B[n1:] - Op(self.Z, True).mul_dense(t2, t1, X1)
        X2 = self.utsolve(t2, B2)
        return np.vstack([X1, X2])

    def rfs_chol(self, t, s):
        """X L_ss^T = Y at block (t, s), in place (P:423-450 with R = L^T; R8 admissible case)."""
        Z, rt, bt = self.Z, self.rt, self.Z.bt
        b = bt.index[(t, s)]
        k = bt.kind[b]
        if k == INADM:
            L = self._diag_tile(s)
            Z.N[b] = solve_triangular(L, Z.N[b].T, lower=True).T
        elif k == ADM:
            S = Z.S[b]
            if S.size == 0:
                return
            Zs = self.lsolve(s, Z.full_col_basis(s))
            U = Z.full_row_basis(t) @ S
            Z.S[b] = np.zeros_like(S)
            self._add(None, t, s, U, Zs)
        else:
            if rt.is_leaf(s):
                for t2 in rt.sons_plus(t):
                    self.rfs_chol(t2, s)
                return
            s1, s2 = rt.sons(s)
            for t2 in rt.sons_plus(t):
                self.rfs_chol(t2, s1)
                self.addmul(-1.0, Op(Z), Op(Z, True), t2, s1, s2)
                self.rfs_chol(t2, s2)

    def chol(self, t=0):
        """In-place H^2 Cholesky of the lower-stored Z|_{t x t}."""
        Z, rt = self.Z, self.rt
        if rt.is_leaf(t):
            b = Z.bt.index[(t, t)]
            N = Z.N[b]
            try:
                L = np.linalg.cholesky(np.tril(N) + np.tril(N, -1).T)
            except np.linalg.LinAlgError as e:
                raise BreakdownError(f"H2_ERR_BREAKDOWN: leaf {t} not positive definite") from e
            Z.N[b] = L
            return
        t1, t2 = rt.sons(t)
        self.chol(t1)
        self.rfs_chol(t2, t1)
        self.addmul(-1.0, Op(Z), Op(Z, True), t2, t1, t2)
        self.chol(t2)

    def lfs(self, t, s):
        """L_tt X = Y at block (t, s), unit-lower L (R8 admissible case)."""
        Z, rt, bt = self.Z, self.rt, self.Z.bt
        b = bt.index[(t, s)]
        k = bt.kind[b]
        if k == INADM:
            Z.N[b] = solve_triangular(self._diag_tile(t), Z.N[b], lower=True, unit_diagonal=True)
        elif k == ADM:
            S = Z.S[b]
            if S.size == 0:
                return
            U = self.lsolve(t, Z.full_row_basis(t), unit=True) @ S
            Ws = Z.full_col_basis(s)
            Z.S[b] = np.zeros_like(S)
            self._add(None, t, s, U, Ws)
        else:
            if rt.is_leaf(t):
                for s2 in rt.sons_plus(s):
                    self.lfs(t, s2)
                return
            t1, t2 = rt.sons(t)
            for s2 in rt.sons_plus(s):
                self.lfs(t1, s2)
                self.addmul(-1.0, Op(Z), Op(Z), t2, t1, s2)
                self.lfs(t2, s2)

    def rfs_lr(self, t, s):
        """X R_ss = Y at block (t, s) (R8 admissible case)."""
        Z, rt, bt = self.Z, self.rt, self.Z.bt
        b = bt.index[(t, s)]
        k = bt.kind[b]
        if k == INADM:
            R = self._diag_tile(s)
            Z.N[b] = solve_triangular(np.triu(R), Z.N[b].T, trans="T", lower=False).T
        elif k == ADM:
            S = Z.S[b]
            if S.size == 0:
                return
            Zs = self.utsolve(s, Z.full_col_basis(s))
            U = Z.full_row_basis(t) @ S
            Z.S[b] = np.zeros_like(S)
            self._add(None, t, s, U, Zs)
        else:
            if rt.is_leaf(s):
                for t2 in rt.sons_plus(t):
                    self.rfs_lr(t2, s)
                return
            s1, s2 = rt.sons(s)
            for t2 in rt.sons_plus(t):
                self.rfs_lr(t2, s1)
                self.addmul(-1.0, Op(Z), Op(Z), t2, s1, s2)
                self.rfs_lr(t2, s2)

    def lr(self, t=0):
        """In-place H^2 LR factorization (Doolittle, unit-lower L, no pivoting)."""
        Z, rt = self.Z, self.rt
        if rt.is_leaf(t):
            b = Z.bt.index[(t, t)]
            N = Z.N[b].copy()
            m = N.shape[0]
            nrm = np.linalg.norm(N)  # Frobenius (reading: breakdown threshold |p| <= 1e-14 ||tile||_F)
            for j in range(m):
                if abs(N[j, j]) <= 1e-14 * nrm:
                    raise BreakdownError(f"H2_ERR_BREAKDOWN: leaf {t} pivot {j}")
                N[j + 1:, j] /= N[j, j]
                N[j + 1:, j + 1:] -= np.outer(N[j + 1:, j], N[j, j + 1:])
            Z.N[b] = N
            return
        t1, t2 = rt.sons(t)
        self.lr(t1)
        self.lfs(t1, t2)
        self.rfs_lr(t2, t1)
        self.addmul(-1.0, Op(Z), Op(Z), t2, t1, t2)
        self.lr(t2)

    # ---- approximate inverse (Remark 1) -------------------------
    def zero_block(self, t, s):
        """Z|_{t x s} <- 0: every coupling and nearfield tile of the block subtree (bases untouched)."""
        Z = self.Z
        for b in Z.bt.subtree(Z.bt.index[(t, s)]):
            if b in Z.S:
                Z.S[b] = np.zeros_like(Z.S[b])
            if b in Z.N:
                Z.N[b] = np.zeros_like(Z.N[b])

    def inv(self, T, t=0, _aT=None):
        """In place Z|_{t x t} <- (Z|_{t x t})^{-1} by block Gauss elimination (Remark 1):
        C11 = A11^{-1};  B12 = C11 A12,  B21 = A21 C11  (into the scratch H^2 matrix T, same trees,
        zero on entry);  S = A22 - A21 B12  (P:1382 prints "A_11 -", reading R20: A_22);
        C22 = S^{-1};  C12 = -B12 C22;  C21 = -C22 B21;  C11 = C11 - C12 B21  -- six products, all
        Z|_{t x r} += alpha X|_{t x s} Y|_{s x r} (addmul) in this order; a leaf tile is inverted
        directly.  Full storage only."""
        Z, rt = self.Z, self.rt
        if rt.is_leaf(t):
            b = Z.bt.index[(t, t)]
            N = Z.N[b]
            nrm = np.linalg.norm(N)
            # breakdown rule of the leaf LR (reading own-2): no-pivot elimination pivots
            M = N.copy()
            for j in range(M.shape[0]):
                if abs(M[j, j]) <= 1e-14 * nrm:
                    raise BreakdownError(f"H2_ERR_BREAKDOWN: leaf {t} pivot {j}")
                M[j + 1:, j] /= M[j, j]
                M[j + 1:, j + 1:] -= np.outer(M[j + 1:, j], M[j, j + 1:])
            Z.N[b] = np.linalg.inv(N)
            return
        aT = _aT if _aT is not None else Arith(T, self.trunc)
        t1, t2 = rt.sons(t)
        self.inv(T, t1, aT)
        aT.addmul(1.0, Op(Z), Op(Z), t1, t1, t2)   # B12 = C11 A12   -> T|_{t1 x t2}
        aT.addmul(1.0, Op(Z), Op(Z), t2, t1, t1)   # B21 = A21 C11   -> T|_{t2 x t1}
        self.addmul(-1.0, Op(Z), Op(T), t2, t1, t2)  # S = A22 - A21 B12
        self.inv(T, t2, aT)                          # C22 = S^{-1}
        self.zero_block(t1, t2)
        self.addmul(-1.0, Op(T), Op(Z), t1, t2, t2)  # C12 = -B12 C22
        self.zero_block(t2, t1)
        self.addmul(-1.0, Op(Z), Op(T), t2, t2, t1)  # C21 = -C22 B21
        self.addmul(-1.0, Op(Z), Op(T), t1, t2, t1)  # C11 = C11 - C12 B21

    # ---- preconditioner application -------------------------------------------------------
    def solve_tree(self, b, cholesky=True):
        """x = (LL^T)^{-1} b or (LR)^{-1} b, vectors in TREE order."""
        B = b[:, None] if b.ndim == 1 else b
        if cholesky:
            X = self.ltsolve(0, self.lsolve(0, B))
        else:
            X = self.usolve(0, self.lsolve(0, B, unit=True))
        return X[:, 0] if b.ndim == 1 else X

    def solve(self, b, cholesky=True):
        """Same, vectors in ORIGINAL order."""
        rt = self.rt
        x = np.empty_like(b)
        x[rt.perm] = self.solve_tree(b[rt.perm], cholesky)
        return x


def dense_factor_product(Z, cholesky=True):
    """L L^T (Cholesky, lower storage) or L R (LR, full storage) of a factored Z, dense, tree order."""
    from .dense import densify
    D = densify(Z)
    if cholesky:
        L = np.tril(D)
        return L @ L.T
    L = np.tril(D, -1) + np.eye(D.shape[0])
    R = np.triu(D)
    return L @ R


def pcg(apply_A, apply_M, b, tol=1e-8, maxit=500):
    """Preconditioned CG [HEST52], x0 = 0, stop at ||r||/||b|| < tol (reading R12).
    Returns (x, m = number of A-applications, final relative residual)."""
    x = np.zeros_like(b)
    r = b.copy()
    nb = np.linalg.norm(b)
    if nb == 0:
        return x, 0, 0.0
    z = apply_M(r)
    p = z.copy()
    rz = r @ z
    m = 0
    while m < maxit:
        Ap = apply_A(p)
        m += 1
        a = rz / (p @ Ap)
        x += a * p
        r -= a * Ap
        rel = np.linalg.norm(r) / nb
        if rel < tol:
            return x, m, rel
        z = apply_M(r)
        rz_new = r @ z
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x, m, np.linalg.norm(r) / nb


def power_error(apply_A, apply_M, x0, iters=50, rtol=1e-4):
    """Power iteration on E = I - M^{-1} A (reading R11): returns the estimate of ||E||."""
    x = x0 / np.linalg.norm(x0)
    lam_old = None
    lam = 0.0
    for _ in range(iters):
        y = x - apply_M(apply_A(x))
        lam = np.linalg.norm(y)
        if lam == 0.0:
            return 0.0
        x = y / lam
        if lam_old is not None and abs(lam - lam_old) <= rtol * lam:
            break
        lam_old = lam
    return lam
