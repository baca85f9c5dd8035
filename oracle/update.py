"""ORACLE (test infrastructure only) — local low-rank update Z|_{t0 x s0} += X Y^T (O1).

Follows PAPER §4-§5 in the paper's order and notation:
  U0  nearfield leaves inside T_{b0} receive X|t Y|s^T exactly
  U1  extension  V~_t = [V_t, X|t], E~_t = diag(E_t, I), E~_{t0} = [E_{t0}; 0],
      S~_b = diag(S_b, I) / [S_b; 0] / [S_b, 0]                             (eq. 4a-c)
  U2  thin-QR R-factors of the extended bases by the nested recursion        ([BO10 Alg. 16])
  U3  weights B~_t: R-factor of [R_{W,s} S~_{t,s}^T (s in row(t)); B~_{t+} E~_t^T],
      top-down over pred(t0) then T_{t0}; blocks outside T_{b0} included
  U4  truncated nested basis: leaf SVD of V~_t B~_t^T, internal SVD of
      V^_t B~_t^T with V^_t = [R_{t1} E~_{t1}; R_{t2} E~_{t2}];
      R_t = Q_t^T V~_t = Q^_t^T V^_t                                         ([BO10 Alg. 30])
  U5  couplings S_b <- R_t S~_b R_s^T (three cases)
  U6  V_t <- Q_t on T_{t0}, E_{t0} <- R_{t0}[E_{t0}; 0]
The column side is the same construction applied to Z~^T.

Readings: R5 truncation rule, R7 actual R-factors of partner bases
(never assumed I), R21 weights over the full block row (stored blocks only),
b0 an inadmissible leaf => dense add only.
"""
from dataclasses import dataclass

import numpy as np
from scipy.linalg import block_diag

from .structure import INADM
from .h2 import H2


@dataclass
class Trunc:
    """TruncationControl.  rank r = #{sigma_i > max(rel_tol*sigma_1, abs_tol)},
    capped by max_rank (<= 0: unbounded).  SURVEY R5.

    blockwise=True (DESIGN reading own-10): "block-relative accuracy eps^"
    (P:874-879): the weight matrices carry the factor 1/||G~_b||_F for every block b
    (weighting factors in B_{t,s}), so their singular values are measured in units of
    the blocks' own norms, and the rank is r = #{sigma_i > max(rel_tol, abs_tol)} -- an ABSOLUTE
    threshold eps^ = rel_tol on the weighted matrix.  Low-rank temporaries (one block each) keep
    the relative rule (relative())."""
    rel_tol: float = 1e-4
    abs_tol: float = 0.0
    max_rank: int = 0
    blockwise: bool = False

    def rank(self, sig: np.ndarray) -> int:
        if sig.size == 0 or sig[0] <= 0.0:
            return 0
        if self.blockwise:
            thr = max(self.rel_tol, self.abs_tol)
        else:
            thr = max(self.rel_tol * sig[0], self.abs_tol)
        r = int(np.count_nonzero(sig > thr))
        if self.max_rank > 0:
            r = min(r, self.max_rank)
        return r

    def relative(self) -> "Trunc":
        """The plain relative rule with the same tolerance (temporaries of the product)."""
        return Trunc(self.rel_tol, self.abs_tol, self.max_rank)


FIXED16 = Trunc(rel_tol=1e-12, abs_tol=0.0, max_rank=16)  # SURVEY R5/R16 fixed-rank mode


def qr_R(A: np.ndarray, ncols: int) -> np.ndarray:
    """R-factor of a thin QR factorization (library primitive), shape min(m,n) x n."""
    if A.shape[0] == 0:
        return np.zeros((0, ncols))
    return np.linalg.qr(A, mode="r")


def svd_left(M: np.ndarray):
    """Left singular vectors and singular values (library primitive)."""
    if M.size == 0:
        return np.zeros((M.shape[0], 0)), np.zeros(0)
    U, sig, _ = np.linalg.svd(M, full_matrices=False)
    return U, sig


class RCache:
    """R-factors R_{V,t} of the CURRENT nested basis, computed by the recursion of
    [BO10 Alg. 16]: leaf qr(V_t), internal qr([R_{t1}E_{t1}; R_{t2}E_{t2}]).
    Memoised; entries on changed subtrees and ancestor paths are dropped."""

    def __init__(self, tree, leaf, transfer):
        self.tree, self.leaf, self.transfer = tree, leaf, transfer
        self.c = {}

    def get(self, t):
        r = self.c.get(t)
        if r is None:
            tr = self.tree
            if tr.is_leaf(t):
                r = qr_R(self.leaf[t], self.leaf[t].shape[1])
            else:
                t1, t2 = tr.sons(t)
                A = np.vstack([self.get(t1) @ self.transfer[t1], self.get(t2) @ self.transfer[t2]])
                r = qr_R(A, self.transfer[t1].shape[1])
            self.c[t] = r
        return r

    def invalidate(self, root):
        tr = self.tree
        for t in tr.subtree(root):
            self.c.pop(t, None)
        for t in tr.pred(root):
            self.c.pop(t, None)


class _Side:
    """One side (row basis V/E of Z, or column basis W/F viewed through Z^T)."""

    def __init__(self, Z: H2, row: bool, root: int, Xf: np.ndarray):
        self.Z = Z
        self.row = row
        self.tree = Z.rt if row else Z.ct
        self.leaf = Z.V if row else Z.W
        self.tr = Z.E if row else Z.F
        self.rank = Z.k if row else Z.l
        self.blocks = Z.bt.row if row else Z.bt.col
        self.root = root
        self.Xf = Xf
        self.k = Xf.shape[1]
        self.sub = self.tree.subtree(root)

    def inside(self, t):
        return self.tree.in_subtree(t, self.root)

    def K(self, t):
        return int(self.rank[t]) + (self.k if self.inside(t) else 0)

    def partner(self, b):
        bt = self.Z.bt
        return int(bt.s[b]) if self.row else int(bt.t[b])

    def coupling(self, b):
        """S_b oriented (this-side rank) x (partner rank)."""
        S = self.Z.S[b]
        return S if self.row else S.T

    def Vext(self, t):
        tr = self.tree
        lo = tr.lo[t] - tr.lo[self.root]
        return np.hstack([self.leaf[t], self.Xf[lo:lo + tr.size(t)]])

    def Eext(self, t):
        """Transfer matrix of t in the extended basis (eq. 4 and E~_{t0} = [E_{t0}; 0])."""
        E = self.tr[t]
        if t == self.root:
            return np.vstack([E, np.zeros((self.k, E.shape[1]))])
        if self.inside(t):
            return block_diag(E, np.eye(self.k))
        return E


def _ext_rfactors(side: _Side):
    """U2: R-factors of V~_t for t in T_{t0}, bottom-up."""
    R = {}
    tr = side.tree
    for t in reversed(side.sub):
        if tr.is_leaf(t):
            R[t] = qr_R(side.Vext(t), side.K(t))
        else:
            t1, t2 = tr.sons(t)
            R[t] = qr_R(np.vstack([R[t1] @ side.Eext(t1), R[t2] @ side.Eext(t2)]), side.K(t))
    return R


def _weights(side: _Side, other: _Side, R_other_ext, other_cache: RCache, blockwise: bool = False,
             R_own_ext=None, own_cache: RCache = None):
    """U3: weight matrices B~_t for t in pred(t0) u T_{t0}.
    blockwise: every block's rows R_{W,s} S~_b^T carry the weight 1/||G~_b||_F, where
    ||G~_b||_F = ||R_{V,t} S~_b R_{W,s}^T||_F (R-factors of the current / extended bases, R7)."""
    tr = side.tree
    B = {}
    order = tr.pred(side.root)[:-1] + side.sub  # father before son
    Z = side.Z
    for t in order:
        rows = []
        for b in side.blocks[t]:
            if b not in Z.S:  # lower storage: only stored blocks (R21)
                continue
            s = side.partner(b)
            S = side.coupling(b)
            in_t, in_s = side.inside(t), other.inside(s)
            if in_t and in_s:
                St = block_diag(S, np.eye(side.k))
                RB = R_other_ext[s]
            elif in_t:
                St = np.vstack([S, np.zeros((side.k, S.shape[1]))])
                RB = other_cache.get(s)
            else:
                assert not in_s, "block of an ancestor inside the partner subtree cannot be a leaf"
                St = S
                RB = other_cache.get(s)
            blk = RB @ St.T
            if blockwise:
                RV = R_own_ext[t] if in_t else own_cache.get(t)
                nrm = np.linalg.norm(blk @ RV.T)
                if nrm == 0.0:
                    continue  # a zero block adds nothing to the weights
                blk = blk / nrm
            rows.append(blk)
        p = tr.parent[t]
        if p >= 0:
            rows.append(B[p] @ side.Eext(t).T)
        K = side.K(t)
        B[t] = qr_R(np.vstack(rows) if rows else np.zeros((0, K)), K)
    return B


def _truncated_basis(side: _Side, B, trunc: Trunc):
    """U4: Q_t, R_t = Q_t^T V~_t, ranks, bottom-up over T_{t0}."""
    tr = side.tree
    Q, R, r, sig_log = {}, {}, {}, {}
    for t in reversed(side.sub):
        if tr.is_leaf(t):
            Vt = side.Vext(t)
        else:
            t1, t2 = tr.sons(t)
            Vt = np.vstack([R[t1] @ side.Eext(t1), R[t2] @ side.Eext(t2)])  # V^_t
        M = Vt @ B[t].T
        U, sig = svd_left(M)
        rt = trunc.rank(sig)
        Q[t] = U[:, :rt]
        R[t] = Q[t].T @ Vt
        r[t] = rt
        sig_log[t] = sig
    return Q, R, r, sig_log


def local_update(Z: H2, t0: int, s0: int, X: np.ndarray, Y: np.ndarray, trunc: Trunc,
                 rcache_row: RCache, rcache_col: RCache, log: dict | None = None):
    """In-place Z|_{t0 x s0} += X Y^T.  X: |t0| x k, Y: |s0| x k, rows in TREE order
    restricted to the clusters' ranges (alpha already folded into X)."""
    bt = Z.bt
    b0 = bt.index.get((int(t0), int(s0)))
    if b0 is None:
        raise ValueError("H2_ERR_ARG: (t0,s0) is not a block of the block tree")
    rt, ct = Z.rt, Z.ct
    X = np.asarray(X, dtype=np.float64).reshape(rt.size(t0), -1)
    Y = np.asarray(Y, dtype=np.float64).reshape(ct.size(s0), -1)
    if X.shape[1] != Y.shape[1]:
        raise ValueError("H2_ERR_SHAPE")
    k = X.shape[1]
    # U0: exact nearfield part
    for b in bt.subtree(b0):
        if bt.kind[b] == INADM and b in Z.N:
            t, s = bt.t[b], bt.s[b]
            Z.N[b] += X[rt.lo[t] - rt.lo[t0]:rt.hi[t] - rt.lo[t0]] @ Y[ct.lo[s] - ct.lo[s0]:ct.hi[s] - ct.lo[s0]].T
    if k == 0 or bt.kind[b0] == INADM:
        return
    row = _Side(Z, True, int(t0), X)
    col = _Side(Z, False, int(s0), Y)
    # U1/U2
    RVe = _ext_rfactors(row)
    RWe = _ext_rfactors(col)
    # U3
    bw = trunc.blockwise
    Brow = _weights(row, col, RWe, rcache_col, bw, RVe, rcache_row)
    Bcol = _weights(col, row, RVe, rcache_row, bw, RWe, rcache_col)
    # U4
    Qr, Rr, rr, sr = _truncated_basis(row, Brow, trunc)
    Qc, Rc, rc, sc = _truncated_basis(col, Bcol, trunc)
    if log is not None:
        log.update(row_sig=sr, col_sig=sc, row_rank=rr, col_rank=rc)
    # U5: couplings of every stored admissible leaf touching T_{t0} or T_{s0}
    done = set()
    for t in row.sub:
        for b in bt.row[t]:
            if b not in Z.S:
                continue
            s = int(bt.s[b])
            S = Z.S[b]
            if col.inside(s):
                Z.S[b] = Rr[t] @ block_diag(S, np.eye(k)) @ Rc[s].T
            else:
                Z.S[b] = Rr[t][:, :int(Z.k[t])] @ S
            done.add(b)
    for s in col.sub:
        for b in bt.col[s]:
            if b not in Z.S or b in done:
                continue
            Z.S[b] = Z.S[b] @ Rc[s][:, :int(Z.l[s])].T
    # U6: install new bases and transfers
    for side, Q, R, r in ((row, Qr, Rr, rr), (col, Qc, Rc, rc)):
        tr = side.tree
        a0 = side.root
        if a0 != 0:
            side.tr[a0] = R[a0][:, :int(side.rank[a0])] @ side.tr[a0]
        for t in side.sub:
            if tr.is_leaf(t):
                side.leaf[t] = Q[t]
            else:
                t1, t2 = tr.sons(t)
                side.tr[t1] = Q[t][:r[t1]]
                side.tr[t2] = Q[t][r[t1]:]
        for t in side.sub:
            side.rank[t] = r[t]
    rcache_row.invalidate(int(t0))
    rcache_col.invalidate(int(s0))


class Updater:
    """Convenience wrapper keeping the R-factor caches of one matrix."""

    def __init__(self, Z: H2, trunc: Trunc):
        self.Z, self.trunc = Z, trunc
        self.crow = RCache(Z.rt, Z.V, Z.E)
        self.ccol = RCache(Z.ct, Z.W, Z.F)

    def __call__(self, t0, s0, X, Y, alpha=1.0, log=None):
        local_update(self.Z, t0, s0, alpha * np.asarray(X, dtype=np.float64), Y, self.trunc,
                     self.crow, self.ccol, log)
