"""ORACLE (test infrastructure only) — H^2-matrix representation.

PAPER Def. 3 (nested cluster basis, eq. (1)), Def. 4 (H^2 matrix, eq. (2)
P:285-287), representation by bases, couplings and nearfield.
Variable per-cluster ranks.  Row basis (V_t leaves, E_t transfers),
column basis (W_s leaves, F_s transfers), couplings S_b (k_t x l_s) on admissible
leaves, dense nearfield N_b on inadmissible leaves.  Everything is in TREE order;
``perm`` maps tree position -> original index.

Storage ``lower``: only blocks with t-range >= s-range are
kept (block-lower triangle including the full dense diagonal tiles); used by the
Cholesky factor.
"""
import numpy as np

from .structure import ClusterTree, BlockTree, ADM, INADM


class H2:
    def __init__(self, bt: BlockTree, lower: bool = False):
        self.bt, self.rt, self.ct = bt, bt.rt, bt.ct
        self.lower = lower
        rt, ct = self.rt, self.ct
        self.k = np.zeros(rt.nclusters, dtype=np.int64)  # row ranks
        self.l = np.zeros(ct.nclusters, dtype=np.int64)  # column ranks
        self.V = {t: np.zeros((rt.size(t), 0)) for t in rt.leaves()}
        self.W = {s: np.zeros((ct.size(s), 0)) for s in ct.leaves()}
        self.E = {t: np.zeros((0, 0)) for t in range(1, rt.nclusters)}
        self.F = {s: np.zeros((0, 0)) for s in range(1, ct.nclusters)}
        self.S = {b: np.zeros((0, 0)) for b in bt.adm if self.stored(b)}
        self.N = {b: np.zeros((rt.size(bt.t[b]), ct.size(bt.s[b]))) for b in bt.inadm if self.stored(b)}

    # -- storage predicate -------------------------------------------------
    def stored(self, b) -> bool:
        if not self.lower:
            return True
        t, s = self.bt.t[b], self.bt.s[b]
        return self.rt.lo[t] >= self.ct.lo[s]

    def copy(self):
        c = H2.__new__(H2)
        c.__dict__.update(self.__dict__)
        c.k, c.l = self.k.copy(), self.l.copy()
        for name in ("V", "W", "E", "F", "S", "N"):
            setattr(c, name, {key: val.copy() for key, val in getattr(self, name).items()})
        return c

    # -- full (expanded) bases, by the nesting eq. (1) ---------------------
    def full_row_basis(self, t):
        rt = self.rt
        if rt.is_leaf(t):
            return self.V[t]
        t1, t2 = rt.sons(t)
        return np.vstack([self.full_row_basis(t1) @ self.E[t1], self.full_row_basis(t2) @ self.E[t2]])

    def full_col_basis(self, s):
        ct = self.ct
        if ct.is_leaf(s):
            return self.W[s]
        s1, s2 = ct.sons(s)
        return np.vstack([self.full_col_basis(s1) @ self.F[s1], self.full_col_basis(s2) @ self.F[s2]])

    # -- matvec, P:1077-1081 ([BO10 Thm 3.42]): forward transform, couplings, backward
    def matvec_tree(self, x: np.ndarray, transpose: bool = False) -> np.ndarray:
        """y = Z x (or Z^T x) for x in TREE order; x may be (n,) or (n, m)."""
        rt, ct, bt = self.rt, self.ct, self.bt
        x = np.asarray(x, dtype=np.float64)
        vec = x.ndim == 1
        if vec:
            x = x[:, None]
        m = x.shape[1]
        if transpose:  # roles of the two bases swap
            src, dst = rt, ct
            srcL, srcT, dstL, dstT = self.V, self.E, self.W, self.F
            src_rank, dst_rank = self.k, self.l
        else:
            src, dst = ct, rt
            srcL, srcT, dstL, dstT = self.W, self.F, self.V, self.E
            src_rank, dst_rank = self.l, self.k
        # forward transform xhat_s = W_s^T x|s, bottom-up
        xh = [None] * src.nclusters
        for s in range(src.nclusters - 1, -1, -1):
            if src.is_leaf(s):
                xh[s] = srcL[s].T @ x[src.lo[s]:src.hi[s]]
            else:
                s1, s2 = src.sons(s)
                xh[s] = srcT[s1].T @ xh[s1] + srcT[s2].T @ xh[s2]
        yh = [np.zeros((int(dst_rank[t]), m)) for t in range(dst.nclusters)]
        y = np.zeros((dst.n, m))
        for b, Sb in self.S.items():
            t, s = bt.t[b], bt.s[b]
            if transpose:
                yh[s] += Sb.T @ xh[t]
            else:
                yh[t] += Sb @ xh[s]
        # backward transform, top-down
        for t in range(dst.nclusters):
            if dst.is_leaf(t):
                y[dst.lo[t]:dst.hi[t]] += dstL[t] @ yh[t]
            else:
                for t2 in dst.sons(t):
                    yh[t2] = yh[t2] + dstT[t2] @ yh[t]
        for b, Nb in self.N.items():
            t, s = bt.t[b], bt.s[b]
            if transpose:
                y[ct.lo[s]:ct.hi[s]] += Nb.T @ x[rt.lo[t]:rt.hi[t]]
            else:
                y[rt.lo[t]:rt.hi[t]] += Nb @ x[ct.lo[s]:ct.hi[s]]
        return y[:, 0] if vec else y

    def matvec(self, x: np.ndarray, transpose: bool = False) -> np.ndarray:
        """y = Z x with x, y in ORIGINAL order."""
        src = self.rt if transpose else self.ct
        dst = self.ct if transpose else self.rt
        yt = self.matvec_tree(np.asarray(x)[src.perm], transpose)
        y = np.empty_like(yt)
        y[dst.perm] = yt
        return y

    def storage(self):
        """Scalars stored: nearfield, leaf bases, transfers, couplings."""
        near = sum(v.size for v in self.N.values())
        leaf = sum(v.size for v in self.V.values()) + sum(v.size for v in self.W.values())
        tr = sum(v.size for v in self.E.values()) + sum(v.size for v in self.F.values())
        cp = sum(v.size for v in self.S.values())
        return near, leaf, tr, cp


def from_sparse(bt: BlockTree, A, lower: bool = False) -> H2:
    """h2_from_sparse: all ranks 0, CSR scattered into the
    nearfield.  A nonzero in an admissible block is a structure error."""
    rt, ct = bt.rt, bt.ct
    Z = H2(bt, lower=lower)
    A = A.tocsr()
    # tree-order copy of A
    Ap = A[rt.perm][:, ct.perm].tocoo()
    owner = {}
    for b in bt.inadm:
        owner[(int(bt.t[b]), int(bt.s[b]))] = b
    # leaf cluster of each tree position
    rleaf = np.empty(rt.n, dtype=np.int64)
    for t in rt.leaves():
        rleaf[rt.lo[t]:rt.hi[t]] = t
    cleaf = np.empty(ct.n, dtype=np.int64)
    for s in ct.leaves():
        cleaf[ct.lo[s]:ct.hi[s]] = s
    for i, j, v in zip(Ap.row, Ap.col, Ap.data):
        if v == 0.0:
            continue
        b = owner.get((int(rleaf[i]), int(cleaf[j])))
        if b is None:
            raise ValueError(f"H2_ERR_STRUCTURE: nonzero ({rt.perm[i]},{ct.perm[j]}) in an admissible block")
        if b not in Z.N:
            if lower:
                continue  # upper part of a symmetric matrix is not stored
            raise AssertionError
        t, s = bt.t[b], bt.s[b]
        Z.N[b][i - rt.lo[t], j - ct.lo[s]] += v
    return Z
