"""ORACLE (test infrastructure only) — cluster tree and block tree.

Cluster tree: PAPER Def. 1, binary.  Construction by
geometric bisection with the conventions of SURVEY §8(c).1 / R2:
  * box = tight axis-aligned bounding box of the cluster's points
  * split axis = largest extent, ties -> lowest axis index
  * son0 gets the points with coord < (lo+hi)/2, original relative order kept
  * stop when #t <= leaf_size; clusters numbered in DFS preorder (root 0, son0 first)
Block tree: PAPER Def. 2, sons(b) = sons+(t) x sons+(s),
t-son-major order.  Admissibility (never stated in the paper; reading
SURVEY R1): (t,s) admissible iff dist > 0 and max(diam_t^2, diam_s^2) <= eta^2 dist^2.
row(t), pred(t): P:594-607.  C_sp: P:981-988.

Domain-decomposition clustering ("a domain decomposition cluster
strategy similar to the one described in [GRKRLE05a]" -- the paper gives no details; DESIGN
reading own-11).  With the sparsity graph of the matrix (adjacency, symmetrised), a DOMAIN
cluster t with more than 2 leaf_size points (smaller ones are bisected plainly: their domains
would be tiny) is bisected geometrically as above into (left, right); the interface gamma is the set
of points of `right` coupled to a point of `left`; dom1 = left, dom2 = right minus gamma.  The
ternary split {dom1, dom2, gamma} of [GRKRLE05a] is realised in the binary tree as
    t -> (interior, gamma),   interior -> (dom1, dom2),
so the tree order is the nested-dissection order [dom1, dom2, gamma].  dom1 and dom2 are DOMAIN
clusters (split again the same way), gamma is an INTERFACE cluster (plain geometric bisection
below it).  If gamma is empty the halves are already decoupled: t -> (left, right) is itself a
decoupled pair; if dom2 is empty, or the interior has at most leaf_size points, t is split
plainly into (left, right) [right an INTERFACE cluster when it is all interface] with no
decoupling claimed.  `ddpair[p]` marks clusters whose two sons are decoupled domains: no matrix
entry couples them, and none is created by the LR / Cholesky factorization in tree order
(nested dissection), so the block (dom1, dom2) is an admissible leaf of rank zero whatever its
geometry (BlockTree below).
"""
import numpy as np

SUBDIV, ADM, INADM = 0, 1, 2


class ClusterTree:
    """Arrays indexed by cluster id (DFS preorder).  Index ranges are in tree order."""

    def __init__(self, points: np.ndarray, leaf_size: int, adjacency=None):
        """adjacency: None (geometric bisection) or a scipy sparse matrix whose pattern (taken
        symmetrically) is the coupling graph -> domain-decomposition clustering (see above)."""
        pts = np.asarray(points, dtype=np.float64)
        if pts.ndim != 2 or pts.shape[0] < 1 or leaf_size < 1:
            raise ValueError("need n >= 1 points and leaf_size >= 1")
        self.n, self.dim = pts.shape
        self.leaf_size = leaf_size
        lo, hi, son0, son1, parent, level, bmin, bmax = [], [], [], [], [], [], [], []
        ddpair = []
        perm = np.empty(self.n, dtype=np.int64)
        if adjacency is not None:
            G = (adjacency != 0).astype(np.int8).tocsr()
            G = (G + G.T).tocsr()
            gptr, gidx = G.indptr, G.indices
            in_left = np.zeros(self.n, dtype=bool)
        DOMAIN, INTERFACE = 0, 1

        def build(idx, start, par, lev, kind=INTERFACE, presplit=None):
            cid = len(lo)
            ddpair.append(False)
            lo.append(start)
            hi.append(start + len(idx))
            son0.append(-1)
            son1.append(-1)
            parent.append(par)
            level.append(lev)
            p = pts[idx]
            bmin.append(p.min(axis=0))
            bmax.append(p.max(axis=0))
            if presplit is not None:  # the interior cluster of a DD split: its sons are the domains
                i0, i1 = presplit
                ddpair[cid] = True
                c0 = build(i0, start, cid, lev + 1, DOMAIN)
                c1 = build(i1, start + len(i0), cid, lev + 1, DOMAIN)
                son0[cid], son1[cid] = c0, c1
                return cid
            if len(idx) <= leaf_size:
                perm[start:start + len(idx)] = idx
                return cid
            ext = bmax[cid] - bmin[cid]
            ax = int(np.argmax(ext))  # first maximal axis = lowest index on ties
            # coord < (lo+hi)/2  <=>  2*coord < lo+hi   (exact for integer-valued coordinates)
            left = 2.0 * p[:, ax] < bmin[cid][ax] + bmax[cid][ax]
            i0, i1 = idx[left], idx[~left]
            if len(i0) == 0 or len(i1) == 0:  # all points coincide on the split axis: stop
                perm[start:start + len(idx)] = idx
                return cid
            if adjacency is not None and kind == DOMAIN and len(idx) > 2 * leaf_size:
                in_left[i0] = True
                coupled = np.array([in_left[gidx[gptr[q]:gptr[q + 1]]].any() for q in i1], dtype=bool)
                in_left[i0] = False
                gam, d2 = i1[coupled], i1[~coupled]
                if len(gam) == 0:  # the halves are not coupled at all
                    ddpair[cid] = True
                    c0 = build(i0, start, cid, lev + 1, DOMAIN)
                    c1 = build(i1, start + len(i0), cid, lev + 1, DOMAIN)
                elif len(d2) == 0 or len(i0) + len(d2) <= leaf_size:  # no decoupling gained
                    c0 = build(i0, start, cid, lev + 1, DOMAIN)
                    c1 = build(i1, start + len(i0), cid, lev + 1, INTERFACE if len(d2) == 0 else DOMAIN)
                else:
                    inner = np.concatenate([i0, d2])
                    c0 = build(inner, start, cid, lev + 1, DOMAIN, presplit=(i0, d2))
                    c1 = build(gam, start + len(inner), cid, lev + 1, INTERFACE)
                son0[cid], son1[cid] = c0, c1
                return cid
            c0 = build(i0, start, cid, lev + 1, kind)
            c1 = build(i1, start + len(i0), cid, lev + 1, kind)
            son0[cid], son1[cid] = c0, c1
            return cid

        import sys
        sys.setrecursionlimit(max(sys.getrecursionlimit(), 10000))
        build(np.arange(self.n), 0, -1, 0, DOMAIN if adjacency is not None else INTERFACE)
        self.ddpair = np.array(ddpair, dtype=bool)
        self.lo = np.array(lo, dtype=np.int64)
        self.hi = np.array(hi, dtype=np.int64)
        self.son0 = np.array(son0, dtype=np.int64)
        self.son1 = np.array(son1, dtype=np.int64)
        self.parent = np.array(parent, dtype=np.int64)
        self.level = np.array(level, dtype=np.int64)
        self.bmin = np.array(bmin)
        self.bmax = np.array(bmax)
        self.perm = perm
        self.nclusters = len(lo)
        self.depth = int(self.level.max())
        # number of clusters in the subtree of t (subtree = contiguous preorder id range)
        self.tsize = np.ones(self.nclusters, dtype=np.int64)
        for t in range(self.nclusters - 1, -1, -1):
            if self.son0[t] >= 0:
                self.tsize[t] = 1 + self.tsize[self.son0[t]] + self.tsize[self.son1[t]]

    def is_leaf(self, t) -> bool:
        return self.son0[t] < 0

    def sons(self, t):
        return [] if self.son0[t] < 0 else [int(self.son0[t]), int(self.son1[t])]

    def sons_plus(self, t):
        """sons+(t)."""
        return [t] if self.son0[t] < 0 else [int(self.son0[t]), int(self.son1[t])]

    def size(self, t) -> int:
        return int(self.hi[t] - self.lo[t])

    def in_subtree(self, t, root) -> bool:
        return root <= t < root + self.tsize[root]

    def subtree(self, t):
        """T_t in preorder."""
        return list(range(int(t), int(t + self.tsize[t])))

    def pred(self, t):
        """pred(t) as a list root ... t."""
        out = []
        while t >= 0:
            out.append(int(t))
            t = self.parent[t]
        return out[::-1]

    def leaves(self):
        return [t for t in range(self.nclusters) if self.son0[t] < 0]

    def diam2(self, t):
        e = self.bmax[t] - self.bmin[t]
        return float(np.dot(e, e))


def dist2(rt: ClusterTree, t, ct: ClusterTree, s):
    g = np.maximum(0.0, np.maximum(ct.bmin[s] - rt.bmax[t], rt.bmin[t] - ct.bmax[s]))
    return float(np.dot(g, g))


def admissible(rt, t, ct, s, eta):
    """SURVEY R1 reading of the (unstated) admissibility condition; with a
    domain-decomposition tree (rt is ct) the two decoupled domains of a split also form an
    admissible (zero) block (reading own-11)."""
    if rt is ct and t != s and rt.parent[t] >= 0 and rt.parent[t] == ct.parent[s] and rt.ddpair[rt.parent[t]]:
        return True
    d2 = dist2(rt, t, ct, s)
    return d2 > 0.0 and max(rt.diam2(t), ct.diam2(s)) <= eta * eta * d2


class BlockTree:
    """Block tree over (rt, ct), nodes in DFS preorder."""

    def __init__(self, rt: ClusterTree, ct: ClusterTree, eta: float):
        self.rt, self.ct, self.eta = rt, ct, float(eta)
        T, S, kind, parent, sons = [], [], [], [], []

        def build(t, s, par):
            b = len(T)
            T.append(t)
            S.append(s)
            parent.append(par)
            sons.append([])
            if admissible(rt, t, ct, s, eta):
                kind.append(ADM)
                return b
            if rt.is_leaf(t) and ct.is_leaf(s):
                kind.append(INADM)
                return b
            kind.append(SUBDIV)
            for t2 in rt.sons_plus(t):
                for s2 in ct.sons_plus(s):
                    sons[b].append(build(t2, s2, b))
            return b

        build(0, 0, -1)
        self.t = np.array(T, dtype=np.int64)
        self.s = np.array(S, dtype=np.int64)
        self.kind = np.array(kind, dtype=np.int64)
        self.parent = np.array(parent, dtype=np.int64)
        self.sons = sons
        self.nblocks = len(T)
        self.index = {(int(a), int(c)): i for i, (a, c) in enumerate(zip(T, S))}
        self.bsize = np.ones(self.nblocks, dtype=np.int64)
        for b in range(self.nblocks - 1, -1, -1):
            self.bsize[b] = 1 + sum(self.bsize[c] for c in sons[b])
        self.adm = [b for b in range(self.nblocks) if kind[b] == ADM]
        self.inadm = [b for b in range(self.nblocks) if kind[b] == INADM]
        # row(t) / col(s): admissible leaves by cluster
        self.row = [[] for _ in range(rt.nclusters)]
        self.col = [[] for _ in range(ct.nclusters)]
        for b in self.adm:
            self.row[self.t[b]].append(b)
            self.col[self.s[b]].append(b)
        self.nrow = [[] for _ in range(rt.nclusters)]  # inadmissible leaves per row cluster
        for b in self.inadm:
            self.nrow[self.t[b]].append(b)

    def subtree(self, b):
        """T_{b}, preorder ids (contiguous)."""
        return range(int(b), int(b + self.bsize[b]))

    def sparsity(self):
        """C_sp: max number of blocks (any kind) sharing a row / column cluster."""
        cr = np.bincount(self.t, minlength=self.rt.nclusters)
        cc = np.bincount(self.s, minlength=self.ct.nclusters)
        return int(max(cr.max(), cc.max()))
