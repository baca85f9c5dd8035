"""ORACLE (test infrastructure only) — O2: dense brute-force definitions (n <= ~4096).

These restate what the paper's construction computes, without weights, R-factors
or nested recursions, so that a mistake in O1 (oracle/update.py) shows up as a
disagreement:
  * densify: G|_b = V_t S_b W_s^T on admissible leaves (eq. (2)) with
    V_t expanded from the leaves by eq. (1) written as explicit products, dense N_b
    on inadmissible leaves.
  * local update: Q_t from the SVD of the materialised block row
      Z~_t = [Z~|_{t x s} : s in row*(t)]
    leaf: left singular vectors of Z~_t; internal: Q_t = (Q_{t1} (+) Q_{t2}) Qhat_t with
    Qhat_t from (Q_{t1} (+) Q_{t2})^T Z~_t
    By P:671-691 and P:841-849 this equals O1 exactly in exact arithmetic, ranks
    included.  New admissible blocks are orthogonal projections P_t Z~|_b P_s
    (P:861-868); for blocks of proper ancestors of t0 only the rows t0 are
    projected by Q_{t0}Q_{t0}^T (E_{t0} <- R_{t0}[E_{t0};0]).
"""
import numpy as np

from .structure import ADM, INADM


def expand_leafwise(tree, leaf, transfer, t):
    """V_t (|t| x k_t) by explicit products down to the leaves: V_t|_{leaf} = V_leaf E_leaf ... E_{son of t}."""
    rows = []
    for q in tree.subtree(t):
        if not tree.is_leaf(q):
            continue
        M = leaf[q]
        a = q
        while a != t:
            M = M @ transfer[a]
            a = tree.parent[a]
        rows.append(M)
    return np.vstack(rows)


def densify(Z) -> np.ndarray:
    """Dense matrix in TREE order (stored blocks only)."""
    rt, ct, bt = Z.rt, Z.ct, Z.bt
    D = np.zeros((rt.n, ct.n))
    for b, S in Z.S.items():
        t, s = bt.t[b], bt.s[b]
        Vt = expand_leafwise(rt, Z.V, Z.E, t)
        Ws = expand_leafwise(ct, Z.W, Z.F, s)
        D[rt.lo[t]:rt.hi[t], ct.lo[s]:ct.hi[s]] = Vt @ S @ Ws.T
    for b, N in Z.N.items():
        t, s = bt.t[b], bt.s[b]
        D[rt.lo[t]:rt.hi[t], ct.lo[s]:ct.hi[s]] = N
    return D


def block_row(D, Z, t, row_side=True, blockwise=False):
    """Z~_t: stored admissible blocks (t*, s), t* in pred(t), restricted to rows t.
    blockwise (NEXT-1): each block scaled by 1 / ||D|_{t* x s}||_F (the whole block's norm)."""
    rt, ct, bt = Z.rt, Z.ct, Z.bt
    tree = rt if row_side else ct
    blocks = bt.row if row_side else bt.col
    cols = []
    for tp in tree.pred(t):
        for b in blocks[tp]:
            if b not in Z.S:
                continue
            if row_side:
                s = bt.s[b]
                blk = D[rt.lo[t]:rt.hi[t], ct.lo[s]:ct.hi[s]]
                full = D[rt.lo[tp]:rt.hi[tp], ct.lo[s]:ct.hi[s]]
            else:
                r = bt.t[b]
                blk = D[rt.lo[r]:rt.hi[r], ct.lo[t]:ct.hi[t]].T
                full = D[rt.lo[r]:rt.hi[r], ct.lo[tp]:ct.hi[tp]]
            if blockwise:
                nrm = np.linalg.norm(full)
                if nrm == 0.0:
                    continue
                blk = blk / nrm
            cols.append(blk)
    if not cols:
        return np.zeros((tree.size(t), 0))
    return np.hstack(cols)


def _dense_bases(D, Z, root, row_side, trunc):
    tree = Z.rt if row_side else Z.ct
    Q, r, sig = {}, {}, {}
    for t in reversed(tree.subtree(root)):
        Zt = block_row(D, Z, t, row_side, getattr(trunc, "blockwise", False))
        if tree.is_leaf(t):
            P = np.eye(tree.size(t))
        else:
            t1, t2 = tree.sons(t)
            P = np.zeros((tree.size(t), Q[t1].shape[1] + Q[t2].shape[1]))
            n1 = tree.size(t1)
            P[:n1, :Q[t1].shape[1]] = Q[t1]
            P[n1:, Q[t1].shape[1]:] = Q[t2]
        M = P.T @ Zt
        if M.size:
            U, s, _ = np.linalg.svd(M, full_matrices=False)
        else:
            U, s = np.zeros((M.shape[0], 0)), np.zeros(0)
        rk = trunc.rank(s)
        Q[t] = P @ U[:, :rk]
        r[t] = rk
        sig[t] = s
    return Q, r, sig


def local_update_dense(Z, t0, s0, X, Y, trunc):
    """O2 result of the local update on densify(Z): (new dense matrix, row ranks, col ranks, sigmas)."""
    rt, ct, bt = Z.rt, Z.ct, Z.bt
    D = densify(Z)
    D[rt.lo[t0]:rt.hi[t0], ct.lo[s0]:ct.hi[s0]] += X @ Y.T
    b0 = bt.index[(t0, s0)]
    # keep the "not stored" region zero (lower storage)
    if Z.lower:
        for b in range(bt.nblocks):
            if bt.kind[b] != 0 and b not in Z.S and b not in Z.N:
                t, s = bt.t[b], bt.s[b]
                D[rt.lo[t]:rt.hi[t], ct.lo[s]:ct.hi[s]] = 0.0
    if X.shape[1] == 0 or bt.kind[b0] == INADM:
        return D, {}, {}, ({}, {})
    Qr, rr, sr = _dense_bases(D, Z, t0, True, trunc)
    Qc, rc, sc = _dense_bases(D, Z, s0, False, trunc)
    out = D.copy()
    for b in Z.S:
        t, s = int(bt.t[b]), int(bt.s[b])
        blk = D[rt.lo[t]:rt.hi[t], ct.lo[s]:ct.hi[s]].copy()
        if rt.in_subtree(t, t0):
            blk = Qr[t] @ (Qr[t].T @ blk)
        elif t in rt.pred(t0):
            a, e = rt.lo[t0] - rt.lo[t], rt.hi[t0] - rt.lo[t]
            blk[a:e] = Qr[t0] @ (Qr[t0].T @ blk[a:e])
        if ct.in_subtree(s, s0):
            blk = (blk @ Qc[s]) @ Qc[s].T
        elif s in ct.pred(s0):
            a, e = ct.lo[s0] - ct.lo[s], ct.hi[s0] - ct.lo[s]
            blk[:, a:e] = (blk[:, a:e] @ Qc[s0]) @ Qc[s0].T
        out[rt.lo[t]:rt.hi[t], ct.lo[s]:ct.hi[s]] = blk
    return out, rr, rc, (sr, sc)
