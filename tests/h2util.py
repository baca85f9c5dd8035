"""Shared test helpers: build the oracle and the CUDA-path matrices for one config."""
import numpy as np

from inputs import config
from inputs.rng import probes
from oracle.structure import ClusterTree, BlockTree, ADM
from oracle.h2 import from_sparse as o_from_sparse


def setup(name, N=None, lower=False, rank_cap=32, update_cap=32, gpu=True, eta=None, dd=False):
    """dd: domain-decomposition cluster tree (NEXT-3) instead of geometric bisection."""
    c = config(name, N=N)
    if eta is not None:
        c["eta"] = eta
    ot = ClusterTree(c["points"], c["leaf"], adjacency=c["A"] if dd else None)
    ob = BlockTree(ot, ot, c["eta"])
    OZ = o_from_sparse(ob, c["A"], lower=lower)
    out = dict(c=c, ot=ot, ob=ob, OZ=OZ)
    if gpu:
        import paper_1402_5056_b200 as P
        t = P.h2_cluster_tree_dd(c["points"], c["leaf"], c["A"]) if dd else P.h2_cluster_tree(c["points"], c["leaf"])
        bt = P.h2_block_tree(t, t, c["eta"])
        Z = P.h2_from_sparse(bt, c["A"], lower=lower, rank_cap=rank_cap, update_cap=update_cap)
        out.update(t=t, bt=bt, Z=Z)
    return out


def adm_targets(ot, ob):
    return [(int(ob.t[b]), int(ob.s[b]), ot.size(ob.t[b]), ot.size(ob.s[b])) for b in ob.adm]


def all_targets(ot, ob):
    return [(int(ob.t[b]), int(ob.s[b]), ot.size(ob.t[b]), ot.size(ob.s[b])) for b in range(ob.nblocks)]


def gpu_apply(Z, Xp):
    """Apply the GPU operator to the columns of Xp (n x m numpy, ORIGINAL order)."""
    import torch
    import paper_1402_5056_b200 as P
    out = np.empty_like(Xp)
    for j in range(Xp.shape[1]):
        x = torch.from_numpy(np.ascontiguousarray(Xp[:, j])).cuda()
        y = P.h2_matvec(Z, x)
        out[:, j] = y.cpu().numpy()
    return out


def operator_rel_diff(Z, OZ, n, count=16, seed=0):
    """North-star operator parity: relative 2-norm difference of Z and the oracle on 16 seeded probes."""
    Xp = probes(n, count, seed).T
    yg = gpu_apply(Z, Xp)
    yo = OZ.matvec(Xp)
    return np.linalg.norm(yg - yo) / np.linalg.norm(yo)
