"""Pins for the oracle's structure code and the FEM inputs (CPU only).

Pinned against: closed forms on 2^a grids, SPEC hand examples, the partition /
son-rule properties of Def. 1-2, a brute-force evaluation of the
admissibility predicate on the raw point sets, and the hand 9x9 stencil."""
import os

import numpy as np
import pytest

from inputs import config, fem2d_csr, grid_points_2d, fem3d_kuhn_csr, jump_sigma_cells
from oracle.structure import ClusterTree, BlockTree, ADM, INADM, SUBDIV

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_fem_l2_hand_stencil():
    M = np.loadtxt(os.path.join(GOLD, "fem_l2_stencil.txt"), comments="#")
    np.testing.assert_array_equal(fem2d_csr(3).toarray(), M)


@pytest.mark.parametrize("N", [7, 31, 127])
def test_fem_n_matches_table1(N):
    # n = (2^l - 1)^2 (P:1421-1426 for l=7: 16 129)
    A = fem2d_csr(N)
    assert A.shape[0] == N * N
    if N == 127:
        assert A.shape[0] == 16129


def test_fem_jump_properties():
    N = 40
    sig = jump_sigma_cells(0)
    A = fem2d_csr(N, sig)
    assert abs(A - A.T).max() == 0.0
    d = A.toarray()
    # 5-point pattern only (hypotenuse couplings vanish, R18)
    i, j = np.nonzero(d)
    di = np.abs(i % N - j % N) + np.abs(i // N - j // N)
    assert di.max() <= 1
    # interior rows away from the boundary sum to zero
    inner = [(jj * N + ii) for jj in range(1, N - 1) for ii in range(1, N - 1)]
    assert np.abs(d[inner].sum(axis=1)).max() < 1e-9 * np.abs(d).max()
    # SPD
    assert np.linalg.eigvalsh(d).min() > 0
    # a single-cell sigma = c scales the Laplacian by c
    A1 = fem2d_csr(N, np.full((16, 16), 3.5)).toarray()
    np.testing.assert_allclose(A1, 3.5 * fem2d_csr(N).toarray(), rtol=0, atol=1e-15)


def test_fem_jump_edge_weights_by_hand():
    # Edge between (i,j) and (i+1,j) borders T_low of square (i,j-1)... hand-computed on a 2-cell sigma
    N = 3
    sig = np.ones((16, 16))
    sig[:, 8:] = 100.0  # x >= 0.5 is "100"
    A = fem2d_csr(N, sig).toarray()
    # node (2,1) -> idx 1 and node (3,1) -> idx 2: triangles sharing the edge have centroids with
    # x in (0.5, 0.75): both sigma 100 -> -(100+100)/2
    assert A[1, 2] == -100.0
    # node (1,1) -> idx 0 and (2,1) -> idx 1: centroids x < 0.5 -> -(1+1)/2
    assert A[0, 1] == -1.0


def test_fem3d_stencil():
    N = 4
    A = fem3d_kuhn_csr(N).toarray()
    h = 1.0 / (N + 1)
    assert np.allclose(np.diag(A), 6 * h)
    assert abs(A - A.T).max() == 0
    assert np.count_nonzero(A[N * N + N + 1]) == 7


def test_cluster_tree_spec_examples():
    # 1 point -> depth 0
    t = ClusterTree(np.zeros((1, 2)), 16)
    assert t.nclusters == 1 and t.depth == 0
    # 8 collinear equispaced points, leaf 2 -> perfect binary tree of depth 2, leaves of size 2
    t = ClusterTree(np.arange(8.0)[:, None], 2)
    assert t.depth == 2 and t.nclusters == 7
    assert [t.size(x) for x in t.leaves()] == [2, 2, 2, 2]
    assert list(t.perm) == list(range(8))


@pytest.mark.parametrize("N,leaf", [(32, 32), (64, 32), (128, 32), (16, 8)])
def test_cluster_tree_closed_forms(N, leaf):
    pts = grid_points_2d(N)
    t = ClusterTree(pts, leaf)
    n = N * N
    assert t.nclusters == 2 * n // leaf - 1
    assert t.depth == int(np.log2(n // leaf))
    assert all(t.size(x) == leaf for x in t.leaves())
    # partition: perm is a permutation and leaf ranges tile [0, n)
    assert sorted(t.perm.tolist()) == list(range(n))
    for c in range(t.nclusters):
        if not t.is_leaf(c):
            a, b = t.sons(c)
            assert t.lo[a] == t.lo[c] and t.hi[a] == t.lo[b] and t.hi[b] == t.hi[c]
            assert t.parent[a] == c and t.parent[b] == c
        # tight box of the cluster's own points
        p = pts[t.perm[t.lo[c]:t.hi[c]]]
        assert np.array_equal(p.min(0), t.bmin[c]) and np.array_equal(p.max(0), t.bmax[c])
    # preorder subtree ranges
    for c in range(t.nclusters):
        assert t.tsize[c] == 2 * (t.size(c) // leaf) - 1


def _brute_adm(pts_t, pts_s, eta):
    lo_t, hi_t = pts_t.min(0), pts_t.max(0)
    lo_s, hi_s = pts_s.min(0), pts_s.max(0)
    diam_t = np.sqrt(((hi_t - lo_t) ** 2).sum())
    diam_s = np.sqrt(((hi_s - lo_s) ** 2).sum())
    gap = np.maximum(0, np.maximum(lo_s - hi_t, lo_t - hi_s))
    dist = np.sqrt((gap ** 2).sum())
    return dist > 0 and max(diam_t, diam_s) <= eta * dist


@pytest.mark.parametrize("name", ["C0"])
def test_block_tree_partition_and_predicate(name):
    c = config(name)
    t = ClusterTree(c["points"], c["leaf"])
    bt = BlockTree(t, t, c["eta"])
    n = t.n
    cover = np.zeros((n, n), dtype=np.int64)
    for b in range(bt.nblocks):
        tt, ss = bt.t[b], bt.s[b]
        # son rule (Def. 2 with sons+)
        if bt.kind[b] == SUBDIV:
            expect = [(a, d) for a in t.sons_plus(tt) for d in t.sons_plus(ss)]
            assert [(bt.t[x], bt.s[x]) for x in bt.sons[b]] == expect
        else:
            assert bt.sons[b] == []
            cover[t.lo[tt]:t.hi[tt], t.lo[ss]:t.hi[ss]] += 1
            pt = c["points"][t.perm[t.lo[tt]:t.hi[tt]]]
            ps = c["points"][t.perm[t.lo[ss]:t.hi[ss]]]
            assert (bt.kind[b] == ADM) == _brute_adm(pt, ps, c["eta"])
            if bt.kind[b] == INADM:
                assert t.is_leaf(tt) and t.is_leaf(ss)
    assert (cover == 1).all()  # leaves partition I x I
    # every stiffness nonzero lands in an inadmissible leaf
    A = c["A"].tocoo()
    inv = np.empty(n, dtype=np.int64)
    inv[t.perm] = np.arange(n)
    near = np.zeros((n, n), dtype=bool)
    for b in bt.inadm:
        tt, ss = bt.t[b], bt.s[b]
        near[t.lo[tt]:t.hi[tt], t.lo[ss]:t.hi[ss]] = True
    assert near[inv[A.row], inv[A.col]].all()


def test_block_tree_counts_match_survey_appendix():
    # SURVEY Appendix A [calc] (same conventions): cross-check, not a paper value
    for name, adm, inadm, csp in (("C0", 264, 220, 18), ("C1", 8064, 4324, 30)):
        c = config(name)
        t = ClusterTree(c["points"], c["leaf"])
        bt = BlockTree(t, t, c["eta"])
        assert (len(bt.adm), len(bt.inadm), bt.sparsity()) == (adm, inadm, csp)


# ---- domain-decomposition clustering (NEXT-3, reading own-11) ----------------------
def _dd_checks(pts, A, leaf, eta):
    """Properties that define the DD tree: partition, nested-dissection order, interface =
    exactly the points of the right half coupled to the left half, decoupled domain pairs (no
    matrix entry, brute force on the dense pattern), block-tree partition with every nonzero in an
    inadmissible leaf."""
    n = pts.shape[0]
    t = ClusterTree(pts, leaf, adjacency=A)
    assert sorted(t.perm.tolist()) == list(range(n))
    D = (A != 0).toarray()
    D = D | D.T
    Dt = D[t.perm][:, t.perm]
    npairs = 0
    for c in range(t.nclusters):
        if t.is_leaf(c):
            assert t.size(c) <= max(leaf, 1)
            continue
        a, b = t.sons(c)
        assert t.lo[a] == t.lo[c] and t.hi[a] == t.lo[b] and t.hi[b] == t.hi[c]
        if t.ddpair[c]:
            npairs += 1
            assert not Dt[t.lo[a]:t.hi[a], t.lo[b]:t.hi[b]].any()  # decoupled domains
            p = t.parent[c]
            if p >= 0 and t.son0[p] == c and not t.ddpair[p]:
                g = t.son1[p]  # the interface of this split: every point coupled to dom1, none of dom2 is
                assert Dt[t.lo[g]:t.hi[g], t.lo[a]:t.hi[a]].any(axis=1).all()
                # geometric rule: dom1 is the left half (coord < mid of the father's box), the rest right
                ext = t.bmax[p] - t.bmin[p]
                ax = int(np.argmax(ext))
                mid2 = t.bmin[p][ax] + t.bmax[p][ax]
                assert (2 * pts[t.perm[t.lo[a]:t.hi[a]], ax] < mid2).all()
                assert (2 * pts[t.perm[t.lo[b]:t.hi[g]], ax] >= mid2).all()
    bt = BlockTree(t, t, eta)
    cover = np.zeros((n, n), dtype=np.int64)
    near = np.zeros((n, n), dtype=bool)
    for b in range(bt.nblocks):
        if bt.kind[b] != SUBDIV:
            tt, ss = bt.t[b], bt.s[b]
            cover[t.lo[tt]:t.hi[tt], t.lo[ss]:t.hi[ss]] += 1
            if bt.kind[b] == INADM:
                near[t.lo[tt]:t.hi[tt], t.lo[ss]:t.hi[ss]] = True
            else:
                pt, ps = pts[t.perm[t.lo[tt]:t.hi[tt]]], pts[t.perm[t.lo[ss]:t.hi[ss]]]
                pair = tt != ss and t.parent[tt] == t.parent[ss] and t.ddpair[t.parent[tt]]
                assert pair or _brute_adm(pt, ps, eta)
    assert (cover == 1).all()
    assert near[Dt].all()
    return t, bt, npairs


def test_dd_tree_nested_dissection_closed_form():
    """(2^l - 1)^2 grid, 5-point stencil: the root split is the classical nested dissection --
    separator = the middle grid line (2^l - 1 points), two domains of (2^(l-1) - 1)(2^l - 1)."""
    l = 5
    N = 2 ** l - 1
    c = config("C1", N=N)
    t, bt, npairs = _dd_checks(c["points"], c["A"], 32, 2.0)
    inner, gam = t.sons(0)
    assert t.ddpair[inner] and not t.ddpair[0]
    assert t.size(gam) == N and all(t.size(d) == (2 ** (l - 1) - 1) * N for d in t.sons(inner))
    assert (c["points"][t.perm[t.lo[gam]:t.hi[gam]], 0] == 2 ** (l - 1)).all()
    assert npairs >= 7
    # without the graph the constructor is the plain bisection tree
    assert not ClusterTree(c["points"], 32).ddpair.any()


def test_dd_tree_irregular_graph():
    """Random points with a k-nearest-neighbour coupling graph (unsymmetric pattern, symmetrised
    by the constructor), and a graph with two components (an empty interface)."""
    rng = np.random.default_rng(3)
    pts = np.round(rng.uniform(0, 100, (400, 2)))
    d2 = ((pts[:, None, :] - pts[None, :, :]) ** 2).sum(-1)
    nb = np.argsort(d2, axis=1)[:, :5]
    import scipy.sparse as sp
    A = sp.csr_matrix((np.ones(nb.size), (np.repeat(np.arange(400), 5), nb.ravel())), shape=(400, 400))
    _dd_checks(pts, A, 16, 2.0)
    # two far-apart clouds coupled only inside themselves: the root itself is a decoupled pair
    pts2 = np.vstack([pts[:100], pts[100:200] + [1000.0, 0.0]])
    B = sp.block_diag([A[:100, :100], A[100:200, 100:200]]).tocsr()
    t, _, _ = _dd_checks(pts2, B, 16, 2.0)
    assert t.ddpair[0]
