"""Pins for the oracle's H^2 representation and local low-rank update (CPU only).

O1 (oracle/update.py, the paper's weighted nested algorithm) is held to things
other than itself:
  * O2 (oracle/dense.py): the SVD of the materialised block rows Z~_t, which the
    paper proves equivalent -- ranks bit-equal, operators 1e-12;
  * exactness with no truncation (rel_tol = 0): densify = old + X Y^T;
  * k = 0 bit-identical; untouched region bit-identical;
  * the C0 exact-rank pin: rank exactly 8 where row* is non-empty and
    densify = A + P_adm(X Y^T)/n;
  * orthonormality of freshly rebuilt subtree bases;
  * matvec against an independent dense product.
"""
import os

import numpy as np
import pytest

from inputs import config, stream, XFAC, YFAC
from oracle.structure import ClusterTree, BlockTree, ADM, INADM
from oracle.h2 import from_sparse
from oracle.update import Updater, Trunc, FIXED16, qr_R
from oracle.dense import densify, local_update_dense, expand_leafwise

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _c0():
    c = config("C0")
    rt = ClusterTree(c["points"], c["leaf"])
    bt = BlockTree(rt, rt, c["eta"])
    return c, rt, bt


def test_linalg_golden_examples():
    lines = [l.split("|") for l in open(os.path.join(GOLD, "linalg_examples.txt")) if not l.startswith("#")]
    g = {l[0].strip(): l[2].split() for l in lines}
    R = qr_R(np.array([[3.0], [4.0]]), 1)
    assert abs(abs(R[0, 0]) - float(g["qr_col34_R"][0])) < 1e-15
    assert Trunc(0.5).rank(np.array([3.0, 1.0])) == int(g["svd_diag31_rank"][0])
    assert Trunc(0.5).rank(np.zeros(2)) == int(g["svd_zero_rank"][0])
    L = np.linalg.cholesky(np.array([[4.0, 2.0], [2.0, 3.0]]))
    np.testing.assert_allclose(L.ravel(), [float(x) for x in g["chol_4223_L"]], atol=1e-15)


def test_from_sparse_densify_exact_and_matvec():
    c, rt, bt = _c0()
    Z = from_sparse(bt, c["A"])
    A = c["A"].toarray()
    np.testing.assert_array_equal(densify(Z), A[rt.perm][:, rt.perm])
    assert Z.k.sum() == 0 and Z.l.sum() == 0
    x = stream(6).standard_normal((rt.n, 3))
    np.testing.assert_allclose(Z.matvec(x), A @ x, rtol=0, atol=1e-12)


def _random_updates(Z, bt, rt, trunc, count, seed, check_o2=True, only_kinds=None):
    rng = np.random.default_rng(seed)
    up = Updater(Z, trunc)
    worst = 0.0
    for _ in range(count):
        while True:
            b = int(rng.integers(bt.nblocks))
            if only_kinds is None or bt.kind[b] in only_kinds:
                break
        t0, s0 = int(bt.t[b]), int(bt.s[b])
        k = int(rng.integers(1, 9))
        X = rng.standard_normal((rt.size(t0), k))
        Y = rng.standard_normal((rt.size(s0), k))
        if check_o2:
            D2, rr, rc, (sr, sc) = local_update_dense(Z, t0, s0, X, Y, trunc)
        log = {}
        up(t0, s0, X, Y, log=log)
        if check_o2:
            D1 = densify(Z)
            worst = max(worst, np.linalg.norm(D1 - D2) / np.linalg.norm(D2))
            for t in rr:
                assert log["row_rank"][t] == rr[t]
            for s in rc:
                assert log["col_rank"][s] == rc[s]
            # weight fidelity: sigma(V~_t B~_t^T) = sigma(Z~_t) at leaves
            for t, sig in sr.items():
                if rt.is_leaf(t):
                    a, b2 = log["row_sig"][t], sig
                    m = min(a.size, b2.size)
                    if m:
                        assert np.allclose(a[:m], b2[:m], rtol=0, atol=1e-10 * max(1.0, b2[0]))
    return worst


@pytest.mark.parametrize("trunc", [Trunc(1e-4), Trunc(1e-2), Trunc(1e-12, 0.0, 4)])
def test_o1_equals_o2_random_updates(trunc):
    c, rt, bt = _c0()
    Z = from_sparse(bt, c["A"])
    worst = _random_updates(Z, bt, rt, trunc, 30, seed=7)
    assert worst < 1e-12


def test_no_truncation_is_exact():
    c, rt, bt = _c0()
    Z = from_sparse(bt, c["A"])
    rng = np.random.default_rng(3)
    up = Updater(Z, Trunc(0.0))
    D = densify(Z)
    for _ in range(12):
        b = bt.adm[int(rng.integers(len(bt.adm)))] if rng.random() < 0.5 else int(rng.integers(bt.nblocks))
        t0, s0 = int(bt.t[b]), int(bt.s[b])
        X = rng.standard_normal((rt.size(t0), 3))
        Y = rng.standard_normal((rt.size(s0), 3))
        up(t0, s0, X, Y)
        D[rt.lo[t0]:rt.hi[t0], rt.lo[s0]:rt.hi[s0]] += X @ Y.T
    assert np.linalg.norm(densify(Z) - D) / np.linalg.norm(D) < 1e-12


def test_k0_bit_identical_and_untouched_region():
    c, rt, bt = _c0()
    Z = from_sparse(bt, c["A"])
    _random_updates(Z, bt, rt, Trunc(1e-4), 10, seed=11, check_o2=False)
    before = Z.copy()
    up = Updater(Z, Trunc(1e-4))
    b = bt.adm[5]
    t0, s0 = int(bt.t[b]), int(bt.s[b])
    up(t0, s0, np.zeros((rt.size(t0), 0)), np.zeros((rt.size(s0), 0)))
    for key in before.S:
        assert np.array_equal(before.S[key], Z.S[key])
    for key in before.E:
        assert np.array_equal(before.E[key], Z.E[key])
    # a real update: blocks away from T_{t0} u pred(t0) and T_{s0} u pred(s0) are bit-identical
    D0 = densify(Z)
    rng = np.random.default_rng(5)
    up(t0, s0, rng.standard_normal((rt.size(t0), 4)), rng.standard_normal((rt.size(s0), 4)))
    D1 = densify(Z)
    near_t = set(rt.subtree(t0)) | set(rt.pred(t0))
    near_s = set(rt.subtree(s0)) | set(rt.pred(s0))
    checked = 0
    for key, S in before.S.items():
        t, s = int(bt.t[key]), int(bt.s[key])
        if t in near_t or s in near_s:
            continue
        assert np.array_equal(S, Z.S[key])
        sl = np.s_[rt.lo[t]:rt.hi[t], rt.lo[s]:rt.hi[s]]
        assert np.array_equal(D0[sl], D1[sl])
        checked += 1
    assert checked > 50


def test_fresh_subtree_bases_orthonormal():
    c, rt, bt = _c0()
    Z = from_sparse(bt, c["A"])
    _random_updates(Z, bt, rt, Trunc(1e-4), 8, seed=21, check_o2=False, only_kinds=(ADM,))
    up = Updater(Z, Trunc(1e-4))
    t0 = s0 = 0  # global update (t0 = s0 = root)
    rng = np.random.default_rng(2)
    up(t0, s0, rng.standard_normal((rt.n, 5)), rng.standard_normal((rt.n, 5)))
    for t in range(rt.nclusters):
        for V in (expand_leafwise(rt, Z.V, Z.E, t), expand_leafwise(rt, Z.W, Z.F, t)):
            if V.shape[1]:
                assert np.abs(V.T @ V - np.eye(V.shape[1])).max() < 1e-12


def test_zero_update_does_not_raise_ranks():
    # recompression of a zero-extended representation recovers the original ranks
    c, rt, bt = _c0()
    Z = from_sparse(bt, c["A"])
    _random_updates(Z, bt, rt, Trunc(1e-10), 6, seed=4, check_o2=False, only_kinds=(ADM,))
    k0, l0 = Z.k.copy(), Z.l.copy()
    D0 = densify(Z)
    Updater(Z, Trunc(1e-10))(0, 0, np.zeros((rt.n, 6)), np.zeros((rt.n, 6)))
    assert (Z.k <= k0).all() and (Z.l <= l0).all()
    assert np.linalg.norm(densify(Z) - D0) <= 1e-8 * np.linalg.norm(D0)


def test_c0_exact_rank8_pin():
    """one global X, Y in R^{n x 8}, alpha = 1/n, one local update per admissible
    leaf in block-tree DFS order.  Result = A + P_adm(X Y^T)/n exactly; rank 8 exactly on every
    cluster whose row*/col* is non-empty, 0 elsewhere."""
    c, rt, bt = _c0()
    n = rt.n
    X = stream(XFAC).standard_normal((n, 8))  # rows in ORIGINAL order
    Y = stream(YFAC).standard_normal((n, 8))
    Xt, Yt = X[rt.perm], Y[rt.perm]
    Z = from_sparse(bt, c["A"])
    up = Updater(Z, Trunc(1e-4))
    for b in bt.adm:
        t0, s0 = int(bt.t[b]), int(bt.s[b])
        up(t0, s0, Xt[rt.lo[t0]:rt.hi[t0]], Yt[rt.lo[s0]:rt.hi[s0]], alpha=1.0 / n)
    D = c["A"].toarray()[rt.perm][:, rt.perm]
    P = np.zeros((n, n))
    for b in bt.adm:
        t, s = bt.t[b], bt.s[b]
        P[rt.lo[t]:rt.hi[t], rt.lo[s]:rt.hi[s]] = 1.0
    expect = D + P * (Xt @ Yt.T) / n
    assert np.linalg.norm(densify(Z) - expect) / np.linalg.norm(expect) < 1e-12
    for t in range(rt.nclusters):
        has_row = any(bt.row[p] for p in rt.pred(t))
        has_col = any(bt.col[p] for p in rt.pred(t))
        assert Z.k[t] == (8 if has_row else 0)
        assert Z.l[t] == (8 if has_col else 0)


def test_transpose_matvec_nonzero_ranks():
    """H.matvec_tree(transpose=True) with non-zero ranks equals densify(Z)^T x (P:1077-1081 with the
    roles of the row and column bases swapped); also the plain product."""
    c, rt, bt = _c0()
    Z = from_sparse(bt, c["A"])
    _random_updates(Z, bt, rt, Trunc(1e-6), 12, seed=31, check_o2=False)
    assert Z.k.max() > 0 and Z.l.max() > 0
    D = densify(Z)
    x = stream(6).standard_normal((rt.n, 2))
    np.testing.assert_allclose(Z.matvec_tree(x, transpose=True), D.T @ x, rtol=0, atol=1e-10 * np.abs(D.T @ x).max())
    np.testing.assert_allclose(Z.matvec_tree(x), D @ x, rtol=0, atol=1e-10 * np.abs(D @ x).max())


@pytest.mark.parametrize("eps", [1e-2, 1e-4])
def test_blockwise_o1_equals_o2(eps):
    """NEXT-1 (reading own-10): the blockwise-relative weights in the paper's nested recursion (O1)
    equal the dense definition -- SVDs of the block rows with every block scaled by 1 / its
    Frobenius norm, absolute threshold eps^ (O2) -- in ranks and result."""
    c, rt, bt = _c0()
    Z = from_sparse(bt, c["A"])
    worst = _random_updates(Z, bt, rt, Trunc(eps, blockwise=True), 24, seed=17)
    assert worst < 1e-12


def test_blockwise_error_bound_per_block():
    """The point of blockwise-relative truncation: after a local update every
    admissible block keeps its own relative accuracy, ||G_b - G~_b||_2 <= 2 (depth + 1) eps^ ||G_b||_F
    (row and column truncation, each accumulating at most depth + 1 levels), whatever the blocks'
    magnitudes -- here blocks scaled over eight orders of magnitude."""
    c, rt, bt = _c0()
    Z = from_sparse(bt, c["A"])
    eps = 1e-3
    up = Updater(Z, Trunc(1e-13))
    rng = np.random.default_rng(3)
    for b in bt.adm:  # build blocks of wildly different size: exact (tight truncation)
        t0, s0 = int(bt.t[b]), int(bt.s[b])
        scale = 10.0 ** rng.uniform(-4, 4)
        up(t0, s0, scale * rng.standard_normal((rt.size(t0), 3)), rng.standard_normal((rt.size(s0), 3)))
    depth = max(rt.level)
    b0 = next(b for b in range(bt.nblocks) if bt.kind[b] == 0 and rt.size(bt.t[b]) >= 128)
    t0, s0 = int(bt.t[b0]), int(bt.s[b0])
    X = rng.standard_normal((rt.size(t0), 4))
    Y = rng.standard_normal((rt.size(s0), 4))
    exact = densify(Z)
    exact[rt.lo[t0]:rt.hi[t0], rt.lo[s0]:rt.hi[s0]] += X @ Y.T
    Updater(Z, Trunc(eps, blockwise=True))(t0, s0, X, Y)
    got = densify(Z)
    worst = 0.0
    for b in bt.adm:
        t, s = int(bt.t[b]), int(bt.s[b])
        G = exact[rt.lo[t]:rt.hi[t], rt.lo[s]:rt.hi[s]]
        if not G.any():
            continue
        err = np.linalg.norm(got[rt.lo[t]:rt.hi[t], rt.lo[s]:rt.hi[s]] - G, 2) / np.linalg.norm(G)
        worst = max(worst, err)
    assert 0.0 < worst <= 2 * (depth + 1) * eps, worst
