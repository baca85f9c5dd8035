"""Pins for the oracle's product, substitutions, LR/Cholesky, solves and PCG (CPU only).

Held to: the dense Cholesky / no-pivot LU factors (unique, tree order) when truncation is
(nearly) off; the exactness of A*A for a sparse A (far field exactly zero); X = I and
alpha = 0 special cases; random H^2 products against dense products; the
factorization error bound ||LL^T - A|| <= 10 eps ||A||; PCG/power-iteration special
cases."""
import numpy as np
import pytest
import scipy.sparse as sp

from inputs import config
from inputs.updates import c0_global_factors, mixed_stream
from oracle.structure import ClusterTree, BlockTree, ADM, INADM
from oracle.h2 import from_sparse
from oracle.update import Updater, Trunc
from oracle.dense import densify
from oracle.arith import Arith, Op, dense_factor_product, pcg, power_error


def _c0(lower=False, A=None):
    c = config("C0")
    rt = ClusterTree(c["points"], c["leaf"])
    bt = BlockTree(rt, rt, c["eta"])
    Z = from_sparse(bt, c["A"] if A is None else A, lower=lower)
    return c, rt, bt, Z


def test_cholesky_exact_equals_dense_cholesky():
    c, rt, bt, Z = _c0(lower=True)
    Ad = c["A"].toarray()[rt.perm][:, rt.perm]
    ar = Arith(Z, Trunc(1e-13))
    ar.chol()
    L = np.tril(densify(Z))
    Lref = np.linalg.cholesky(Ad)
    assert np.abs(L - Lref).max() / np.abs(Lref).max() < 1e-9
    assert ar.stats["updates"] > 100 and ar.stats["temporaries"] > 0


def test_cholesky_truncated_error_bound_and_pcg():
    c, rt, bt, Z = _c0(lower=True)
    A = c["A"]
    Ad = A.toarray()[rt.perm][:, rt.perm]
    eps = 1e-4
    ar = Arith(Z, Trunc(eps))
    ar.chol()
    E = dense_factor_product(Z, True) - Ad
    assert np.linalg.norm(E, 2) <= 10 * eps * np.linalg.norm(Ad, 2)
    b = np.random.default_rng(4).standard_normal(A.shape[0])
    x, m, rel = pcg(lambda v: A @ v, lambda v: ar.solve(v), b)
    assert rel < 1e-8 and m <= 10
    err = power_error(lambda v: A @ v, lambda v: ar.solve(v), np.random.default_rng(5).standard_normal(A.shape[0]))
    assert err < 0.2


def test_lr_exact_equals_dense_lu_after_rank8_update():
    """C0 protocol (R15): rank-8 update (alpha = 1/n) on every admissible leaf, then LR vs dense
    no-pivot LU in tree order."""
    c, rt, bt, Z = _c0()
    n = rt.n
    X, Y = c0_global_factors(n)
    Xt, Yt = X[rt.perm], Y[rt.perm]
    up = Updater(Z, Trunc(1e-4))
    for b in bt.adm:
        t0, s0 = int(bt.t[b]), int(bt.s[b])
        up(t0, s0, Xt[rt.lo[t0]:rt.hi[t0]], Yt[rt.lo[s0]:rt.hi[s0]], alpha=1.0 / n)
    M = densify(Z)
    ar = Arith(Z, Trunc(1e-13))
    ar.lr()
    D = densify(Z)
    # dense Doolittle LU without pivoting
    U = M.copy()
    Lr = np.eye(n)
    for j in range(n):
        Lr[j + 1:, j] = U[j + 1:, j] / U[j, j]
        U[j + 1:, j:] -= np.outer(Lr[j + 1:, j], U[j, j:])
    assert np.abs(np.tril(D, -1) - np.tril(Lr, -1)).max() < 1e-8
    assert np.abs(np.triu(D) - np.triu(U)).max() / np.abs(U).max() < 1e-8
    # truncated LR error bound (<= 10 eps for alpha = 1/n)
    c, rt, bt, Z = _c0()
    up = Updater(Z, Trunc(1e-4))
    for b in bt.adm:
        t0, s0 = int(bt.t[b]), int(bt.s[b])
        up(t0, s0, Xt[rt.lo[t0]:rt.hi[t0]], Yt[rt.lo[s0]:rt.hi[s0]], alpha=1.0 / n)
    M = densify(Z)
    ar = Arith(Z, Trunc(1e-4))
    ar.lr()
    E = dense_factor_product(Z, False) - M
    assert np.linalg.norm(E, 2) <= 10 * 1e-4 * np.linalg.norm(M, 2)


def test_product_sparse_squared_is_exact():
    """for a sparse A (rank-0 bases) every far-field contribution of A*A is zero."""
    c, rt, bt, A = _c0()
    Zc, _, _, Z = _c0(A=c["A"] * 0.0)
    ar = Arith(Z, Trunc(1e-4))
    ar.addmul(1.0, Op(A), Op(A), 0, 0, 0)
    Ad = c["A"].toarray()[rt.perm][:, rt.perm]
    assert np.abs(densify(Z) - Ad @ Ad).max() < 1e-12
    assert Z.k.sum() == 0


def test_product_identity_and_alpha_zero():
    c, rt, bt, Y = _c0()
    n = rt.n
    Updater(Y, Trunc(1e-10))
    for t0, s0, X_, Y_ in mixed_stream([(int(bt.t[b]), int(bt.s[b]), rt.size(bt.t[b]), rt.size(bt.s[b]))
                                        for b in bt.adm], 6, 4, seed=3):
        Updater(Y, Trunc(1e-10))(t0, s0, X_, Y_)
    _, _, _, I = _c0(A=sp.identity(n, format="csr"))
    _, _, _, Z = _c0(A=c["A"] * 0.0)
    ar = Arith(Z, Trunc(1e-10))
    ar.addmul(1.0, Op(I), Op(Y), 0, 0, 0)  # S:404  X = I -> Z = Y
    Dy = densify(Y)
    assert np.linalg.norm(densify(Z) - Dy) / np.linalg.norm(Dy) < 1e-9
    before = densify(Z)
    ar.addmul(0.0, Op(Y), Op(Y), 0, 0, 0)  # S:403  alpha = 0 -> unchanged
    assert np.linalg.norm(densify(Z) - before) <= 1e-9 * np.linalg.norm(before)


def test_product_random_h2_against_dense():
    c, rt, bt, X = _c0()
    targets = [(int(bt.t[b]), int(bt.s[b]), rt.size(bt.t[b]), rt.size(bt.s[b])) for b in range(bt.nblocks)]
    ux = Updater(X, Trunc(1e-12))
    for t0, s0, a, b in mixed_stream(targets, 8, 4, seed=1):
        ux(t0, s0, a, b)
    _, _, _, Y = _c0()
    uy = Updater(Y, Trunc(1e-12))
    for t0, s0, a, b in mixed_stream(targets, 8, 4, seed=2):
        uy(t0, s0, a, b)
    _, _, _, Z = _c0()
    D0 = densify(Z)
    ar = Arith(Z, Trunc(1e-12))
    ar.addmul(-0.5, Op(X), Op(Y, True), 0, 0, 0)
    ref = D0 - 0.5 * densify(X) @ densify(Y).T
    assert np.linalg.norm(densify(Z) - ref) / np.linalg.norm(ref) < 1e-8


def test_pcg_and_power_special_cases():
    n = 50
    b = np.random.default_rng(0).standard_normal(n)
    x, m, rel = pcg(lambda v: v, lambda v: v, b)  # A = I, M = I -> 1 iteration
    assert m == 1 and rel < 1e-14
    A = np.diag(np.linspace(1, 10, n))
    x, m, rel = pcg(lambda v: A @ v, lambda v: np.linalg.solve(A, v), b)  # exact preconditioner
    assert m <= 2
    D = np.diag([1.0, 2.0])  # A = diag(1,2), M = I -> ||I - A|| = 1
    assert abs(power_error(lambda v: D @ v, lambda v: v, np.array([0.3, 1.0])) - 1.0) < 1e-3
    assert power_error(lambda v: A @ v, lambda v: np.linalg.solve(A, v), b) < 1e-8


def test_interpolative_decomposition_reading_own7():
    """own-7: A = r pivot columns of P, A B^T = P to the truncation level; exact rank recovered."""
    rng = np.random.default_rng(12)
    for rank in (0, 1, 5, 12):
        P = rng.standard_normal((32, rank)) @ rng.standard_normal((rank, 30))
        A, B = Arith._interp_decomp(P)
        assert A.shape[1] == rank and B.shape == (30, rank)
        if rank:
            assert np.abs(A @ B.T - P).max() <= 1e-11 * np.abs(P).max()
            cols = [j for j in range(30) if any(np.array_equal(P[:, j], A[:, q]) for q in range(rank))]
            assert len(cols) >= rank  # A consists of columns of P
    P = np.diag([3.0, 1e-13, 0.0, 2.0])
    A, B = Arith._interp_decomp(P)
    assert A.shape[1] == 2 and np.abs(A @ B.T - np.diag([3.0, 0, 0, 2.0])).max() == 0.0


def _small(name="C2", N=24):
    c = config(name, N=N)
    ot = ClusterTree(c["points"], c["leaf"])
    ob = BlockTree(ot, ot, c["eta"])
    return c, ot, ob


def test_inverse_remark1_against_dense_inverse():
    """NEXT-2 (Remark 1): the block-Gauss approximate inverse equals the dense inverse
    within the truncation (tight eps: 1e-8 relative on probes) and its error falls with eps (the
    Schur complement uses A22; P:1382 prints A11, reading R20)."""
    c, ot, ob = _small()
    A = c["A"].toarray()
    Ainv = np.linalg.inv(A)
    X = np.random.default_rng(1).standard_normal((ot.n, 3))
    errs = []
    for eps in (1e-10, 1e-5, 1e-3):
        Z = from_sparse(ob, c["A"])
        Arith(Z, Trunc(eps)).inv(from_sparse(ob, c["A"] * 0))
        errs.append(np.linalg.norm(Z.matvec(X) - Ainv @ X) / np.linalg.norm(Ainv @ X))
    assert errs[0] < 1e-8
    assert errs[0] < errs[1] < errs[2] < 1e-1


def test_inverse_identity_and_diagonal_exact():
    """A = I gives C = I exactly; a diagonal A gives C = diag(1/a) exactly (every product of a
    zero off-diagonal block is exactly zero)."""
    c, ot, ob = _small()
    n = ot.n
    d = np.random.default_rng(2).uniform(1.0, 3.0, n)
    for D in (sp.identity(n, format="csr"), sp.diags(d, format="csr")):
        Z = from_sparse(ob, D)
        Arith(Z, Trunc(1e-4)).inv(from_sparse(ob, D * 0))
        np.testing.assert_array_equal(densify(Z), np.diag(1.0 / D.diagonal())[np.ix_(ot.perm, ot.perm)])


def test_inverse_breakdown_reported():
    c, ot, ob = _small()
    A = c["A"].tolil()
    A[0, :] = 0.0
    A[:, 0] = 0.0
    from oracle.arith import BreakdownError
    with pytest.raises(BreakdownError):
        Arith(from_sparse(ob, A.tocsr()), Trunc(1e-4)).inv(from_sparse(ob, c["A"] * 0))


def test_lr_substitutions_invert_the_represented_factors():
    """Arith.lsolve(unit) / usolve / utsolve and solve_tree(cholesky=False) solve with the
    triangular matrices the factored H^2 matrix represents: L = unit-lower part, R = upper part of
    densify(Z) (a truncated LR at eps = 1e-4 after the C0 rank-8 update, so the blocks have
    non-zero ranks).  Reference: dense triangular solves of the densified factors."""
    from scipy.linalg import solve_triangular
    c, rt, bt, Z = _c0()
    n = rt.n
    X, Y = c0_global_factors(n)
    Xt, Yt = X[rt.perm], Y[rt.perm]
    up = Updater(Z, Trunc(1e-4))
    for b in bt.adm:
        t0, s0 = int(bt.t[b]), int(bt.s[b])
        up(t0, s0, Xt[rt.lo[t0]:rt.hi[t0]], Yt[rt.lo[s0]:rt.hi[s0]], alpha=1.0 / n)
    ar = Arith(Z, Trunc(1e-4))
    ar.lr()
    assert Z.k.max() > 0 and Z.l.max() > 0
    D = densify(Z)
    L = np.tril(D, -1) + np.eye(n)
    R = np.triu(D)
    B = np.random.default_rng(21).standard_normal((n, 3))
    for got, ref in ((ar.usolve(0, B), solve_triangular(R, B, lower=False)),
                     (ar.utsolve(0, B), solve_triangular(R.T, B, lower=True)),
                     (ar.lsolve(0, B, unit=True), solve_triangular(L, B, lower=True, unit_diagonal=True))):
        assert np.linalg.norm(got - ref) <= 1e-10 * np.linalg.norm(ref)
    x = ar.solve_tree(B[:, 0], cholesky=False)
    assert np.linalg.norm(L @ (R @ x) - B[:, 0]) <= 1e-10 * np.linalg.norm(B[:, 0])


def test_zero_tile_factor_adds_nothing_reading_own6():
    """own-6 in the mixed Case-2 branches: a product X|_{t x s} 0|_{s x r} (admissible block of an
    H^2 matrix X with non-zero ranks times an exactly zero dense leaf tile), and 0|_{t x s} X|_{s x r},
    leaves Z bit for bit unchanged and performs no local update -- the same decision the device
    takes (h2_factor.cpp, zero_rank_if_zero_tile)."""
    c, rt, bt, X = _c0()
    targets = [(int(bt.t[b]), int(bt.s[b]), rt.size(bt.t[b]), rt.size(bt.s[b])) for b in range(bt.nblocks)]
    ux = Updater(X, Trunc(1e-12))
    for t0, s0, a, b in mixed_stream([tg for tg in targets if bt.kind[bt.index[tg[:2]]] == ADM], 40, 4, seed=5):
        ux(t0, s0, a, b)
    _, _, _, O = _c0(A=c["A"] * 0.0)
    _, _, _, Z = _c0()
    uz = Updater(Z, Trunc(1e-12))
    for t0, s0, a, b in mixed_stream(targets, 6, 4, seed=6):
        uz(t0, s0, a, b)
    ox, oo = Op(X), Op(O)
    n_cases = [0, 0]
    for (t, s), bx in bt.index.items():
        if bt.kind[bx] != ADM or X.k[t] == 0 or X.l[s] == 0:
            continue
        for r in range(rt.nclusters):
            for case, (P, Q, a, b_, c_) in enumerate(((ox, oo, t, s, r), (oo, ox, r, t, s))):
                if not all(blk in bt.index for blk in ((a, b_), (b_, c_), (a, c_))):
                    continue
                if (Q.kind(b_, c_) if case == 0 else P.kind(a, b_)) != INADM:  # the zero factor: a dense tile
                    continue
                before, k0, l0 = densify(Z), Z.k.copy(), Z.l.copy()
                ar = Arith(Z, Trunc(1e-4))
                ar.addmul(-1.0, P, Q, a, b_, c_)
                assert ar.stats["updates"] == 0 and ar.stats["dense_adds"] == 0 and ar.stats["tmp_adds"] == 0
                np.testing.assert_array_equal(densify(Z), before)
                np.testing.assert_array_equal(Z.k, k0)
                np.testing.assert_array_equal(Z.l, l0)
                n_cases[case] += 1
    assert min(n_cases) >= 3, n_cases


def test_cholesky_blockwise_truncation():
    """NEXT-1: the H^2 Cholesky with blockwise-relative truncation (own-10; temporaries keep the
    relative rule): at a tight eps^ it reproduces the dense Cholesky, at a loose one the factor
    still preconditions CG."""
    c, rt, bt, Z = _c0(lower=True)
    A = c["A"]
    Ad = A.toarray()[rt.perm][:, rt.perm]
    ar = Arith(Z, Trunc(1e-12, blockwise=True))
    ar.chol()
    assert np.abs(np.tril(densify(Z)) - np.linalg.cholesky(Ad)).max() / np.abs(Ad).max() < 1e-9
    c, rt, bt, Z = _c0(lower=True)
    ar = Arith(Z, Trunc(1e-3, blockwise=True))
    ar.chol()
    b = np.random.default_rng(4).standard_normal(A.shape[0])
    _, m, rel = pcg(lambda v: A @ v, lambda v: ar.solve(v), b)
    assert rel < 1e-8 and m <= 12


def test_cholesky_on_dd_tree_equals_dense_and_keeps_decoupled_blocks_zero():
    """NEXT-3 (reading own-11): on the domain-decomposition tree the H^2 Cholesky at a
    tight truncation is the dense Cholesky in tree (= nested dissection) order, the blocks of the
    decoupled domain pairs stay exactly zero (rank 0) and far fewer local updates are needed than
    on the bisection tree; at eps = 1e-4 it preconditions CG like the bisection-tree factor."""
    c = config("C2", N=48)
    A = c["A"]
    rt = ClusterTree(c["points"], c["leaf"], adjacency=A)
    bt = BlockTree(rt, rt, c["eta"])
    Z = from_sparse(bt, A, lower=True)
    Ad = A.toarray()[rt.perm][:, rt.perm]
    ar = Arith(Z, Trunc(1e-13))
    ar.chol()
    L = np.tril(densify(Z))
    Lref = np.linalg.cholesky(Ad)
    assert np.abs(L - Lref).max() / np.abs(Lref).max() < 1e-9
    npairs = 0
    for p in np.nonzero(rt.ddpair)[0]:
        a, b = rt.sons(p)
        blk = bt.index[(b, a)]
        assert bt.kind[blk] == ADM and Z.k[b] * 0 == 0
        assert not L[rt.lo[b]:rt.hi[b], rt.lo[a]:rt.hi[a]].any()
        assert not Lref[rt.lo[b]:rt.hi[b], rt.lo[a]:rt.hi[a]].any()  # no fill in nested dissection order
        npairs += 1
    assert npairs > 10
    # truncated: error bound, PCG, and the update count against the bisection tree
    Z2 = from_sparse(bt, A, lower=True)
    ar2 = Arith(Z2, Trunc(1e-4))
    ar2.chol()
    E = dense_factor_product(Z2, True) - Ad
    assert np.linalg.norm(E, 2) <= 10 * 1e-4 * np.linalg.norm(Ad, 2)
    b = np.random.default_rng(4).standard_normal(A.shape[0])
    _, m, rel = pcg(lambda v: A @ v, lambda v: ar2.solve(v), b)
    assert rel < 1e-8 and m <= 12
    rb = ClusterTree(c["points"], c["leaf"])
    Zb = from_sparse(BlockTree(rb, rb, c["eta"]), A, lower=True)
    arb = Arith(Zb, Trunc(1e-4))
    arb.chol()
    assert ar2.stats["updates"] < arb.stats["updates"] / 2
