"""NEXT-4 (Table 2; reading own-12): the boundary element workload -- the Galerkin
matrix of the single layer potential on a circle -- compressed into an H^2 matrix by the paper's
own tool, one local low-rank update per admissible leaf, then factored and used in PCG.

CPU part: pins of the workload generator (closed series vs direct quadrature, circulant structure,
positive definiteness, the radius-1 singularity that motivates the reading) and of the oracle on
it (H^2 matrix built by local updates = dense Galerkin matrix to the interpolation/truncation
accuracy; Cholesky; PCG).  GPU part: the same build through the C ABI against the oracle."""
import numpy as np
import pytest
from scipy import integrate

from inputs import bem
from inputs.rng import stream, RHS
from oracle.structure import ClusterTree, BlockTree
from oracle.h2 import from_sparse
from oracle.update import Updater, Trunc
from oracle.dense import densify
from oracle.arith import Arith, pcg


def _oracle_build(n, eps, lower=False, leaf=32, eta=2.0, bw=False):
    ot = ClusterTree(bem.circle_points(n), leaf)
    ob = BlockTree(ot, ot, eta)
    A_near, far = bem.pieces(n, ot.perm, ot.lo, ot.hi, ob.t, ob.s, ob.kind, lower=lower)
    Z = from_sparse(ob, A_near, lower=lower)
    up = Updater(Z, Trunc(eps, blockwise=bw))
    for t, s, X, Y in far:
        up(t, s, X, Y)
    return ot, ob, Z, A_near, far


def test_bem_generator_pins():
    n = 64
    g = bem.first_row(n)
    G = bem.dense_matrix(n)
    h, R = 2 * np.pi / n, bem.R
    # the folded series against direct adaptive quadrature of the definition (smooth entries)
    for d in (2, 7, 31):
        f = lambda v, u: -(R * R / (2 * np.pi)) * (np.log(R) + np.log(2 * abs(np.sin((d * h + u - v) / 2))))  # noqa: E731
        assert abs(g[d] - integrate.dblquad(f, 0, h, 0, h, epsabs=1e-14, epsrel=1e-12)[0]) < 1e-15
    # the singular diagonal entry against the unfolded series
    m = np.arange(1, 400001)
    d0 = R * R * (-h * h * np.log(R) / (2 * np.pi) + (2 / np.pi) * np.sum(np.sin(m * h / 2) ** 2 / m ** 3))
    assert abs(g[0] - d0) <= R * R / (np.pi * 400000.0 ** 2)  # the tail of the unfolded series (terms <= 1/m^3)
    # symmetric circulant, positive definite; eigenvalue of the constants = -n h^2 R^2 log(R) / (2 pi)
    assert np.abs(G - G.T).max() < 1e-18 and np.allclose(G[3], np.roll(G[0], 3))
    ev = np.linalg.eigvalsh(G)
    assert ev[0] > 0
    assert abs(np.ones(n) @ G @ np.ones(n) / n + n * h * h * R * R * np.log(R) / (2 * np.pi)) < 1e-15
    # degenerate-kernel factors of separated arc ranges (also across the wrap at 2 pi)
    for rows, cols in ((np.arange(0, 8), np.arange(24, 40)), (np.array([62, 63, 0, 1]), np.arange(20, 30))):
        X, Y = bem.far_factors(n, rows, cols)
        ref = G[np.ix_(rows, cols)]
        assert np.abs(X @ Y.T - ref).max() < 1e-12 * np.abs(ref).max()


def test_bem_h2_by_local_updates_matches_dense_oracle():
    """The oracle's H^2 matrix, built from the nearfield entries by one local update per admissible
    leaf, is the dense Galerkin matrix up to the truncation; its Cholesky
    factorization preconditions CG."""
    n = 512
    G = bem.dense_matrix(n)
    errs = []
    for eps in (1e-4, 1e-8):
        ot, ob, Z, _, far = _oracle_build(n, eps)
        D = densify(Z)
        Gt = G[ot.perm][:, ot.perm]
        errs.append(np.linalg.norm(D - Gt, 2) / np.linalg.norm(Gt, 2))
    assert errs[0] < 10 * 1e-4 and errs[1] < 1e-7 and errs[1] < errs[0]
    assert len(far) > 100 and Z.k.max() <= 12
    # Cholesky of the lower-stored H^2 matrix + PCG on the dense operator
    ot, ob, ZL, _, _ = _oracle_build(n, 1e-6, lower=True)
    ar = Arith(ZL, Trunc(1e-6))
    ar.chol()
    b = stream(RHS).standard_normal(n)
    x, m, rel = pcg(lambda v: G @ v, lambda v: ar.solve(v), b)
    assert rel < 1e-8 and m <= 4
    assert np.linalg.norm(G @ x - b) <= 1e-7 * np.linalg.norm(b)


# ---- GPU parity ------------------------------------------------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("n,eps,bw", [(1024, 1e-6, False), (2048, 1e-4, False), (2048, 2.4e-4, True)])
def test_bem_gpu_parity(n, eps, bw):
    """The last case is the paper's own setting (Table 2: eta = 2, block-relative eps^ ~ h,
    P:1461-1481, here eps^ = 1.2e-4 * 8192 / n)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1402_5056_b200 as P
    from h2util import operator_rel_diff

    def _t(a):
        return torch.from_numpy(np.ascontiguousarray(a)).cuda()

    pts = bem.circle_points(n)
    t = P.h2_cluster_tree(pts, 32)
    bt = P.h2_block_tree(t, t, 2.0)
    tr = P.Trunc(eps, blockwise=bw)
    mats = {}
    for lower in (False, True):
        ot, ob, OZ, A_near, far = _oracle_build(n, eps, lower=lower, bw=bw)
        np.testing.assert_array_equal(t.perm, ot.perm)
        np.testing.assert_array_equal(bt.kind, ob.kind)
        Z = P.h2_from_sparse(bt, A_near, lower=lower, rank_cap=32, update_cap=32)
        keep = [P.h2_lowrank_update(Z, t0, s0, _t(X), _t(Y), trunc=tr) for t0, s0, X, Y in far]
        kr, kc = P.h2_ranks(Z)
        np.testing.assert_array_equal(kr, OZ.k)
        np.testing.assert_array_equal(kc, OZ.l)
        assert P.h2_check_device_flags(Z) == 0
        d = operator_rel_diff(Z, OZ, n)
        assert d <= 10 * eps
        mats[lower] = (Z, OZ, d)
        del keep
    # the compressed operator against the dense Galerkin matrix (full storage)
    G = bem.dense_matrix(n)
    x = np.random.default_rng(2).standard_normal(n)
    y = P.h2_matvec(mats[False][0], _t(x)).cpu().numpy()
    assert np.linalg.norm(y - G @ x) <= 10 * eps * np.linalg.norm(G @ x)
    # Cholesky of the lower-stored copy on both sides, PCG with the H^2 operator
    ZL, OZL, _ = mats[True]
    ar = Arith(OZL, Trunc(eps, blockwise=bw))
    ar.chol()
    P.h2_lr_factor(ZL, cholesky=True, trunc=tr)
    assert P.h2_check_device_flags(ZL) == 0
    kr, kc = P.h2_ranks(ZL)
    np.testing.assert_array_equal(kr, OZL.k)
    np.testing.assert_array_equal(kc, OZL.l)
    dL = operator_rel_diff(ZL, OZL, n)
    b = stream(RHS).standard_normal(n)
    _, m_o, _ = pcg(lambda v: G @ v, lambda v: ar.solve(v), b)
    xg = _t(np.zeros(n))
    _, m_g, rel = P.h2_pcg(mats[False][0], ZL, _t(b), xg, tol=1e-8)
    print(f"BEM n={n} eps={eps}: build diff {mats[False][2]:.2e}/{mats[True][2]:.2e}, factor diff {dL:.2e}, "
          f"max rank {OZL.k.max()}, PCG m gpu {m_g} oracle {m_o}")
    assert dL <= 10 * eps and rel < 1e-8 and abs(m_g - m_o) <= 1


@pytest.mark.gpu
def test_update_capacity_overrun_is_reported():
    """A contribution inside the factorization whose rank exceeds update_cap (a dense x dense product
    of 32-point leaves can reach rank 32, reading own-7) is dropped and reported (flag bit 2,
    H2_ERR_NOMEM), not written past the extended-rank workspace."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1402_5056_b200 as P

    n, eps = 1024, 1e-6
    t = P.h2_cluster_tree(bem.circle_points(n), 32)
    bt = P.h2_block_tree(t, t, 2.0)
    A_near, far = bem.pieces(n, t.perm, t.lo, t.hi, bt.t, bt.s, bt.kind, lower=True)
    Z = P.h2_from_sparse(bt, A_near, lower=True, rank_cap=32, update_cap=16)
    keep = [P.h2_lowrank_update(Z, t0, s0, torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda(), trunc=P.Trunc(eps))
            for t0, s0, X, Y in far]
    assert P.h2_check_device_flags(Z) == 0
    P.h2_lr_factor(Z, cholesky=True, trunc=P.Trunc(eps))
    with pytest.raises(P.H2Error) as e:
        P.h2_check_device_flags(Z)
    assert e.value.status == "H2_ERR_NOMEM" and "update_cap" in str(e.value)
    del keep
