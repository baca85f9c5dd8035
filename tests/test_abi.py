"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/h2.h declares,
validates arguments, and its host structure code (cluster tree, block tree) is bit-exact with
the oracle (SURVEY §8(c).4 "structure ... bit-exact").  No compute calls need a GPU here."""
import os
import re
import ctypes

import numpy as np
import pytest

from inputs import config, grid_points_2d, grid_points_3d
from oracle.structure import ClusterTree, BlockTree

P = pytest.importorskip("paper_1402_5056_b200")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_header_symbols_exported():
    hdr = open(os.path.join(ROOT, "include", "h2.h")).read()
    declared = set(re.findall(r"^\s*(?:h2_status|void|const char\*)\s+(h2_\w+)\s*\(", hdr, re.M))
    assert declared == set(P.EXPORTED_SYMBOLS)
    lib = ctypes.CDLL(P.library_path())
    for name in declared:
        assert hasattr(lib, name), name


@pytest.mark.parametrize("name,N", [("C0", None), ("C1", None), ("C2", 64), ("C3", 8)])
def test_structure_bit_exact_vs_oracle(name, N):
    c = config(name, N=N)
    t = P.h2_cluster_tree(c["points"], c["leaf"])
    bt = P.h2_block_tree(t, t, c["eta"])
    ot = ClusterTree(c["points"], c["leaf"])
    ob = BlockTree(ot, ot, c["eta"])
    np.testing.assert_array_equal(t.perm, ot.perm)
    for a, b in ((t.lo, ot.lo), (t.hi, ot.hi), (t.son0, ot.son0), (t.son1, ot.son1), (t.level, ot.level)):
        np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(bt.t, ob.t)
    np.testing.assert_array_equal(bt.s, ob.s)
    np.testing.assert_array_equal(bt.kind, ob.kind)
    assert bt.csp == ob.sparsity()


def test_structure_irregular_points_bit_exact():
    rng = np.random.default_rng(9)
    pts = rng.integers(0, 50, size=(700, 2)).astype(float)
    for leaf, eta in ((16, 2.0), (7, 1.0)):
        t = P.h2_cluster_tree(pts, leaf)
        ot = ClusterTree(pts, leaf)
        np.testing.assert_array_equal(t.perm, ot.perm)
        bt = P.h2_block_tree(t, t, eta)
        ob = BlockTree(ot, ot, eta)
        np.testing.assert_array_equal(bt.kind, ob.kind)
        np.testing.assert_array_equal(bt.t, ob.t)


@pytest.mark.parametrize("name,N", [("C1", 63), ("C2", 96), ("C3", 10)])
def test_dd_structure_bit_exact_vs_oracle(name, N):
    """Domain-decomposition cluster tree (NEXT-3, reading own-11) and its block tree."""
    c = config(name, N=N)
    t = P.h2_cluster_tree_dd(c["points"], c["leaf"], c["A"])
    bt = P.h2_block_tree(t, t, c["eta"])
    ot = ClusterTree(c["points"], c["leaf"], adjacency=c["A"])
    ob = BlockTree(ot, ot, c["eta"])
    np.testing.assert_array_equal(t.perm, ot.perm)
    for a, b in ((t.lo, ot.lo), (t.hi, ot.hi), (t.son0, ot.son0), (t.son1, ot.son1), (t.level, ot.level),
                 (t.ddpair, ot.ddpair)):
        np.testing.assert_array_equal(a, b)
    assert t.ddpair.sum() > 0
    np.testing.assert_array_equal(bt.t, ob.t)
    np.testing.assert_array_equal(bt.s, ob.s)
    np.testing.assert_array_equal(bt.kind, ob.kind)


def test_dd_structure_irregular_graph_bit_exact():
    import scipy.sparse as sp
    rng = np.random.default_rng(5)
    pts = rng.integers(0, 80, size=(900, 2)).astype(float)
    d2 = ((pts[:, None, :] - pts[None, :, :]) ** 2).sum(-1)
    nb = np.argsort(d2, axis=1, kind="stable")[:, :4]
    A = sp.csr_matrix((np.ones(nb.size), (np.repeat(np.arange(900), 4), nb.ravel())), shape=(900, 900))
    t = P.h2_cluster_tree_dd(pts, 12, A)
    ot = ClusterTree(pts, 12, adjacency=A)
    np.testing.assert_array_equal(t.perm, ot.perm)
    np.testing.assert_array_equal(t.ddpair, ot.ddpair)
    bt = P.h2_block_tree(t, t, 1.5)
    ob = BlockTree(ot, ot, 1.5)
    np.testing.assert_array_equal(bt.kind, ob.kind)
    np.testing.assert_array_equal(bt.t, ob.t)


def test_argument_errors():
    with pytest.raises(P.H2Error) as e:
        P.h2_cluster_tree(np.zeros((0, 2)), 4)
    assert e.value.status == "H2_ERR_ARG"
    with pytest.raises(P.H2Error) as e:
        P.h2_cluster_tree(np.array([[0.0, np.nan]]), 4)
    assert e.value.status == "H2_ERR_NONFINITE"
    t = P.h2_cluster_tree(grid_points_2d(8), 4)
    with pytest.raises(P.H2Error) as e:
        P.h2_block_tree(t, t, -1.0)
    assert e.value.status == "H2_ERR_ARG"
