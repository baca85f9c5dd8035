"""Diagnostic (test infrastructure; run from the repo root as python tests/diag_...py): the sequence of non-zero-rank local updates (t0, s0, k) of the GPU Cholesky
(H2_UPD_LOG) against the oracle's, on the DD tree; prints the first difference."""
import os
import sys

import numpy as np

os.environ["H2_UPD_LOG"] = "/tmp/h2_updlog.txt"
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_1402_5056_b200 as P  # noqa: E402
from h2util import setup  # noqa: E402
from oracle.arith import Arith  # noqa: E402
from oracle.update import Trunc  # noqa: E402

name, N, dd = sys.argv[1], int(sys.argv[2]), sys.argv[3] == "dd"
s = setup(name, N, lower=True, dd=dd)
ar = Arith(s["OZ"], Trunc(1e-4))
orig = ar.up
seq = []


def rec(t, r, A, B, **k):
    seq.append((t, r, A.shape[1], int(s["OZ"].k[t]), int(s["OZ"].l[r]), float(np.abs(A).max()), float(np.abs(B).max())))
    return orig(t, r, A, B, **k)


ar.up = rec
last = {}
of = ar._factors


def fac(X, Y, t, s_, r, dense_target=False):
    A, B = of(X, Y, t, s_, r, dense_target)
    last.update(kx=int(X.kind(t, s_)), ky=int(Y.kind(s_, r)), t=t, s=s_, r=r, k=A.shape[1])
    return A, B


ar._factors = fac
info = []
orig_rec = rec


def rec2(t, r, A, B, **k):
    info.append(dict(last))
    return orig_rec(t, r, A, B, **k)


ar.up = rec2
ar.chol()
P.h2_lr_factor(s["Z"], cholesky=True, trunc=P.Trunc(1e-4))
P.h2_check_device_flags(s["Z"])
g = [tuple(int(v) for v in l.split()) for l in open("/tmp/h2_updlog.txt")]
print(name, N, "oracle", len(seq), "gpu", len(g))
i = 0
while i < min(len(seq), len(g)) and seq[i][:5] == g[i]:
    i += 1
print("first difference at", i, "oracle", seq[i - 1:i + 3], "gpu", g[i - 1:i + 3])
ot, ob = s["ot"], s["ob"]
if i < len(seq):
    print("last Case-2 factor call before the oracle's update:", info[i], "(kind 1 = admissible, 2 = inadmissible)")
    t, r = seq[i][0], seq[i][1]
    print("oracle update target", t, r, "sizes", ot.size(t), ot.size(r), "kind", ob.kind[ob.index[(t, r)]], "leaf", ot.is_leaf(t), ot.is_leaf(r))
