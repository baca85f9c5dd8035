"""Sensitivity of the C1 protocol itself (DESIGN own-9): two ORACLE runs of the same 10,000-update
fixed-rank-16 chain whose inputs differ by one ulp in a single entry of the first update's X.
Prints the relative operator difference between the two oracle matrices (16 seeded probes) and
whether the ranks agree at every 1,000-update checkpoint.  A difference that grows like the
GPU-vs-oracle drift shows the amplification belongs to the truncation, not to either
implementation.  Imports oracle/ and inputs/ only.

    python tools/c1_drift_oracle.py [k_u]
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from inputs import config  # noqa: E402
from inputs.rng import probes  # noqa: E402
from inputs.updates import c1_stream  # noqa: E402
from oracle.structure import ClusterTree, BlockTree  # noqa: E402
from oracle.h2 import from_sparse  # noqa: E402
from oracle.update import Updater, Trunc  # noqa: E402


def main():
    ku = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    c = config("C1")
    ot = ClusterTree(c["points"], c["leaf"])
    ob = BlockTree(ot, ot, c["eta"])
    tg = [(int(ob.t[b]), int(ob.s[b]), ot.size(ob.t[b]), ot.size(ob.s[b])) for b in ob.adm]
    ups = c1_stream(tg, 10000, ku, seed=0)
    Z1, Z2 = from_sparse(ob, c["A"]), from_sparse(ob, c["A"])
    u1, u2 = Updater(Z1, Trunc(1e-12, 0.0, 16)), Updater(Z2, Trunc(1e-12, 0.0, 16))
    Xp = probes(ot.n, 16).T
    out = []
    for i, (t0, s0, X, Y) in enumerate(ups):
        u1(t0, s0, X, Y)
        if i == 0:
            X = X.copy()
            X[0, 0] = np.nextafter(X[0, 0], np.inf)  # one ulp
        u2(t0, s0, X, Y)
        if (i + 1) % 1000 == 0:
            y1, y2 = Z1.matvec(Xp), Z2.matvec(Xp)
            out.append(dict(updates=i + 1, rel_diff=float(np.linalg.norm(y1 - y2) / np.linalg.norm(y1)),
                            ranks_equal=bool((Z1.k == Z2.k).all() and (Z1.l == Z2.l).all())))
            print(json.dumps(out[-1]), flush=True)
    print(json.dumps({"k_u": ku, "checkpoints": out}))


if __name__ == "__main__":
    main()
