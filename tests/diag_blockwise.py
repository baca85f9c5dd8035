"""Diagnostic (test infrastructure; run from the repo root as python tests/diag_...py): oracle vs GPU Cholesky with the block-relative rule; prints rank statistics,
the first differing cluster and the device flags instead of asserting."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_1402_5056_b200 as P  # noqa: E402
from h2util import setup, operator_rel_diff  # noqa: E402
from oracle.arith import Arith  # noqa: E402
from oracle.update import Trunc  # noqa: E402

CASES = [("C2", 128, e, 32) for e in (5e-3, 7e-3, 9e-3, 1.1e-2, 2e-2, 5e-2)] + [("C2", 96, 1e-2, 32), ("C1", 128, 1e-2, 32),
                                                                                ("C1", 128, 5e-2, 32)]
for name, N, eps, cap in CASES:
    s = setup(name, N, lower=True, rank_cap=cap, update_cap=cap)
    ar = Arith(s["OZ"], Trunc(eps, blockwise=True))
    ar.chol()
    try:
        P.h2_lr_factor(s["Z"], cholesky=True, trunc=P.Trunc(eps, blockwise=True))
        err = None
    except P.H2Error as e:
        err = str(e)
    kr, kc = P.h2_ranks(s["Z"])
    ok, oc = s["OZ"].k, s["OZ"].l
    dr = np.nonzero(kr != ok)[0]
    dc = np.nonzero(kc != oc)[0]
    try:
        fl = P.h2_check_device_flags(s["Z"])
    except P.H2Error as e:
        fl = str(e)
    print(name, N, eps, cap, "err", err, "flags", fl, "oracle kmax", ok.max(), oc.max(), "gpu kmax", kr.max(), kc.max(),
          "row diffs", len(dr), dr[:5], kr[dr[:5]], ok[dr[:5]], "col diffs", len(dc), dc[:5], kc[dc[:5]], oc[dc[:5]],
          "stats", P.h2_stats(s["Z"]), ar.stats, flush=True)
    if err is None:
        print("   operator diff", operator_rel_diff(s["Z"], s["OZ"], s["ot"].n), flush=True)
