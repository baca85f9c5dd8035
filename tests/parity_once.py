"""One Cholesky parity check outside pytest (test infrastructure): oracle vs GPU on config NAME at side N and
truncation eps: ranks, device flags, non-zero update counts, operator difference on 16 probes.

    python tests/parity_once.py NAME N eps [rank_cap]
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))  # tests/ -> repo root
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1402_5056_b200 as P  # noqa: E402
from h2util import setup, operator_rel_diff  # noqa: E402
from oracle.arith import Arith, BreakdownError  # noqa: E402
from oracle.update import Trunc  # noqa: E402

name, N, eps = sys.argv[1], int(sys.argv[2]), float(sys.argv[3])
cap = int(sys.argv[4]) if len(sys.argv) > 4 else 32
s = setup(name, N, lower=True, rank_cap=cap, update_cap=cap)
OZ, Z = s["OZ"], s["Z"]
t0 = time.perf_counter()
ar = Arith(OZ, Trunc(eps))
try:
    ar.chol()
    ob = "ok"
except BreakdownError as e:
    ob = str(e)
t1 = time.perf_counter()
P.h2_lr_factor(Z, cholesky=True, trunc=P.Trunc(eps))
torch.cuda.synchronize()
t2 = time.perf_counter()
try:
    flags = P.h2_check_device_flags(Z)
except P.H2Error as e:
    flags = str(e)
kr, kc = P.h2_ranks(Z)
out = dict(name=name, N=N, eps=eps, oracle=ob, oracle_s=round(t1 - t0, 1), gpu_s=round(t2 - t1, 2), flags=flags,
           ranks_equal=bool((kr == OZ.k).all() and (kc == OZ.l).all()),
           nz=[P.h2_stats(Z)["updates_nonzero"], ar.stats["updates"]], maxrank=[int(kr.max()), int(kc.max())])
if ob == "ok" and flags == 0:
    out["op_rel_diff"] = operator_rel_diff(Z, OZ, s["ot"].n)
print(json.dumps(out))
