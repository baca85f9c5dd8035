"""Time h2_matvec (CUDA events, median of back-to-back calls) on C2-shaped matrices of side N:
the sparse input A (rank-0 H^2 form) and, with "factor", the Cholesky factor L. GB/s uses the
algorithmic bytes 8 * (stored scalars) + 16 n."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_1402_5056_b200 as P
from inputs import config

N = int(sys.argv[1]) if len(sys.argv) > 1 else 256
do_factor = "factor" in sys.argv[2:]
c = config("C2", N=N)
n = c["n"]
t = P.h2_cluster_tree(c["points"], c["leaf"])
bt = P.h2_block_tree(t, t, c["eta"])
dev = torch.device("cuda", 0)


def time_mv(Z, reps=50, transpose=False):
    x = torch.randn(n, dtype=torch.float64, device=dev)
    y = torch.empty_like(x)
    for _ in range(3):
        P.h2_matvec(Z, x, y, transpose=transpose)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for e0, e1 in evs:
        e0.record()
        P.h2_matvec(Z, x, y, transpose=transpose)
        e1.record()
    torch.cuda.synchronize()
    ts = sorted(e0.elapsed_time(e1) for e0, e1 in evs)
    ms = ts[len(ts) // 2]
    byt = 8.0 * float(P.h2_storage_report(Z).sum()) + 16.0 * n
    return dict(ms=ms, MB=byt / 1e6, GBps=byt / ms / 1e6)


out = {"N": N, "n": n}
A = P.h2_from_sparse(bt, c["A"], lower=False)
out["A"] = time_mv(A)
out["A_T"] = time_mv(A, transpose=True)
if do_factor:
    Z = P.h2_from_sparse(bt, c["A"], lower=True, rank_cap=32, update_cap=32)
    P.h2_lr_factor(Z, cholesky=True, trunc=P.Trunc(1e-4))
    torch.cuda.synchronize()
    out["L"] = time_mv(Z)
print(json.dumps(out))
