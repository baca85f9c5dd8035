"""Time h2_solve (one right-hand side; CUDA events) on the C2-shaped Cholesky factor of side N."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_1402_5056_b200 as P
from inputs import config

N = int(sys.argv[1]) if len(sys.argv) > 1 else 256
c = config("C2", N=N)
n = c["n"]
t = P.h2_cluster_tree(c["points"], c["leaf"])
bt = P.h2_block_tree(t, t, c["eta"])
Z = P.h2_from_sparse(bt, c["A"], lower=True, rank_cap=32, update_cap=32)
P.h2_lr_factor(Z, cholesky=True, trunc=P.Trunc(1e-4))
x = torch.randn(n, dtype=torch.float64, device="cuda")
for _ in range(2):
    P.h2_solve(Z, x)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    P.h2_solve(Z, x)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(json.dumps({"N": N, "n": n, "leaves": n // 32, "solve_ms": ms, "us_per_leaf_per_sweep": ms * 1e3 / (2 * (n // 32))}))
