"""Per-phase cycle breakdown of the substitution sweep (k_sweep) on the C2-shaped Cholesky factor of side N:
   python tools/sweep_profile.py 256"""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1402_5056_b200 as P
from paper_1402_5056_b200 import h2 as H
from inputs import config
c = config("C2", N=int(sys.argv[1]))
t = P.h2_cluster_tree(c["points"], c["leaf"]); bt = P.h2_block_tree(t, t, c["eta"])
Z = P.h2_from_sparse(bt, c["A"], lower=True, rank_cap=32, update_cap=32)
P.h2_lr_factor(Z, cholesky=True, trunc=P.Trunc(1e-4))
x = torch.randn(c["n"], dtype=torch.float64, device="cuda")
P.h2_solve(Z, x); torch.cuda.synchronize()
P.h2_profile_enable(True)
P.h2_solve(Z, x); torch.cuda.synchronize()
ns = np.zeros(64); cnt = np.zeros(64)
H._check(H._lib.h2_profile_ops(H._ptr(ns), H._ptr(cnt), 64, None))
names = ["enter || near", "residual", "diag solve", "done/push"]
tot = ns[40:44].sum()
for i in range(4):
    print(f"{names[i]:16s} cycles/leaf-step {ns[40+i]/max(cnt[40+i],1):8.0f}  share {ns[40+i]/tot*100:5.1f}%")
