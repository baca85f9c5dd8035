"""Time the GPU H^2 Cholesky on a C2-shaped problem of side N; per-kernel breakdown (profiling hook)."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1402_5056_b200 as P
from inputs import config

N = int(sys.argv[1]) if len(sys.argv) > 1 else 128
prof = len(sys.argv) > 2 and sys.argv[2] == "prof"
c = config("C2", N=N)
t = P.h2_cluster_tree(c["points"], c["leaf"])
bt = P.h2_block_tree(t, t, c["eta"])
Z = P.h2_from_sparse(bt, c["A"], lower=True, rank_cap=32, update_cap=32)
torch.cuda.synchronize()
if prof:
    P.h2_profile_enable(True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
w0 = time.perf_counter()
e0.record()
P.h2_lr_factor(Z, cholesky=True, trunc=P.Trunc(1e-4))
w1 = time.perf_counter()
e1.record()
torch.cuda.synchronize()
w2 = time.perf_counter()
out = dict(N=N, n=c["n"], gpu_s=e0.elapsed_time(e1) / 1e3, host_enqueue_s=w1 - w0, wall_s=w2 - w0,
           stats=P.h2_stats(Z), flags=P.h2_check_device_flags(Z))
if prof:
    out["kernels"] = {k: (v["launches"], round(v["ms"], 1)) for k, v in P.h2_profile_read().items()}
    d = P.h2.h2_profile_debug()
    out["host_wait_s"] = round(d[15], 3)
    out["ops"] = P.h2.h2_profile_ops()
    if d[3]:
        out["svd_phases_cycles_per_call"] = [round(d[0] / d[3]), round(d[1] / d[3]), round(d[2] / d[3])]
        out["svd_avg_K_m_sweeps"] = [d[4] / d[3], d[5] / d[3], d[6] / d[3]]
        out["svd_paths_calls_avg_cycles"] = {name: [int(d[7 + i]), round(d[10 + i] / d[7 + i]) if d[7 + i] else 0]
                                             for i, name in enumerate(("regs_m<=16", "K<=32", "K>32 cta"))}
    P.h2_profile_enable(False)
kr, kc = P.h2_ranks(Z)
out["maxrank"] = [int(kr.max()), int(kc.max())]
out["storage_KB_per_dof"] = float(P.h2_storage_report(Z).sum() * 8 / c["n"] / 1e3)
print(json.dumps(out))
