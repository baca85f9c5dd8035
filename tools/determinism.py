"""Determinism stress of the GPU H^2 Cholesky.

Factors the C2-shaped jump problem of side N `runs` times, each on a fresh h2_from_sparse copy,
and fingerprints every result bit for bit: row/column ranks, the update counters, the device
flags, the factor applied to 4 seeded probe vectors (h2_matvec of the stored L) and the PCG
iteration count / relative residual.  Environment knobs of the library (H2_EXEC_BIG, H2_EXEC_CL,
H2_POISON, H2_NO_SKIP ...) are read by the library itself.

    python tools/determinism.py N runs [--pcg]
prints one JSON line per run and a summary line {"identical": bool, ...}.
"""
import hashlib
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1402_5056_b200 as P  # noqa: E402
from inputs import config  # noqa: E402
from inputs.rng import stream, RHS, PROBES  # noqa: E402


def sha(*arrs):
    h = hashlib.sha1()
    for a in arrs:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:16]


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    runs = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    do_pcg = "--pcg" in sys.argv
    c = config("C2", N=N)
    n = c["n"]
    tree = P.h2_cluster_tree(c["points"], c["leaf"])
    bt = P.h2_block_tree(tree, tree, c["eta"])
    probes = torch.from_numpy(stream(PROBES).standard_normal((4, n))).cuda()
    Aop = P.h2_from_sparse(bt, c["A"], lower=False, rank_cap=32, update_cap=32) if do_pcg else None
    b = torch.from_numpy(stream(RHS).standard_normal(n)).cuda()
    prints = []
    for r in range(runs):
        Z = P.h2_from_sparse(bt, c["A"], lower=True, rank_cap=32, update_cap=32)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        P.h2_lr_factor(Z, cholesky=True, trunc=P.Trunc(1e-4))
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        try:
            flags = P.h2_check_device_flags(Z)
            err = ""
        except P.H2Error as e:
            flags, err = -1, str(e)
        kr, kc = P.h2_ranks(Z)
        ys = [P.h2_matvec(Z, probes[i]).cpu().numpy() for i in range(4)]
        finite = bool(all(np.isfinite(y).all() for y in ys))
        rec = dict(run=r, N=N, seconds=round(dt, 3), flags=flags, err=err, stats=P.h2_stats(Z),
                   ranks=sha(kr, kc), maxrank=[int(kr.max()), int(kc.max())], probes=sha(*ys), finite=finite,
                   probe_norm=[float(np.linalg.norm(y)) for y in ys])
        if do_pcg:
            x = torch.zeros(n, dtype=torch.float64, device="cuda")
            try:
                _, m, rel = P.h2_pcg(Aop, Z, b, x, tol=1e-8)
                rec["pcg"] = [m, rel]
            except P.H2Error as e:
                rec["pcg"] = str(e)
        print(json.dumps(rec), flush=True)
        prints.append((rec["ranks"], rec["probes"], json.dumps(rec["stats"], sort_keys=True), rec["flags"]))
        del Z
        torch.cuda.synchronize()
    env = {k: v for k, v in os.environ.items() if k.startswith("H2_")}
    print(json.dumps({"summary": True, "N": N, "runs": runs, "env": env, "identical": len(set(prints)) == 1,
                      "distinct": len(set(prints))}), flush=True)


if __name__ == "__main__":
    main()
