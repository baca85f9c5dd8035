"""Write the oracle's result for the C2 headline problem (north_star target).

Imports ONLY oracle/ and inputs/ (no CUDA path): builds the C2 jump problem of side N
(BASELINE.json configs[2]: 512 x 512, n = 262,144, leaf 32, eta 2), runs the oracle's H^2
Cholesky at eps = 1e-4, and stores

  ranks_row / ranks_col   cluster ranks after the factorization (bit-exact parity)
  stats                   local updates / dense adds / temporaries performed
  probes_out              L p for the first 4 seeded probe vectors (inputs.rng.probes(n, 4)),
                          float32 (the bar is 10 eps = 1e-3 relative; float32 keeps 1e-7)
  pcg_m, pcg_relres       PCG to 1e-8 with b = stream(RHS) (reading R12)
  err                     ||I - (LL^T)^{-1} A|| by power iteration (reading R11)
  fact_s, host            oracle factorization seconds and the host it ran on (context)

into tests/golden/c2_oracle_N{N}.npz (+ a .json summary beside it).

    python tools/oracle_golden_c2.py [N]
"""
import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from inputs import config  # noqa: E402
from inputs.rng import stream, probes, RHS, POWER  # noqa: E402
from oracle.structure import ClusterTree, BlockTree  # noqa: E402
from oracle.h2 import from_sparse  # noqa: E402
from oracle.update import Trunc  # noqa: E402
from oracle.arith import Arith, pcg, power_error  # noqa: E402

EPS = 1e-4


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    c = config("C2", N=N)
    n = c["n"]
    t0 = time.perf_counter()
    ot = ClusterTree(c["points"], c["leaf"])
    ob = BlockTree(ot, ot, c["eta"])
    Z = from_sparse(ob, c["A"], lower=True)
    t1 = time.perf_counter()
    ar = Arith(Z, Trunc(EPS))
    ar.chol()
    t2 = time.perf_counter()
    print(f"structure {t1 - t0:.1f} s, Cholesky {t2 - t1:.1f} s, stats {ar.stats}", flush=True)
    P4 = probes(n, 4).T  # n x 4, ORIGINAL order
    Y = Z.matvec(P4)
    A = c["A"]
    b = stream(RHS).standard_normal(n)
    t3 = time.perf_counter()
    _, m, rel = pcg(lambda v: A @ v, lambda v: ar.solve(v), b)
    t4 = time.perf_counter()
    print(f"PCG m={m} relres={rel:.3e} ({t4 - t3:.1f} s)", flush=True)
    err = power_error(lambda v: A @ v, lambda v: ar.solve(v), stream(POWER).standard_normal(n))
    t5 = time.perf_counter()
    print(f"Err={err:.5f} ({t5 - t4:.1f} s)", flush=True)
    out = os.path.join(ROOT, "tests", "golden", f"c2_oracle_N{N}")
    np.savez_compressed(out + ".npz", ranks_row=Z.k.astype(np.int16), ranks_col=Z.l.astype(np.int16),
                        probes_out=Y.astype(np.float32), pcg_m=np.int32(m), pcg_relres=np.float64(rel),
                        err=np.float64(err))
    summary = dict(config="C2", N=N, n=n, eps=EPS, leaf=c["leaf"], eta=c["eta"], stats=ar.stats,
                   max_rank=[int(Z.k.max()), int(Z.l.max())], pcg_m=int(m), pcg_relres=float(rel), err=float(err),
                   structure_s=round(t1 - t0, 1), fact_s=round(t2 - t1, 1), pcg_s=round(t4 - t3, 1),
                   power_s=round(t5 - t4, 1), host=dict(cpu=cpu_model(), nproc=os.cpu_count()),
                   written_by="tools/oracle_golden_c2.py (imports oracle/ and inputs/ only)",
                   cites="BASELINE.json configs[2]; P:338-390, P:1406-1408 (Cholesky), P:1440-1443 (Err, PCG)")
    json.dump(summary, open(out + ".json", "w"), indent=1)
    print(json.dumps(summary))


if __name__ == "__main__":
    main()
