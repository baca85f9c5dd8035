"""Timings of the BASELINE configs beyond the bench's C2 line; one JSON line each.

  python tools/time_configs.py c1 [count]        C1: `count` (10,000) seeded random rank-k_u updates
                                                 at fixed rank 16, k_u in {4, 8, 16, 32}; updates/s
                                                 = count / device time of the dependent stream
                                                 (inputs resident in HBM), median of 3 fresh runs
  python tools/time_configs.py c3 [N]            C3: 3D Kuhn P1 Laplacian N^3 (64^3), leaf 64:
                                                 H^2 Cholesky at eps 1e-4 + PCG to 1e-8
  python tools/time_configs.py c4 [N] [eps...]   C4: 2D jump problem N^2 (1024^2): Z = A A (h2_addmul
                                                 into a fresh rank-0 Z), then H^2 Cholesky of A
                                                 (reading own-8: A^2 is numerically singular here)

  python tools/time_configs.py table1 [l...]      the paper's own FEM parameters (Table 1):
                                                 Poisson on (2^l - 1)^2 nodes, eta = 4, block-relative
                                                 accuracy eps^ ~ h^2 (NEXT-1, reading own-10), geometric
                                                 bisection tree (the paper: DD clustering, NEXT-3);
                                                 Time/n, Mem/n, Err (power iteration, R11), m

Every call goes through the C ABI (paper_1402_5056_b200); times are CUDA events on the stream.
"""
import json
import sys
import time

import numpy as np
import scipy.sparse as sp
import torch

sys.path.insert(0, ".")
import paper_1402_5056_b200 as P  # noqa: E402
from inputs import config  # noqa: E402
from inputs.rng import stream, RHS  # noqa: E402
from inputs.updates import c1_stream  # noqa: E402

dev = torch.device("cuda", 0)
ADM = 1  # h2_btree_export kind of an admissible leaf (include/h2.h)


def ev():
    return torch.cuda.Event(enable_timing=True)


def structure(c):
    t = P.h2_cluster_tree(c["points"], c["leaf"])
    bt = P.h2_block_tree(t, t, c["eta"])
    return t, bt


def adm_targets(t, bt):
    """Admissible leaves (t0, s0, |t0|, |s0|) in block-tree DFS order, from the ABI exports."""
    adm = np.nonzero(bt.kind == ADM)[0]
    return [(int(bt.t[i]), int(bt.s[i]), t.size(bt.t[i]), t.size(bt.s[i])) for i in adm]


def run_c1(count):
    c = config("C1")
    t, bt = structure(c)
    targets = adm_targets(t, bt)
    out = {"config": "C1", "n": c["n"], "count": count, "trunc": "fixed rank 16 (rel 1e-12, max_rank 16)"}
    for ku in (4, 8, 16, 32):
        ups = c1_stream(targets, count, ku, seed=0)
        # all factors resident in HBM before the clock starts (one buffer, column-major slices)
        Xs = [torch.from_numpy(np.asfortranarray(X)).to(dev) for _, _, X, _ in ups]
        Ys = [torch.from_numpy(np.asfortranarray(Y)).to(dev) for _, _, _, Y in ups]
        res = {}
        for mode in ("batched", "per_call"):
            runs = []
            for rep in range(3):
                Z = P.h2_from_sparse(bt, c["A"], lower=False, rank_cap=16, update_cap=32)
                torch.cuda.synchronize()
                e0, e1 = ev(), ev()
                w0 = time.perf_counter()
                e0.record()
                if mode == "batched":  # one op list for the whole dependent stream (h2_batch_begin)
                    P.h2_batch_begin(torch.cuda.current_stream().cuda_stream)
                for (t0, s0, _, _), X, Y in zip(ups, Xs, Ys):
                    P.h2_lowrank_update(Z, t0, s0, X, Y, trunc=P.Trunc(1e-12, 0.0, 16),
                                        stream=torch.cuda.current_stream().cuda_stream)
                if mode == "batched":
                    P.h2_batch_end()
                e1.record()
                torch.cuda.synchronize()
                runs.append((e0.elapsed_time(e1) / 1e3, time.perf_counter() - w0))
                kr, kc = P.h2_ranks(Z)
                flags = P.h2_check_device_flags(Z)
                del Z
            dev_s = sorted(r[0] for r in runs)[1]
            res[mode] = {"updates_per_s": count / dev_s, "device_s": dev_s, "wall_s": sorted(r[1] for r in runs)[1],
                         "max_rank": [int(kr.max()), int(kc.max())], "flags": flags}
        out[f"k{ku}"] = res
    print(json.dumps(out), flush=True)


def matvec_gbps(Z, n, reps=20):
    """Algorithmic bytes (8 per stored scalar + 16 n) / median time of h2_matvec."""
    x = torch.randn(n, dtype=torch.float64, device=dev)
    y = torch.empty_like(x)
    for _ in range(3):
        P.h2_matvec(Z, x, y)
    evs = [(ev(), ev()) for _ in range(reps)]
    for a, b in evs:
        a.record()
        P.h2_matvec(Z, x, y)
        b.record()
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in evs)[reps // 2]
    byt = 8.0 * float(P.h2_storage_report(Z).sum()) + 16.0 * n
    return {"ms": ms, "MB": byt / 1e6, "GBps": byt / ms / 1e6}


def factor_and_pcg(c, bt, Z, Aop, eps, label, extra):
    e0, e1, e2 = ev(), ev(), ev()
    torch.cuda.synchronize()
    e0.record()
    P.h2_lr_factor(Z, cholesky=True, trunc=P.Trunc(eps))
    e1.record()
    torch.cuda.synchronize()
    try:
        flags = P.h2_check_device_flags(Z)
    except P.H2Error as err:  # leaf breakdown: report it, no PCG
        print(json.dumps({"config": label, "n": c["n"], "eps": eps, "setup_s": e0.elapsed_time(e1) / 1e3,
                          "breakdown": str(err), "stats": P.h2_stats(Z), **extra}), flush=True)
        return
    b = torch.from_numpy(stream(RHS).standard_normal(c["n"])).to(dev)
    x = torch.zeros_like(b)
    e1b = ev()
    e1b.record()
    try:
        _, m, rel = P.h2_pcg(Aop, Z, b, x, tol=1e-8)
    except P.H2Error as err:
        m, rel = -1, str(err)
    e2.record()
    torch.cuda.synchronize()
    kr, kc = P.h2_ranks(Z)
    out = {"config": label, "n": c["n"], "eps": eps, "setup_s": e0.elapsed_time(e1) / 1e3,
           "pcg_iterations": m, "pcg_relres": rel, "pcg_s": e1b.elapsed_time(e2) / 1e3, "stats": P.h2_stats(Z),
           "max_rank": [int(kr.max()), int(kc.max())], "flags": flags,
           "storage_KB_per_dof": float(P.h2_storage_report(Z).sum() * 8 / c["n"] / 1e3),
           "matvec_factor": matvec_gbps(Z, c["n"])}
    out.update(extra)
    print(json.dumps(out), flush=True)


def run_c3(N):
    c = config("C3", N=N)
    w0 = time.perf_counter()
    t, bt = structure(c)
    st = time.perf_counter() - w0
    # 3D ranks exceed 32 ("larger ranks"): the largest stored capacity, 48 + 48
    Aop = P.h2_from_sparse(bt, c["A"], lower=False, rank_cap=48, update_cap=48)
    Z = P.h2_from_sparse(bt, c["A"], lower=True, rank_cap=48, update_cap=48)
    factor_and_pcg(c, bt, Z, Aop, 1e-4, f"C3 {N}^3", {"structure_s": st, "rank_cap": 48})


def run_c4(N, epss):
    """C4 (reading own-8): the full H^2 product Z = A A into a fresh rank-0 Z (exact, R14; checked on
    a probe against the sparse A^2), then the H^2 Cholesky of A at each eps.  A^2 itself is not
    factored at this size: its condition number (~1e18 for the 10^6 coefficient contrast at
    h = 1/1025) exceeds 1/eps_machine, so every truncated Cholesky of it breaks down."""
    c = config("C4", N=N)
    w0 = time.perf_counter()
    t, bt = structure(c)
    st = time.perf_counter() - w0
    A = P.h2_from_sparse(bt, c["A"], lower=False, rank_cap=32, update_cap=32)
    Aop = A
    zero = sp.csr_matrix(c["A"].shape)
    Z = P.h2_from_sparse(bt, zero, lower=False, rank_cap=32, update_cap=32)
    torch.cuda.synchronize()
    e0, e1 = ev(), ev()
    e0.record()
    P.h2_addmul(Z, 1.0, A, A, trunc=P.Trunc(epss[0]))
    e1.record()
    torch.cuda.synchronize()
    prod_s = e0.elapsed_time(e1) / 1e3
    xv = np.random.default_rng(3).standard_normal(c["n"])
    zx = P.h2_matvec(Z, torch.from_numpy(xv).to(dev)).cpu().numpy()
    ref = c["A"] @ (c["A"] @ xv)
    prod = {"product_s": prod_s, "product_stats": P.h2_stats(Z),
            "product_rel_err": float(np.linalg.norm(zx - ref) / np.linalg.norm(ref)),
            "product_storage_KB_per_dof": float(P.h2_storage_report(Z).sum() * 8 / c["n"] / 1e3),
            "matvec_product": matvec_gbps(Z, c["n"])}
    print(json.dumps({"config": f"C4 {N}^2 A*A", "n": c["n"], "structure_s": st, **prod}), flush=True)
    del Z
    for eps in epss:
        cap = 32 if eps >= 1e-4 else 48  # tighter truncation, larger ranks
        L = P.h2_from_sparse(bt, c["A"], lower=True, rank_cap=cap, update_cap=cap)
        factor_and_pcg(c, bt, L, Aop, eps, f"C4 {N}^2 Cholesky of A", {"rank_cap": cap})
        del L


def run_inv(N, eps):
    """NEXT-2: approximate inverse (Remark 1) of the C2-shaped jump problem at N x N nodes; the
    quality ||I - C A|| on probes and the PCG iterations with C as preconditioner."""
    c = config("C2", N=N)
    t, bt = structure(c)
    Aop = P.h2_from_sparse(bt, c["A"], lower=False, rank_cap=32, update_cap=32)
    Z = P.h2_from_sparse(bt, c["A"], lower=False, rank_cap=32, update_cap=32)
    torch.cuda.synchronize()
    e0, e1 = ev(), ev()
    e0.record()
    P.h2_inverse(Z, trunc=P.Trunc(eps))
    e1.record()
    torch.cuda.synchronize()
    X = np.random.default_rng(7).standard_normal((c["n"], 4))
    r = []
    for j in range(4):
        x = torch.from_numpy(X[:, j].copy()).to(dev)
        ax = P.h2_matvec(Aop, x)
        cax = P.h2_matvec(Z, ax).cpu().numpy()
        r.append(np.linalg.norm(cax - X[:, j]) / np.linalg.norm(X[:, j]))
    kr, kc = P.h2_ranks(Z)
    print(json.dumps({"config": f"inverse C2-shaped {N}^2", "n": c["n"], "eps": eps, "inverse_s": e0.elapsed_time(e1) / 1e3,
                      "I_minus_CA_probe_rel": max(r), "stats": P.h2_stats(Z), "max_rank": [int(kr.max()), int(kc.max())],
                      "flags": P.h2_check_device_flags(Z),
                      "storage_KB_per_dof": float(P.h2_storage_report(Z).sum() * 8 / c["n"] / 1e3)}), flush=True)


TABLE1 = {7: (3.1e-3, 7.0e-5, 1.0, 0.06, 3), 8: (7.7e-4, 8.4e-5, 1.1, 0.07, 3), 9: (1.9e-4, 1.1e-4, 1.2, 0.07, 3),
          10: (4.8e-5, 1.3e-4, 1.2, 0.10, 3), 11: (1.2e-5, 1.5e-4, 1.2, 0.11, 3)}  # l: eps^, Time/n, Mem/n KB, Err, m


def run_table1(levels, dd=False, jump=False):
    """dd: the domain-decomposition cluster tree (NEXT-3, reading own-11) instead of geometric
    bisection; jump: the C2 jump-coefficient problem at N = 512 with eta = 2, eps = 1e-4 relative
    (the BASELINE C2 matrix on the DD tree) instead of the paper's Poisson settings."""
    from inputs.rng import POWER
    for l in levels:
        N = 2 ** l - 1
        eps = TABLE1[l][0]
        c = config("C1", N=N)  # the constant-coefficient 5-point problem
        eta, trunc = 4.0, P.Trunc(eps, abs_tol=1e-13 if dd else 0.0, blockwise=True)
        if jump:
            N = 2 ** l
            c = config("C2", N=N)
            eta, eps, trunc = 2.0, 1e-4, P.Trunc(1e-4, abs_tol=1e-13)
        t = P.h2_cluster_tree_dd(c["points"], c["leaf"], c["A"]) if dd else P.h2_cluster_tree(c["points"], c["leaf"])
        bt = P.h2_block_tree(t, t, eta)
        Aop = P.h2_from_sparse(bt, c["A"], lower=False, rank_cap=32, update_cap=32)
        Z = P.h2_from_sparse(bt, c["A"], lower=True, rank_cap=32, update_cap=32)
        torch.cuda.synchronize()
        e0, e1 = ev(), ev()
        e0.record()
        P.h2_lr_factor(Z, cholesky=True, trunc=trunc)
        e1.record()
        torch.cuda.synchronize()
        flags = P.h2_check_device_flags(Z)
        n = c["n"]
        b = torch.from_numpy(stream(RHS).standard_normal(n)).to(dev)
        x = torch.zeros_like(b)
        e2, e3 = ev(), ev()
        e2.record()
        _, m, rel = P.h2_pcg(Aop, Z, b, x, tol=1e-8)
        e3.record()
        torch.cuda.synchronize()
        # Err = ||I - (L L^T)^-1 A||_2 by plain power iteration (R11): 50 its or rel. change < 1e-4
        v = torch.from_numpy(stream(POWER).standard_normal(n)).to(dev)
        v /= torch.linalg.norm(v)
        lam = 0.0
        for it in range(50):
            w = P.h2_matvec(Aop, v)
            P.h2_solve(Z, w)
            w = v - w
            new = float(torch.linalg.norm(w))
            v = w / new
            if it > 0 and abs(new - lam) <= 1e-4 * new:
                lam = new
                break
            lam = new
        kr, kc = P.h2_ranks(Z)
        setup_s = e0.elapsed_time(e1) / 1e3
        ref = TABLE1[l]
        print(json.dumps({"config": ("C2 jump problem" if jump else f"Table 1 l={l}"), "n": n, "eta": eta, "eps_hat": eps,
                          "truncation": "relative 1e-4 (+ abs 1e-13)" if jump else "block-relative (own-10)",
                          "tree": ("domain decomposition (own-11)" if dd else "geometric bisection") + ", leaf 32",
                          "clusters": int(t.nclusters), "blocks": int(bt.nblocks),
                          "setup_s": setup_s, "setup_s_per_dof": setup_s / n,
                          "mem_KB_per_dof": float(P.h2_storage_report(Z).sum() * 8 / n / 1e3),
                          "Err": lam, "m": m, "pcg_relres": rel, "solve_s_per_step_per_dof": e2.elapsed_time(e3) / 1e3 / max(m, 1) / n,
                          "max_rank": [int(kr.max()), int(kc.max())], "mean_rank": float(kr.mean()), "flags": flags,
                          "stats": P.h2_stats(Z), "matvec_factor": matvec_gbps(Z, n),
                          "paper_table1": {"setup_s_per_dof": ref[1], "mem_KB_per_dof": ref[2], "Err": ref[3], "m": ref[4],
                                           "machine": "one Opteron 8431 core; DD clustering (P:1403-1405)"}}), flush=True)
        del Z, Aop


TABLE2 = {17: (1.9e-6, 3.3e-4, 0.8, 0.02, 3), 18: (9.5e-7, 3.5e-4, 0.8, 0.01, 4),
          11: (1.2e-4, 1.6e-4, 0.8, 0.05, 3), 12: (6.1e-5, 1.9e-4, 0.8, 0.03, 3), 13: (3.1e-5, 2.1e-4, 0.8, 0.03, 3),
          14: (1.5e-5, 2.4e-4, 0.8, 0.02, 3), 15: (7.6e-6, 2.6e-4, 0.8, 0.02, 3), 16: (3.8e-6, 3.0e-4, 0.8, 0.02, 3)}


def run_bem(levels):
    """NEXT-4 (Table 2; reading own-12): single layer potential on the circle, n = 2^(l+2)
    arcs (the paper's l = 11 row has n = 8,192), eta = 2, block-relative eps^ ~ h.  The H^2 matrix is built from the exact nearfield
    entries by one h2_lowrank_update per admissible leaf (factors from inputs/bem.py, resident in
    HBM before the clock starts), then factored (Cholesky, lower storage) and used in PCG."""
    from inputs import bem
    from inputs.rng import POWER
    for l in levels:
        n = 2 ** (l + 2)
        eps = TABLE2[l][0]
        tr = P.Trunc(eps, blockwise=True)
        t = P.h2_cluster_tree(bem.circle_points(n), 32)
        bt = P.h2_block_tree(t, t, 2.0)
        res = {}
        mats = {}
        for lower in (False, True):
            w0 = time.perf_counter()
            A_near, far = bem.pieces(n, t.perm, t.lo, t.hi, bt.t, bt.s, bt.kind, lower=lower)
            gen_s = time.perf_counter() - w0
            Z = P.h2_from_sparse(bt, A_near, lower=lower, rank_cap=48, update_cap=32)
            Xs = [torch.from_numpy(np.asfortranarray(X)).to(dev) for _, _, X, _ in far]
            Ys = [torch.from_numpy(np.asfortranarray(Y)).to(dev) for _, _, _, Y in far]
            torch.cuda.synchronize()
            e0, e1 = ev(), ev()
            e0.record()
            P.h2_batch_begin(torch.cuda.current_stream().cuda_stream)
            for (t0, s0, _, _), X, Y in zip(far, Xs, Ys):
                P.h2_lowrank_update(Z, t0, s0, X, Y, trunc=tr, stream=torch.cuda.current_stream().cuda_stream)
            P.h2_batch_end()
            e1.record()
            torch.cuda.synchronize()
            res["lower" if lower else "full"] = {"updates": len(far), "build_s": e0.elapsed_time(e1) / 1e3,
                                                 "updates_per_s": len(far) / (e0.elapsed_time(e1) / 1e3), "generator_s": gen_s}
            mats[lower] = Z
            del Xs, Ys
        Aop, Z = mats[False], mats[True]
        # accuracy of the compressed operator against the exact circulant matrix (FFT product)
        g = bem.first_row(n)
        xv = np.random.default_rng(3).standard_normal(n)
        ref = np.real(np.fft.ifft(np.fft.fft(g) * np.fft.fft(xv)))
        yv = P.h2_matvec(Aop, torch.from_numpy(xv).to(dev)).cpu().numpy()
        e0, e1 = ev(), ev()
        e0.record()
        P.h2_lr_factor(Z, cholesky=True, trunc=tr)
        e1.record()
        torch.cuda.synchronize()
        flags = P.h2_check_device_flags(Z)
        b = torch.from_numpy(stream(RHS).standard_normal(n)).to(dev)
        x = torch.zeros_like(b)
        e2, e3 = ev(), ev()
        e2.record()
        _, m, rel = P.h2_pcg(Aop, Z, b, x, tol=1e-8)
        e3.record()
        torch.cuda.synchronize()
        v = torch.from_numpy(stream(POWER).standard_normal(n)).to(dev)
        v /= torch.linalg.norm(v)
        lam = 0.0
        for it in range(50):
            w = P.h2_matvec(Aop, v)
            P.h2_solve(Z, w)
            w = v - w
            new = float(torch.linalg.norm(w))
            v = w / new
            if it > 0 and abs(new - lam) <= 1e-4 * new:
                lam = new
                break
            lam = new
        kr, kc = P.h2_ranks(Z)
        setup_s = e0.elapsed_time(e1) / 1e3
        ref2 = TABLE2[l]
        print(json.dumps({"config": f"Table 2 l={l} (BEM single layer potential, circle r=1/2)", "n": n, "eta": 2.0, "eps_hat": eps,
                          "compression_by_local_updates": res,
                          "operator_rel_err_vs_exact": float(np.linalg.norm(yv - ref) / np.linalg.norm(ref)),
                          "setup_s": setup_s, "setup_s_per_dof": setup_s / n,
                          "mem_KB_per_dof": float(P.h2_storage_report(Z).sum() * 8 / n / 1e3),
                          "Err": lam, "m": m, "pcg_relres": rel,
                          "solve_s_per_step_per_dof": e2.elapsed_time(e3) / 1e3 / max(m, 1) / n,
                          "max_rank": [int(kr.max()), int(kc.max())], "flags": flags, "stats": P.h2_stats(Z),
                          "matvec_operator": matvec_gbps(Aop, n), "matvec_factor": matvec_gbps(Z, n),
                          "paper_table2": {"setup_s_per_dof": ref2[1], "mem_KB_per_dof": ref2[2], "Err": ref2[3], "m": ref2[4],
                                           "machine": "one Opteron 8431 core"}}), flush=True)
        del mats, Aop, Z


if __name__ == "__main__":
    what = sys.argv[1]
    if what == "bem":
        run_bem([int(a) for a in sys.argv[2:]] or [11, 13])
        sys.exit(0)
    if what in ("table1", "table1dd", "c2dd"):
        run_table1([int(a) for a in sys.argv[2:]] or [7, 8, 9], dd=what != "table1", jump=what == "c2dd")
        sys.exit(0)
    if what == "c1":
        run_c1(int(sys.argv[2]) if len(sys.argv) > 2 else 10000)
    elif what == "c3":
        run_c3(int(sys.argv[2]) if len(sys.argv) > 2 else 64)
    elif what == "c4":
        N = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
        epss = [float(e) for e in sys.argv[3:]] or [1e-2, 1e-4, 1e-6]
        run_c4(N, epss)
    elif what == "inv":
        run_inv(int(sys.argv[2]) if len(sys.argv) > 2 else 256, float(sys.argv[3]) if len(sys.argv) > 3 else 1e-4)
