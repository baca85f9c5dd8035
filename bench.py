"""Benchmark of the B200 H^2 hot path (contract: one JSON line on rank 0).

Workload C2 (BASELINE.json configs[2], the configuration the metric is quoted on, "at n=262k";
SURVEY §8(d)): 2D -div(sigma grad u), P1 FEM on 512 x 512 nodes (n = 262,144), sigma on a 16 x 16
checkerboard, 10^U with U ~ U[-3,3] (seeded), leaf 32, eta = 2.  One step = the whole hot path
on a fresh rank-0 H^2 copy of A: H^2 Cholesky at eps = 1e-4 (h2_lr_factor: recursive product,
block substitutions, ~4e5 local low-rank updates U0-U6, dense leaf factorizations) followed by
preconditioned CG to ||r||/||b|| < 1e-8 with a seeded b ~ N(0,1) (h2_pcg: H^2 matvec + H^2
triangular solves).  The cluster/block trees (host) and h2_from_sparse are built outside the
timed region (reported separately).

metric value: local low-rank updates with non-zero rank per second during the factorization
(the count is identical to the oracle's, which is checked by the parity tests); `setup_s` is the
LR-factor setup time in seconds (the paper's Table-1 quantity) and is reported beside it.

Multi-GPU: the update chain does not shard (replicas only); --gpus N runs N
independent replicas, value = total updates / max-over-ranks time.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--N 512]
"""
import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "H2 LR-factor setup s and rank-k updates/s (FP64) at n=262k; % of roofline"
UNIT = "updates/s"
EPS = 1e-4


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    d = json.load(open(p)) if os.path.exists(p) else {}
    f = os.path.join(ROOT, "profiles", "fp64_peak.json")
    fp = json.load(open(f)) if os.path.exists(f) else {}
    return d, fp


def _clock_sampler_start():
    try:
        f = open(os.path.join("/tmp", f"h2_clocks_{os.getpid()}.csv"), "w")
        p = subprocess.Popen(
            ["nvidia-smi", "--query-gpu=index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
             "--format=csv,noheader,nounits", "-lms", "200"], stdout=f, stderr=subprocess.DEVNULL)
        return p, f
    except Exception:
        return None, None


def _clock_sampler_stop(p, f, gpu_index):
    if p is None:
        return None
    p.terminate()
    try:
        p.wait(timeout=5)
    except Exception:
        p.kill()
    f.close()
    sm, mx, reasons = [], 0.0, set()
    names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    for line in open(f.name):
        parts = [x.strip() for x in line.split(",")]
        if len(parts) < 8 or parts[0] != str(gpu_index):
            continue
        try:
            sm.append(float(parts[1]))
            mx = max(mx, float(parts[2]))
        except ValueError:
            continue
        for nm, v in zip(names, parts[4:8]):
            if v.lower().startswith("active"):
                reasons.add(nm)
    if not sm:
        return None
    return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def max_over_ranks(vals, dist, device):
    """Element-wise MAX of a list of floats over all ranks (the step time of a multi-GPU run is the
    slowest rank's).  Backend-agnostic: nccl with CUDA tensors, gloo with CPU tensors (tests)."""
    import torch
    t = torch.tensor([float(v) for v in vals], device=device, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(v) for v in t.tolist()]


def job_throughput(nz_per_rank, world, fact_ms_max):
    """Whole-job updates/s: every replica factors the same workload, so the job processed
    world x nz updates in the slowest rank's factorization time."""
    return nz_per_rank * world / (fact_ms_max / 1e3)


def run_gpu(args, rank, world):
    import torch
    import paper_1402_5056_b200 as P
    from inputs import config
    from inputs.rng import stream, RHS

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    cs = torch.cuda.current_stream()
    c = config("C2", N=args.N)
    n = c["n"]
    A = c["A"]
    t0 = time.perf_counter()
    tree = P.h2_cluster_tree(c["points"], c["leaf"])
    bt = P.h2_block_tree(tree, tree, c["eta"])
    structure_s = time.perf_counter() - t0
    Aop = P.h2_from_sparse(bt, A, lower=False, rank_cap=32, update_cap=32)  # operator for PCG (nearfield form)
    b_host = stream(RHS).standard_normal(n)
    b = torch.from_numpy(b_host).to(dev)
    x = torch.zeros(n, dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # 256 MiB > 126 MB L2
    trunc = P.Trunc(EPS)

    def check_step(Z, m=None, rel=None):
        """A step counts only if the factorization is clean: no device flag (rank clamp, leaf
        breakdown) and PCG converged to a finite residual (h2_pcg raises otherwise)."""
        f = P.h2_check_device_flags(Z)
        if f != 0:
            raise P.H2Error(8, f"device flags {f} after the factorization")
        if rel is not None and not (np.isfinite(rel) and rel < 1e-8):
            raise P.H2Error(9, f"PCG relres {rel}")

    def fresh():
        t = time.perf_counter()
        Z = P.h2_from_sparse(bt, A, lower=True, rank_cap=32, update_cap=32)
        torch.cuda.synchronize()
        return Z, time.perf_counter() - t

    prof = None
    e2e_samples = []
    # ---- warm-up steps (the first one is profiled, the others are end-to-end measurements) ----
    for w in range(args.warmup):
        if w >= 1:
            # e2e: host CSR -> h2_from_sparse (upload) -> factor -> PCG with b from pinned host -> x back
            bh = torch.from_numpy(b_host).pin_memory()
            xh = torch.empty(n, dtype=torch.float64).pin_memory()
            torch.cuda.synchronize()
            te = time.perf_counter()
            Z = P.h2_from_sparse(bt, A, lower=True, rank_cap=32, update_cap=32)
            P.h2_lr_factor(Z, cholesky=True, trunc=trunc)
            bd = bh.to(dev, non_blocking=True)
            P.h2_pcg(Aop, Z, bd, x, tol=1e-8)
            xh.copy_(x, non_blocking=True)
            torch.cuda.synchronize()
            e2e_s = time.perf_counter() - te
            check_step(Z)
            e2e_samples.append((P.h2_stats(Z)["updates_nonzero"], e2e_s))
            del Z
            continue
        Z, _ = fresh()
        P.h2_profile_enable(True)
        P.h2_lr_factor(Z, cholesky=True, trunc=trunc)
        P.h2_pcg(Aop, Z, b, x, tol=1e-8)
        torch.cuda.synchronize()
        prof = P.h2_profile_read()
        P.h2_profile_enable(False)
        check_step(Z)
        del Z
    e2e = None
    if e2e_samples:
        secs = sorted(t for _, t in e2e_samples)
        med = secs[len(secs) // 2]
        nz = e2e_samples[0][0]
        csr_bytes = A.indptr.nbytes + A.indices.nbytes + A.data.nbytes
        e2e = {"value": nz / med, "unit": UNIT, "seconds": med, "samples_s": [round(t, 3) for _, t in e2e_samples],
               "h2d_bytes_per_step": int(csr_bytes + 8 * n), "d2h_bytes_per_step": int(8 * n),
               "path": "h2_from_sparse(host CSR) + h2_lr_factor + h2_pcg(b from pinned host) + x to host; "
                       "median over the non-profiled warm-up steps"}
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    clk_p, clk_f = _clock_sampler_start() if rank == 0 else (None, None)
    fact_ms, pcg_ms, nz_total, iters, rels, launches = 0.0, 0.0, 0, [], [], 0
    stats, failed, good = None, [], 0
    for j in range(args.steps):
        Z, fs = fresh()  # outside the timed events
        flush.fill_(float(j))  # L2 flush between timed steps
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        l0 = P.h2_launch_count()
        e0.record(cs)
        P.h2_lr_factor(Z, cholesky=True, trunc=trunc)
        e1.record(cs)
        try:
            _, m, rel = P.h2_pcg(Aop, Z, b, x, tol=1e-8)
            e2.record(cs)
            torch.cuda.synchronize()
            check_step(Z, m, rel)
        except P.H2Error as err:  # a failed step is dropped from the totals and reported
            torch.cuda.synchronize()
            failed.append({"step": j, "error": str(err)})
            del Z
            continue
        launches += P.h2_launch_count() - l0
        fact_ms += e0.elapsed_time(e1)
        pcg_ms += e1.elapsed_time(e2)
        stats = P.h2_stats(Z)
        nz_total += stats["updates_nonzero"]
        iters.append(m)
        rels.append(rel)
        good += 1
        if good == 1:
            sto = P.h2_storage_report(Z)
            # matvecs (HBM-bound, both larger than L2): the factor L (~1.4 KB/DOF) and the sparse
            # input A in H^2 form (rank-0 bases; the matvec PCG applies every iteration)
            xv = torch.randn(n, dtype=torch.float64, device=dev)
            yv = torch.empty_like(xv)

            def time_mv(M):
                for _ in range(3):
                    P.h2_matvec(M, xv, yv)
                m0, m1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                m0.record(cs)
                for _ in range(20):
                    P.h2_matvec(M, xv, yv)
                m1.record(cs)
                torch.cuda.synchronize()
                return m0.elapsed_time(m1) / 20

            mv_ms = time_mv(Z)
            mvA_ms = time_mv(Aop)
            mvA_bytes = 8.0 * float(P.h2_storage_report(Aop).sum()) + 16.0 * n
        del Z
    step_ms = fact_ms + pcg_ms
    if dist is not None:
        step_ms, fact_ms = max_over_ranks([step_ms, fact_ms], dist, dev)
    clocks = _clock_sampler_stop(clk_p, clk_f, dev.index) if rank == 0 else None
    mv_bytes = 8.0 * float(sto.sum()) + 16.0 * n
    return dict(n=n, structure_s=structure_s, fact_ms=fact_ms, pcg_ms=pcg_ms, step_ms=step_ms, nz=nz_total,
                good=good, failed=failed,
                stats=stats, iters=iters, rels=rels, launches=launches, prof=prof, e2e=e2e, clocks=clocks,
                sto=sto.tolist(), mv_ms=mv_ms, mv_bytes=mv_bytes, mvA_ms=mvA_ms, mvA_bytes=mvA_bytes)


def host_cpu():
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"model": model, "nproc": os.cpu_count()}


class _Budget(Exception):
    pass


def oracle_setup(N, seed=0):
    """The oracle's structure and rank-0 H^2 copy of the C2 jump problem (outside any timing)."""
    from inputs import config
    from oracle.structure import ClusterTree, BlockTree
    import oracle.arith  # noqa: F401  (loads scipy.linalg's BLAS before the thread limit below)
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)  # the oracle as it stands, on ONE host core (every loaded BLAS)
    except Exception:
        pass
    c = config("C2", N=N, seed=seed)
    ot = ClusterTree(c["points"], c["leaf"])
    ob = BlockTree(ot, ot, c["eta"])
    return c, ot, ob


def oracle_sample(setup, budget_s):
    """A bounded sample of the C2 workload on the oracle (as it stands, one thread): its H^2
    Cholesky of the same n = N^2 jump problem, stopped after `budget_s` seconds of factorization.
    The factorization order is the paper's (chol(t1) first), so the sample is the first part of
    the very recursion the GPU runs.  Returns (local updates performed, seconds, finished)."""
    from oracle.h2 import from_sparse
    from oracle.update import Trunc
    from oracle.arith import Arith
    c, ot, ob = setup
    Z = from_sparse(ob, c["A"], lower=True)

    class Bounded(Arith):  # stops the recursion at the budget; the arithmetic is the oracle's
        def _add(self, *a, **k):
            if time.perf_counter() - self.t_start > budget_s:
                raise _Budget()
            return super()._add(*a, **k)

    ar = Bounded(Z, Trunc(EPS))
    ar.t_start = time.perf_counter()
    done = True
    try:
        ar.chol()
    except _Budget:
        done = False
    return ar.stats["updates"], time.perf_counter() - ar.t_start, done


def full_size_oracle():
    """The oracle's full C2 factorization as measured by tools/oracle_golden_c2.py (context)."""
    p = os.path.join(ROOT, "tests", "golden", "c2_oracle_N512.json")
    if not os.path.exists(p):
        return None
    g = json.load(open(p))
    return {"fact_s": g["fact_s"], "updates": g["stats"]["updates"], "updates_per_s": g["stats"]["updates"] / g["fact_s"],
            "host": g["host"], "note": "full n=262,144 oracle Cholesky, tools/oracle_golden_c2.py, build host"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--N", type=int, default=512, help="grid side (512: BASELINE C2, n = 262,144)")
    ap.add_argument("--cpu-budget", type=float, default=20.0, help="seconds of oracle factorization (cpu_baseline)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    config = {"workload": "C2", "n": args.N * args.N, "mesh": f"{args.N}x{args.N} 2D P1, sigma 16x16 checkerboard 10^U[-3,3]",
              "leaf": 32, "eta": 2.0, "eps": EPS, "factorization": "H2 Cholesky (lower storage)",
              "step": "h2_lr_factor (Cholesky) + h2_pcg to 1e-8 on a fresh h2_from_sparse copy",
              "l2": "flushed between timed steps (256 MiB write)", "parallelism": f"replicas x{args.gpus}"}

    if args.impl == "reference":
        if rank != 0:
            return
        # each step: a bounded sample of the same C2 workload, sized so the whole run stays within a
        # few minutes (the oracle needs ~515 s for the full factorization)
        per_step = min(20.0, max(3.0, 150.0 / (args.steps + args.warmup)))
        st = oracle_setup(args.N)
        for _ in range(args.warmup):
            oracle_sample(st, per_step)
        tot_u, tot_s = 0, 0.0
        for _ in range(args.steps):
            u, dt, _ = oracle_sample(st, per_step)
            tot_u += u
            tot_s += dt
        value = tot_u / tot_s
        sample = (f"oracle (numpy/scipy, 1 thread) H2 Cholesky of the same C2 problem (n={args.N * args.N}), "
                  f"each step the first {per_step:.1f} s of the factorization in the paper's order; "
                  f"updates/s = local updates performed / factorization seconds")
        line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_s / args.steps,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": dict(config, sample_s_per_step=per_step),
                "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample,
                                 "host": host_cpu()},
                "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                "full_size_oracle": full_size_oracle()}
        print(json.dumps(line))
        return

    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        dist.init_process_group("nccl")
    res = run_gpu(args, rank, world)
    if rank != 0:
        return
    if res["good"] == 0:
        print(json.dumps({"metric": METRIC, "error": "every timed step failed", "failed_steps": res["failed"]}))
        sys.exit(1)
    measured, fp = _peaks()
    good = res["good"]
    fact_s = res["fact_ms"] / 1e3 / good
    value = job_throughput(res["nz"], world, res["fact_ms"])
    prof = res["prof"] or {}
    # the executor kernel is the dominant kernel of the step (every op of the factorization runs in it)
    ex_ms = sum(v["ms"] for k, v in prof.items() if k not in ("k_matvec", "k_solve_sweep"))
    ex_flops = sum(v["flops"] for k, v in prof.items() if k not in ("k_matvec", "k_solve_sweep"))
    fp64_peak = fp.get("fp64_fma_tflops") or 37.0
    # achieved: the algorithmic FP64 flops of one factorization (device counters of the profiled
    # warm-up step: fixed formulas, the same workload every step) over the factorization time
    # measured by CUDA events in the TIMED region (the executor launches are ~99.9 % of it)
    roof = {"kernel": "k_exec_cluster (+k_exec_big): all factorization ops", "bound": "alu",
            "achieved": ex_flops / fact_s / 1e12 if ex_flops else None, "peak": fp64_peak, "unit": "TFLOP/s",
            "flops_per_step": ex_flops, "profiled_executor_ms": ex_ms,
            "traffic": None,
            "peak_source": "profiles/fp64_peak.json (FP64 DFMA microbenchmark, measured)" if fp else
                           "B200 FP64 nominal 37 TFLOP/s (148 SMs x 64 DFMA/clk x 1.965 GHz)",
            "note": "latency-bound dependent chain of tiny dense problems (avg extended rank ~6); see DESIGN.md"}
    tr = os.path.join(ROOT, "profiles", "r02", "exec_traffic.json")
    if os.path.exists(tr):
        t = json.load(open(tr))
        roof["traffic"] = t.get("dram_bytes_per_launch")
        roof["traffic_source"] = t.get("source")
    if roof["achieved"] is not None:
        roof["frac"] = roof["achieved"] / roof["peak"]
    mv_gbs = res["mv_bytes"] / (res["mv_ms"] / 1e3) / 1e9
    hbm = measured.get("hbm_gbs", 6650.0)
    cpu_u, cpu_s, _ = oracle_sample(oracle_setup(args.N), args.cpu_budget)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": res["step_ms"] / good, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config,
        "setup_s": fact_s, "setup_s_paper_l9_opteron": 28.7,
        "steps_valid": good, "failed_steps": res["failed"],
        "pcg": {"iterations": res["iters"], "relres": res["rels"], "ms": res["pcg_ms"] / good},
        "structure_s": res["structure_s"],
        "updates": res["stats"],
        "storage_KB_per_dof": 8.0 * sum(res["sto"]) / res["n"] / 1e3,
        "roofline": roof,
        "matvec": {"GBps": mv_gbs, "ms": res["mv_ms"], "bytes": res["mv_bytes"], "peak": hbm, "frac": mv_gbs / hbm,
                   "bound": "hbm", "of": "factor L"},
        "matvec_A": {"GBps": res["mvA_bytes"] / (res["mvA_ms"] / 1e3) / 1e9, "ms": res["mvA_ms"],
                     "bytes": res["mvA_bytes"], "peak": hbm,
                     "frac": res["mvA_bytes"] / (res["mvA_ms"] / 1e3) / 1e9 / hbm, "bound": "hbm",
                     "of": "input A (H2 form, the PCG operator)"},
        "cpu_baseline": {"value": cpu_u / cpu_s, "unit": UNIT, "cores": 1, "kind": "oracle", "host": host_cpu(),
                         "sample": f"oracle (numpy/scipy, 1 thread) H2 Cholesky of the same C2 problem "
                                   f"(n={res['n']}), stopped after {cpu_s:.1f} s: {cpu_u} local updates "
                                   f"(the first part of the factorization in the paper's order)",
                         "full_size_oracle": full_size_oracle()},
        "e2e": res["e2e"],
        "gpu_launches": res["launches"],
        "clocks": res["clocks"],
        # per op kind of the profiled warm-up step: op count, device time, counted FP64 flops and the
        # rate they give (the ops are latency-bound: see DESIGN §4/§6)
        "executor_ops": {k: {"ops": v["launches"], "ms": round(v["ms"], 2), "gflop": round(v["flops"] / 1e9, 3),
                             "gflops_per_s": round(v["flops"] / max(v["ms"], 1e-9) / 1e6, 2)}
                         for k, v in prof.items() if k not in ("k_matvec", "k_solve_sweep")},
        "kernels": {k: {"launches": v["launches"], "ms": round(v["ms"], 2)} for k, v in prof.items()
                    if k in ("k_matvec", "k_solve_sweep")},
    }
    print(json.dumps(line))


if __name__ == "__main__":
    main()
