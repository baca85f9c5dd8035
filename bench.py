"""Benchmark of the B200 H^2 hot path (contract: one JSON line on rank 0).

Workload C1 (BASELINE.json configs[1]): 2D P1 Laplacian on 128x128 nodes
(n = 16,384), leaf 32, eta = 2, fixed rank 16.  One step = U seeded random rank-k_u local
low-rank updates on random admissible blocks (h2_lowrank_update, U0-U6) followed by one H^2
matvec (h2_matvec).  The matrix is not reset between steps (the update stream continues; after
the warm-up the ranks sit at the fixed-rank steady state).  metric value = updates per second.

Multi-GPU: the update chain does not shard (replicas only); --gpus N runs N
independent replicas (one process per GPU), value = total updates / max-over-ranks time.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--ku 16] [--updates 1000]
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


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    d = json.load(open(p)) if os.path.exists(p) else {}
    f = os.path.join(ROOT, "profiles", "fp64_peak.json")
    fp = json.load(open(f)) if os.path.exists(f) else {}
    return d, fp


def _workload(args):
    from inputs import config
    from inputs.updates import c1_stream
    c = config("C1")
    return c


def _clock_sampler_start():
    try:
        f = open(os.path.join("/tmp", f"h2_clocks_{os.getpid()}.csv"), "w")
        p = subprocess.Popen(
            ["nvidia-smi", "--query-gpu=index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
             "--format=csv,noheader,nounits", "-lms", "100"], stdout=f, stderr=subprocess.DEVNULL)
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


def run_gpu(args, rank, world):
    import torch
    import paper_1402_5056_b200 as P
    from inputs.updates import c1_stream

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream()
    c = _workload(args)
    n = c["n"]
    t = P.h2_cluster_tree(c["points"], c["leaf"])
    bt = P.h2_block_tree(t, t, c["eta"])
    Z = P.h2_from_sparse(bt, c["A"], rank_cap=32, update_cap=32)
    trunc = P.Trunc(1e-12, 0.0, 16)
    adm = [(int(bt.t[b]), int(bt.s[b]), t.size(bt.t[b]), t.size(bt.s[b])) for b in np.nonzero(bt.kind == 1)[0]]
    U = args.updates
    nsteps = args.warmup + args.steps + 1  # +1: profiled pass
    ups = c1_stream(adm, U * nsteps, args.ku, seed=args.seed)
    # inputs resident in HBM before the clock starts: one flat buffer per step
    def pack(batch):
        offs, flat = [], []
        pos = 0
        for (t0, s0, X, Y) in batch:
            xs, ys = X.T.ravel(), Y.T.ravel()  # column-major
            offs.append((t0, s0, pos, X.shape[0], pos + xs.size, Y.shape[0]))
            flat += [xs, ys]
            pos += xs.size + ys.size
        return offs, np.concatenate(flat)
    packed = [pack(ups[i * U:(i + 1) * U]) for i in range(nsteps)]
    dbufs = [torch.from_numpy(p[1]).to(dev) for p in packed]
    x = torch.from_numpy(np.random.default_rng(0).standard_normal(n)).to(dev)
    y = torch.zeros(n, dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # 256 MiB > 126 MB L2
    lib = P.h2._lib
    C = P.h2.C
    ctr = P.h2._ctrunc(trunc)
    sptr = C.c_void_p(stream.cuda_stream)
    k = args.ku

    def step(i, buf):
        base = buf.data_ptr()
        for (t0, s0, xo, mt, yo, ms) in packed[i][0]:
            rc = lib.h2_lowrank_update(Z.h, t0, s0, k, 1.0, C.c_void_p(base + 8 * xo), mt,
                                       C.c_void_p(base + 8 * yo), ms, C.byref(ctr), sptr)
            if rc:
                P.h2._check(rc)
        P.h2._check(lib.h2_matvec(Z.h, 0, 1.0, C.c_void_p(x.data_ptr()), 0.0, C.c_void_p(y.data_ptr()), sptr))

    for i in range(args.warmup):
        step(i, dbufs[i])
    torch.cuda.synchronize()
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    clk_p, clk_f = _clock_sampler_start() if rank == 0 else (None, None)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for j in range(args.steps):
        flush.fill_(float(j))  # L2 flush between timed steps (outside the timed events)
        ev[j][0].record(stream)
        step(args.warmup + j, dbufs[args.warmup + j])
        ev[j][1].record(stream)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = _clock_sampler_stop(clk_p, clk_f, dev.index) if rank == 0 else None
    ms = sum(a.elapsed_time(b) for a, b in ev)
    if dist is not None:
        tt = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    # profiled pass (one more step, same structure) -> per-kernel launches, time, flops, bytes
    P.h2_profile_enable(True)
    step(nsteps - 1, dbufs[nsteps - 1])
    prof = P.h2_profile_read()
    P.h2_profile_enable(False)
    flags = P.h2_check_device_flags(Z)
    # matvec GB/s: 100 back-to-back calls, algorithmic bytes of the current representation
    sto = P.h2_storage_report(Z)
    mv_bytes = 8.0 * float(sto.sum()) + 16.0 * n
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(5):
        P.h2_matvec(Z, x, y)
    e0.record(stream)
    for _ in range(100):
        P.h2_matvec(Z, x, y)
    e1.record(stream)
    torch.cuda.synchronize()
    mv_ms = e0.elapsed_time(e1) / 100
    # e2e: same steps through host buffers (pinned), H2D of the step's factors and D2H of y inside
    host = [torch.from_numpy(p[1]).pin_memory() for p in packed[:min(3, args.steps)]]
    yh = torch.empty(n, dtype=torch.float64).pin_memory()
    ebuf = torch.empty_like(dbufs[0])
    torch.cuda.synchronize()
    e2e_ms = 0.0
    for j, hb in enumerate(host):
        if ebuf.numel() < hb.numel():
            ebuf = torch.empty(hb.numel(), dtype=torch.float64, device=dev)
        s0e, s1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0e.record(stream)
        ebuf[:hb.numel()].copy_(hb, non_blocking=True)
        step(j, ebuf)
        yh.copy_(y, non_blocking=True)
        s1e.record(stream)
        torch.cuda.synchronize()
        e2e_ms += s0e.elapsed_time(s1e)
    e2e_ms /= len(host)
    h2d = int(np.mean([hb.numel() * 8 for hb in host]))
    return dict(ms=ms, prof=prof, flags=flags, mv_ms=mv_ms, mv_bytes=mv_bytes, sto=sto.tolist(), clocks=clocks,
                e2e_ms=e2e_ms, h2d=h2d, d2h=n * 8, n=n)


def oracle_rate(n_updates, ku, seed, with_matvec=True):
    """Time the oracle (as it stands) on a bounded sample of the same workload: the first
    n_updates of the seeded C1 stream on a fresh matrix, plus one matvec.  Single thread."""
    try:
        from threadpoolctl import threadpool_limits
        lim = threadpool_limits(1)
    except Exception:
        lim = None
    from inputs import config
    from inputs.updates import c1_stream
    from oracle.structure import ClusterTree, BlockTree
    from oracle.h2 import from_sparse
    from oracle.update import Updater, Trunc
    c = config("C1")
    ot = ClusterTree(c["points"], c["leaf"])
    ob = BlockTree(ot, ot, c["eta"])
    OZ = from_sparse(ob, c["A"])
    up = Updater(OZ, Trunc(1e-12, 0.0, 16))
    adm = [(int(ob.t[b]), int(ob.s[b]), ot.size(ob.t[b]), ot.size(ob.s[b])) for b in ob.adm]
    ups = c1_stream(adm, n_updates, ku, seed=seed)
    t0 = time.perf_counter()
    for (a, b, X, Y) in ups:
        up(a, b, X, Y)
    if with_matvec:
        OZ.matvec(np.ones(ot.n))
    dt = time.perf_counter() - t0
    return n_updates / dt, dt


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ku", type=int, default=16)
    ap.add_argument("--updates", type=int, default=1000)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--cpu-sample", type=int, default=1500, help="oracle updates timed for cpu_baseline")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    config = {"workload": "C1", "n": 16384, "mesh": "128x128 2D P1 Laplacian", "leaf": 32, "eta": 2.0,
              "rank": "fixed 16 (rel guard 1e-12)", "k_u": args.ku, "updates_per_step": args.updates,
              "step": f"{args.updates} local low-rank updates + 1 matvec", "l2": "flushed between timed steps (256 MiB write)",
              "parallelism": f"replicas x{args.gpus}"}

    if args.impl == "reference":
        if rank != 0:
            return
        per = max(10, args.updates // 10)
        t_all = 0.0
        for _ in range(args.warmup):
            oracle_rate(per, args.ku, args.seed)
        for _ in range(args.steps):
            r, dt = oracle_rate(per, args.ku, args.seed)
            t_all += dt
        value = args.steps * per / t_all
        line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_all / args.steps,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic", "config": dict(config, updates_per_step=per),
                "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                                 "sample": f"first {per} updates of the seeded C1 stream (fresh matrix) + 1 matvec per step"},
                "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
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
    measured, fp = _peaks()
    total_updates = args.updates * args.steps * world
    value = total_updates / (res["ms"] / 1e3)
    prof = res["prof"]
    upd_kernels = {k: v for k, v in prof.items() if k.startswith("k_upd")}
    launches_per_step = sum(v["launches"] for v in prof.values())
    # dominant kernel of the step (largest summed event time in the profiled step)
    dom_name, dom = max(prof.items(), key=lambda kv: kv[1]["ms"])
    fp64_peak = fp.get("fp64_fma_tflops") or 37.0
    if dom["bytes"] > 0 and dom["flops"] / max(dom["bytes"], 1) < 6:
        achieved = dom["bytes"] / dom["launches"] / (dom["ms"] / dom["launches"] / 1e3) / 1e9
        roof = {"kernel": dom_name, "bound": "hbm", "achieved": achieved, "peak": measured.get("hbm_gbs", 6650.0),
                "unit": "GB/s", "traffic": None}
    else:
        achieved = dom["flops"] / dom["launches"] / (dom["ms"] / dom["launches"] / 1e3) / 1e12
        roof = {"kernel": dom_name, "bound": "alu", "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s",
                "traffic": None, "peak_source": "profiles/fp64_peak.json (FP64 FMA microbenchmark)" if fp else
                "B200 FP64 nominal 37 TFLOP/s (148 SMs x 64 DFMA/clk x 1.965 GHz)"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["share_of_step"] = dom["ms"] / sum(v["ms"] for v in prof.values())
    roof["launches_per_step"] = dom["launches"]
    cpu_rate, cpu_dt = oracle_rate(args.cpu_sample, args.ku, args.seed)
    mv_gbs = res["mv_bytes"] / (res["mv_ms"] / 1e3) / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": res["ms"] / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config,
        "roofline": roof,
        "cpu_baseline": {"value": cpu_rate, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"first {args.cpu_sample} updates of the seeded C1 stream on a fresh matrix "
                                   f"+ 1 matvec ({cpu_dt:.1f} s, numpy single thread)"},
        "e2e": {"value": args.updates / (res["e2e_ms"] / 1e3), "unit": UNIT,
                "h2d_bytes_per_step": res["h2d"], "d2h_bytes_per_step": res["d2h"]},
        "gpu_launches": launches_per_step * args.steps,
        "clocks": res["clocks"],
        "matvec": {"GBps": mv_gbs, "ms": res["mv_ms"], "bytes": res["mv_bytes"],
                   "frac_of_hbm": mv_gbs / measured.get("hbm_gbs", 6650.0),
                   "note": "C1 matrix (~%.0f MB) is L2-resident: HBM does not bind here" % (res["mv_bytes"] / 1e6)},
        "kernels": {k: {"launches": v["launches"], "ms": round(v["ms"], 4),
                        "gflops_per_s": (v["flops"] / (v["ms"] / 1e3) / 1e9) if v["ms"] else None}
                    for k, v in prof.items()},
        "device_flags": res["flags"],
        "storage_scalars": res["sto"],
    }
    print(json.dumps(line))


if __name__ == "__main__":
    main()
