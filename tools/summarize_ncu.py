"""Summaries of the ncu outputs of tools/prof_r02.sh (gpurun_out/) into profiles/r02/ (text)."""
import collections
import csv
import io
import json
import subprocess
import sys

out = sys.argv[1] if len(sys.argv) > 1 else "profiles/r02"
rows = list(csv.reader(open("gpurun_out/launches_bench.csv")))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
kn, mv = h.index("Kernel Name"), h.index("Metric Value")
ex, agg = [], collections.defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if len(r) <= mv:
        continue
    name = r[kn].split("(")[0].split("::")[-1]
    v = float(r[mv].replace(",", ""))
    agg[name][0] += 1
    agg[name][1] += v
    if name == "k_exec_cluster":
        ex.append(v)
tot = sum(v[1] for v in agg.values())
with open(f"{out}/ncu_launches_bench_C2_summary.txt", "w") as f:
    f.write("ncu --metrics gpu__time_duration.sum --clock-control none --csv  python bench.py --warmup 3 --steps 1 --cpu-budget 2\n"
            "(C2, n = 262,144; 4 factorizations + PCG + matvecs; per-launch times are cold-cache and serialised)\n")
    f.write(f"{'kernel':28s} {'launches':>9s} {'total ms':>12s} {'share':>8s}\n")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        f.write(f"{k:28s} {v[0]:9d} {v[1] / 1e6:12.2f} {100 * v[1] / tot:7.2f}%\n")
    f.write(f"k_exec_cluster launches: {len(ex)}, median {sorted(ex)[len(ex) // 2] / 1e6:.1f} ms, max {max(ex) / 1e6:.1f} ms\n")


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(txt)))
    return r[0], r[1], r[2:]


h, u, body = raw("gpurun_out/prof_matvec_L.ncu-rep")
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size",
        "launch__block_size", "launch__registers_per_thread", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active"]
idx = [(w, h.index(w)) for w in want if w in h]
with open(f"{out}/ncu_matvec_L_C2_raw.txt", "w") as f:
    f.write(str([w for w, _ in idx]) + "\n" + str([u[i] for _, i in idx]) + "\n")
    rd = wr = 0.0
    n = 0
    for row in body:
        f.write(str([row[i][:28] for _, i in idx]) + "\n")
        rd += float(row[h.index("dram__bytes_read.sum")])
        wr += float(row[h.index("dram__bytes_write.sum")])
        n += 1
    f.write(f"sum over {n} launches: dram read {rd:.1f} + write {wr:.1f} (units as above, per 2 products if 12 launches)\n")
h, u, body = raw("gpurun_out/prof_exec.ncu-rep")
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size", "launch__cluster_size",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio"]
d = {k: (body[0][h.index(k)], u[h.index(k)]) for k in keys if k in h}
json.dump(d, open(f"{out}/ncu_exec_cluster_C2_raw.json", "w"), indent=1)
print(open(f"{out}/ncu_launches_bench_C2_summary.txt").read())
print(open(f"{out}/ncu_matvec_L_C2_raw.txt").read())
print(d)
