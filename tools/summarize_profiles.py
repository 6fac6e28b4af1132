"""Summarise ncu outputs from gpurun_out/ into committed profiles/ files.

    python tools/summarize_profiles.py <round-tag> <launches.csv | -> <full.ncu-rep> <sweeps-in-capture> <workload>
profiles/traffic.json keeps one entry per workload (the bench's roofline `traffic`).
"""
import csv
import json
import subprocess
import sys
from collections import defaultdict

tag, launches, rep, sweeps, workload = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]), sys.argv[5]

rows = [r for r in csv.reader(open(launches)) if len(r) > 14 and r[0] not in ("ID",)] if launches != "-" else []
by = defaultdict(lambda: [0, 0.0])
for r in rows:
    name = r[4].replace("<unnamed>::", "").replace("(anonymous namespace)::", "").replace("void ", "").split("(")[0].split("<")[0].strip()
    by[name][0] += 1
    by[name][1] += float(r[14]) * (1e-3 if r[13] == "ns" else 1.0)   # -> us
tot = sum(v[1] for v in by.values())
out = [f"# {tag}: ncu launch list (`--metrics gpu__time_duration.sum --clock-control none`) of "
       f"`python bench.py --steps 2 --warmup 3 --no-cpu-baseline` ({workload})", "",
       "Cold-cache, serialised per-launch times: compare SHARES, not absolutes.", "",
       "| kernel | launches | total us | share |", "|---|---:|---:|---:|"]
for k, (n, us) in sorted(by.items(), key=lambda kv: -kv[1][1]):
    out.append(f"| `{k}` | {n} | {us:.1f} | {100 * us / tot:.1f}% |")
if rows:
    open(f"profiles/{tag}_launches.md", "w").write("\n".join(out) + "\n")

raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h, u, v = r[0], r[1], r[2]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio"]
m = {k: (x, uu) for k, uu, x in zip(h, u, v) if k in want}
scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
dr = float(m["dram__bytes_read.sum"][0]) * scale.get(m["dram__bytes_read.sum"][1], 1)
dw = float(m["dram__bytes_write.sum"][0]) * scale.get(m["dram__bytes_write.sum"][1], 1)
lines = [f"# {tag}: `ncu --set full` of the top kernel ({workload}, {sweeps} sweeps in one launch)", "",
         "| metric | unit | value |", "|---|---|---:|"]
for k in want:
    if k in m:
        lines.append(f"| {k} | {m[k][1]} | {m[k][0]} |")
lines += ["", f"DRAM bytes per sweep (read+write) = {(dr + dw) / sweeps / 1e6:.1f} MB"]
open(f"profiles/{tag}_top_kernel_ncu.md", "w").write("\n".join(lines) + "\n")
try:
    tj = json.load(open("profiles/traffic.json"))
    if "workload" in tj:  # (the one-entry format of earlier rounds)
        tj = {tj["workload"]: tj}
except Exception:
    tj = {}
tj[workload] = {"workload": workload, "kernel": "wavefront", "dram_bytes_per_sweep": (dr + dw) / sweeps,
                "source": f"profiles/{tag}_top_kernel_ncu.md"}
json.dump(tj, open("profiles/traffic.json", "w"), indent=1)
print("\n".join(out if rows else [])); print("\n".join(lines))
