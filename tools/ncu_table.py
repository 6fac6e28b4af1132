"""Markdown table of one ncu --set full capture (development/reporting aid).
    python tools/ncu_table.py <rep> <out.md> <title> <sweeps-in-capture>"""
import csv, subprocess, sys
rep, out, title, sweeps = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4])
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h, u, v = r[0], r[1], r[2]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio"]
m = {k: (x, uu) for k, uu, x in zip(h, u, v) if k in want}
lines = [f"# {title} ({sweeps} sweeps in one launch)", "", "| metric | unit | value |", "|---|---|---:|"]
lines += [f"| {k} | {m[k][1]} | {m[k][0]} |" for k in want if k in m]
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
