"""Top SASS instructions by warp-stall samples from an ncu report (development aid).
    python tools/ncu_hot.py report.ncu-rep [N]"""
import csv, subprocess, sys, io
rep = sys.argv[1]; N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["/usr/local/cuda/bin/ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]; data = rows[2:]
ia, isrc, iss = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[iss] or 0) for r in data if len(r) > iss)
print("total samples", tot)
idx = sorted(range(len(data)), key=lambda i: -int(data[i][iss] or 0))[:N]
for i in sorted(idx):
    r = data[i]
    print(f"{i:6d} {int(r[iss]):7d} {100*int(r[iss])/tot:5.1f}%  {r[isrc].strip()[:90]}")
