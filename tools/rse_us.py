"""Development: K2 us/sweep with and without the per-sweep RSE check on one config (min of 5),
with the stop sweep, final RSE and a checksum of x (bitwise comparisons across builds).
    PYTHONPATH=. python tools/rse_us.py [workload] [tol]"""
import hashlib
import sys

import torch

import paper_2401_00672_b200 as pk
from workloads import gen

name = sys.argv[1] if len(sys.argv) > 1 else "geoknn_1m"
tol = float(sys.argv[2]) if len(sys.argv) > 2 else 0.1
s = gen.make(name, 0)
plan = pk.Plan.from_system(s, kernel="wavefront")
f, xs = torch.from_numpy(s.f).cuda(), torch.from_numpy(s.x_star).cuda()
x = torch.zeros(s.m, dtype=torch.float64, device="cuda")
for stop in ("rse", "none"):
    best, r = 1e9, None
    for i in range(6):
        x.zero_()
        r = plan.solve(f, x, xs, tol=tol, stop=stop, max_sweeps=50 if stop == "none" else 500000)
        if i:
            best = min(best, r.sweep_seconds / r.sweeps * 1e6)
    h = hashlib.sha1(x.cpu().numpy().tobytes()).hexdigest()[:12]
    print(f"{name} stop={stop:4s} {best:7.2f} us/sweep sweeps={r.sweeps} final={r.final_value!r} x={h}")
