"""Quick per-kernel timing of fixed-count sweeps on one config (development aid, not the bench)."""
import sys, time, json
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2401_00672_b200 as pk
from workloads import gen

name = sys.argv[1] if len(sys.argv) > 1 else "geoknn_1m"
n = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "-" else None
kernels = sys.argv[3].split(",") if len(sys.argv) > 3 else ["launch", "wavefront"]
nsw = int(sys.argv[4]) if len(sys.argv) > 4 else 50
t = time.time(); s = gen.make(name, n=n) if n else gen.make(name); print("gen", round(time.time() - t, 1), "s", s.m, s.nnz, flush=True)
B = 12 * s.nnz + 12 * s.m
f = torch.from_numpy(s.f).cuda(); xs = torch.from_numpy(s.x_star).cuda()
for k in kernels:
    try:
        t = time.time(); plan = pk.Plan.from_system(s, kernel=k); tp = time.time() - t
    except pk.PobkError as e:
        print(k, "n/a", e); continue
    print(k, plan.layout_stats(), flush=True)
    x = torch.zeros(s.m, dtype=torch.float64, device="cuda")
    plan.solve(f, x, xs, max_sweeps=3, stop="none")
    for stop in ("none", "rse"):
        x.zero_()
        r = plan.solve(f, x, xs, max_sweeps=nsw, stop=stop, tol=0.0)
        us = r.sweep_seconds / max(r.sweeps, 1) * 1e6
        print(json.dumps({"kernel": k, "stop": stop, "prep_s": round(tp, 2), "sweeps": r.sweeps, "us_per_sweep": round(us, 2),
                          "GBps": round(B / (us * 1e-6) / 1e9, 1), "frac_hbm": round(B / (us * 1e-6) / 6556.5e9, 3),
                          "value": r.final_value, "launches": r.launches}), flush=True)
    plan.close()
