"""NEXT-1 measurement: the thr > 0 mode (near-orthogonal rows share a category) --
categories per sweep, Gershgorin guard, sweeps and GPU time to the RSE tolerance -- beside thr = 0.
    python tools/thr_perf.py"""
import json, sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2401_00672_b200 as pk
from workloads import gen
cases = [("lap2d5_32", None, [0.0, 0.11], 1e-6, 500000), ("geoknn_1m", None, [0.0, 0.05], 0.1, 5000),
         ("lap3d7_64", None, [0.0, 0.06], 0.1, 5000)]
for name, n, thrs, tol, cap in cases:
    s = gen.make(name, n=n) if n else gen.make(name)
    f, xs = torch.from_numpy(s.f).cuda(), torch.from_numpy(s.x_star).cuda()
    for thr in thrs:
        guard_ok = True
        try:
            pk.Plan.from_system(s, thr=thr, guard=1, device=-1).close()
        except pk.PobkError:
            guard_ok = False
        p = pk.Plan.from_system(s, thr=thr)
        x = torch.zeros(s.m, dtype=torch.float64, device="cuda")
        p.solve(f, x, xs, max_sweeps=2, stop="none")
        x.zero_()
        r = p.solve(f, x, xs, tol=tol, max_sweeps=cap)
        print(json.dumps({"config": name, "thr": thr, "categories": p.nsteps, "gershgorin_guard_ok": guard_ok,
                          "kernel": r.as_dict()["kernel"], "sweeps": r.sweeps, "termination": r.as_dict()["termination"],
                          "final_rse": r.final_value, "ms_to_tol": round(r.solve_seconds * 1e3, 3),
                          "us_per_sweep": round(r.sweep_seconds / max(1, r.sweeps) * 1e6, 2)}), flush=True)
        p.close()
