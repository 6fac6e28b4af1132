"""NEXT-4 measurement: the residual-ordered sweep (opts.order = residual) against the paper's cyclic
schedule -- sweeps and GPU time to the RSE tolerance on the BASELINE configs.
    python tools/order_perf.py"""
import json, sys
sys.path.insert(0, ".")
import torch
import paper_2401_00672_b200 as pk
from workloads import gen
for name, tol, cap in [("lap2d5_32", 1e-6, 500000), ("randband_20k", 1e-6, 5000), ("lap3d7_64", 0.1, 5000),
                       ("geoknn_1m", 0.1, 5000)]:
    s = gen.make(name)
    p = pk.Plan.from_system(s)
    f, xs = torch.from_numpy(s.f).cuda(), torch.from_numpy(s.x_star).cuda()
    for order in ("schedule", "residual"):
        x = torch.zeros(s.m, dtype=torch.float64, device="cuda")
        p.solve(f, x, xs, max_sweeps=2, stop="none", order=order)
        x.zero_()
        r = p.solve(f, x, xs, tol=tol, max_sweeps=cap, order=order)
        print(json.dumps({"config": name, "order": order, "kernel": r.as_dict()["kernel"], "sweeps": r.sweeps,
                          "termination": r.as_dict()["termination"], "ms_to_tol": round(r.solve_seconds * 1e3, 3),
                          "us_per_sweep": round(r.sweep_seconds / max(1, r.sweeps) * 1e6, 2)}), flush=True)
