"""NEXT-2 / NEXT-4 measurement: the paper-literal k-block POBK (K5) on the small BASELINE configs --
per k: the zn/nn diagnostics (Definitions 1-2), Oclass pairs / Nclass, iterations to
RSE < tol, time per iteration and time to tolerance on the GPU, beside the row-level POBK
(the hot path).  Prints one JSON line per case.
    python tools/blocks_perf.py"""
import json, sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2401_00672_b200 as pk
from workloads import gen

cases = [("lap2d5_32", None, [2, 5, 7, 10, 19], 0.05, 1e-6), ("randband_20k", None, [10, 19], 0.3, 1e-6)]
for name, n, ks, thr, tol in cases:
    s = gen.make(name, n=n) if n else gen.make(name)
    d = lambda a: torch.from_numpy(a).cuda()
    f, xs = d(s.f), d(s.x_star)
    row = pk.Plan.from_system(s)
    x = torch.zeros(s.m, dtype=torch.float64, device="cuda")
    r = row.solve(f, x, xs, tol=tol)
    print(json.dumps({"config": name, "method": "row-level POBK (hot path)", "kernel": r.as_dict()["kernel"],
                      "iterations": r.sweeps, "ms_to_tol": round(r.solve_seconds * 1e3, 3),
                      "us_per_iteration": round(r.sweep_seconds / max(r.sweeps, 1) * 1e6, 2)}), flush=True)
    for k in ks:
        t0 = time.time()
        try:
            p = pk.Plan.from_system_blocks(s, k=k, thr=thr)
        except pk.PobkError as e:
            print(json.dumps({"config": name, "k": k, "error": str(e)})); continue
        tp = time.time() - t0
        info = p.blocks_info()
        x.zero_()
        p.solve(f, x, xs, max_sweeps=2, stop="none")
        x.zero_()
        r = p.solve(f, x, xs, tol=tol, max_sweeps=20000)
        print(json.dumps({"config": name, "method": "k-block POBK (K5)", "k": k, "thr": thr, "pairs": len(info["pairs"]),
                          "nclass": len(info["nclass"]), "zn": round(info["zn"], 4), "nn": round(info["nn"], 4),
                          "iterations": r.sweeps, "termination": r.as_dict()["termination"], "final_rse": r.final_value,
                          "ms_to_tol": round(r.solve_seconds * 1e3, 3),
                          "us_per_iteration": round(r.sweep_seconds / max(r.sweeps, 1) * 1e6, 2),
                          "preprocess_s": round(tp, 2)}), flush=True)
        p.close()
