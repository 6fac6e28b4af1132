"""NEXT-3 measurement: R right-hand sides of config 4's matrix (one plan) -- pobk_solve_multi
(A read once per step for all R) against R single solves on the fast single-RHS path (K2),
fixed 50 sweeps each; nnz-updates/s counts every right-hand side's updates.
    python tools/multi_rhs_perf.py [config] [sweeps]"""
import json, sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2401_00672_b200 as pk
from workloads import gen
name = sys.argv[1] if len(sys.argv) > 1 else "geoknn_1m"
nsw = int(sys.argv[2]) if len(sys.argv) > 2 else 50
base = gen.make(name)
plan = pk.Plan.from_system(base)
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for R in (1, 2, 4, 8):
    systems = [base] + [gen.make(name, b) for b in range(1, R)]
    fs = [torch.from_numpy(s.f).cuda() for s in systems]
    xs = [torch.zeros(s.m, dtype=torch.float64, device="cuda") for s in systems]
    plan.solve_multi(fs, xs, None, stop="none", max_sweeps=2)
    for x in xs: x.zero_()
    ev0.record(); plan.solve_multi(fs, xs, None, stop="none", max_sweeps=nsw); ev1.record(); torch.cuda.synchronize()
    t_multi = ev0.elapsed_time(ev1) * 1e-3
    for x in xs: x.zero_()
    ev0.record()
    for f, x in zip(fs, xs): plan.solve(f, x, None, stop="none", max_sweeps=nsw)
    ev1.record(); torch.cuda.synchronize()
    t_single = ev0.elapsed_time(ev1) * 1e-3
    upd = R * base.nnz * nsw
    print(json.dumps({"config": name, "R": R, "sweeps": nsw, "multi_s": round(t_multi, 5), "singles_s": round(t_single, 5),
                      "multi_nnz_updates_per_s": upd / t_multi, "singles_nnz_updates_per_s": upd / t_single,
                      "single_kernel": plan.layout_stats()["kernel"], "speedup": round(t_single / t_multi, 3)}), flush=True)
