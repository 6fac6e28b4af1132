"""Batched systems (config 5): back-to-back full-GPU solves vs two concurrent half-GPU lanes
(development aid; results must be bitwise equal).   python tools/batch_lanes.py [nsys]"""
import sys, time, json
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2401_00672_b200 as pk
from workloads import gen
nb = int(sys.argv[1]) if len(sys.argv) > 1 else 8
systems = [gen.make("batch9pt_1024", b) for b in range(nb)]
fs = [torch.from_numpy(s.f).cuda() for s in systems]
xss = [torch.from_numpy(s.x_star).cuda() for s in systems]
out = {}
for mode in ("full", "half"):
    tr = 0 if mode == "full" else pk.half_gpu_tile_rows(systems[0].m)
    plans = [pk.Plan.from_system(s, tile_rows=tr) for s in systems]
    xs = [torch.zeros(s.m, dtype=torch.float64, device="cuda") for s in systems]
    for it in range(3):
        for x in xs: x.zero_()
        torch.cuda.synchronize(); t0 = time.perf_counter()
        reps = pk.solve_batch(plans, fs, xs, xss, tol=0.1, stop="rse")
        torch.cuda.synchronize(); t = time.perf_counter() - t0
    sweeps = [r.sweeps for r in reps]
    nnz = sum(r.sweeps * p.nnz for r, p in zip(reps, plans))
    out[mode] = [x.cpu().numpy() for x in xs]
    print(json.dumps({"mode": mode, "tiles": plans[0].layout_stats().get("ntiles"), "ms": round(t * 1e3, 2), "sweeps": sweeps,
                      "G_nnz_updates_per_s": round(nnz / t / 1e9, 1)}), flush=True)
    for p in plans: p.close()
print("bitwise equal:", all(np.array_equal(a, b) for a, b in zip(out["full"], out["half"])))
