"""Several right-hand sides of ONE matrix through pobk_solve_batch: one
plan per right-hand side (the matrix's preprocessing is shared on the host: perm and partition are
bitwise the same), half-GPU K2 tilings so two solves run side by side.  Compares with back-to-back
full-GPU solves; results must be bitwise equal (development/reporting aid).

    python tools/multi_rhs.py [config] [R] [lanes]
"""
import sys, time, json
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2401_00672_b200 as pk
from workloads import gen
from bench import TOL
name = sys.argv[1] if len(sys.argv) > 1 else "geoknn_1m"
R = int(sys.argv[2]) if len(sys.argv) > 2 else 2
s = gen.make(name)
rng = np.random.default_rng(7)
import scipy.sparse as sp
A = sp.csr_matrix((s.data, s.indices, s.indptr), shape=(s.m, s.m))
xstars = [s.x_star] + [rng.standard_normal(s.m) for _ in range(R - 1)]
fs = [torch.from_numpy(A @ xs).cuda() for xs in xstars]
xss = [torch.from_numpy(xs).cuda() for xs in xstars]
tol = TOL[name]
res = {}
nl = int(sys.argv[3]) if len(sys.argv) > 3 else 2  # lanes (tiles per system: SMs / nl)
sms = torch.cuda.get_device_properties(0).multi_processor_count
for mode in ("back-to-back", "lanes"):
    tr = 0 if mode == "back-to-back" else -(-s.m // max(1, sms // nl - 2))
    plans = [pk.Plan.from_system(s, tile_rows=tr) for _ in range(R)]
    xs = [torch.zeros(s.m, dtype=torch.float64, device="cuda") for _ in range(R)]
    for it in range(3):
        for x in xs: x.zero_()
        torch.cuda.synchronize(); t0 = time.perf_counter()
        if mode == "lanes":
            reps = pk.solve_batch(plans, fs, xs, xss, tol=tol, stop="rse")
        else:
            reps = [p.solve(f, x, xst, tol=tol, stop="rse") for p, f, x, xst in zip(plans, fs, xs, xss)]
        torch.cuda.synchronize(); t = time.perf_counter() - t0
    upd = sum(r.sweeps * s.nnz for r in reps)
    res[mode] = [x.cpu().numpy() for x in xs]
    print(json.dumps({"config": name, "rhs": R, "mode": mode, "tiles": plans[0].layout_stats()["ntiles"],
                      "ms": round(t * 1e3, 2), "sweeps": [r.sweeps for r in reps],
                      "G_nnz_updates_per_s": round(upd / t / 1e9, 1), "sweep_ms": [round(r.sweep_seconds * 1e3, 2) for r in reps], "solve_ms": [round(r.solve_seconds * 1e3, 2) for r in reps]}), flush=True)
    for p in plans: p.close()
print("bitwise equal:", all(np.array_equal(a, b) for a, b in zip(res["back-to-back"], res["lanes"])))
