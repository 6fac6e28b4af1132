"""Small solves on every kernel family, for compute-sanitizer:
    compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize_run.py
K1 (launch), K3 (smem, both layouts via the two systems), K4 (cluster), K2 (wavefront: RSE,
RELRES, fixed count, a nonzero x0, small tiles so most rows cross tiles) and the batch lanes; each
result is checked against the oracle's iterates (bitwise, thr = 0)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import torch
import oracle as O
import paper_2401_00672_b200 as pk
from workloads import gen

torch.cuda.set_device(0)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()
cases = [("lap2d5_32", None, "launch", {}), ("lap2d5_32", None, "smem", {}), ("lap2d5_32", None, "cluster", {}),
         ("lap3d7_64", 16, "wavefront", {"tile_rows": 64}), ("randband_20k", 3000, "wavefront", {}),
         ("geoknn_1m", 6000, "wavefront", {})]
bad = 0
for name, n, kernel, kw in cases:
    s = gen.make(name, n=n) if n else gen.make(name)
    pre = O.preprocess(s.m, s.indptr, s.indices, s.data)
    try:
        plan = pk.Plan.from_system(s, kernel=kernel, **kw)
    except pk.PobkError as e:
        print(f"{name} {kernel}: n/a ({e})"); continue
    x0 = np.random.default_rng(3).standard_normal(s.m)
    x = d(x0)
    plan.solve(d(s.f), x, d(s.x_star), max_sweeps=4, stop="none")
    ok = np.array_equal(x.cpu().numpy(), O.run_sweeps(pre, s.f, 4, x0=x0))
    x = d(np.zeros(s.m))
    r1 = plan.solve(d(s.f), x, d(s.x_star), tol=0.3, max_sweeps=50)
    x = d(np.zeros(s.m))
    r2 = plan.solve(d(s.f), x, None, tol=0.3, max_sweeps=50, stop="relres")
    rn = plan.residual_norm(d(s.f), x)
    print(f"{name}@{s.m} {kernel}: fixed-count bitwise {ok}, rse stop {r1.sweeps}, relres stop {r2.sweeps}, "
          f"kernel {r2.as_dict()['kernel']}, residual {rn:.3e}", flush=True)
    bad += not ok
systems = [gen.make("batch9pt_1024", b, n=64) for b in range(3)]
tr = pk.half_gpu_tile_rows(systems[0].m)
plans = [pk.Plan.from_system(s, kernel="wavefront", tile_rows=tr) for s in systems]
xs = [d(np.zeros(s.m)) for s in systems]
reps = pk.solve_batch(plans, [d(s.f) for s in systems], xs, [d(s.x_star) for s in systems], tol=0.2)
print("batch lanes:", [r.sweeps for r in reps])
torch.cuda.synchronize()
print("SANITIZE-RUN", "FAIL" if bad else "OK")
