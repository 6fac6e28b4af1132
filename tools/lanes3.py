"""Config 5 on 2 vs 3 concurrent lanes (development aid): pobk_solve_batch of the GPU's 8 systems
with K2 plans built by lane_tile_rows(m, L); times, kernel, tiles, and bitwise agreement."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2401_00672_b200 as pk  # noqa: E402
from workloads import gen  # noqa: E402

systems = [gen.make("batch9pt_1024", b) for b in range(8)]
fs = [torch.from_numpy(s.f).cuda() for s in systems]
xss = [torch.from_numpy(s.x_star).cuda() for s in systems]
out = {}
for lanes in (2, 3):
    tr = pk.lane_tile_rows(systems[0].m, lanes)
    plans = [pk.Plan.from_system(s, kernel="auto", tile_rows=tr) for s in systems]
    xs = [torch.zeros(s.m, dtype=torch.float64, device="cuda") for s in systems]
    best = 1e9
    for it in range(4):
        for x in xs:
            x.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        reps = pk.solve_batch(plans, fs, xs, xss, tol=0.1, stop="rse")
        torch.cuda.synchronize()
        if it:
            best = min(best, time.perf_counter() - t0)
    nnz = sum(r.sweeps * p.nnz for r, p in zip(reps, plans))
    out[lanes] = [x.cpu().numpy() for x in xs]
    st = plans[0].layout_stats()
    print(json.dumps({"lanes": lanes, "tile_rows": tr, "kernel": st.get("kernel"), "tiles": st.get("ntiles"),
                      "threads": st.get("threads"), "private": round(st.get("private_nnz_frac", 0), 3),
                      "ms": round(best * 1e3, 2), "G": round(nnz / best / 1e9, 1), "sweeps": [r.sweeps for r in reps]}), flush=True)
    for p in plans:
        p.close()
print("bitwise", all(np.array_equal(a, b) for a, b in zip(out[2], out[3])))
