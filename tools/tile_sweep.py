"""us/sweep of K2 as a function of the tile size (development aid).
    python tools/tile_sweep.py config tile_rows[,tile_rows...] [sweeps]"""
import sys, json
import torch
sys.path.insert(0, ".")
import paper_2401_00672_b200 as pk
from workloads import gen
name = sys.argv[1]
trs = [int(v) for v in sys.argv[2].split(",")]
nsw = int(sys.argv[3]) if len(sys.argv) > 3 else 50
s = gen.make(name)
f = torch.from_numpy(s.f).cuda(); xs = torch.from_numpy(s.x_star).cuda()
for tr in trs:
    plan = pk.Plan.from_system(s, kernel="wavefront", tile_rows=tr)
    x = torch.zeros(s.m, dtype=torch.float64, device="cuda")
    plan.solve(f, x, xs, max_sweeps=3, stop="none")
    x.zero_()
    r = plan.solve(f, x, xs, max_sweeps=nsw, stop="rse", tol=0.0)
    st = plan.layout_stats()
    print(json.dumps({"cfg": name, "tile_rows": tr, "tiles": st.get("tiles", st.get("T")), "private": round(st.get("private_nnz_frac", 0), 3),
                      "us_per_sweep": round(r.sweep_seconds / r.sweeps * 1e6, 2), "rse": r.final_value}), flush=True)
    plan.close()
