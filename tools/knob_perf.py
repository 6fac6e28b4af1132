"""K2 us/sweep on one config for several runtime knob settings (development aid).
    python tools/knob_perf.py CONFIG "VL=-1" "STRICT=1,IREG=1;STRICT=0,IREG=0" [nsweeps]
Each semicolon-separated setting sets POBK_K2_<KEY> for the solves of one plan (per VL)."""
import os, sys, json
sys.path.insert(0, ".")
import torch
import paper_2401_00672_b200 as pk
from workloads import gen
name = sys.argv[1]; vls = sys.argv[2].split(","); sets = sys.argv[3].split(";")
nsw = int(sys.argv[4]) if len(sys.argv) > 4 else 50
s = gen.make(name)
B = 12 * s.nnz + 12 * s.m
f = torch.from_numpy(s.f).cuda(); xs = torch.from_numpy(s.x_star).cuda()
x = torch.zeros(s.m, dtype=torch.float64, device="cuda")
ref = None
for vl in vls:
    os.environ["POBK_K2_VL"] = vl.split("=")[-1]
    plan = pk.Plan.from_system(s, kernel="wavefront")
    for st in sets:
        for kv in st.split(","):
            k, v = kv.split("=")
            os.environ["POBK_K2_" + k] = v
        x.zero_(); plan.solve(f, x, xs, max_sweeps=3, stop="none")
        best = 1e9
        for rep in range(3):
            x.zero_()
            r = plan.solve(f, x, xs, max_sweeps=nsw, stop="none", tol=0.0)
            best = min(best, r.sweep_seconds / r.sweeps * 1e6)
        xc = x.cpu().numpy()
        same = None if ref is None else bool((xc == ref).all())
        if ref is None: ref = xc
        print(json.dumps({"config": name, "VL": vl, "set": st, "us_per_sweep": round(best, 2),
                          "frac_hbm": round(B / (best * 1e-6) / 6542.4e9, 3), "bitwise_same": same}), flush=True)
    plan.close()
