"""K1 on the sliced ELL copy (K1E) beside the CSR kernels (POBK_K1_CSR=1): fixed sweeps on the
launch path, thr = 0 and thr > 0, bitwise check between the two.
    python tools/k1e_perf.py"""
import json, os, sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2401_00672_b200 as pk
from workloads import gen
cases = [("geoknn_1m", 0.0, 20), ("geoknn_1m", 0.05, 20), ("lap3d7_64", 0.0, 20), ("lap3d7_64", 0.06, 20),
         ("randband_20k", 0.0, 50)]
for name, thr, nsw in cases:
    s = gen.make(name)
    f, xs = torch.from_numpy(s.f).cuda(), torch.from_numpy(s.x_star).cuda()
    out = {}
    for mode in ("csr", "ell"):
        if mode == "csr":
            os.environ["POBK_K1_CSR"] = "1"
        else:
            os.environ.pop("POBK_K1_CSR", None)
        p = pk.Plan.from_system(s, thr=thr, kernel="launch")
        x = torch.zeros(s.m, dtype=torch.float64, device="cuda")
        p.solve(f, x, xs, max_sweeps=2, stop="none")
        x.zero_()
        r = p.solve(f, x, xs, max_sweeps=nsw, stop="none")
        out[mode] = (x.cpu().numpy().copy(), r.sweep_seconds / max(1, r.sweeps) * 1e6, r.as_dict()["kernel"], p.nsteps)
        p.close()
    print(json.dumps({"config": name, "thr": thr, "categories": out["ell"][3], "kernel": out["ell"][2], "sweeps": nsw,
                      "us_per_sweep_csr": round(out["csr"][1], 2), "us_per_sweep_ell": round(out["ell"][1], 2),
                      "bitwise_equal": bool(np.array_equal(out["csr"][0], out["ell"][0]))}), flush=True)
