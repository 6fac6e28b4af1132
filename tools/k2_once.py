"""One K2 solve of a fixed sweep count on one config (development aid: the ncu target).
    python tools/k2_once.py CONFIG NSWEEPS"""
import sys
sys.path.insert(0, ".")
import torch
import paper_2401_00672_b200 as pk
from workloads import gen
name = sys.argv[1]; nsw = int(sys.argv[2]) if len(sys.argv) > 2 else 20
s = gen.make(name)
f = torch.from_numpy(s.f).cuda(); xs = torch.from_numpy(s.x_star).cuda()
x = torch.zeros(s.m, dtype=torch.float64, device="cuda")
plan = pk.Plan.from_system(s, kernel="wavefront")
for i in range(2):
    x.zero_()
    r = plan.solve(f, x, xs, max_sweeps=nsw, stop="none", tol=0.0)
    print("us/sweep", r.sweep_seconds / r.sweeps * 1e6, flush=True)
