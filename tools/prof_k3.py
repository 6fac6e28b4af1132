"""Run one K3 solve on config 1 (for ncu; development aid)."""
import sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2401_00672_b200 as pk
from workloads import gen
s = gen.make("lap2d5_32")
plan = pk.Plan.from_system(s, kernel="smem")
f = torch.from_numpy(s.f).cuda(); xs = torch.from_numpy(s.x_star).cuda()
x = torch.zeros(s.m, dtype=torch.float64, device="cuda")
for _ in range(2):
    x.zero_()
    r = plan.solve(f, x, xs, max_sweeps=2000, stop="none")
torch.cuda.synchronize()
print(r.as_dict())
