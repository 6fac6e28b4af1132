"""Run one short K2 solve on config 4 (for ncu)."""
import sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2401_00672_b200 as pk
from workloads import gen
name = sys.argv[1] if len(sys.argv) > 1 else "geoknn_1m"
kernel = sys.argv[2] if len(sys.argv) > 2 else "wavefront"
nsw = int(sys.argv[3]) if len(sys.argv) > 3 else 10
s = gen.make(name)
plan = pk.Plan.from_system(s, kernel=kernel)
f = torch.from_numpy(s.f).cuda(); xs = torch.from_numpy(s.x_star).cuda()
x = torch.zeros(s.m, dtype=torch.float64, device="cuda")
for _ in range(2):
    x.zero_()
    r = plan.solve(f, x, xs, max_sweeps=nsw, stop="none")
torch.cuda.synchronize()
print(r.as_dict(), plan.layout_stats())
