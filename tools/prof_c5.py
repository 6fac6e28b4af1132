"""ncu target: one config-5 system (batch9pt_1024, system 0) on the bench's half-GPU K2 tiling,
50 sweeps without a stop check, after one untimed warm-up solve (the capture is the 2nd launch)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2401_00672_b200 as pk  # noqa: E402
from workloads import gen  # noqa: E402

s = gen.make("batch9pt_1024", 0)
plan = pk.Plan.from_system(s, kernel="wavefront", tile_rows=pk.half_gpu_tile_rows(s.m))
f, xs = torch.from_numpy(s.f).cuda(), torch.from_numpy(s.x_star).cuda()
x = torch.zeros(s.m, dtype=torch.float64, device="cuda")
for _ in range(2):
    x.zero_()
    r = plan.solve(f, x, xs, max_sweeps=50, stop="none")
torch.cuda.synchronize()
print("sweeps", r.sweeps, "us/sweep", r.sweep_seconds / r.sweeps * 1e6, plan.layout_stats())
