"""(Needs a development build: POBK_EXTRA_FLAGS=-DPOBK_K2_DEV=1, e.g. via tools/with_lib.sh.)
Cycle-level phases of K2's first boundary slice per task (development aid; needs a libpobk.so
built with -DPOBK_K2_FT=1): runs a traced solve and prints p10/p50/p90 cycles per phase.

    python tools/k2_ft.py [config] [sweep]
"""
import os, sys
import numpy as np
sw = int(sys.argv[2]) if len(sys.argv) > 2 else 10
os.environ["POBK_K2_TRACE"] = str(sw)
os.environ.setdefault("POBK_K2_TRACE_OUT", "gpurun_out/k2_ft.bin")
sys.path.insert(0, ".")
import torch
import paper_2401_00672_b200 as pk
from workloads import gen

name = sys.argv[1] if len(sys.argv) > 1 else "geoknn_1m"
s = gen.make(name)
plan = pk.Plan.from_system(s, kernel="wavefront")
f = torch.from_numpy(s.f).cuda(); xs = torch.from_numpy(s.x_star).cuda()
x = torch.zeros(s.m, dtype=torch.float64, device="cuda")
r = plan.solve(f, x, xs, max_sweeps=sw + 3, stop="none", tol=0.0)
print(name, "us/sweep (traced)", round(r.sweep_seconds / r.sweeps * 1e6, 2))
raw = open(os.environ["POBK_K2_TRACE_OUT"], "rb").read()
T, ntm, nst, ntt = np.frombuffer(raw[:16], np.int32)
st = np.frombuffer(raw[16:16 + T * ntm * 96], np.uint64).reshape(T, ntm, 12).astype(np.int64)
ok = np.all(st[:, :, [0, 4, 8, 1, 3, 2, 9, 6, 7, 10, 5, 11]] > 0, axis=2)
seq = [("task start->slice ready", 0, 4), ("pre", 4, 8), ("poll", 8, 1), ("barrier wait", 1, 3), ("sum: x~ loads", 3, 11), ("sum: chain", 11, 2),
       ("division", 2, 9), ("new x", 9, 6), ("write-back issue", 6, 7), ("syncwarp", 7, 10), ("release", 10, 5),
       ("TOTAL start->released", 0, 5)]
print("tasks", int(ok.sum()))
for n, a, b in seq:
    v = (st[:, :, b] - st[:, :, a])[ok]
    print(f"{n:26s} cycles p10/p50/p90", np.percentile(v, [10, 50, 90]).astype(int))
s0 = st[:, 1:, 0]; e0 = st[:, :-1, 5]
g = (s0 - e0)[ok[:, 1:] & ok[:, :-1]]
print(f"{'released->next task start':26s} cycles p10/p50/p90", np.percentile(g, [10, 50, 90]).astype(int))
