"""Which warp closes each task barrier in K2 (development aid; libpobk.so built with
-DPOBK_K2_WT=1, 256 threads): per (tile, task) the compute warps' arrival clocks at the barrier
that closes the task; reports how late the last warp is and whether it was a look-ahead warp
(waiting for its poll = neighbours' data) or a warp still working on the task's slices.

    python tools/k2_wt.py [config] [sweep]
"""
import os, sys
import numpy as np
sw = int(sys.argv[2]) if len(sys.argv) > 2 else 10
os.environ["POBK_K2_TRACE"] = str(sw)
os.environ.setdefault("POBK_K2_TRACE_OUT", "gpurun_out/k2_wt.bin")
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
arr = st[:, :, :7]; lam = st[:, :, 7]; rel = st[:, :, 8]
ok = np.all(arr > 0, axis=2) & (rel > 0)
last = np.argmax(np.where(ok[..., None], arr, 0), axis=2)
srt = np.sort(arr, axis=2)
gap = (srt[:, :, -1] - srt[:, :, -2])[ok]
spread = (srt[:, :, -1] - srt[:, :, 0])[ok]
last_la = ((lam >> last) & 1)[ok].astype(bool)
q = lambda v: np.percentile(v, [10, 50, 90]).astype(int) if len(v) else []
print("barriers", int(ok.sum()), " last arrival is a look-ahead (poll) warp:", round(last_la.mean(), 3))
print("last - second-last arrival (cycles) p10/p50/p90:", q(gap))
print("last - first arrival (cycles) p10/p50/p90:", q(spread))
print("  ... when the last is a look-ahead warp:", q(spread[last_la]), " else:", q(spread[~last_la]))
per = np.diff(np.where(ok, rel, 0), axis=1)
print("barrier-to-barrier (cycles) p10/p50/p90:", q(per[(per > 0) & (per < 1e6)]))
