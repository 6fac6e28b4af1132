"""(Needs a development build: POBK_EXTRA_FLAGS=-DPOBK_K2_DEV=1, e.g. via tools/with_lib.sh.)
Which warp closes each task barrier in K2 (development aid; libpobk.so built with
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
# per-warp detail for one tile: arrival at the barrier closing task ti, relative to the release of
# barrier ti-1, with the warp's slices in task ti (b = boundary, i = interior; rot as the kernel)
o = 16 + T * ntm * 96
tm = np.frombuffer(raw[o:o + ntt * 16], np.int32).reshape(ntt, 4); o += ntt * 16
tt = np.frombuffer(raw[o:o + (T + 1) * 4], np.int32)
t = int(sys.argv[3]) if len(sys.argv) > 3 else T // 2
nw = 7; rot = 0
print("tile", t)
for ti in range(tt[t + 1] - tt[t]):
    nb = tm[tt[t] + ti][1] & 0xffff; ni = tm[tt[t] + ti][1] >> 16; ntot = nb + ni
    own = {w: "" for w in range(nw)}
    for q in range(ntot):
        own[(q + rot) % nw] += "b" if q < nb else "i"
    rot = (rot + ntot % nw) % nw
    if ti == 0 or not ok[t, ti]:
        continue
    base = rel[t, ti - 1]
    cells = " ".join(f"w{w}:{own[w] or '-':>3s}{'*' if (lam[t, ti] >> w) & 1 else ' '}{arr[t, ti, w] - base:6d}" for w in range(nw))
    print(f"task {ti:2d} nb {nb} ni {ni} | {cells} | release {rel[t, ti] - base}")
