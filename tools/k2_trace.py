"""(Needs a development build: POBK_EXTRA_FLAGS=-DPOBK_K2_DEV=1, e.g. via tools/with_lib.sh.)
K2 per-task timeline of one sweep (development aid): POBK_K2_TRACE=<sweep> makes libpobk.so
dump %globaltimer stamps per tile and task; this script runs a solve and summarises where a
sweep's time goes.  Stamps: 0 task start (warp 0), 1 boundary poll satisfied (warp 0), 3 task
barrier passed, 4/5 first slice (q=0) ready/done, 6/7 first interior slice ready/done.

    python tools/k2_trace.py [config] [sweep] [nsweeps]
"""
import os, sys
import numpy as np
sw = int(sys.argv[2]) if len(sys.argv) > 2 else 10
os.environ["POBK_K2_TRACE"] = str(sw)
os.environ.setdefault("POBK_K2_TRACE_OUT", "gpurun_out/k2_trace.bin")
sys.path.insert(0, ".")
import torch
import paper_2401_00672_b200 as pk
from workloads import gen

name = sys.argv[1] if len(sys.argv) > 1 else "geoknn_1m"
nsw = int(sys.argv[3]) if len(sys.argv) > 3 else 20
s = gen.make(name)
plan = pk.Plan.from_system(s, kernel="wavefront")
print(plan.layout_stats())
f = torch.from_numpy(s.f).cuda(); xs = torch.from_numpy(s.x_star).cuda()
x = torch.zeros(s.m, dtype=torch.float64, device="cuda")
r = plan.solve(f, x, xs, max_sweeps=nsw, stop="rse", tol=0.0)
print("us/sweep (whole solve)", r.sweep_seconds / r.sweeps * 1e6)

raw = open(os.environ["POBK_K2_TRACE_OUT"], "rb").read()
T, ntm, nst, ntt = np.frombuffer(raw[:16], np.int32)
o = 16
st = np.frombuffer(raw[o:o + T * ntm * 12 * 8], np.uint64).reshape(T, ntm, 12).astype(np.int64); o += T * ntm * 96
tm = np.frombuffer(raw[o:o + ntt * 16], np.int32).reshape(ntt, 4); o += ntt * 16
tt = np.frombuffer(raw[o:o + (T + 1) * 4], np.int32); o += (T + 1) * 4
t0 = st[:, :, 0][st[:, :, 0] > 0].min()
st = np.where(st > 0, st - t0, -1)


def q(v):
    v = np.asarray(v, float)
    if not len(v):
        return {}
    return {"n": len(v), "mean": round(v.mean()), "p50": round(np.median(v)), "p90": round(np.percentile(v, 90)), "max": round(v.max())}


print("sweep span ns", int(st[:, :, 3].max()))
task_len, poll, bslice, islice, ready_b, bar_after = [], [], [], [], [], []
pm, ps, pf, pr = [], [], [], []
pa, pb, pc, pd = [], [], [], []
for t in range(T):
    n = tt[t + 1] - tt[t]
    for ti in range(n):
        a = tm[tt[t] + ti]
        nb, ni = a[1] & 0xffff, a[1] >> 16
        s0, sp, m2, s3, r0, d0, r1, d1, m8, m9, m10, _ = st[t, ti]
        task_len.append(s3 - s0)
        if nb > 0 and sp >= 0:
            poll.append(sp - s0); ready_b.append(r0 - sp); bslice.append(d0 - r0); bar_after.append(s3 - d0)
            pm.append(m8 - r0); ps.append(sp - m8); pf.append(d0 - sp); pa.append(m2 - sp); pb.append(m9 - m2); pc.append(m10 - m9); pd.append(d0 - m10)
        if ni > 0 and r1 >= 0:
            islice.append(d1 - r1)
print("task (start -> barrier passed)", q(task_len))
rb = [st[t, ti, 4] - st[t, ti, 0] for t in range(T) for ti in range(tt[t + 1] - tt[t]) if (tm[tt[t] + ti][1] & 0xffff) > 0 and st[t, ti, 4] >= 0]
ri = [st[t, ti, 6] - st[t, ti, 0] for t in range(T) for ti in range(tt[t + 1] - tt[t]) if (tm[tt[t] + ti][1] >> 16) > 0 and st[t, ti, 6] >= 0]
print("  start -> first boundary slice data ready", q(rb), " start -> first interior slice data ready", q(ri))
print("  start -> mailboxes full", q(poll))
print("  first boundary slice: polled->ready", q(ready_b), "compute+publish", q(bslice), "done->barrier", q(bar_after))
print("  first interior slice compute", q(islice))
print("  boundary slice: pre", q(pm), " mailbox poll", q(ps), " post (math+stores)", q(pf))
print("  post: sum", q(pa), " ddiv", q(pb), " pass 2", q(pc), " release", q(pd))
span = [st[t, tt[t + 1] - tt[t] - 1, 3] - st[t, 0, 0] for t in range(T) if tt[t + 1] > tt[t]]
print("tile sweep span", q(span))
t = int(np.argmax([st[t, tt[t + 1] - tt[t] - 1, 3] if tt[t + 1] > tt[t] else -1 for t in range(T)]))
print("slowest tile", t)
for ti in range(tt[t + 1] - tt[t]):
    a = tm[tt[t] + ti]
    print("  task %2d step %2d nb %2d ni %2d | start %7d polled %7d q0 %7d..%7d int %7d..%7d end %7d" %
          ((ti, a[2], a[1] & 0xffff, a[1] >> 16, st[t, ti, 0], st[t, ti, 1], st[t, ti, 4], st[t, ti, 5], st[t, ti, 6], st[t, ti, 7], st[t, ti, 3])))

# per-step fronts: when do tiles finish step k (task end stamp), and how fast does the front move
ends = {}
starts = {}
for t in range(T):
    for ti in range(tt[t + 1] - tt[t]):
        k = int(tm[tt[t] + ti][2])
        ends.setdefault(k, []).append(st[t, ti, 3])
        starts.setdefault(k, []).append(st[t, ti, 0])
print("step | tiles | start min/med/max | end min/med/max | end-max delta")
prev = None
for k in sorted(ends):
    e = np.array(ends[k]); s_ = np.array(starts[k])
    d = (e.max() - prev) if prev is not None else 0
    prev = e.max()
    print("%4d | %5d | %7d %7d %7d | %7d %7d %7d | %6d" % (k, len(e), s_.min(), np.median(s_), s_.max(), e.min(), np.median(e), e.max(), d))
