"""Per-phase latency of K2's first boundary slice from a POBK_K2_TRACE dump (development aid):
pre (4->8), poll wait (8->1), sum (1->2), division (2->9), write-back (9->10), and the gap from
one task's barrier to the next task's start.

    python tools/k2_phases.py [gpurun_out/k2_trace.bin]
"""
import sys
import numpy as np

raw = open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/k2_trace.bin", "rb").read()
T, ntm, nst, ntt = np.frombuffer(raw[:16], np.int32)
st = np.frombuffer(raw[16:16 + T * ntm * 96], np.uint64).reshape(T, ntm, 12).astype(np.int64)
ok = (st[:, :, 10] > 0) & (st[:, :, 9] > 0) & (st[:, :, 8] > 0) & (st[:, :, 1] > 0)
print("tiles", T, "tasks/tile (max)", ntm)
for n, (a, b) in {"start->data ready (0->4)": (0, 4), "pre (4->8)": (4, 8), "poll wait (8->1)": (8, 1),
                  "sum (1->2)": (1, 2), "division (2->9)": (2, 9), "write-back (9->10)": (9, 10),
                  "release (10->5)": (10, 5), "q0 done -> barrier (5->3)": (5, 3)}.items():
    v = (st[:, :, b] - st[:, :, a])[ok]
    print(f"{n:28s} p10/p50/p90 ns", np.percentile(v, [10, 50, 90]).astype(int))
s0 = st[:, 1:, 0]; b0 = st[:, :-1, 3]
g = (s0 - b0)[(s0 > 0) & (b0 > 0)]
print(f"{'barrier -> next start':28s} p10/p50/p90 ns", np.percentile(g, [10, 50, 90]).astype(int))
