"""(Needs a development build: POBK_EXTRA_FLAGS=-DPOBK_K2_DEV=1, e.g. via tools/with_lib.sh.)
In-situ mailbox hop latency of K2 (development aid).  Runs a traced solve (POBK_K2_TRACE), then
for every task's first boundary slice (q0) finds the producers of its shared inputs (previous
toucher of each shared column in schedule order, wrapping to the previous sweep) and compares the
consumer's poll-satisfied stamp with the latest producer's slice-done stamp.

    python tools/k2_hops.py [config] [sweep]
"""
import os, sys
import numpy as np, scipy.sparse as sp
sw = int(sys.argv[2]) if len(sys.argv) > 2 else 10
os.environ["POBK_K2_TRACE"] = str(sw)
os.environ.setdefault("POBK_K2_TRACE_OUT", "gpurun_out/k2_trace.bin")
sys.path.insert(0, ".")
import torch
import paper_2401_00672_b200 as pk
from workloads import gen

name = sys.argv[1] if len(sys.argv) > 1 else "randband_20k"
s = gen.make(name)
plan = pk.Plan.from_system(s, kernel="wavefront")
f = torch.from_numpy(s.f).cuda(); xs = torch.from_numpy(s.x_star).cuda()
x = torch.zeros(s.m, dtype=torch.float64, device="cuda")
r = plan.solve(f, x, xs, max_sweeps=sw + 3, stop="rse", tol=0.0)
print(name, "us/sweep", round(r.sweep_seconds / r.sweeps * 1e6, 2))
raw = open(os.environ["POBK_K2_TRACE_OUT"], "rb").read()
T, ntm, nst, ntt = np.frombuffer(raw[:16], np.int32)
o = 16
st = np.frombuffer(raw[o:o + T * ntm * 96], np.uint64).reshape(T, ntm, 12).astype(np.int64); o += T * ntm * 96
tm = np.frombuffer(raw[o:o + ntt * 16], np.int32).reshape(ntt, 4); o += ntt * 16
tt = np.frombuffer(raw[o:o + (T + 1) * 4], np.int32)
# task index of (tile, step); boundary slice count per task
nsteps = plan.nsteps
tix = np.full((T, nsteps), -1); nb = np.zeros((T, nsteps), int)
for t in range(T):
    for i in range(tt[t], tt[t + 1]):
        tix[t, tm[i, 2]] = i - tt[t]; nb[t, tm[i, 2]] = tm[i, 1] & 0xffff

perm = plan.perm(); colour, cat_ptr, cat_rows = plan.partition(); _, tile = plan.tiles()
m = s.m
A = sp.csr_matrix((s.data, s.indices, s.indptr), shape=(m, m))
At = A[perm][:, perm].tocsr()
step = np.empty(m, np.int64); pos = np.empty(m, np.int64)
for k in range(nsteps):
    step[cat_rows[cat_ptr[k]:cat_ptr[k + 1]]] = k
pos[cat_rows] = np.arange(m)
rlen = np.diff(At.indptr)
rows = np.repeat(np.arange(m), rlen); cols = At.indices
# shared columns: touched by more than one tile
ntc = {}
o2 = np.lexsort((tile[rows], cols)); cs, ts = cols[o2], tile[rows][o2]
newc = np.r_[True, cs[1:] != cs[:-1]]; newct = newc | np.r_[True, ts[1:] != ts[:-1]]
cnt = np.add.reduceat(newct.astype(int), np.flatnonzero(newc))
shared = np.zeros(m, bool); shared[cs[newc]] = cnt > 1
boundary = np.zeros(m, bool); boundary[np.unique(rows[shared[cols]])] = True
# q0 rows of each (tile, step): boundary rows in schedule order, stable-sorted by length desc, first 32
q0 = np.zeros(m, bool)
order = np.lexsort((pos, -rlen, step, tile))
ob = order[boundary[order]]
key = tile[ob] * nsteps + step[ob]
first = np.r_[True, key[1:] != key[:-1]]
rank = np.arange(len(ob)) - np.maximum.accumulate(np.where(first, np.arange(len(ob)), 0))
q0[ob[rank < 32]] = True
# previous toucher of each shared entry (schedule order, wrapping)
e = shared[cols]
er, ec = rows[e], cols[e]
o3 = np.lexsort((pos[er], ec)); er, ec = er[o3], ec[o3]
g0 = np.r_[True, ec[1:] != ec[:-1]]
gstart = np.maximum.accumulate(np.where(g0, np.arange(len(ec)), 0))
gl = np.r_[np.flatnonzero(g0)[1:], len(ec)] - np.flatnonzero(g0)
gend = np.repeat(np.flatnonzero(g0) + gl - 1, gl)
prev = np.where(g0, gend, np.arange(len(ec)) - 1)
wrap = g0
pr = er[prev]
cons = q0[er]
ct_, ck = tile[er][cons], step[er][cons]
pt_, pk_ = tile[pr][cons], step[pr][cons]
pw = wrap[cons]
done = np.where(nb[pt_, pk_] == 1, st[pt_, tix[pt_, pk_], 5], st[pt_, tix[pt_, pk_], 3])
done = np.where(pw, -1, done)  # producer in the previous sweep: not traced
kk = ct_ * nsteps + ck
import pandas as pd
df = pd.DataFrame({"k": kk, "done": done, "same": pt_ == ct_})
g = df.groupby("k").agg(done=("done", "max"), same=("same", "all"))
kt, ks = g.index.values // nsteps, g.index.values % nsteps
ti = tix[kt, ks]
sat = st[kt, ti, 1]; pre = st[kt, ti, 8]; start = st[kt, ti, 0]
okm = (g["done"].values > 0) & (sat > 0)
hop = (sat - g["done"].values)[okm]
late = (g["done"].values > pre)[okm]
print("tasks", okm.sum(), "where the last input arrived after pre:", late.sum())
q = lambda v: np.percentile(v, [10, 50, 90]).astype(int) if len(v) else []
print("producer done -> consumer poll satisfied (ns) p10/p50/p90, all:", q(hop))
print("  ... when the input was late (on the chain):", q(hop[late]))
print("  ... same-tile producer only:", q(hop[g["same"].values[okm]]))
gap = (g["done"].values - start)[okm]
print("consumer task start -> producer done (ns):", q(gap))
its = st[kt, ti, 11][okm]
wait = (sat - pre)[okm]
print("poll iterations p10/p50/p90:", q(its), " ns per iteration (wait / iterations, >1 iteration):",
      q((wait / np.maximum(its, 1))[its > 1]))
