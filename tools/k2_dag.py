"""Critical-path model of one K2 sweep (development aid): per-task barriers (the current kernel)
versus slice-level dependencies (a slice waits only for the earlier-step slices it shares a
column with).  Slices are approximated like the builder (per tile and step: boundary rows then
interior rows, sorted by length, 32 per slice).  Costs in us: interior slice, boundary slice,
hand-off inside a tile (shared memory) and across tiles (mailbox hop).

    python tools/k2_dag.py [config]
"""
import sys, time
import numpy as np, scipy.sparse as sp
sys.path.insert(0, ".")
import paper_2401_00672_b200 as pk
from workloads import gen

name = sys.argv[1] if len(sys.argv) > 1 else "geoknn_1m"
s = gen.make(name)
plan = pk.Plan.from_system(s, kernel="wavefront")
perm = plan.perm()
colour, cat_ptr, cat_rows = plan.partition()
T, tile = plan.tiles()
m = s.m
A = sp.csr_matrix((s.data, s.indices, s.indptr), shape=(m, m))
At = A[perm][:, perm].tocsr()
nst = len(cat_ptr) - 1
step = np.empty(m, np.int64)
for k in range(nst):
    step[cat_rows[cat_ptr[k]:cat_ptr[k + 1]]] = k
rows = np.repeat(np.arange(m), np.diff(At.indptr)); cols = At.indices
# shared columns and boundary rows
ct = np.full(m, -1); sh = np.zeros(m, bool)
for r, c in zip(rows, cols):
    pass
order = np.lexsort((tile[rows], cols)); cs_, ts_ = cols[order], tile[rows][order]
first = np.r_[True, cs_[1:] != cs_[:-1]]
nt = np.add.reduceat(np.r_[True, (cs_[1:] != cs_[:-1]) | (ts_[1:] != ts_[:-1])].astype(np.int64), np.flatnonzero(first))
sh[cs_[first]] = nt > 1
bnd = np.zeros(m, bool); bnd[np.unique(rows[sh[cols]])] = True
rlen = np.diff(At.indptr)
# slices: (tile, step, kind) groups of 32 rows sorted by length desc
key = (tile.astype(np.int64) * nst + step) * 2 + (~bnd).astype(np.int64)
o = np.lexsort((-rlen, key))
ks = key[o]
starts = np.flatnonzero(np.r_[True, ks[1:] != ks[:-1]])
slice_of = np.empty(m, np.int64)
sl_tile, sl_step, sl_bnd = [], [], []
sid = 0
for a, b in zip(starts, np.r_[starts[1:], m]):
    for c0 in range(a, b, 32):
        slice_of[o[c0:min(b, c0 + 32)]] = sid
        kk = ks[c0]
        sl_tile.append(kk // 2 // nst); sl_step.append(kk // 2 % nst); sl_bnd.append(kk % 2 == 0)
        sid += 1
S = sid
sl_tile, sl_step, sl_bnd = np.array(sl_tile), np.array(sl_step), np.array(sl_bnd)
print("slices", S, "boundary", sl_bnd.sum(), "T", T, "steps", nst)
# slice dependencies through columns: for each column, the slices touching it in step order
t0 = time.time()
cs = slice_of[rows]
o2 = np.lexsort((sl_step[cs], cols))
cc, ss = cols[o2], cs[o2]
# consecutive (by step) distinct slices on the same column -> edge prev -> next (and the chain gives transitivity)
same = (cc[1:] == cc[:-1]) & (ss[1:] != ss[:-1])
src, dst = ss[:-1][same], ss[1:][same]
E = np.unique(src * S + dst)
src, dst = E // S, E % S
print("edges", len(src), round(time.time() - t0, 1), "s")
preds = [[] for _ in range(S)]
for a_, b_ in zip(src, dst):
    if sl_step[a_] < sl_step[b_]:
        preds[b_].append(a_)
order_s = np.lexsort((sl_tile, sl_step))


def run(cost_i, cost_b, handoff_local, hop, barrier):
    fin = np.zeros(S)
    task_end = {}
    for x in order_s:
        t, k = sl_tile[x], sl_step[x]
        st = 0.0
        for p in preds[x]:
            st = max(st, fin[p] + (handoff_local if sl_tile[p] == t else hop))
        if barrier:  # all slices of the tile's previous task
            st = max(st, task_end.get((t, 'prev'), 0.0))
        fin[x] = st + (cost_b if sl_bnd[x] else cost_i)
        if barrier:
            task_end[(t, k)] = max(task_end.get((t, k), 0.0), fin[x])
            # previous task end for the next task of the tile
        if barrier and (x == order_s[-1] or True):
            pass
    return fin.max()


def run_barrier(cost_i, cost_b, hop):
    # per tile: task k starts when its previous task ended; boundary slices also wait for the
    # other tiles' slices they depend on (+hop); interior slices only for the task start
    fin = np.zeros(S)
    tile_ready = np.zeros(T)
    for k in range(nst):
        xs = np.flatnonzero(sl_step == k)
        ends = {}
        for x in xs:
            t = sl_tile[x]
            st = tile_ready[t]
            if sl_bnd[x]:
                for p in preds[x]:
                    if sl_tile[p] != t:
                        st = max(st, fin[p] + hop)
            fin[x] = st + (cost_b if sl_bnd[x] else cost_i)
            ends[t] = max(ends.get(t, 0.0), fin[x])
        for t, e in ends.items():
            tile_ready[t] = e
    return fin.max()


for ci, cb, hl, hop in ((1.2, 2.2, 0.1, 1.0), (1.2, 1.5, 0.1, 0.7), (0.6, 1.0, 0.05, 0.6)):
    a = run_barrier(ci, cb, hop)
    b = run(ci, cb, hl, hop, False)
    print(f"costs int {ci} bnd {cb} local {hl} hop {hop}: per-task barrier {a:.1f} us/sweep, slice dataflow {b:.1f} us/sweep")
