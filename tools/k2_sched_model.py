"""K2 schedule model (development aid): list-schedules one config-4 sweep on T = 144 tiles
(a 12 x 12 grid of the unit square the geo-kNN points live in: ~16% boundary rows, close to K2's
tiling) with NW warps per tile, interior slices of DI us, boundary slices of DB us, and a
cross-tile hand-off of H us; prints the sweep time with one barrier per (tile, step) task, and
with per-slice dependencies (each slice waits only for the slices that last wrote its columns).
    python tools/k2_sched_model.py prep          (writes /tmp/k2_model_c4.pkl; ~1 min)
    python tools/k2_sched_model.py NW DI DB H
Measured (r02f): barrier 76.9 vs per-slice dataflow 75.4 us at (7, 1.4, 1.2, 0.7) -- dropping
the task barrier buys nothing; DI dominates in the model (0.7 -> 56.8)."""
import sys
if len(sys.argv) > 1 and sys.argv[1] == "prep":
    import pickle
    import numpy as np
    sys.path.insert(0, ".")
    import paper_2401_00672_b200 as pk
    from workloads import gen
    s = gen.make("geoknn_1m")
    plan = pk.Plan.from_system(s, kernel="wavefront", device=-1)  # host preprocessing only
    colour, cat_ptr, cat_rows = plan.partition()
    perm = plan.perm()
    A = s.csr()[perm][:, perm].tocsr()
    pts = gen._rng(304).random((s.m, 2))      # the generator's points (workloads/gen.py geoknn)
    q = gen._rng(104).permutation(s.m)        # its scramble
    pickle.dump(dict(indptr=A.indptr, indices=A.indices, cat_ptr=cat_ptr, cat_rows=cat_rows, pts=pts[q[perm]]),
                open("/tmp/k2_model_c4.pkl", "wb"))
    sys.exit(0)
import numpy as np, pickle
d = pickle.load(open("/tmp/k2_model_c4.pkl","rb"))
ip, ix, cp, cr = d["indptr"], d["indices"], d["cat_ptr"], d["cat_rows"]
m = len(ip)-1; T = 144; NW = int(sys.argv[1]) if len(sys.argv)>1 else 7
DI = float(sys.argv[2]) if len(sys.argv)>2 else 1.4   # interior slice us
DB = float(sys.argv[3]) if len(sys.argv)>3 else 1.2   # boundary post us
H = float(sys.argv[4]) if len(sys.argv)>4 else 0.7    # cross-tile hand-off us
K = len(cp)-1
step = np.empty(m, np.int64)
for k in range(K): step[cr[cp[k]:cp[k+1]]] = k
G = 12; P = d['pts']; tile = np.minimum((P[:,0]*G).astype(np.int64), G-1) * G + np.minimum((P[:,1]*G).astype(np.int64), G-1)
rl = np.diff(ip)
erow = np.repeat(np.arange(m), rl)
ecol = ix.astype(np.int64)
# shared columns
ct_min = np.full(m, T, np.int64); ct_max = np.full(m, -1, np.int64)
np.minimum.at(ct_min, ecol, tile[erow]); np.maximum.at(ct_max, ecol, tile[erow])
shared = ct_min != ct_max
bnd = np.zeros(m, bool); np.logical_or.at(bnd, erow, shared[ecol])
print("boundary row frac", bnd.mean())
# slices
slice_of = np.empty(m, np.int64); sl_tile=[]; sl_step=[]; sl_bnd=[]; sl_n=[]
order = np.lexsort((-rl, ~bnd, step, tile))  # tile, step, boundary first, longer first
key = tile[order]*K*2 + step[order]*2 + (~bnd[order]).astype(np.int64)
brk = np.flatnonzero(np.diff(key)) + 1
grp = np.split(order, brk)
ns = 0
for g in grp:
    for a in range(0, len(g), 32):
        rows = g[a:a+32]; slice_of[rows] = ns
        r0 = rows[0]; sl_tile.append(tile[r0]); sl_step.append(step[r0]); sl_bnd.append(bnd[r0]); sl_n.append(len(rows)); ns += 1
sl_tile=np.array(sl_tile); sl_step=np.array(sl_step); sl_bnd=np.array(sl_bnd)
print("slices", ns)
# prev toucher per entry (same sweep)
o = np.lexsort((step[erow], ecol))
c_s = ecol[o]; r_s = erow[o]
same = np.r_[False, c_s[1:] == c_s[:-1]]
prev_row = np.full(len(o), -1); prev_row[1:] = r_s[:-1]; prev_row[~same] = -1
has = prev_row >= 0
si = slice_of[r_s[has]]; sp_ = slice_of[prev_row[has]]
cross = tile[r_s[has]] != tile[prev_row[has]]
pairs_in = np.unique(si[~cross]*ns + sp_[~cross]); pairs_x = np.unique(si[cross]*ns + sp_[cross])
def lists(pairs):
    a = pairs // ns; b = pairs % ns
    ptr = np.searchsorted(a, np.arange(ns+1))
    return ptr, b
pin, din = lists(pairs_in); px, dx = lists(pairs_x)
print("intra deps/slice", len(din)/ns, "cross deps/slice", len(dx)/ns)
# process slices in (step, tile, index) order
proc = np.lexsort((np.arange(ns), sl_tile, sl_step))
def run(barrier):
    fin = np.zeros(ns); wfree = [[0.0]*NW for _ in range(T)]; task_end = np.zeros(T); cur_step = np.full(T, -1)
    task_max = np.zeros(T)
    for s_ in proc:
        t = sl_tile[s_]
        if barrier and sl_step[s_] != cur_step[t]:
            task_end[t] = task_max[t] if cur_step[t] >= 0 else 0.0
            cur_step[t] = sl_step[s_]
        r = 0.0
        if barrier: r = task_end[t]
        if pin[s_] < pin[s_+1]: r = max(r, fin[din[pin[s_]:pin[s_+1]]].max())
        if px[s_] < px[s_+1]: r = max(r, fin[dx[px[s_]:px[s_+1]]].max() + H)
        w = wfree[t]; i = min(range(NW), key=lambda j: w[j])
        st = max(r, w[i]); dur = DB if sl_bnd[s_] else DI
        fin[s_] = st + dur; w[i] = fin[s_]
        task_max[t] = max(task_max[t], fin[s_]) if barrier else 0
    return fin.max()
print("barrier model us/sweep", round(run(True), 1), " per-slice dataflow", round(run(False), 1))
