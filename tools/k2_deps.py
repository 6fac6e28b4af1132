"""Dependency analysis of the K2 tiling (development aid): compares the coarse task rule (a tile's
boundary rows at step k wait for every neighbour's boundary rows of ALL steps < k) with the exact
row-level rule (wait only for the latest step < k at which the neighbour has a row sharing a
column with one of ours), by the longest path of the per-sweep task DAG.

    python tools/k2_deps.py [config]
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
step = np.empty(m, np.int64)
for k in range(len(cat_ptr) - 1):
    step[cat_rows[cat_ptr[k]:cat_ptr[k + 1]]] = k
nsteps = len(cat_ptr) - 1
# shared columns: touched by >1 tile
rows = np.repeat(np.arange(m), np.diff(At.indptr)); cols = At.indices
ct = tile[rows]
order = np.lexsort((ct, cols))
cs, ts = cols[order], ct[order]
first = np.r_[True, cs[1:] != cs[:-1]]
ntile_per_col = np.add.reduceat(np.r_[True, (cs[1:] != cs[:-1]) | (ts[1:] != ts[:-1])].astype(np.int64), np.flatnonzero(first))
shared = np.zeros(m, bool); shared[cs[first]] = ntile_per_col > 1
print("T", T, "nsteps", nsteps, "shared cols", shared.sum())
# conflict pairs through shared columns, across tiles
AtT = At.T.tocsr()  # column -> rows
need_exact = {}  # (t, k, u) -> max step < k of a conflicting row in u  (or -1 - (max step) for previous sweep)
t0 = time.time()
pairs_t, pairs_k, pairs_u, pairs_ku = [], [], [], []
for c in np.flatnonzero(shared):
    r = AtT.indices[AtT.indptr[c]:AtT.indptr[c + 1]]
    tr, kr = tile[r], step[r]
    I, J = np.meshgrid(np.arange(len(r)), np.arange(len(r)), indexing="ij")
    msk = tr[I] != tr[J]
    pairs_t.append(tr[I][msk]); pairs_k.append(kr[I][msk]); pairs_u.append(tr[J][msk]); pairs_ku.append(kr[J][msk])
pt, pk_, pu, pku = (np.concatenate(x) for x in (pairs_t, pairs_k, pairs_u, pairs_ku))
print("pairs", len(pt), "in", round(time.time() - t0, 1), "s")
# exact need: latest step of u before k (same sweep) if any, else latest step of u overall (previous sweep)
key = (pt * nsteps + pk_) * T + pu
before = pku < pk_
v_same = np.full(len(pt), -1); v_same[before] = pku[before]
import pandas as pd
df = pd.DataFrame({"key": key, "same": v_same, "prev": np.where(before, -1, pku)})
g = df.groupby("key").agg({"same": "max", "prev": "max"})
keys = g.index.values
t_, rest = keys // T, keys % T
tk = t_ // 1
tt_, kk = tk // nsteps, tk % nsteps
slack = np.where(g["same"].values >= 0, kk - g["same"].values, kk + nsteps - g["prev"].values)
print("exact slack (k - latest conflicting neighbour step), over (tile, step, neighbour):",
      {int(a): int(b) for a, b in zip(*np.unique(np.minimum(slack, 6), return_counts=True))})
# DAG longest path over 3 sweeps (node = (tile, step) present in tile), unit cost per cross hop + local cost
has = np.zeros((T, nsteps), bool); has[tile, step] = True
bnd = np.zeros((T, nsteps), bool); brow = np.zeros(m, bool)
brow[np.unique(rows[shared[cols]])] = True
bnd[tile[brow], step[brow]] = True
nbrs = [set() for _ in range(T)]
for a_, b_ in zip(tt_, rest): nbrs[a_].add(b_)
def longest(exact, c_local=1.0, c_cross=2.0, sweeps=3):
    INF = -1e18
    fin = np.full((sweeps, T, nsteps), INF)
    exact_need = {}
    if exact:
        for (kk_, t__, u__), sm, pv in zip(zip(kk, tt_, rest), g["same"].values, g["prev"].values):
            exact_need[(t__, kk_, u__)] = (0, sm) if sm >= 0 else (-1, pv)
    last_local = np.full(T, 0.0)
    for sw in range(sweeps):
        for k in range(nsteps):
            for t in range(T):
                if not has[t, k]: continue
                st = last_local[t]
                if bnd[t, k]:
                    for u in nbrs[t]:
                        if exact:
                            d = exact_need.get((t, k, u))
                            if d is None: continue
                            s2, kp = sw + d[0], d[1]
                            if s2 < 0: continue
                            ready = fin[s2, u, kp]
                        else:
                            # all boundary tasks of u before k in this sweep, else previous sweep's last
                            ks = np.flatnonzero(has[u, :k] & bnd[u, :k])
                            if len(ks): ready = fin[sw, u, ks[-1]]
                            else:
                                ks = np.flatnonzero(has[u] & bnd[u])
                                if sw == 0 or not len(ks): continue
                                ready = fin[sw - 1, u, ks[-1]]
                        st = max(st, ready + c_cross)
                fin[sw, t, k] = st + c_local
                last_local[t] = fin[sw, t, k]
    return last_local.max() / sweeps
for cl, cc in ((1.0, 2.0), (1.0, 1.0), (1.0, 0.5)):
    print(f"per-sweep critical path (task cost {cl}, hop cost {cc}): coarse {longest(False, cl, cc):.1f}  exact {longest(True, cl, cc):.1f}  (nsteps {nsteps})")
