"""Fraction of consecutive K2 tasks of a tile that share no column (their barrier could be dropped; development aid)."""
import sys
import numpy as np, scipy.sparse as sp
sys.path.insert(0, ".")
import paper_2401_00672_b200 as pk
from workloads import gen
name = sys.argv[1] if len(sys.argv) > 1 else "geoknn_1m"
s = gen.make(name)
plan = pk.Plan.from_system(s, kernel="wavefront")
colour, cat_ptr, cat_rows = plan.partition(); _, tile = plan.tiles(); perm = plan.perm()
m = s.m; K = plan.nsteps
A = sp.csr_matrix((s.data, s.indices, s.indptr), shape=(m, m))[perm][:, perm].tocsr()
step = np.empty(m, np.int64)
for k in range(K): step[cat_rows[cat_ptr[k]:cat_ptr[k + 1]]] = k
rows = np.repeat(np.arange(m), np.diff(A.indptr)); cols = A.indices
T = tile.max() + 1
# for each (tile, step): set of columns touched
key = tile[rows].astype(np.int64) * K + step[rows]
order = np.lexsort((cols, key))
kk, cc = key[order], cols[order]
from collections import defaultdict
touched = defaultdict(set)
for k_, c_ in zip(kk.tolist(), cc.tolist()):
    touched[k_].add(c_)
tot = free = 0; tail_tot = tail_free = 0
for t in range(T):
    prev = None
    for k in range(K):
        cur = touched.get(t * K + k)
        if cur is None: continue
        if prev is not None:
            tot += 1; f = not (prev & cur); free += f
            if k >= K - 10: tail_tot += 1; tail_free += f
        prev = cur
print(name, "task pairs", tot, "conflict-free consecutive pairs", round(free / tot, 3), "tail (last 10 steps)", tail_tot, round(tail_free / max(tail_tot, 1), 3))
