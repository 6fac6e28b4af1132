"""How many K2 boundary rows could run before their tile's previous task completes (development
aid): a boundary row is 'early' when none of its private columns is touched by a row of the
tile's previous (non-empty) task.  Also: the fraction of boundary rows whose shared inputs all
come from early producers.

    python tools/k2_early.py [config]
"""
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
# shared columns
ct = np.full(m, -1); sh = np.zeros(m, bool)
for r, c in zip(rows, cols):
    pass
o = np.lexsort((tile[rows], cols)); cs, ts = cols[o], tile[rows][o]
newc = np.r_[True, cs[1:] != cs[:-1]]; newct = newc | np.r_[True, ts[1:] != ts[:-1]]
cnt = np.add.reduceat(newct.astype(int), np.flatnonzero(newc)); sh[cs[newc]] = cnt > 1
bnd = np.zeros(m, bool); bnd[np.unique(rows[sh[cols]])] = True
# previous non-empty task of each (tile, step)
T = tile.max() + 1
has = np.zeros((T, K), bool); has[tile, step] = True
prev = np.full((T, K), -1)
for t in range(T):
    last = -1
    for k in range(K):
        prev[t, k] = last
        if has[t, k]: last = k
# private column touched by tile's task k: set of (col, k)
priv_e = ~sh[cols]
touch = set(zip(cols[priv_e].tolist(), step[rows[priv_e]].tolist()))
early = np.zeros(m, bool)
for r in np.flatnonzero(bnd):
    pk_ = prev[tile[r], step[r]]
    cs_r = A.indices[A.indptr[r]:A.indptr[r + 1]]
    early[r] = not any((c, pk_) in touch for c in cs_r if not sh[c])
print(name, "boundary rows", int(bnd.sum()), "early-eligible", round(early[bnd].mean(), 3))
