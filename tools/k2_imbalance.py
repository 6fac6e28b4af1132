"""Per-step load imbalance of the K2 tiling (development aid): nnz per (tile, step), max vs mean."""
import sys, numpy as np
sys.path.insert(0, ".")
import paper_2401_00672_b200 as pk
from workloads import gen
name = sys.argv[1]
s = gen.make(name)
plan = pk.Plan.from_system(s, kernel="wavefront")
colour, cat_ptr, cat_rows = plan.partition()
_, tile = plan.tiles()
T = tile.max() + 1; K = plan.nsteps
step = np.empty(s.m, np.int64)
for k in range(K): step[cat_rows[cat_ptr[k]:cat_ptr[k+1]]] = k
perm = plan.perm()
import scipy.sparse as sp
A = sp.csr_matrix((s.data, s.indices, s.indptr), shape=(s.m, s.m))[perm][:, perm].tocsr()
rl = np.diff(A.indptr)
cnt = np.zeros((T, K)); nz = np.zeros((T, K))
np.add.at(cnt, (tile, step), 1); np.add.at(nz, (tile, step), rl)
mean = nz.mean(0); mx = nz.max(0)
print(name, "T", T, "K", K)
print("sum over steps of max-tile nnz / sum of mean-tile nnz:", mx.sum() / mean.sum())
print("per step max/mean:", np.round(mx / np.maximum(mean, 1e-9), 2)[:40])
print("slices per task (rows/32 ceil) mean", np.ceil(cnt / 32).mean(), "max per step", np.ceil(cnt / 32).max(0)[:40])
