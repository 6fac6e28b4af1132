"""Seeded synthetic workloads for the POBK sweep (SURVEY.md §8(d) "Concrete synthetic inputs").

This module is shared by the oracle side (tests, bench cpu_baseline) and the
product side (bench, smoke).  It builds INPUTS only: the system matrix A in the
user's (scrambled) frame, the exact solution x* and the right-hand side
f = A x*.  It holds none of the method's arithmetic (no RCM, no partition, no
projection, no norm): f = A x* is the consistent-system construction the paper
states as its experimental protocol ("we set the initial value x0 = 0 and the
exact solution is x*", §5.1), computed with one SciPy CSR
mat-vec.

The paper measures on 20 SuiteSparse matrices (Table 2)
which are not available offline; the configs below are synthetic stand-ins
with the paper's structural features (scattered patterns that RCM fixes,
2-D/3-D meshes, FEM-like graphs, random banded systems, fp64).  No SuiteSparse
content is reproduced.

Every matrix returned is canonical CSR: int64 indptr, int32 indices strictly
increasing within a row, no duplicates, no explicitly stored zeros.

RNG: numpy.random.Generator(PCG64(seed)) throughout.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

__all__ = [
    "System", "CONFIGS", "make", "canonical", "scramble",
    "lap2d5", "randband", "lap3d7", "geoknn", "box9",
    "random_banded", "random_pattern_graph",
]


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


@dataclass
class System:
    """One square system A x = f in the user's frame (before any preprocessing)."""
    name: str
    m: int
    indptr: np.ndarray   # int64 [m+1]
    indices: np.ndarray  # int32 [nnz]
    data: np.ndarray     # float64 [nnz]
    f: np.ndarray        # float64 [m]
    x_star: np.ndarray   # float64 [m]

    @property
    def nnz(self) -> int:
        return int(self.indptr[-1])

    def csr(self) -> sp.csr_matrix:
        return sp.csr_matrix((self.data, self.indices, self.indptr), shape=(self.m, self.m))


def canonical(A: sp.spmatrix) -> sp.csr_matrix:
    """Canonical CSR: summed duplicates, sorted indices, no stored zeros.

    SciPy's kron/diags can store explicit zeros (SURVEY.md §8(c) "Hazard found
    during the survey"), so zeros are always eliminated here.
    """
    A = sp.csr_matrix(A, dtype=np.float64)
    A.sum_duplicates()
    A.eliminate_zeros()
    A.sort_indices()
    return A


def scramble(A: sp.csr_matrix, seed: int) -> sp.csr_matrix:
    """Symmetric random permutation q = rng.permutation(m); A_s = A[q][:, q]."""
    q = _rng(seed).permutation(A.shape[0])
    return canonical(A[q][:, q])


# ---------------------------------------------------------------- matrices

def lap2d5(n: int) -> sp.csr_matrix:
    """5-point Dirichlet Laplacian on an n x n grid: diagonal 4, -1 to in-grid neighbours.
    nnz = 5n^2 - 4n (BASELINE.json configs[0])."""
    m = n * n
    ii = np.arange(m)
    r, c = ii // n, ii % n
    rows, cols, vals = [ii], [ii], [np.full(m, 4.0)]
    for dr, dc in ((-1, 0), (1, 0), (0, -1), (0, 1)):
        ok = (r + dr >= 0) & (r + dr < n) & (c + dc >= 0) & (c + dc < n)
        rows.append(ii[ok]); cols.append(((r + dr) * n + (c + dc))[ok]); vals.append(np.full(ok.sum(), -1.0))
    return canonical(sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(m, m)))


def box9(n: int) -> sp.csr_matrix:
    """9-point box stencil on an n x n grid: diagonal 8, -1 to each of the 8 in-grid neighbours.
    nnz = 9n^2 - 12n + 4 (BASELINE.json configs[4])."""
    m = n * n
    ii = np.arange(m)
    r, c = ii // n, ii % n
    rows, cols, vals = [ii], [ii], [np.full(m, 8.0)]
    for dr in (-1, 0, 1):
        for dc in (-1, 0, 1):
            if dr == 0 and dc == 0:
                continue
            ok = (r + dr >= 0) & (r + dr < n) & (c + dc >= 0) & (c + dc < n)
            rows.append(ii[ok]); cols.append(((r + dr) * n + (c + dc))[ok]); vals.append(np.full(ok.sum(), -1.0))
    return canonical(sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(m, m)))


def randband(m: int, seed: int, half: int = 50, n_in: int = 3, n_far: int = 1) -> sp.csr_matrix:
    """BASELINE.json configs[1]: per row i, `n_in` distinct in-band partners uniform from
    [i-half, i+half] \\ {i} (clipped) and `n_far` partner(s) uniform from {j : |j-i| > half};
    pattern := P u P^T; every stored off-diagonal value independent U(-1,1) (values are
    nonsymmetric); diagonal = 1 + sum_j |a_ij| (strictly diagonally dominant)."""
    rng = _rng(seed)
    rows, cols = [], []
    for i in range(m):
        lo, hi = max(0, i - half), min(m - 1, i + half)
        cand = np.concatenate([np.arange(lo, i), np.arange(i + 1, hi + 1)])
        k = min(n_in, cand.size)
        if k:
            pick = rng.choice(cand, size=k, replace=False)
            rows.extend([i] * k); cols.extend(pick.tolist())
        n_out = m - (hi - lo + 1)
        for _ in range(n_far if n_out > 0 else 0):
            u = int(rng.integers(n_out))
            j = u if u < lo else u + (hi - lo + 1)
            rows.append(i); cols.append(j)
    r = np.array(rows, dtype=np.int64); c = np.array(cols, dtype=np.int64)
    P = sp.coo_matrix((np.ones(r.size), (r, c)), shape=(m, m)).tocsr()
    P = P + P.T
    P.sum_duplicates(); P.sort_indices()
    P.data = rng.uniform(-1.0, 1.0, size=P.nnz)  # independent values in CSR order
    diag = 1.0 + np.asarray(abs(P).sum(axis=1)).ravel()
    return canonical(P + sp.diags(diag))


def lap3d7(n: int, seed: int) -> sp.csr_matrix:
    """BASELINE.json configs[2]: 7-point stencil on n^3; per grid edge {i,j}: a_ij = a_ji = -u,
    u ~ U(0.9, 1.1) drawn edge by edge (x-, then y-, then z-edges, ascending lower endpoint);
    diagonal = sum_j |a_ij| + (6 - #grid neighbours) (Dirichlet ghost edges of weight 1, SPD;
    SURVEY.md §8(d) config 3 reading)."""
    rng = _rng(seed)
    m = n ** 3
    ii = np.arange(m)
    z, y, x = ii // (n * n), (ii // n) % n, ii % n
    er, ec = [], []
    for ok, step in ((x + 1 < n, 1), (y + 1 < n, n), (z + 1 < n, n * n)):
        er.append(ii[ok]); ec.append(ii[ok] + step)
    er = np.concatenate(er); ec = np.concatenate(ec)
    u = rng.uniform(0.9, 1.1, size=er.size)
    nb = np.bincount(er, minlength=m) + np.bincount(ec, minlength=m)
    off = sp.coo_matrix((np.concatenate([-u, -u]), (np.concatenate([er, ec]), np.concatenate([ec, er]))), shape=(m, m)).tocsr()
    diag = np.asarray(abs(off).sum(axis=1)).ravel() + (6 - nb)
    return canonical(off + sp.diags(diag))


def geoknn(m: int, seed: int, k: int = 14) -> sp.csr_matrix:
    """BASELINE.json configs[3]: m points U([0,1]^2); k nearest neighbours (cKDTree.query(k+1),
    self removed); pattern = union (symmetric); per undirected edge a_ij = a_ji = -w,
    w ~ U(0.5, 1) drawn in ascending (i, j), i < j order; diagonal = sum |off| + 0.01."""
    from scipy.spatial import cKDTree
    rng = _rng(seed)
    pts = rng.random((m, 2))
    _, idx = cKDTree(pts).query(pts, k=k + 1, workers=-1)
    ii = np.repeat(np.arange(m), k + 1)
    jj = idx.ravel()
    keep = ii != jj
    ii, jj = ii[keep], jj[keep]
    lo, hi = np.minimum(ii, jj), np.maximum(ii, jj)
    key = np.unique(lo.astype(np.int64) * m + hi)
    lo, hi = key // m, key % m
    w = rng.uniform(0.5, 1.0, size=key.size)
    off = sp.coo_matrix((np.concatenate([-w, -w]), (np.concatenate([lo, hi]), np.concatenate([hi, lo]))), shape=(m, m)).tocsr()
    diag = np.asarray(abs(off).sum(axis=1)).ravel() + 0.01
    return canonical(off + sp.diags(diag))


# ---------------------------------------------------------------- tiny test systems

def random_banded(m: int, seed: int, half: int = 3, density: float = 0.6) -> sp.csr_matrix:
    """Small random banded, diagonally dominant system (SPEC.md:473-style acceptance inputs)."""
    rng = _rng(seed)
    rows, cols = [], []
    for i in range(m):
        for j in range(max(0, i - half), min(m, i + half + 1)):
            if j != i and rng.random() < density:
                rows.append(i); cols.append(j)
    off = sp.coo_matrix((rng.uniform(-1, 1, len(rows)), (rows, cols)), shape=(m, m)).tocsr()
    diag = 1.0 + np.asarray(abs(off).sum(axis=1)).ravel()
    return canonical(off + sp.diags(diag))


def random_pattern_graph(m: int, seed: int, p: float) -> sp.csr_matrix:
    """Random symmetric pattern (Erdos-Renyi, edge prob p) with a unit-dominant diagonal;
    isolated vertices and several components occur at small p."""
    rng = _rng(seed)
    mask = np.triu(rng.random((m, m)) < p, 1)
    r, c = np.nonzero(mask)
    v = rng.uniform(-1, 1, r.size)
    off = sp.coo_matrix((np.concatenate([v, v]), (np.concatenate([r, c]), np.concatenate([c, r]))), shape=(m, m)).tocsr()
    diag = 1.0 + np.asarray(abs(off).sum(axis=1)).ravel()
    return canonical(off + sp.diags(diag))


# ---------------------------------------------------------------- configs

# name -> (builder(system_id, scale) -> csr, scramble seed(system_id), x* seed(system_id)).
# Single-system configs: system b > 0 (a replica on rank b of a multi-GPU run) keeps the matrix
# and scramble and draws its own x* (seed + 1000 b); b = 0 is the BASELINE config itself.
CONFIGS = {
    # BASELINE.json configs[0]
    "lap2d5_32": dict(build=lambda b, n=32: lap2d5(n), scramble=lambda b: 101, xstar=lambda b: 201 + 1000 * b, n=32),
    # BASELINE.json configs[1]
    "randband_20k": dict(build=lambda b, n=20000: randband(n, 302), scramble=lambda b: 102, xstar=lambda b: 202 + 1000 * b, n=20000),
    # BASELINE.json configs[2]
    "lap3d7_64": dict(build=lambda b, n=64: lap3d7(n, 303), scramble=lambda b: 103, xstar=lambda b: 203 + 1000 * b, n=64),
    # BASELINE.json configs[3]
    "geoknn_1m": dict(build=lambda b, n=1000000: geoknn(n, 304), scramble=lambda b: 104, xstar=lambda b: 204 + 1000 * b, n=1000000),
    # BASELINE.json configs[4]: 64 independent systems b = 0..63
    "batch9pt_1024": dict(build=lambda b, n=1024: box9(n), scramble=lambda b: 1050 + b, xstar=lambda b: 2050 + b, n=1024),
}


def make(config: str, system_id: int = 0, n: int | None = None) -> System:
    """Build system `system_id` of `config` (optionally at a reduced size parameter `n`:
    grid side for the stencils, m for randband/geoknn) in the user's scrambled frame."""
    spec = CONFIGS[config]
    size = spec["n"] if n is None else n
    A0 = spec["build"](system_id, size)
    A = scramble(A0, spec["scramble"](system_id))
    x_star = _rng(spec["xstar"](system_id)).standard_normal(A.shape[0])
    f = A @ x_star
    return System(config if n is None else f"{config}@{size}", A.shape[0], A.indptr.astype(np.int64),
                  A.indices.astype(np.int32), A.data, np.ascontiguousarray(f), x_star)


def from_csr(name: str, A: sp.spmatrix, xstar_seed: int) -> System:
    """Wrap an arbitrary (test) matrix as a consistent system with x* ~ N(0,1)."""
    A = canonical(A)
    x_star = _rng(xstar_seed).standard_normal(A.shape[0])
    return System(name, A.shape[0], A.indptr.astype(np.int64), A.indices.astype(np.int32), A.data,
                  np.ascontiguousarray(A @ x_star), x_star)
