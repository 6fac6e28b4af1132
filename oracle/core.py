"""POBK oracle (TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py for who may use it).

Follows SURVEY.md §8(c) O1-O9 in the paper's order.  Citations: PAPER.md line numbers
(arXiv 2401.00672 LaTeX source), SPEC.md line numbers.  Loop-heavy steps call the plain C
in oracle/c/pobk_oracle.c; everything else is NumPy/SciPy library primitives used as
single steps (a permutation, a sort, a mat-vec), never blocked or fused.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

__all__ = [
    "OracleError", "ERR_ARG", "ERR_BAD_CSR", "ERR_ZERO_ROW",
    "TERM_CONVERGED", "TERM_MAX_SWEEPS", "TERM_NONFINITE",
    "canonicalize", "row_nrm2", "graph_pattern", "rcm", "rcm_py", "bandwidth",
    "permute_matrix", "permute_vector", "unpermute_vector",
    "first_fit", "first_fit_py", "schedule", "category_overlap",
    "Preprocessed", "preprocess", "sweep", "sweep_rows_py", "sweep_numpy",
    "rse", "relres", "residual_norm", "SolveResult", "solve", "run_sweeps", "block_step_pinv",
    "row_residuals", "seq_sum", "two_level_sum", "step_scores", "residual_order", "sweep_ordered",
    "run_sweeps_ordered", "solve_ordered", "CHUNK",
    "build_c",
]

ERR_ARG, ERR_BAD_CSR, ERR_ZERO_ROW = 1, 2, 3
TERM_CONVERGED, TERM_MAX_SWEEPS, TERM_NONFINITE = 0, 1, 2


class OracleError(ValueError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


# ------------------------------------------------------------------ the C part
_HERE = os.path.dirname(os.path.abspath(__file__))
_CSRC = os.path.join(_HERE, "c", "pobk_oracle.c")
_SO = os.path.join(_HERE, "c", "_pobk_oracle.so")
_lock = threading.Lock()
_lib_handle = None


def build_c(force: bool = False) -> str:
    """Compile oracle/c/pobk_oracle.c (plain C, -ffp-contract=off: no FMA contraction)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_CSRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
                               "-o", tmp, _CSRC, "-lm"])
        os.replace(tmp, _SO)
    return _SO


def _lib():
    global _lib_handle
    with _lock:
        if _lib_handle is None:
            lib = ctypes.CDLL(build_c())
            P = ctypes.c_void_p
            I64 = ctypes.c_int64
            lib.orc_row_nrm2.argtypes = [I64, P, P, P]
            lib.orc_rcm.argtypes = [I64, P, P, P]
            lib.orc_first_fit.argtypes = [I64, P, P, P, P, ctypes.c_double, P]
            lib.orc_category_overlap.argtypes = [I64, P, P, P, I64, P]
            lib.orc_sweep.argtypes = [I64, P, P, P, P, P, P, I64, P, P, P, P]
            lib.orc_row_residuals.argtypes = [I64, P, P, P, P, P, P]
            lib.orc_rse.argtypes = [I64, P, P]
            lib.orc_rse.restype = ctypes.c_double
            lib.orc_relres.argtypes = [I64, P, P, P, P, P]
            lib.orc_relres.restype = ctypes.c_double
            lib.orc_residual_sumsq.argtypes = [I64, P, P, P, P, P]
            lib.orc_residual_sumsq.restype = ctypes.c_double
            lib.orc_solve.argtypes = [I64, P, P, P, P, P, P, P, I64, P, P, P, ctypes.c_int32, ctypes.c_double,
                                      I64, P, P, P, P]
            _lib_handle = lib
        return _lib_handle


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# ------------------------------------------------------------------ O1 canonicalise
def canonicalize(m: int, indptr, indices, data):
    """O1 (SURVEY.md §8(b) input contract): validate 0-based canonical CSR
    (row_ptr[0] = 0, non-decreasing, row_ptr[m] = nnz, 0 <= col < m strictly increasing
    within a row; duplicates rejected), then drop explicitly stored zeros.  A row that is
    empty afterwards has ||a_i|| = 0, for which Eq 1.2 is undefined: error."""
    if m < 1:
        raise OracleError(ERR_ARG, "m must be >= 1")
    indptr = np.asarray(indptr, dtype=np.int64)
    indices = np.asarray(indices, dtype=np.int64)
    data = np.asarray(data, dtype=np.float64)
    if indptr.shape != (m + 1,) or indptr[0] != 0 or np.any(np.diff(indptr) < 0) or indptr[-1] != indices.size \
            or indices.size != data.size:
        raise OracleError(ERR_BAD_CSR, "row_ptr not a valid CSR offset array")
    if indices.size and (indices.min() < 0 or indices.max() >= m):
        raise OracleError(ERR_BAD_CSR, "column index out of range")
    rows = np.repeat(np.arange(m), np.diff(indptr))
    same_row = rows[1:] == rows[:-1]
    if np.any(same_row & (indices[1:] <= indices[:-1])):
        bad = int(rows[1:][same_row & (indices[1:] <= indices[:-1])][0])
        raise OracleError(ERR_BAD_CSR, f"row {bad}: columns not strictly increasing (unsorted or duplicate)")
    keep = data != 0.0
    counts = np.bincount(rows[keep], minlength=m)
    if np.any(counts == 0):
        raise OracleError(ERR_ZERO_ROW, f"row {int(np.argmin(counts))} is zero")
    new_ptr = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(counts, out=new_ptr[1:])
    return new_ptr, indices[keep].astype(np.int32), data[keep].copy()


def row_nrm2(m: int, indptr, data) -> np.ndarray:
    """nrm2_i = sum_p a_ip^2, ascending p, plain sum from 0.0 (Eq 1.2 denominator)."""
    out = np.empty(m)
    _lib().orc_row_nrm2(m, _p(np.ascontiguousarray(indptr, np.int64)), _p(np.ascontiguousarray(data, np.float64)), _p(out))
    return out


# ------------------------------------------------------------------ O2/O3 RCM
def graph_pattern(m: int, indptr, indices) -> list[list[int]]:
    """O2: adjacency lists of pattern(A + A^T) without self loops."""
    adj = [set() for _ in range(m)]
    for i in range(m):
        for j in indices[indptr[i]:indptr[i + 1]]:
            j = int(j)
            if j != i:
                adj[i].add(j)
                adj[j].add(i)
    return [sorted(a) for a in adj]


def rcm(m: int, indptr, indices) -> np.ndarray:
    """O3 (Eq 3.1; rule pinned in SURVEY.md §8(c) O3):
    returns perm with perm[new] = old.  Plain C implementation."""
    perm = np.empty(m, dtype=np.int32)
    rc = _lib().orc_rcm(m, _p(np.ascontiguousarray(indptr, np.int64)), _p(np.ascontiguousarray(indices, np.int32)), _p(perm))
    if rc != 0:
        raise MemoryError("orc_rcm failed")
    return perm


def rcm_py(m: int, indptr, indices) -> np.ndarray:
    """The same O3 rule written out in pure Python (small cases only)."""
    adj = graph_pattern(m, indptr, indices)
    deg = [len(a) for a in adj]
    key = lambda v: (deg[v], v)  # noqa: E731

    def levels(r):
        dist = {r: 0}
        frontier, out = [r], [[r]]
        while True:
            nxt = []
            for v in frontier:
                for u in adj[v]:
                    if u not in dist:
                        dist[u] = dist[v] + 1
                        nxt.append(u)
            if not nxt:
                return out
            out.append(nxt)
            frontier = nxt

    visited = [False] * m
    order = []
    for s0 in range(m):
        if visited[s0]:
            continue
        comp = [v for lvl in levels(s0) for v in lvl]
        r = min(comp, key=key)
        L = levels(r)
        x = r
        for _ in range(10):
            x = min(L[-1], key=key)
            Lx = levels(x)
            if len(Lx) > len(L):
                r, L = x, Lx
            else:
                break
        root = x
        queue = [root]
        visited[root] = True
        head = 0
        while head < len(queue):
            v = queue[head]
            head += 1
            order.append(v)
            for u in sorted((u for u in adj[v] if not visited[u]), key=key):
                visited[u] = True
                queue.append(u)
    return np.array(order[::-1], dtype=np.int32)


def bandwidth(m: int, indptr, indices) -> int:
    """max over stored entries of |i - j|."""
    rows = np.repeat(np.arange(m), np.diff(indptr))
    return int(np.max(np.abs(rows - np.asarray(indices, dtype=np.int64)))) if rows.size else 0


# ------------------------------------------------------------------ O4 / O9 permutation
def permute_matrix(m: int, indptr, indices, data, perm):
    """O4: A~ = P A P^T (Eq 3.1): row i of A~ is row perm[i] of A, with
    column c renamed iperm[c] and columns re-sorted ascending."""
    A = sp.csr_matrix((data, indices, indptr), shape=(m, m))
    At = A[perm][:, perm].tocsr()
    At.sort_indices()
    return At.indptr.astype(np.int64), At.indices.astype(np.int32), At.data.astype(np.float64)


def permute_vector(v, perm):
    """f~ = P f, i.e. f~[i] = f[perm[i]]."""
    return np.asarray(v, dtype=np.float64)[perm].copy()


def unpermute_vector(vt, perm):
    """O9: x = P^T x~, i.e. x[perm[i]] = x~[i]."""
    x = np.empty_like(vt)
    x[perm] = vt
    return x


# ------------------------------------------------------------------ O5/O6 partition
def first_fit(m: int, indptr, indices, data, nrm2, thr: float = 0.0) -> np.ndarray:
    """O5/O6: color[i] = mex{color[l] : l < i, conflict(i, l)} over the
    rows of A~.  Plain C implementation."""
    color = np.empty(m, dtype=np.int32)
    _lib().orc_first_fit(m, _p(np.ascontiguousarray(indptr, np.int64)), _p(np.ascontiguousarray(indices, np.int32)),
                         _p(np.ascontiguousarray(data, np.float64)), _p(np.ascontiguousarray(nrm2, np.float64)),
                         float(thr), _p(color))
    return color


def first_fit_py(m: int, indptr, indices, data, nrm2, thr: float = 0.0) -> np.ndarray:
    """The same O5/O6 rule in pure Python, by brute force over all pairs (small cases only)."""
    rows = [dict(zip(indices[indptr[i]:indptr[i + 1]].tolist(), data[indptr[i]:indptr[i + 1]].tolist())) for i in range(m)]
    color = [0] * m
    for i in range(m):
        used = set()
        for l in range(i):
            shared = sorted(set(rows[i]) & set(rows[l]))
            if not shared:
                continue
            if thr > 0.0:
                d = 0.0
                for c in shared:
                    d = d + rows[i][c] * rows[l][c]
                if not (d * d >= (thr * thr) * (nrm2[i] * nrm2[l])):
                    continue
            used.add(color[l])
        k = 0
        while k in used:
            k += 1
        color[i] = k
    return np.array(color, dtype=np.int32)


def schedule(color: np.ndarray):
    """O6 schedule sigma: Oclass = categories K_c = {i : color[i] = c} with |K_c| >= 2, in
    ascending c, each one step (rows ascending); then the Nclass rows (singleton categories)
    in ascending row index, each its own step.
    Returns (cat_ptr int64[nsteps+1], cat_rows int32[m], n_oclass)."""
    color = np.asarray(color)
    ncol = int(color.max()) + 1 if color.size else 0
    sizes = np.bincount(color, minlength=ncol)
    steps = []
    for c in range(ncol):
        if sizes[c] >= 2:
            steps.append(np.nonzero(color == c)[0])
    n_oclass = len(steps)
    singles = np.nonzero(sizes[color] == 1)[0]
    steps.extend([np.array([i]) for i in singles])
    cat_ptr = np.zeros(len(steps) + 1, dtype=np.int64)
    cat_ptr[1:] = np.cumsum([s.size for s in steps])
    cat_rows = np.concatenate(steps).astype(np.int32) if steps else np.zeros(0, np.int32)
    return cat_ptr, cat_rows, n_oclass


def category_overlap(m: int, indptr, indices, cat_ptr, cat_rows) -> np.ndarray:
    """Per step: 1 if two of its rows share a column (only possible with thr > 0)."""
    nsteps = cat_ptr.size - 1
    step_of = np.empty(m, dtype=np.int32)
    for k in range(nsteps):
        step_of[cat_rows[cat_ptr[k]:cat_ptr[k + 1]]] = k
    out = np.zeros(nsteps, dtype=np.uint8)
    _lib().orc_category_overlap(m, _p(np.ascontiguousarray(indptr, np.int64)), _p(np.ascontiguousarray(indices, np.int32)),
                                _p(step_of), nsteps, _p(out))
    return out


# ------------------------------------------------------------------ preprocess (Alg 5 steps 1-4)
@dataclass
class Preprocessed:
    m: int
    perm: np.ndarray       # int32 [m], new -> old
    iperm: np.ndarray      # int32 [m], old -> new
    indptr: np.ndarray     # A~ (RCM frame)
    indices: np.ndarray
    data: np.ndarray
    nrm2: np.ndarray       # ||a~_i||^2, RCM frame
    color: np.ndarray      # int32 [m], RCM-frame rows
    cat_ptr: np.ndarray    # int64 [nsteps+1]
    cat_rows: np.ndarray   # int32 [m], schedule order
    n_oclass: int
    overlap: np.ndarray    # uint8 [nsteps]
    bw_before: int
    bw_after: int
    thr: float = 0.0
    extras: dict = field(default_factory=dict)

    @property
    def nsteps(self) -> int:
        return int(self.cat_ptr.size - 1)


def preprocess(m: int, indptr, indices, data, thr: float = 0.0, reorder: int = 1) -> Preprocessed:
    """Alg 5 steps 1-4 at row granularity:
    O1 canonicalise, O3 RCM (or identity), O4 permute, nrm2 on A~ rows,
    O6 first-fit + schedule."""
    indptr, indices, data = canonicalize(m, indptr, indices, data)
    perm = rcm(m, indptr, indices) if reorder else np.arange(m, dtype=np.int32)
    iperm = np.empty(m, dtype=np.int32)
    iperm[perm] = np.arange(m, dtype=np.int32)
    tp, ti, td = permute_matrix(m, indptr, indices, data, perm)
    nrm2 = row_nrm2(m, tp, td)
    color = first_fit(m, tp, ti, td, nrm2, thr)
    cat_ptr, cat_rows, n_oclass = schedule(color)
    overlap = category_overlap(m, tp, ti, cat_ptr, cat_rows) if thr > 0 else np.zeros(cat_ptr.size - 1, np.uint8)
    return Preprocessed(m, perm, iperm, tp, ti, td, nrm2, color, cat_ptr, cat_rows, n_oclass, overlap,
                        bandwidth(m, indptr, indices), bandwidth(m, tp, ti), float(thr))


# ------------------------------------------------------------------ O7 sweep
def sweep(pre: Preprocessed, f_t: np.ndarray, x_t: np.ndarray, nsweeps: int = 1) -> np.ndarray:
    """O7: `nsweeps` sweeps of Eq 1.2 in schedule order on A~ x~ = f~ (in place on x_t, RCM
    frame).  Plain C, row by row."""
    lib = _lib()
    scratch = np.empty(max(pre.m, 1))
    for _ in range(nsweeps):
        lib.orc_sweep(pre.m, _p(pre.indptr), _p(pre.indices), _p(pre.data), _p(pre.nrm2), _p(f_t), _p(x_t),
                      pre.nsteps, _p(pre.cat_ptr), _p(pre.cat_rows), _p(pre.overlap), _p(scratch))
    return x_t


def sweep_rows_py(pre: Preprocessed, f_t: np.ndarray, x_t: np.ndarray, on_step=None) -> np.ndarray:
    """One sweep of Eq 1.2 in pure Python, row by row (small cases).
    on_step(k, rows, x_before, x_after) is called after every schedule step (for pins)."""
    ip, ix, vd = pre.indptr, pre.indices, pre.data
    for k in range(pre.nsteps):
        rows = pre.cat_rows[pre.cat_ptr[k]:pre.cat_ptr[k + 1]]
        x_before = x_t.copy() if on_step is not None else None
        if not pre.overlap[k]:
            for i in rows:
                s = 0.0
                for p in range(ip[i], ip[i + 1]):
                    s = s + vd[p] * x_t[ix[p]]
                alpha = (f_t[i] - s) / pre.nrm2[i]
                for p in range(ip[i], ip[i + 1]):
                    x_t[ix[p]] = x_t[ix[p]] + alpha * vd[p]
        else:
            alphas = []
            for i in rows:
                s = 0.0
                for p in range(ip[i], ip[i + 1]):
                    s = s + vd[p] * x_t[ix[p]]
                alphas.append((f_t[i] - s) / pre.nrm2[i])
            for i, alpha in zip(rows, alphas):
                for p in range(ip[i], ip[i + 1]):
                    x_t[ix[p]] = x_t[ix[p]] + alpha * vd[p]
        if on_step is not None:
            on_step(k, rows, x_before, x_t.copy())
    return x_t


def sweep_numpy(pre: Preprocessed, f_t: np.ndarray, x_t: np.ndarray) -> np.ndarray:
    """One sweep in the block form of Eq 1.3 with the Lemma-1 collapse:
    for each step K: r = f~_K - A~_K x~; x~ += A~_K^T (r / nrm2_K).  For disjoint categories this
    is the same arithmetic as the row-by-row form (each x~ entry receives one product)."""
    A = sp.csr_matrix((pre.data, pre.indices, pre.indptr), shape=(pre.m, pre.m))
    for k in range(pre.nsteps):
        rows = pre.cat_rows[pre.cat_ptr[k]:pre.cat_ptr[k + 1]]
        AK = A[rows]
        r = f_t[rows] - AK @ x_t
        x_t += AK.T @ (r / pre.nrm2[rows])
    return x_t


def block_step_pinv(AK_dense: np.ndarray, fK: np.ndarray, x: np.ndarray) -> np.ndarray:
    """Eq 1.3 literally: x + A_tau^dagger (f_tau - A_tau x), pseudo-inverse via
    numpy.linalg.pinv (the paper's lsqminnorm/pinv).  Used only by pins."""
    return x + np.linalg.pinv(AK_dense) @ (fK - AK_dense @ x)


# ------------------------------------------------------------------ O8 check values
def rse(x, x_star) -> float:
    """RSE = ||x - x*||_2 / ||x*||_2; frame independent (Eq 4.1)."""
    x = np.ascontiguousarray(x, np.float64)
    xs = np.ascontiguousarray(x_star, np.float64)
    return float(_lib().orc_rse(x.size, _p(x), _p(xs)))


def relres(pre: Preprocessed, f_t, x_t) -> float:
    return float(_lib().orc_relres(pre.m, _p(pre.indptr), _p(pre.indices), _p(pre.data), _p(f_t), _p(x_t)))


def residual_norm(m: int, indptr, indices, data, f, x) -> float:
    """||f - A x||_2 in the user's frame (SPEC.md:55-58 spmv, ascending-column sums)."""
    ip = np.ascontiguousarray(indptr, np.int64)
    ix = np.ascontiguousarray(indices, np.int32)
    vd = np.ascontiguousarray(data, np.float64)
    f = np.ascontiguousarray(f, np.float64)
    x = np.ascontiguousarray(x, np.float64)
    return float(np.sqrt(_lib().orc_residual_sumsq(m, _p(ip), _p(ix), _p(vd), _p(f), _p(x))))


# ------------------------------------------------------------------ solve (Alg 5)
@dataclass
class SolveResult:
    x: np.ndarray          # user frame
    sweeps: int
    termination: int
    value: float           # final RSE or RELRES
    trace: np.ndarray | None
    pre: Preprocessed


def solve(m, indptr, indices, data, f, x_star=None, x0=None, thr: float = 0.0, reorder: int = 1,
          tol: float = 1e-6, max_sweeps: int = 500000, stop: str = "rse", keep_trace: bool = False,
          pre: Preprocessed | None = None) -> SolveResult:
    """Algorithm 5 at row granularity: preprocess, sweep until the §5.1 rule
    (x0 = 0, RSE < 1e-6 or the 5e5 cap), back-permute."""
    if pre is None:
        pre = preprocess(m, indptr, indices, data, thr=thr, reorder=reorder)
    f_t = permute_vector(f, pre.perm)
    x_t = permute_vector(np.zeros(m) if x0 is None else x0, pre.perm)
    if stop == "rse":
        if x_star is None:
            raise OracleError(ERR_ARG, "RSE stop needs x_star")
        xs_t = permute_vector(x_star, pre.perm)
        code = 0
    else:
        xs_t = np.zeros(1)
        code = 1
    sweeps = ctypes.c_int64()
    term = ctypes.c_int32()
    val = ctypes.c_double()
    trace = np.empty(max_sweeps) if keep_trace else None
    _lib().orc_solve(m, _p(pre.indptr), _p(pre.indices), _p(pre.data), _p(pre.nrm2), _p(f_t), _p(x_t), _p(xs_t),
                     pre.nsteps, _p(pre.cat_ptr), _p(pre.cat_rows), _p(pre.overlap), code, float(tol),
                     int(max_sweeps), ctypes.byref(sweeps), ctypes.byref(term), ctypes.byref(val),
                     _p(trace) if trace is not None else None)
    if trace is not None:
        trace = trace[:sweeps.value].copy()
    return SolveResult(unpermute_vector(x_t, pre.perm), int(sweeps.value), int(term.value), float(val.value), trace, pre)


def run_sweeps(pre: Preprocessed, f, nsweeps: int, x0=None) -> np.ndarray:
    """Exactly `nsweeps` sweeps from x0 (default 0); returns x in the user frame."""
    f_t = permute_vector(f, pre.perm)
    x_t = permute_vector(np.zeros(pre.m) if x0 is None else x0, pre.perm)
    sweep(pre, f_t, x_t, nsweeps)
    return unpermute_vector(x_t, pre.perm)


# ------------------------------------------------------------------ NEXT-4: residual-ordered sweep
# Reading R-G: not the paper's POBK rule (P:248 avoids
# residual selection) but the greedy "largest residual block first" idea of GRBK / GRMK
# (Alg 1): at the start of every sweep each schedule step (category) K gets the score
#     rho_K = ||f~_K - A~_K x~||^2 / ||A~_K||_F^2          (residuals and norms at the sweep start)
# and the sweep applies the steps in decreasing rho (ties: ascending step index), each as in O7.
# The two sums of a step run over its rows in schedule order in a fixed two-level grouping:
# chunks of CHUNK consecutive rows summed left to right, then the chunk sums left to right.
CHUNK = 256


def row_residuals(pre: Preprocessed, f_t, x_t) -> np.ndarray:
    r = np.empty(pre.m)
    _lib().orc_row_residuals(pre.m, _p(pre.indptr), _p(pre.indices), _p(pre.data), _p(np.ascontiguousarray(f_t)),
                             _p(np.ascontiguousarray(x_t)), _p(r))
    return r


def seq_sum(v) -> float:
    """Left-to-right sum from 0.0 (no pairwise summation)."""
    s = 0.0
    for a in np.asarray(v, dtype=np.float64).tolist():
        s = s + a
    return s


def two_level_sum(v, chunk: int = CHUNK) -> float:
    v = np.asarray(v, dtype=np.float64)
    return seq_sum([seq_sum(v[a:a + chunk]) for a in range(0, v.size, chunk)])


def step_scores(pre: Preprocessed, f_t, x_t) -> np.ndarray:
    r = row_residuals(pre, f_t, x_t)
    out = np.empty(pre.nsteps)
    for k in range(pre.nsteps):
        rows = pre.cat_rows[pre.cat_ptr[k]:pre.cat_ptr[k + 1]]
        out[k] = two_level_sum(r[rows] * r[rows]) / two_level_sum(pre.nrm2[rows])
    return out


def residual_order(scores) -> np.ndarray:
    """Steps by decreasing score, ties by ascending index (a stable sort of -score)."""
    return np.argsort(-np.asarray(scores), kind="stable").astype(np.int32)


def _apply_step(pre: Preprocessed, k: int, f_t, x_t, scratch):
    ptr = np.ascontiguousarray(pre.cat_ptr[k:k + 2], dtype=np.int64)
    ov = np.ascontiguousarray(pre.overlap[k:k + 1], dtype=np.uint8)
    _lib().orc_sweep(pre.m, _p(pre.indptr), _p(pre.indices), _p(pre.data), _p(pre.nrm2), _p(f_t), _p(x_t), 1,
                     _p(ptr), _p(pre.cat_rows), _p(ov), _p(scratch))


def sweep_ordered(pre: Preprocessed, f_t, x_t, nsweeps: int = 1, orders=None) -> np.ndarray:
    """nsweeps residual-ordered sweeps (in place, RCM frame); `orders` collects each sweep's order."""
    scratch = np.empty(max(pre.m, 1))
    for _ in range(nsweeps):
        order = residual_order(step_scores(pre, f_t, x_t))
        if orders is not None:
            orders.append(order)
        for k in order:
            _apply_step(pre, int(k), f_t, x_t, scratch)
    return x_t


def run_sweeps_ordered(pre: Preprocessed, f, nsweeps: int, x0=None) -> np.ndarray:
    f_t = permute_vector(f, pre.perm)
    x_t = permute_vector(np.zeros(pre.m) if x0 is None else x0, pre.perm)
    sweep_ordered(pre, f_t, x_t, nsweeps)
    return unpermute_vector(x_t, pre.perm)


def solve_ordered(pre: Preprocessed, f, x_star, tol: float, max_sweeps: int):
    """Residual-ordered sweeps to RSE < tol; returns (x user frame, sweeps, term, value)."""
    f_t = permute_vector(f, pre.perm)
    xs_t = permute_vector(x_star, pre.perm)
    x_t = np.zeros(pre.m)
    term, v, s = TERM_MAX_SWEEPS, float("nan"), 0
    for s in range(1, max_sweeps + 1):
        sweep_ordered(pre, f_t, x_t, 1)
        v = rse(x_t, xs_t)
        if not np.isfinite(v):
            term = TERM_NONFINITE
            break
        if v < tol:
            term = TERM_CONVERGED
            break
    return unpermute_vector(x_t, pre.perm), s, term, v
