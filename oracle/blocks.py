"""Paper-literal POBK oracle: k uniform row blocks (TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py).

Algorithm 5 as written, step by step in the paper's order and notation, for
the NEXT-2 row of SURVEY.md §8(f).  The row-granularity hot path (oracle/core.py) reads the
blocks as single rows; here they are the paper's k < 20 uniform chunks:

  1. RCM: A~ = P A P^T, f~ = P f                                (Eq 3.1; core.preprocess)
  2. uniform chunking: blocks 1..k-1 take [m/k] consecutive rows, block k the rest
     centroids  A-bar_i = mean of block i's rows (a dense m-vector)                  (Alg 5 step 2)
  3. cosine table C(i,j) = |G(i,j)| / (||A-bar_i|| ||A-bar_j||), G(i,j) = (A-bar_i, A-bar_j),
     diagonal 1                                                          (|.|: SURVEY Z6)
  4. classes: C(i,j) < thr counts as orthogonal; for i = 1..k not yet used, the first
     unused j > i with C(i,j) < thr forms class{i} = (i, j), no block in two classes;
     Oclass = those pairs, Nclass = the unpaired blocks ascending
  5. one iteration (sweep, SURVEY Z9 / S:345-349): for each pair (tau1, tau2) in Oclass order
     x~ <- x~ + A_tau1^+ (f_tau1 - A_tau1 x~), then the same with tau2 (Alg 5 lines 7-8); then each
     Nclass block in ascending order (lines 9-10); A_tau^+ as the minimum-norm least-squares
     operator (MATLAB lsqminnorm): numpy.linalg.pinv once per block (block_step: the same
     step through numpy.linalg.lstsq) -- library steps
  6. stop when RSE < tol, x = P^T x~

Diagnostics (Definitions 1-2): zn = n1/(k k), nn = n2 nm/(k k) on the table with
C(i,j) < thr set to 0 -- n1 zero entries, n2 nonzero entries of mean nm (the diagonal,
1, counts as nonzero).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from . import core

__all__ = ["uniform_blocks", "centroids", "cosine_table", "classify", "zn_nn", "BlockPre", "block_preprocess",
           "block_step", "block_sweep", "block_solve", "block_schedule"]


def uniform_blocks(m: int, k: int) -> np.ndarray:
    """Block boundaries [k+1]: blocks 1..k-1 take floor(m/k) rows each in order, block k the
    remaining rows."""
    if not (1 <= k <= m):
        raise core.OracleError(core.ERR_ARG, f"k must be in [1, m], got k={k}, m={m}")
    q = m // k
    ptr = [i * q for i in range(k)] + [m]
    return np.asarray(ptr, dtype=np.int64)


def centroids(A: sp.csr_matrix, ptr: np.ndarray) -> np.ndarray:
    """A-bar_i = (1/|tau_i|) sum_{r in tau_i} row_r (dense k x m, P:218 / Alg 5 step 2)."""
    k = ptr.size - 1
    out = np.zeros((k, A.shape[1]))
    for i in range(k):
        rows = A[ptr[i]:ptr[i + 1]].toarray()
        out[i] = rows.sum(axis=0) / rows.shape[0]
    return out


def cosine_table(cent: np.ndarray) -> np.ndarray:
    """C(i,j) = |G(i,j)| / (||A-bar_i|| ||A-bar_j||), G(i,j) = (A-bar_i, A-bar_j), once per
    unordered pair (k(k-1)/2 inner products), C(i,i) = 1."""
    k = cent.shape[0]
    nrm = np.sqrt((cent * cent).sum(axis=1))
    if np.any(nrm == 0.0):
        raise core.OracleError(core.ERR_ARG, f"zero centroid in block {int(np.argmin(nrm))}")
    C = np.eye(k)
    for i in range(k):
        for j in range(i + 1, k):
            g = float(np.dot(cent[i], cent[j]))
            C[i, j] = C[j, i] = abs(g) / (nrm[i] * nrm[j])
    return C


def classify(C: np.ndarray, thr: float):
    """Oclass pairs and Nclass blocks: scan i ascending; an unused i takes the first unused
    j > i with C(i,j) < thr (the pair is class{i}); unpaired blocks form Nclass, ascending."""
    k = C.shape[0]
    used = [False] * k
    pairs = []
    for i in range(k):
        if used[i]:
            continue
        for j in range(i + 1, k):
            if not used[j] and C[i, j] < thr:
                pairs.append((i, j))
                used[i] = used[j] = True
                break
    nclass = [i for i in range(k) if not used[i]]
    return pairs, nclass


def zn_nn(C: np.ndarray, thr: float):
    """Definitions 1-2 on the table with entries < thr set to 0 (thr = 0:
    exact zeros only): zn = n1/(k k), nn = n2 * nm / (k k)."""
    k = C.shape[0]
    Ct = np.where(C < thr, 0.0, C)
    nz = Ct[Ct != 0.0]
    n1 = k * k - nz.size
    nm = float(nz.mean()) if nz.size else 0.0
    return n1 / (k * k), nz.size * nm / (k * k)


def block_schedule(pairs, nclass) -> list[int]:
    """One iteration's block order: each Oclass pair (tau1 then tau2), then Nclass ascending."""
    return [b for pr in pairs for b in pr] + list(nclass)


@dataclass
class BlockPre:
    pre: core.Preprocessed   # RCM (step 1) -- the row-level preprocessing's permutation and A~
    k: int
    thr: float
    ptr: np.ndarray          # [k+1] block boundaries in the RCM frame
    C: np.ndarray            # k x k cosine table
    pairs: list
    nclass: list
    zn: float
    nn: float

    @property
    def order(self) -> list[int]:
        return block_schedule(self.pairs, self.nclass)

    def block(self, i: int) -> sp.csr_matrix:
        pre = self.pre
        A = sp.csr_matrix((pre.data, pre.indices, pre.indptr), shape=(pre.m, pre.m))
        return A[self.ptr[i]:self.ptr[i + 1]]


def block_preprocess(m: int, indptr, indices, data, k: int, thr: float, reorder: int = 1) -> BlockPre:
    """Alg 5 steps 1-4 with k uniform blocks."""
    pre = core.preprocess(m, indptr, indices, data, reorder=reorder)
    A = sp.csr_matrix((pre.data, pre.indices, pre.indptr), shape=(m, m))
    ptr = uniform_blocks(m, k)
    C = cosine_table(centroids(A, ptr))
    pairs, nclass = classify(C, thr)
    zn, nn = zn_nn(C, thr)
    return BlockPre(pre, k, float(thr), ptr, C, pairs, nclass, zn, nn)


def block_step(A_tau, f_tau: np.ndarray, x: np.ndarray) -> np.ndarray:
    """Eq 1.3 / 3.3: x + A_tau^+ (f_tau - A_tau x), the pseudo-inverse applied as
    the minimum-norm least-squares solve (lsqminnorm)."""
    Ad = A_tau.toarray() if sp.issparse(A_tau) else np.asarray(A_tau)
    r = f_tau - Ad @ x
    dx = np.linalg.lstsq(Ad, r, rcond=None)[0]
    return x + dx


def _pinvs(bp: BlockPre):
    """A_tau^+ of every block, computed once (numpy.linalg.pinv: the SVD pseudo-inverse, equal to
    the minimum-norm least-squares operator of lsqminnorm) -- SPEC.md:366 'block
    factorizations are computed once and reused'."""
    out = []
    for i in range(bp.k):
        Ad = bp.block(i).toarray()
        out.append((Ad, np.linalg.pinv(Ad), bp.ptr[i], bp.ptr[i + 1]))
    return out


def _apply(blocks, order, f_t, x):
    for b in order:  # Eq 3.3: x + A_tau^+ (f_tau - A_tau x)
        Ad, Pd, r0, r1 = blocks[b]
        x = x + Pd @ (f_t[r0:r1] - Ad @ x)
    return x


def block_sweep(bp: BlockPre, f_t: np.ndarray, x_t: np.ndarray, nsweeps: int = 1) -> np.ndarray:
    """nsweeps iterations of the Alg 5 loop in the RCM frame; returns the new x~."""
    x = np.array(x_t, dtype=np.float64)
    blocks = _pinvs(bp)
    for _ in range(nsweeps):
        x = _apply(blocks, bp.order, f_t, x)
    return x


def block_solve(bp: BlockPre, f, x_star, tol: float = 1e-6, max_sweeps: int = 500000, x0=None):
    """Alg 5 to the paper's rule: RSE < tol after an iteration or the cap; returns
    (x in the user frame, sweeps, termination, final RSE)."""
    pre = bp.pre
    f_t = core.permute_vector(f, pre.perm)
    xs_t = core.permute_vector(x_star, pre.perm)
    x = core.permute_vector(np.zeros(pre.m) if x0 is None else x0, pre.perm)
    blocks = _pinvs(bp)
    den = np.linalg.norm(xs_t)
    term, v, s = core.TERM_MAX_SWEEPS, float("nan"), 0
    for s in range(1, max_sweeps + 1):
        x = _apply(blocks, bp.order, f_t, x)
        v = float(np.linalg.norm(x - xs_t) / den)
        if not np.isfinite(v):
            term = core.TERM_NONFINITE
            break
        if v < tol:
            term = core.TERM_CONVERGED
            break
    return core.unpermute_vector(x, pre.perm), s, term, v
