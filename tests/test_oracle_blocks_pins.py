"""Pins of the paper-literal k-block POBK oracle (oracle/blocks.py)
against what the paper and the mathematics fix: the chunking rule, hand values of the
centroid cosine table, hand traces of the first-orthogonal pairing,
the Definition 1-2 examples, exactness of the block projection (Eq 3.3,
Lemma 1), closed-form one-sweep cases and a dense direct solve."""
import numpy as np
import pytest
import scipy.sparse as sp

import oracle as O
from oracle import blocks as OB
from workloads import gen


@pytest.mark.parametrize("m,k,sizes", [(10, 2, [5, 5]), (10, 3, [3, 3, 4]), (5, 5, [1] * 5), (7, 1, [7]), (9, 4, [2, 2, 2, 3])])
def test_uniform_blocks(m, k, sizes):
    """the first k-1 blocks take [m/k] rows each in order, the k-th the rest."""
    ptr = OB.uniform_blocks(m, k)
    assert np.diff(ptr).tolist() == sizes and ptr[0] == 0 and ptr[-1] == m


def test_uniform_blocks_errors():
    with pytest.raises(O.OracleError):
        OB.uniform_blocks(5, 6)
    with pytest.raises(O.OracleError):
        OB.uniform_blocks(5, 0)


def test_centroids_hand_values():
    """a block of identical rows has that row as centroid; {e1, e2} -> (0.5, 0.5, 0)."""
    A = sp.csr_matrix(np.array([[1.0, 2.0, 0.0], [1.0, 2.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0]]))
    c = OB.centroids(A, np.array([0, 2, 4]))
    assert c.tolist() == [[1.0, 2.0, 0.0], [0.5, 0.5, 0.0]]


@pytest.mark.parametrize("a,b,cos", [((1, 0, 0), (0, 1, 0), 0.0), ((1, 2, 3), (2, 4, 6), 1.0),
                                     ((1, 1, 0), (1, 0, 1), 0.5), ((1, 1, 0), (-1, 0, -1), 0.5)])
def test_cosine_table_hand_values(a, b, cos):
    """P:218 C = G/(||.|| ||.||), absolute: axes 0, collinear 1, 1/(sqrt2 sqrt2);
    a negative inner product gives the same |cos|; diagonal 1, symmetric."""
    C = OB.cosine_table(np.array([a, b], dtype=float))
    assert abs(C[0, 1] - cos) < 1e-15 and C[0, 1] == C[1, 0] and C[0, 0] == C[1, 1] == 1.0


def test_cosine_table_zero_centroid_is_an_error():
    with pytest.raises(O.OracleError):
        OB.cosine_table(np.array([[1.0, 0.0], [0.0, 0.0]]))


def _table(k, small):
    C = np.full((k, k), 0.9)
    np.fill_diagonal(C, 1.0)
    for i, j in small:
        C[i, j] = C[j, i] = 0.01
    return C


@pytest.mark.parametrize("k,small,pairs,nclass", [
    (4, [(0, 2), (1, 3)], [(0, 2), (1, 3)], []),        # oclass = [(1,3),(2,4)]
    (4, [], [], [0, 1, 2, 3]),                           # nothing orthogonal
    (3, [(0, 1), (0, 2)], [(0, 1)], [2]),                # the first j wins; 3 cannot re-pair
    (5, [(0, 3), (1, 3), (1, 4), (2, 4)], [(0, 3), (1, 4)], [2]),   # a used j is skipped
])
def test_classify_hand_traces(k, small, pairs, nclass):
    """for each block i the first (unused) block j > i orthogonal to it joins class{i}; no
    block in two classes; the rest is Nclass (hand-traced greedy scans)."""
    p, n = OB.classify(_table(k, small), 0.05)
    assert p == pairs and n == nclass
    assert OB.block_schedule(p, n) == [b for pr in pairs for b in pr] + nclass


@pytest.mark.parametrize("C,thr,zn,nn", [
    ([[1, 0], [0, 1]], 0.0, 0.5, 0.5),
    ([[1, 1], [1, 1]], 0.0, 0.0, 1.0),
    ([[1, 0, 0], [0, 1, 0.4], [0, 0.4, 1]], 0.0, 4 / 9, 3.8 / 9),
    ([[1, 0.02, 0.3], [0.02, 1, 0.4], [0.3, 0.4, 1]], 0.05, 2 / 9, (3 + 0.6 + 0.8) / 9),  # thr zeroes 0.02
])
def test_zn_nn_definitions(C, thr, zn, nn):
    """Definitions 1-2: zn = n1/(k k); nn = n2 * (mean of the nonzeros) / (k k)."""
    a, b = OB.zn_nn(np.array(C, dtype=float), thr)
    assert abs(a - zn) < 1e-15 and abs(b - nn) < 1e-15


def test_block_step_single_row_is_eq_1_2():
    """A one-row block reproduces Eq 1.2: a = (3,4), f = 5, x = 0 -> (0.6, 0.8)."""
    x = OB.block_step(np.array([[3.0, 4.0]]), np.array([5.0]), np.zeros(2))
    assert np.allclose(x, [0.6, 0.8], rtol=0, atol=1e-15)


@pytest.mark.parametrize("seed", range(4))
def test_block_step_projection_properties(seed):
    """Eq 3.3 with A_tau^+ (Lemma 1): for a full-row-rank block the new point satisfies
    the block's equations exactly and moves only within range(A_tau^T) (minimum norm); the error
    never grows (Eq 4.6)."""
    rng = np.random.default_rng(seed)
    Ad = rng.standard_normal((4, 9))
    xs = rng.standard_normal(9)
    x = rng.standard_normal(9)
    xn = OB.block_step(Ad, Ad @ xs, x)
    assert np.linalg.norm(Ad @ xn - Ad @ xs) <= 1e-12 * np.linalg.norm(Ad @ xs)
    z, res, *_ = np.linalg.lstsq(Ad.T, xn - x, rcond=None)
    assert np.linalg.norm(Ad.T @ z - (xn - x)) <= 1e-12 * np.linalg.norm(xn - x)
    assert np.linalg.norm(xn - xs) <= np.linalg.norm(x - xs) + 1e-12


def test_one_block_is_a_direct_solve():
    """k = 1: the single block is A~ itself (nonsingular), so one iteration gives x* (A~^+ = A~^-1)."""
    s = gen.from_csr("rb", gen.scramble(gen.random_banded(30, 5, half=3), 6), 7)
    bp = OB.block_preprocess(s.m, s.indptr, s.indices, s.data, k=1, thr=0.05)
    x, sweeps, term, v = OB.block_solve(bp, s.f, s.x_star, tol=1e-10)
    assert sweeps == 1 and term == O.TERM_CONVERGED and np.linalg.norm(x - s.x_star) <= 1e-10 * np.linalg.norm(s.x_star)


def test_orthonormal_blocks_exact_after_one_sweep():
    """orthonormal rows in k = 2 mutually orthogonal blocks: one iteration (two projections
    onto orthogonal subspaces) reaches x*."""
    Q, _ = np.linalg.qr(np.random.default_rng(1).standard_normal((8, 8)))
    A = sp.csr_matrix(Q)
    s = gen.from_csr("q", A, 2)
    bp = OB.block_preprocess(s.m, s.indptr, s.indices, s.data, k=2, thr=0.05, reorder=0)
    x, sweeps, term, v = OB.block_solve(bp, s.f, s.x_star, tol=1e-10)
    assert sweeps == 1 and term == O.TERM_CONVERGED


@pytest.mark.parametrize("seed", range(4))
def test_dense_solve_agreement(seed):
    """random 50x50 banded system, k = 5 -> RSE <= 1e-6 and the dense direct solve to 1e-5."""
    A = gen.scramble(gen.random_banded(50, 700 + seed, half=3), 800 + seed)
    s = gen.from_csr("rb", A, seed)
    bp = OB.block_preprocess(50, s.indptr, s.indices, s.data, k=5, thr=0.05)
    x, sweeps, term, v = OB.block_solve(bp, s.f, s.x_star, tol=1e-6, max_sweeps=10000)
    assert term == O.TERM_CONVERGED
    xd = np.linalg.solve(A.toarray(), s.f)
    assert np.linalg.norm(x - xd) <= 1e-5 * np.linalg.norm(xd)


def test_blocks_cover_and_schedule_is_a_permutation_of_blocks():
    s = gen.make("lap2d5_32")
    bp = OB.block_preprocess(s.m, s.indptr, s.indices, s.data, k=7, thr=0.05)
    assert sorted(bp.order) == list(range(7))
    assert all(bp.C[i, j] < 0.05 for i, j in bp.pairs)
    # RCM-banded blocks far apart share no columns: exactly zero centroid cosines ("natural
    # orthogonality of banded matrices")
    assert bp.C[0, 6] == 0.0 and bp.zn > 0


@pytest.mark.parametrize("seed", range(3))
def test_pinv_step_equals_lstsq_step_and_gram_form(seed):
    """The cached operator numpy.linalg.pinv(A_tau) applies the same step as the per-step minimum-
    norm solve (lstsq), and for a full-row-rank block both equal A_tau^T (A_tau A_tau^T)^-1 (Lemma 1,
    P:257-261): three library routes to A_tau^+ agree to rounding."""
    rng = np.random.default_rng(50 + seed)
    Ad = rng.standard_normal((5, 12))
    x, f = rng.standard_normal(12), rng.standard_normal(5)
    a = OB.block_step(Ad, f, x)
    b = x + np.linalg.pinv(Ad) @ (f - Ad @ x)
    c = x + Ad.T @ np.linalg.solve(Ad @ Ad.T, f - Ad @ x)
    assert np.linalg.norm(a - b) <= 1e-12 * np.linalg.norm(a) and np.linalg.norm(a - c) <= 1e-12 * np.linalg.norm(a)
