"""Pins for the oracle (-m "not gpu"): the oracle checked against facts fixed by the paper and
by mathematics -- hand-traced fixtures, brute force, closed forms, invariants, special cases
that reduce to a library routine -- never against a retyped copy of itself.
(SURVEY.md §8(c) "What pins each part".)"""
import itertools
import json
import math
import os

import numpy as np
import pytest
import scipy.sparse as sp

import oracle as O
from workloads import gen

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _from_edges(m, edges, diag=4.0):
    r = [i for i in range(m)] + [a for a, b in edges] + [b for a, b in edges]
    c = [i for i in range(m)] + [b for a, b in edges] + [a for a, b in edges]
    v = [diag] * m + [-1.0] * (2 * len(edges))
    return gen.canonical(sp.coo_matrix((v, (r, c)), shape=(m, m)))


def _pre_from_matrix(A, thr=0.0, reorder=1):
    A = gen.canonical(A)
    return O.preprocess(A.shape[0], A.indptr, A.indices, A.data, thr=thr, reorder=reorder)


HAND = json.load(open(os.path.join(GOLDEN, "handtraced_rcm_partition.json")))["cases"]


# ------------------------------------------------------------------ O3 RCM + O6 partition: hand traces
@pytest.mark.parametrize("case", HAND, ids=[c["name"] for c in HAND])
def test_handtraced_rcm_and_partition(case):
    A = _from_edges(case["m"], case["edges"])
    pre = O.preprocess(case["m"], A.indptr, A.indices, A.data)
    assert pre.perm.tolist() == case["perm"]
    assert pre.bw_after == case["bandwidth_after"]
    assert pre.color.tolist() == case["color"]
    assert pre.cat_ptr.tolist() == case["cat_ptr"]
    assert pre.cat_rows.tolist() == case["cat_rows"]
    assert pre.n_oclass == case["n_oclass"]
    # the pure-Python restatements agree on these too
    assert O.rcm_py(case["m"], A.indptr, A.indices).tolist() == case["perm"]
    assert O.first_fit_py(case["m"], pre.indptr, pre.indices, pre.data, pre.nrm2).tolist() == case["color"]


def test_gl_termination_reading_matters():
    """Z11: returning r instead of x gives a different permutation (recorded in the fixture)."""
    case = [c for c in HAND if c["name"] == "path_with_mid_leaf_two_gl_rounds"][0]
    assert case["perm"] != case["perm_if_root_were_r"]


# ------------------------------------------------------------------ O3: brute force + properties
def test_rcm_path5_matches_bruteforce_minimum():
    """a 5-node path in scrambled order -> bandwidth 1 = min over all 5! orderings."""
    A = gen.scramble(_from_edges(5, [(0, 1), (1, 2), (2, 3), (3, 4)]), 7)
    best = min(O.bandwidth(5, *_perm_csr(A, np.array(p))) for p in itertools.permutations(range(5)))
    perm = O.rcm(5, A.indptr, A.indices)
    assert best == 1
    assert O.bandwidth(5, *_perm_csr(A, perm)) == best


def _perm_csr(A, perm):
    ip, ix, _ = O.permute_matrix(A.shape[0], A.indptr, A.indices, A.data, perm)
    return ip, ix


def test_rcm_scrambled_path_2000_bandwidth_1():
    """SPEC.md:477 (acceptance #5, synthetic part): scrambled tridiagonal m=2000 -> bandwidth <= 5;
    RCM from a path endpoint reproduces the path, bandwidth exactly 1."""
    m = 2000
    A = gen.scramble(_from_edges(m, [(i, i + 1) for i in range(m - 1)]), 11)
    assert O.bandwidth(m, A.indptr, A.indices) > 100
    perm = O.rcm(m, A.indptr, A.indices)
    assert O.bandwidth(m, *_perm_csr(A, perm)) == 1


def _check_rcm_properties(m, indptr, indices, perm):
    """Independent checker of the pinned O3 rule (shares no code with the oracle): reverse(perm)
    is a concatenation of FIFO BFS orders, one per component in ascending min-index order, each
    enqueueing unvisited neighbours in ascending (deg, idx), from a root satisfying the
    George-Liu termination condition."""
    adj = [set() for _ in range(m)]
    for i in range(m):
        for j in indices[indptr[i]:indptr[i + 1]]:
            if j != i:
                adj[i].add(int(j)); adj[int(j)].add(i)
    deg = [len(a) for a in adj]
    assert sorted(perm.tolist()) == list(range(m))          # bijection
    order = perm[::-1].tolist()
    pos = 0
    seen = set()
    comp_mins = []
    while pos < m:
        root = order[pos]
        # re-run the BFS the rule prescribes from this root and compare
        q, vis, out = [root], {root}, []
        while q:
            v = q.pop(0)
            out.append(v)
            for u in sorted((u for u in adj[v] if u not in vis and u not in seen), key=lambda u: (deg[u], u)):
                vis.add(u); q.append(u)
        assert order[pos:pos + len(out)] == out
        comp = set(out)
        comp_mins.append(min(comp))
        # George-Liu: the root is the (deg, idx)-minimal node of the last BFS level of some r in
        # its component (or the component is a single node)
        def last_min(s):
            d = {s: 0}; f = [s]
            while f:
                nf = []
                for v in f:
                    for u in adj[v]:
                        if u not in d:
                            d[u] = d[v] + 1; nf.append(u)
                f = nf
            e = max(d.values())
            return min((v for v, k in d.items() if k == e), key=lambda v: (deg[v], v))
        assert len(comp) == 1 or any(last_min(r) == root for r in comp)
        seen |= comp
        pos += len(out)
    assert comp_mins == sorted(comp_mins)


@pytest.mark.parametrize("seed", range(60))
def test_rcm_properties_random_graphs(seed):
    rng = np.random.default_rng(seed)
    m = int(rng.integers(1, 50))
    A = gen.random_pattern_graph(m, seed, p=float(rng.choice([0.02, 0.05, 0.1, 0.3])))
    perm = O.rcm(m, A.indptr, A.indices)
    _check_rcm_properties(m, A.indptr, A.indices, perm)
    assert perm.tolist() == O.rcm_py(m, A.indptr, A.indices).tolist()
    assert perm.tolist() == O.rcm(m, A.indptr, A.indices).tolist()          # determinism


def test_rcm_magnitudes():
    """SURVEY.md A.6 magnitudes: 32x32 5-point (scrambled) -> bandwidth 32, 7 categories."""
    s = gen.make("lap2d5_32")
    pre = O.preprocess(s.m, s.indptr, s.indices, s.data)
    assert pre.bw_before > 900 and pre.bw_after == 32
    assert pre.nsteps == 7 and pre.n_oclass == 7


def test_explicit_zeros_do_not_change_preprocessing():
    """SURVEY.md §8(c) hazard: the same matrix with stored zeros gives the identical perm and
    partition (zeros dropped first)."""
    A = gen.lap2d5(3).tocoo()
    r = np.concatenate([A.row, [0, 0, 8]]); c = np.concatenate([A.col, [8, 5, 0]])
    v = np.concatenate([A.data, [0.0, 0.0, 0.0]])
    B = sp.csr_matrix((v, (r, c)), shape=(9, 9)); B.sort_indices()
    assert B.nnz == A.nnz + 3
    p1 = O.preprocess(9, A.tocsr().indptr, A.tocsr().indices, A.tocsr().data)
    p2 = O.preprocess(9, B.indptr, B.indices, B.data)
    assert p1.perm.tolist() == p2.perm.tolist() and p1.color.tolist() == p2.color.tolist()


# ------------------------------------------------------------------ O1 validation
def test_canonicalize_errors():
    ok = (np.array([0, 1, 2]), np.array([0, 1]), np.array([1.0, 2.0]))
    O.canonicalize(2, *ok)
    with pytest.raises(O.OracleError) as e:
        O.canonicalize(2, np.array([0, 2, 1]), np.array([0, 1]), np.array([1.0, 2.0]))
    assert e.value.code == O.ERR_BAD_CSR
    with pytest.raises(O.OracleError) as e:
        O.canonicalize(2, np.array([0, 2, 2]), np.array([1, 0]), np.array([1.0, 2.0]))   # unsorted
    assert e.value.code == O.ERR_BAD_CSR
    with pytest.raises(O.OracleError) as e:
        O.canonicalize(2, np.array([0, 2, 3]), np.array([0, 0, 1]), np.array([1.0, 2.0, 3.0]))   # duplicate
    assert e.value.code == O.ERR_BAD_CSR
    with pytest.raises(O.OracleError) as e:
        O.canonicalize(2, np.array([0, 1, 2]), np.array([0, 2]), np.array([1.0, 2.0]))   # out of range
    assert e.value.code == O.ERR_BAD_CSR
    with pytest.raises(O.OracleError) as e:
        O.canonicalize(2, np.array([0, 1, 2]), np.array([0, 1]), np.array([1.0, 0.0]))   # zero row
    assert e.value.code == O.ERR_ZERO_ROW


# ------------------------------------------------------------------ O6 partition
def _mex_certificate(pre):
    """color[i] = mex{color[l] : l < i, rows share a column} -- characterises first-fit uniquely."""
    A = sp.csr_matrix((pre.data, pre.indices, pre.indptr), shape=(pre.m, pre.m))
    S = (abs(A) @ abs(A).T).tocsr()   # S_il != 0 iff rows i, l share a column (nonnegative entries)
    for i in range(pre.m):
        nb = S.indices[S.indptr[i]:S.indptr[i + 1]]
        used = {int(pre.color[l]) for l in nb if l < i}
        k = 0
        while k in used:
            k += 1
        assert pre.color[i] == k


def _pairwise_disjoint(pre):
    owner = {}
    for k in range(pre.nsteps):
        for i in pre.cat_rows[pre.cat_ptr[k]:pre.cat_ptr[k + 1]]:
            for c in pre.indices[pre.indptr[i]:pre.indptr[i + 1]]:
                assert owner.get((k, int(c))) is None, "two rows of one category share a column"
                owner[(k, int(c))] = i


@pytest.mark.parametrize("seed", range(40))
def test_partition_certificate_random(seed):
    rng = np.random.default_rng(100 + seed)
    m = int(rng.integers(1, 60))
    A = gen.random_pattern_graph(m, 100 + seed, p=float(rng.choice([0.03, 0.1, 0.3])))
    pre = O.preprocess(m, A.indptr, A.indices, A.data)
    _mex_certificate(pre)
    _pairwise_disjoint(pre)
    assert sorted(pre.cat_rows.tolist()) == list(range(m))
    sizes = np.diff(pre.cat_ptr)
    assert np.all(sizes[:pre.n_oclass] >= 2) and np.all(sizes[pre.n_oclass:] == 1)
    singles = pre.cat_rows[pre.cat_ptr[pre.n_oclass]:]
    assert singles.tolist() == sorted(singles.tolist())          # Nclass ascending
    oc = [int(pre.color[pre.cat_rows[pre.cat_ptr[k]]]) for k in range(pre.n_oclass)]
    assert oc == sorted(oc)                                       # Oclass ascending colour


def test_partition_certificate_config1_and_3():
    for name, n in (("lap2d5_32", None), ("lap3d7_64", 16)):
        s = gen.make(name, n=n) if n else gen.make(name)
        pre = O.preprocess(s.m, s.indptr, s.indices, s.data)
        _mex_certificate(pre)
        _pairwise_disjoint(pre)


def _row_system(rows_support, m, seed=0):
    rng = np.random.default_rng(seed)
    r, c = [], []
    for i, sup in enumerate(rows_support):
        r += [i] * len(sup); c += list(sup)
    return gen.canonical(sp.coo_matrix((rng.uniform(0.5, 1.5, len(r)), (r, c)), shape=(m, m)))


def test_spec_classify_traces_at_row_level():
    """SPEC.md:234-236, with blocks = rows and structural orthogonality (reorder off):
    (a) C(1,3), C(2,4) orthogonal only -> Oclass {1,3},{2,4};  (c) 1 _|_ 2, 1 _|_ 3 -> {1,2},{3}."""
    A = _row_system([(0, 1), (1, 2), (2, 3), (0, 3)], 4)
    pre = _pre_from_matrix(A, reorder=0)
    assert pre.cat_rows.tolist() == [0, 2, 1, 3] and pre.cat_ptr.tolist() == [0, 2, 4] and pre.n_oclass == 2
    A = _row_system([(0,), (1, 2), (2,)], 3)
    pre = _pre_from_matrix(A, reorder=0)
    assert pre.cat_rows.tolist() == [0, 1, 2] and pre.cat_ptr.tolist() == [0, 2, 3] and pre.n_oclass == 1


# ------------------------------------------------------------------ O7 sweep
def test_eq12_hand_values():
    """a=(3,4), f=5, x=0 -> (0.6, 0.8); a=(1,0), f=1 -> (1,0); on-hyperplane x
    unchanged.  2x2 systems with the second row orthogonal and consistent (zero residual)."""
    A = sp.csr_matrix(np.array([[3.0, 4.0], [4.0, -3.0]]))
    pre = _pre_from_matrix(A, reorder=0)
    assert pre.cat_rows.tolist() == [0, 1]
    x = np.zeros(2)
    O.sweep_rows_py(pre, np.array([5.0, 0.0]), x, on_step=lambda k, r, a, b: k == 0 and np.testing.assert_allclose(b, [0.6, 0.8], rtol=0, atol=2e-16))
    np.testing.assert_allclose(x, [0.6, 0.8], rtol=0, atol=2e-16)
    A = sp.csr_matrix(np.array([[1.0, 0.0], [0.0, 1.0]]))
    pre = _pre_from_matrix(A, reorder=0)
    x = O.run_sweeps(pre, np.array([1.0, 0.0]), 1)
    assert x.tolist() == [1.0, 0.0]
    x = O.run_sweeps(pre, np.array([1.0, 0.0]), 1, x0=np.array([1.0, 0.0]))
    assert x.tolist() == [1.0, 0.0]


def test_survey_2x2_worked_example():
    """SURVEY.md §8(c) sweep check: A = [[1,1],[1,-1]], x* = (1,2): thr=0 -> two steps, x = x* after
    one sweep (alpha = 3/2 then -1/2); thr>0 -> one overlapping category, same x."""
    A = sp.csr_matrix(np.array([[1.0, 1.0], [1.0, -1.0]]))
    f = np.array([3.0, -1.0])
    pre0 = _pre_from_matrix(A)
    assert pre0.nsteps == 2
    assert O.run_sweeps(pre0, f, 1).tolist() == [1.0, 2.0]
    pre1 = _pre_from_matrix(A, thr=0.5)
    assert pre1.nsteps == 1 and pre1.overlap.tolist() == [1]
    assert O.run_sweeps(pre1, f, 1).tolist() == [1.0, 2.0]


@pytest.mark.parametrize("kind", ["diag", "scaled_perm", "hadamard4", "hadamard8"])
def test_fully_orthogonal_converges_in_one_sweep(kind):
    """Fig 1 right panel: mutually orthogonal hyperplanes -> exact after one pass
    (SPEC.md:351); Hadamard rows exercise the overlapping-category (atomic) path at thr > 0."""
    rng = np.random.default_rng(5)
    if kind == "diag":
        A = sp.diags(rng.uniform(0.5, 3, 30)).tocsr()
    elif kind == "scaled_perm":
        p = rng.permutation(30)
        A = sp.csr_matrix((rng.uniform(0.5, 3, 30), (np.arange(30), p)), shape=(30, 30))
    else:
        H = np.array([[1.0]])
        while H.shape[0] < int(kind[-1]):
            H = np.block([[H, H], [H, -H]])
        A = sp.csr_matrix(H)
    s = gen.from_csr(kind, A, 3)
    for thr in ([0.0, 0.5] if kind.startswith("hadamard") else [0.0]):
        pre = O.preprocess(s.m, s.indptr, s.indices, s.data, thr=thr)
        if kind.startswith("hadamard") and thr > 0:
            assert pre.nsteps == 1 and pre.overlap.tolist() == [1]
        x = O.run_sweeps(pre, s.f, 1)
        assert O.rse(x, s.x_star) < 1e-14


@pytest.mark.parametrize("theta_deg", [10, 45, 80])
def test_cos_theta_ratio(theta_deg):
    """Eq 4.12-4.13: per projection the error shrinks by cos(theta); per sweep
    (two projections) by cos^2(theta), within 1e-9."""
    t = math.radians(theta_deg)
    A = sp.csr_matrix(np.array([[1.0, 0.0], [math.cos(t), math.sin(t)]]))
    s = gen.from_csr("2x2", A, 9)
    pre = O.preprocess(2, s.indptr, s.indices, s.data)
    assert pre.nsteps == 2
    res = O.solve(2, s.indptr, s.indices, s.data, s.f, s.x_star, tol=1e-300, max_sweeps=6, keep_trace=True, pre=pre)
    tr = res.trace
    checked = 0
    for k in range(1, 5):
        if tr[k + 1] > 1e-6:
            assert abs(tr[k + 1] / tr[k] - math.cos(t) ** 2) < 1e-9
            checked += 1
    assert checked >= 1


@pytest.mark.parametrize("seed", range(8))
def test_monotone_error_every_step_and_lemma1_collapse(seed):
    """Eq 4.5-4.6: ||x - x*|| never increases across a block projection
    (slack 1e-12 ||x*||).  Lemma 1: for a category of pairwise
    orthogonal rows, the parallel row projections equal the block step x + A_tau^+ (f_tau - A_tau x)
    computed with numpy.linalg.pinv (Eq 1.3)."""
    rng = np.random.default_rng(seed)
    m = int(rng.integers(10, 40))
    s = gen.from_csr("rb", gen.random_banded(m, seed, half=int(rng.integers(1, 5))), seed)
    pre = O.preprocess(s.m, s.indptr, s.indices, s.data)
    f_t = O.permute_vector(s.f, pre.perm)
    xs_t = O.permute_vector(s.x_star, pre.perm)
    At = sp.csr_matrix((pre.data, pre.indices, pre.indptr), shape=(m, m)).toarray()
    errs = []

    def on_step(k, rows, xb, xa):
        errs.append((np.linalg.norm(xb - xs_t), np.linalg.norm(xa - xs_t)))
        xp = O.block_step_pinv(At[rows], f_t[rows], xb)
        np.testing.assert_allclose(xa, xp, rtol=0, atol=1e-12 * max(1.0, np.linalg.norm(xb)))

    x = np.zeros(m)
    for _ in range(3):
        O.sweep_rows_py(pre, f_t, x, on_step=on_step)
    slack = 1e-12 * np.linalg.norm(s.x_star)
    assert all(a <= b + slack for b, a in errs)


@pytest.mark.parametrize("seed", range(6))
def test_vectorised_equals_row_by_row_bitwise(seed):
    """Disjoint categories: the block form (SciPy mat-vecs) and the row form
    (Eq 1.2, both the pure-Python and the C restatement) give bitwise-identical iterates
    (SURVEY.md A.7)."""
    s = gen.make("lap2d5_32") if seed == 0 else gen.from_csr("rb", gen.random_banded(50, seed), seed)
    pre = O.preprocess(s.m, s.indptr, s.indices, s.data)
    f_t = O.permute_vector(s.f, pre.perm)
    xa, xb, xc = np.zeros(s.m), np.zeros(s.m), np.zeros(s.m)
    for _ in range(5):
        O.sweep_numpy(pre, f_t, xa)
        O.sweep_rows_py(pre, f_t, xb)
    O.sweep(pre, f_t, xc, 5)
    assert np.array_equal(xa, xb) and np.array_equal(xb, xc)


def test_one_row_category_is_eq12():
    """A singleton step applies exactly Eq 1.2: the pseudo-inverse of one row is
    a^T/||a||^2, so the step equals numpy.linalg.pinv's block step (Eq 1.3) on that row."""
    rng = np.random.default_rng(3)
    a = rng.standard_normal(6)
    A = sp.csr_matrix(np.vstack([a, np.eye(6)[1:]]))   # row 0 conflicts with all others
    pre = _pre_from_matrix(A, reorder=0)
    assert pre.cat_ptr.tolist() == [0, 5, 6] and pre.cat_rows.tolist() == [1, 2, 3, 4, 5, 0]
    f = rng.standard_normal(6)
    seen = []

    def on_step(k, rows, xb, xa):
        if rows.tolist() == [0]:
            seen.append(1)
            np.testing.assert_allclose(xa, O.block_step_pinv(a[None, :], f[:1], xb), rtol=0, atol=1e-14)

    O.sweep_rows_py(pre, f, rng.standard_normal(6), on_step=on_step)
    assert seen == [1]


@pytest.mark.parametrize("seed", range(10))
def test_dense_solve_agreement_relres(seed):
    """SPEC.md:473 (acceptance #1): iterate with the RELRES stop (no x* used) to 1e-12 and compare
    with a dense direct solve (numpy.linalg.solve) within 1e-5 relative; m <= 60."""
    rng = np.random.default_rng(seed)
    m = int(rng.integers(5, 61))
    A = gen.scramble(gen.random_banded(m, 200 + seed, half=int(rng.integers(1, 6))), 300 + seed)
    s = gen.from_csr("rb", A, seed)
    res = O.solve(m, s.indptr, s.indices, s.data, s.f, stop="relres", tol=1e-12, max_sweeps=200000)
    assert res.termination == O.TERM_CONVERGED
    xd = np.linalg.solve(A.toarray(), s.f)
    assert np.linalg.norm(res.x - xd) <= 1e-5 * np.linalg.norm(xd)


@pytest.mark.parametrize("seed", range(5))
def test_permutation_invariance(seed):
    """Eq 4.1 / SPEC.md:481: solving (A, f) and a pre-shuffled copy (P0 A P0^T,
    P0 f) gives solutions equal after alignment (1e-8 relative)."""
    A = gen.random_banded(40, 400 + seed, half=3)
    s = gen.from_csr("rb", A, seed)
    q = np.random.default_rng(seed).permutation(40)
    B = gen.canonical(A[q][:, q])
    r1 = O.solve(40, s.indptr, s.indices, s.data, s.f, s.x_star, tol=1e-12)
    r2 = O.solve(40, B.indptr, B.indices, B.data, s.f[q], s.x_star[q], tol=1e-12)
    assert np.linalg.norm(r1.x[q] - r2.x) <= 1e-8 * np.linalg.norm(r1.x)


def test_frame_invariance_of_error():
    """Eq 4.1: ||x_j - x*|| = ||x~_j - x~*|| for corresponding iterates."""
    s = gen.make("lap2d5_32")
    pre = O.preprocess(s.m, s.indptr, s.indices, s.data)
    f_t = O.permute_vector(s.f, pre.perm)
    x_t = O.sweep(pre, f_t, np.zeros(s.m), 7)
    x = O.unpermute_vector(x_t, pre.perm)
    assert abs(np.linalg.norm(x - s.x_star) - np.linalg.norm(x_t - O.permute_vector(s.x_star, pre.perm))) < 1e-13


# ------------------------------------------------------------------ O8 / O9
def test_rse_closed_forms():
    """SPEC.md:360-362."""
    xs = np.array([3.0, 4.0])
    assert O.rse(xs, xs) == 0.0
    assert O.rse(np.zeros(2), xs) == 1.0
    assert O.rse(np.array([3.0, 9.0]), xs) == 1.0


def _relres_pre(A, reorder):
    A = gen.canonical(sp.csr_matrix(A))
    return A, O.preprocess(A.shape[0], A.indptr, A.indices, A.data, reorder=reorder)


@pytest.mark.parametrize("reorder", [0, 1])
def test_relres_closed_forms(reorder):
    """RELRES = ||f - A x||_2 / ||f||_2 (the residual stop of SURVEY Z13, beside the RSE of
    PAPER.md:365), evaluated by the oracle in the RCM frame.  Pins, each failing a plausible
    slip: x = 0 gives exactly 1 (a missing normalisation gives ||f||); a hand-computed 2x2 value
    sqrt(5)/5 for A = [[2,1],[0,3]], f = (3,4), x = (0,1) (r = (2,1)), which a missing sqrt (0.2),
    a squared numerator (1.0), a missing ||f|| (sqrt 5) or a swapped operand (A^T x: r = (3,0),
    0.6) all miss; the exact solution gives 0."""
    A, pre = _relres_pre(np.array([[2.0, 1.0], [0.0, 3.0]]), reorder)
    f = np.array([3.0, 4.0])
    f_t = O.permute_vector(f, pre.perm)
    assert O.relres(pre, f_t, np.zeros(2)) == 1.0
    x = np.array([0.0, 1.0])
    v = O.relres(pre, f_t, O.permute_vector(x, pre.perm))
    assert abs(v - np.sqrt(5.0) / 5.0) <= 1e-16
    assert O.relres(pre, f_t, O.permute_vector(np.array([5.0 / 6.0, 4.0 / 3.0]), pre.perm)) <= 1e-15
    # the user-frame residual norm of the same point
    assert abs(O.residual_norm(2, A.indptr, A.indices, A.data, f, x) - np.sqrt(5.0)) <= 1e-15


@pytest.mark.parametrize("seed", range(3))
def test_relres_frame_invariant_and_scale_free(seed):
    """RELRES does not depend on the frame (P^T P = E, Eq 4.1) and is invariant under
    f -> c f, x -> c x (homogeneous of degree 0): a reordering of the sum or a missing ||f||
    normalisation breaks one of the two."""
    rng = np.random.default_rng(seed)
    A = gen.scramble(gen.random_banded(40, 500 + seed, half=3), 600 + seed)
    A = gen.canonical(A)
    f = rng.standard_normal(40)
    x = rng.standard_normal(40)
    pre0 = O.preprocess(40, A.indptr, A.indices, A.data, reorder=0)
    pre1 = O.preprocess(40, A.indptr, A.indices, A.data, reorder=1)
    v0 = O.relres(pre0, f, x)
    v1 = O.relres(pre1, O.permute_vector(f, pre1.perm), O.permute_vector(x, pre1.perm))
    ref = np.linalg.norm(f - A @ x) / np.linalg.norm(f)
    assert abs(v0 - ref) <= 1e-13 * ref and abs(v1 - ref) <= 1e-13 * ref
    assert abs(O.relres(pre0, 8.0 * f, 8.0 * x) - v0) <= 1e-15 * v0  # (8: exact power-of-two scaling)


def test_stop_is_strict_less_than():
    """PAPER.md:364 'less than 1e-6': value == tol does not stop."""
    s = gen.make("lap2d5_32")
    r = O.solve(s.m, s.indptr, s.indices, s.data, s.f, s.x_star, tol=0.0, max_sweeps=5, keep_trace=True)
    assert r.termination == O.TERM_MAX_SWEEPS and r.sweeps == 5
    v1 = r.trace[0]
    assert O.solve(s.m, s.indptr, s.indices, s.data, s.f, s.x_star, tol=v1, max_sweeps=5).sweeps == 2
    assert O.solve(s.m, s.indptr, s.indices, s.data, s.f, s.x_star, tol=np.nextafter(v1, 1.0), max_sweeps=5).sweeps == 1


def test_nonfinite_termination():
    A = sp.csr_matrix(np.array([[1.0, 0.5], [0.5, 1.0]]))
    s = gen.from_csr("nf", A, 1)
    f = s.f.copy(); f[0] = np.inf
    r = O.solve(2, s.indptr, s.indices, s.data, f, s.x_star, tol=1e-6, max_sweeps=10)
    assert r.termination == O.TERM_NONFINITE and r.sweeps == 1


def test_permutation_round_trip():
    """inverse(forward(v)) = v."""
    rng = np.random.default_rng(0)
    v = rng.standard_normal(50)
    p = rng.permutation(50).astype(np.int32)
    assert np.array_equal(O.unpermute_vector(O.permute_vector(v, p), p), v)
    assert np.array_equal(O.permute_vector(v, p), v[p])


def test_thr_positive_partition_pins():
    """PAPER.md:220 with the absolute cosine: rows sharing columns but with
    |cos| < thr are treated as orthogonal (same category, overlapping -> simultaneous update);
    the mex certificate holds for the thresholded conflict relation."""
    A = sp.csr_matrix(np.array([[1.0, 1.0, 0.0], [1.0, -1.0, 0.1], [0.0, 0.1, 1.0]]))
    pre = _pre_from_matrix(A, thr=0.2, reorder=0)
    # rows 0,1: cos = 0/(sqrt2*sqrt2.01) = 0 < 0.2 -> no conflict; rows 1,2: dot=-0.1+0.1=0 -> none;
    # rows 0,2: dot 0.1/(sqrt2*sqrt1.01) = 0.0704 < 0.2 -> none: one category
    assert pre.color.tolist() == [0, 0, 0] and pre.overlap.tolist() == [1]
    pre = _pre_from_matrix(A, thr=0.05, reorder=0)
    # rows 0,2 now conflict (0.0704 >= 0.05)
    assert pre.color.tolist() == [0, 0, 1]
    assert pre.color.tolist() == O.first_fit_py(3, pre.indptr, pre.indices, pre.data, pre.nrm2, 0.05).tolist()


# ------------------------------------------------------------------ NEXT-4 residual-ordered sweep (reading R-G)
def test_residual_order_ties_and_permutation():
    """Decreasing score, ties by ascending step index; always a permutation of the steps."""
    assert O.residual_order([1.0, 3.0, 3.0, 2.0]).tolist() == [1, 2, 3, 0]
    sc = np.random.default_rng(3).random(40)
    assert sorted(O.residual_order(sc).tolist()) == list(range(40))


def test_two_level_sum_grouping():
    """Chunks summed left to right, then the chunk sums: 1 + 1e-16 + 1e-16 + 1e-16 in chunks of 2
    is (1) + (2e-16) = 1 + 2^-52 (rounded up), while the plain left-to-right sum stays 1."""
    v = [1.0, 1e-16, 1e-16, 1e-16]
    assert O.seq_sum(v) == 1.0
    assert O.two_level_sum(v, chunk=2) == 1.0 + 2.0 ** -52
    assert O.two_level_sum([0.5, 0.25, 0.125, 1.0], chunk=2) == 1.875


def test_step_scores_hand_value():
    """rho_K = ||f_K - A_K x||^2 / ||A_K||_F^2: A = [[1,1],[1,-1]] (two one-row steps at thr = 0),
    f = (3,-1), x = 0: rho = (9/2, 1/2) -> step 0 first; after x = (1.5, 1.5): rho = (0, 1/2)."""
    A = sp.csr_matrix(np.array([[1.0, 1.0], [1.0, -1.0]]))
    pre = _pre_from_matrix(A, reorder=0)
    f = np.array([3.0, -1.0])
    assert O.step_scores(pre, f, np.zeros(2)).tolist() == [4.5, 0.5]
    assert O.step_scores(pre, f, np.array([1.5, 1.5])).tolist() == [0.0, 0.5]


def test_ordered_steps_in_cyclic_order_equal_the_sweep():
    """Applying the steps one at a time in schedule order is the O7 sweep, bitwise (the ordered
    sweep differs only in the order)."""
    s = gen.make("lap2d5_32")
    pre = O.preprocess(s.m, s.indptr, s.indices, s.data)
    f_t = O.permute_vector(s.f, pre.perm)
    x1 = O.sweep(pre, f_t, np.zeros(s.m), 1)
    x2 = np.zeros(s.m)
    scratch = np.empty(s.m)
    for k in range(pre.nsteps):
        O.core._apply_step(pre, k, f_t, x2, scratch)
    assert np.array_equal(x1, x2)


@pytest.mark.parametrize("seed", range(3))
def test_ordered_sweep_monotone_and_converges(seed):
    """Any order of exact projections keeps Eq 4.6 (error never increases) and the ordered
    iteration reaches the dense solve."""
    A = gen.scramble(gen.random_banded(40, 900 + seed, half=3), 950 + seed)
    s = gen.from_csr("rb", A, seed)
    pre = O.preprocess(40, s.indptr, s.indices, s.data)
    f_t, xs_t = O.permute_vector(s.f, pre.perm), O.permute_vector(s.x_star, pre.perm)
    x = np.zeros(40)
    prev = np.linalg.norm(xs_t)
    for _ in range(30):
        O.sweep_ordered(pre, f_t, x, 1)
        e = np.linalg.norm(x - xs_t)
        assert e <= prev + 1e-12 * np.linalg.norm(xs_t)
        prev = e
    xo, sweeps, term, v = O.solve_ordered(pre, s.f, s.x_star, 1e-10, 100000)
    assert term == O.TERM_CONVERGED
    assert np.linalg.norm(xo - np.linalg.solve(A.toarray(), s.f)) <= 1e-8 * np.linalg.norm(s.x_star)
