"""Host-side parity (-m "not gpu"): libpobk.so's native preprocessing (host-only plans, device=-1)
against the oracle, bit-exact on the integer work (perm, colour, schedule), and the C ABI surface.
SURVEY.md §4 T2; DESIGN.md §6."""
import ctypes
import os
import re

import numpy as np
import pytest
import scipy.sparse as sp

import oracle as O
from workloads import gen

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def pk():
    import paper_2401_00672_b200 as pk
    return pk


def test_library_exports_every_declared_symbol(pk):
    """Every function include/pobk.h declares is exported by libpobk.so with that name."""
    hdr = open(os.path.join(ROOT, "include", "pobk.h")).read()
    declared = set(re.findall(r"^\s*(?:pobk_status|void|const char\*|int32_t)\s+(pobk_\w+)\s*\(", hdr, re.M))
    assert len(declared) >= 15
    lib = ctypes.CDLL(pk._lib.LIB_PATH)
    for name in sorted(declared):
        assert hasattr(lib, name), name
    assert set(pk._lib.SIGNATURES) == declared
    assert lib.pobk_abi_version() == 3


def _compare(pk, m, indptr, indices, data, thr=0.0, reorder=1):
    pre = O.preprocess(m, indptr, indices, data, thr=thr, reorder=reorder)
    plan = pk.Plan.from_csr(m, indptr, indices, data, thr=thr, reorder=reorder, device=-1)
    colour, cat_ptr, cat_rows = plan.partition()
    assert np.array_equal(plan.perm(), pre.perm)
    assert np.array_equal(colour, pre.color)
    assert np.array_equal(cat_ptr, pre.cat_ptr)
    assert np.array_equal(cat_rows, pre.cat_rows)
    assert plan.n_oclass == pre.n_oclass and plan.nsteps == pre.nsteps
    assert plan.bw_before == pre.bw_before and plan.bw_after == pre.bw_after
    plan.close()
    return pre


@pytest.mark.parametrize("seed", range(200))
def test_random_graphs_bit_exact(pk, seed):
    """~200 random tiny graphs: disconnected, isolated vertices, dense, sparse."""
    rng = np.random.default_rng(1000 + seed)
    m = int(rng.integers(1, 51))
    kind = seed % 4
    if kind == 0:
        A = gen.random_pattern_graph(m, 1000 + seed, p=float(rng.choice([0.01, 0.05, 0.2, 0.6])))
    elif kind == 1:
        A = gen.random_banded(m, 1000 + seed, half=int(rng.integers(1, 6)))
        A = gen.scramble(A, seed)
    elif kind == 2:   # nonsymmetric pattern
        D = (rng.random((m, m)) < 0.08) * rng.uniform(-1, 1, (m, m)) + np.eye(m) * 3
        A = gen.canonical(sp.csr_matrix(D))
    else:             # grids and paths with degree ties, scrambled
        n = int(rng.integers(1, 8))
        A = gen.scramble(gen.lap2d5(n) if seed % 8 == 3 else gen.box9(n), seed)
    A = gen.canonical(A)
    _compare(pk, A.shape[0], A.indptr.astype(np.int64), A.indices.astype(np.int32), A.data)


@pytest.mark.parametrize("thr", [0.02, 0.1, 0.3])
@pytest.mark.parametrize("seed", range(10))
def test_thr_positive_bit_exact(pk, thr, seed):
    """thr > 0: float-decided conflicts (DESIGN.md §3 P2) still bit-exact with the oracle."""
    A = gen.scramble(gen.random_banded(40, 77 + seed, half=4, density=0.8), seed)
    _compare(pk, 40, A.indptr.astype(np.int64), A.indices.astype(np.int32), A.data, thr=thr)


def test_reorder_off_identity(pk):
    A = gen.scramble(gen.lap2d5(6), 3)
    pre = _compare(pk, 36, A.indptr.astype(np.int64), A.indices.astype(np.int32), A.data, reorder=0)
    assert np.array_equal(pre.perm, np.arange(36))


@pytest.mark.parametrize("name,n", [("lap2d5_32", None), ("randband_20k", None), ("lap3d7_64", 24),
                                    ("geoknn_1m", 20000), ("batch9pt_1024", 64)])
def test_configs_bit_exact(pk, name, n):
    """BASELINE configs (configs 3-5 at reduced size here; full sizes run in the GPU suite)."""
    s = gen.make(name, n=n) if n else gen.make(name)
    _compare(pk, s.m, s.indptr, s.indices, s.data)


def test_explicit_zero_and_errors(pk):
    m = 3
    ip = np.array([0, 2, 3, 5], np.int64)
    ix = np.array([0, 1, 1, 0, 2], np.int32)
    v = np.array([1.0, 0.0, 2.0, 1.0, 3.0])
    plan = pk.Plan.from_csr(m, ip, ix, v, device=-1)
    assert plan.nnz == 4   # stored zero dropped
    with pytest.raises(pk.PobkError) as e:
        pk.Plan.from_csr(m, ip, np.array([1, 0, 1, 0, 2], np.int32), v, device=-1)
    assert e.value.code == 2 and "row 0" in str(e.value)
    with pytest.raises(pk.PobkError) as e:
        pk.Plan.from_csr(m, ip, ix, np.array([1.0, 0.0, 0.0, 1.0, 3.0]), device=-1)
    assert e.value.code == 3 and "row 1" in str(e.value)
    with pytest.raises(pk.PobkError) as e:
        pk.Plan.from_csr(m, ip, np.array([0, 1, 1, 0, 3], np.int32), v, device=-1)
    assert e.value.code == 2
    with pytest.raises(pk.PobkError) as e:
        pk.Plan.from_csr(m, np.array([0, 2, 1, 5]), ix, v, device=-1)
    assert e.value.code == 2
    with pytest.raises(pk.PobkError) as e:
        pk.Plan.from_csr(m, ip, ix, v, thr=1.5, device=-1)
    assert e.value.code == 1


def test_host_plan_refuses_solve(pk):
    A = gen.lap2d5(4)
    plan = pk.Plan.from_csr(16, A.indptr, A.indices, A.data, device=-1)
    f = np.ones(16)
    x = np.zeros(16)
    with pytest.raises(pk.PobkError) as e:
        plan.solve_host(f, x, f, stream=0)
    assert e.value.code == 7


def test_gershgorin_guard(pk):
    """NEXT-1 guard: a thr so large that a category's overlaps can expand the error is refused."""
    A = gen.lap2d5(8)
    s = gen.from_csr("g", A, 1)
    with pytest.raises(pk.PobkError) as e:
        pk.Plan.from_csr(s.m, s.indptr, s.indices, s.data, thr=0.45, guard=1, device=-1)
    assert e.value.code == 4
    pk.Plan.from_csr(s.m, s.indptr, s.indices, s.data, thr=0.45, guard=0, device=-1).close()
