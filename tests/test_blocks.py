"""The paper-literal k-block POBK (SURVEY §8(f) NEXT-2, NEXT-4 diagnostics): the product's host
layout (pobk_blocks_preprocess, device = -1) against the oracle (oracle/blocks.py) -- block
boundaries, Oclass pairs and Nclass bit-exact, the cosine table and zn/nn to rounding -- and, on
the GPU, K5's iterates and stop sweeps against the oracle's Alg 5."""
import numpy as np
import pytest

import oracle as O
from oracle import blocks as OB
from workloads import gen


@pytest.fixture(scope="module")
def pk():
    import paper_2401_00672_b200 as pk
    return pk


CASES = [("lap2d5_32", None, 7, 0.05), ("lap2d5_32", None, 19, 0.0), ("randband_20k", 3000, 10, 0.3),
         ("lap3d7_64", 12, 13, 0.05), ("geoknn_1m", 5000, 5, 0.2)]


@pytest.mark.parametrize("name,n,k,thr", CASES)
def test_host_layout_matches_oracle(pk, name, n, k, thr):
    s = gen.make(name, n=n) if n else gen.make(name)
    bp = OB.block_preprocess(s.m, s.indptr, s.indices, s.data, k=k, thr=thr)
    plan = pk.Plan.from_system_blocks(s, k=k, thr=thr, device=-1)
    info = plan.blocks_info()
    assert np.array_equal(plan.perm(), bp.pre.perm)
    assert info["k"] == k and np.array_equal(info["ptr"], bp.ptr)
    np.testing.assert_allclose(info["C"], bp.C, rtol=1e-13, atol=1e-15)
    assert info["pairs"] == bp.pairs and info["nclass"] == bp.nclass
    assert abs(info["zn"] - bp.zn) < 1e-15 and abs(info["nn"] - bp.nn) < 1e-12
    colour, cat_ptr, cat_rows = plan.partition()
    assert np.array_equal(cat_ptr, bp.ptr) and np.array_equal(cat_rows, np.arange(s.m))
    plan.close()


def test_bad_k_is_an_error(pk):
    s = gen.make("lap2d5_32")
    with pytest.raises(pk.PobkError):
        pk.Plan.from_system_blocks(s, k=0, thr=0.05, device=-1)
    with pytest.raises(pk.PobkError):
        pk.Plan.from_system_blocks(s, k=s.m + 1, thr=0.05, device=-1)


def _dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


@pytest.mark.gpu
@pytest.mark.parametrize("name,n,k,thr,tol", [("lap2d5_32", None, 7, 0.05, 0.1), ("lap2d5_32", None, 2, 0.05, 0.1),
                                              ("randband_20k", 3000, 10, 0.3, 1e-6), ("lap3d7_64", 12, 13, 0.05, 0.1)])
def test_k5_iterates_and_stop_parity(pk, name, n, k, thr, tol):
    """K5 (Gram-inverse block projections) against the oracle's lstsq block steps: iterates within
    1e-9 relative after a fixed count, and the RSE stop sweep +-1."""
    import torch
    s = gen.make(name, n=n) if n else gen.make(name)
    bp = OB.block_preprocess(s.m, s.indptr, s.indices, s.data, k=k, thr=thr)
    plan = pk.Plan.from_system_blocks(s, k=k, thr=thr)
    assert plan.layout_stats()["kernel"] == "blocks"
    x = _dev(torch, np.zeros(s.m))
    rep = plan.solve(_dev(torch, s.f), x, _dev(torch, s.x_star), max_sweeps=6, stop="none")
    assert rep.sweeps == 6 and rep.kernel == 5
    ref = O.unpermute_vector(OB.block_sweep(bp, O.permute_vector(s.f, bp.pre.perm), np.zeros(s.m), 6), bp.pre.perm)
    assert np.linalg.norm(x.cpu().numpy() - ref) <= 1e-9 * np.linalg.norm(ref)
    xr, sweeps, term, v = OB.block_solve(bp, s.f, s.x_star, tol=tol, max_sweeps=3000)
    x = _dev(torch, np.zeros(s.m))
    rep = plan.solve(_dev(torch, s.f), x, _dev(torch, s.x_star), tol=tol, max_sweeps=3000)
    assert rep.termination == term and abs(rep.sweeps - sweeps) <= 1, (rep.sweeps, sweeps)
