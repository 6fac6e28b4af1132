"""GPU parity of the K2 wavefront kernel's specific paths, against the oracle
on the same seeded inputs: rows longer than the register cache (tail entries on interior and
boundary slices), many small tiles (mailbox hand-offs on most rows), a nonzero x0 (mailbox
seeding), repeated solves on one plan (mailbox re-initialisation) and the RSE stop evaluated
from owned columns / wrap slots.  thr = 0 iterates must be bitwise the oracle's (common.cuh)."""
import numpy as np
import pytest

import oracle as O
from workloads import gen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch

    import paper_2401_00672_b200 as pk
    torch.cuda.set_device(0)
    return pk, torch


def _dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def _wave(env, s, **kw):
    pk, _ = env
    plan = pk.Plan.from_system(s, kernel="wavefront", **kw)
    st = plan.layout_stats()
    assert st["kernel"] == "wavefront" and st["ntiles"] > 1, st
    return plan


def _sweeps(env, plan, s, n, x0=None):
    _, torch = env
    x = _dev(torch, np.zeros(s.m) if x0 is None else x0)
    rep = plan.solve(_dev(torch, s.f), x, _dev(torch, s.x_star), max_sweeps=n, stop="none")
    assert rep.sweeps == n
    return x.cpu().numpy()


def test_long_rows_tails(env):
    """geo-kNN with k = 30: rows of ~31-50 entries, past the 24-entry register cache on both
    interior and boundary slices."""
    A = gen.scramble(gen.geoknn(40000, 11, k=30), 12)
    s = gen.from_csr("geoknn40k_k30", A, 13)
    assert np.diff(s.indptr).max() > 40
    pre = O.preprocess(s.m, s.indptr, s.indices, s.data)
    plan = _wave(env, s)
    x = _sweeps(env, plan, s, 6)
    assert np.array_equal(x, O.run_sweeps(pre, s.f, 6))


def test_many_small_tiles_nonzero_x0_repeat(env):
    """3-D 7-point, 24^3, ~100 rows per tile: most rows on tile boundaries (mailboxes), a random
    x0 (seeds the mailboxes), and a second solve on the same plan (mailboxes re-armed)."""
    s = gen.make("lap3d7_64", n=24)
    pre = O.preprocess(s.m, s.indptr, s.indices, s.data)
    plan = _wave(env, s, tile_rows=120)
    x0 = np.random.default_rng(5).standard_normal(s.m)
    ref = O.run_sweeps(pre, s.f, 9, x0=x0)
    x1 = _sweeps(env, plan, s, 9, x0=x0)
    assert np.array_equal(x1, ref)
    x2 = _sweeps(env, plan, s, 9, x0=x0)
    assert np.array_equal(x2, ref)


@pytest.mark.parametrize("tol", [1e-1, 3e-2])
def test_rse_stop_parity(env, tol):
    """RSE stop evaluated by K2 from owned columns and wrap slots: same
    stop sweep +-1 and the same value to 1e-9 as the oracle."""
    pk, torch = env
    s = gen.make("geoknn_1m", n=60000)
    ref = O.solve(s.m, s.indptr, s.indices, s.data, s.f, s.x_star, tol=tol)
    plan = _wave(env, s)
    x = _dev(torch, np.zeros(s.m))
    rep = plan.solve(_dev(torch, s.f), x, _dev(torch, s.x_star), tol=tol)
    assert rep.termination == ref.termination
    assert abs(rep.sweeps - ref.sweeps) <= 1, (rep.sweeps, ref.sweeps)
    assert abs(rep.final_value - ref.value) <= 1e-9 * ref.value
    if rep.sweeps == ref.sweeps:
        pre = O.preprocess(s.m, s.indptr, s.indices, s.data)
        assert np.array_equal(x.cpu().numpy(), O.run_sweeps(pre, s.f, rep.sweeps))
