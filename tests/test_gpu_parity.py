"""GPU parity (-m gpu): the CUDA path, called through the C ABI, against the oracle on the same
seeded inputs.

Bars (BASELINE.json north_star): integer work bit-exact; fp64 iterates within
||x_gpu - x_oracle|| / ||x_oracle|| <= 1e-9 after a fixed sweep count; the same stop sweep +-1.
thr = 0 iterates are additionally bitwise identical across kernel families and repeat runs."""
import numpy as np
import pytest

import oracle as O
from workloads import gen

pytestmark = pytest.mark.gpu

REL = 1e-9


@pytest.fixture(scope="module")
def env():
    import torch

    import paper_2401_00672_b200 as pk
    torch.cuda.set_device(0)
    return pk, torch


def _dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def _run(env, s, nsweeps, kernel="auto", thr=0.0, plan=None, pre=None, x0=None):
    pk, torch = env
    plan = plan or pk.Plan.from_system(s, kernel=kernel, thr=thr)
    x = _dev(torch, np.zeros(s.m) if x0 is None else x0)
    rep = plan.solve(_dev(torch, s.f), x, _dev(torch, s.x_star), max_sweeps=nsweeps, stop="none")
    assert rep.sweeps == nsweeps
    return plan, x.cpu().numpy(), rep


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


SMALL = [("lap2d5_32", None), ("randband_20k", None), ("lap3d7_64", 20), ("geoknn_1m", 30000),
         ("batch9pt_1024", 100)]


@pytest.mark.parametrize("kernel", ["launch", "smem", "cluster", "wavefront", "auto"])
@pytest.mark.parametrize("name,n", SMALL)
def test_fixed_sweeps_parity(env, name, n, kernel):
    s = gen.make(name, n=n) if n else gen.make(name)
    pre = O.preprocess(s.m, s.indptr, s.indices, s.data)
    pk, _ = env
    try:
        plan = pk.Plan.from_system(s, kernel=kernel)
    except pk.PobkError as e:
        if kernel in ("smem", "cluster", "wavefront") and e.code == 1:
            pytest.skip(f"{kernel} not applicable: {e}")
        raise
    assert np.array_equal(plan.perm(), pre.perm)
    nf = 25
    _, x, rep = _run(env, s, nf, plan=plan)
    ref = O.run_sweeps(pre, s.f, nf)
    assert _rel(x, ref) <= REL, (rep.as_dict(), _rel(x, ref))
    assert np.array_equal(x, ref), "thr = 0 iterates are bitwise the oracle's (common.cuh contract)"


@pytest.mark.parametrize("name,n", [("lap2d5_32", None), ("lap3d7_64", 11), ("randband_20k", 3000),
                                    ("geoknn_1m", 120000)])
def test_kernel_families_bitwise_equal(env, name, n):
    """Same per-row arithmetic contract (common.cuh) -> bitwise-identical iterates (T3), and -- since
    the contract is the oracle's own operation order -- bitwise equal to the oracle (thr = 0)."""
    pk, _ = env
    s = gen.make(name, n=n) if n else gen.make(name)
    outs = {}
    for kernel in ("launch", "smem", "cluster", "wavefront"):
        try:
            _, outs[kernel], _ = _run(env, s, 12, kernel=kernel)
        except pk.PobkError:
            continue
    assert len(outs) >= 2
    vals = list(outs.values())
    for v in vals[1:]:
        assert np.array_equal(v, vals[0]), list(outs)
    pre = O.preprocess(s.m, s.indptr, s.indices, s.data)
    assert np.array_equal(vals[0], O.run_sweeps(pre, s.f, 12))


def test_repeatable_bitwise(env):
    s = gen.make("lap3d7_64", n=24)
    plan, x1, _ = _run(env, s, 30)
    _, x2, _ = _run(env, s, 30, plan=plan)
    assert np.array_equal(x1, x2)


def test_stop_sweep_config1_tol_1e6(env):
    """BASELINE config 1 to the paper's tolerance (RSE < 1e-6): same stop sweep +-1."""
    pk, torch = env
    s = gen.make("lap2d5_32")
    ref = O.solve(s.m, s.indptr, s.indices, s.data, s.f, s.x_star, tol=1e-6)
    assert ref.termination == O.TERM_CONVERGED
    plan = pk.Plan.from_system(s)
    x = _dev(torch, np.zeros(s.m))
    rep = plan.solve(_dev(torch, s.f), x, _dev(torch, s.x_star), tol=1e-6)
    assert rep.termination == 0
    assert abs(rep.sweeps - ref.sweeps) <= 1, (rep.sweeps, ref.sweeps)
    assert O.rse(x.cpu().numpy(), s.x_star) < 1e-6


@pytest.mark.parametrize("name,n,tol", [("randband_20k", None, 1e-6), ("lap3d7_64", None, 1e-1),
                                        ("lap2d5_32", None, 1e-3)])
@pytest.mark.parametrize("kernel", ["auto", "launch"])
def test_stop_sweep_parity(env, name, n, tol, kernel):
    pk, torch = env
    s = gen.make(name, n=n) if n else gen.make(name)
    ref = O.solve(s.m, s.indptr, s.indices, s.data, s.f, s.x_star, tol=tol)
    plan = pk.Plan.from_system(s, kernel=kernel)
    x = _dev(torch, np.zeros(s.m))
    rep = plan.solve(_dev(torch, s.f), x, _dev(torch, s.x_star), tol=tol)
    assert rep.termination == ref.termination
    assert abs(rep.sweeps - ref.sweeps) <= 1, (rep.sweeps, ref.sweeps)
    assert abs(rep.final_value - ref.value) <= 1e-9 * ref.value + 1e-15


def test_relres_stop_and_residual_norm(env):
    pk, torch = env
    s = gen.make("randband_20k")
    pre = O.preprocess(s.m, s.indptr, s.indices, s.data)
    ref = O.solve(s.m, s.indptr, s.indices, s.data, s.f, stop="relres", tol=1e-8, pre=pre)
    for kernel in ("launch", "auto"):
        plan = pk.Plan.from_system(s, kernel=kernel)
        x = _dev(torch, np.zeros(s.m))
        f = _dev(torch, s.f)
        rep = plan.solve(f, x, None, tol=1e-8, stop="relres")
        assert abs(rep.sweeps - ref.sweeps) <= 1
        r = plan.residual_norm(f, x)
        r_ref = O.residual_norm(s.m, s.indptr, s.indices, s.data, s.f, x.cpu().numpy())
        assert abs(r - r_ref) <= 1e-9 * r_ref
        # row-sharded residual (C2): shards sum to the whole
        h = s.m // 3
        parts = [plan.residual_sumsq_rows(a, b, f, x) for a, b in ((0, h), (h, 2 * h), (2 * h, s.m))]
        assert abs(np.sqrt(sum(parts)) - r) <= 1e-12 * r


@pytest.mark.parametrize("thr", [0.05, 0.12])
def test_thr_positive_parity(env, thr, monkeypatch):
    """Overlapping categories (a3'): every alpha of the step at the same x~, then the
    scatter as one ordered fold per column (the step's contributions in ascending row order, each
    product and sum rounded -- the oracle's rows-then-entries order): bitwise the oracle's
    iterates on K1 and K3.  The fp64-atomic scatter (POBK_THR_ATOMIC=1, order nondeterministic)
    stays within 1e-9."""
    pk, torch = env
    s = gen.make("lap2d5_32")
    pre = O.preprocess(s.m, s.indptr, s.indices, s.data, thr=thr)
    assert pre.overlap.any()
    ref = O.run_sweeps(pre, s.f, 20)
    for kernel in ("launch", "smem"):
        plan = pk.Plan.from_system(s, thr=thr, kernel=kernel)
        colour, _, cat_rows = plan.partition()
        assert np.array_equal(colour, pre.color) and np.array_equal(cat_rows, pre.cat_rows)
        _, x, _ = _run(env, s, 20, plan=plan)
        assert np.array_equal(x, ref), kernel
    monkeypatch.setenv("POBK_THR_ATOMIC", "1")
    for kernel in ("launch", "smem"):
        plan = pk.Plan.from_system(s, thr=thr, kernel=kernel)  # (K1 captures its graph with the atomic scatter)
        _, x, _ = _run(env, s, 20, plan=plan)
        assert _rel(x, ref) <= REL, kernel


@pytest.mark.parametrize("kind", ["hadamard8", "diag"])
def test_fully_orthogonal_one_sweep(env, kind):
    pk, torch = env
    if kind == "diag":
        import scipy.sparse as sp
        A = sp.diags(np.linspace(0.5, 2.0, 4000)).tocsr()
        s = gen.from_csr(kind, A, 4)
        thr = 0.0
    else:
        H = np.array([[1.0]])
        while H.shape[0] < 8:
            H = np.block([[H, H], [H, -H]])
        import scipy.sparse as sp
        s = gen.from_csr(kind, sp.csr_matrix(H), 5)
        thr = 0.5
    plan = pk.Plan.from_system(s, thr=thr)
    x = _dev(torch, np.zeros(s.m))
    rep = plan.solve(_dev(torch, s.f), x, _dev(torch, s.x_star), tol=1e-12)
    assert rep.sweeps == 1 and rep.termination == 0


def test_edge_cases(env):
    pk, torch = env
    import scipy.sparse as sp
    # m = 1
    s = gen.from_csr("one", sp.csr_matrix(np.array([[2.0]])), 1)
    plan = pk.Plan.from_system(s)
    x = _dev(torch, np.zeros(1))
    rep = plan.solve(_dev(torch, s.f), x, _dev(torch, s.x_star), tol=1e-12)
    assert rep.sweeps == 1 and abs(x.item() - s.x_star[0]) < 1e-15
    # max_sweeps = 0 leaves x0
    s = gen.make("lap2d5_32")
    plan = pk.Plan.from_system(s)
    x0 = np.arange(s.m, dtype=np.float64)
    x = _dev(torch, x0)
    rep = plan.solve(_dev(torch, s.f), x, _dev(torch, s.x_star), max_sweeps=0)
    assert rep.sweeps == 0 and np.array_equal(x.cpu().numpy(), x0)
    # all-singleton Nclass (star: every pair of rows overlaps) and a nonzero x0 (resume)
    star = sp.lil_matrix((60, 60))
    star[0, :] = 1.0
    star[:, 0] = 1.0
    star.setdiag(5.0)
    s = gen.from_csr("star", star.tocsr(), 2)
    pre = O.preprocess(s.m, s.indptr, s.indices, s.data)
    assert pre.n_oclass <= 1
    x0 = np.random.default_rng(0).standard_normal(s.m)
    for kernel in ("launch", "smem"):
        _, x, _ = _run(env, s, 7, kernel=kernel, x0=x0)
        assert _rel(x, O.run_sweeps(pre, s.f, 7, x0=x0)) <= REL
    # argument errors: the RSE stop needs x*
    plan = pk.Plan.from_system(s)
    with pytest.raises(pk.PobkError):
        plan.solve(_dev(torch, s.f), _dev(torch, np.zeros(s.m)), None, stop="rse")


def test_solve_host_matches_device(env):
    pk, torch = env
    s = gen.make("randband_20k")
    plan = pk.Plan.from_system(s)
    x = _dev(torch, np.zeros(s.m))
    r1 = plan.solve(_dev(torch, s.f), x, _dev(torch, s.x_star), tol=1e-6)
    xh = np.zeros(s.m)
    r2 = plan.solve_host(s.f.copy(), xh, s.x_star.copy(), tol=1e-6)
    assert r1.sweeps == r2.sweeps and np.array_equal(xh, x.cpu().numpy())


def test_batch_equals_single(env):
    """T5: a system's iterates are bitwise the same alone or inside a batch."""
    pk, torch = env
    systems = [gen.make("batch9pt_1024", b, n=48) for b in range(3)]
    plans = [pk.Plan.from_system(s) for s in systems]
    xs = [_dev(torch, np.zeros(s.m)) for s in systems]
    reps = pk.solve_batch(plans, [_dev(torch, s.f) for s in systems], xs, [_dev(torch, s.x_star) for s in systems],
                          tol=1e-3)
    for s, p, xb, r in zip(systems, plans, xs, reps):
        x = _dev(torch, np.zeros(s.m))
        r1 = p.solve(_dev(torch, s.f), x, _dev(torch, s.x_star), tol=1e-3)
        assert r1.sweeps == r.sweeps and np.array_equal(x.cpu().numpy(), xb.cpu().numpy())


@pytest.mark.parametrize("nb", [2, 5])
def test_batch_lanes_equal_single(env, nb):
    """Concurrent lanes (pobk_solve_batch with half-GPU K2 tilings): every system's stop sweep,
    final RSE and iterates are bitwise those of its own back-to-back solve, and of the oracle's
    sweeps (config-5 generator at m = 160^2, odd and even batch sizes)."""
    pk, torch = env
    systems = [gen.make("batch9pt_1024", b, n=160) for b in range(nb)]
    tr = pk.half_gpu_tile_rows(systems[0].m)
    plans = [pk.Plan.from_system(s, kernel="wavefront", tile_rows=tr) for s in systems]
    assert all(2 * p.layout_stats()["ntiles"] <= torch.cuda.get_device_properties(0).multi_processor_count for p in plans)
    xs = [_dev(torch, np.zeros(s.m)) for s in systems]
    reps = pk.solve_batch(plans, [_dev(torch, s.f) for s in systems], xs, [_dev(torch, s.x_star) for s in systems],
                          tol=0.2)
    for s, p, xb, r in zip(systems, plans, xs, reps):
        x = _dev(torch, np.zeros(s.m))
        r1 = p.solve(_dev(torch, s.f), x, _dev(torch, s.x_star), tol=0.2)
        assert r1.sweeps == r.sweeps and r1.final_value == r.final_value
        assert np.array_equal(x.cpu().numpy(), xb.cpu().numpy())
    s0 = systems[0]
    pre = O.preprocess(s0.m, s0.indptr, s0.indices, s0.data)
    assert np.array_equal(xs[0].cpu().numpy(), O.run_sweeps(pre, s0.f, reps[0].sweeps))


# ---------------------------------------------------------------- full BASELINE sizes
@pytest.mark.slow
def test_config3_full_parity(env):
    s = gen.make("lap3d7_64")
    pre = O.preprocess(s.m, s.indptr, s.indices, s.data)
    plan, x, _ = _run(env, s, 100)
    assert np.array_equal(plan.perm(), pre.perm)
    assert np.array_equal(plan.partition()[0], pre.color)
    assert _rel(x, O.run_sweeps(pre, s.f, 100)) <= REL


@pytest.mark.slow
def test_config4_full_parity(env):
    """geoknn_1m at full size, in the bench's launch configuration: bit-exact perm/partition and
    iterates within 1e-9 after N_fix = 100 sweeps."""
    s = gen.make("geoknn_1m")
    pre = O.preprocess(s.m, s.indptr, s.indices, s.data)
    plan, x, rep = _run(env, s, 100)
    colour, cat_ptr, cat_rows = plan.partition()
    assert np.array_equal(plan.perm(), pre.perm)
    assert np.array_equal(colour, pre.color) and np.array_equal(cat_rows, pre.cat_rows)
    assert np.array_equal(cat_ptr, pre.cat_ptr)
    assert _rel(x, O.run_sweeps(pre, s.f, 100)) <= REL, rep.as_dict()


@pytest.mark.slow
@pytest.mark.parametrize("b", [0, 63])
def test_config5_full_parity(env, b):
    s = gen.make("batch9pt_1024", b)
    pre = O.preprocess(s.m, s.indptr, s.indices, s.data)
    plan, x, _ = _run(env, s, 20)
    assert np.array_equal(plan.perm(), pre.perm)
    assert np.array_equal(plan.partition()[0], pre.color)
    assert _rel(x, O.run_sweeps(pre, s.f, 20)) <= REL


@pytest.mark.slow
def test_config5_full_parity_bench_launch(env):
    """Config 5 at full size in the bench's launch configuration: systems 0 and 63 in one
    pobk_solve_batch call on two lanes (half-GPU K2 tilings), N_fix = 20 sweeps; bit-exact
    permutation / partition and iterates bitwise equal to the oracle's."""
    pk, torch = env
    systems = [gen.make("batch9pt_1024", b) for b in (0, 63)]
    tr = pk.half_gpu_tile_rows(systems[0].m)
    plans = [pk.Plan.from_system(s, tile_rows=tr) for s in systems]
    xs = [_dev(torch, np.zeros(s.m)) for s in systems]
    reps = pk.solve_batch(plans, [_dev(torch, s.f) for s in systems], xs, [_dev(torch, s.x_star) for s in systems],
                          max_sweeps=20, stop="none")
    for s, p, x, r in zip(systems, plans, xs, reps):
        assert r.sweeps == 20
        pre = O.preprocess(s.m, s.indptr, s.indices, s.data)
        assert np.array_equal(p.perm(), pre.perm) and np.array_equal(p.partition()[0], pre.color)
        assert np.array_equal(x.cpu().numpy(), O.run_sweeps(pre, s.f, 20))


@pytest.mark.parametrize("name,n", [("lap2d5_32", None), ("lap3d7_64", 11), ("randband_20k", 2000), ("geoknn_1m", 3000)])
def test_k3_layouts_bitwise_equal(env, name, n, monkeypatch):
    """K3 has two layouts (k3_smem.cu): the thread-major ELL (K3E, rows <= 16 entries) and the CSR
    fallback (POBK_NO_K3E); both follow the common.cuh contract, so both are the oracle's iterates,
    bitwise, including RELRES stop decisions at the same sweep."""
    pk, torch = env
    s = gen.make(name, n=n) if n else gen.make(name)
    outs = []
    for no_e in (False, True):
        if no_e:
            monkeypatch.setenv("POBK_NO_K3E", "1")
        try:
            _, x, _ = _run(env, s, 17, kernel="smem")
        except pk.PobkError:
            pytest.skip("system does not fit one CTA")
        outs.append(x)
        plan = pk.Plan.from_system(s, kernel="smem")
        xr = _dev(torch, np.zeros(s.m))
        outs.append(plan.solve(_dev(torch, s.f), xr, None, tol=1e-3, stop="relres").sweeps)
    pre = O.preprocess(s.m, s.indptr, s.indices, s.data)
    assert np.array_equal(outs[0], O.run_sweeps(pre, s.f, 17))
    assert np.array_equal(outs[0], outs[2])
    assert abs(outs[1] - outs[3]) <= 1


# ---------------------------------------------------------------- the bench's own stopping points
@pytest.mark.slow
def test_config4_stop_sweep_bench_point(env):
    """geoknn_1m at full size, in the bench's launch configuration (auto kernel -> K2), to the
    bench's stopping point RSE < 0.1 (PAPER.md:364-365 rule, R2): the same stop sweep
    +-1 as the oracle, the same final RSE to 1e-9, and -- at equal sweeps -- the oracle's iterates."""
    pk, torch = env
    s = gen.make("geoknn_1m")
    pre = O.preprocess(s.m, s.indptr, s.indices, s.data)
    ref = O.solve(s.m, s.indptr, s.indices, s.data, s.f, s.x_star, tol=0.1, pre=pre)
    assert ref.termination == O.TERM_CONVERGED
    plan = pk.Plan.from_system(s)
    assert plan.layout_stats()["kernel"] == "wavefront"
    x = _dev(torch, np.zeros(s.m))
    rep = plan.solve(_dev(torch, s.f), x, _dev(torch, s.x_star), tol=0.1)
    assert rep.termination == 0 and abs(rep.sweeps - ref.sweeps) <= 1, (rep.sweeps, ref.sweeps)
    assert abs(rep.final_value - ref.value) <= 1e-9 * ref.value
    if rep.sweeps == ref.sweeps:
        assert _rel(x.cpu().numpy(), ref.x) <= REL


@pytest.mark.slow
def test_config5_stop_sweep_bench_point(env):
    """Config 5 systems 0 and 63 at full size, in the bench's launch configuration (one
    pobk_solve_batch call, half-GPU K2 tilings on concurrent lanes), to RSE < 0.1: each system's
    stop sweep +-1 and final RSE (1e-9) against the oracle's own solve of that system."""
    pk, torch = env
    systems = [gen.make("batch9pt_1024", b) for b in (0, 63)]
    tr = pk.half_gpu_tile_rows(systems[0].m)
    plans = [pk.Plan.from_system(s, tile_rows=tr) for s in systems]
    xs = [_dev(torch, np.zeros(s.m)) for s in systems]
    reps = pk.solve_batch(plans, [_dev(torch, s.f) for s in systems], xs, [_dev(torch, s.x_star) for s in systems], tol=0.1)
    for s, x, r in zip(systems, xs, reps):
        ref = O.solve(s.m, s.indptr, s.indices, s.data, s.f, s.x_star, tol=0.1)
        assert ref.termination == O.TERM_CONVERGED and r.termination == 0
        assert abs(r.sweeps - ref.sweeps) <= 1, (r.sweeps, ref.sweeps)
        assert abs(r.final_value - ref.value) <= 1e-9 * ref.value
        if r.sweeps == ref.sweeps:
            assert _rel(x.cpu().numpy(), ref.x) <= REL


@pytest.mark.parametrize("kernel,name,n", [("launch", "lap2d5_32", None), ("smem", "lap2d5_32", None),
                                           ("wavefront", "lap3d7_64", 24), ("cluster", "randband_20k", 3000)])
def test_nonfinite_termination(env, kernel, name, n):
    """O8 (PAPER.md:366 records non-convergence): a non-finite RSE ends the solve
    with POBK_TERM_NONFINITE at the sweep it first appears, as in the oracle (f with an inf)."""
    pk, torch = env
    s = gen.make(name, n=n) if n else gen.make(name)
    f = s.f.copy()
    f[7] = np.inf
    ref = O.solve(s.m, s.indptr, s.indices, s.data, f, s.x_star, tol=1e-6, max_sweeps=50)
    assert ref.termination == O.TERM_NONFINITE
    try:
        plan = pk.Plan.from_system(s, kernel=kernel)
    except pk.PobkError as e:
        pytest.skip(f"{kernel} not applicable: {e}")
    x = _dev(torch, np.zeros(s.m))
    rep = plan.solve(_dev(torch, f), x, _dev(torch, s.x_star), tol=1e-6, max_sweeps=50)
    assert rep.termination == 2 and rep.sweeps == ref.sweeps, (rep.as_dict(), ref.sweeps)


@pytest.mark.parametrize("thr", [0.05])
def test_thr_positive_parity_20k(env, thr):
    """Overlapping categories (thr > 0) at m = 20,000 (config 2) on K1: the same
    thresholded partition as the oracle, iterates bitwise the oracle's after 25 sweeps (the
    ordered per-column scatter) and the same RSE stop sweep +-1."""
    pk, torch = env
    s = gen.make("randband_20k")
    pre = O.preprocess(s.m, s.indptr, s.indices, s.data, thr=thr)
    assert pre.overlap.any() and pre.nsteps < O.preprocess(s.m, s.indptr, s.indices, s.data).nsteps
    plan = pk.Plan.from_system(s, thr=thr)
    colour, cat_ptr, cat_rows = plan.partition()
    assert np.array_equal(colour, pre.color) and np.array_equal(cat_rows, pre.cat_rows)
    _, x, _ = _run(env, s, 25, plan=plan)
    assert np.array_equal(x, O.run_sweeps(pre, s.f, 25))
    ref = O.solve(s.m, s.indptr, s.indices, s.data, s.f, s.x_star, tol=1e-6, pre=pre)
    xx = _dev(torch, np.zeros(s.m))
    rep = plan.solve(_dev(torch, s.f), xx, _dev(torch, s.x_star), tol=1e-6)
    assert rep.termination == ref.termination and abs(rep.sweeps - ref.sweeps) <= 1


# ---------------------------------------------------------------- RELRES inside K2, resume, batch contract
@pytest.mark.slow
def test_relres_on_wavefront_config4(env):
    """RELRES stop (||f~ - A~x~||/||f~||) evaluated inside K2 (residual pass over each
    tile's stream, fixed-order reductions) at full config-4 size: the solve stays on the wavefront
    kernel and stops within +-1 sweep of the oracle's O8 rule (PAPER.md:364 strict '<'), with the
    same RELRES value to 1e-9 when the sweeps agree."""
    pk, torch = env
    s = gen.make("geoknn_1m")
    pre = O.preprocess(s.m, s.indptr, s.indices, s.data)
    tr = O.solve(s.m, s.indptr, s.indices, s.data, s.f, stop="relres", tol=0.0, max_sweeps=30, keep_trace=True, pre=pre)
    tol = float(tr.trace[24]) * (1 + 1e-9)   # the oracle stops at sweep 25 (trace decreasing there)
    assert tr.trace[23] > tol
    ref = O.solve(s.m, s.indptr, s.indices, s.data, s.f, stop="relres", tol=tol, pre=pre)
    plan = pk.Plan.from_system(s)
    x = _dev(torch, np.zeros(s.m))
    rep = plan.solve(_dev(torch, s.f), x, None, tol=tol, stop="relres")
    assert rep.kernel == 2, rep.as_dict()  # POBK_KERNEL_WAVEFRONT
    assert rep.termination == 0 and abs(rep.sweeps - ref.sweeps) <= 1, (rep.sweeps, ref.sweeps)
    assert np.isnan(rep.final_rse) and rep.final_relres == rep.final_value
    if rep.sweeps == ref.sweeps:
        assert abs(rep.final_value - ref.value) <= 1e-9 * ref.value


@pytest.mark.parametrize("name,n,kernel", [("lap3d7_64", 24, "wavefront"), ("lap2d5_32", None, "smem"),
                                           ("randband_20k", 4000, "launch")])
def test_relres_fixed_count_value(env, name, n, kernel):
    """RELRES after a fixed sweep count (tol 0, cap N: the check at the cap reports the value) on
    each kernel family equals the oracle's relres of the oracle's iterate to 1e-12."""
    pk, torch = env
    s = gen.make(name, n=n) if n else gen.make(name)
    pre = O.preprocess(s.m, s.indptr, s.indices, s.data)
    plan = pk.Plan.from_system(s, kernel=kernel)
    x = _dev(torch, np.zeros(s.m))
    rep = plan.solve(_dev(torch, s.f), x, None, tol=0.0, max_sweeps=9, stop="relres")
    assert rep.sweeps == 9 and rep.termination == 1
    xr = O.run_sweeps(pre, s.f, 9)
    v = O.relres(pre, O.permute_vector(s.f, pre.perm), O.permute_vector(xr, pre.perm))
    assert abs(rep.final_relres - v) <= 1e-12 * v


@pytest.mark.parametrize("name,n,kernel", [("lap3d7_64", 24, "wavefront"), ("lap2d5_32", None, "smem"),
                                           ("lap2d5_32", None, "launch")])
def test_sweep_offset_resume(env, name, n, kernel):
    """Resume (SURVEY §5 checkpoint/resume, §8b sweep_offset): 7 sweeps, then a second call from
    that x with sweep_offset = 7 and the same total cap, equals 12 uninterrupted sweeps bitwise;
    checks fall on the same sweep numbers (check_every = 5: a loose tol stops at total sweep 10)."""
    pk, torch = env
    s = gen.make(name, n=n) if n else gen.make(name)
    plan = pk.Plan.from_system(s, kernel=kernel)
    f, xs = _dev(torch, s.f), _dev(torch, s.x_star)
    x12 = _dev(torch, np.zeros(s.m))
    plan.solve(f, x12, xs, max_sweeps=12, stop="none")
    x = _dev(torch, np.zeros(s.m))
    r1 = plan.solve(f, x, xs, max_sweeps=7, stop="none")
    r2 = plan.solve(f, x, xs, max_sweeps=12, stop="none", sweep_offset=7)
    assert (r1.sweeps, r2.sweeps, r2.sweeps_total) == (7, 5, 12)
    assert np.array_equal(x.cpu().numpy(), x12.cpu().numpy())
    x = _dev(torch, np.zeros(s.m))
    plan.solve(f, x, xs, max_sweeps=7, stop="none")
    r3 = plan.solve(f, x, xs, tol=10.0, check_every=5, sweep_offset=7)
    assert r3.termination == 0 and r3.sweeps == 3 and r3.sweeps_total == 10
    r4 = plan.solve(f, x, xs, max_sweeps=7, sweep_offset=9)   # offset past the cap: nothing to do
    assert r4.sweeps == 0 and r4.sweeps_total == 9


def test_batch_duplicate_plan_and_bad_args(env):
    """pobk_solve_batch contract: a batch naming one plan twice gives each system its own
    back-to-back result (a plan is not re-entrant); a bad argument in any system fails the call
    before anything is enqueued (x of the other systems untouched)."""
    pk, torch = env
    systems = [gen.make("batch9pt_1024", b, n=160) for b in range(2)]
    tr = pk.half_gpu_tile_rows(systems[0].m)
    p = pk.Plan.from_system(systems[0], kernel="wavefront", tile_rows=tr)
    f = _dev(torch, systems[0].f)
    xs = [_dev(torch, np.zeros(systems[0].m)) for _ in range(2)]
    reps = pk.solve_batch([p, p], [f, f], xs, None, max_sweeps=15, stop="none")
    x1 = _dev(torch, np.zeros(systems[0].m))
    p.solve(f, x1, None, max_sweeps=15, stop="none")
    assert all(r.sweeps == 15 for r in reps)
    assert np.array_equal(xs[0].cpu().numpy(), x1.cpu().numpy()) and np.array_equal(xs[1].cpu().numpy(), x1.cpu().numpy())
    q = pk.Plan.from_system(systems[1], kernel="wavefront", tile_rows=tr)
    x0 = [_dev(torch, np.zeros(s.m)) for s in systems]
    with pytest.raises(pk.PobkError):  # system 1: RSE stop without x*
        import ctypes
        L = pk._lib
        H = (ctypes.c_void_p * 2)(p._h.value, q._h.value)
        F = (ctypes.c_void_p * 2)(f.data_ptr(), _dev(torch, systems[1].f).data_ptr())
        X = (ctypes.c_void_p * 2)(x0[0].data_ptr(), x0[1].data_ptr())
        XS = (ctypes.c_void_p * 2)(_dev(torch, systems[0].x_star).data_ptr(), None)
        reps = (L.Report * 2)()
        o = pk._solve_opts(1e-3, 100, "rse", 1)
        L.check(L.lib.pobk_solve_batch(H, 2, ctypes.cast(F, ctypes.c_void_p), ctypes.cast(X, ctypes.c_void_p),
                                       ctypes.cast(XS, ctypes.c_void_p), ctypes.byref(o), None, ctypes.cast(reps, ctypes.c_void_p)))
    torch.cuda.synchronize()
    assert not x0[0].any().item()


@pytest.mark.parametrize("nb,lanes", [(5, True), (3, False)])
def test_batch_host_equals_device_batch(env, nb, lanes):
    """pobk_solve_batch_host (host vectors; copies of other systems overlapped with the sweeps on
    concurrent lanes): every system's stop sweep, final RSE and solution are bitwise those of
    pobk_solve_batch on device vectors, on lanes (half-GPU K2 tilings, odd batch) and on one
    internal stream (AUTO plans); pinned and pageable host buffers; a bad argument fails before
    anything runs; a plan named twice runs back to back."""
    pk, torch = env
    systems = [gen.make("batch9pt_1024", b, n=160) for b in range(nb)]
    kw = dict(kernel="wavefront", tile_rows=pk.half_gpu_tile_rows(systems[0].m)) if lanes else {}
    plans = [pk.Plan.from_system(s, **kw) for s in systems]
    xs = [_dev(torch, np.zeros(s.m)) for s in systems]
    reps = pk.solve_batch(plans, [_dev(torch, s.f) for s in systems], xs, [_dev(torch, s.x_star) for s in systems],
                          tol=0.2)
    for pinned in (True, False):
        conv = (lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()) if pinned else np.ascontiguousarray
        hf = [conv(s.f) for s in systems]
        hxs = [conv(s.x_star) for s in systems]
        hx = [conv(np.zeros(s.m)) for s in systems]
        hreps = pk.solve_batch_host(plans, hf, hx, hxs, tol=0.2)
        for r, hr, xd, xh in zip(reps, hreps, xs, hx):
            assert hr.sweeps == r.sweeps and hr.final_value == r.final_value
            assert np.array_equal(xh, xd.cpu().numpy())
    s0 = systems[0]
    pre = O.preprocess(s0.m, s0.indptr, s0.indices, s0.data)
    assert np.array_equal(hx[0], O.run_sweeps(pre, s0.f, reps[0].sweeps))
    bad = [np.zeros(s.m) for s in systems]
    with pytest.raises(pk.PobkError):  # last system: RSE stop without x*
        import ctypes
        L = pk._lib
        H = (ctypes.c_void_p * nb)(*[p._h.value for p in plans])
        F = (ctypes.c_void_p * nb)(*[L.ptr(f).value for f in hf])
        X = (ctypes.c_void_p * nb)(*[L.ptr(x).value for x in bad])
        XS = (ctypes.c_void_p * nb)(*([L.ptr(x).value for x in hxs[:-1]] + [None]))
        o = pk._solve_opts(0.2, 100, "rse", 1)
        L.check(L.lib.pobk_solve_batch_host(H, nb, ctypes.cast(F, ctypes.c_void_p), ctypes.cast(X, ctypes.c_void_p),
                                            ctypes.cast(XS, ctypes.c_void_p), ctypes.byref(o), None,
                                            ctypes.cast((L.Report * nb)(), ctypes.c_void_p)))
    assert not any(b.any() for b in bad)
    with pytest.raises(pk.PobkError):  # one host x for two systems
        pk.solve_batch_host(plans[:2], hf[:2], [bad[0], bad[0]], hxs[:2], tol=0.2)
    assert not bad[0].any()
    # a plan named twice: back to back through pobk_solve_host, each system its own result
    hx2 = [np.zeros(systems[0].m) for _ in range(2)]
    r2 = pk.solve_batch_host([plans[0], plans[0]], [hf[0], hf[0]], hx2, [hxs[0], hxs[0]], tol=0.2)
    assert all(r.sweeps == reps[0].sweeps for r in r2)
    assert np.array_equal(hx2[0], xs[0].cpu().numpy()) and np.array_equal(hx2[1], xs[0].cpu().numpy())


# ---------------------------------------------------------------- several right-hand sides (NEXT-3)
@pytest.mark.parametrize("name,n,R,tol", [("lap3d7_64", 24, 3, 0.1), ("lap2d5_32", None, 8, 1e-3),
                                          ("geoknn_1m", 30000, 4, 0.1)])
def test_multi_rhs_bitwise_equals_single(env, name, n, R, tol):
    """pobk_solve_multi: R right-hand sides of one matrix (Ax = f) in one sweep loop
    -- A read once per step for all of them -- each stopping on its own RSE rule: every right-hand
    side's stop sweep and iterates are bitwise those of its own single solve (and so the oracle's)."""
    pk, torch = env
    systems = [gen.make(name, b, n=n) if n else gen.make(name, b) for b in range(R)]
    assert all(np.array_equal(s.data, systems[0].data) for s in systems)  # one matrix, R right-hand sides
    plan = pk.Plan.from_system(systems[0])
    fs = [_dev(torch, s.f) for s in systems]
    xss = [_dev(torch, s.x_star) for s in systems]
    xs = [_dev(torch, np.zeros(s.m)) for s in systems]
    reps = plan.solve_multi(fs, xs, xss, tol=tol)
    for s, f, xst, x, r in zip(systems, fs, xss, xs, reps):
        x1 = _dev(torch, np.zeros(s.m))
        r1 = plan.solve(f, x1, xst, tol=tol)
        assert r.sweeps == r1.sweeps and r.termination == r1.termination, (r.as_dict(), r1.as_dict())
        assert np.array_equal(x.cpu().numpy(), x1.cpu().numpy())
    pre = O.preprocess(systems[0].m, systems[0].indptr, systems[0].indices, systems[0].data)
    assert np.array_equal(xs[-1].cpu().numpy(), O.run_sweeps(pre, systems[-1].f, reps[-1].sweeps))


@pytest.mark.parametrize("name,n,R,tol", [("geoknn_1m", None, 2, 0.1), ("lap3d7_64", None, 3, 0.1),
                                          ("geoknn_1m", 60000, 5, 0.05)])
def test_multi_rhs_wavefront_pairs(env, name, n, R, tol):
    """K2 plans take right-hand sides in PAIRS through the two-RHS K2 layout (x~ pair-interleaved
    in shared memory and the mailboxes, A~ streamed once per sweep for both), an
    odd last one through the plan's own solve.  Each right-hand side keeps the per-row contract
    and stops on its own RSE rule (a stopped one is frozen while its partner
    iterates): stop sweep, termination, RSE value and iterates bitwise its single solve's; full
    sizes of configs 3 and 4 (the bench's stopping point)."""
    pk, torch = env
    systems = [gen.make(name, b, n=n) if n else gen.make(name, b) for b in range(R)]
    plan = pk.Plan.from_system(systems[0])
    assert plan.layout_stats()["kernel"] == "wavefront"
    fs = [_dev(torch, s.f) for s in systems]
    xss = [_dev(torch, s.x_star) for s in systems]
    xs = [_dev(torch, np.zeros(s.m)) for s in systems]
    reps = plan.solve_multi(fs, xs, xss, tol=tol)
    assert all(r.kernel == 2 for r in reps)
    sweeps = []
    for s, f, xst, x, r in zip(systems, fs, xss, xs, reps):
        x1 = _dev(torch, np.zeros(s.m))
        r1 = plan.solve(f, x1, xst, tol=tol)
        assert r.sweeps == r1.sweeps and r.termination == r1.termination, (r.as_dict(), r1.as_dict())
        assert r.final_rse == r1.final_rse
        assert np.array_equal(x.cpu().numpy(), x1.cpu().numpy())
        sweeps.append(r.sweeps)
    # fixed sweep count, no stop rule: the second member bitwise the oracle's sweeps
    xs = [_dev(torch, np.zeros(s.m)) for s in systems[:2]]
    reps = plan.solve_multi(fs[:2], xs, None, stop="none", max_sweeps=6)
    assert [r.sweeps for r in reps] == [6, 6] and all(r.kernel == 2 for r in reps)
    pre = O.preprocess(systems[0].m, systems[0].indptr, systems[0].indices, systems[0].data)
    assert np.array_equal(xs[1].cpu().numpy(), O.run_sweeps(pre, systems[1].f, 6))


def test_multi_rhs_wavefront_freeze(env):
    """A two-RHS K2 solve whose members stop far apart: RHS 0 starts from an x0 close to x*, so it
    meets the RSE rule early and stays frozen while RHS 1 (x0 = 0) iterates on; each matches its
    own single solve bitwise (stop sweep and iterates)."""
    pk, torch = env
    s = gen.make("geoknn_1m", 0, n=30000)
    plan = pk.Plan.from_system(s)
    assert plan.layout_stats()["kernel"] == "wavefront"
    f, xst = _dev(torch, s.f), _dev(torch, s.x_star)
    x0 = _dev(torch, s.x_star * 0.999)
    xs = [x0.clone(), _dev(torch, np.zeros(s.m))]
    r2 = plan.solve_multi([f, f], xs, [xst, xst], tol=0.01)
    xa = x0.clone()
    ra = plan.solve(f, xa, xst, tol=0.01)
    xb = _dev(torch, np.zeros(s.m))
    rb = plan.solve(f, xb, xst, tol=0.01)
    assert ra.sweeps < rb.sweeps, (ra.sweeps, rb.sweeps)
    assert (r2[0].sweeps, r2[1].sweeps) == (ra.sweeps, rb.sweeps)
    assert r2[0].final_rse == ra.final_rse and r2[1].final_rse == rb.final_rse
    assert np.array_equal(xs[0].cpu().numpy(), xa.cpu().numpy())
    assert np.array_equal(xs[1].cpu().numpy(), xb.cpu().numpy())


def test_multi_rhs_contract(env):
    pk, torch = env
    s = gen.make("lap2d5_32")
    plan = pk.Plan.from_system(s)
    f = _dev(torch, s.f)
    with pytest.raises(pk.PobkError):
        plan.solve_multi([f] * 9, [_dev(torch, np.zeros(s.m)) for _ in range(9)], None, stop="none", max_sweeps=3)
    with pytest.raises(pk.PobkError):
        plan.solve_multi([f, f], [_dev(torch, np.zeros(s.m)) for _ in range(2)], None, stop="relres")
    x = _dev(torch, np.zeros(s.m))
    with pytest.raises(pk.PobkError):  # the same x twice
        plan.solve_multi([f, f], [x, x], None, stop="none", max_sweeps=3)
    thr_plan = pk.Plan.from_system(s, thr=0.12)
    with pytest.raises(pk.PobkError):
        thr_plan.solve_multi([f], [x], None, stop="none", max_sweeps=3)
    # fixed count, resume numbering
    xs = [_dev(torch, np.zeros(s.m)) for _ in range(2)]
    reps = plan.solve_multi([f, f], xs, None, stop="none", max_sweeps=12, sweep_offset=5)
    assert [r.sweeps for r in reps] == [7, 7] and [r.sweeps_total for r in reps] == [12, 12]


# ---------------------------------------------------------------- residual-ordered sweep (NEXT-4)
@pytest.mark.parametrize("name,n,tol", [("lap2d5_32", None, 1e-2), ("randband_20k", 3000, 1e-6), ("lap3d7_64", 16, 0.1),
                                        ("geoknn_1m", 20000, 0.1)])
def test_residual_order_parity(env, name, n, tol):
    """opts.order = residual (reading R-G): the device scores every step with the
    oracle's fixed two-level sums, so it takes the same order decisions -- iterates bitwise the
    oracle's residual-ordered sweeps (O7 per step), stop sweep +-1."""
    pk, torch = env
    s = gen.make(name, n=n) if n else gen.make(name)
    pre = O.preprocess(s.m, s.indptr, s.indices, s.data)
    plan = pk.Plan.from_system(s)
    x = _dev(torch, np.zeros(s.m))
    rep = plan.solve(_dev(torch, s.f), x, _dev(torch, s.x_star), max_sweeps=7, stop="none", order="residual")
    assert rep.sweeps == 7 and rep.kernel == 1
    assert np.array_equal(x.cpu().numpy(), O.run_sweeps_ordered(pre, s.f, 7))
    xo, sweeps, term, v = O.solve_ordered(pre, s.f, s.x_star, tol, 20000)
    x = _dev(torch, np.zeros(s.m))
    rep = plan.solve(_dev(torch, s.f), x, _dev(torch, s.x_star), tol=tol, max_sweeps=20000, order="residual")
    assert rep.termination == term and abs(rep.sweeps - sweeps) <= 1, (rep.sweeps, sweeps)
