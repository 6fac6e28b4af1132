"""N > 1 host-side path on CPU (-m "not gpu"): world-size-2 gloo process group exercising the
driver's sharding, max-over-ranks timing, report gathering and the row-sharded residual (C2)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch.distributed as dist

    import oracle as O
    from paper_2401_00672_b200 import driver
    from workloads import gen
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # independent systems: every system id lands on exactly one rank
        ids = driver.shard(64, world, rank)
        all_ids = sum(driver.gather_objects(ids), [])
        # max over ranks
        t = driver.max_over_ranks(1.0 + rank)
        # row-sharded residual of one system at some x: ranks sum their own rows
        s = gen.make("lap2d5_32")
        x = np.linspace(-1, 1, s.m)
        lo, hi = driver.row_range(s.m, world, rank)
        A = s.csr()
        r = s.f[lo:hi] - A[lo:hi] @ x
        local = float(np.dot(r, r))
        res = driver.sharded_residual_norm(local)
        full = O.residual_norm(s.m, s.indptr, s.indices, s.data, s.f, x)
        reports = driver.gather_objects({"rank": rank, "systems": len(ids)})
        # the bench's report path (C1): per-system reports -> gather_reports on every rank
        local = [driver.system_report(i, 100 + i, {"sweeps": 10 + i, "termination": "converged", "final_value": 0.05})
                 for i in ids]
        agg = driver.gather_reports(local, 0.5 + rank)
        out[rank] = (sorted(all_ids), t, res, full, reports, agg)
    finally:
        dist.destroy_process_group()


def test_two_rank_driver():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    for rank in range(world):
        ids, t, res, full, reports, agg = out[rank]
        assert ids == list(range(64))
        assert t == 2.0
        assert abs(res - full) <= 1e-12 * full
        assert [r["rank"] for r in reports] == [0, 1] and sum(r["systems"] for r in reports) == 64
        assert agg["systems"] == 64 and agg["seconds"] == 1.5
        assert [r["id"] for pr in agg["ranks"] for r in pr["systems"]] == list(range(64))
        assert agg["nnz_updates"] == float(sum((100 + i) * (10 + i) for i in range(64)))


@pytest.mark.parametrize("n,world", [(64, 8), (10, 3), (3, 4), (0, 2)])
def test_shard_partition(n, world):
    from paper_2401_00672_b200 import driver
    parts = [driver.shard(n, world, r) for r in range(world)]
    assert sum(parts, []) == list(range(n))
    assert max(map(len, parts)) - min(map(len, parts)) <= 1


def _nccl_worker(rank, world, port, out):
    """The product's multi-GPU path on the GPU box (world size 1 -- gpurun has one GPU): NCCL
    process group, a shard of config-5 systems solved with pobk_solve_batch, per-system reports
    through gather_reports, and the row-sharded residual (C2) from pobk_residual_sumsq_rows +
    all_reduce, checked against pobk_residual_norm and the oracle."""
    import torch
    import torch.distributed as dist

    import oracle as O
    import paper_2401_00672_b200 as pk
    from paper_2401_00672_b200 import driver
    from workloads import gen
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        dev = torch.device("cuda", rank)
        ids = driver.shard(4, world, rank)
        systems = [gen.make("batch9pt_1024", i, n=96) for i in ids]
        plans = [pk.Plan.from_system(s) for s in systems]
        fs = [torch.from_numpy(s.f).to(dev) for s in systems]
        xs = [torch.zeros(s.m, dtype=torch.float64, device=dev) for s in systems]
        reps = pk.solve_batch(plans, fs, xs, [torch.from_numpy(s.x_star).to(dev) for s in systems], tol=1e-2)
        agg = driver.gather_reports([driver.system_report(i, p.nnz, r) for i, p, r in zip(ids, plans, reps)], 1.0, dev)
        s, p, f, x = systems[0], plans[0], fs[0], xs[0]
        lo, hi = driver.row_range(s.m, world, rank)
        res = driver.sharded_residual_norm(p.residual_sumsq_rows(lo, hi, f, x), dev)
        full = p.residual_norm(f, x)
        ref = O.residual_norm(s.m, s.indptr, s.indices, s.data, s.f, x.cpu().numpy())
        out[rank] = (agg["systems"], [r.termination for r in reps], res, full, ref)
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_nccl_world1_driver_path():
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_nccl_worker, args=(1, port, out), nprocs=1, join=True)
    nsys, terms, res, full, ref = out[0]
    assert nsys == 4 and all(t == 0 for t in terms)
    assert abs(res - full) <= 1e-12 * full and abs(full - ref) <= 1e-9 * ref
