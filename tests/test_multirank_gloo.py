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
        out[rank] = (sorted(all_ids), t, res, full, reports)
    finally:
        dist.destroy_process_group()


def test_two_rank_driver():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    for rank in range(world):
        ids, t, res, full, reports = out[rank]
        assert ids == list(range(64))
        assert t == 2.0
        assert abs(res - full) <= 1e-12 * full
        assert [r["rank"] for r in reports] == [0, 1] and sum(r["systems"] for r in reports) == 64


@pytest.mark.parametrize("n,world", [(64, 8), (10, 3), (3, 4), (0, 2)])
def test_shard_partition(n, world):
    from paper_2401_00672_b200 import driver
    parts = [driver.shard(n, world, r) for r in range(world)]
    assert sum(parts, []) == list(range(n))
    assert max(map(len, parts)) - min(map(len, parts)) <= 1
