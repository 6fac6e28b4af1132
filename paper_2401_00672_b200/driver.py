"""Multi-GPU plumbing (torch.distributed): one process per GPU, independent systems per rank.

The POBK sweep of one system does not shard: ranks solve DIFFERENT systems (a
batch such as BASELINE config 5, 8 systems per GPU) with no data-path collective.  The only
collectives are control/reporting: a start barrier, the max-over-ranks elapsed time, the
gathering of per-system reports, and the row-sharded residual (C2): each rank
computes sum (f_i - a_i.x)^2 over its rows with pobk_residual_sumsq_rows and an all-reduce SUM
forms ||f - Ax||.  Everything here is backend-agnostic (NCCL on the GPU box, gloo in the CPU
tests).
"""
from __future__ import annotations

import math

import torch
import torch.distributed as dist

__all__ = ["shard", "row_range", "max_over_ranks", "sum_over_ranks", "gather_objects", "sharded_residual_norm",
           "system_report", "gather_reports"]


def shard(n_items: int, world: int, rank: int) -> list[int]:
    """Contiguous block of item ids for `rank` (sizes differ by at most one)."""
    base, extra = divmod(n_items, world)
    lo = rank * base + min(rank, extra)
    return list(range(lo, lo + base + (1 if rank < extra else 0)))


def row_range(m: int, world: int, rank: int) -> tuple[int, int]:
    ids = shard(m, world, rank)
    return (ids[0], ids[-1] + 1) if ids else (0, 0)


def _tensor(v: float, device) -> torch.Tensor:
    return torch.tensor([float(v)], dtype=torch.float64, device=device)


def max_over_ranks(v: float, device="cpu") -> float:
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(v)
    t = _tensor(v, device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(v: float, device="cpu") -> float:
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(v)
    t = _tensor(v, device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def gather_objects(obj) -> list:
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return [obj]
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, obj)
    return out


def sharded_residual_norm(local_sumsq: float, device="cpu") -> float:
    """||f - Ax||_2 from every rank's sum over its own rows (pobk_residual_sumsq_rows)."""
    return math.sqrt(sum_over_ranks(local_sumsq, device))


def system_report(system_id: int, nnz: int, rep) -> dict:
    """One system's solve as reported by pobk_solve / pobk_solve_batch (pobk_report), reduced to
    what the run summary keeps: id, stored nonzeros, sweeps, termination, final stop value."""
    d = rep.as_dict() if hasattr(rep, "as_dict") else dict(rep)
    return {"id": int(system_id), "nnz": int(nnz), "sweeps": int(d["sweeps"]), "termination": d["termination"],
            "final": float(d["final_value"])}


def gather_reports(local: list[dict], seconds: float, device="cpu") -> dict:
    """C1: every rank's per-system reports gathered to every rank, the elapsed time
    as the max over ranks, and the whole job's nnz-updates (sum of nnz x sweeps over all systems)."""
    per_rank = gather_objects({"rank": dist.get_rank() if dist.is_initialized() else 0, "systems": local})
    t = max_over_ranks(seconds, device)
    updates = sum(r["nnz"] * r["sweeps"] for pr in per_rank for r in pr["systems"])
    return {"ranks": per_rank, "seconds": t, "nnz_updates": float(updates),
            "systems": sum(len(pr["systems"]) for pr in per_rank)}
