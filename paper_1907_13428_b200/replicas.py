"""Multi-GPU = replicas only: the hot path does not
shard under the north star, so N GPUs run N independent solves.  This module
holds the host logic around that: splitting independent work items (e.g. the
reference CLI's delta sweep, fdeopt_main.cpp:133-195) over ranks and reducing
per-rank timings the way the bench contract requires (max over ranks for
time, sum over ranks for work).  It is backend-agnostic (nccl on GPUs, gloo
in the CPU tests).
"""
from __future__ import annotations


def shard(items, rank: int, world: int):
    """Round-robin assignment of independent work items (order preserved)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("shard: bad rank/world")
    return [it for i, it in enumerate(items) if i % world == rank]


def aggregate(elapsed_ms: float, units: float, dist=None, device=None):
    """(max elapsed over ranks, sum of units over ranks)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(elapsed_ms), float(units)
    import torch
    t = torch.tensor([float(elapsed_ms)], dtype=torch.float64, device=device)
    u = torch.tensor([float(units)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(u, op=dist.ReduceOp.SUM)
    return float(t.item()), float(u.item())


def gather_records(records, dist=None):
    """All ranks' per-item result records (lists of dicts), rank-major, on every rank."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return list(records)
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, list(records))
    merged = []
    for part in out:
        merged.extend(part)
    return merged
