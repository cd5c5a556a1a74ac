"""Slice sharding for multi-GPU runs.

Slices of a 3-D stack are independent, so each rank takes a contiguous
range of slices and runs its own plan; the only cross-rank traffic is a
barrier and the max-reduction of timings (no collective on the data path).
"""
from __future__ import annotations


def stack_shard(n_slices: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [start, start + count) share of rank `rank`; shares differ by
    at most one slice and partition the stack."""
    if world < 1 or not 0 <= rank < world or n_slices < 0:
        raise ValueError("stack_shard: bad arguments")
    base, extra = divmod(n_slices, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (timings are reported as the slowest rank)."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
