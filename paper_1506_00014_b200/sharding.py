"""Slice sharding for multi-GPU runs.

Slices of a 3-D stack are independent, so each rank takes a contiguous
range of slices and runs its own plan; the only cross-rank traffic on the
sharded path is a barrier and the max-reduction of timings (no collective on
the data path). The optional final gather of every rank's outputs to one
rank is `gather_to_root`: grouped point-to-point
sends/receives (NCCL ncclSend/ncclRecv inside one group over NVLink/NVSwitch
on GPUs, gloo on CPU).
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


def gather_to_root(local, root: int = 0, out=None):
    """Gather every rank's shard `local` (same shape and dtype on every rank)
    to `root` with one grouped batch of point-to-point ops: root posts a
    receive per peer, every other rank one send (torch batch_isend_irecv ->
    ncclGroupStart / ncclSend / ncclRecv / ncclGroupEnd). Returns on root the
    shards concatenated in rank order along dim 0 (written into `out`, shape
    (world * local.shape[0], ...), when given), None on the other ranks.
    Single process: returns `local`."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return local
    ws, rank = dist.get_world_size(), dist.get_rank()
    if not 0 <= root < ws:
        raise ValueError("gather_to_root: bad root")
    n = local.shape[0]
    if rank == root:
        if out is None:
            out = torch.empty((ws * n,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
        elif tuple(out.shape) != (ws * n,) + tuple(local.shape[1:]) or out.dtype != local.dtype:
            raise ValueError("gather_to_root: out has the wrong shape or dtype")
        out[root * n:(root + 1) * n].copy_(local)
        ops = [dist.P2POp(dist.irecv, out[r * n:(r + 1) * n], r) for r in range(ws) if r != root]
    else:
        ops = [dist.P2POp(dist.isend, local.contiguous(), root)]
    for w in dist.batch_isend_irecv(ops):
        w.wait()
    return out if rank == root else None
