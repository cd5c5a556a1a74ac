"""CPU (gloo, world_size 2) coverage of the multi-GPU plumbing: slice shards
partition the stack, and timings reduce to the slowest rank."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_slices, out):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1506_00014_b200.sharding import max_over_ranks, stack_shard

    start, count = stack_shard(n_slices, world, rank)
    slowest = max_over_ranks(10.0 + rank)
    out[rank] = (start, count, slowest)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_slices", [2048, 7])
def test_shards_partition_and_max_reduce(n_slices):
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), n_slices, out), nprocs=world, join=True)
    covered = []
    for r in range(world):
        start, count, slowest = out[r]
        covered.extend(range(start, start + count))
        assert slowest == 10.0 + world - 1
    assert covered == list(range(n_slices))


def test_shard_arguments():
    from paper_1506_00014_b200.sharding import stack_shard

    assert stack_shard(10, 4, 0) == (0, 3) and stack_shard(10, 4, 3) == (8, 2)
    with pytest.raises(ValueError):
        stack_shard(10, 2, 2)
