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


def _gather_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1506_00014_b200.sharding import gather_to_root

    local = torch.full((2, 3, 4), float(rank + 1))
    buf = torch.empty(2 * world, 3, 4) if rank == 1 else None
    got = gather_to_root(local, root=1, out=buf)
    out[rank] = None if got is None else got.tolist()
    dist.barrier()
    dist.destroy_process_group()


def test_gather_to_root_gloo():
    """The final gather: grouped send/recv to a root, shards
    in rank order; non-root ranks get None."""
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_gather_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    assert out[0] is None
    import numpy as np

    got = np.array(out[1])
    assert got.shape == (4, 3, 4)
    assert (got[:2] == 1).all() and (got[2:] == 2).all()


def test_bench_dry_run_two_ranks():
    """bench.py --gpus 2 outside torchrun re-executes itself under
    torch.distributed.run with 2 ranks; --dry-run drives the rank / shard /
    gather path with gloo on CPU and prints n_gpus and the gather bytes."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--dry-run", "--size", "32",
                        "--batch", "3"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    line = lines[0]
    assert line["n_gpus"] == 2 and line["dry_run"] is True
    assert line["gathered"]["verified"] is True
    assert line["gathered"]["bytes_to_rank0_per_step"] == 3 * 48 * 32 * 4
    assert line["max_over_ranks"] == 1.0
    # the config-4 stack (2048 slices) split over the ranks: contiguous, disjoint, complete
    assert line["stack"] == {"slices": 2048, "slices_per_rank0": 1024, "partition_verified": True}
