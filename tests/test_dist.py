"""Multi-process (world_size 2, gloo, CPU) coverage of the sharded inference
plumbing: contiguous shards, padded all-gather, input-order reassembly."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1711_03637_b200.distributed import gather_counts, shard_bounds
    a, b = shard_bounds(n, world)[rank]
    # stand-in for the per-rank GPU result: counts that encode the global index
    local = torch.stack([torch.arange(a, b, dtype=torch.int32) * 10 + k for k in range(10)], dim=1)
    allc = gather_counts(local, n)
    if rank == 0:
        out_q.put(allc.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [1, 9, 101])
def test_gather_counts_world2(n):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    want = np.stack([np.arange(n) * 10 + k for k in range(10)], axis=1)
    assert np.array_equal(got, want)
