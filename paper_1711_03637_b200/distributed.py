"""Data-parallel inference over GPUs: one process per GPU, contiguous shards,
one collective (an all-gather of the int32 counts) at the end.

The reference's only parallel strategy is process-level data parallelism over
images in batch_counts (evaluate.py:34-39: np.array_split chunks, results
concatenated in input order).  Here each rank owns one B200; the shard
boundaries are np.array_split's, so the gathered result is in input order.
Training is sequential online NormAD and stays on one GPU (replicas only).
"""
from __future__ import annotations

import numpy as np

from .params import N_OUTPUTS


def shard_bounds(n: int, world: int):
    """[(start, stop)] per rank, identical to np.array_split(range(n), world)."""
    q, r = divmod(n, world)
    bounds, start = [], 0
    for k in range(world):
        stop = start + q + (1 if k < r else 0)
        bounds.append((start, stop))
        start = stop
    return bounds


def gather_counts(local, n_total: int, group=None):
    """All-gather per-rank int32 [n_k,10] device tensors into [n_total,10] in
    rank order.  Pads every shard to the largest one (NCCL needs equal sizes)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    bounds = shard_bounds(n_total, world)
    width = max(b - a for a, b in bounds)
    send = torch.zeros((width, N_OUTPUTS), dtype=torch.int32, device=local.device)
    send[: local.shape[0]] = local
    recv = torch.empty((world * width, N_OUTPUTS), dtype=torch.int32, device=local.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(recv, send, group=group)
    else:  # gloo (CPU tests)
        dist.all_gather(list(recv.chunk(world)), send, group=group)
    parts = [recv[k * width: k * width + (b - a)] for k, (a, b) in enumerate(bounds)]
    return torch.cat(parts, dim=0)


def sharded_counts_device(images_dev_shard, w_dev, consts, n_total: int, engine, group=None):
    """Device-resident sharded inference: this rank's shard -> all counts."""
    local = engine.infer(consts, images_dev_shard, w_dev)["counts"]
    engine.stream.synchronize()
    return gather_counts(local, n_total, group)


def sharded_batch_counts(images, weights, filters, cfg, group=None) -> np.ndarray:
    """batch_counts over all ranks of the process group: every rank passes the
    full image set, simulates its contiguous shard on its own GPU, and gets
    back the (n, 10) int64 counts of the whole set in input order."""
    import torch
    import torch.distributed as dist

    from .api import _consts_cached, _weights
    from .engine import get_engine
    from .params import as_pixel_batch

    imgs = as_pixel_batch(images)
    n = len(imgs)
    if n == 0:
        return np.zeros((0, N_OUTPUTS), dtype=np.int64)
    if not (dist.is_available() and dist.is_initialized()):
        from .api import batch_counts
        return batch_counts(imgs, weights, filters, cfg)
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    a, b = shard_bounds(n, world)[rank]
    c = _consts_cached(cfg, filters)
    eng = get_engine()
    with eng.lock:
        d_w = eng.weights(weights, check=_weights)
        if b > a:
            d_img = eng.upload("images", imgs[a:b]).view(b - a, -1)
            local = eng.infer(c, d_img, d_w)["counts"]
        else:
            local = torch.zeros((0, N_OUTPUTS), dtype=torch.int32, device=eng.device)
        eng.stream.synchronize()
    allc = gather_counts(local, n, group)
    from .api import _fetch
    torch.cuda.current_stream(eng.device).synchronize()  # the gather ran on the caller's stream
    with eng.lock:
        return _fetch(eng, allc, np.int64)  # one DMA through the engine's pinned staging buffer
