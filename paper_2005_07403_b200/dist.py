"""Multi-GPU plumbing: one process per GPU, contiguous lane shards.

The batched 2x2 SVD is embarrassingly parallel -- lane k of the output
depends only on lane k of the input (reference test_svd2.py:428-440,
test_driver.py:165-177) -- so N GPUs each own one contiguous lane range of
the batch (the multi-process analogue of driver._slabs, driver.py:134-146)
and there is no collective on the data path.  torch.distributed (NCCL on
GPUs, gloo on CPU tests) is used only for the timing barrier, the
max-over-ranks of measured times, and gathering per-shard digests.
"""

from __future__ import annotations

import hashlib
import os

from .driver import shards

__all__ = ["rank_span", "world_info", "barrier", "max_over_ranks",
           "sum_over_ranks", "gather", "shard_digest", "combine_digests"]


def world_info():
    """(world_size, rank, local_rank) from the torchrun environment."""
    return (int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def rank_span(n, rank, world):
    """This rank's contiguous lane range [lo, hi) of an n-lane batch
    (empty when there are more ranks than 256-lane units)."""
    spans = shards(n, world)
    if rank < len(spans):
        return spans[rank]
    return (n, n)


def _dist():
    import torch.distributed as dist
    return dist if dist.is_available() and dist.is_initialized() else None


def _tensor(x):
    import torch
    dist = _dist()
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    return torch.tensor([float(x)], dtype=torch.float64, device=dev)


def barrier():
    dist = _dist()
    if dist is not None and dist.get_world_size() > 1:
        dist.barrier()


def max_over_ranks(x):
    """Maximum of a scalar over all ranks (identity without a process group)."""
    dist = _dist()
    if dist is None or dist.get_world_size() == 1:
        return float(x)
    t = _tensor(x)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x):
    dist = _dist()
    if dist is None or dist.get_world_size() == 1:
        return float(x)
    t = _tensor(x)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def gather(obj):
    """All ranks' picklable objects, in rank order."""
    dist = _dist()
    if dist is None or dist.get_world_size() == 1:
        return [obj]
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, obj)
    return out


def shard_digest(trains):
    """Incremental SHA-256 state of a shard's output trains: a dict name ->
    raw bytes of the train (uint64 view), in a fixed key order."""
    return {k: hashlib.sha256(bytes(memoryview(v).cast("B"))).hexdigest()
            for k, v in sorted(trains.items())}


def combine_digests(per_rank):
    """Checksum of checksums: one digest over the ordered per-rank digests."""
    h = hashlib.sha256()
    for d in per_rank:
        for k in sorted(d):
            h.update(k.encode())
            h.update(d[k].encode())
    return h.hexdigest()
