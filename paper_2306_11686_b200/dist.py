"""Multi-GPU plumbing: lookups shard by contiguous global index range, the grid
is replicated by a local build on every rank, and the only exchange is one int64 all-reduce (SUM)
of the raw verification sum per batch.  Works with any torch.distributed backend (NCCL on the B200
box; gloo in the CPU tests)."""
from __future__ import annotations

from . import shard_range, verify, weak_range

__all__ = ["shard_range", "weak_range", "reduce_raw", "max_over_ranks", "finish_hash"]


def reduce_raw(vsum, group=None):
    """In-place SUM of the per-rank raw sums (int64 tensor of one element)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(vsum, op=dist.ReduceOp.SUM, group=group)
    return vsum


def max_over_ranks(values, device, group=None):
    """Element-wise MAX over ranks of a list of floats (device-timed milliseconds)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return t.tolist()


def finish_hash(raw: int, expected: int | None = None) -> int:
    """R-MOD: the modulus is applied once, after the cross-rank sum."""
    return verify(raw, expected)
