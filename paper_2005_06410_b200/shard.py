"""Batch sharding of the convolution across GPUs (one process per GPU).

The batch index is the outermost (slowest) dimension of both I (h_i x w_i x c_i x b)
and O (k_n x h_o x w_o x b) (tensor.hpp:28-50), so a contiguous batch range of I
maps to a contiguous batch range of O and each rank's shard is an independent
convolution -- no data-path collective. Shards follow the reference's static
split (threads.hpp:20-25: contiguous ranges, the first count % n ranks take one
extra). Filters are replicated once with a broadcast before any timed work.
"""
from __future__ import annotations

from dataclasses import replace


def split_range(count: int, rank: int, nranks: int) -> tuple[int, int]:
    """convgemm::split_range (threads.hpp:20-25)."""
    if nranks < 1 or not 0 <= rank < nranks:
        raise ValueError("rank out of range")
    base, rem = divmod(count, nranks)
    begin = rank * base + min(rank, rem)
    return begin, begin + base + (1 if rank < rem else 0)


def shard_params(cp, rank: int, world: int):
    """(b0, b1, cp_local): this rank's batch range and its ConvParams (b = b1 - b0).
    Ranks with an empty range get b0 == b1 and cp_local None."""
    from . import ConvParams
    cp = ConvParams.of(cp)
    b0, b1 = split_range(cp.b, rank, world)
    return b0, b1, (replace(cp, b=b1 - b0) if b1 > b0 else None)


def batch_slice(t, b0: int, b1: int):
    """Batch range [b0, b1) of a leftmost-fastest rank-4 tensor: a view (no copy)."""
    return t[..., b0:b1]


def broadcast_filters(F, src: int = 0):
    """Replicate the filters from `src` to every rank (outside any timed region).
    F is a leftmost-fastest rank-4 CUDA tensor; its storage is broadcast in place."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.broadcast(F.permute(3, 2, 1, 0), src=src)
    return F


def max_over_ranks(value: float, device=None) -> float:
    """Job time = the slowest rank (timed on each device, reduced across ranks)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
