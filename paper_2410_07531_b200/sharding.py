"""Batch x head sharding of the dropout path across ranks.

The (b, h) slices are independent: rank r of n takes a contiguous slice range
and the Philox counter range that the global layout assigns to it
(base_offset + s0*SQ^2/4, element_source in mask.hpp:72-85), so the per-rank
masks concatenate byte-exactly to the single-device mask and no collective is
needed on the data path.  For weak-scaling replicas (bench.py) each rank runs
a whole block with its own disjoint counter range.
"""
from __future__ import annotations

from typing import Tuple


def shard_slices(batch: int, heads: int, seq: int, world: int, rank: int,
                 base_offset: int = 0) -> Tuple[int, int, int]:
    """(first slice, end slice, base_offset of the shard).  Requires
    batch*heads % world == 0 and the shard's first element to start a whole
    byte (s0*SQ^2 % 8 == 0) so the bytes concatenate."""
    slices = batch * heads
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    if slices % world:
        raise ValueError(f"{slices} (b,h) slices do not split over {world} ranks")
    per = slices // world
    s0 = rank * per
    if (s0 * seq * seq) % 8:
        raise ValueError("shard boundary is not byte aligned (SQ^2 * slices_per_rank % 8 != 0)")
    return s0, s0 + per, (base_offset + s0 * seq * seq // 4) & 0xFFFFFFFFFFFFFFFF


def replica_base_offset(batch: int, heads: int, seq: int, rank: int, base_offset: int = 0) -> int:
    """Counter base of replica `rank` when every rank runs a whole B x nH x SQ^2
    layout (weak scaling): replicas own consecutive, disjoint counter ranges."""
    return (base_offset + rank * (batch * heads * seq * seq // 4)) & 0xFFFFFFFFFFFFFFFF


def max_over_ranks(x: float, group=None) -> float:
    """Max of a per-rank scalar (the bench's timing rule); works on any backend."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return x
    dev = torch.device("cuda") if dist.get_backend(group) == "nccl" else torch.device("cpu")
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
