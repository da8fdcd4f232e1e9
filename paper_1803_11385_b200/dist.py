"""Data parallelism over whole shapes.

Every model of a super-PSH batch is an independent segment (psh_batch.hpp:24-29), so
a global batch of b shapes shards across G ranks as contiguous groups of whole
shapes; each rank builds its OWN super-PSH from its shapes (local M*/R*/N* prefix
arrays) and runs forward and input-gradient with no communication. The only
exchange is the weight gradient: dW_global = sum_r dW_r, one all-reduce (NCCL over
NVLink on the GPU path, gloo in the CPU tests). The reference scales the loss by the
GLOBAL batch size (net.cpp:281), so per-rank gradients are summed, never averaged.
"""
from __future__ import annotations

from typing import List, Sequence

import torch
import torch.distributed as dist


def shard_range(n_shapes: int, world: int, rank: int) -> range:
    """Contiguous, balanced block of shape indices owned by `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(n_shapes, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def local_levels(levels: Sequence, world: int, rank: int) -> List:
    """This rank's PshLevels of one pyramid level of the global batch (net.cpp:40-53
    build_batch, restricted to the rank's shapes)."""
    return [levels[i] for i in shard_range(len(levels), world, rank)]


def allreduce_gradients(grads: Sequence[torch.Tensor], group=None) -> None:
    """Sum weight gradients over ranks in place. All tensors are flattened into ONE
    bucket so the whole step costs a single collective (latency-bound at these sizes:
    a 64->64 3x3x3 layer's dW is 442 KB)."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return
    if len(grads) == 1:
        dist.all_reduce(grads[0], op=dist.ReduceOp.SUM, group=group)
        return
    flat = torch.cat([g.reshape(-1) for g in grads])
    dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    off = 0
    for g in grads:
        n = g.numel()
        g.copy_(flat[off:off + n].view_as(g))
        off += n


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a per-rank timing (multi-GPU numbers are the slowest rank's)."""
    if not dist.is_available() or not dist.is_initialized():
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def sum_over_ranks(t: torch.Tensor, group=None) -> None:
    """In-place sum over the data-parallel ranks (the NativeHashNet sync_bn hook: batch-norm
    statistics over the global batch). No-op without an initialised multi-rank group."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
