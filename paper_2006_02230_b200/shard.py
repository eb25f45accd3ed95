"""Batch sharding across GPUs: one process per GPU, each rank
runs the tile engine on its own contiguous slice of the minibatch; the only
collectives are set-up (weights broadcast once) and measurement (max of the
per-rank device times).  Images are independent in a forward conv, so there is
no exchange step on the data path and no fused compute+collective kernel to
write.  The reference is single-node, single-socket OpenMP (the `img` loop is
its `parallel for`, Fig. 9); this is the same loop split across GPUs.

Works with any torch.distributed backend: NCCL on the B200 box, gloo in the
CPU tests (tests/test_shard.py, world_size 2).
"""
from __future__ import annotations

from typing import Iterable, Sequence


def shard_images(n_global: int, world: int, rank: int) -> tuple:
    """(start, count) of rank's contiguous slice; the first n % world ranks
    take one extra image, ranks beyond n_global get an empty slice."""
    if world < 1 or not 0 <= rank < world or n_global < 0:
        raise ValueError(f"bad shard request n={n_global} world={world} rank={rank}")
    base, extra = divmod(n_global, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def shard_table(n_global: int, world: int) -> list:
    return [shard_images(n_global, world, r) for r in range(world)]


def replicate_(tensors: Iterable, src: int = 0, group=None) -> None:
    """Make every rank's copy equal to rank `src`'s (in place)."""
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return
    for t in tensors:
        dist.broadcast(t, src, group=group)


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a per-rank scalar (device time of the timed region)."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def gather_images(local, n_global: int, group=None):
    """Concatenate the ranks' output slices along the image axis (validation
    only -- the benchmark never gathers).  Ragged slices are padded for the
    collective and trimmed afterwards."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return local
    world = dist.get_world_size(group)
    table = shard_table(n_global, world)
    cap = max(c for _, c in table)
    pad = torch.zeros((cap,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[:local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[:c] for p, (_, c) in zip(parts, table)], dim=0)
