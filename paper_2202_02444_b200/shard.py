"""Sharding of the hot path across GPUs (one process per GPU).

Boxes, rays and frontier nodes are independent, so no collective runs in
any inner loop; torch.distributed is used only to combine
timings/counts (max of times, sum of units) and, optionally, to gather
results.  These helpers hold the host-side logic so it can be tested on CPU
with the gloo backend.
"""

from __future__ import annotations

import numpy as np


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [first, first+count) slice of n units for `rank` (C5 boxes)."""
    base, extra = divmod(int(n), int(world))
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


def split_frontier(open_idx, rank: int, world: int) -> np.ndarray:
    """Contiguous slice of the UNKNOWN frontier (tree) for `rank`."""
    return np.array_split(np.asarray(open_idx), world)[rank]


def first_cut(world: int, min_roots_per_rank: int, max_depth: int) -> int:
    """Depth at which an all-UNKNOWN binary frontier first holds
    >= min_roots_per_rank * world nodes (2^d nodes at depth d)."""
    target = max(1, min_roots_per_rank * world)
    return min(max_depth, int(np.ceil(np.log2(target))))


def pixel_tiles(width: int, height: int, tile: int, rank: int, world: int):
    """Interleaved tile assignment for ray casting: tile i -> rank i mod world."""
    tiles = [(ty, tx) for ty in range(0, height, tile) for tx in range(0, width, tile)]
    return tiles[rank::world]


def reduce_time_units(local_time: float, local_units: float, device=None):
    """(max over ranks of time, sum over ranks of units); identity when not distributed."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return float(local_time), float(local_units)
    t = torch.tensor([float(local_time)], dtype=torch.float64, device=device)
    u = torch.tensor([float(local_units)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(u, op=dist.ReduceOp.SUM)
    return float(t.item()), float(u.item())
