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


def interleaved_roots(n_open: int, rank: int, world: int) -> np.ndarray:
    """Positions (into the frontier) of this rank's roots when the cut frontier
    is dealt round-robin: spatially adjacent roots land on different ranks, so
    convergence-mode builds (whose refinement depth varies over space) stay
    balanced without a data-path collective."""
    return np.arange(rank, int(n_open), int(world), dtype=np.int64)


# --------------------------------------------------------------------------
# Final gather of a frontier-sharded tree.
#
# Level order of the unsharded tree (spatial.py:246-256, reproduced by the
# device builder): level k+1 lists the low children of level k's split nodes
# in level-k order, then their high children.  Below a cut whose split nodes
# (the roots) are numbered g = 0..R-1 in frontier order, the position of a
# node is therefore lexicographic in (b_j, b_{j-1}, ..., b_1, g) where b_i is
# its low/high choice i levels below the cut -- the integer
#     key_j = b_j * 2^(j-1) * R + key_{j-1}(parent),   key_0 = g.
# Every rank computes the keys of its own sub-tree; sorting the union of the
# ranks' level-j nodes by key gives the unsharded level j, and the parent of
# a node is the position of key mod 2^(j-1)R in level j-1.

def subtree_keys(parents, root_ids, n_roots: int):
    """Order keys of a sub-build's levels.  `parents[j]` is level j's parent
    index array (j >= 1; parents[0] is ignored), `root_ids` the global frontier
    positions of the sub-build's level-0 nodes."""
    keys = [np.asarray(root_ids, dtype=np.int64)]
    for j in range(1, len(parents)):
        par = np.asarray(parents[j], dtype=np.int64)
        k = len(par) // 2
        bit = np.zeros(len(par), dtype=np.int64)
        bit[k:] = 1
        keys.append(bit * ((1 << (j - 1)) * int(n_roots)) + keys[j - 1][par])
    return keys


def merge_shard_levels(parts, open_idx, n_fields_f64: int):
    """Merge the ranks' sub-tree levels into the unsharded levels below the cut.

    parts: per rank, a list over levels j = 1..J of (f64 rows (n, F), i64 rows
    (n, 3) = [key, label, face]).  open_idx: the cut level's split-node
    indices (frontier order; root g is node open_idx[g]).  Returns a list over
    j of (f64 rows, label, face, parent) in the unsharded order."""
    open_idx = np.asarray(open_idx, dtype=np.int64)
    n_roots = len(open_idx)
    depth = max((len(p) for p in parts), default=0)
    out = []
    prev_keys = None
    for j in range(1, depth + 1):
        fs = [p[j - 1][0] for p in parts if len(p) >= j]
        ks = [p[j - 1][1] for p in parts if len(p) >= j]
        f = np.concatenate(fs, axis=0) if fs else np.zeros((0, n_fields_f64))
        k = np.concatenate(ks, axis=0) if ks else np.zeros((0, 3), dtype=np.int64)
        order = np.argsort(k[:, 0], kind="stable")
        f, k = f[order], k[order]
        span = (1 << (j - 1)) * n_roots
        pkey = k[:, 0] % span
        if j == 1:
            parent = open_idx[pkey]
        else:
            parent = np.searchsorted(prev_keys, pkey)
        out.append((f, k[:, 1].astype(np.int8), k[:, 2].astype(np.int8), parent.astype(np.int64)))
        prev_keys = k[:, 0]
    return out


def allgather_rows(rows: np.ndarray, device=None):
    """all_gather of a per-rank (n_r, F) array with n_r varying by rank
    (sizes first, then one padded all_gather).  Returns the list over ranks."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size()
    rows = np.ascontiguousarray(rows)
    n = torch.tensor([rows.shape[0]], dtype=torch.int64, device=device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n)
    sizes = [int(s.item()) for s in sizes]
    cap = max(sizes) if sizes else 0
    t = torch.zeros((cap,) + rows.shape[1:], dtype=torch.from_numpy(rows[:0]).dtype, device=device)
    if rows.shape[0]:
        t[: rows.shape[0]] = torch.from_numpy(rows).to(device)
    bufs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(bufs, t)
    return [b[:s].cpu().numpy() for b, s in zip(bufs, sizes)]


# --------------------------------------------------------------------------
# Device-resident gathers (torch tensors end to end: NCCL over NVLink on GPUs
# -- the level arrays never leave HBM -- and the same code on CPU tensors with
# gloo).  Results equal the NumPy merge above.

def allgather_tensor(t, device=None):
    """all_gather of a per-rank (n_r, ...) tensor with n_r varying by rank:
    sizes first, then one padded all_gather on `device` (the collective's
    device: the rank's GPU for NCCL, "cpu" for gloo).  Returns the list over
    ranks, on `device`."""
    import torch
    import torch.distributed as dist

    dev = torch.device(device) if device is not None else t.device
    t = t.to(dev)
    world = dist.get_world_size()
    n = torch.tensor([t.shape[0]], dtype=torch.int64, device=dev)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n)
    sizes = [int(s.item()) for s in sizes]
    cap = max(sizes) if sizes else 0
    buf = torch.zeros((cap,) + tuple(t.shape[1:]), dtype=t.dtype, device=dev)
    if t.shape[0]:
        buf[: t.shape[0]] = t
    bufs = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(bufs, buf)
    return [b[:s] for b, s in zip(bufs, sizes)]


def subtree_keys_t(parents, root_ids, n_roots: int):
    """subtree_keys on torch tensors (int64, on the levels' device)."""
    import torch

    keys = [root_ids.to(torch.int64)]
    for j in range(1, len(parents)):
        par = parents[j].to(torch.int64)
        k = par.numel() // 2
        bit = torch.zeros_like(par)
        bit[k:] = 1
        keys.append(bit * ((1 << (j - 1)) * int(n_roots)) + keys[j - 1][par])
    return keys


def merge_shard_levels_t(parts, open_idx):
    """merge_shard_levels on torch tensors: per rank a list over levels j of
    (f64 rows (n, F), i64 rows (n, 3) = [key, label, face]); open_idx an int64
    tensor.  Stable key sort and searchsorted on the device."""
    import torch

    depth = max((len(p) for p in parts), default=0)
    out = []
    prev_keys = None
    n_roots = int(open_idx.numel())
    for j in range(1, depth + 1):
        fs = [p[j - 1][0] for p in parts if len(p) >= j]
        ks = [p[j - 1][1] for p in parts if len(p) >= j]
        f = torch.cat(fs, dim=0)
        k = torch.cat(ks, dim=0)
        order = torch.sort(k[:, 0], stable=True).indices
        f, k = f[order], k[order]
        span = (1 << (j - 1)) * n_roots
        pkey = k[:, 0] % span
        parent = open_idx[pkey] if j == 1 else torch.searchsorted(prev_keys, pkey)
        out.append((f, k[:, 1].to(torch.int8), k[:, 2].to(torch.int8), parent.to(torch.int64)))
        prev_keys = k[:, 0].contiguous()
    return out


# --------------------------------------------------------------------------
# Mesh shards (C4): contiguous slices of the surviving blocks in visiting
# order (spk_mesh_extract_shard).  Concatenated in rank order, the shards'
# triangles -- as edge-key triples -- are the unsharded triangle stream; the
# reference's _MeshBuilder numbers vertices by first visit and fixes a
# vertex's position at the first cell that visits its edge, so a global
# sort-unique on the edge keys with first occurrence (lowest rank, then the
# shard's own first visit) reproduces extract_mesh's arrays exactly.

def merge_mesh_parts_t(parts):
    """parts: per rank, in rank order, (tri_keys (T_r, 3) int64, vertex_keys
    (V_r,) int64, vertices (V_r, 3) f64) torch tensors on one device.
    Returns (vertices, triangles, vertex_keys) of the unsharded mesh."""
    import torch

    dev = parts[0][0].device if parts else torch.device("cpu")
    tk = torch.cat([p[0].reshape(-1, 3) for p in parts], dim=0) if parts else torch.zeros((0, 3), dtype=torch.int64)
    if tk.numel() == 0:
        return (torch.zeros((0, 3), dtype=torch.float64, device=dev), torch.zeros((0, 3), dtype=torch.int64, device=dev),
                torch.zeros(0, dtype=torch.int64, device=dev))

    def first_occurrence(x):
        uk, inv = torch.unique(x, return_inverse=True)
        pos = torch.arange(x.numel(), device=x.device)
        first = torch.full((uk.numel(),), x.numel(), dtype=torch.int64, device=x.device)
        first.scatter_reduce_(0, inv, pos, reduce="amin")
        return uk, inv, first

    flat = tk.reshape(-1)
    uk, inv, first = first_occurrence(flat)
    order = torch.argsort(first)                     # unique keys in first-visit order
    new_id = torch.empty_like(order)
    new_id[order] = torch.arange(order.numel(), device=dev)
    triangles = new_id[inv].reshape(-1, 3)
    vertex_keys = uk[order]
    vk = torch.cat([p[1].reshape(-1) for p in parts], dim=0)
    vp = torch.cat([p[2].reshape(-1, 3) for p in parts], dim=0)
    uk2, _, first2 = first_occurrence(vk)
    vertices = vp[first2][torch.searchsorted(uk2, vertex_keys)]
    return vertices, triangles, vertex_keys


# --------------------------------------------------------------------------
# Frontier rebalancing (segmented refinement below the cut).

def _order_keys(parents, root_keys, j0: int, n_roots: int):
    """Order keys of a segment's levels 1.. from its roots' keys (level j0 of
    the tree below the cut): key_j = b_j 2^(j-1) R + key_(j-1)(parent)."""
    keys = [np.asarray(root_keys, np.int64)]
    for l in range(1, len(parents)):
        j = j0 + l
        if (j - 1) + int(np.ceil(np.log2(max(2, n_roots)))) >= 62:
            raise OverflowError("tree too deep for 64-bit order keys")
        par = np.asarray(parents[l], np.int64)
        bit = np.zeros(len(par), np.int64)
        bit[len(par) // 2:] = 1
        keys.append(bit * ((1 << (j - 1)) * int(n_roots)) + keys[-1][par])
    return keys


def allgather_sizes(n: int, device=None):
    """Every rank's count (one small all_gather)."""
    import torch
    import torch.distributed as dist

    if device is None:
        device = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([int(n)], dtype=torch.int64, device=device)
    out = [torch.zeros_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return [int(x.item()) for x in out]


def rebalance_frontier(lo, hi, keys, sizes, rank: int, world: int):
    """Redistribute the open frontier evenly: one all_gather of every rank's
    (corners, key) rows -- NCCL over NVLink on GPUs -- and each rank keeps its
    contiguous slice of the concatenation (rank order).  Returns the new
    (lo, hi, keys)."""
    import torch

    d = lo.shape[1] if lo.ndim == 2 else 0
    rows = np.concatenate([lo, hi, keys[:, None].astype(np.float64)], axis=1) if len(keys) else \
        np.zeros((0, 2 * d + 1))
    # keys travel as exact integers inside FP64 rows (< 2^53 is checked)
    if len(keys) and int(keys.max()) >= (1 << 53):
        raise OverflowError("order key beyond 2^53")
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    allr = np.concatenate(allgather_rows(rows, dev), axis=0)
    total = allr.shape[0]
    first, count = shard_range(total, rank, world)
    mine = allr[first:first + count]
    return mine[:, :d].copy(), mine[:, d:2 * d].copy(), mine[:, 2 * d].astype(np.int64)


def refine_segmented(build_segment, lo, hi, root_keys, n_roots: int, segment_levels: int, stop: float,
                     cut: int, max_depth, rank: int, world: int, imbalance: float = 1.25):
    """Refine this rank's frontier below the cut in segments, rebalancing the
    open frontier between segments when max/mean > imbalance.

    build_segment(lo, hi, j0) -> levels [(lo, hi, bound_lo, bound_hi, label,
    face, parent)] of a capped build rooted at the given nodes (level 0 = the
    roots, at depth cut + j0).  Returns ((sizes per level j = 1..J, f rows,
    i rows [key, label, face]) in the gather's packed layout, record)."""
    import torch.distributed as dist

    distributed = dist.is_available() and dist.is_initialized() and world > 1
    lo = np.asarray(lo, np.float64)
    hi = np.asarray(hi, np.float64)
    d = lo.shape[1]
    keys = np.asarray(root_keys, np.int64)
    per_level = {}
    record = []
    j0 = 0
    while True:
        sizes = allgather_sizes(len(keys)) if distributed else [len(keys)]
        total = sum(sizes)
        if total == 0:
            break
        mean = total / len(sizes)
        moved = False
        if distributed and max(sizes) > imbalance * mean:
            lo, hi, keys = rebalance_frontier(lo, hi, keys, sizes, rank, world)
            moved = True
        record.append({"level": cut + j0, "sizes": sizes, "rebalanced": moved})
        if len(keys) == 0:
            lo, hi, keys = np.zeros((0, d)), np.zeros((0, d)), np.zeros(0, np.int64)
            j0 += segment_levels
            continue
        levels = build_segment(lo, hi, j0)
        lkeys = _order_keys([l[6] for l in levels], keys, j0, n_roots)
        for l in range(1, len(levels)):
            llo, lhi, blo, bhi, lab, face, _ = levels[l]
            f = np.concatenate([llo, lhi, blo[:, None], bhi[:, None]], axis=1)
            i = np.stack([lkeys[l], lab.astype(np.int64), face.astype(np.int64)], axis=1)
            per_level.setdefault(j0 + l, []).append((f, i))
        # the capped last level: nodes that would split are the next segment's roots
        if len(levels) == segment_levels + 1:
            llo, lhi, _, _, lab, _, _ = levels[-1]
            open_ = lab == 0
            if max_depth is None:
                open_ &= (lhi - llo).max(axis=1) >= stop
            else:
                open_ &= (cut + j0 + segment_levels) < max_depth
            lo, hi, keys = llo[open_], lhi[open_], lkeys[-1][open_]
        else:
            lo, hi, keys = np.zeros((0, d)), np.zeros((0, d)), np.zeros(0, np.int64)
        j0 += segment_levels
    J = max(per_level) if per_level else 0
    sizes, fs, is_ = [], [], []
    for j in range(1, J + 1):
        parts = per_level.get(j, [])
        f = np.concatenate([p[0] for p in parts], axis=0) if parts else np.zeros((0, 2 * d + 2))
        i = np.concatenate([p[1] for p in parts], axis=0) if parts else np.zeros((0, 3), np.int64)
        sizes.append(len(f))
        fs.append(f)
        is_.append(i)
    packed = (np.asarray(sizes, np.int64),
              np.concatenate(fs, axis=0) if fs else np.zeros((0, 2 * d + 2)),
              np.concatenate(is_, axis=0) if is_ else np.zeros((0, 3), np.int64))
    return packed, record
