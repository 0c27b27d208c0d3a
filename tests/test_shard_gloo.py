"""Multi-process (world_size 2, gloo, CPU) tests of the sharding host logic.

The GPU kernels are replaced by the oracle here (test infrastructure): each
rank refines its slice of the frontier with oracle.tree_levels, ranks
combine timings with shard.reduce_time_units (the helper bench.py uses) and
gather their levels; rank 0 checks that the union of the slices equals the
unsharded tree below the cut.
"""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import spelunk_oracle as orc
from paper_2202_02444_b200 import shard

NET = os.path.join(os.path.dirname(__file__), "golden", "nets", "relu4x32.json")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, depth, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        net = orc.load_net(NET)
        cut = shard.first_cut(world, 2, depth)
        top = orc.tree_levels(net, -np.ones(3), np.ones(3), "affine-fixed", max_depth=cut)
        last = top[-1]
        open_idx = np.flatnonzero(last["label"] == 0)
        mine = shard.split_frontier(open_idx, rank, world)
        sub = orc.tree_levels(net, last["lo"][mine], last["hi"][mine], "affine-fixed", max_depth=depth,
                              start_depth=cut) if mine.size else []
        own = sum(len(l["label"]) for l in sub[1:])
        units = own + (sum(len(l["label"]) for l in top) if rank == 0 else 0)
        t_max, u_sum = shard.reduce_time_units(0.1 * (rank + 1), units)
        gathered = [None] * world
        dist.all_gather_object(gathered, [
            np.concatenate([l["lo"], l["hi"], l["label"][:, None].astype(float)], axis=1) for l in sub[1:]
        ])
        if rank == 0:
            out_q.put((cut, t_max, u_sum, gathered))
    finally:
        dist.destroy_process_group()


def test_frontier_sharding_union_gloo():
    depth = 9
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, depth, q)) for r in range(world)]
    for p in procs:
        p.start()
    cut, t_max, u_sum, gathered = q.get(timeout=600)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = orc.tree_levels(orc.load_net(NET), -np.ones(3), np.ones(3), "affine-fixed", max_depth=depth)
    assert t_max == pytest.approx(0.2)
    assert u_sum == sum(len(l["label"]) for l in full)
    for d in range(cut + 1, depth + 1):
        got = [g[d - cut - 1] for g in gathered if len(g) > d - cut - 1]
        got = np.concatenate(got) if got else np.zeros((0, 7))
        ref = full[d]
        want = np.concatenate([ref["lo"], ref["hi"], ref["label"][:, None].astype(float)], axis=1)
        np.testing.assert_array_equal(np.unique(got, axis=0), np.unique(want, axis=0))


def test_shard_range_partition():
    for n in (0, 1, 7, 1000, 2 ** 24 + 3):
        for world in (1, 2, 3, 8):
            parts = [shard.shard_range(n, r, world) for r in range(world)]
            assert sum(c for _, c in parts) == n
            assert parts[0][0] == 0
            for (f0, c0), (f1, _) in zip(parts, parts[1:]):
                assert f1 == f0 + c0


def test_pixel_tiles_cover_image():
    tiles = [t for r in range(3) for t in shard.pixel_tiles(64, 48, 16, r, 3)]
    assert sorted(tiles) == sorted((y, x) for y in range(0, 48, 16) for x in range(0, 64, 16))
