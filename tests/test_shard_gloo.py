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


def _oracle_shard(net, depth, rank, world, roots):
    """A rank's build_spatial_tree_sharded result with the oracle standing in
    for the device builder (same cut, same root assignment, same level layout)."""
    from paper_2202_02444_b200.spatial import TreeArrays, TreeLevel

    cut = shard.first_cut(world, 2, depth)
    top = orc.tree_levels(net, -np.ones(3), np.ones(3), "affine-fixed", max_depth=cut)

    def level(l):
        blo, bhi = orc.bound_aabbs(net, l["lo"], l["hi"], "affine-fixed")
        return TreeLevel(l["lo"], l["hi"], blo, bhi, l["label"], l["face"], l["parent"])

    open_idx = np.flatnonzero(top[-1]["label"] == 0)
    if roots == "contiguous":
        root_ids = shard.split_frontier(np.arange(len(open_idx)), rank, world)
    else:
        root_ids = shard.interleaved_roots(len(open_idx), rank, world)
    part = open_idx[root_ids]
    sub = orc.tree_levels(net, top[-1]["lo"][part], top[-1]["hi"][part], "affine-fixed", max_depth=depth,
                          start_depth=cut) if part.size else []
    meta = dict(cut=cut, top=[level(l) for l in top], open_idx=open_idx, root_ids=np.asarray(root_ids),
                own_sub=bool(part.size), world=world)
    return TreeArrays([level(l) for l in sub] if sub else [level(l) for l in top], cut, meta=meta)


def _gather_worker(rank, world, port, depth, roots, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2202_02444_b200 import gather_camera_image, gather_spatial_tree

        net = orc.load_net(NET)
        tree = gather_spatial_tree(_oracle_shard(net, depth, rank, world, roots))
        # camera image: this rank's interleaved tiles with synthetic results
        w, h = 40, 24
        pix = np.concatenate([(np.arange(ty, min(ty + 16, h))[:, None] * w
                               + np.arange(tx, min(tx + 16, w))[None, :]).ravel()
                              for ty, tx in shard.pixel_tiles(w, h, 16, rank, world)])
        img = gather_camera_image(pix, pix % 3 == 0, np.where(pix % 3 == 0, pix * 0.5, np.inf), pix % 7,
                                  w * h)
        if rank == 0:
            out_q.put(([(l.lo, l.hi, l.label, l.face, l.parent) for l in tree.levels], img))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("roots", ["contiguous", "interleaved"])
def test_gather_sharded_tree_gloo(roots):
    """The final gather of a frontier-sharded build reproduces the unsharded
    tree in the reference's level order (AABBs, labels, faces, parents)."""
    depth, world = 9, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, depth, roots, q)) for r in range(world)]
    for p in procs:
        p.start()
    levels, (hit, t, steps) = q.get(timeout=600)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = orc.tree_levels(orc.load_net(NET), -np.ones(3), np.ones(3), "affine-fixed", max_depth=depth)
    assert len(levels) == len(full)
    for got, ref in zip(levels, full):
        for g, k in zip(got, ("lo", "hi", "label", "face", "parent")):
            if k == "parent" and ref["parent"][0] < 0:
                continue  # root
            np.testing.assert_array_equal(g, ref[k])
    idx = np.arange(40 * 24)
    np.testing.assert_array_equal(hit, idx % 3 == 0)
    np.testing.assert_array_equal(t, np.where(idx % 3 == 0, idx * 0.5, np.inf))
    np.testing.assert_array_equal(steps, idx % 7)


def test_subtree_keys_order():
    """Keys of two complete sub-trees interleave into the unsharded order."""
    # 2 roots, each split fully for 2 levels: level 1 = [lo(r0), lo(r1), hi(r0), hi(r1)]
    par1 = np.array([0, 0])
    k = shard.subtree_keys([None, par1], [1], 2)
    assert list(k[1]) == [1, 3]
    k0 = shard.subtree_keys([None, par1], [0], 2)
    assert sorted(list(k0[1]) + list(k[1])) == [0, 1, 2, 3]


# ---------------------------------------------------------------- C4 meshes
MESH_NET = os.path.join(os.path.dirname(__file__), "golden", "nets", "relu_sdf.json")


def _oracle_mesh_shard(net, m, rank, world):
    """A rank's extract_mesh_sharded result with the oracle standing in for
    the device kernels: its contiguous slice of the surviving blocks."""
    from paper_2202_02444_b200.meshing import MeshResult

    blocks, coords = orc.mesh_blocks(net, -np.ones(3), np.ones(3), m, 3, "affine-fixed")
    first, count = shard.shard_range(len(blocks), rank, world)
    builder = orc._Builder(coords)
    for blk in blocks[first:first + count]:
        orc._polygonize(builder, orc._grid_values(net, coords, blk), (blk[0][0], blk[1][0], blk[2][0]))
    v, t, k = builder.result()
    return MeshResult(v, t, k, count, meta={"block_first": first, "blocks_total": len(blocks)})


def test_merge_mesh_shards_single_process():
    """Shards merged in one process equal the unsharded extraction (arrays,
    first-visit vertex numbering)."""
    from paper_2202_02444_b200.meshing import merge_sharded_meshes

    net = orc.load_net(MESH_NET)
    want_v, want_t, want_k = orc.mesh_extract(net, -np.ones(3), np.ones(3), 5, 3, "affine-fixed")
    for world in (1, 3):
        got = merge_sharded_meshes([_oracle_mesh_shard(net, 5, r, world) for r in range(world)])
        np.testing.assert_array_equal(got.triangles, want_t)
        np.testing.assert_array_equal(got.vertex_keys, want_k)
        np.testing.assert_array_equal(got.vertices, want_v)


def _mesh_worker(rank, world, port, m, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2202_02444_b200.meshing import gather_mesh

        net = orc.load_net(MESH_NET)
        res = gather_mesh(_oracle_mesh_shard(net, m, rank, world), device="cpu")
        if rank == 0:
            out_q.put((res.vertices, res.triangles, res.vertex_keys))
    finally:
        dist.destroy_process_group()


def test_gather_mesh_gloo():
    """C4 mesh sharding: block slices per rank, one all_gather of edge-key
    triangles and vertex rows, global sort-unique dedup -> extract_mesh's arrays."""
    m, world = 5, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_mesh_worker, args=(r, world, port, m, q)) for r in range(world)]
    for p in procs:
        p.start()
    v, t, k = q.get(timeout=600)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want_v, want_t, want_k = orc.mesh_extract(orc.load_net(MESH_NET), -np.ones(3), np.ones(3), m, 3, "affine-fixed")
    np.testing.assert_array_equal(t, want_t)
    np.testing.assert_array_equal(k, want_k)
    np.testing.assert_array_equal(v, want_v)


# ---------------------------------------------------------------- rebalancing
def _oracle_segment(net, delta, cut, seg):
    """Capped segment build with the oracle standing in for the device:
    the full convergence subtree truncated to seg levels below the roots."""
    def build(lo, hi, j0):
        lv = orc.tree_levels(net, lo, hi, "affine-fixed", delta=delta, start_depth=cut + j0)[: seg + 1]
        return [(l["lo"], l["hi"], *orc.bound_aabbs(net, l["lo"], l["hi"], "affine-fixed"), l["label"], l["face"],
                 l["parent"]) for l in lv]
    return build


def _rebalance_worker(rank, world, port, delta, seg, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2202_02444_b200.spatial import TreeArrays, TreeLevel, gather_spatial_tree

        net = orc.load_net(NET)
        cut = 3
        top = orc.tree_levels(net, -np.ones(3), np.ones(3), "affine-fixed", max_depth=cut)
        open_idx = np.flatnonzero(top[-1]["label"] == 0)
        # deliberately unbalanced start: rank 0 takes every root
        mine = np.arange(len(open_idx)) if rank == 0 else np.zeros(0, np.int64)
        stop = delta / np.sqrt(3.0)
        packed, record = shard.refine_segmented(_oracle_segment(net, delta, cut, seg), top[-1]["lo"][open_idx[mine]],
                                                top[-1]["hi"][open_idx[mine]], mine, len(open_idx), seg, stop, cut,
                                                None, rank, world, imbalance=1.1)

        def level(l):
            blo, bhi = orc.bound_aabbs(net, l["lo"], l["hi"], "affine-fixed")
            return TreeLevel(l["lo"], l["hi"], blo, bhi, l["label"], l["face"], l["parent"])

        arr = TreeArrays([level(l) for l in top], 0,
                         meta=dict(cut=cut, top=[level(l) for l in top], open_idx=open_idx, packed=packed))
        tree = gather_spatial_tree(arr, device="cpu")
        if rank == 0:
            out_q.put(([(l.lo, l.hi, l.label, l.face, l.parent) for l in tree.levels], record))
    finally:
        dist.destroy_process_group()


def test_rebalanced_convergence_build_gloo():
    """Segmented refinement with frontier rebalancing (all_gather of the open
    nodes when max/mean > 1.1) from a maximally unbalanced start reproduces
    the unsharded convergence-mode tree node for node."""
    delta, seg, world = 0.08, 2, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rebalance_worker, args=(r, world, port, delta, seg, q)) for r in range(world)]
    for p in procs:
        p.start()
    levels, record = q.get(timeout=900)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert any(r["rebalanced"] for r in record)
    full = orc.tree_levels(orc.load_net(NET), -np.ones(3), np.ones(3), "affine-fixed", delta=delta)
    assert len(levels) == len(full)
    for got, ref in zip(levels, full):
        for g, k in zip(got, ("lo", "hi", "label", "face", "parent")):
            if k == "parent" and ref["parent"][0] < 0:
                continue
            np.testing.assert_array_equal(g, ref[k])
