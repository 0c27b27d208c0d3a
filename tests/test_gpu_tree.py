"""K5 tree build on the GPU vs the reference's golden trees and the oracle.

FP64 kernels: topology, AABBs (bit-exact), labels and face annotations equal
the reference's.  FP32 kernels: on the common subtree (nodes present in both
trees, matched by path key) AABBs are bit-identical and labels agree wherever
both are definite; every node FP32 certifies is checked by dense sampling.
"""

import numpy as np
import pytest

import paper_2202_02444_b200 as sp
from oracle import spelunk_oracle as orc
from paper_2202_02444_b200 import spatial
from tests.test_oracle_golden import TREES, golden_tree

pytestmark = pytest.mark.gpu
BOUNDS = spatial.AABB(-np.ones(3), np.ones(3))
GPU_TREES = dict(TREES)


def by_key(keys, *arrays):
    order = np.argsort(keys)
    return (keys[order],) + tuple(a[order] for a in arrays)


@pytest.mark.parametrize("tag", sorted(GPU_TREES))
def test_tree_fp64_equals_reference(golden, net_paths, tag):
    """FP64: identical topology, AABBs, labels and face annotations -- except
    where the reference certified a node whose exact range touches zero (its
    unrounded FP64 bound lands a few ulps on the definite side; the sound
    GPU bound keeps the node UNKNOWN and splits it).  Such nodes must have
    |oracle bound| <= 1e-9 and only their sub-trees may differ."""
    netname, kw = GPU_TREES[tag]
    net = sp.load_network(net_paths[netname])
    arr = spatial.build_spatial_tree_arrays(net, BOUNDS, precision="fp64", **kw)
    want = golden_tree(golden, tag)
    onet = orc.as_oracle_net(net)
    policy = kw["policy"]
    touching = 0
    for lv, k, w in zip(arr.levels, arr.keys(), want):
        common, ia, ib = np.intersect1d(k, w["keys"], return_indices=True)
        np.testing.assert_array_equal(lv.lo[ia], w["lo"][ib])
        np.testing.assert_array_equal(lv.hi[ia], w["hi"][ib])
        a, b = lv.label[ia], w["sign"][ib]
        diff = np.flatnonzero(a != b)
        if diff.size:
            assert np.all(a[diff] == 0), "GPU certified a node the reference did not"
            blo, bhi = orc.bound_aabbs(onet, w["lo"][ib][diff], w["hi"][ib][diff], policy)
            near = np.minimum(np.abs(blo), np.abs(bhi))
            assert np.all(near <= 1e-9), near.max()
            touching += diff.size
        same = a == b
        np.testing.assert_array_equal(lv.face[ia][same], w["face"][ib][same])
    if touching == 0:
        assert len(arr.levels) == len(want)
        assert [len(l) for l in arr.levels] == [len(w["keys"]) for w in want]
    print(f"{tag}: FP64 touching-zero label differences {touching}")


@pytest.mark.parametrize("tag", sorted(GPU_TREES))
def test_tree_fp32_common_subtree(golden, net_paths, tag):
    netname, kw = GPU_TREES[tag]
    net = sp.load_network(net_paths[netname])
    arr = spatial.build_spatial_tree_arrays(net, BOUNDS, precision="fp32", **kw)
    want = golden_tree(golden, tag)
    rng = np.random.default_rng(0)
    onet = orc.as_oracle_net(net)
    mism = 0
    for lv, k, w in zip(arr.levels, arr.keys(), want):
        common, ia, ib = np.intersect1d(k, w["keys"], return_indices=True)
        np.testing.assert_array_equal(lv.lo[ia], w["lo"][ib])
        np.testing.assert_array_equal(lv.hi[ia], w["hi"][ib])
        a, b = lv.label[ia], w["sign"][ib]
        both = (a != 0) & (b != 0)
        np.testing.assert_array_equal(a[both], b[both])
        mism += int(np.sum(a != b))
        # soundness of FP32 certifications
        cert = np.flatnonzero(lv.label != 0)[:200]
        if cert.size:
            pts = rng.uniform(lv.lo[cert][:, None, :], lv.hi[cert][:, None, :], (cert.size, 16, 3))
            vals = orc.eval_points(onet, pts.reshape(-1, 3)).reshape(cert.size, -1)
            sign = lv.label[cert][:, None]
            assert np.all(np.where(sign > 0, vals > 0, vals < 0))
    print(f"{tag}: FP32 label mismatches on common subtree {mism}")


def test_tree_materialize_matches_reference_api(net_paths):
    net = sp.load_network(net_paths["box"])
    root = spatial.build_spatial_tree(net, BOUNDS, policy=sp.AFFINE_FIXED, max_depth=6)
    depths = [l.depth for l in spatial.iter_leaves(root)]
    assert max(depths) == 6
    vol = sum(l.aabb.volume for l in spatial.iter_leaves(root))
    assert abs(vol - 8.0) <= 1e-9
    for leaf in spatial.iter_leaves(root):
        if leaf.depth < 6:
            assert leaf.sign is not sp.SignClass.UNKNOWN


def test_tree_convergence_mode_interval(golden, net_paths):
    """Convergence mode with face annotations vs the oracle (interval policy)."""
    net = sp.load_network(net_paths["box"])
    arr = spatial.build_spatial_tree_arrays(net, BOUNDS, delta=0.1, policy="interval", precision="fp64")
    levels = orc.tree_levels(orc.as_oracle_net(net), -np.ones(3), np.ones(3), "interval", delta=0.1)
    okeys = orc.node_keys(levels)
    assert len(arr.levels) == len(levels)
    for lv, k, ol, ok in zip(arr.levels, arr.keys(), levels, okeys):
        k1, lab, face = by_key(k, lv.label, lv.face)
        k2, wl, wf = by_key(ok, ol["label"], ol["face"])
        np.testing.assert_array_equal(k1, k2)
        np.testing.assert_array_equal(lab, wl)
        np.testing.assert_array_equal(face, wf)


def test_depth_overflow(net_paths):
    net = sp.load_network(net_paths["box"])
    with pytest.raises(sp.errors.DepthOverflow):
        spatial.build_spatial_tree(net, BOUNDS, max_depth=61)


def test_sharded_union_equals_full(net_paths):
    """Frontier sharding: the union of 4 ranks' sub-trees = the full tree."""
    net = sp.load_network(net_paths["relu4x32"])
    full = spatial.build_spatial_tree_arrays(net, BOUNDS, policy="affine-fixed", max_depth=9)
    fk = full.keys()
    world = 4
    parts = [spatial.build_spatial_tree_sharded(net, BOUNDS, 9, "affine-fixed", r, world, min_roots_per_rank=2, to_host=True)
             for r in range(world)]
    cut = parts[0].meta["cut"]
    for depth in range(cut + 1, 10):
        got = []
        for p in parts:
            if "top_levels" not in p.meta or depth - cut >= len(p.levels):
                continue
            # keys of a shard are relative to its roots; compare labels+AABBs as sets
            lv = p.levels[depth - cut]
            got.append(np.concatenate([lv.lo, lv.hi, lv.label[:, None].astype(float)], axis=1))
        got = np.concatenate(got) if got else np.zeros((0, 7))
        ref = full.levels[depth]
        want = np.concatenate([ref.lo, ref.hi, ref.label[:, None].astype(float)], axis=1)
        assert got.shape == want.shape
        np.testing.assert_array_equal(np.unique(got, axis=0), np.unique(want, axis=0))


@pytest.mark.parametrize("roots,world,precision", [("contiguous", 4, "fp32"), ("interleaved", 3, "fp64"),
                                                   ("interleaved", 8, "fp32")])
def test_sharded_merge_equals_full(net_paths, roots, world, precision):
    """Final gather (merge_sharded_trees, the local form of gather_spatial_tree):
    the merged shards equal the unsharded device tree array-for-array, in the
    reference's level order -- AABBs, bounds, labels, faces, parents."""
    net = sp.load_network(net_paths["relu4x32"])
    full = spatial.build_spatial_tree_arrays(net, BOUNDS, policy="affine-fixed", max_depth=10,
                                             precision=precision)
    parts = [spatial.build_spatial_tree_sharded(net, BOUNDS, 10, "affine-fixed", r, world, precision=precision,
                                                min_roots_per_rank=2, to_host=True, roots=roots)
             for r in range(world)]
    merged = spatial.merge_sharded_trees(parts)
    assert merged.n_levels == full.n_levels and merged.n_nodes == full.n_nodes
    for d, (g, f) in enumerate(zip(merged.levels, full.levels)):
        for k in ("lo", "hi", "bound_lo", "bound_hi", "label", "face"):
            np.testing.assert_array_equal(getattr(g, k), getattr(f, k), err_msg=f"{k} at depth {d}")
        if d:
            np.testing.assert_array_equal(g.parent, f.parent, err_msg=f"parent at depth {d}")


@pytest.mark.parametrize("policy", ["affine-fixed", "interval"])
def test_live_row_skipping_is_exact(policy):
    """Live-row masks skip all-zero (ReLU-inactive) X rows of a box group.
    The tree bounds its levels in sibling-pair order (coherent box groups,
    many rows skipped); bounding the same AABBs in level order pairs
    unrelated boxes (other rows skipped).  Skipping exact zeros must not
    change a single bit of the FP32 bounds, and the tree must stay the
    reference's topology."""
    import torch

    from paper_2202_02444_b200 import synth

    net = synth.random_mlp(256, 6, "relu", "torch-uniform", seed=5)
    arr = spatial.build_spatial_tree_arrays(net, BOUNDS, policy=policy, max_depth=12, precision="fp32",
                                            to_host=True)
    for d in range(1, arr.n_levels):
        lv = arr.levels[d]
        lo, hi, _ = sp.bound_aabb(net, torch.from_numpy(lv.lo).cuda(), torch.from_numpy(lv.hi).cuda(), policy)
        np.testing.assert_array_equal(lo.cpu().numpy(), lv.bound_lo, err_msg=f"lo at depth {d}")
        np.testing.assert_array_equal(hi.cpu().numpy(), lv.bound_hi, err_msg=f"hi at depth {d}")
    # and an odd-sized batch (no pair order possible) through the same kernels
    lv = arr.levels[-1]
    m = len(lv) - 1
    lo, hi, _ = sp.bound_aabb(net, torch.from_numpy(lv.lo[:m]).cuda(), torch.from_numpy(lv.hi[:m]).cuda(), policy)
    np.testing.assert_array_equal(lo.cpu().numpy(), lv.bound_lo[:m])


@pytest.mark.parametrize("policy", ["affine-fixed", "interval"])
def test_processing_orders_are_exact(policy):
    """The small tile, spread, natural and Morton processing orders all give
    bit-identical FP32 bounds: each box is bounded on its own, skipped rows
    are exact zeros, and every tile shape sums in the same k order."""
    import torch

    from paper_2202_02444_b200 import synth

    net = synth.random_mlp(256, 5, "relu", "torch-uniform", seed=9)
    rng = np.random.default_rng(4)
    n_big = 70_000  # >= 65,536: Morton order
    c = rng.uniform(-1, 1, (n_big, 3))
    h = 10.0 ** rng.uniform(-3, -1, (n_big, 1))
    lo_t, hi_t = torch.from_numpy(c - h).cuda(), torch.from_numpy(c + h).cuda()
    big_lo, big_hi, _ = sp.bound_aabb(net, lo_t, hi_t, policy)
    # small tile, spread, natural order (vs the Morton-ordered big batch)
    for a, b in ((0, 300), (1000, 1900), (5000, 12000)):
        lo, hi, _ = sp.bound_aabb(net, lo_t[a:b], hi_t[a:b], policy)
        np.testing.assert_array_equal(lo.cpu().numpy(), big_lo[a:b].cpu().numpy())
        np.testing.assert_array_equal(hi.cpu().numpy(), big_hi[a:b].cpu().numpy())


@pytest.mark.parametrize("netname", ["c1", "relu_sdf"])
def test_narrow_warp_live_masks_are_exact(net_paths, netname):
    """Width-32 nets skip X rows that are zero for every box a warp computes
    (the union of its box groups' masks).  A batch sorted along z (coherent
    warps, many rows skipped) and the same boxes in a random permutation
    (incoherent warps, few skipped) must give bit-identical bounds."""
    import torch

    from paper_2202_02444_b200 import synth

    net = synth.config_net("C1") if netname == "c1" else sp.load_network(net_paths[netname])
    rng = np.random.default_rng(11)
    n = 50_000
    c = rng.uniform(-1, 1, (n, 3))
    c = c[np.argsort(c[:, 2])]
    h = 10.0 ** rng.uniform(-3, -1.5, (n, 1))
    perm = rng.permutation(n)
    for policy in ("affine-fixed", "interval"):
        lo_a, hi_a, _ = sp.bound_aabb(net, torch.from_numpy(c - h).cuda(), torch.from_numpy(c + h).cuda(), policy)
        lo_b, hi_b, _ = sp.bound_aabb(net, torch.from_numpy(c[perm] - h[perm]).cuda(),
                                      torch.from_numpy(c[perm] + h[perm]).cuda(), policy)
        np.testing.assert_array_equal(lo_b.cpu().numpy(), lo_a.cpu().numpy()[perm])
        np.testing.assert_array_equal(hi_b.cpu().numpy(), hi_a.cpu().numpy()[perm])


@pytest.mark.parametrize("mode", ["convergence", "fixed"])
def test_segmented_build_equals_unsharded(net_paths, mode):
    """The rebalancing builder refines in capped segments (SPK_TREE_LEVEL_CAP)
    and reassembles by order key: in one process (no rebalancing needed) the
    gathered tree equals the unsharded build array for array."""
    net = sp.load_network(net_paths["relu_sdf"])
    b = spatial.AABB(-np.ones(3), np.ones(3))
    kw = dict(delta=0.02, max_depth=None) if mode == "convergence" else dict(delta=1.0, max_depth=9)
    full = spatial.build_spatial_tree_arrays(net, b, policy=sp.AFFINE_FIXED, precision="fp64", to_host=True, **kw)
    arr = spatial.build_spatial_tree_rebalanced(net, b, 0, 1, policy=sp.AFFINE_FIXED, precision="fp64",
                                                min_roots_per_rank=16, segment_levels=3, **kw)
    got = spatial.gather_spatial_tree(arr, device="cpu")
    assert got.n_levels == full.n_levels
    for g, f in zip(got.levels, full.levels):
        for k in ("lo", "hi", "bound_lo", "bound_hi", "label", "face"):
            np.testing.assert_array_equal(np.asarray(getattr(g, k)), np.asarray(getattr(f, k)))
        if len(f) and f.parent[0] >= 0:
            np.testing.assert_array_equal(np.asarray(g.parent), np.asarray(f.parent))


def test_fp64_live_masks_are_exact():
    """FP64 width-256 tiles skip X rows that are zero for both boxes of a box
    group (16-row W tiles, round 2).  Coherent sibling-like batches (many rows
    skipped) and the same boxes permuted (dense tiles) must give bit-identical
    FP64 bounds, and those match the oracle."""
    import torch

    from oracle import spelunk_oracle as orc
    from paper_2202_02444_b200 import synth

    net = synth.random_mlp(256, 4, "relu", "torch-uniform", seed=5)
    rng = np.random.default_rng(12)
    n = 20_000
    c = rng.uniform(-1, 1, (n, 3))
    c = c[np.lexsort((c[:, 0], c[:, 1], np.round(c[:, 2] * 8)))]
    h = np.full((n, 1), 1.0 / 128)
    perm = rng.permutation(n)
    for policy in ("affine-fixed", "interval"):
        lo_a, hi_a, _ = sp.bound_aabb(net, torch.from_numpy(c - h).cuda(), torch.from_numpy(c + h).cuda(), policy,
                                      precision="fp64")
        lo_b, hi_b, _ = sp.bound_aabb(net, torch.from_numpy(c[perm] - h[perm]).cuda(),
                                      torch.from_numpy(c[perm] + h[perm]).cuda(), policy, precision="fp64")
        lo_a, hi_a = lo_a.cpu().numpy(), hi_a.cpu().numpy()
        np.testing.assert_array_equal(lo_b.cpu().numpy(), lo_a[perm])
        np.testing.assert_array_equal(hi_b.cpu().numpy(), hi_a[perm])
        sel = rng.choice(n, 256, replace=False)
        axes = np.zeros((256, 3, 3))
        axes[:, np.arange(3), np.arange(3)] = 1.0 / 128
        wl, wh = orc.bound_batch(orc.as_oracle_net(net), c[sel], axes, policy)
        s = np.maximum(1.0, np.maximum(np.abs(wl), np.abs(wh)))
        assert np.all(np.abs(lo_a[sel] - wl) <= 1e-10 * s) and np.all(np.abs(hi_a[sel] - wh) <= 1e-10 * s)
