"""A trained net of the headline shape (3->8x256->1 ReLU torus SDF,
synth.trained_net; tools/train_sdf_net.py) against golden vectors from the
unmodified reference (tests/golden/make_golden_trained.py).

The random-init BASELINE nets certify (almost) nothing, so they cannot show
what the FP32 rounding budget costs in labels; this net certifies 61% of the
1/256 cubes in the reference.  FP64 kernels reproduce the reference's labels
and tree; plain FP32 bounds contain the reference's enclosure and agree on
every box both certify; precision="fp32-refine" gives the reference's labels.
"""

from pathlib import Path

import numpy as np
import pytest

import paper_2202_02444_b200 as sp
from paper_2202_02444_b200 import spatial, synth

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden" / "trained.npz"
BOUNDS = spatial.AABB(-np.ones(3), np.ones(3))


@pytest.fixture(scope="module")
def gold():
    with np.load(GOLD) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="module")
def net():
    return synth.trained_net("torus")


def _labels(lo, hi):
    return np.where(lo > 0, 1, np.where(hi < 0, -1, 0)).astype(np.int8)


def _check_labels(got, ref, wl, wh, tol=1e-9):
    """Equal except boxes the reference certifies with a bound within tol of
    zero (the sound bound may keep those UNKNOWN)."""
    diff = np.flatnonzero(got != ref)
    if diff.size:
        assert np.all(got[diff] == 0), "certified a box the reference did not"
        assert np.all(np.minimum(np.abs(wl[diff]), np.abs(wh[diff])) <= tol)
    return diff.size


@pytest.mark.parametrize("h", [64, 256])
def test_trained_cubes(gold, net, h):
    c = gold["cubes/centres"]
    wl, wh = gold[f"cubes/{h}/lo"], gold[f"cubes/{h}/hi"]
    ref = _labels(wl, wh)
    s = np.maximum(1.0, np.maximum(np.abs(wl), np.abs(wh)))
    axes = np.zeros((len(c), 3, 3))
    axes[:, np.arange(3), np.arange(3)] = 1.0 / h
    got = {}
    for prec in ("fp64", "fp32", "fp32-refine"):
        lo, hi, cls = sp.range_bound_batch(net, c, axes, sp.AFFINE_FIXED, precision=prec, return_class=True)
        assert np.all(lo <= wl + 1e-12 * s) and np.all(hi >= wh - 1e-12 * s), f"{prec}: contains the reference"
        got[prec] = cls
        if prec == "fp64":
            assert np.max(np.abs(lo - wl) / s) <= 1e-8
    _check_labels(got["fp64"], ref, wl, wh)
    _check_labels(got["fp32-refine"], ref, wl, wh)
    both = (got["fp32"] != 0) & (ref != 0)
    np.testing.assert_array_equal(got["fp32"][both], ref[both])
    rate = {k: float((v != 0).mean()) for k, v in got.items()}
    print(f"torus 1/{h} cubes: certified reference {(ref != 0).mean():.4f}, fp64 {rate['fp64']:.4f}, "
          f"fp32 {rate['fp32']:.4f}, fp32-refine {rate['fp32-refine']:.4f}")


@pytest.mark.parametrize("policy", ["affine-fixed", "interval"])
def test_trained_tree(gold, net, policy):
    """build_spatial_tree to depth 10: FP64 and fp32-refine give the
    reference's tree (AABBs and labels, level by level); FP64 bounds within
    1e-8 S of the reference's, FP32 / refined bounds contain them."""
    want = []
    k = 0
    while f"tree/{policy}/{k}/lo" in gold:
        want.append({n: gold[f"tree/{policy}/{k}/{n}"] for n in ("lo", "hi", "label", "bound_lo", "bound_hi")})
        k += 1
    for prec in ("fp64", "fp32-refine", "fp32"):
        arr = spatial.build_spatial_tree_arrays(net, BOUNDS, policy=policy, max_depth=10, precision=prec,
                                                to_host=True)
        if prec != "fp32":
            assert arr.n_levels == len(want)
        for lv, w in zip(arr.levels, want):
            if prec != "fp32" or len(lv.lo) == len(w["lo"]):
                np.testing.assert_array_equal(lv.lo, w["lo"])
                np.testing.assert_array_equal(lv.hi, w["hi"])
                S = np.maximum(1.0, np.maximum(np.abs(w["bound_lo"]), np.abs(w["bound_hi"])))
                assert np.all(lv.bound_lo <= w["bound_lo"] + 1e-12 * S)
                assert np.all(lv.bound_hi >= w["bound_hi"] - 1e-12 * S)
                if prec == "fp64":
                    assert np.max(np.abs(lv.bound_lo - w["bound_lo"]) / S) <= 1e-8
                if prec != "fp32":
                    _check_labels(lv.label, w["label"], w["bound_lo"], w["bound_hi"])


def test_trained_sharded_refine_equals_unsharded(net):
    """fp32-refine through the sharded builder: every rank's net calibrates the
    same band and each node's bound is independent of its batch, so the
    merged shards equal the unsharded refined tree array for array."""
    full = spatial.build_spatial_tree_arrays(net, BOUNDS, policy=sp.AFFINE_FIXED, max_depth=20,
                                             precision="fp32-refine", to_host=True)
    world = 4
    parts = [spatial.build_spatial_tree_sharded(net, BOUNDS, 20, sp.AFFINE_FIXED, r, world, precision="fp32-refine",
                                                min_roots_per_rank=2, to_host=True, roots="interleaved")
             for r in range(world)]
    merged = spatial.merge_sharded_trees(parts)
    assert merged.n_nodes == full.n_nodes and sum(int((lv.label != 0).sum()) for lv in full.levels) > 0
    for d, (g, f) in enumerate(zip(merged.levels, full.levels)):
        for k in ("lo", "hi", "bound_lo", "bound_hi", "label"):
            np.testing.assert_array_equal(getattr(g, k), getattr(f, k), err_msg=f"{k} at depth {d}")


def test_host_mirror_equals_device_levels(net):
    """The host mirror (to_host=True; the last level's AABBs and parents copied
    while its bounds compute, in sections sized by the level's capacity, which
    certification leaves larger than its count) equals the device levels."""
    kw = dict(policy=sp.AFFINE_FIXED, max_depth=19)
    host = spatial.build_spatial_tree_arrays(net, BOUNDS, to_host=True, **kw)
    dev = spatial.build_spatial_tree_arrays(net, BOUNDS, to_host=False, **kw)
    assert sum(int((lv.label != 0).sum().item()) for lv in dev.levels) > 0  # certification: capacity > count
    assert host.n_levels == dev.n_levels
    for d, (h, g) in enumerate(zip(host.levels, dev.levels)):
        for k in ("lo", "hi", "bound_lo", "bound_hi", "label", "face", "parent"):
            np.testing.assert_array_equal(getattr(h, k), getattr(g, k).cpu().numpy(), err_msg=f"{k} at depth {d}")
