"""precision="fp32-refine" (SPK_FP32_REFINE): FP32 bounds, then the boxes the
FP32 pass leaves UNKNOWN within tau * (S + w) of certifying are re-bounded in
FP64 in place.

The FP32 rounding budget on deep nets costs certifications the reference
(FP64, range_core.py:547-642) makes -- e.g. 4.0% of the C5_64 cubes against
0.006% in plain FP32.  With the refinement the labels
are the reference's on every golden tree and on the C5 cubes, i.e. the
topology of every golden tree is the reference's (spatial.py:214-289), while
the bounds stay sound (FP32 or FP64, both contain the reference enclosure).
"""

import numpy as np
import pytest

import paper_2202_02444_b200 as sp
from oracle import spelunk_oracle as orc
from paper_2202_02444_b200 import spatial
from tests.test_gpu_configs import _c5_axes, config_net, gold  # noqa: F401  (fixture)
from tests.test_oracle_golden import TREES, golden_tree

pytestmark = pytest.mark.gpu
BOUNDS = spatial.AABB(-np.ones(3), np.ones(3))


def _labels_match_reference(onet, policy, got, want_sign, lo_ref, hi_ref, tol=1e-9):
    """Labels equal except where the reference certified a box whose exact
    range touches zero (its unrounded FP64 bound lands ulps on the definite
    side; the sound bound keeps it UNKNOWN): those must sit within tol of 0."""
    diff = np.flatnonzero(got != want_sign)
    if diff.size:
        assert np.all(got[diff] == 0), "refined labels certified a box the reference did not"
        near = np.minimum(np.abs(lo_ref[diff]), np.abs(hi_ref[diff]))
        assert np.all(near <= tol), near.max()
    return diff.size


# every golden tree: interval, affine-fixed, affine-truncate, affine-full
# (the symbol-carrying policies re-bound their candidates with the FP64
# symbolic kernels), fixed-depth and convergence-mode builds
REFINED_TREES = dict(TREES)


@pytest.mark.parametrize("tag", sorted(REFINED_TREES))
def test_refined_tree_equals_reference(golden, net_paths, tag):
    netname, kw = REFINED_TREES[tag]
    net = sp.load_network(net_paths[netname])
    onet = orc.as_oracle_net(net)
    policy = kw["policy"]
    want = golden_tree(golden, tag)
    arr = spatial.build_spatial_tree_arrays(net, BOUNDS, precision="fp32-refine", **kw)
    plain = spatial.build_spatial_tree_arrays(net, BOUNDS, precision="fp32", **kw)
    touching = 0
    for lv, k, w in zip(arr.levels, arr.keys(), want):
        common, ia, ib = np.intersect1d(k, w["keys"], return_indices=True)
        np.testing.assert_array_equal(lv.lo[ia], w["lo"][ib])
        a, b = lv.label[ia], w["sign"][ib]
        blo, bhi = orc.bound_aabbs(onet, w["lo"][ib], w["hi"][ib], policy)
        touching += _labels_match_reference(onet, policy, a, b, blo, bhi)
        # refined bounds contain the reference's enclosure where the FP32 rules
        # are inclusion-monotone (fused policies on these ReLU fixtures; FP32
        # truncation may keep other symbols than FP64 -- sound, not nested)
        if policy in ("affine-fixed", "interval"):
            s = np.maximum(1.0, np.maximum(np.abs(blo), np.abs(bhi)))
            assert np.all(lv.bound_lo[ia] <= blo + 1e-12 * s) and np.all(lv.bound_hi[ia] >= bhi - 1e-12 * s)
    if touching == 0:
        assert [len(l) for l in arr.levels] == [len(w["keys"]) for w in want], "topology"
    n_plain = sum(len(l) for l in plain.levels)
    print(f"{tag}: refined tree {arr.n_nodes} nodes (reference {sum(len(w['keys']) for w in want)}, "
          f"plain FP32 {n_plain}); touching-zero differences {touching}")


@pytest.mark.parametrize("tagnet", ["C5_64", "C5_512"])
@pytest.mark.parametrize("policy", ["affine-fixed", "interval"])
def test_refined_c5_labels_equal_reference(gold, tagnet, policy):  # noqa: F811
    net = config_net(gold, tagnet)
    c = gold["C5/centres"]
    wl, wh = gold[f"{tagnet}/{policy}/lo"], gold[f"{tagnet}/{policy}/hi"]
    ref = np.where(wl > 0, 1, np.where(wh < 0, -1, 0)).astype(np.int8)
    s = np.maximum(1.0, np.maximum(np.abs(wl), np.abs(wh)))
    lo, hi, cls = sp.bound_random_cubes(net, len(c), seed=5, half=1.0 / 64, policy=policy, precision="fp32-refine")
    lo, hi, cls = lo.cpu().numpy(), hi.cpu().numpy(), cls.cpu().numpy()
    assert np.all(lo <= wl + 1e-12 * s) and np.all(hi >= wh - 1e-12 * s), "sound"
    _labels_match_reference(None, policy, cls, ref, wl, wh)
    p_lo, p_hi, p_cls = sp.bound_random_cubes(net, len(c), seed=5, half=1.0 / 64, policy=policy)
    p_cls = p_cls.cpu().numpy()
    # boxes plain FP32 certifies keep their FP32 bounds bit for bit
    cert = p_cls != 0
    np.testing.assert_array_equal(lo[cert], p_lo.cpu().numpy()[cert])
    band = sp.net_refine_band(net, policy)
    assert 0.0 <= band <= 0.25
    print(f"{tagnet} {policy}: band {band:.3e}; certified ref {(ref != 0).mean():.4f} refined {(cls != 0).mean():.4f} "
          f"plain fp32 {cert.mean():.4f}")
    # the same through the host-array API (range_bound_batch, spk_bound_batch_host)
    hlo, hhi, hcls = sp.range_bound_batch(net, c, _c5_axes(len(c)), policy, precision="fp32-refine",
                                          return_class=True)
    np.testing.assert_array_equal(hcls, cls)


def test_refine_band_semantics(gold):  # noqa: F811
    """tau = 0 refines only boxes touching zero; a huge tau refines every
    UNKNOWN box, whose bounds then equal the FP64 kernels' bit for bit, while
    the boxes FP32 certifies keep their FP32 bounds."""
    net = config_net(gold, "C5_64")
    c = gold["C5/centres"]
    ax = _c5_axes(len(c))
    prev = sp.refine_band()
    assert prev == -1.0  # per-net calibration by default
    try:
        assert sp.refine_band(1e30) == -1.0
        assert sp.refine_band() == 1e30
        lo, hi, cls = sp.range_bound_batch(net, c, ax, "affine-fixed", precision="fp32-refine", return_class=True)
        lo32, hi32, cls32 = sp.range_bound_batch(net, c, ax, "affine-fixed", precision="fp32", return_class=True)
        lo64, hi64, cls64 = sp.range_bound_batch(net, c, ax, "affine-fixed", precision="fp64", return_class=True)
        u = cls32 == 0
        np.testing.assert_array_equal(lo[u], lo64[u])
        np.testing.assert_array_equal(hi[u], hi64[u])
        np.testing.assert_array_equal(lo[~u], lo32[~u])
        sp.refine_band(0.0)
        lo0, hi0, cls0 = sp.range_bound_batch(net, c, ax, "affine-fixed", precision="fp32-refine", return_class=True)
        keep = (lo32 != 0.0) & (hi32 != 0.0)
        np.testing.assert_array_equal(lo0[keep], lo32[keep])
        with pytest.raises(sp.errors.InvalidParameter):
            sp.refine_band(float("nan"))
        assert sp.refine_band("auto") == 0.0
        assert sp.refine_band() == -1.0
    finally:
        sp.refine_band("auto")


@pytest.mark.parametrize("policy", ["affine-truncate:8", "affine-truncate:40", "affine-full"])
def test_refine_symbolic_policies(net_paths, policy):
    """fp32-refine with the symbol-carrying kernels (K3 register tile for
    truncate:8, K3F for truncate:40 and affine-full on the 7x32 fixture): with
    an all-covering band every UNKNOWN box is re-bounded through the FP64
    kernels' processing order -- bit-identical to their own bounds -- and the
    boxes FP32 certifies keep their FP32 bounds."""
    net = sp.load_network(net_paths["relu_sdf"])
    rng = np.random.default_rng(4)
    n = 3000
    c = rng.uniform(-1, 1, (n, 3))
    ax = np.zeros((n, 3, 3))
    ax[:, np.arange(3), np.arange(3)] = rng.uniform(0.005, 0.08, (n, 1))
    prev = sp.refine_band(1e30)
    try:
        lo, hi, cls = sp.range_bound_batch(net, c, ax, policy, precision="fp32-refine", return_class=True)
    finally:
        sp.refine_band("auto") if prev < 0 else sp.refine_band(prev)
    lo32, hi32, cls32 = sp.range_bound_batch(net, c, ax, policy, precision="fp32", return_class=True)
    lo64, hi64, cls64 = sp.range_bound_batch(net, c, ax, policy, precision="fp64", return_class=True)
    u = cls32 == 0
    assert u.any() and (~u).any()
    np.testing.assert_array_equal(lo[u], lo64[u])
    np.testing.assert_array_equal(hi[u], hi64[u])
    np.testing.assert_array_equal(lo[~u], lo32[~u])
    # and with the calibrated band the labels are the FP64 kernels'
    lo_c, hi_c, cls_c = sp.range_bound_batch(net, c, ax, policy, precision="fp32-refine", return_class=True)
    np.testing.assert_array_equal(cls_c, cls64)
