"""GPU parity of the fused bound / point-evaluation kernels (K1, K2, K4)
against the pinned CPU oracle and the reference's golden vectors.

Tolerances (stated, not tuned per run):
  * FP64 kernels vs reference: |d| <= 1e-10 * S, S = max(1, |lo|, |hi|)
    (the reference allows last-ulp summation differences, range_core.py:552).
  * FP32 kernels: sound enclosures.  Every dense sample evaluated by the FP64
    oracle lies inside [lo, hi]; vs the reference |d| <= tau * (S + w),
    w = hi_ref - lo_ref, tau = 3e-3 for ReLU/ELU/tanh nets and 1e-2 for nets
    with sin (measured maxima 2.1e-3 -- 3x512 ReLU, tiny boxes, where the
    a-priori FMA rounding budget gamma * sum|W| |base| dominates the radius --
    and 3.8e-3: sin nets carry |pre-activations| ~ 100 whose FP32
    representation error is amplified by the slope of the linearisation).
  * Labels: where both sides are definite they are identical.
"""

import numpy as np
import pytest

import paper_2202_02444_b200 as sp
from oracle import spelunk_oracle as orc
from paper_2202_02444_b200 import synth

pytestmark = pytest.mark.gpu

GPU_POLICIES = ["interval", "affine-fixed"]


def tau32(net):
    kinds = {getattr(l, "value", l) for l in net.layers if not hasattr(l, "weights")}
    return 1e-2 if "sin" in kinds else 3e-3


@pytest.fixture(scope="module")
def nets(net_paths):
    return {k: sp.load_network(p) for k, p in net_paths.items()}


def scale(lo, hi):
    return np.maximum(1.0, np.maximum(np.abs(lo), np.abs(hi)))


def test_eval_fp64_matches_reference(golden, nets):
    for name, net in nets.items():
        x = golden[f"eval/{name}/x"]
        want = golden[f"eval/{name}/f"]
        got = sp.eval_batch(net, x, precision="fp64")
        assert np.max(np.abs(got - want) / scale(want, want)) <= 1e-12, name


def test_eval_fp32_close(golden, nets):
    for name, net in nets.items():
        x = golden[f"eval/{name}/x"]
        want = golden[f"eval/{name}/f"]
        got = sp.eval_batch(net, x, precision="fp32")
        assert np.max(np.abs(got - want) / scale(want, want)) <= 1e-4, name


def test_eval_batch_invariant(nets):
    net = nets["relu_sdf"]
    x = np.random.default_rng(3).uniform(-1, 1, (4097, 3))
    full = sp.eval_batch(net, x, precision="fp32")
    for n in (1, 2, 33, 1000, 4097):
        np.testing.assert_array_equal(sp.eval_batch(net, x[:n], precision="fp32"), full[:n])


@pytest.mark.parametrize("policy", GPU_POLICIES)
def test_bounds_fp64_match_reference(golden, nets, policy):
    for name, net in nets.items():
        c, a = golden[f"bounds/{name}/centers"], golden[f"bounds/{name}/axes"]
        lo, hi = sp.range_bound_batch(net, c, a, policy, precision="fp64")
        wl, wh = golden[f"bounds/{name}/{policy}/lo"], golden[f"bounds/{name}/{policy}/hi"]
        s = scale(wl, wh)
        assert np.max(np.abs(lo - wl) / s) <= 1e-10, name
        assert np.max(np.abs(hi - wh) / s) <= 1e-10, name


@pytest.mark.parametrize("policy", GPU_POLICIES)
def test_bounds_fp32_within_tolerance(golden, nets, policy):
    for name, net in nets.items():
        c, a = golden[f"bounds/{name}/centers"], golden[f"bounds/{name}/axes"]
        lo, hi = sp.range_bound_batch(net, c, a, policy, precision="fp32")
        wl, wh = golden[f"bounds/{name}/{policy}/lo"], golden[f"bounds/{name}/{policy}/hi"]
        tol = tau32(net) * (scale(wl, wh) + (wh - wl))
        assert np.all(np.abs(lo - wl) <= tol), (name, np.max(np.abs(lo - wl) / tol))
        assert np.all(np.abs(hi - wh) <= tol), (name, np.max(np.abs(hi - wh) / tol))
        # labels: never opposite-definite
        g = orc.sign_labels(lo, hi)
        r = orc.sign_labels(wl, wh)
        both = (g != 0) & (r != 0)
        np.testing.assert_array_equal(g[both], r[both])


def _sample_boxes(rng, c, a, k):
    eps = rng.uniform(-1.0, 1.0, (c.shape[0], k, a.shape[1]))
    return c[:, None, :] + np.einsum("nks,nsd->nkd", eps, a)


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
@pytest.mark.parametrize("policy", GPU_POLICIES)
def test_soundness_dense_samples(nets, policy, precision):
    """Zero dense-sample escapes, no slack beyond FP64 evaluation noise."""
    rng = np.random.default_rng(11)
    for name, net in nets.items():
        n = 512
        c = rng.uniform(-1.1, 1.1, (n, 3))
        sizes = 10.0 ** rng.uniform(-4, 0, n)
        a = np.zeros((n, 3, 3))
        one_d = rng.random(n) < 0.5
        a[:, np.arange(3), np.arange(3)] = (sizes / 2.0)[:, None]
        dirs = rng.standard_normal((n, 3))
        dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
        a[one_d] = 0.0
        a[one_d, 0, :] = (sizes[one_d, None] / 2.0) * dirs[one_d]
        lo, hi = sp.range_bound_batch(net, c, a, policy, precision=precision)
        pts = _sample_boxes(rng, c, a, 32)
        vals = orc.eval_points(orc.as_oracle_net(net), pts.reshape(-1, 3)).reshape(n, -1)
        slack = 1e-12 * scale(lo, hi)
        assert np.all(vals >= (lo - slack)[:, None]), name
        assert np.all(vals <= (hi + slack)[:, None]), name


def test_c1_grid_parity():
    """C1: 4x32 ReLU, affine-fixed over the uniform 64^3 grid, vs the oracle."""
    net = synth.config_net("C1")
    c, a = synth.grid_cubes(64)
    lo, hi, cls = sp.range_bound_batch(net, c, a, "affine-fixed", return_class=True)
    wl, wh = orc.bound_batch(orc.as_oracle_net(net), c, a, "affine-fixed", chunk=32768)
    tol = tau32(net) * (scale(wl, wh) + (wh - wl))
    assert np.all(np.abs(lo - wl) <= tol) and np.all(np.abs(hi - wh) <= tol)
    r = orc.sign_labels(wl, wh)
    both = (cls != 0) & (r != 0)
    np.testing.assert_array_equal(cls[both], r[both])
    np.testing.assert_array_equal(cls, orc.sign_labels(lo, hi))
    # FP32 may lose only a sliver of the reference's certifications
    assert (r != 0).sum() - ((cls != 0) & (r != 0)).sum() <= 0.01 * max(1, (r != 0).sum())


def test_aabb_path_equals_box_path(nets):
    import torch

    net = nets["relu_sdf"]
    rng = np.random.default_rng(5)
    lo_c = rng.uniform(-1, 0.9, (3000, 3))
    hi_c = lo_c + rng.uniform(1e-3, 0.1, (3000, 3))
    axes = np.zeros((3000, 3, 3))
    axes[:, np.arange(3), np.arange(3)] = (hi_c - lo_c) / 2.0
    want = sp.range_bound_batch(net, (lo_c + hi_c) / 2.0, axes, "affine-fixed")
    got = sp.bound_aabb(net, torch.from_numpy(lo_c).cuda(), torch.from_numpy(hi_c).cuda(), "affine-fixed")
    np.testing.assert_array_equal(got[0].cpu().numpy(), want[0])
    np.testing.assert_array_equal(got[1].cpu().numpy(), want[1])


def test_random_cubes_match_host_stream():
    net = synth.config_net("C5_64")
    n = 20000
    lo, hi, cls = sp.bound_random_cubes(net, n, seed=7, half=1 / 64, first_index=123)
    cen = synth.random_cube_centres(n, 7, 123)
    axes = np.zeros((n, 3, 3))
    axes[:, np.arange(3), np.arange(3)] = 1 / 64
    wl, wh = sp.range_bound_batch(net, cen, axes, "affine-fixed")
    np.testing.assert_array_equal(lo.cpu().numpy(), wl)
    np.testing.assert_array_equal(hi.cpu().numpy(), wh)


def test_device_tensor_path_matches_host(nets):
    import torch

    net = nets["elu_sdf"]
    rng = np.random.default_rng(9)
    c = rng.uniform(-1, 1, (777, 3))
    a = np.zeros((777, 3, 3))
    a[:, np.arange(3), np.arange(3)] = 0.02
    lo_h, hi_h = sp.range_bound_batch(net, c, a, "affine-fixed")
    lo_d, hi_d = sp.range_bound_batch(net, torch.from_numpy(c).cuda(), torch.from_numpy(a).cuda(), "affine-fixed")
    np.testing.assert_array_equal(lo_d.cpu().numpy(), lo_h)
    np.testing.assert_array_equal(hi_d.cpu().numpy(), hi_h)


def test_widths_and_activations_sweep():
    """Every compiled MMAX (32..512) and every activation, vs the oracle."""
    rng = np.random.default_rng(1)
    for width, act in ((48, "tanh"), (64, "relu"), (100, "elu"), (256, "sin"), (512, "relu")):
        net = synth.random_mlp(width, 3, act, "ref-normal", seed=width)
        c = rng.uniform(-1, 1, (300, 3))
        a = np.zeros((300, 3, 3))
        a[:, np.arange(3), np.arange(3)] = 10.0 ** rng.uniform(-3, -1, (300, 1))
        for policy in GPU_POLICIES:
            wl, wh = orc.bound_batch(orc.as_oracle_net(net), c, a, policy)
            lo, hi = sp.range_bound_batch(net, c, a, policy, precision="fp64")
            s = scale(wl, wh)
            assert np.max(np.abs(lo - wl) / s) <= 1e-10, (width, act, policy)
            lo32, hi32 = sp.range_bound_batch(net, c, a, policy, precision="fp32")
            tol = tau32(net) * (s + (wh - wl))
            assert np.all(np.abs(lo32 - wl) <= tol), (width, act, policy)
            assert np.all(np.abs(hi32 - wh) <= tol), (width, act, policy)


def test_errors_map_to_reference_exceptions(nets):
    net = nets["relu12"]
    with pytest.raises(sp.errors.DimensionMismatch):
        sp.range_bound_batch(net, np.zeros((4, 2)), np.zeros((4, 1, 2)), "affine-fixed")
    with pytest.raises(sp.errors.InvalidParameter):
        sp.range_bound_batch(net, np.zeros((4, 3)), np.zeros((4, 1, 3)), "bogus")
