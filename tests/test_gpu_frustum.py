"""§8(f1) frustum casting (spk_frustum_cast) vs the reference.

FP64: hit / t / amortised steps bit-identical to the reference's
cast_frustum_image (golden vectors, make_golden.py:gen_frustum) and to the
oracle restatement for the other policies.  Both precisions: the reference's
own acceptance contract (test_rays.py:222-256, test_acceptance.py:98-122) --
per-pixel-equal hit masks against per-ray casting except sub-delta slivers,
|dt| <= delta, strictly fewer total marching steps.
"""

import numpy as np
import pytest

import paper_2202_02444_b200 as sp
from oracle import spelunk_oracle as orc

pytestmark = pytest.mark.gpu

FRONT_CAM = dict(position=np.array([0.13, 0.11, 2.4]), look_at=np.array([0.02, -0.03, 0.0]),
                 up=np.array([0.0, 1.0, 0.0]), vertical_fov=40.0)
PARAMS = sp.RayCastParams(t_max=4.0)
DEFAULT_CAM = dict(position=np.array([1.6, 1.2, 2.0]), look_at=np.zeros(3), up=np.array([0.0, 1.0, 0.0]),
                   vertical_fov=40.0)


@pytest.fixture(scope="module")
def nets(net_paths):
    return {k: sp.load_network(p) for k, p in net_paths.items()}


def box_chords(origins, dirs, halfwidth=0.5):
    """Exact ray / cube chord lengths (0 for misses), slab intersection."""
    with np.errstate(divide="ignore", invalid="ignore"):
        t1 = (-halfwidth - origins) / dirs
        t2 = (halfwidth - origins) / dirs
    t_in = np.minimum(t1, t2).max(axis=1)
    t_out = np.maximum(t1, t2).min(axis=1)
    return np.maximum(t_out - np.maximum(t_in, 0.0), 0.0) * (t_out >= t_in)


CASES = {
    "box_front64": ("box", sp.Camera(resolution=(64, 64), **FRONT_CAM), PARAMS, 16),
    "relu_sdf_default48": ("relu_sdf", sp.Camera(resolution=(48, 32), **DEFAULT_CAM), sp.RayCastParams(), 8),
}


@pytest.mark.parametrize("tag", sorted(CASES))
def test_frustum_fp64_bit_exact(golden, nets, tag):
    netname, cam, params, grid = CASES[tag]
    fr = sp.cast_frustum_image(nets[netname], cam, params, "affine-fixed", initial_grid=grid, precision="fp64")
    np.testing.assert_array_equal(fr.hit, golden[f"frustum/{tag}/hit"])
    np.testing.assert_array_equal(fr.t, golden[f"frustum/{tag}/t"])
    np.testing.assert_array_equal(fr.steps, golden[f"frustum/{tag}/steps"])
    assert fr.stats.meta["frustum_steps"] > 0 and fr.stats.meta["pixel_handoffs"] > 0


@pytest.mark.parametrize("policy", ["interval", "affine-truncate:8"])
def test_frustum_fp64_other_policies_vs_oracle(nets, policy):
    cam = sp.Camera(resolution=(32, 32), **DEFAULT_CAM)
    fr = sp.cast_frustum_image(nets["relu_sdf"], cam, sp.RayCastParams(), policy, initial_grid=8, precision="fp64")
    hit, t, steps = orc.frustum_cast(orc.as_oracle_net(nets["relu_sdf"]), cam.position, cam.look_at, cam.up,
                                     cam.vertical_fov, 32, 32, orc.MarchParams(), policy, 8)
    np.testing.assert_array_equal(fr.hit, hit)
    np.testing.assert_array_equal(fr.t, t)
    np.testing.assert_array_equal(fr.steps, steps)


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("res", [64, 256])
def test_frustum_matches_per_ray(nets, precision, res):
    """Reference acceptance criterion, at its 256x256 size too."""
    box = nets["box"]
    cam = sp.Camera(resolution=(res, res), **FRONT_CAM)
    fr = sp.cast_frustum_image(box, cam, PARAMS, precision=precision)
    hit, t, steps, _ = sp.cast_camera(box, cam, PARAMS, "affine-fixed", precision="fp64")
    hit, t, steps = hit.cpu().numpy().reshape(-1), t.cpu().numpy().reshape(-1), steps.cpu().numpy().reshape(-1)
    dirs = cam.pixel_dirs().reshape(-1, 3)
    origins = np.broadcast_to(cam.position, dirs.shape)
    sliver = box_chords(origins, dirs) <= PARAMS.delta
    disagree = fr.hit.reshape(-1) != hit
    assert not np.any(disagree & ~sliver), int(np.sum(disagree & ~sliver))
    both = hit & fr.hit.reshape(-1)
    assert np.max(np.abs(fr.t.reshape(-1)[both] - t[both])) <= PARAMS.delta
    assert fr.total_steps() < steps.sum()


def test_frustum_empty_scene(nets):
    cam = sp.Camera(position=np.array([0.0, 0.0, 3.0]), look_at=np.array([0.0, 0.0, 6.0]),
                    up=np.array([0.0, 1.0, 0.0]), vertical_fov=40.0, resolution=(32, 32))
    fr = sp.cast_frustum_image(nets["box"], cam, PARAMS)
    assert not fr.hit.any() and np.all(np.isinf(fr.t))
    _, _, steps, _ = sp.cast_camera(nets["box"], cam, PARAMS)
    assert fr.total_steps() <= float(steps.sum())


def test_frustum_camera_on_surface(nets):
    cam = sp.Camera(position=np.array([0.5, 0.0, 0.0]), look_at=np.array([2.0, 0.0, 0.0]),
                    up=np.array([0.0, 1.0, 0.0]), vertical_fov=40.0, resolution=(16, 16))
    fr = sp.cast_frustum_image(nets["box"], cam, PARAMS)
    assert fr.hit.all() and np.all(fr.t == 0.0) and fr.total_steps() == 0.0


def test_frustum_indivisible_resolution(nets):
    cam = sp.Camera(resolution=(50, 50), **FRONT_CAM)
    with pytest.raises(sp.errors.InvalidCamera):
        sp.cast_frustum_image(nets["box"], cam, PARAMS)


def test_frustum_device_output_and_grid_one(nets):
    cam = sp.Camera(resolution=(24, 16), **DEFAULT_CAM)
    a = sp.cast_frustum_image(nets["relu_sdf"], cam, sp.RayCastParams(), initial_grid=1, device_output=True)
    b = sp.cast_frustum_image(nets["relu_sdf"], cam, sp.RayCastParams(), initial_grid=8)
    assert a.hit.is_cuda and a.t.shape == (16, 24)
    h = a.hit.cpu().numpy()
    # different initial grids change the frustum tree, not the contract
    both = h & b.hit
    assert np.max(np.abs(a.t.cpu().numpy()[both] - b.t[both]), initial=0.0) <= sp.RayCastParams().delta


def test_frustum_termination_guard_siren():
    """C3 SIREN (outputs ~1e-11): the FP32 bound cannot certify the camera
    point, so every t = 0 frustum dissolves into pixel hand-offs instead of
    looping; the per-ray contract still holds."""
    from paper_2202_02444_b200 import synth
    from paper_2202_02444_b200.camera import default_camera

    net = synth.config_net("C3")
    cam = default_camera(32)
    p = sp.RayCastParams()
    fr = sp.cast_frustum_image(net, cam, p, "affine-fixed", precision="fp32")
    assert fr.stats.meta["dissolved_frusta"] > 0
    hit, t, _, _ = sp.cast_camera(net, cam, p, "affine-fixed", precision="fp32")
    hit, t = hit.cpu().numpy(), t.cpu().numpy()
    np.testing.assert_array_equal(fr.hit, hit)
    assert np.max(np.abs(fr.t[hit] - t[hit]), initial=0.0) <= p.delta
