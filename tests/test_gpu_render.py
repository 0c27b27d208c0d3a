"""§8(f2) rendering (spk_render_shade / spk_fixed_step_march) vs the reference.

FP64 end to end: the rendered images equal the reference's render_image
(golden vectors, make_golden.py:gen_render) in every mode -- identical hit
masks, and gray levels identical up to a +-1 rounding tie on at most 0.5% of
the hit pixels (the FP64 point kernel agrees with the reference's einsum to
~1e-12, not to the last bit, and the 48-step bisection and the
central-difference normal amplify that into the last gray level only at
rint ties).  FP32 marching keeps the reference's per-pixel contract: hit
masks equal except sub-delta silhouette slivers.
"""

import numpy as np
import pytest

import paper_2202_02444_b200 as sp
from paper_2202_02444_b200.render import BACKGROUND

pytestmark = pytest.mark.gpu

FRONT_CAM = dict(position=np.array([0.13, 0.11, 2.4]), look_at=np.array([0.02, -0.03, 0.0]),
                 up=np.array([0.0, 1.0, 0.0]), vertical_fov=40.0)
SDF_CAM = sp.Camera(np.array([1.6, 1.2, 2.0]), np.zeros(3), np.array([0.0, 1.0, 0.0]), 40.0, (40, 24))
BOX_CAM = sp.Camera(resolution=(48, 48), **FRONT_CAM)
CASES = {
    "box_per_ray": ("box", BOX_CAM, sp.RayCastParams(t_max=4.0), "per_ray", None),
    "box_frustum": ("box", BOX_CAM, sp.RayCastParams(t_max=4.0), "frustum", None),
    "box_fixed": ("box", BOX_CAM, sp.RayCastParams(t_max=4.0), "fixed_step", 0.01),
    "relu_sdf_per_ray": ("relu_sdf", SDF_CAM, sp.RayCastParams(), "per_ray", None),
    "elu_sdf_fixed": ("elu_sdf", SDF_CAM, sp.RayCastParams(t_max=5.0), "fixed_step", 0.02),
}


@pytest.fixture(scope="module")
def nets(net_paths):
    return {k: sp.load_network(p) for k, p in net_paths.items()}


def hit_mask(px):
    return np.any(px != BACKGROUND, axis=-1)


@pytest.mark.parametrize("tag", sorted(CASES))
def test_render_fp64_matches_reference(golden, nets, tag):
    netname, cam, params, mode, step = CASES[tag]
    img = sp.render_image(nets[netname], cam, params, sp.AFFINE_FIXED, mode, step, precision="fp64")
    want = golden[f"render/{tag}/pixels"]
    assert img.pixels.shape == want.shape and img.pixels.dtype == np.uint8
    np.testing.assert_array_equal(hit_mask(img.pixels), hit_mask(want))
    diff = np.abs(img.pixels.astype(int) - want.astype(int)).max(axis=-1)
    assert diff.max() <= 1
    assert np.count_nonzero(diff) <= max(1, 0.005 * hit_mask(want).sum())


def box_chords(origins, dirs, halfwidth=0.5):
    with np.errstate(divide="ignore", invalid="ignore"):
        t1 = (-halfwidth - origins) / dirs
        t2 = (halfwidth - origins) / dirs
    t_in = np.minimum(t1, t2).max(axis=1)
    t_out = np.maximum(t1, t2).min(axis=1)
    return np.maximum(t_out - np.maximum(t_in, 0.0), 0.0) * (t_out >= t_in)


@pytest.mark.parametrize("mode", ["per_ray", "frustum"])
def test_render_fp32_march_contract(golden, nets, mode):
    img = sp.render_image(nets["box"], BOX_CAM, sp.RayCastParams(t_max=4.0), sp.AFFINE_FIXED, mode,
                          precision="fp32")
    want = golden[f"render/box_{mode}/pixels"]
    dirs = BOX_CAM.pixel_dirs().reshape(-1, 3)
    sliver = (box_chords(np.broadcast_to(BOX_CAM.position, dirs.shape), dirs) <= 1e-3).reshape(48, 48)
    got_m, want_m = hit_mask(img.pixels), hit_mask(want)
    assert not np.any((got_m != want_m) & ~sliver)
    both = got_m & want_m
    diff = np.abs(img.pixels.astype(int) - want.astype(int)).max(axis=-1)[both]
    assert np.mean(diff <= 1) >= 0.99


def test_render_modes_and_errors(nets):
    cam = sp.Camera(resolution=(16, 16), **FRONT_CAM)
    with pytest.raises(sp.errors.InvalidParameter):
        sp.render_image(nets["box"], cam, sp.RayCastParams(t_max=4.0), mode="fixed_step")
    with pytest.raises(sp.errors.InvalidParameter):
        sp.render_image(nets["box"], cam, sp.RayCastParams(t_max=4.0), mode="bogus")
    # a camera looking away: all background
    away = sp.Camera(position=np.array([0.0, 0.0, 3.0]), look_at=np.array([0.0, 0.0, 6.0]),
                     up=np.array([0.0, 1.0, 0.0]), vertical_fov=40.0, resolution=(8, 8))
    img = sp.render_image(nets["box"], away, sp.RayCastParams(t_max=4.0))
    assert np.all(img.pixels == BACKGROUND)


def test_fixed_step_matches_oracle(nets):
    from oracle import spelunk_oracle as orc
    from paper_2202_02444_b200.render import fixed_step_march

    cam = sp.Camera(resolution=(24, 24), **FRONT_CAM)
    hit, t, rounds = fixed_step_march(nets["box"], cam, 0.013, sp.RayCastParams(t_max=4.0), precision="fp64")
    dirs = cam.pixel_dirs().reshape(-1, 3)
    h2, t2 = orc.fixed_step_march(orc.as_oracle_net(nets["box"]), np.broadcast_to(cam.position, dirs.shape).copy(),
                                  dirs, 0.013, 4.0)
    np.testing.assert_array_equal(hit.cpu().numpy().astype(bool), h2)
    np.testing.assert_array_equal(t.cpu().numpy(), t2)
    assert rounds > 0
