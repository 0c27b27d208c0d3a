"""Pin the CPU oracle to vectors produced by the unmodified reference
(tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from oracle import spelunk_oracle as orc
from tests.conftest import golden_group

POLICIES = ["interval", "affine-fixed", "affine-full", "affine-truncate:8", "affine-truncate:16"]


def test_rules_match_reference(golden):
    lo, hi = golden["rules/lo"], golden["rules/hi"]
    for kind in ("relu", "elu", "sin", "tanh"):
        with np.errstate(all="ignore"):
            a, b, g = orc.LINEAR_RULES[kind](lo, hi)
            il, ih = orc.IMAGE_RULES[kind](lo, hi)
        np.testing.assert_array_equal(a, golden[f"rules/{kind}/alpha"])
        np.testing.assert_array_equal(b, golden[f"rules/{kind}/beta"])
        np.testing.assert_array_equal(g, golden[f"rules/{kind}/gamma"])
        np.testing.assert_array_equal(il, golden[f"rules/{kind}/ilo"])
        np.testing.assert_array_equal(ih, golden[f"rules/{kind}/ihi"])


def test_point_eval_bit_exact(golden, net_paths):
    for name, path in net_paths.items():
        net = orc.load_net(path)
        got = orc.eval_points(net, golden[f"eval/{name}/x"])
        np.testing.assert_array_equal(got, golden[f"eval/{name}/f"])


@pytest.mark.parametrize("policy", POLICIES)
def test_bounds_match_reference(golden, net_paths, policy):
    for name, path in net_paths.items():
        net = orc.load_net(path)
        c = golden[f"bounds/{name}/centers"]
        a = golden[f"bounds/{name}/axes"]
        lo, hi = orc.bound_batch(net, c, a, policy)
        want_lo = golden[f"bounds/{name}/{policy}/lo"]
        want_hi = golden[f"bounds/{name}/{policy}/hi"]
        scale = np.maximum(1.0, np.maximum(np.abs(want_lo), np.abs(want_hi)))
        assert np.max(np.abs(lo - want_lo) / scale) <= 1e-12, name
        assert np.max(np.abs(hi - want_hi) / scale) <= 1e-12, name


TREES = {
    "box_d8_fixed": ("box", dict(policy="affine-fixed", max_depth=8)),
    "box_conv_full": ("box", dict(policy="affine-full", delta=0.1)),
    "relu_sdf_d10_fixed": ("relu_sdf", dict(policy="affine-fixed", max_depth=10)),
    "relu_sdf_d7_interval": ("relu_sdf", dict(policy="interval", max_depth=7)),
    "relu4x32_d9_fixed": ("relu4x32", dict(policy="affine-fixed", max_depth=9)),
    "elu_sdf_conv_trunc": ("elu_sdf", dict(policy="affine-truncate:8", delta=0.15)),
    "relu_sdf_d7_full": ("relu_sdf", dict(policy="affine-full", max_depth=7)),
}


def golden_tree(golden, tag):
    g = golden_group(golden, f"tree/{tag}")
    n = 1 + max(int(k.split("/")[0]) for k in g)
    return [{f: g[f"{i}/{f}"] for f in ("keys", "lo", "hi", "sign", "face")} for i in range(n)]


@pytest.mark.parametrize("tag", sorted(TREES))
def test_tree_matches_reference(golden, net_paths, tag):
    netname, kw = TREES[tag]
    levels = orc.tree_levels(orc.load_net(net_paths[netname]), -np.ones(3), np.ones(3), **kw)
    keys = orc.node_keys(levels)
    want = golden_tree(golden, tag)
    assert len(levels) == len(want)
    for lv, k, w in zip(levels, keys, want):
        order = np.argsort(k)
        worder = np.argsort(w["keys"])
        np.testing.assert_array_equal(k[order], w["keys"][worder])
        np.testing.assert_array_equal(lv["label"][order], w["sign"][worder])
        np.testing.assert_array_equal(lv["face"][order], w["face"][worder])
        np.testing.assert_array_equal(lv["lo"][order], w["lo"][worder])
        np.testing.assert_array_equal(lv["hi"][order], w["hi"][worder])


@pytest.mark.parametrize("netname", ["box", "relu_sdf", "sin3x48"])
@pytest.mark.parametrize("policy", ["affine-fixed", "interval", "affine-truncate:8"])
def test_march_matches_reference(golden, net_paths, netname, policy):
    net = orc.load_net(net_paths[netname])
    p = orc.MarchParams(t_max=4.0)
    hit, t, steps = orc.march(net, golden[f"rays/{netname}/origins"], golden[f"rays/{netname}/dirs"], p, policy)
    np.testing.assert_array_equal(hit, golden[f"rays/{netname}/{policy}/hit"])
    np.testing.assert_array_equal(t, golden[f"rays/{netname}/{policy}/t"])
    np.testing.assert_array_equal(steps, golden[f"rays/{netname}/{policy}/steps"])


def test_camera_and_march(golden, net_paths):
    dirs = orc.pixel_dirs([1.6, 1.2, 2.0], [0, 0, 0], [0, 1, 0], 40.0, 24, 16)
    np.testing.assert_array_equal(dirs, golden["camera/dirs"])
    d = dirs.reshape(-1, 3)
    o = np.broadcast_to(np.array([1.6, 1.2, 2.0]), d.shape)
    hit, t, steps = orc.march(orc.load_net(net_paths["relu_sdf"]), o, d, orc.MarchParams(), "affine-fixed")
    np.testing.assert_array_equal(hit, golden["camera/relu_sdf/hit"])
    np.testing.assert_array_equal(t, golden["camera/relu_sdf/t"])
    np.testing.assert_array_equal(steps, golden["camera/relu_sdf/steps"])


def test_mc_tables(golden):
    flat = [(c, *tri) for c in range(256) for tri in orc.MC_TRIANGLES[c]]
    np.testing.assert_array_equal(np.array(flat), golden["mc/tri_table"])
    assert len(flat) == 820


MESHES = {
    "offset_box_m5_fixed": ("offset_box", 5, "affine-fixed"),
    "offset_box_m5_full": ("offset_box", 5, "affine-full"),
    "relu_sdf_m5_fixed": ("relu_sdf", 5, "affine-fixed"),
    "elu_sdf_m5_fixed": ("elu_sdf", 5, "affine-fixed"),
    "relu_sdf_m5_full": ("relu_sdf", 5, "affine-full"),
}


@pytest.mark.parametrize("tag", sorted(MESHES))
def test_mesh_matches_reference(golden, net_paths, tag):
    netname, m, pol = MESHES[tag]
    v, t, _ = orc.mesh_extract(orc.load_net(net_paths[netname]), -np.ones(3), np.ones(3), m, 3, pol)
    np.testing.assert_array_equal(v, golden[f"mesh/{tag}/vertices"])
    np.testing.assert_array_equal(t, golden[f"mesh/{tag}/triangles"])


def test_dense_mesh_matches_reference(golden, net_paths):
    v, t, _ = orc.mesh_extract_dense(orc.load_net(net_paths["relu_sdf"]), -np.ones(3), np.ones(3), 5)
    np.testing.assert_array_equal(v, golden["mesh/relu_sdf_m5_dense/vertices"])
    np.testing.assert_array_equal(t, golden["mesh/relu_sdf_m5_dense/triangles"])


def test_package_mc_tables_match_reference(golden):
    """The product's table generator (paper_2202_02444_b200/mc_tables.py)
    reproduces the reference's generated TRI_TABLE / EDGE_TABLE."""
    from paper_2202_02444_b200 import mc_tables

    flat = [(c, *tri) for c in range(256) for tri in mc_tables.TRI_TABLE[c]]
    np.testing.assert_array_equal(np.array(flat), golden["mc/tri_table"])
    np.testing.assert_array_equal(np.array(mc_tables.EDGE_TABLE), golden["mc/edge_table"])
    table, count = mc_tables.flat_tables()
    assert table.shape == (256, 15) and int(count.sum()) == 820


# cast_frustum_image cases in make_golden.py:gen_frustum
FRUSTA = {
    "box_front64": ("box", ([0.13, 0.11, 2.4], [0.02, -0.03, 0.0], [0.0, 1.0, 0.0], 40.0, 64, 64),
                    orc.MarchParams(t_max=4.0), 16),
    "relu_sdf_default48": ("relu_sdf", ([1.6, 1.2, 2.0], [0.0, 0.0, 0.0], [0.0, 1.0, 0.0], 40.0, 48, 32),
                           orc.MarchParams(), 8),
}


@pytest.mark.parametrize("tag", sorted(FRUSTA))
def test_frustum_cast_matches_reference(golden, net_paths, tag):
    netname, cam, params, grid = FRUSTA[tag]
    hit, t, steps = orc.frustum_cast(orc.load_net(net_paths[netname]), *cam, params, "affine-fixed", grid)
    np.testing.assert_array_equal(hit, golden[f"frustum/{tag}/hit"])
    np.testing.assert_array_equal(t, golden[f"frustum/{tag}/t"])
    np.testing.assert_array_equal(steps, golden[f"frustum/{tag}/steps"])


SDF_CAM = ([1.6, 1.2, 2.0], [0.0, 0.0, 0.0], [0.0, 1.0, 0.0], 40.0, 40, 24)
BOX_CAM = ([0.13, 0.11, 2.4], [0.02, -0.03, 0.0], [0.0, 1.0, 0.0], 40.0, 48, 48)
RENDERS = {
    "box_per_ray": ("box", BOX_CAM, orc.MarchParams(t_max=4.0), "per_ray", None),
    "box_frustum": ("box", BOX_CAM, orc.MarchParams(t_max=4.0), "frustum", None),
    "box_fixed": ("box", BOX_CAM, orc.MarchParams(t_max=4.0), "fixed_step", 0.01),
    "relu_sdf_per_ray": ("relu_sdf", SDF_CAM, orc.MarchParams(), "per_ray", None),
    "elu_sdf_fixed": ("elu_sdf", SDF_CAM, orc.MarchParams(t_max=5.0), "fixed_step", 0.02),
}


@pytest.mark.parametrize("tag", sorted(RENDERS))
def test_render_matches_reference(golden, net_paths, tag):
    netname, cam, params, mode, step = RENDERS[tag]
    img = orc.render(orc.load_net(net_paths[netname]), *cam, params, "affine-fixed", mode, step)
    np.testing.assert_array_equal(img, golden[f"render/{tag}/pixels"])


def test_ppm_bytes_and_round_trip(tmp_path):
    """write_image P6 layout (render.py:158-162) and read_ppm round trip."""
    from paper_2202_02444_b200.render import Image, read_ppm, write_image

    px = np.arange(2 * 3 * 3, dtype=np.uint8).reshape(2, 3, 3)
    write_image(Image(3, 2, px), tmp_path / "a.ppm")
    assert (tmp_path / "a.ppm").read_bytes() == b"P6\n3 2\n255\n" + px.tobytes()
    np.testing.assert_array_equal(read_ppm(tmp_path / "a.ppm").pixels, px)
    write_image(Image(3, 2, px), tmp_path / "a.png")
    assert (tmp_path / "a.png").read_bytes()[:8] == b"\x89PNG\r\n\x1a\n"


# ---- volumetric queries (make_golden.py:gen_queries) ----

def test_queries_radii_match_reference(golden, net_paths):
    box, sdf = orc.load_net(net_paths["box"]), orc.load_net(net_paths["relu_sdf"])
    pts, rin = golden["queries/ebr/box/points"], golden["queries/ebr/box/r_init"]
    got = [orc.certified_radii(box, p[None, :], [r], 0.001)[0] for p, r in zip(pts, rin)]
    np.testing.assert_array_equal(got, golden["queries/ebr/box/radius"])
    got = orc.certified_radii(sdf, golden["queries/radii/relu_sdf/points"], 1.0, 0.002)
    np.testing.assert_array_equal(got, golden["queries/radii/relu_sdf/radii"])


def test_queries_walk_and_sample_match_reference(golden, net_paths):
    box, sdf = orc.load_net(net_paths["box"]), orc.load_net(net_paths["relu_sdf"])
    m, se = orc.walk_on_spheres_stats(box, [0.2, 0.0, 0.0], lambda q: q[0], 300, rng_seed=0)
    np.testing.assert_array_equal([m, se], golden["queries/wos/box"])
    lo, hi = -np.ones(3), np.ones(3)
    np.testing.assert_array_equal(orc.sample_near_surface(box, lo, hi, 500, 0.01, 12, rng_seed=1),
                                  golden["queries/sample/box"])
    np.testing.assert_array_equal(orc.sample_near_surface(sdf, lo, hi, 300, 0.05, 7, rng_seed=2),
                                  golden["queries/sample/relu_sdf"])


def test_queries_bulk_intersection_closest_match_reference(golden, net_paths):
    box, sdf = orc.load_net(net_paths["box"]), orc.load_net(net_paths["relu_sdf"])
    lo, hi = -np.ones(3), np.ones(3)
    for tag, net, depth in (("box", box, 9), ("relu_sdf", sdf, 6)):
        mass, err, c, inertia = orc.bulk_properties(net, lo, hi, depth, rng_seed=0)
        np.testing.assert_array_equal(np.concatenate([[mass, err], c, inertia.reshape(-1)]),
                                      golden[f"queries/bulk/{tag}"])
    for tag, off, delta in (("overlap", 0.4, 0.01), ("disjoint", 2.0, 0.01), ("touch", 1.0, 0.05)):
        other = orc.as_oracle_net(build_box(np.array([off, 0.0, 0.0]), 0.5))
        top = 3.0 if tag == "disjoint" else 2.0
        kind, info = orc.test_intersection(box, other, np.full(3, -2.0), np.full(3, top), delta)
        assert ["disjoint", "intersecting", "inconclusive"].index(kind) == int(golden[f"queries/isect/{tag}/kind"])
        if kind == "intersecting":
            np.testing.assert_array_equal(np.concatenate(info), golden[f"queries/isect/{tag}/witness"])
        if kind == "inconclusive":
            np.testing.assert_array_equal(np.array([np.concatenate(n) for n in info]),
                                          golden[f"queries/isect/{tag}/nodes"])
    for tag, net in (("box", box), ("relu_sdf", sdf)):
        for q, want in zip(golden[f"queries/closest/{tag}/q"], golden[f"queries/closest/{tag}/result"]):
            p, dist = orc.closest_point(net, q, lo, hi, delta=0.01)
            np.testing.assert_array_equal(np.concatenate([p, [dist]]), want)


def build_box(center, half):
    from paper_2202_02444_b200.network import build_box_oracle

    return build_box_oracle(center, half)
