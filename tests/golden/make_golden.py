"""Generate the golden vectors that pin the oracle to the real reference.

Runs ONLY in the build container, where the unmodified reference package is
importable from /root/reference/pkg/src (override with SPELUNK_REF_SRC).
Everything it writes lands in tests/golden/ and is committed, so the GPU box
never needs the reference:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Inputs are seeded; nets are written with the reference's own save_network so
both sides load bit-identical weights.
"""

from __future__ import annotations

import json
import os
import shutil
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_SRC = os.environ.get("SPELUNK_REF_SRC", "/root/reference/pkg/src")
REF_FIXTURES = Path(REF_SRC).parent / "tests" / "fixtures"
sys.path.insert(0, REF_SRC)
sys.dont_write_bytecode = True

import spelunk as sp  # noqa: E402  (the reference)
from spelunk import mc_tables  # noqa: E402
from spelunk.network import ActivationKind, DenseLayer, NetworkSpec  # noqa: E402
from spelunk.range_core import AFFINE_RULES, INTERVAL_RULES  # noqa: E402
from spelunk.rays import _march_arrays  # noqa: E402

NETS = HERE / "nets"
OFFSET = np.array([0.031, 0.017, -0.023])


def random_mlp(rng, hidden, activation, scale=1.0, d=3):
    """Reference conftest recipe (tests/conftest.py:43-61)."""
    layers = []
    dims = [d, *hidden, 1]
    for i in range(len(dims) - 1):
        w = rng.standard_normal((dims[i + 1], dims[i])) * (scale / np.sqrt(dims[i]))
        b = rng.standard_normal(dims[i + 1]) * 0.1
        layers.append(DenseLayer(w, b))
        if i < len(dims) - 2:
            layers.append(activation)
    return NetworkSpec(d, tuple(layers), "sdf", "random_mlp")


def make_nets():
    NETS.mkdir(exist_ok=True)
    rng = np.random.default_rng(2024)
    nets = {
        "box": sp.build_box_oracle(np.zeros(3), 0.5),
        "offset_box": sp.build_box_oracle(OFFSET, 0.5),
        "relu12": random_mlp(rng, (12, 12), ActivationKind.RELU),
        "elu12": random_mlp(rng, (12, 12), ActivationKind.ELU),
        "sin12": random_mlp(rng, (12, 12), ActivationKind.SIN),
        "tanh12": random_mlp(rng, (12, 12), ActivationKind.TANH),
        "wide_sin": random_mlp(rng, (6,), ActivationKind.SIN, scale=8.0),
        "relu4x32": random_mlp(rng, (32, 32, 32, 32), ActivationKind.RELU),
        "sin3x48": random_mlp(rng, (48, 48, 48), ActivationKind.SIN, scale=3.0),
    }
    for name, net in nets.items():
        sp.save_network(net, NETS / f"{name}.json")
    for name in ("relu_sdf", "elu_sdf"):
        shutil.copyfile(REF_FIXTURES / f"{name}.json", NETS / f"{name}.json")
        nets[name] = sp.load_network(NETS / f"{name}.json")
    return nets


def random_boxes(rng, n, d=3):
    """Oriented boxes, s in 1..3 (zero-row padded), log-uniform sizes."""
    centers = rng.uniform(-1.1, 1.1, (n, d))
    axes = np.zeros((n, d, d))
    for i in range(n):
        s = int(rng.integers(1, d + 1))
        q, _ = np.linalg.qr(rng.standard_normal((d, d)))
        half = 10.0 ** rng.uniform(-3.5, -0.3, s)
        axes[i, :s] = q[:, :s].T * half[:, None]
    return centers, axes


POLICIES = ["interval", "affine-fixed", "affine-full", "affine-truncate:8", "affine-truncate:16"]


def gen_bounds(nets, out):
    rng = np.random.default_rng(7)
    for name, net in nets.items():
        c, a = random_boxes(rng, 48)
        # axis-aligned cubes too (tree / mesh boxes)
        cc = rng.uniform(-1, 1, (16, 3))
        half = 10.0 ** rng.uniform(-3, -0.5, 16)
        ca = np.zeros((16, 3, 3))
        ca[:, np.arange(3), np.arange(3)] = half[:, None]
        centers = np.concatenate([c, cc])
        axes = np.concatenate([a, ca])
        out[f"bounds/{name}/centers"] = centers
        out[f"bounds/{name}/axes"] = axes
        for pol in POLICIES:
            lo, hi = sp.range_bound_batch(net, centers, axes, sp.parse_policy(pol))
            out[f"bounds/{name}/{pol}/lo"] = lo
            out[f"bounds/{name}/{pol}/hi"] = hi
        pts = rng.uniform(-1.2, 1.2, (257, 3))
        out[f"eval/{name}/x"] = pts
        out[f"eval/{name}/f"] = sp.eval_batch(net, pts)


def gen_rules(out):
    rng = np.random.default_rng(9)
    lo = rng.uniform(-6, 6, 4000)
    hi = lo + rng.uniform(0, 8, 4000) * (rng.random(4000) > 0.1)
    # pin the degenerate and far-left (secant underflow) branches too
    lo = np.concatenate([lo, [-800.0, -50.0, 0.0, -1e-9, 3.0, -3.0]])
    hi = np.concatenate([hi, [-799.0, -49.5, 0.0, 1e-9, 3.0, -3.0]])
    out["rules/lo"] = lo
    out["rules/hi"] = hi
    for kind in (ActivationKind.RELU, ActivationKind.ELU, ActivationKind.SIN, ActivationKind.TANH):
        with np.errstate(all="ignore"):
            a, b, g = AFFINE_RULES[kind](lo, hi)
            il, ih = INTERVAL_RULES[kind](lo, hi)
        out[f"rules/{kind.value}/alpha"] = np.asarray(a, float)
        out[f"rules/{kind.value}/beta"] = np.asarray(b, float)
        out[f"rules/{kind.value}/gamma"] = np.asarray(g, float)
        out[f"rules/{kind.value}/ilo"] = np.asarray(il, float)
        out[f"rules/{kind.value}/ihi"] = np.asarray(ih, float)


def flatten_tree(root):
    """Breadth-first level arrays with path keys (root 1, child 2k / 2k+1)."""
    levels = []
    frontier = [(root, 1)]
    while frontier:
        lo = np.array([n.aabb.lo for n, _ in frontier])
        hi = np.array([n.aabb.hi for n, _ in frontier])
        sign = np.array([{"positive": 1, "negative": -1, "unknown": 0}[n.sign.value] for n, _ in frontier], np.int8)
        face = np.array([0 if n.face_sign is None else n.face_sign for n, _ in frontier], np.int8)
        keys = np.array([k for _, k in frontier], np.int64)
        levels.append((keys, lo, hi, sign, face))
        nxt = []
        for n, k in frontier:
            if n.children:
                nxt.append((n.children[0], 2 * k))
                nxt.append((n.children[1], 2 * k + 1))
        frontier = nxt
    return levels


def gen_trees(nets, out):
    bounds = sp.AABB(np.full(3, -1.0), np.full(3, 1.0))
    cases = [
        ("box_d8_fixed", "box", dict(policy=sp.AFFINE_FIXED, max_depth=8)),
        ("box_conv_full", "box", dict(policy=sp.AFFINE_FULL, delta=0.1)),
        ("relu_sdf_d10_fixed", "relu_sdf", dict(policy=sp.AFFINE_FIXED, max_depth=10)),
        ("relu_sdf_d7_interval", "relu_sdf", dict(policy=sp.INTERVAL_ONLY, max_depth=7)),
        ("relu4x32_d9_fixed", "relu4x32", dict(policy=sp.AFFINE_FIXED, max_depth=9)),
        ("elu_sdf_conv_trunc", "elu_sdf", dict(policy=sp.affine_truncate(8), delta=0.15)),
        # the reference's DEFAULT policy on a 227-symbol net (large-capacity affine-full)
        ("relu_sdf_d7_full", "relu_sdf", dict(policy=sp.AFFINE_FULL, max_depth=7)),
    ]
    for tag, netname, kw in cases:
        root = sp.build_spatial_tree(nets[netname], bounds, **kw)
        for lv, (keys, lo, hi, sign, face) in enumerate(flatten_tree(root)):
            p = f"tree/{tag}/{lv}"
            out[p + "/keys"] = keys
            out[p + "/lo"] = lo
            out[p + "/hi"] = hi
            out[p + "/sign"] = sign
            out[p + "/face"] = face


def random_rays(rng, n):
    """Reference test_rays.py:126-133 recipe."""
    o = rng.standard_normal((n, 3))
    o *= 2.0 / np.linalg.norm(o, axis=1, keepdims=True)
    tgt = rng.uniform(-0.75, 0.75, (n, 3))
    d = tgt - o
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return o, d


def gen_rays(nets, out):
    rng = np.random.default_rng(5)
    params = sp.RayCastParams(t_max=4.0)
    for netname in ("box", "relu_sdf", "sin3x48"):
        o, d = random_rays(rng, 64)
        out[f"rays/{netname}/origins"] = o
        out[f"rays/{netname}/dirs"] = d
        for pol in ("affine-fixed", "interval", "affine-truncate:8"):
            hit, t, steps = _march_arrays(nets[netname], o, d, params, sp.parse_policy(pol))
            out[f"rays/{netname}/{pol}/hit"] = hit
            out[f"rays/{netname}/{pol}/t"] = t
            out[f"rays/{netname}/{pol}/steps"] = steps
    cam = sp.Camera(np.array([1.6, 1.2, 2.0]), np.zeros(3), np.array([0.0, 1.0, 0.0]), 40.0, (24, 16))
    out["camera/dirs"] = cam.pixel_dirs()
    dirs = cam.pixel_dirs().reshape(-1, 3)
    orig = np.broadcast_to(cam.position, dirs.shape).copy()
    hit, t, steps = _march_arrays(nets["relu_sdf"], orig, dirs, sp.RayCastParams(), sp.AFFINE_FIXED)
    out["camera/relu_sdf/hit"] = hit
    out["camera/relu_sdf/t"] = t
    out["camera/relu_sdf/steps"] = steps


FRONT_CAM = dict(position=np.array([0.13, 0.11, 2.4]), look_at=np.array([0.02, -0.03, 0.0]),
                 up=np.array([0.0, 1.0, 0.0]), vertical_fov=40.0)


def gen_frustum(nets, out):
    """cast_frustum_image (rays.py:232-341) on the box oracle (reference
    test_rays.py:226-242 camera) and on relu_sdf with the bench camera."""
    cases = [
        ("box_front64", "box", sp.Camera(resolution=(64, 64), **FRONT_CAM), sp.RayCastParams(t_max=4.0), 16),
        ("relu_sdf_default48", "relu_sdf",
         sp.Camera(np.array([1.6, 1.2, 2.0]), np.zeros(3), np.array([0.0, 1.0, 0.0]), 40.0, (48, 32)),
         sp.RayCastParams(), 8),
    ]
    for tag, netname, cam, params, grid in cases:
        res = sp.cast_frustum_image(nets[netname], cam, params, sp.AFFINE_FIXED, initial_grid=grid)
        out[f"frustum/{tag}/hit"] = res.hit
        out[f"frustum/{tag}/t"] = res.t
        out[f"frustum/{tag}/steps"] = res.steps


def gen_render(nets, out):
    """render_image (render.py:91-141) in its three modes."""
    from spelunk.render import render_image

    box_cam = sp.Camera(resolution=(48, 48), **FRONT_CAM)
    sdf_cam = sp.Camera(np.array([1.6, 1.2, 2.0]), np.zeros(3), np.array([0.0, 1.0, 0.0]), 40.0, (40, 24))
    cases = [
        ("box_per_ray", "box", box_cam, sp.RayCastParams(t_max=4.0), "per_ray", None),
        ("box_frustum", "box", box_cam, sp.RayCastParams(t_max=4.0), "frustum", None),
        ("box_fixed", "box", box_cam, sp.RayCastParams(t_max=4.0), "fixed_step", 0.01),
        ("relu_sdf_per_ray", "relu_sdf", sdf_cam, sp.RayCastParams(), "per_ray", None),
        ("elu_sdf_fixed", "elu_sdf", sdf_cam, sp.RayCastParams(t_max=5.0), "fixed_step", 0.02),
    ]
    for tag, netname, cam, params, mode, step in cases:
        img = render_image(nets[netname], cam, params, sp.AFFINE_FIXED, mode, step)
        out[f"render/{tag}/pixels"] = img.pixels


def gen_queries(nets, out):
    """Volumetric queries (spatial.py:292-684), reference default policies."""
    from spelunk.spatial import (_certified_radii, bulk_properties, closest_point, empty_box_radius,
                                 sample_near_surface, test_intersection, walk_on_spheres_stats)

    box, sdf = nets["box"], nets["relu_sdf"]
    cube = sp.AABB(np.full(3, -1.0), np.full(3, 1.0))
    rng = np.random.default_rng(41)
    # empty-box radii: single points and one batched call
    pts = np.array([[0.9, 0.9, 0.9], [0.0, 0.0, 0.0], [0.4999, 0.0, 0.0], [0.3, -0.7, 0.2]])
    rin = np.array([0.5, 0.25, 0.5, 1.0])
    out["queries/ebr/box/points"] = pts
    out["queries/ebr/box/r_init"] = rin
    out["queries/ebr/box/radius"] = np.array([empty_box_radius(box, q, r).radius for q, r in zip(pts, rin)])
    sp_pts = rng.uniform(-1.0, 1.0, (48, 3))
    out["queries/radii/relu_sdf/points"] = sp_pts
    out["queries/radii/relu_sdf/radii"] = _certified_radii(sdf, sp_pts, np.full(48, 1.0), 0.002, sp.AFFINE_FULL)
    # walk on spheres (harmonic data x0)
    m, se = walk_on_spheres_stats(box, [0.2, 0.0, 0.0], lambda q: q[0], 300, rng_seed=0)
    out["queries/wos/box"] = np.array([m, se])
    # band sampling
    out["queries/sample/box"] = sample_near_surface(box, cube, 500, 0.01, 12, rng_seed=1)
    out["queries/sample/relu_sdf"] = sample_near_surface(sdf, cube, 300, 0.05, 7, rng_seed=2)
    # mass properties
    for tag, net, depth in (("box", box, 9), ("relu_sdf", sdf, 6)):
        bp = bulk_properties(net, cube, depth, rng_seed=0)
        out[f"queries/bulk/{tag}"] = np.concatenate([[bp.mass, bp.mass_error_bound], bp.centroid,
                                                     bp.inertia.reshape(-1)])
    # intersection: overlapping / disjoint / touching
    big = sp.AABB(np.full(3, -2.0), np.full(3, 2.0))
    for tag, off, delta in (("overlap", 0.4, 0.01), ("disjoint", 2.0, 0.01), ("touch", 1.0, 0.05)):
        other = sp.build_box_oracle(np.array([off, 0.0, 0.0]), 0.5)
        bounds = sp.AABB(np.full(3, -2.0), np.full(3, 3.0)) if tag == "disjoint" else big
        res = test_intersection(box, other, bounds, delta=delta)
        out[f"queries/isect/{tag}/kind"] = np.array(["disjoint", "intersecting", "inconclusive"].index(res.kind))
        if res.witness is not None:
            out[f"queries/isect/{tag}/witness"] = np.concatenate([res.witness.lo, res.witness.hi])
        out[f"queries/isect/{tag}/nodes"] = (np.array([np.concatenate([n.lo, n.hi]) for n in res.nodes])
                                             if res.nodes else np.zeros((0, 6)))
    # closest point
    qs = rng.uniform(-1.2, 1.2, (4, 3))
    out["queries/closest/box/q"] = qs
    out["queries/closest/box/result"] = np.array([np.concatenate(
        [p, [dd]]) for p, dd in (closest_point(box, q, cube, delta=0.01) for q in qs)])
    qs2 = rng.uniform(-0.9, 0.9, (2, 3))
    out["queries/closest/relu_sdf/q"] = qs2
    out["queries/closest/relu_sdf/result"] = np.array([np.concatenate(
        [p, [dd]]) for p, dd in (closest_point(sdf, q, cube, delta=0.01) for q in qs2)])


def gen_variants(nets, out):
    """bench_variants region sizes and a fuzz report (bench.py:128-319)."""
    from spelunk.bench import bench_variants, fuzz_soundness

    rows = bench_variants([nets["relu_sdf"], nets["elu_sdf"]], n_regions=2000, rng_seed=0, raycast_res=16, runs=1)
    out["variants/region_size"] = np.array([r.region_size for r in rows])
    out["variants/dim"] = np.array([r.dim for r in rows])
    rep = fuzz_soundness([nets["relu_sdf"], nets["sin12"]], n_regions=20_000, rng_seed=3, threads=1)
    out["variants/fuzz"] = np.array([rep.n_regions, rep.n_checks, rep.n_violations])


def gen_mesh(nets, out):
    bounds = sp.AABB(np.full(3, -1.0), np.full(3, 1.0))
    for tag, netname, m, pol in (
        ("offset_box_m5_fixed", "offset_box", 5, sp.AFFINE_FIXED),
        ("offset_box_m5_full", "offset_box", 5, sp.AFFINE_FULL),
        ("relu_sdf_m5_fixed", "relu_sdf", 5, sp.AFFINE_FIXED),
        ("elu_sdf_m5_fixed", "elu_sdf", 5, sp.AFFINE_FIXED),
        ("relu_sdf_m5_full", "relu_sdf", 5, sp.AFFINE_FULL),  # extract_mesh's default policy
    ):
        mesh = sp.extract_mesh(nets[netname], bounds, m, policy=pol)
        out[f"mesh/{tag}/vertices"] = mesh.vertices
        out[f"mesh/{tag}/triangles"] = mesh.triangles
    dense = sp.extract_mesh_dense(nets["relu_sdf"], bounds, 5)
    out["mesh/relu_sdf_m5_dense/vertices"] = dense.vertices
    out["mesh/relu_sdf_m5_dense/triangles"] = dense.triangles
    flat = []
    for case in range(256):
        for tri in mc_tables.TRI_TABLE[case]:
            flat.append((case, *tri))
    out["mc/tri_table"] = np.array(flat, np.int64)
    out["mc/edge_table"] = np.array(mc_tables.EDGE_TABLE, np.int64)


def main():
    nets = make_nets()
    out = {}
    gen_rules(out)
    gen_bounds(nets, out)
    gen_trees(nets, out)
    gen_rays(nets, out)
    gen_mesh(nets, out)
    gen_frustum(nets, out)
    gen_render(nets, out)
    gen_queries(nets, out)
    gen_variants(nets, out)
    np.savez_compressed(HERE / "golden.npz", **out)
    meta = {"reference": REF_SRC, "numpy": np.__version__, "n_arrays": len(out)}
    (HERE / "golden_meta.json").write_text(json.dumps(meta, indent=1))
    print(f"wrote {len(out)} arrays")


if __name__ == "__main__":
    main()
