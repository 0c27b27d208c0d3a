"""K7 hierarchical marching cubes on the GPU vs the reference's golden meshes.

Connectivity: the triangle lists as edge-key triples must equal the
reference's exactly (FP64 point evaluation; vertex ids are numbered in
first-visit order like _MeshBuilder, so even the triangle arrays match).
Vertex positions agree to 1e-12 (FP64 evaluation differs from the
reference's einsum only in summation order).
"""

import numpy as np
import pytest

import paper_2202_02444_b200 as sp
from oracle import spelunk_oracle as orc
from paper_2202_02444_b200 import mc_tables, meshing
from paper_2202_02444_b200.spatial import AABB

pytestmark = pytest.mark.gpu
BOUNDS = AABB(-np.ones(3), np.ones(3))
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
    net = sp.load_network(net_paths[netname])
    res = meshing.extract_mesh_arrays(net, BOUNDS, m, 3, pol, precision="fp64")
    wv, wt = golden[f"mesh/{tag}/vertices"], golden[f"mesh/{tag}/triangles"]
    assert res.triangles.shape == wt.shape
    np.testing.assert_array_equal(res.triangles, wt)          # first-visit numbering: identical arrays
    assert np.max(np.abs(res.vertices - wv)) <= 1e-12
    # oracle edge keys agree too
    ov, ot, okeys = orc.mesh_extract(orc.as_oracle_net(net), -np.ones(3), np.ones(3), m, 3, pol)
    np.testing.assert_array_equal(res.vertex_keys, okeys)


def test_dense_matches_hierarchical(net_paths):
    net = sp.load_network(net_paths["offset_box"])
    h = meshing.extract_mesh_arrays(net, BOUNDS, 5, 3, "affine-fixed")
    d = meshing.extract_mesh_arrays(net, BOUNDS, 5, 3, "affine-fixed", prune=False)
    np.testing.assert_array_equal(meshing.triangle_key_set(h.triangles, h.vertex_keys),
                                  meshing.triangle_key_set(d.triangles, d.vertex_keys))
    assert h.point_evals < d.point_evals


@pytest.mark.parametrize("netname", ["relu_sdf", "elu_sdf"])
def test_mesh_fp32_connectivity(net_paths, netname):
    """FP32 evaluation (the north-star rule): the triangles of every grid cell
    whose 8 corner signs agree between FP32 and FP64 are identical."""
    from tests.mesh_rules import agreeing_triangle_sets

    net = sp.load_network(net_paths[netname])
    a = meshing.extract_mesh_arrays(net, BOUNDS, 6, 3, "affine-fixed", precision="fp64")
    b = meshing.extract_mesh_arrays(net, BOUNDS, 6, 3, "affine-fixed", precision="fp32")
    ka, kb, na, nb, bad = agreeing_triangle_sets(net, a, b, 6)
    assert len(ka) > 0
    np.testing.assert_array_equal(ka, kb)
    print(f"MESH {netname} fp32 vs fp64: {len(ka)} triangles identical on agreeing cells; "
          f"{na} / {nb} on {bad} disagreeing cells")


def test_mesh_edge_cases(net_paths):
    const = sp.NetworkSpec(3, (sp.DenseLayer(np.zeros((1, 3)), np.array([1.0])),))
    res = meshing.extract_mesh_arrays(const, BOUNDS, 4, 3, "affine-fixed")
    assert len(res.vertices) == 0 and len(res.triangles) == 0
    with pytest.raises(sp.errors.ResolutionTooSmall):
        meshing.extract_mesh(const, BOUNDS, 3)


def test_watertight_and_volume(net_paths):
    from collections import Counter

    net = sp.load_network(net_paths["offset_box"])
    mesh = meshing.extract_mesh(net, BOUNDS, 5, policy="affine-fixed")
    v, t = mesh.vertices, mesh.triangles
    directed = Counter()
    for a, b, c in t:
        for e in ((a, b), (b, c), (c, a)):
            directed[e] += 1
    assert all(directed[(b, a)] == n for (a, b), n in directed.items())
    v0, v1, v2 = v[t[:, 0]], v[t[:, 1]], v[t[:, 2]]
    assert abs(np.einsum("ij,ij->", v0, np.cross(v1, v2)) / 6.0 - 1.0) <= 0.01


@pytest.mark.parametrize("world", [2, 3, 5])
def test_mesh_shards_merge_to_unsharded(net_paths, world):
    """C4 sharding (spk_mesh_extract_shard): block slices per rank, merged by
    the global edge-key dedup, reproduce the unsharded arrays exactly."""
    net = sp.load_network(net_paths["relu_sdf"])
    full = meshing.extract_mesh_arrays(net, BOUNDS, 6, 3, "affine-fixed", precision="fp64")
    parts = [meshing.extract_mesh_sharded(net, BOUNDS, 6, r, world, 3, "affine-fixed", precision="fp64")
             for r in range(world)]
    assert sum(p.n_blocks for p in parts) == full.n_blocks
    assert [p.meta["block_first"] for p in parts] == sorted(p.meta["block_first"] for p in parts)
    got = meshing.merge_sharded_meshes(parts)
    np.testing.assert_array_equal(got.triangles, full.triangles)
    np.testing.assert_array_equal(got.vertex_keys, full.vertex_keys)
    np.testing.assert_array_equal(got.vertices, full.vertices)
    # single process: gather_mesh of the whole mesh is the identity
    one = meshing.gather_mesh(meshing.extract_mesh_sharded(net, BOUNDS, 6, 0, 1, 3, "affine-fixed"))
    np.testing.assert_array_equal(one.triangles, full.triangles)
