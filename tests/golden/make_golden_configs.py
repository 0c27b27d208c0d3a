"""Golden vectors for BASELINE.json's configs C3, C4 and C5, produced by the
unmodified reference.

Runs ONLY in the build container, where the reference package is importable
from /root/reference/pkg/src (override with SPELUNK_REF_SRC):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_configs.py

The config nets are not committed (the 8x512 weight file would be ~40 MB):
they are regenerated deterministically by paper_2202_02444_b200.synth (seeded
NumPy), converted to the reference's NetworkSpec here, and fingerprinted
(sum and sum of squares of every parameter, in order) so the tests can assert
they rebuilt the same net.  Output: tests/golden/configs.npz.

  C3  SIREN 3->8x256->1, default bench camera (reference bench.py:119-126) at
      32x32, RayCastParams() defaults: _march_arrays (rays.py:88-138) for 128
      pixels (every 8th) under interval and affine-fixed, 32 pixels (every
      32nd) under affine-truncate:16, 16 pixels (every 64th) under
      affine-truncate:32.
  C4  ELU 3->8x512->1 occupancy net: extract_mesh (meshing.py:111-169), m=4
      and m=5, dense_levels=3, affine-fixed (passed explicitly: the reference
      default affine-full needs 4,099 symbols).
  C2  the headline net (8x256 ReLU) at depth 12: build_spatial_tree levels
      (AABBs, labels) and each level's range_bound_batch bounds.
  C5  4096 cubes of half-extent 1/64 with centres from the on-device stream
      (synth.random_cube_centres, seed 5): range_bound_batch
      (range_core.py:547-642) for the 8-layer width-64 and width-512 nets,
      affine-fixed and interval.
"""

from __future__ import annotations

import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
REF_SRC = os.environ.get("SPELUNK_REF_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF_SRC)
sys.path.insert(0, str(ROOT))
sys.dont_write_bytecode = True

C3_STRIDE = {"interval": 8, "affine-fixed": 8, "affine-truncate:16": 32, "affine-truncate:32": 64}
C3_RES = 32
C5_N = 4096
C5_SEED = 5
C5_HALF = 1.0 / 64


def fingerprint(net) -> np.ndarray:
    ps = [np.concatenate([L.weights.ravel(), L.bias.ravel()]) for L in net.layers if hasattr(L, "weights")]
    p = np.concatenate(ps)
    return np.array([p.size, p.sum(), (p * p).sum()])


def ref_net(tag):
    import spelunk as ref
    from spelunk.network import ActivationKind, DenseLayer, NetworkSpec

    from paper_2202_02444_b200 import synth

    net = synth.config_net(tag)
    layers = []
    for L in net.layers:
        if hasattr(L, "weights"):
            layers.append(DenseLayer(np.array(L.weights), np.array(L.bias)))
        else:
            layers.append(ActivationKind(L.value))
    assert ref is not None
    return NetworkSpec(net.input_dim, tuple(layers), "sdf", net.name), fingerprint(net)


def c3_rays():
    import spelunk as ref

    cam = ref.Camera(np.array([1.6, 1.2, 2.0]), np.zeros(3), np.array([0.0, 1.0, 0.0]), 40.0, (C3_RES, C3_RES))
    dirs = cam.pixel_dirs().reshape(-1, 3)
    return cam.position, dirs


def job_c3(policy, lo, hi):
    import spelunk as ref
    from spelunk.rays import _march_arrays

    net, _ = ref_net("C3")
    pos, dirs = c3_rays()
    idx = np.arange(0, C3_RES * C3_RES, C3_STRIDE[policy])[lo:hi]
    d = dirs[idx]
    o = np.broadcast_to(pos, d.shape).copy()
    hit, t, steps = _march_arrays(net, o, d, ref.RayCastParams(), ref.parse_policy(policy))
    return ("C3", policy, lo, hit, t, steps)


def job_c4(m):
    import spelunk as ref

    net, _ = ref_net("C4")
    mesh = ref.extract_mesh(net, ref.AABB(np.full(3, -1.0), np.full(3, 1.0)), m, policy=ref.AFFINE_FIXED)
    return ("C4", m, mesh.vertices, mesh.triangles)


def job_c2(depth):
    """The headline config itself at a depth the reference finishes in
    seconds: build_spatial_tree (spatial.py:214-289), affine-fixed, with each
    level's node bounds from range_bound_batch (the same boxes the tree
    bounded)."""
    import spelunk as ref

    net, _ = ref_net("C2")
    root = ref.build_spatial_tree(net, ref.AABB(np.full(3, -1.0), np.full(3, 1.0)), policy=ref.AFFINE_FIXED,
                                  max_depth=depth)
    levels, frontier = [], [root]
    while frontier:
        lo = np.array([n.aabb.lo for n in frontier])
        hi = np.array([n.aabb.hi for n in frontier])
        lab = np.array([{"positive": 1, "negative": -1}.get(n.sign.value, 0) for n in frontier], np.int8)
        axes = np.zeros((len(frontier), 3, 3))
        axes[:, np.arange(3), np.arange(3)] = (hi - lo) / 2.0
        blo, bhi = ref.range_bound_batch(net, (lo + hi) / 2.0, axes, ref.AFFINE_FIXED)
        levels.append((lo, hi, lab, blo, bhi))
        nxt_lo = [c for n in frontier if n.children for c in n.children[:1]]
        nxt_hi = [c for n in frontier if n.children for c in n.children[1:]]
        frontier = nxt_lo + nxt_hi
    return ("C2", depth, levels)


def job_c5(tag, policy):
    import spelunk as ref

    from paper_2202_02444_b200 import synth

    net, _ = ref_net(tag)
    c = synth.random_cube_centres(C5_N, C5_SEED)
    axes = np.zeros((C5_N, 3, 3))
    axes[:, np.arange(3), np.arange(3)] = C5_HALF
    lo, hi = ref.range_bound_batch(net, c, axes, ref.parse_policy(policy))
    return ("C5", tag, policy, lo, hi)


def main():
    t0 = time.time()
    out = {}
    for tag in ("C2", "C3", "C4", "C5_64", "C5_512"):
        out[f"configs/{tag}/fingerprint"] = ref_net(tag)[1]
    pos, dirs = c3_rays()
    out["configs/C3/position"] = pos
    out["configs/C3/dirs"] = dirs
    jobs = []
    with ProcessPoolExecutor(max_workers=os.cpu_count()) as pool:
        for pol, stride in C3_STRIDE.items():
            n = C3_RES * C3_RES // stride
            per = 8 if "truncate" not in pol else 1
            for lo in range(0, n, per):
                jobs.append(pool.submit(job_c3, pol, lo, min(n, lo + per)))
        for m in (4, 5):
            jobs.append(pool.submit(job_c4, m))
        for tag in ("C5_64", "C5_512"):
            for pol in ("affine-fixed", "interval"):
                jobs.append(pool.submit(job_c5, tag, pol))
        jobs.append(pool.submit(job_c2, 12))
        c3 = {}
        for f in jobs:
            r = f.result()
            if r[0] == "C3":
                c3.setdefault(r[1], []).append(r[2:])
            elif r[0] == "C4":
                out[f"configs/C4/m{r[1]}/vertices"] = r[2]
                out[f"configs/C4/m{r[1]}/triangles"] = r[3]
            elif r[0] == "C2":
                for k, (lo, hi, lab, blo, bhi) in enumerate(r[2]):
                    for name, v in (("lo", lo), ("hi", hi), ("label", lab), ("bound_lo", blo), ("bound_hi", bhi)):
                        out[f"configs/C2/d{r[1]}/{k}/{name}"] = v
            else:
                out[f"configs/{r[1]}/{r[2]}/lo"] = r[3]
                out[f"configs/{r[1]}/{r[2]}/hi"] = r[4]
    for pol, parts in c3.items():
        parts.sort(key=lambda p: p[0])
        idx = np.arange(0, C3_RES * C3_RES, C3_STRIDE[pol])
        out[f"configs/C3/{pol}/pixels"] = idx
        out[f"configs/C3/{pol}/hit"] = np.concatenate([p[1] for p in parts])
        out[f"configs/C3/{pol}/t"] = np.concatenate([p[2] for p in parts])
        out[f"configs/C3/{pol}/steps"] = np.concatenate([p[3] for p in parts])
    c = __import__("paper_2202_02444_b200.synth", fromlist=["x"]).random_cube_centres(C5_N, C5_SEED)
    out["configs/C5/centres"] = c
    np.savez_compressed(HERE / "configs.npz", **out)
    meta = {"reference": REF_SRC, "numpy": np.__version__, "n_arrays": len(out),
            "seconds": round(time.time() - t0, 1)}
    (HERE / "configs_meta.json").write_text(json.dumps(meta, indent=1))
    print(f"wrote {len(out)} arrays in {time.time() - t0:.0f} s")


if __name__ == "__main__":
    main()
