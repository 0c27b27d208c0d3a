"""Golden vectors for the trained 3->8x256->1 ReLU torus SDF net
(synth.trained_net, weights in tests/golden/nets/torus_8x256.npz, made by
tools/train_sdf_net.py), produced by the unmodified reference.

Runs ONLY in the build container, where the reference package is importable
from /root/reference/pkg/src (override with SPELUNK_REF_SRC):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_trained.py

Output tests/golden/trained.npz:
  tree/<policy>/<k>/{lo,hi,label,bound_lo,bound_hi}  build_spatial_tree
      (spatial.py:214-289) to depth 10, levels in the reference's order, with
      each level's range_bound_batch bounds (affine-fixed and interval)
  cubes/<h>/{lo,hi}, cubes/centres  range_bound_batch (range_core.py:547-642),
      affine-fixed, 8192 cubes of half-extent 1/h, h in {64, 256}
      (synth.random_cube_centres, seed 7)
"""

from __future__ import annotations

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

DEPTH = 10
N_CUBES = 8192
SEED = 7
HALVES = (64, 256)


def ref_net():
    from spelunk.network import ActivationKind, DenseLayer, NetworkSpec

    from paper_2202_02444_b200 import synth

    net = synth.trained_net("torus")
    layers = []
    for L in net.layers:
        if hasattr(L, "weights"):
            layers.append(DenseLayer(np.array(L.weights), np.array(L.bias)))
        else:
            layers.append(ActivationKind(L.value))
    return NetworkSpec(net.input_dim, tuple(layers), "sdf", net.name)


def job_tree(policy):
    import spelunk as ref

    net = ref_net()
    pol = ref.parse_policy(policy)
    root = ref.build_spatial_tree(net, ref.AABB(np.full(3, -1.0), np.full(3, 1.0)), policy=pol, max_depth=DEPTH)
    levels, frontier = [], [root]
    while frontier:
        lo = np.array([n.aabb.lo for n in frontier])
        hi = np.array([n.aabb.hi for n in frontier])
        lab = np.array([{"positive": 1, "negative": -1}.get(n.sign.value, 0) for n in frontier], np.int8)
        axes = np.zeros((len(frontier), 3, 3))
        axes[:, np.arange(3), np.arange(3)] = (hi - lo) / 2.0
        blo, bhi = ref.range_bound_batch(net, (lo + hi) / 2.0, axes, pol)
        levels.append((lo, hi, lab, blo, bhi))
        nxt_lo = [c for n in frontier if n.children for c in n.children[:1]]
        nxt_hi = [c for n in frontier if n.children for c in n.children[1:]]
        frontier = nxt_lo + nxt_hi
    return policy, levels


def job_cubes(h, lo_i, hi_i):
    import spelunk as ref

    from paper_2202_02444_b200 import synth

    net = ref_net()
    c = synth.random_cube_centres(N_CUBES, SEED)[lo_i:hi_i]
    axes = np.zeros((len(c), 3, 3))
    axes[:, np.arange(3), np.arange(3)] = 1.0 / h
    lo, hi = ref.range_bound_batch(net, c, axes, ref.AFFINE_FIXED)
    return h, lo_i, lo, hi


def main():
    from paper_2202_02444_b200 import synth

    t0 = time.time()
    out = {}
    with ProcessPoolExecutor(max_workers=os.cpu_count()) as pool:
        trees = [pool.submit(job_tree, p) for p in ("affine-fixed", "interval")]
        step = 1024
        cubes = [pool.submit(job_cubes, h, i, i + step) for h in HALVES for i in range(0, N_CUBES, step)]
        for f in trees:
            policy, levels = f.result()
            for k, (lo, hi, lab, blo, bhi) in enumerate(levels):
                for name, v in (("lo", lo), ("hi", hi), ("label", lab), ("bound_lo", blo), ("bound_hi", bhi)):
                    out[f"tree/{policy}/{k}/{name}"] = v
        parts = sorted(f.result() for f in cubes)
    out["cubes/centres"] = synth.random_cube_centres(N_CUBES, SEED)
    for h in HALVES:
        out[f"cubes/{h}/lo"] = np.concatenate([p[2] for p in parts if p[0] == h])
        out[f"cubes/{h}/hi"] = np.concatenate([p[3] for p in parts if p[0] == h])
    np.savez_compressed(HERE / "trained.npz", **out)
    print(f"wrote {len(out)} arrays in {time.time() - t0:.0f} s")


if __name__ == "__main__":
    main()
