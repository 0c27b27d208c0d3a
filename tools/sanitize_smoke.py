"""Small run of every kernel family, for compute-sanitizer (one tool per run):
fused bound (interval / fixed / truncate / full, FP32 + FP64), point eval, tree
build (fixed + convergence), fused and unfused march, marching cubes; round 2
adds the width-256/512 instantiations (fused ReLU, running-error layer, FP64
live-row masks, small-batch tile), large-capacity truncate (top-k), 5-axis
boxes and a mesh shard; late round 2: fp32-refine on every policy,
speculative tree levels, the 32-row width-512 affine tile."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2202_02444_b200 as sp  # noqa: E402
from paper_2202_02444_b200 import meshing, spatial, synth  # noqa: E402

net = synth.random_mlp(64, 3, "relu", "torch-uniform", seed=1)
small = sp.load_network("tests/golden/nets/relu12.json")
rng = np.random.default_rng(0)
c = rng.uniform(-1, 1, (700, 3))
a = np.zeros((700, 3, 3))
a[:, np.arange(3), np.arange(3)] = 0.05
for pol in ("interval", "affine-fixed", "affine-truncate:8"):
    for prec in ("fp32", "fp64"):
        sp.range_bound_batch(net, c, a, pol, precision=prec)
sp.range_bound_batch(small, c, a, "affine-full")
sp.eval_batch(net, c, precision="fp32")
b = spatial.AABB(-np.ones(3), np.ones(3))
spatial.build_spatial_tree_arrays(net, b, policy="affine-fixed", max_depth=6)
spatial.build_spatial_tree_arrays(small, b, delta=0.3, policy="interval")
cam = sp.Camera(np.array([1.6, 1.2, 2.0]), np.zeros(3), np.array([0.0, 1.0, 0.0]), 40.0, (16, 8))
sp.cast_camera(net, cam, sp.RayCastParams(t_max=3.0), "affine-fixed", precision="fp32")
sp.cast_camera(net, cam, sp.RayCastParams(t_max=3.0), "affine-truncate:8", precision="fp32")
meshing.extract_mesh_arrays(net, b, 4, 3, "affine-fixed")
# round 2 paths
w256 = synth.random_mlp(256, 3, "relu", "torch-uniform", seed=2)
w512 = synth.random_mlp(512, 2, "relu", "torch-uniform", seed=3)
c3, a3 = c[:300], a[:300]
for prec in ("fp32", "fp64"):
    sp.range_bound_batch(w256, c3, a3, "affine-fixed", precision=prec)
    sp.range_bound_batch(w512, c3[:100], a3[:100], "affine-fixed", precision=prec)
sp.range_bound_batch(w256, c3[:64], a3[:64], "affine-truncate:32", precision="fp64")
spatial.build_spatial_tree_arrays(w256, b, policy="affine-fixed", max_depth=4)
hd = synth.random_mlp(32, 2, "relu", "ref-normal", seed=1, input_dim=5)
c5 = rng.uniform(-1, 1, (200, 5))
a5 = np.zeros((200, 5, 5))
a5[:, np.arange(5), np.arange(5)] = 0.05
sp.range_bound_batch(hd, c5, a5, "affine-fixed", precision="fp32")
meshing.extract_mesh_sharded(net, b, 4, 1, 2, 3, "affine-fixed", precision="fp32")
# late round 2: fp32-refine (calibration, candidate selection, FP64 re-bound
# through a processing order; fused, K3 and K3F), speculative tree levels,
# width-512 affine tile with 32-row W tiles and live-row masks
for pol in ("affine-fixed", "interval", "affine-truncate:8", "affine-full"):
    sp.range_bound_batch(small, c, a, pol, precision="fp32-refine")
spatial.build_spatial_tree_arrays(net, b, policy="affine-fixed", max_depth=8, precision="fp32-refine")
sp.range_bound_batch(w512, c3[:200], a3[:200], "affine-fixed", precision="fp32")
print("sanitize smoke done")
