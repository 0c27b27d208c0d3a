"""FP64 kernel timings (A/B with SPK_LIB_PATH)."""
import json
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2202_02444_b200 as sp  # noqa: E402
from paper_2202_02444_b200 import spatial, synth  # noqa: E402
from paper_2202_02444_b200.camera import default_camera  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


c3 = synth.config_net("C3")
c2 = synth.config_net("C2")
cam = default_camera(96)
x = torch.rand((1 << 20, 3), device="cuda", dtype=torch.float64) * 2 - 1
res = {"c3_interval_96sq_ms": timed(lambda: sp.cast_camera(c3, cam, sp.RayCastParams(), "interval", precision="fp64")),
       "c2_eval_1M_fp64_ms": timed(lambda: sp.eval_batch(c2, x, precision="fp64")),
       "c2_fixed_256K_fp64_ms": timed(lambda: sp.bound_random_cubes(c2, 1 << 18, seed=1, precision="fp64")),
       "c2_tree_d18_fp64_ms": timed(lambda: spatial.build_spatial_tree_arrays(
           c2, sp.AABB([-1.0] * 3, [1.0] * 3), policy=sp.AFFINE_FIXED, max_depth=18, precision="fp64",
           to_host=False)),
       "c5_512_1M_fp64_ms": timed(lambda: sp.bound_random_cubes(synth.config_net("C5_512"), 1 << 20, seed=1,
                                                                 precision="fp64"))}
print(json.dumps(res))
