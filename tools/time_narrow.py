"""CUDA-event timings of the narrow-net paths (A/B with SPK_LIB_PATH)."""
import json
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2202_02444_b200 as sp  # noqa: E402
from paper_2202_02444_b200 import synth  # noqa: E402
from paper_2202_02444_b200.camera import default_camera  # noqa: E402


def timed(fn, reps=5):
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


sdf = sp.load_network("tests/golden/nets/relu_sdf.json")
c1 = synth.config_net("C1")
res = {}
cam = default_camera(1024)
for pol in ("affine-fixed", "interval"):
    res[f"rays_{pol}_ms"] = timed(lambda: sp.cast_camera(sdf, cam, sp.RayCastParams(), pol, precision="fp32"))
    res[f"frustum_{pol}_ms"] = timed(lambda: sp.cast_frustum_image(sdf, cam, sp.RayCastParams(), pol,
                                                                   precision="fp32", device_output=True))
gc, ga = synth.grid_cubes(64)
gc, ga = torch.from_numpy(gc).cuda(), torch.from_numpy(ga).cuda()
res["c1_ms"] = timed(lambda: sp.range_bound_batch(c1, gc, ga, sp.AFFINE_FIXED))
x = torch.rand((1 << 22, 3), device="cuda", dtype=torch.float64) * 2 - 1
res["eval_4M_sdf_ms"] = timed(lambda: sp.eval_batch(sdf, x, precision="fp32"))
print(json.dumps(res))
