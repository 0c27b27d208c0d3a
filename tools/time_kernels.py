"""CUDA-event timings of the fused bound kernel on the bench workloads, for
A/B builds (SPK_LIB_PATH): C1 grid (4x32, 64^3), C5 cubes at widths 64 / 256
/ 512, and one C2 tree build.  Median of 5 (L2 flushed).  One JSON line."""
import json
import os
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2202_02444_b200 as sp  # noqa: E402
from paper_2202_02444_b200 import spatial, synth  # noqa: E402

flush_buf = torch.empty(64 << 20, dtype=torch.float32, device="cuda")


def t(fn, reps=5):
    fn()
    ts = []
    for _ in range(reps):
        flush_buf.fill_(1.0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


out = {"lib": os.environ.get("SPK_LIB_PATH", "in-tree")}
c1 = synth.config_net("C1")
c, a = synth.grid_cubes(64)
ct, at = torch.from_numpy(c).cuda(), torch.from_numpy(a).cuda()
out["C1_ms"] = t(lambda: sp.range_bound_batch(c1, ct, at, sp.AFFINE_FIXED))
for tag, n in (("C5_64", 1 << 22), ("C5_256", 1 << 20), ("C5_512", 1 << 18)):
    net = synth.config_net(tag)
    o = tuple(torch.empty(n, dtype=dt, device="cuda") for dt in (torch.float64, torch.float64, torch.int8))
    out[tag + "_ms"] = t(lambda: sp.bound_random_cubes(net, n, seed=1, half=1 / 64, out=o))
c2 = synth.config_net("C2")
b = spatial.AABB(-np.ones(3), np.ones(3))
out["C2_tree_ms"] = t(lambda: spatial.build_spatial_tree_arrays(c2, b, policy=sp.AFFINE_FIXED, max_depth=18,
                                                               to_host=False), reps=3)
print(json.dumps(out), flush=True)
