"""CUDA-event timing of the C2 tree build (A/B with SPK_LIB_PATH)."""
import json
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2202_02444_b200 as sp  # noqa: E402
from paper_2202_02444_b200 import spatial, synth  # noqa: E402

net = synth.config_net("C2")
bounds = spatial.AABB(-np.ones(3), np.ones(3))
run = lambda: spatial.build_spatial_tree_arrays(net, bounds, policy=sp.AFFINE_FIXED, max_depth=18, to_host=False)
run()
torch.cuda.synchronize()
best, kern = 1e9, None
for _ in range(4):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    arr = run()
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1)
    if t < best:
        best, kern = t, arr.bound_ms
print(json.dumps({"tree_ms": best, "bound_kernel_ms": kern}))
