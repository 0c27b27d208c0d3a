"""Wall-clock of the C2 build through the public API: device levels vs host
levels (to_host=True, overlapped host mirror)."""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2202_02444_b200 as sp  # noqa: E402
from paper_2202_02444_b200 import spatial, synth  # noqa: E402

net = synth.config_net("C2")
bounds = spatial.AABB(-np.ones(3), np.ones(3))
res = {}
for to_host in (False, True, False, True):
    arr = spatial.build_spatial_tree_arrays(net, bounds, policy=sp.AFFINE_FIXED, max_depth=18, to_host=to_host)
    ts = []
    for _ in range(3):
        del arr
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        arr = spatial.build_spatial_tree_arrays(net, bounds, policy=sp.AFFINE_FIXED, max_depth=18, to_host=to_host)
        if not to_host:
            arr.levels
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    res[f"to_host={to_host}"] = round(1e3 * float(np.median(ts)), 2)
    print(json.dumps(res))
