"""Where the C4 mesh extraction's time goes: per-kernel device time (CUPTI via
torch.profiler, which sees the library's own launches) against the wall
clock of extract_mesh_arrays, at 2^m cells per axis.  Usage:
python tools/c4_breakdown.py [m ...]"""

import collections
import json
import os
import sys
import time

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2202_02444_b200 as sp  # noqa: E402
from paper_2202_02444_b200 import meshing, synth  # noqa: E402
from paper_2202_02444_b200.spatial import AABB  # noqa: E402


def run(m):
    net = synth.config_net("C4")
    b = AABB(-np.ones(3), np.ones(3))
    meshing.extract_mesh_arrays(net, b, 6, 3, sp.AFFINE_FIXED, precision="fp32")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = meshing.extract_mesh_arrays(net, b, m, 3, sp.AFFINE_FIXED, precision="fp32")
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        t1 = time.perf_counter()
        meshing.extract_mesh_arrays(net, b, m, 3, sp.AFFINE_FIXED, precision="fp32")
        torch.cuda.synchronize()
        wall_prof = time.perf_counter() - t1
    agg = collections.defaultdict(lambda: [0, 0.0])
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            k = e.name if len(e.name) < 90 else e.name[:90]
            agg[k][0] += 1
            agg[k][1] += e.device_time_total / 1e3 if hasattr(e, "device_time_total") else e.cuda_time_total / 1e3
    tot = sum(v[1] for v in agg.values())
    top = sorted(agg.items(), key=lambda kv: -kv[1][1])[:15]
    print(json.dumps({"m": m, "wall_s": wall, "wall_profiled_s": wall_prof, "device_ms_total": tot,
                      "point_evals": int(res.point_evals) if hasattr(res, "point_evals") else None,
                      "top": [[k, v[0], round(v[1], 2)] for k, v in top]}), flush=True)


if __name__ == "__main__":
    for m in [int(a) for a in sys.argv[1:]] or [8, 9]:
        run(m)
