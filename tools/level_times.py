"""Per-launch device times of one C2 tree build (CUPTI through torch.profiler,
which sees the library's own launches), in launch order: where the small top
levels' time goes.  Usage: python tools/level_times.py [depth]"""
import json
import os
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2202_02444_b200 as sp  # noqa: E402
from paper_2202_02444_b200 import spatial, synth  # noqa: E402


def main():
    depth = int(sys.argv[1]) if len(sys.argv) > 1 else 18
    net = synth.config_net("C2")
    b = spatial.AABB(-np.ones(3), np.ones(3))
    run = lambda: spatial.build_spatial_tree_arrays(net, b, policy=sp.AFFINE_FIXED, max_depth=depth, to_host=False)
    run()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        run()
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ev.sort(key=lambda e: e.time_range.start)
    t0 = ev[0].time_range.start
    rows = []
    for e in ev:
        rows.append([e.name[:60], round((e.time_range.start - t0), 1), round(e.time_range.end - e.time_range.start, 1)])
    end = ev[-1].time_range.end - t0
    busy = sum(r[2] for r in rows)
    print(json.dumps({"depth": depth, "span_us": end, "busy_us": busy, "launches": len(rows)}))
    for r in rows:
        print(json.dumps(r))


if __name__ == "__main__":
    main()
