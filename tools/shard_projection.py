"""Per-rank work of the sharded paths, measured one rank at a time on ONE GPU.

The sharded builds have no collective inside (each rank refines its share of
the frontier / renders its pixel tiles alone), so a rank's device time does
not depend on the other ranks running: timing every rank's shard in turn on
one B200 gives the compute part of an N-GPU run exactly -- max over ranks --
while the final gather (one all_gather over NVLink) is not included.  This is
a projection of the strong-scaling curve, not a multi-GPU measurement (the
driver's SCALE run is that); each line states which.

    python tools/shard_projection.py
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2202_02444_b200 as sp  # noqa: E402
from paper_2202_02444_b200 import spatial, synth  # noqa: E402
from paper_2202_02444_b200.camera import default_camera  # noqa: E402

flush_buf = torch.empty(64 << 20, dtype=torch.float32, device="cuda")


def dev_ms(fn, reps=3):
    fn()
    ts = []
    for _ in range(reps):
        flush_buf.fill_(1.0)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def project(case, units, run_rank, worlds=(1, 2, 4, 8)):
    t1 = None
    for w in worlds:
        per = [dev_ms(lambda r=r: run_rank(r, w)) for r in range(w)]
        tmax = max(per)
        if w == 1:
            t1 = tmax
        print(json.dumps({"case": case, "world": w, "rank_ms": [round(x, 3) for x in per], "max_ms": round(tmax, 3),
                          "projected_units_per_s": units / tmax * 1e3, "projected_efficiency": t1 / (w * tmax),
                          "note": "per-rank shard work timed one rank at a time on one GPU; final gather excluded"}),
              flush=True)


def main():
    b = spatial.AABB(-np.ones(3), np.ones(3))
    c2 = synth.config_net("C2")
    project("C2 tree depth 18 (524,287 node bounds)", 524287,
            lambda r, w: spatial.build_spatial_tree_sharded(c2, b, 18, sp.AFFINE_FIXED, r, w, to_host=False))
    torus = synth.trained_net("torus")
    full = spatial.build_spatial_tree_arrays(torus, b, policy=sp.AFFINE_FIXED, max_depth=21, to_host=False)
    project(f"trained torus 8x256 tree depth 21 ({full.n_nodes} node bounds, interleaved roots)", full.n_nodes,
            lambda r, w: spatial.build_spatial_tree_sharded(torus, b, 21, sp.AFFINE_FIXED, r, w, to_host=False,
                                                            roots="interleaved"))
    del full
    c3 = synth.config_net("C3")
    cam = default_camera(256)
    project("C3 SIREN rays 256^2 interval FP64 (65,536 rays)", 65536,
            lambda r, w: sp.cast_camera_sharded(c3, cam, r, w, sp.RayCastParams(), "interval", precision="fp64"),
            worlds=(1, 2, 4, 8))


if __name__ == "__main__":
    main()
