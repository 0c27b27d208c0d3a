"""FP32 vs fp32-refine vs FP64 on the trained 8x256 torus SDF net (the
headline architecture with a real surface): certified fractions of random
cubes at several sizes, and deep k-d trees (the C2 build, to depths where
this net certifies), with device times.  One JSON line per case.

    python tools/trained_study.py
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2202_02444_b200 as sp  # noqa: E402
from paper_2202_02444_b200 import spatial, synth  # noqa: E402


def timed(fn, reps=3):
    fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        r = fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts)), r


def main():
    net = synth.trained_net("torus")
    print(json.dumps({"refine_band": sp.net_refine_band(net)}), flush=True)
    n = 1 << 22
    for h in (64, 128, 256, 512):
        row = {"case": f"cubes_1/{h}", "n": n}
        labs = {}
        for prec in ("fp32", "fp32-refine", "fp64"):
            ms, (lo, hi, cls) = timed(lambda: sp.bound_random_cubes(net, n, seed=3, half=1.0 / h, precision=prec))
            labs[prec] = cls
            row[prec] = {"ms": round(ms, 3), "certified": float((cls != 0).float().mean())}
        row["refine_labels_equal_fp64"] = bool(torch.equal(labs["fp32-refine"], labs["fp64"]))
        row["fp32_lost_vs_fp64"] = float(((labs["fp32"] == 0) & (labs["fp64"] != 0)).float().mean())
        print(json.dumps(row), flush=True)
    b = spatial.AABB(-np.ones(3), np.ones(3))
    for depth in (18, 21, 24):
        row = {"case": f"tree_depth{depth}"}
        res = {}
        for prec in ("fp32", "fp32-refine", "fp64"):
            ms, a = timed(lambda: spatial.build_spatial_tree_arrays(net, b, policy=sp.AFFINE_FIXED, max_depth=depth,
                                                                    precision=prec, to_host=False), reps=1)
            n_cert = sum(int((lv.label != 0).sum().item()) for lv in a.levels)
            res[prec] = [len(lv.label) for lv in a.levels]
            row[prec] = {"ms": round(ms, 2), "nodes": a.n_nodes, "certified_nodes": n_cert,
                         "node_bounds_per_s": a.n_nodes / ms * 1e3}
            del a
            torch.cuda.empty_cache()
        row["refine_topology_equals_fp64"] = res["fp32-refine"] == res["fp64"]
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
