"""Cost / effect of precision="fp32-refine" against plain FP32 and FP64.

For the C2 depth-18 tree and the C5 cube streams, at several refine bands:
device time (CUDA events, L2 not flushed -- relative numbers), certified
fraction, and the fraction of boxes whose bound the FP64 pass rewrote.
Prints one JSON line per case.  Usage: python tools/refine_probe.py
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


def c5(tag, n, taus):
    net = synth.config_net(tag)
    res = {}
    for prec in ["fp32", "fp64"]:
        ms, (lo, hi, cls) = timed(lambda: sp.bound_random_cubes(net, n, seed=1, half=1 / 64, precision=prec))
        res[prec] = (ms, lo.clone(), cls.clone())
        print(json.dumps({"case": tag, "n": n, "precision": prec, "ms": ms,
                          "certified": float((cls != 0).float().mean())}), flush=True)
    for tau in taus:
        sp.refine_band(tau)
        if tau == "auto":  # calibrate outside the timed region
            print(json.dumps({"case": tag, "calibrated_band": sp.net_refine_band(net)}), flush=True)
        ms, (lo, hi, cls) = timed(lambda: sp.bound_random_cubes(net, n, seed=1, half=1 / 64, precision="fp32-refine"))
        rewritten = float((lo != res["fp32"][1]).float().mean())
        agree = float((cls == res["fp64"][2]).float().mean())
        print(json.dumps({"case": tag, "n": n, "precision": "fp32-refine", "tau": tau, "ms": ms,
                          "certified": float((cls != 0).float().mean()), "rewritten": rewritten,
                          "labels_equal_fp64": agree}), flush=True)


def c2(taus, depth=18):
    net = synth.config_net("C2")
    b = spatial.AABB(-np.ones(3), np.ones(3))
    run = lambda prec: spatial.build_spatial_tree_arrays(net, b, policy=sp.AFFINE_FIXED, max_depth=depth,
                                                         precision=prec, to_host=False)
    ms32, a32 = timed(lambda: run("fp32"), 2)
    print(json.dumps({"case": "C2", "precision": "fp32", "ms": ms32, "nodes": a32.n_nodes}), flush=True)
    for tau in taus:
        sp.refine_band(tau)
        if tau == "auto":
            print(json.dumps({"case": "C2", "calibrated_band": sp.net_refine_band(net)}), flush=True)
        ms, a = timed(lambda: run("fp32-refine"), 2)
        lv = a.levels[-1]
        print(json.dumps({"case": "C2", "precision": "fp32-refine", "tau": tau, "ms": ms, "nodes": a.n_nodes}),
              flush=True)


if __name__ == "__main__":
    taus = ["auto", 0.0, 0.003, 0.01, 0.06]
    c2(taus)
    c5("C5_64", 4 << 20, taus)
    c5("C5_256", 4 << 20, taus)
    c5("C5_512", 1 << 20, taus)
    sp.refine_band("auto")
