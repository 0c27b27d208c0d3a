"""Distribution of the FP32 affine-fixed excess over the FP64 enclosure, per
box, relative to the box's FP32 width and to S + w -- the data behind the
fp32-refine candidate rule.  Usage:
python tools/excess_dist.py"""

import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2202_02444_b200 as sp  # noqa: E402
from paper_2202_02444_b200 import spatial, synth  # noqa: E402


def report(tag, lo32, hi32, lo64, hi64):
    w32 = hi32 - lo32
    s = np.maximum(1.0, np.maximum(np.abs(lo32), np.abs(hi32)))
    ex = np.maximum(lo64 - lo32, hi32 - hi64)
    unk = (lo32 <= 0) & (hi32 >= 0)
    gain = unk & ((lo64 > 0) | (hi64 < 0))  # FP64 certifies, FP32 does not
    q = lambda a: [float(np.quantile(a, p)) for p in (0.5, 0.99, 1.0)] if a.size else None
    margin = np.minimum(-lo32, hi32)  # distance of the nearer end from zero (UNKNOWN boxes)
    out = {"case": tag, "n": int(lo32.size), "ex_over_w32": q(ex / w32), "ex_over_Sw": q(ex / (s + w32)),
           "gain": int(gain.sum()),
           "gain_margin_over_w32": q(margin[gain] / w32[gain]),
           "gain_margin_over_Sw": q(margin[gain] / (s[gain] + w32[gain]))}
    for k in (0.02, 0.05, 0.1, 0.2):
        out[f"cand_frac_w32_{k}"] = float((unk & (margin <= k * w32)).mean())
    print(json.dumps(out), flush=True)


def c5(tag, n, net=None, half=1 / 64):
    net = net if net is not None else synth.config_net(tag)
    r = {}
    for prec in ("fp32", "fp64"):
        lo, hi, _ = sp.bound_random_cubes(net, n, seed=1, half=half, precision=prec)
        r[prec] = (lo.cpu().numpy(), hi.cpu().numpy())
    report(tag, *r["fp32"], *r["fp64"])


def c2(depth=18):
    net = synth.config_net("C2")
    b = spatial.AABB(-np.ones(3), np.ones(3))
    a = spatial.build_spatial_tree_arrays(net, b, policy=sp.AFFINE_FIXED, max_depth=depth, precision="fp32",
                                          to_host=True)
    for d in (12, 15, depth):
        lv = a.levels[d]
        lo64, hi64, _ = sp.bound_aabb(net, torch.from_numpy(lv.lo).cuda(), torch.from_numpy(lv.hi).cuda(),
                                      precision="fp64")
        report(f"C2_level{d}", lv.bound_lo, lv.bound_hi, lo64.cpu().numpy(), hi64.cpu().numpy())


if __name__ == "__main__":
    c2()
    c5("C5_64", 1 << 20)
    c5("C5_256", 1 << 20)
    c5("C5_512", 1 << 18)
    c5("C1", 1 << 20)
    nets = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "nets")
    for f in sorted(os.listdir(nets)):
        net = sp.load_network(os.path.join(nets, f))
        for half in (1 / 64, 1 / 16):
            c5(f"{f[:-5]}_h{int(1 / half)}", 1 << 18, net, half)
