"""A/B of the narrow-net (width 32) live-row masks: bounds of C1 and random
cubes through width-32 ReLU nets, saved for a bit-exact comparison between two
library builds, plus CUDA-event timings.

    python tools/ab_live_warp.py OUT.npz            # in-tree library
    SPK_LIB_PATH=var/nolw/_spk.so python tools/ab_live_warp.py OUT.npz
"""
import json
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2202_02444_b200 as sp  # noqa: E402
from paper_2202_02444_b200 import synth  # noqa: E402


def timed(fn, reps=7):
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


def main():
    out = {}
    res = {}
    c1 = synth.config_net("C1")
    sdf = sp.load_network("tests/golden/nets/relu_sdf.json")
    gc, ga = synth.grid_cubes(64)
    gc, ga = torch.from_numpy(gc).cuda(), torch.from_numpy(ga).cuda()
    for tag, pol in (("fixed", sp.AFFINE_FIXED), ("interval", sp.parse_policy("interval"))):
        lo, hi = sp.range_bound_batch(c1, gc, ga, pol)
        out[f"c1_{tag}_lo"], out[f"c1_{tag}_hi"] = np.asarray(lo.cpu()), np.asarray(hi.cpu())
        res[f"c1_{tag}_ms"] = timed(lambda: sp.range_bound_batch(c1, gc, ga, pol))
    for name, net in (("c1net", c1), ("sdf", sdf)):
        for half in (1 / 64, 1 / 8):
            lo, hi, cls = sp.bound_random_cubes(net, 1 << 20, seed=5, half=half)
            out[f"cubes_{name}_{half}_lo"] = lo.cpu().numpy()
            out[f"cubes_{name}_{half}_hi"] = hi.cpu().numpy()
        n = 1 << 24
        res[f"cubes16M_{name}_ms"] = timed(lambda: sp.bound_random_cubes(net, n, seed=1), reps=3)
        res[f"cubes16M_{name}_boxes_per_s"] = n / res[f"cubes16M_{name}_ms"] * 1e3
    res["c1_boxes_per_s"] = 262144 / res["c1_fixed_ms"] * 1e3
    np.savez(sys.argv[1], **out)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
