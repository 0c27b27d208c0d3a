"""A/B of width-64 FP32 paths (W tile rows, Morton order): C5_64 random
cubes (affine-fixed, interval), point evaluation; bounds saved for a
bit-exact comparison between library builds.

    SPK_LIB_PATH=var/<v>/_spk.so python tools/ab_w64.py OUT.npz
"""
import json
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2202_02444_b200 as sp  # noqa: E402
from paper_2202_02444_b200 import synth  # noqa: E402
from tools.ab_live_warp import timed  # noqa: E402


def main():
    out, res = {}, {}
    net = synth.config_net("C5_64")
    for tag, pol in (("fixed", sp.AFFINE_FIXED), ("interval", sp.parse_policy("interval"))):
        lo, hi, _ = sp.bound_random_cubes(net, 1 << 20, seed=5, policy=pol)
        out[f"{tag}_lo"], out[f"{tag}_hi"] = lo.cpu().numpy(), hi.cpu().numpy()
        n = 1 << 24
        res[f"c5_64_{tag}_16M_ms"] = timed(lambda: sp.bound_random_cubes(net, n, seed=1, policy=pol), reps=3)
        res[f"c5_64_{tag}_boxes_per_s"] = n / res[f"c5_64_{tag}_16M_ms"] * 1e3
    x = torch.rand((1 << 22, 3), device="cuda", dtype=torch.float64) * 2 - 1
    out["eval"] = sp.eval_batch(net, x[: 1 << 16], precision="fp32").cpu().numpy()
    res["eval_4M_ms"] = timed(lambda: sp.eval_batch(net, x, precision="fp32"))
    np.savez(sys.argv[1], **out)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
