"""One warm launch of a fused bound kernel, for ncu captures.

    python tools/prof_one.py c2level   # depth-18 level of C2 (262,144 AABBs, 8x256 ReLU, affine-fixed)
    python tools/prof_one.py c5 [n]    # n on-device cubes through 8x256 (default 2^20)
    python tools/prof_one.py c1        # 64^3 grid through 4x32
    python tools/prof_one.py c5_64 [n] # n on-device cubes through 8x64 (default 2^20)
    python tools/prof_one.py c5_512 [n] # n on-device cubes through 8x512 (default 2^17)
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2202_02444_b200 as sp  # noqa: E402
from paper_2202_02444_b200 import synth  # noqa: E402


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "c2level"
    torch.cuda.set_device(0)
    if which == "c2level":
        net = synth.config_net("C2")
        c, a = synth.grid_cubes(64)
        lo_c = torch.from_numpy(c - 1 / 64).cuda()
        hi_c = torch.from_numpy(c + 1 / 64).cuda()
        run = lambda: sp.bound_aabb(net, lo_c, hi_c, sp.AFFINE_FIXED)
    elif which == "small":  # a top tree level: one sibling pair (the SM = 1 small tile, one CTA)
        n = int(sys.argv[2]) if len(sys.argv) > 2 else 2
        net = synth.config_net("C2")
        c, a = synth.grid_cubes(64)
        lo_c = torch.from_numpy(c[:n] - 1 / 64).cuda()
        hi_c = torch.from_numpy(c[:n] + 1 / 64).cuda()
        run = lambda: sp.bound_aabb(net, lo_c, hi_c, sp.AFFINE_FIXED)
    elif which == "c5":
        n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 20
        net = synth.config_net("C5_256")
        run = lambda: sp.bound_random_cubes(net, n, seed=1, half=1 / 64)
    elif which in ("c5_64", "c5_512"):
        n = int(sys.argv[2]) if len(sys.argv) > 2 else (1 << 20 if which == "c5_64" else 1 << 17)
        net = synth.config_net("C5_64" if which == "c5_64" else "C5_512")
        run = lambda: sp.bound_random_cubes(net, n, seed=1, half=1 / 64)
    elif which in ("eval256", "eval512"):
        net = synth.config_net("C2" if which == "eval256" else "C4")
        n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 22
        x = torch.rand((n, 3), dtype=torch.float64, device="cuda") * 2 - 1
        run = lambda: sp.eval_batch(net, x, precision="fp32")
    elif which == "c5interval":
        n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 22
        net = synth.config_net("C5_256")
        run = lambda: sp.bound_random_cubes(net, n, seed=1, half=1 / 64, policy=sp.INTERVAL_ONLY)
    elif which == "c5trunc":
        n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 18
        net = synth.config_net("C5_256")
        c = torch.rand((n, 3), dtype=torch.float64, device="cuda") * 2 - 1
        a = torch.zeros((n, 1, 3), dtype=torch.float64, device="cuda")
        a[:, 0, 0] = 1 / 64
        run = lambda: sp.range_bound_batch(net, c, a, sp.affine_truncate(16))
    else:
        net = synth.config_net("C1")
        c, a = synth.grid_cubes(64)
        ct, at = torch.from_numpy(c).cuda(), torch.from_numpy(a).cuda()
        run = lambda: sp.range_bound_batch(net, ct, at, sp.AFFINE_FIXED)
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{which}: {ms:.3f} ms")


if __name__ == "__main__":
    main()
