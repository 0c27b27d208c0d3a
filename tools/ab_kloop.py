"""A/B timings of the fused bound pass across widths (run twice: default
library and SPK_LIB_PATH=var/<name>/_spk.so)."""
import json
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2202_02444_b200 as sp  # noqa: E402
from paper_2202_02444_b200 import synth  # noqa: E402


def timed(fn, reps=5):
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


res = {}
net = synth.config_net("C2")
c, _ = synth.grid_cubes(64)
lo = torch.from_numpy(c - 1 / 64).cuda()
hi = torch.from_numpy(c + 1 / 64).cuda()
res["c2level_ms"] = timed(lambda: sp.bound_aabb(net, lo, hi, sp.AFFINE_FIXED))
l2, h2, _ = sp.bound_aabb(net, lo, hi, sp.AFFINE_FIXED)
res["c2level_width_mean"] = float((h2 - l2).mean().item())
res["interval_2M_ms"] = timed(lambda: sp.bound_random_cubes(net, 1 << 21, seed=1, half=1 / 64,
                                                            policy=sp.INTERVAL_ONLY))
x = torch.rand((1 << 22, 3), device="cuda", dtype=torch.float64) * 2 - 1
res["eval256_4M_ms"] = timed(lambda: sp.eval_batch(net, x, precision="fp32"))
for tag, n in (("C5_64", 1 << 24), ("C5_512", 1 << 19)):
    nt = synth.config_net(tag)
    res[tag + "_ms"] = timed(lambda: sp.bound_random_cubes(nt, n, seed=1, half=1 / 64))
n1 = synth.config_net("C1")
cg, ag = synth.grid_cubes(64)
ct, at = torch.from_numpy(cg).cuda(), torch.from_numpy(ag).cuda()
res["C1_ms"] = timed(lambda: sp.range_bound_batch(n1, ct, at, sp.AFFINE_FIXED), reps=20)
print(json.dumps(res))
