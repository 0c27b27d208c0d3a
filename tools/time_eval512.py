"""CUDA-event timing of FP32 point evaluation through the C4 net (8x512 ELU)."""
import json
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2202_02444_b200 as sp  # noqa: E402
from paper_2202_02444_b200 import synth  # noqa: E402

net = synth.config_net("C4")
x = torch.rand((1 << 22, 3), dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(0)) * 2 - 1
sp.eval_batch(net, x, precision="fp32")
torch.cuda.synchronize()
best = 1e9
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    y = sp.eval_batch(net, x, precision="fp32")
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
ref = sp.eval_batch(net, x, precision="fp64")
err = float(((y - ref).abs() / ref.abs().clamp(min=1.0)).max().item())
print(json.dumps({"eval512_4M_ms": best, "evals_per_s": (1 << 22) / best * 1e3, "max_rel_err_vs_fp64": err}))
