"""Point-eval timings of non-ReLU nets (A/B with SPK_LIB_PATH)."""
import json, sys
sys.path.insert(0, ".")
import torch
import paper_2202_02444_b200 as sp
from paper_2202_02444_b200 import synth


def timed(fn, reps=3):
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


x = torch.rand((1 << 22, 3), device="cuda", dtype=torch.float64) * 2 - 1
res = {}
for tag in ("C4", "C3"):
    net = synth.config_net(tag)
    res[f"{tag}_eval_4M_fp32_ms"] = timed(lambda: sp.eval_batch(net, x, precision="fp32"))
sdf = sp.load_network("tests/golden/nets/elu_sdf.json")
res["elu_sdf_eval_4M_fp32_ms"] = timed(lambda: sp.eval_batch(sdf, x, precision="fp32"))
print(json.dumps(res))
