"""One warm FP32 point-evaluation launch through the C4 net (8x512 ELU)."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2202_02444_b200 as sp  # noqa: E402
from paper_2202_02444_b200 import synth  # noqa: E402

net = synth.config_net("C4")
x = torch.rand((1 << 21, 3), dtype=torch.float64, device="cuda") * 2 - 1
for _ in range(4):
    sp.eval_batch(net, x, precision="fp32")
torch.cuda.synchronize()
