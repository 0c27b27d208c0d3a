"""Train a non-degenerate 3->8x256->1 ReLU SDF net (the C2 architecture) for
the FP32-vs-FP64 certification study: the random-init configs certify
nothing, so they cannot show what the FP32 rounding budget costs in labels.

Target: the signed distance of a torus (R = 0.5, r = 0.2) over [-1, 1]^3,
fitted with Adam (lr 1e-3 -> 1e-4, 800 steps, batches of 8192, seed 0) in
FP32 on the CPU.  The weights are FP32 values, stored as FP32 in
tests/golden/nets/torus_8x256.npz (loaded by synth.trained_net("torus")).

    python tools/train_sdf_net.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def torus_sdf(p, R=0.5, r=0.2):
    q = torch.stack([torch.linalg.norm(p[:, [0, 2]], dim=1) - R, p[:, 1]], dim=1)
    return torch.linalg.norm(q, dim=1) - r


def main():
    torch.manual_seed(0)
    torch.use_deterministic_algorithms(True)
    torch.set_num_threads(os.cpu_count() or 8)
    dims = [3] + [256] * 8 + [1]
    mods = []
    for i in range(len(dims) - 1):
        mods.append(torch.nn.Linear(dims[i], dims[i + 1]))
        if i < len(dims) - 2:
            mods.append(torch.nn.ReLU())
    net = torch.nn.Sequential(*mods)
    opt = torch.optim.Adam(net.parameters(), lr=1e-3)
    steps = 800
    sched = torch.optim.lr_scheduler.CosineAnnealingLR(opt, steps, eta_min=1e-4)
    g = torch.Generator().manual_seed(1)
    for it in range(steps):
        x = torch.rand(8192, 3, generator=g) * 2 - 1
        loss = torch.nn.functional.mse_loss(net(x).squeeze(1), torch_sdf := torus_sdf(x))
        opt.zero_grad()
        loss.backward()
        opt.step()
        sched.step()
        if it % 100 == 0 or it == steps - 1:
            print(f"step {it} loss {loss.item():.3e}", flush=True)
    arrays = {}
    k = 0
    for m in net:
        if isinstance(m, torch.nn.Linear):
            arrays[f"W{k}"] = m.weight.detach().numpy().astype(np.float32)
            arrays[f"b{k}"] = m.bias.detach().numpy().astype(np.float32)
            k += 1
    out = os.path.join(ROOT, "tests", "golden", "nets", "torus_8x256.npz")
    np.savez_compressed(out, **arrays)
    with torch.no_grad():
        x = torch.rand(100000, 3, generator=g) * 2 - 1
        err = (net(x).squeeze(1) - torus_sdf(x)).abs()
    print(f"saved {out}: max |f - sdf| {err.max():.3e}, mean {err.mean():.3e}")


if __name__ == "__main__":
    sys.exit(main())
