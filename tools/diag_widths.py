"""Diagnostic (not a test): FP32 vs FP64 vs oracle bound statistics on
3-layer width-256/512 nets, printed on the GPU box:

    python -m pytest tools/diag_widths.py -s
"""

import numpy as np
import pytest

import paper_2202_02444_b200 as sp
from oracle import spelunk_oracle as orc
from paper_2202_02444_b200 import synth



@pytest.mark.parametrize("width", [256, 512])
def test_print_width_stats(width):
    rng = np.random.default_rng(1)
    net = synth.random_mlp(width, 3, "relu", "ref-normal", seed=width)
    c = rng.uniform(-1, 1, (300, 3))
    a = np.zeros((300, 3, 3))
    a[:, np.arange(3), np.arange(3)] = 10.0 ** rng.uniform(-3, -1, (300, 1))
    for policy in ("interval", "affine-fixed"):
        wl, wh = orc.bound_batch(orc.as_oracle_net(net), c, a, policy)
        l64, h64 = sp.range_bound_batch(net, c, a, policy, precision="fp64")
        l32, h32 = sp.range_bound_batch(net, c, a, policy, precision="fp32")
        s = np.maximum(1, np.maximum(abs(wl), abs(wh))) + (wh - wl)
        e = np.abs(l32 - wl) / s
        i = int(np.argmax(e))
        print(f"DIAG w={width} {policy}: fp32 max rel {e.max():.3e} at {i}: ref [{wl[i]:.6g},{wh[i]:.6g}] "
              f"fp64 [{l64[i]:.6g},{h64[i]:.6g}] fp32 [{l32[i]:.6g},{h32[i]:.6g}]; "
              f"tighter-than-fp64 count lo {(l32 > l64 + 1e-9 * s).sum()} hi {(h32 < h64 - 1e-9 * s).sum()}")
