"""Diagnostics printed on the GPU box (always passes when the kernels run):
FP32-vs-reference error statistics used to state the tolerances."""

import numpy as np
import pytest

import paper_2202_02444_b200 as sp

pytestmark = pytest.mark.gpu


def test_print_fp32_error_stats(golden, net_paths):
    for name, path in sorted(net_paths.items()):
        net = sp.load_network(path)
        c, a = golden[f"bounds/{name}/centers"], golden[f"bounds/{name}/axes"]
        for pol in ("interval", "affine-fixed"):
            lo, hi = sp.range_bound_batch(net, c, a, pol, precision="fp32")
            lo64, hi64 = sp.range_bound_batch(net, c, a, pol, precision="fp64")
            wl, wh = golden[f"bounds/{name}/{pol}/lo"], golden[f"bounds/{name}/{pol}/hi"]
            w = (wh - wl) + np.maximum(1, np.maximum(abs(wl), abs(wh)))
            print(f"STAT {name:10s} {pol:13s} fp32 rel {np.max(np.abs(lo-wl)/w):.2e} {np.max(np.abs(hi-wh)/w):.2e}"
                  f" | fp64 {np.max(np.abs(lo64-wl)/w):.2e} {np.max(np.abs(hi64-wh)/w):.2e}"
                  f" | widen32 {np.median((hi-lo)/(wh-wl+1e-300)):.6f}")
