"""FP32 vs FP64 enclosure on every golden net (reference golden vectors):
FP64 kernels within 1e-10 * S of the reference; FP32 kernels within
tau * (S + w) of it (tau as in test_gpu_bounds.py).  Where the FP32 and FP64
enclosures are computed by inclusion-monotone rules -- interval arithmetic on
every net, and affine-fixed on pure-ReLU nets -- FP32 also CONTAINS the FP64
enclosure (never tighter, up to the FP64 rounding 1e-12 * S).  (ELU / sin /
tanh affine rules pick their slope from the input range, so a looser FP32
input can legitimately give a tighter output on one side.)  The measured
maxima are printed for DESIGN.md §2."""

import numpy as np
import pytest

import paper_2202_02444_b200 as sp

pytestmark = pytest.mark.gpu


def test_fp32_contains_fp64_on_golden_nets(golden, net_paths):
    for name, path in sorted(net_paths.items()):
        net = sp.load_network(path)
        kinds = {getattr(l, "value", l) for l in net.layers if not hasattr(l, "weights")}
        tau = 1e-2 if "sin" in kinds else 3e-3
        c, a = golden[f"bounds/{name}/centers"], golden[f"bounds/{name}/axes"]
        for pol in ("interval", "affine-fixed"):
            lo, hi = sp.range_bound_batch(net, c, a, pol, precision="fp32")
            lo64, hi64 = sp.range_bound_batch(net, c, a, pol, precision="fp64")
            wl, wh = golden[f"bounds/{name}/{pol}/lo"], golden[f"bounds/{name}/{pol}/hi"]
            s = np.maximum(1, np.maximum(abs(wl), abs(wh)))
            w = (wh - wl) + s
            assert np.max(np.abs(lo64 - wl) / s) <= 1e-10 and np.max(np.abs(hi64 - wh) / s) <= 1e-10, (name, pol)
            if pol == "interval" or kinds <= {"relu", "identity"}:
                assert np.all(lo <= lo64 + 1e-12 * s) and np.all(hi >= hi64 - 1e-12 * s), (name, pol)
            e32 = max(np.max(np.abs(lo - wl) / w), np.max(np.abs(hi - wh) / w))
            assert e32 <= tau, (name, pol, e32)
            print(f"STAT {name:10s} {pol:13s} fp32 rel {e32:.2e} | fp64 "
                  f"{max(np.max(np.abs(lo64 - wl) / w), np.max(np.abs(hi64 - wh) / w)):.2e}"
                  f" | widen32 {np.median((hi - lo) / (wh - wl + 1e-300)):.6f}")
