"""FP32 enclosure excess over the FP64 kernel (within 1e-9 of the reference)
on the C5 cube workloads, for A/B builds of the library (SPK_LIB_PATH): used
with the measurement-only SPK_DEBUG_GAMMA_KEEP_MASK variants to attribute the
excess to the rounding budgets of individual layers, and to evaluate budget
changes.  Prints one JSON line per net.

    SPK_LIB_PATH=var/g_keep1/_spk.so python tools/excess_attrib.py
"""
import json
import os
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2202_02444_b200 as sp  # noqa: E402
from paper_2202_02444_b200 import synth  # noqa: E402

n = 1 << 14
for tag in ("C5_64", "C5_256", "C5_512"):
    net = synth.config_net(tag)
    lo, hi, cls = sp.bound_random_cubes(net, n, seed=1, half=1 / 64)
    l64, h64, c64 = sp.bound_random_cubes(net, n, seed=1, half=1 / 64, precision="fp64")
    lo, hi, cls, l64, h64, c64 = (t.cpu().numpy() for t in (lo, hi, cls, l64, h64, c64))
    w = h64 - l64
    S = np.maximum(1, np.maximum(np.abs(l64), np.abs(h64)))
    d = np.maximum(np.abs(lo - l64), np.abs(hi - h64))
    print(json.dumps({"lib": os.environ.get("SPK_LIB_PATH", "in-tree"), "net": tag,
                      "rel_Sw_max": float((d / (S + w)).max()), "rel_Sw_median": float(np.median(d / (S + w))),
                      "rel_w_max": float((d / w).max()), "rel_w_median": float(np.median(d / w)),
                      "cert32": float((cls != 0).mean()), "cert64": float((c64 != 0).mean())}), flush=True)
