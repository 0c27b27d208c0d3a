"""Range-marching ray casting on the trained 8x256 torus SDF (the C3 image
size, 1024^2, the reference bench camera, RayCastParams() defaults) in FP32
and FP64, interval and affine-fixed: rays/s, steps per ray, and agreement
(hit flags equal; |t32 - t64| <= delta where both hit).  The C3 SIREN config
is FP64-only (its outputs sit at 1e-11); this shows the FP32 march on a net
with a real surface.  One JSON line per case.

    python tools/trained_rays.py [res]
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2202_02444_b200 as sp  # noqa: E402
from paper_2202_02444_b200 import synth  # noqa: E402
from paper_2202_02444_b200.camera import default_camera  # noqa: E402


def main():
    res = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    net = synth.trained_net("torus")
    cam = default_camera(res)
    params = sp.RayCastParams()
    for policy in ("interval", "affine-fixed"):
        out = {}
        for prec in ("fp64", "fp32"):
            sp.cast_camera(net, default_camera(64), params, policy, precision=prec)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            hit, t, steps, st = sp.cast_camera(net, cam, params, policy, precision=prec)
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b)
            out[prec] = (hit.cpu().numpy(), t.cpu().numpy(), steps.cpu().numpy(), ms)
        h64, t64, s64, ms64 = out["fp64"]
        h32, t32, s32, ms32 = out["fp32"]
        both = h64 & h32
        dt = np.abs(t32[both] - t64[both])
        print(json.dumps({
            "case": f"torus 8x256 rays {res}^2 {policy}", "rays": res * res,
            "fp64": {"ms": ms64, "rays_per_s": res * res / ms64 * 1e3, "hit_fraction": float(h64.mean()),
                     "steps_per_ray": float(s64.mean())},
            "fp32": {"ms": ms32, "rays_per_s": res * res / ms32 * 1e3, "hit_fraction": float(h32.mean()),
                     "steps_per_ray": float(s32.mean())},
            "hit_flags_equal": float((h32 == h64).mean()), "max_dt_where_both_hit": float(dt.max()) if dt.size else 0.0,
            "delta": params.delta}), flush=True)


if __name__ == "__main__":
    main()
