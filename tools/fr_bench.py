"""Frustum casting timing probe (C3 SIREN net, default camera)."""
import json
import sys
import time

sys.path.insert(0, '.')
import torch  # noqa: E402

import paper_2202_02444_b200 as sp  # noqa: E402
from paper_2202_02444_b200 import synth  # noqa: E402
from paper_2202_02444_b200.camera import default_camera  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
net = sp.load_network(cfg) if cfg.endswith(".json") else synth.config_net(cfg)
for res in [int(r) for r in (sys.argv[2] if len(sys.argv) > 2 else "32,64,128").split(",")]:
    for pol in (sys.argv[3] if len(sys.argv) > 3 else "affine-fixed,interval").split(","):
        t0 = time.time()
        fr = sp.cast_frustum_image(net, default_camera(res), sp.RayCastParams(), pol, precision="fp32",
                                   device_output=True)
        torch.cuda.synchronize()
        dt = time.time() - t0
        t1 = time.time()
        hit, t, steps, st = sp.cast_camera(net, default_camera(res), sp.RayCastParams(), pol, precision="fp32")
        torch.cuda.synchronize()
        print(json.dumps({"res": res, "pol": pol, "frustum_s": round(dt, 3), "perray_s": round(time.time() - t1, 3),
                          **fr.stats.meta, "handoff_steps": fr.stats.ray_steps,
                          "amort": float(fr.steps.sum()) / res / res, "perray_steps": st.ray_steps / res / res}),
              flush=True)
