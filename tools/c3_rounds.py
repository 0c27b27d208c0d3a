"""K6 tail analysis: per-round active rays and host
time of the C3 SIREN march (FP64, default camera), from spk_march_round_log.
Reports the share of time spent in tail rounds (active < 10% / 1% of the
rays) and the fixed per-round cost (launches + count read-back + one
synchronisation), measured on rounds with almost no work.

    python tools/c3_rounds.py [res] [policy]   -> one JSON line
"""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2202_02444_b200 as sp  # noqa: E402
from paper_2202_02444_b200 import rays, synth  # noqa: E402
from paper_2202_02444_b200.camera import default_camera  # noqa: E402

res = int(sys.argv[1]) if len(sys.argv) > 1 else 256
pol = sys.argv[2] if len(sys.argv) > 2 else "interval"
net = synth.config_net("C3")
sp.cast_camera(net, default_camera(16), sp.RayCastParams(), pol, precision="fp64")
torch.cuda.synchronize()
t0 = time.perf_counter()
hit, t, steps, st = sp.cast_camera(net, default_camera(res), sp.RayCastParams(), pol, precision="fp64")
torch.cuda.synchronize()
wall = time.perf_counter() - t0
active, ms = rays.last_march_rounds()
n = res * res
tot = float(ms.sum())
tail10 = active < 0.10 * n
tail1 = active < 0.01 * n
small = active <= 256
fixed = float(np.median(ms[small])) if small.any() else None
# ideal time of the rounds at full-round efficiency: per-ray-step cost of the big rounds
big = active >= 0.5 * n
per_step = float(ms[big].sum() / active[big].sum()) if big.any() else None
print(json.dumps({
    "res": res, "policy": pol, "rays": n, "rounds": int(len(ms)), "ray_steps": int(active.sum()),
    "wall_ms": 1e3 * wall, "rounds_ms": tot,
    "tail10_rounds": int(tail10.sum()), "tail10_ms": float(ms[tail10].sum()), "tail10_share": float(ms[tail10].sum() / tot),
    "tail1_rounds": int(tail1.sum()), "tail1_ms": float(ms[tail1].sum()), "tail1_share": float(ms[tail1].sum() / tot),
    "fixed_ms_per_round": fixed, "fixed_share": (fixed * len(ms) / tot) if fixed else None,
    "per_ray_step_us_full_rounds": 1e3 * per_step if per_step else None,
    "tail10_ideal_ms": float(active[tail10].sum() * per_step) if per_step else None,
    "active_by_round_every10": active[::10].tolist(),
}))
