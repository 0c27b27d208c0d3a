"""Diagnose the frustum loop: oracle control flow, GPU FP32 bounds."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_2202_02444_b200 as sp
from paper_2202_02444_b200 import synth
from paper_2202_02444_b200.camera import default_camera
from oracle import spelunk_oracle as orc

net = synth.config_net(sys.argv[1] if len(sys.argv) > 1 else "C3")
res = int(sys.argv[2]) if len(sys.argv) > 2 else 32
prec = sys.argv[3] if len(sys.argv) > 3 else "fp32"
rounds = [0]
t0 = time.time()
def gpu_bound(onet, centres, axes, policy):
    rounds[0] += 1
    lo, hi = sp.range_bound_batch(net, centres, axes, policy, precision=prec)
    if rounds[0] % 50 == 1 or rounds[0] < 5:
        ext = np.abs(axes).sum(axis=(1, 2))
        print(f"round {rounds[0]} n={len(lo)} t={time.time()-t0:.1f}s ext[min,max]=({ext.min():.3g},{ext.max():.3g}) "
              f"width[min]={np.min(hi-lo):.3g} lo/hi sample={lo[:2]},{hi[:2]} nan={np.isnan(lo).sum()}", flush=True)
    if rounds[0] > 3000:
        raise SystemExit("too many rounds")
    return lo, hi
orc.bound_batch = gpu_bound
cam = default_camera(res)
print("f(pos) =", sp.eval_batch(net, cam.position[None, :]), flush=True)
h, t, s = orc.frustum_cast(orc.as_oracle_net(net), cam.position, cam.look_at, cam.up, cam.vertical_fov, res, res,
                           orc.MarchParams(), "affine-fixed", 16)
print("done rounds", rounds[0], "hits", h.sum(), time.time() - t0)
