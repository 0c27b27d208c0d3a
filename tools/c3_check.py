"""C3 SIREN: GPU FP64 march vs the oracle on a 16x16 default-camera view."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_2202_02444_b200 as sp
from paper_2202_02444_b200 import synth
from paper_2202_02444_b200.camera import default_camera
from oracle import spelunk_oracle as orc
net = synth.config_net("C3")
cam = default_camera(16)
for pol in ("interval", "affine-fixed"):
    h, t, s, st = sp.cast_camera(net, cam, sp.RayCastParams(), pol, precision="fp64")
    dirs = cam.pixel_dirs().reshape(-1, 3)
    t0 = time.time()
    oh, ot, os_ = orc.march(orc.as_oracle_net(net), np.broadcast_to(cam.position, dirs.shape).copy(), dirs,
                            orc.MarchParams(), pol)
    print(pol, "gpu steps/ray", float(s.sum()) / 256, "oracle", os_.sum() / 256, "same t:",
          bool(np.array_equal(t.cpu().numpy().reshape(-1), ot)), "oracle s", round(time.time() - t0, 1))
