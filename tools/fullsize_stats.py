import sys; sys.path.insert(0,'.')
import numpy as np
import paper_2202_02444_b200 as sp
from oracle import spelunk_oracle as orc
from paper_2202_02444_b200 import spatial, synth
net = synth.config_net("C2")
arr = spatial.build_spatial_tree_arrays(net, spatial.AABB(-np.ones(3), np.ones(3)), policy=sp.AFFINE_FIXED, max_depth=18, precision="fp32", to_host=False)
onet = orc.as_oracle_net(net); rng = np.random.default_rng(11)
for k, lv in enumerate(arr.levels):
    n=len(lv); idx=rng.choice(n, size=min(n,256), replace=False)
    lo, hi = lv.lo.cpu().numpy()[idx], lv.hi.cpu().numpy()[idx]
    glo, ghi = lv.bound_lo.cpu().numpy()[idx], lv.bound_hi.cpu().numpy()[idx]
    wl, wh = orc.bound_aabbs(onet, lo, hi, "affine-fixed")
    s = np.maximum(1.0, np.maximum(np.abs(wl), np.abs(wh))) + (wh - wl)
    r = np.maximum(np.abs(glo-wl), np.abs(ghi-wh))/s
    print(k, "max rel %.2e" % r.max(), "width %.3g" % np.median(wh-wl), "sound", bool(np.all(glo <= wl+1e-12*s) and np.all(ghi >= wh-1e-12*s)))
