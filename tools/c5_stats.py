import sys; sys.path.insert(0,'.')
import numpy as np
import paper_2202_02444_b200 as sp
from oracle import spelunk_oracle as orc
from paper_2202_02444_b200 import synth
net = synth.config_net("C5_256"); onet = orc.as_oracle_net(net)
n = 1 << 16
lo, hi, _ = sp.bound_random_cubes(net, n, seed=1, half=1 / 64)
idx = np.random.default_rng(5).choice(n, size=1024, replace=False)
c = np.concatenate([synth.random_cube_centres(1, 1, int(i)) for i in idx])
wl, wh = orc.bound_aabbs(onet, c - 1/64, c + 1/64, "affine-fixed")
glo, ghi = lo.cpu().numpy()[idx], hi.cpu().numpy()[idx]
d = np.maximum(np.abs(glo - wl), np.abs(ghi - wh)); w = wh - wl; S = np.maximum(1, np.maximum(np.abs(wl), np.abs(wh)))
print("abs excess: max %.3f median %.3f" % (d.max(), np.median(d)))
print("rel to S+w: max %.3f median %.4f" % ((d/(S+w)).max(), np.median(d/(S+w))))
print("rel to w: max %.3f" % (d/w).max(), "width min %.3f median %.3f" % (w.min(), np.median(w)))
print("sound", bool(np.all(glo <= wl + 1e-12*(S+w)) and np.all(ghi >= wh - 1e-12*(S+w))))
i = np.argmax(d/(S+w)); print("worst: w=%.3f d=%.3f wl=%.3f wh=%.3f" % (w[i], d[i], wl[i], wh[i]))
