import sys, time; sys.path.insert(0, '.')
import numpy as np, torch
import paper_2202_02444_b200 as sp
from paper_2202_02444_b200 import meshing, synth
from paper_2202_02444_b200.spatial import AABB
net = synth.config_net("C4")
b = AABB(-np.ones(3), np.ones(3))
meshing.extract_mesh_arrays(net, b, 5, 3, sp.AFFINE_FIXED, precision="fp32")
f0, tot = torch.cuda.mem_get_info()
t = time.time()
r = meshing.extract_mesh_arrays(net, b, 10, 3, sp.AFFINE_FIXED, precision="fp32")
torch.cuda.synchronize()
f1, _ = torch.cuda.mem_get_info()
print({"seconds": time.time() - t, "triangles": len(r.triangles), "evals": r.point_evals,
       "used_before_gb": (tot - f0) / 1e9, "used_after_gb": (tot - f1) / 1e9})
