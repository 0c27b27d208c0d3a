"""C4 mesh extraction at 2^m cells per axis (for an ncu launch list)."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2202_02444_b200 as sp  # noqa: E402
from paper_2202_02444_b200 import meshing, synth  # noqa: E402
from paper_2202_02444_b200.spatial import AABB  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 8
net = synth.config_net("C4")
b = AABB(-np.ones(3), np.ones(3))
meshing.extract_mesh_arrays(net, b, 5, 3, sp.AFFINE_FIXED, precision="fp32")
torch.cuda.synchronize()
t0 = time.perf_counter()
res = meshing.extract_mesh_arrays(net, b, m, 3, sp.AFFINE_FIXED, precision="fp32")
torch.cuda.synchronize()
print(f"m={m}: {time.perf_counter() - t0:.3f} s, {len(res.triangles)} triangles, {res.point_evals} evals")
