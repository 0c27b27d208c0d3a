"""C3 SIREN FP64 interval march at 128^2 (for an ncu capture of march_round_kernel)."""
import sys
sys.path.insert(0, '.')
import torch
import paper_2202_02444_b200 as sp
from paper_2202_02444_b200 import synth
from paper_2202_02444_b200.camera import default_camera
net = synth.config_net("C3")
hit, t, s, st = sp.cast_camera(net, default_camera(128), sp.RayCastParams(), sys.argv[1] if len(sys.argv) > 1 else "interval",
                               precision="fp64")
torch.cuda.synchronize()
print(st.rounds, st.ray_steps)
