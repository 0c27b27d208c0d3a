import sys; sys.path.insert(0,'.')
import torch, numpy as np
import paper_2202_02444_b200 as sp
from paper_2202_02444_b200 import synth
net=synth.config_net("C2")
c,_=synth.grid_cubes(64)
lo=torch.from_numpy(c[:64]-1/64).cuda(); hi=torch.from_numpy(c[:64]+1/64).cuda()
for _ in range(4): sp.bound_aabb(net, lo, hi, sp.AFFINE_FIXED)
torch.cuda.synchronize()
