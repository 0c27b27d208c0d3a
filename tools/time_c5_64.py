import sys, json
sys.path.insert(0, ".")
import torch
import paper_2202_02444_b200 as sp
from paper_2202_02444_b200 import synth
from tools.time_act import timed
net = synth.config_net("C5_64")
c1 = synth.config_net("C1")
print(json.dumps({"c5_64_16M_ms": timed(lambda: sp.bound_random_cubes(net, 1 << 24, seed=1)),
                  "c1_4x32_16M_ms": timed(lambda: sp.bound_random_cubes(c1, 1 << 24, seed=1))}))
