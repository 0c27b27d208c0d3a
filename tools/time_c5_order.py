import sys, json
sys.path.insert(0,'.')
import torch
import paper_2202_02444_b200 as sp
from paper_2202_02444_b200 import synth
net=synth.config_net("C5_256")
def timed(fn,reps=3):
    fn(); torch.cuda.synchronize(); best=1e9
    for _ in range(reps):
        e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); best=min(best,e0.elapsed_time(e1))
    return best
n=1<<22
lo,hi,_=sp.bound_random_cubes(net, n, seed=1, half=1/64)
print(json.dumps({"c5_4M_ms": timed(lambda: sp.bound_random_cubes(net, n, seed=1, half=1/64)), "lo_sum": float(lo.sum().item()), "hi_sum": float(hi.sum().item())}))
