import sys, json
sys.path.insert(0, '.')
import torch, bench
import paper_2202_02444_b200 as sp
from paper_2202_02444_b200 import synth
print(json.dumps(bench.bench_c3(torch, sp, synth, "interval", 1024)))
print(json.dumps(bench.bench_c3(torch, sp, synth, "affine-truncate:16", 256)))
print(json.dumps(bench.bench_c3(torch, sp, synth, "affine-fixed", 256)))
