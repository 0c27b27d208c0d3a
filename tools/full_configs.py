"""One-off measurements at the exact BASELINE.json sizes that are too long for
the default bench.py run (the bench measures bounded samples of them):

  C3: SIREN 3->8x256->1, default camera at 1024x1024, RayCastParams() defaults,
      interval and affine-truncate:16 (FP64 kernels: the recipe's outputs are
      ~1e-11, below FP32 evaluation noise)
  C4: ELU 3->8x512->1, hierarchical marching cubes at 1024^3 (m = 10,
      dense_levels = 3), affine-fixed prune, FP32 corner evaluation

    python tools/full_configs.py [c3i] [c3t] [c4] > profiles/r02_full_configs.json

Each measurement carries its own nvidia-smi clock record (bench.ClockSampler).
"""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2202_02444_b200 as sp  # noqa: E402
from paper_2202_02444_b200 import synth  # noqa: E402


def main():
    which = sys.argv[1:] or ["c3i", "c3t", "c4"]
    out = {"device": torch.cuda.get_device_name(0)}
    def clocked(fn, *a):
        with bench.ClockSampler(0) as ck:
            r = fn(*a)
        r["clocks"] = ck.summary()
        return r

    if "c3i" in which:
        out["C3_siren_rays_interval_1024sq_fp64"] = clocked(bench.bench_c3, torch, sp, synth, "interval", 1024)
    if "c3t" in which:
        out["C3_siren_rays_truncate16_1024sq_fp64"] = clocked(bench.bench_c3, torch, sp, synth, "affine-truncate:16",
                                                              1024)
    if "c3t512" in which:
        out["C3_siren_rays_truncate16_512sq_fp64"] = clocked(bench.bench_c3, torch, sp, synth, "affine-truncate:16",
                                                             512)
    if "c4" in which:
        out["C4_elu8x512_mesh_1024cubed"] = clocked(bench.bench_c4, torch, sp, synth, 10)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
