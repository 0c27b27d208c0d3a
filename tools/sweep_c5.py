"""C5 sweep (BASELINE configs[4]): affine-fixed bounds of N
on-device random cubes (half-extent 1/64) through 8-layer ReLU MLPs of width
64 / 256 / 512; one launch per point, CUDA events, FP32 sound kernels.

    python tools/sweep_c5.py > profiles/r02_c5_sweep.json

Every point carries its own nvidia-smi clock record (bench.ClockSampler) and
its fraction of both the measured FFMA probe and the nominal FFMA peak
2 x 128 x SMs x the sampled SM clock.
"""
import json
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2202_02444_b200 as sp  # noqa: E402
from paper_2202_02444_b200 import synth  # noqa: E402
from paper_2202_02444_b200._lib import load  # noqa: E402

SIGMA = {"C5_64": 28928, "C5_256": 459776, "C5_512": 1837056}


def main():
    import ctypes as C
    peak = C.c_double()
    load().spk_ffma_peak(4096, C.byref(peak), None)
    rows = []
    for tag, sizes in (("C5_64", [1, 4, 16, 64, 256]), ("C5_256", [1, 4, 16, 64, 256]), ("C5_512", [1, 4, 16])):
        net = synth.config_net(tag)
        flop = 2 * (3 + 2) * SIGMA[tag]
        sp.bound_random_cubes(net, 1 << 16, seed=3)
        for m in sizes:
            n = m << 20
            out = (torch.empty(n, dtype=torch.float64, device="cuda"), torch.empty(n, dtype=torch.float64, device="cuda"),
                   torch.empty(n, dtype=torch.int8, device="cuda"))
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with bench.ClockSampler(0) as ck:
                e0.record()
                sp.bound_random_cubes(net, n, seed=1, half=1 / 64, out=out)
                e1.record()
                torch.cuda.synchronize()
            s = e0.elapsed_time(e1) / 1e3
            clk = ck.summary()
            mhz = clk["sm_mhz"] or 1965.0
            nominal = 2 * 128 * torch.cuda.get_device_properties(0).multi_processor_count * mhz * 1e6
            rows.append({"net": tag, "width": int(tag.split("_")[1]), "boxes": n, "seconds": s, "boxes_per_s": n / s,
                         "tflops": n * flop / s / 1e12, "frac_of_ffma_peak": n * flop / s / peak.value,
                         "frac_of_nominal_ffma": n * flop / s / nominal, "clocks": clk,
                         "certified_fraction": float((out[2] != 0).float().mean().item())})
            print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
            del out
    print(json.dumps({"sweep": "C5", "ffma_peak_tflops": peak.value / 1e12, "points": rows}, indent=1))


if __name__ == "__main__":
    main()
