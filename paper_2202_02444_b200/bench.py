"""Variant study and soundness fuzzer on the device (reference bench.py:1-319).

`fuzz_soundness` draws exactly the reference's regions and sample offsets
(same numpy Generator calls, same 4096-region chunking, so a seed gives
the same regions), but evaluates them in large batches: the sample values
through the FP64 point kernel and every policy's bounds through the fused
bound kernels -- the production FP32 kernels by default -- so the
reference's 10^6-region acceptance fuzz takes seconds.  `bench_variants`
replicates the paper's Table 1 study (bound-able region size per variant by
binary search over the same size grid, bound cost relative to a point
evaluation, ray-cast time) with CUDA-event timings of the device kernels.
"""

from __future__ import annotations

import csv
from dataclasses import dataclass, field

import numpy as np

from . import device as dv
from .camera import Camera
from .errors import NoNetworks
from .network import eval_batch
from .range_core import AFFINE_FIXED, AFFINE_FULL, INTERVAL_ONLY, affine_truncate, range_bound_batch
from .rays import RayCastParams, cast_camera

BENCH_POLICIES = (INTERVAL_ONLY, AFFINE_FIXED, AFFINE_FULL, affine_truncate(16))
SIZE_GRID = np.geomspace(1e-4, 1.0, 32)


@dataclass(frozen=True)
class BenchRow:
    variant: str
    dim: int
    time_ratio: float
    region_size: float  # a length for 1-d regions, a volume for 3-d ones
    raycast_seconds: float


@dataclass
class FuzzViolation:
    net: str
    policy: str
    center: np.ndarray
    axes: np.ndarray
    value: float
    lo: float
    hi: float


@dataclass
class FuzzReport:
    n_regions: int
    n_checks: int
    n_violations: int = 0
    violations: list = field(default_factory=list)  # capped sample

    @property
    def ok(self) -> bool:
        return self.n_violations == 0


# ----------------------------------------------------------------- fuzzing

def _draw_chunk(rng, n, samples):
    """One reference chunk (bench.py:271-283), same Generator call order."""
    centers = rng.uniform(-1.1, 1.1, (n, 3))
    sizes = 10.0 ** rng.uniform(-4.0, 0.0, n)
    one_d = rng.random(n) < 0.5
    dirs = rng.standard_normal((n, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    axes = np.zeros((n, 3, 3))
    axes[:, np.arange(3), np.arange(3)] = (sizes / 2.0)[:, None]
    axes[one_d] = 0.0
    axes[one_d, 0, :] = (sizes[one_d, None] / 2.0) * dirs[one_d]
    eps = rng.uniform(-1.0, 1.0, (n, samples, 3))
    return centers, axes, eps


def _fuzz_batch(net, centers, axes, eps, policies, slack, precision, report, chunk_sizes, max_reported):
    torch = dv._torch()
    dev = torch.device(f"cuda:{dv._torch().cuda.current_device()}")
    c = torch.from_numpy(centers).to(dev)
    a = torch.from_numpy(axes).to(dev)
    pts = c[:, None, :] + torch.einsum("nsk,nkd->nsd", torch.from_numpy(eps).to(dev), a)
    vals = eval_batch(net, pts.reshape(-1, 3), precision="fp64").reshape(len(centers), -1)
    bad_masks, bounds = [], []
    for pol in policies:
        lo, hi = range_bound_batch(net, c, a, pol, precision=precision)
        bad = (vals < (lo - slack)[:, None]) | (vals > (hi + slack)[:, None])
        bad_masks.append(bad)
        bounds.append((lo, hi))
        report.n_checks += len(centers)
    any_bad = [m.any(dim=1) for m in bad_masks]
    report.n_violations += int(sum(int(b.sum().item()) for b in any_bad))
    if len(report.violations) >= max_reported or not any(bool(b.any().item()) for b in any_bad):
        return
    # report in the reference's order: chunk by chunk, policy by policy
    start = 0
    for n in chunk_sizes:
        for p, pol in enumerate(policies):
            rows = torch.nonzero(any_bad[p][start:start + n]).flatten().cpu().numpy() + start
            for i in rows:
                if len(report.violations) >= max_reported:
                    return
                j = int(torch.nonzero(bad_masks[p][i]).flatten()[0].item())
                lo, hi = bounds[p]
                report.violations.append(FuzzViolation(
                    net=getattr(net, "name", ""), policy=str(pol), center=centers[i].copy(), axes=axes[i].copy(),
                    value=float(vals[i, j].item()), lo=float(lo[i].item()), hi=float(hi[i].item())))
        start += n


def fuzz_soundness(nets, n_regions: int = 1_000_000, rng_seed: int = 0, policies=BENCH_POLICIES,
                   samples_per_region: int = 32, slack: float = 1e-5, max_reported: int = 10, chunk: int = 4096,
                   threads: int = 2, precision: str = "fp32", batch_regions: int = 262_144) -> FuzzReport:
    """Containment fuzzing of every policy (bench.py:228-319): random regions
    (centres in [-1.1, 1.1]^3, log-uniform extent in [1e-4, 1], half 1-d
    random segments, half axis-aligned cubes); every sampled value must lie
    inside the bounds widened by `slack`.  Each network has its own seeded
    stream, so the report is deterministic.  `threads` is accepted for API
    compatibility (the device batches replace the thread pool)."""
    if not nets:
        raise NoNetworks("fuzz needs at least one network")
    per_net = [n_regions // len(nets)] * len(nets)
    per_net[0] += n_regions - sum(per_net)
    report = FuzzReport(n_regions=n_regions, n_checks=0)
    for net, quota in zip(nets, per_net):
        rng = np.random.default_rng(rng_seed)
        remaining = quota
        while remaining > 0:
            parts, sizes = [], []
            while remaining > 0 and sum(sizes) < batch_regions:
                n = min(chunk, remaining)
                remaining -= n
                parts.append(_draw_chunk(rng, n, samples_per_region))
                sizes.append(n)
            centers = np.concatenate([p[0] for p in parts])
            axes = np.concatenate([p[1] for p in parts])
            eps = np.concatenate([p[2] for p in parts])
            _fuzz_batch(net, centers, axes, eps, policies, slack, precision, report, sizes, max_reported)
    return report


# ----------------------------------------------------------------- variants

def _timed_best(fn, runs: int) -> float:
    """Fastest of `runs` CUDA-event-timed calls after one warm-up (seconds)."""
    torch = dv._torch()
    fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(runs):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    return best


def _region_axes(rng, n, dim, size):
    if dim == 1:
        dirs = rng.standard_normal((n, 3))
        dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
        return (size / 2.0) * dirs[:, None, :]
    axes = np.zeros((n, 3, 3))
    axes[:, np.arange(3), np.arange(3)] = size / 2.0
    return axes


def _classified(net, policy, c, a_unit, size, precision):
    lo, hi = range_bound_batch(net, c, a_unit * size, policy, precision=precision)
    return float(((lo > 0.0) | (hi < 0.0)).double().mean().item())


def _threshold_size(net, policy, dim, n_regions, rng, precision):
    """Largest SIZE_GRID entry at which >= 50% of the regions classify
    (bench.py:100-116: binary search over the monotone grid)."""
    torch = dv._torch()
    dev = f"cuda:{torch.cuda.current_device()}"
    c = torch.from_numpy(rng.uniform(-1.0, 1.0, (n_regions, 3))).to(dev)
    a = torch.from_numpy(_region_axes(rng, n_regions, dim, 1.0)).to(dev)
    if _classified(net, policy, c, a, SIZE_GRID[0], precision) < 0.5:
        return 0.0
    lo, hi = 0, len(SIZE_GRID) - 1
    if _classified(net, policy, c, a, SIZE_GRID[hi], precision) >= 0.5:
        return float(SIZE_GRID[hi])
    while hi - lo > 1:
        mid = (lo + hi) // 2
        if _classified(net, policy, c, a, SIZE_GRID[mid], precision) >= 0.5:
            lo = mid
        else:
            hi = mid
    return float(SIZE_GRID[lo])


def bench_variants(nets, n_regions: int = 10_000, rng_seed: int = 0, timing_size: float = 0.05,
                   raycast_res: int = 256, runs: int = 5, params: RayCastParams = RayCastParams(),
                   precision: str = "fp32") -> list:
    """The variant study (bench.py:128-178): per policy and region dimension,
    the bound-able region size (averaged over nets; a volume for 3-d), the
    bound/eval cost ratio and the ray-cast time of a raycast_res^2 view of
    nets[0] (fastest of `runs`, one warm-up)."""
    if not nets:
        raise NoNetworks("bench needs at least one network")
    torch = dv._torch()
    dev = f"cuda:{torch.cuda.current_device()}"
    cam = Camera(np.array([1.6, 1.2, 2.0]), np.zeros(3), np.array([0.0, 1.0, 0.0]), 40.0,
                 (raycast_res, raycast_res))
    rows = []
    for policy in BENCH_POLICIES:
        raycast = _timed_best(lambda: cast_camera(nets[0], cam, params, policy, precision=precision), runs)
        for dim in (1, 3):
            rng = np.random.default_rng(rng_seed)
            sizes, ratios = [], []
            for net in nets:
                sizes.append(_threshold_size(net, policy, dim, n_regions, rng, precision))
                c = torch.from_numpy(rng.uniform(-1.0, 1.0, (n_regions, 3))).to(dev)
                a = torch.from_numpy(_region_axes(rng, n_regions, dim, timing_size)).to(dev)
                t_bound = _timed_best(lambda: range_bound_batch(net, c, a, policy, precision=precision), runs)
                t_eval = _timed_best(lambda: eval_batch(net, c, precision=precision), runs)
                ratios.append(t_bound / t_eval)
            size = float(np.mean(sizes))
            rows.append(BenchRow(variant=str(policy), dim=dim, time_ratio=float(np.mean(ratios)),
                                 region_size=size if dim == 1 else size ** 3, raycast_seconds=raycast))
    return rows


def write_bench_csv(rows, path) -> None:
    """bench.py:181-193 layout."""
    with open(path, "w", newline="", encoding="utf-8") as f:
        w = csv.writer(f)
        w.writerow(["variant", "dim", "time_ratio", "region_size", "raycast_seconds"])
        w.writerows([r.variant, r.dim, f"{r.time_ratio:.6g}", f"{r.region_size:.6g}", f"{r.raycast_seconds:.6g}"]
                    for r in rows)


def write_bench_figure(rows, path) -> None:
    """Bar charts of the study (bench.py:196-225); needs matplotlib."""
    import matplotlib

    matplotlib.use("Agg")
    import matplotlib.pyplot as plt

    variants = list(dict.fromkeys(r.variant for r in rows))
    x = np.arange(len(variants))
    fig, axs = plt.subplots(1, 3, figsize=(12, 3.6))
    for dim, dx in ((1, -0.2), (3, 0.2)):
        pick = {r.variant: r for r in rows if r.dim == dim}
        axs[0].bar(x + dx, [max(pick[v].region_size, 1e-12) for v in variants], width=0.4, label=f"{dim}d")
        axs[1].bar(x + dx, [pick[v].time_ratio for v in variants], width=0.4, label=f"{dim}d")
    axs[2].bar(x, [next(r.raycast_seconds for r in rows if r.variant == v) for v in variants], width=0.5)
    for ax, title in zip(axs, ("bound-able region size", "time vs scalar eval", "raycast seconds")):
        ax.set_xticks(x)
        ax.set_xticklabels(variants, rotation=20, ha="right", fontsize=8)
        ax.set_title(title, fontsize=10)
        ax.set_yscale("log")
    axs[0].legend(fontsize=8)
    axs[1].legend(fontsize=8)
    fig.tight_layout()
    fig.savefig(path, dpi=130)
    plt.close(fig)
