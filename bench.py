#!/usr/bin/env python
"""Benchmark of the B200 range-analysis hot path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Headline workload (BASELINE.json configs[1], "C2"): k-d tree build to depth
18 over [-1,1]^3 with affine-fixed bounds on a random-init (torch-uniform,
seed 0) 3->8x256->1 ReLU MLP.  A step is one full tree build; `value` is
affine box bounds per second (tree nodes bounded / step time, whole job).
At N > 1 the frontier below a redundant top cut is split across ranks (one
process per GPU, no collective in the build): total work is fixed, so
scaling is "strong".  `extra` carries the C5 throughput sweep point
(16M on-device cubes, 8x256, one launch), C1 (4x32, 64^3 grid) and C3
(SIREN 8x256 ray casting in FP64 -- the recipe's outputs are ~1e-11, below
FP32 noise: rays/s, interval at 256^2, truncate:16 at 128^2; 250 steps/ray),
C4 (ELU 8x512 mesh at 256^3) and F1 (frustum vs per-pixel casting, 1024^2,
on the reference's relu_sdf fixture).

Timing: W untimed warm-up steps, then K steps, each bracketed by a barrier
and torch.cuda.synchronize(), timed with CUDA events on the launching
stream; the max over ranks is taken.  L2 (126 MB) is flushed by writing a
256 MB buffer before every timed step.  SM clocks and throttle reasons are
sampled with nvidia-smi during the timed region.

--impl reference times the reference's own CPU implementation on all host
cores: the unmodified reference package staged in baseline/_ref
(integration/stage_reference.sh; it travels to the GPU box with the repo
snapshot) -- its range_bound_batch (range_core.py:547) -- in P processes with
one BLAS thread each, bounding 4096-box chunks of the same depth-18 level
(spatial.py:172-186 calls range_bound_batch in 4096-box chunks).  If
baseline/_ref is absent it falls back to the pinned NumPy oracle port
(oracle/spelunk_oracle.py) and says so (cpu_baseline.kind "port").
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "affine box bounds/sec (8x256 MLP)"
UNIT = "boxes/s"
DEPTH = 18
CHUNK = 4096


# --------------------------------------------------------------------------- CPU legs
REF_PKG = ROOT / "baseline" / "_ref"


def reference_kind():
    """'reference' when the unmodified reference is staged in baseline/_ref,
    else 'port' (the pinned oracle restatement)."""
    return "reference" if (REF_PKG / "spelunk" / "range_core.py").exists() else "port"


def _ref_path():
    if str(REF_PKG) not in sys.path:
        sys.path.insert(0, str(REF_PKG))


def _ref_net(net_doc):
    """The reference's own NetworkSpec (baseline/_ref) for a network document."""
    _ref_path()
    from spelunk.network import ActivationKind, DenseLayer, NetworkSpec

    layers = []
    for L in net_doc["layers"]:
        if L["type"] == "dense":
            layers.append(DenseLayer(np.asarray(L["weights"], np.float64), np.asarray(L["bias"], np.float64)))
        else:
            layers.append(ActivationKind(L["type"] if L["type"] != "activation" else L["kind"]))
    return NetworkSpec(int(net_doc["input_dim"]), tuple(layers), net_doc.get("output_semantics", "sdf"),
                       net_doc.get("name", "net"))


def _ref_bounder(net_doc, kind):
    """range_bound_batch(centres, axes) of the reference (or the port)."""
    if kind == "reference":
        _ref_path()
        import spelunk

        net = _ref_net(net_doc)
        return lambda c, a: spelunk.range_bound_batch(net, c, a, spelunk.AFFINE_FIXED)
    from oracle import spelunk_oracle as orc

    onet = orc.net_from_json_doc(net_doc)
    return lambda c, a: orc.bound_batch(onet, c, a, "affine-fixed")


def _cpu_worker(args):
    """One single-BLAS-thread process bounding its share of boxes."""
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    net_doc, centers, axes, reps, kind = args
    try:
        from threadpoolctl import threadpool_limits

        lim = threadpool_limits(1)
    except Exception:  # pragma: no cover
        lim = None
    bound = _ref_bounder(net_doc, kind)
    bound(centers[:64], axes[:64])  # warm
    t0 = time.perf_counter()
    for _ in range(reps):
        for s in range(0, len(centers), CHUNK):
            bound(centers[s : s + CHUNK], axes[s : s + CHUNK])
    dt = time.perf_counter() - t0
    del lim
    return len(centers) * reps, dt


def _cpu_ray_worker(args):
    """One single-BLAS-thread process marching its rays with the reference's
    _march_arrays (rays.py:88-138; cast_rays' own kernel)."""
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    net_doc, origins, dirs, kind, policy = args
    from threadpoolctl import threadpool_limits

    with threadpool_limits(1):
        if kind == "reference":
            _ref_path()
            from spelunk.range_core import parse_policy
            from spelunk.rays import RayCastParams, _march_arrays

            net = _ref_net(net_doc)
            pol = parse_policy(policy)
            run = lambda o, d: _march_arrays(net, o, d, RayCastParams(), pol)
        else:
            from oracle import spelunk_oracle as orc

            onet = orc.net_from_json_doc(net_doc)
            run = lambda o, d: orc.march(onet, o, d, orc.MarchParams(), policy)
        run(origins[:1], dirs[:1])  # warm
        t0 = time.perf_counter()
        hit, t, steps = run(origins, dirs)[:3]
        dt = time.perf_counter() - t0
    return len(origins), int(np.sum(steps)), dt


class CpuPool:
    def __init__(self, procs, kind):
        import multiprocessing as mp

        os.environ["OPENBLAS_NUM_THREADS"] = "1"
        os.environ["OMP_NUM_THREADS"] = "1"
        self.procs = procs
        self.kind = kind
        self.pool = mp.get_context("spawn").Pool(procs)

    def run(self, net_doc, centers, axes, per_proc, reps=1):
        parts = []
        for p in range(self.procs):
            sl = slice(p * per_proc, (p + 1) * per_proc)
            parts.append((net_doc, centers[sl], axes[sl], reps, self.kind))
        t0 = time.perf_counter()
        res = self.pool.map(_cpu_worker, parts)
        wall = time.perf_counter() - t0
        boxes = sum(r[0] for r in res)
        busy = max(r[1] for r in res)
        return boxes, busy, wall

    def run_rays(self, net_doc, origins, dirs, policy):
        parts = [(net_doc, o, d, self.kind, policy) for o, d in zip(np.array_split(origins, self.procs),
                                                          np.array_split(dirs, self.procs)) if len(o)]
        t0 = time.perf_counter()
        res = self.pool.map(_cpu_ray_worker, parts)
        wall = time.perf_counter() - t0
        return sum(r[0] for r in res), sum(r[1] for r in res), wall

    def close(self):
        self.pool.close()
        self.pool.join()


def level18_boxes():
    """The depth-18 level of the C2 tree when every node is UNKNOWN (the
    random-init case): the 64^3 grid of cubes of half 1/64."""
    from paper_2202_02444_b200 import synth

    return synth.grid_cubes(64)


def cpu_info():
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return model, os.cpu_count() or 1


def run_reference(args, rank):
    """--impl reference: the reference algorithm on the host cores."""
    if rank != 0:
        return None
    from paper_2202_02444_b200 import network, synth

    net = synth.config_net("C2")
    doc = network.network_to_doc(net)
    centers, axes = level18_boxes()
    model, cores = cpu_info()
    kind = reference_kind()
    pool = CpuPool(cores, kind)
    per_proc = CHUNK
    rng = np.random.default_rng(0)
    sel = rng.permutation(len(centers))[: per_proc * cores]
    c, a = centers[sel], axes[sel]
    for _ in range(args.warmup):
        pool.run(doc, c, a, per_proc)
    tot_boxes, tot_time = 0, 0.0
    for _ in range(args.steps):
        boxes, busy, wall = pool.run(doc, c, a, per_proc)
        tot_boxes += boxes
        tot_time += wall
    pool.close()
    value = tot_boxes / tot_time
    what = ("the unmodified reference's spelunk.range_bound_batch (baseline/_ref)" if kind == "reference"
            else "the oracle port of range_bound_batch (baseline/_ref not staged)")
    sample = (f"{cores} procs x 1 BLAS thread, each one {CHUNK}-box chunk of the depth-18 level per step "
              f"(range_bound_batch chunking of spatial.py:38) through {what}; CPU {model}")
    return {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * tot_time / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": "C2 k-d tree depth 18, 8x256 ReLU (torch-uniform seed 0), affine-fixed; "
                               "reference arm bounds the depth-18 level in 4096-box chunks",
                   "flush": "n/a (CPU)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


# --------------------------------------------------------------------------- GPU helpers
class ClockSampler:
    """nvidia-smi sampling during the timed region (recipe's clocks line)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            # nvidia-smi's start-up (NVML init, GPU attach) contends with the
            # CUDA driver for tens of ms: let it finish before the timed
            # region opens, then keep only the samples taken inside it
            t0 = time.perf_counter()
            while not self.lines and time.perf_counter() - t0 < 5.0 and self.proc.poll() is None:
                time.sleep(0.01)
            self.lines.clear()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for name, flag in zip(names, parts[3:7]):
                if flag.lower() in ("active", "1", "yes"):
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def physical_gpu_index(local_rank):
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if vis:
        ids = [v.strip() for v in vis.split(",") if v.strip()]
        if local_rank < len(ids) and ids[local_rank].isdigit():
            return int(ids[local_rank])
    return local_rank


def timed(fn, torch, flush, barrier):
    """Barrier + sync, flush L2, CUDA-event time of fn() on the current stream.

    The start event is queued right behind the L2 flush (a 256 MB write, tens
    of microseconds on the device) and a short device spin, without a host
    sync in between, so the host prepares fn's first launch while they run: the event pair
    measures fn's device time, not the Python launch latency of its first
    kernel (the e2e number measures the API end to end).  Python's cyclic
    garbage collector runs before the step, not inside it (a collection pass
    mid-build stalls the launching thread while the GPU drains)."""
    gc.collect()
    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    gc.disable()
    try:
        flush()
        # a ~0.2 ms device spin between the flush and the start event: the host
        # enqueues fn's first launch while the GPU is still busy, so a slow
        # host's Python preamble (argument conversion, output allocation) is
        # not counted as device time (measured: C1's 0.27 ms kernel read as
        # 0.34 ms on a box with a slower host)
        torch.cuda._sleep(400_000)
        e0.record()
        out = fn()
        e1.record()
        torch.cuda.synchronize()
    finally:
        gc.enable()
    barrier()
    return e0.elapsed_time(e1) / 1e3, out


def load_traffic():
    p = ROOT / "profiles" / "traffic.json"
    if p.exists():
        try:
            return json.loads(p.read_text())
        except ValueError:
            return {}
    return {}


# --------------------------------------------------------------------------- main GPU arm
def run_ours(args, rank, world, local_rank):
    import torch

    import paper_2202_02444_b200 as sp
    from paper_2202_02444_b200 import _lib, spatial, synth

    torch.cuda.set_device(local_rank % max(1, torch.cuda.device_count()))
    dev = torch.cuda.current_device()
    dist = world > 1
    if dist:
        import torch.distributed as tdist

        def barrier():
            tdist.barrier()
    else:
        def barrier():
            return None

    flush_buf = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def flush():
        flush_buf.fill_(1.0)

    net = synth.config_net("C2")
    dn = sp.network.device_net(net, dev)
    flop_box = 2.0 * (3 + 2) * dn.macs  # affine-fixed, s = 3
    bounds = spatial.AABB(-np.ones(3), np.ones(3))

    def step():
        if world == 1:
            return spatial.build_spatial_tree_arrays(net, bounds, policy=sp.AFFINE_FIXED, max_depth=DEPTH,
                                                     precision="fp32", to_host=False)
        return spatial.build_spatial_tree_sharded(net, bounds, DEPTH, sp.AFFINE_FIXED, rank, world,
                                                  precision="fp32", to_host=False)

    def useful_units(arr):
        """Tree nodes this rank contributes, each node of the unsharded tree once."""
        if "top_levels" in arr.meta:  # sharded: own sub-tree below the cut (+ the top, on rank 0)
            own = arr.n_nodes - arr.first_level_len
            return own + (arr.meta["top_nodes"] if rank == 0 else 0)
        return arr.n_nodes if rank == 0 else 0

    for _ in range(args.warmup):
        timed(step, torch, flush, barrier)

    times, launches, kernel_ms, kernel_boxes, units_local = [], 0, 0.0, 0, 0
    clock = ClockSampler(physical_gpu_index(local_rank))
    with clock:
        for _ in range(args.steps):
            dt, arr = timed(step, torch, flush, barrier)
            times.append(dt)
            launches += arr.launches
            kernel_ms += arr.bound_ms
            kernel_boxes += arr.bound_evals
            units_local += useful_units(arr)
    from paper_2202_02444_b200.shard import reduce_time_units

    # certification of the (last) build, outside the timed region
    certified = None
    if world == 1:
        labs = [lv.label for lv in arr.levels]
        n_cert = sum(int((l != 0).sum().item()) for l in labs)
        certified = n_cert / max(1, arr.n_nodes)

    coll_dev = dev if args.dist_backend == "nccl" else "cpu"
    total_time, units = reduce_time_units(float(np.sum(times)), float(units_local), device=coll_dev)
    value = units / total_time

    sharded = {}
    if world > 1:
        # final gather of the last build (the one collective of the tree path,
        # outside the timed region): every rank receives the unsharded tree
        barrier()
        g0 = time.perf_counter()
        tree = spatial.gather_spatial_tree(arr, device=coll_dev)
        barrier()
        sharded["tree_gather"] = {"ms": 1e3 * (time.perf_counter() - g0), "nodes": tree.n_nodes,
                                  "levels": tree.n_levels, "complete": tree.n_nodes == 2 ** (DEPTH + 1) - 1,
                                  "collective": f"all_gather ({args.dist_backend})"}
        del tree
        sharded["C5_8x256_16M_per_rank"] = bench_c5_sharded(torch, sp, synth, 16 << 20, rank, world, coll_dev,
                                                             barrier, flush)
        if not args.no_mesh:
            sharded["C4_elu8x512_mesh_256cubed"] = bench_c4_sharded(torch, sp, synth, 8, rank, world, coll_dev,
                                                                    barrier)
        if not args.no_rays:
            sharded["C3_siren_rays_interval_256sq_fp64"] = bench_c3_sharded(torch, sp, synth, 256, rank, world,
                                                                            coll_dev, barrier)

    # ---- e2e at N>1: the multi-GPU public API (sharded build + final gather
    # to host arrays on every rank), max over ranks; rank 0 reports it
    e2e_sharded = None
    if world > 1:
        e2e_sharded = bench_e2e_tree_sharded(torch, sp, spatial, net, bounds, args, rank, world, coll_dev, barrier)

    if rank != 0:
        return None

    # ---- roofline of the dominant kernel (fused bound kernel, FFMA-bound)
    import ctypes as C

    pk = C.c_double()
    _lib.call("spk_ffma_peak", 20000, C.byref(pk), torch.cuda.current_stream().cuda_stream)
    peak_tf = pk.value / 1e12
    achieved_tf = kernel_boxes * flop_box / (kernel_ms / 1e3) / 1e12
    # nominal FFMA peak at the SM clock sampled during the timed region
    # (2 FLOP x 128 lanes x SMs x f); MEASURED_PEAKS.json has no FP32 entry
    sm_mhz = (clock.summary().get("sm_mhz") or 1965.0)
    nominal_tf = 2 * 128 * torch.cuda.get_device_properties(dev).multi_processor_count * sm_mhz * 1e6 / 1e12
    traffic = load_traffic().get("C2_bound_kernel_bytes_per_launch")

    # ---- extra workloads (single GPU, rank 0), each with its own clock record
    extra = {}
    gpu_idx = physical_gpu_index(local_rank)

    def clocked(fn, *a):
        with ClockSampler(gpu_idx) as ck_x:
            out = fn(*a)
        out["clocks"] = ck_x.summary()
        return out

    extra["C2_tree_fp64"] = clocked(bench_c2_fp64, torch, sp, spatial, net, bounds, flush)
    extra["C2_build_spatial_tree_api"] = clocked(bench_tree_api, torch, sp, spatial, net, bounds)
    extra["C5_8x256_16M"] = clocked(bench_c5, torch, sp, synth, "C5_256", 16 << 20, flush, peak_tf)
    extra["C5_8x64_16M"] = clocked(bench_c5, torch, sp, synth, "C5_64", 16 << 20, flush, peak_tf)
    extra["C5_8x512_4M"] = clocked(bench_c5, torch, sp, synth, "C5_512", 4 << 20, flush, peak_tf)
    # FP32 bounds + FP64 re-bound of near-certifiable UNKNOWN boxes: the
    # reference's labels (tests/test_gpu_refine.py) at close to FP32 cost
    extra["C2_tree_fp32_refine"] = clocked(bench_c2_fp64, torch, sp, spatial, net, bounds, flush, "fp32-refine")
    extra["C5_8x64_16M_fp32_refine"] = clocked(bench_c5, torch, sp, synth, "C5_64", 16 << 20, flush, peak_tf,
                                               "fp32-refine")
    extra["C5_8x64_16M_fp64"] = clocked(bench_c5, torch, sp, synth, "C5_64", 16 << 20, flush, peak_tf, "fp64")
    # the headline architecture with a real surface (trained torus SDF): what
    # plain FP32 costs in certifications and what fp32-refine recovers
    extra["trained_torus_8x256_tree_d21"] = clocked(bench_trained_tree, torch, sp, spatial, synth, bounds, flush)
    extra["C1_4x32_64cubed"] = clocked(bench_c1, torch, sp, synth, flush, peak_tf)
    extra["host_range_bound_batch_4096"] = clocked(bench_host_calls, sp, synth)
    if not args.no_mesh:
        extra["C4_elu8x512_mesh_256cubed"] = clocked(bench_c4, torch, sp, synth, 8)
    if not args.no_rays:
        extra["C3_siren_rays_interval_256sq_fp64"] = clocked(bench_c3, torch, sp, synth, "interval", 256)
        extra["C3_siren_rays_truncate16_128sq_fp64"] = clocked(bench_c3, torch, sp, synth, "affine-truncate:16", 128)
        extra["F1_frustum_relu_sdf_1024sq"] = clocked(bench_frustum, torch, sp, 1024)

    # ---- e2e through the public API (host arrays out)
    e2e = e2e_sharded if e2e_sharded is not None else bench_e2e_tree(torch, sp, spatial, net, bounds, args)

    # ---- CPU baseline: oracle port on the host cores, bounded sample
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        cpu = cpu_baseline(sp)
        extra["cpu_reference"] = cpu_reference_extras(extra)

    ck = clock.summary()
    return {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * total_time / args.steps,
        "step_ms": [round(1e3 * t, 3) for t in times], "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "fp32", "data": "synthetic",
        "config": {"workload": "C2: k-d tree build to depth 18 over [-1,1]^3, affine-fixed, 3->8x256->1 ReLU "
                               "random-init (torch-uniform, seed 0); 524,287 node bounds per build",
                   "global_batch": int(units / args.steps), "parallelism": f"frontier-sharded x{world}",
                   "flush": "L2 flushed (256 MB write) before every timed step",
                   "certified_fraction": certified,
                   "net": "3->8x256->1 ReLU, torch-uniform init (nn.Linear default), final bias recentred, seed 0"},
        "roofline": {"bound": "fp32", "achieved": achieved_tf, "peak": peak_tf, "unit": "TFLOP/s",
                     "frac": achieved_tf / peak_tf, "traffic": traffic,
                     "kernel": "spk::bound_kernel<float,5,256,AFFINE> (all tree levels)",
                     "flop_per_box": flop_box,
                     "peak_source": "measured FFMA probe (spk_ffma_peak) on this GPU at run time",
                     "peak_nominal": nominal_tf, "frac_nominal": achieved_tf / nominal_tf,
                     "flop_counting": "algorithmic (dense) FLOPs; the kernel skips X rows that are exactly zero "
                                      "(ReLU-inactive neurons of both boxes of a sibling pair) with identical "
                                      "results -- it executes ~69% of the dense FMAs on the depth-18 level "
                                      "(tools/live_rows_estimate.py), so the FFMA pipe itself runs at ~0.69 x frac",
                     "kernel_ms_per_step": kernel_ms / args.steps},
        "e2e": e2e,
        "cpu_baseline": cpu,
        "gpu_launches": int(launches / args.steps),
        "clocks": ck,
        "extra": extra,
        "sharded": sharded or None,
    }


def bench_c2_fp64(torch, sp, spatial, net, bounds, flush, precision="fp64"):
    """The headline build with the FP64 kernels -- the reference's arithmetic
    (sound-padded FP64; topology identical to the reference's tree) -- or
    with precision="fp32-refine" (FP32, near-certifiable UNKNOWN nodes
    re-bounded in FP64)."""
    run = lambda: spatial.build_spatial_tree_arrays(net, bounds, policy=sp.AFFINE_FIXED, max_depth=DEPTH,
                                                    precision=precision, to_host=False)
    run()
    ts = []
    for _ in range(2):
        dt, arr = timed(run, torch, flush, lambda: None)
        ts.append(dt)
    dt = float(np.median(ts))
    return {"nodes": arr.n_nodes, "boxes_per_s": arr.n_nodes / dt, "ms": dt * 1e3,
            "bound_kernel_ms": arr.bound_ms, "precision": precision}


def bench_trained_tree(torch, sp, spatial, synth, bounds, flush, depth=21):
    """k-d tree to depth 21 on the trained 3->8x256->1 ReLU torus SDF
    (synth.trained_net; the C2 architecture, certifying 6.6% of its nodes):
    FP32, fp32-refine and FP64 node counts, certifications and times.
    fp32-refine reproduces the FP64 (= reference) topology."""
    net = synth.trained_net("torus")
    out = {"net": "trained 3->8x256->1 ReLU torus SDF (tests/golden/nets/torus_8x256.npz)", "depth": depth,
           "refine_band": sp.net_refine_band(net)}
    levels = {}
    for prec in ("fp32", "fp32-refine", "fp64"):
        run = lambda: spatial.build_spatial_tree_arrays(net, bounds, policy=sp.AFFINE_FIXED, max_depth=depth,
                                                        precision=prec, to_host=False)
        run()
        dt, arr = timed(run, torch, flush, lambda: None)
        levels[prec] = [len(lv.label) for lv in arr.levels]
        cert = sum(int((lv.label != 0).sum().item()) for lv in arr.levels)
        out[prec] = {"ms": dt * 1e3, "nodes": arr.n_nodes, "certified_nodes": cert,
                     "node_bounds_per_s": arr.n_nodes / dt}
        del arr
    out["refine_topology_equals_fp64"] = levels["fp32-refine"] == levels["fp64"]
    return out


def bench_tree_api(torch, sp, spatial, net, bounds):
    """The reference-signature call (spatial.py:214): build_spatial_tree(...)
    -> root TreeNode.  Nodes are materialised lazily from the host level
    arrays on first access (a full Python traversal of the 524,287 nodes costs
    ~7 s whichever way they are built; eager construction alone took 6.7 s)."""
    spatial.build_spatial_tree(net, bounds, policy=sp.AFFINE_FIXED, max_depth=10)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    root = spatial.build_spatial_tree(net, bounds, policy=sp.AFFINE_FIXED, max_depth=DEPTH)
    dt = time.perf_counter() - t0
    return {"nodes": (1 << (DEPTH + 1)) - 1, "seconds": dt, "root_children": len(root.children or ()),
            "api": "build_spatial_tree(net, AABB([-1]*3,[1]*3), policy=AFFINE_FIXED, max_depth=18)"}


def bench_host_calls(sp, synth):
    """The reference's calling pattern through the host-array entry point
    (spk_bound_batch_host): 4096-box chunks (spatial.py:38) of the depth-18
    level, NumPy in / out, one caller and 8 concurrent ThreadPoolExecutor
    callers (rays.py:170-181).  Wall clock, copies included."""
    from concurrent.futures import ThreadPoolExecutor

    net = synth.config_net("C2")
    c, a = level18_boxes()
    chunks = [(c[i:i + CHUNK], a[i:i + CHUNK]) for i in range(0, 64 * CHUNK, CHUNK)]
    for cc, aa in chunks[:4]:
        sp.range_bound_batch(net, cc, aa, sp.AFFINE_FIXED)
    t0 = time.perf_counter()
    for cc, aa in chunks:
        sp.range_bound_batch(net, cc, aa, sp.AFFINE_FIXED)
    serial = time.perf_counter() - t0
    with ThreadPoolExecutor(max_workers=8) as pool:
        # warm every worker thread's staging (pinned + device buffers, streams)
        for _ in range(2):
            list(pool.map(lambda x: sp.range_bound_batch(net, x[0], x[1], sp.AFFINE_FIXED), chunks))
        t0 = time.perf_counter()
        list(pool.map(lambda x: sp.range_bound_batch(net, x[0], x[1], sp.AFFINE_FIXED), chunks))
        threaded = time.perf_counter() - t0
    n = len(chunks) * CHUNK
    return {"calls": len(chunks), "boxes_per_call": CHUNK, "serial_ms_per_call": 1e3 * serial / len(chunks),
            "serial_boxes_per_s": n / serial, "threads8_boxes_per_s": n / threaded,
            "api": "range_bound_batch(net, centers[4096,3], axes[4096,3,3], AFFINE_FIXED) with NumPy arrays"}


def bench_c5(torch, sp, synth, tag, n, flush, peak_tf, precision="fp32"):
    net = synth.config_net(tag)
    dn = sp.network.device_net(net)
    lo = torch.empty(n, dtype=torch.float64, device="cuda")
    hi = torch.empty(n, dtype=torch.float64, device="cuda")
    cls = torch.empty(n, dtype=torch.int8, device="cuda")
    out = (lo, hi, cls)
    run = lambda: sp.bound_random_cubes(net, n, seed=1, half=1.0 / 64, out=out, precision=precision)
    run()
    ts = []
    for _ in range(3):
        dt, _ = timed(run, torch, flush, lambda: None)
        ts.append(dt)
    dt = float(np.median(ts))
    flop = 2.0 * 5 * dn.macs
    cert = float((cls != 0).float().mean().item())
    return {"boxes": n, "boxes_per_s": n / dt, "ms": dt * 1e3, "tflops": n * flop / dt / 1e12,
            "frac_of_ffma_peak": n * flop / dt / 1e12 / peak_tf, "certified_fraction": cert,
            "half_extent": 1 / 64, "precision": precision}


def bench_c1(torch, sp, synth, flush, peak_tf):
    net = synth.config_net("C1")
    dn = sp.network.device_net(net)
    c, a = synth.grid_cubes(64)
    ct = torch.from_numpy(c).cuda()
    at = torch.from_numpy(a).cuda()
    run = lambda: sp.range_bound_batch(net, ct, at, sp.AFFINE_FIXED, return_class=True)
    run()
    ts = []
    for _ in range(5):
        dt, res = timed(run, torch, flush, lambda: None)
        ts.append(dt)
    dt = float(np.median(ts))
    n = len(c)
    flop = 2.0 * 5 * dn.macs
    cert = float((res[2] != 0).float().mean().item())
    return {"boxes": n, "boxes_per_s": n / dt, "ms": dt * 1e3, "tflops": n * flop / dt / 1e12,
            "frac_of_ffma_peak": n * flop / dt / 1e12 / peak_tf, "certified_fraction": cert}


def bench_c3(torch, sp, synth, policy, res):
    """C3: SIREN 3->8x256->1 (w0 = 30 folded into the first layer, recentred),
    default camera (reference bench.py:119-126), RayCastParams() defaults.
    FP64 kernels: this recipe's outputs are ~1e-11 (median |f| over [-1,1]^3),
    below FP32 evaluation noise, so only FP64 -- the reference's arithmetic --
    gives meaningful hit decisions (then bit-identical to the reference)."""
    from paper_2202_02444_b200.camera import default_camera

    net = synth.config_net("C3")
    cam = default_camera(res)
    sp.cast_camera(net, default_camera(16), sp.RayCastParams(), policy, precision="fp64")  # warm
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    hit, t, steps, st = sp.cast_camera(net, cam, sp.RayCastParams(), policy, precision="fp64")
    e1.record()
    torch.cuda.synchronize()
    dt = e0.elapsed_time(e1) / 1e3
    n = res * res
    return {"rays": n, "rays_per_s": n / dt, "ms": dt * 1e3, "ray_steps": st.ray_steps,
            "steps_per_ray": st.ray_steps / n, "certified_steps": st.certified_steps,
            "lockstep_rounds": st.rounds, "hit_fraction": float(hit.float().mean().item()), "policy": policy,
            "precision": "fp64"}


def bench_c3_sharded(torch, sp, synth, res, rank, world, coll_dev, barrier):
    """C3 interval rays sharded over ranks (interleaved 16x16 pixel tiles, no
    collective in the march), rays/s over the max rank time, then the NCCL
    final gather of the image (gather_camera_image)."""
    from paper_2202_02444_b200.camera import default_camera
    from paper_2202_02444_b200.shard import reduce_time_units

    net = synth.config_net("C3")
    cam = default_camera(res)
    sp.cast_camera(net, default_camera(16), sp.RayCastParams(), "interval", precision="fp64")  # warm
    torch.cuda.synchronize()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    pix, hit, t, steps, st = sp.cast_camera_sharded(net, cam, rank, world, sp.RayCastParams(), "interval",
                                                    precision="fp64")
    e1.record()
    torch.cuda.synchronize()
    dt, n = reduce_time_units(e0.elapsed_time(e1) / 1e3, float(pix.numel()), device=coll_dev)
    barrier()
    g0 = time.perf_counter()
    img_hit, img_t, img_steps = sp.gather_camera_image(pix, hit, t, steps, res * res, device=coll_dev)
    barrier()
    return {"rays": int(n), "rays_per_s": n / dt, "ms": dt * 1e3, "gather_ms": 1e3 * (time.perf_counter() - g0),
            "hit_fraction": float(img_hit.mean()), "steps_per_ray": float(img_steps.mean()),
            "parallelism": f"pixel tiles 16x16 interleaved x{world}"}


def bench_c5_sharded(torch, sp, synth, n_per_rank, rank, world, coll_dev, barrier, flush):
    """C5 sharded by contiguous index ranges of the on-device cube stream
    (rank r bounds cubes [r*n, (r+1)*n): first_index), no collective in the
    data path -- weak scaling; boxes/s over the max rank time."""
    from paper_2202_02444_b200.shard import reduce_time_units

    net = synth.config_net("C5_256")
    out = tuple(torch.empty(n_per_rank, dtype=dt, device="cuda")
                for dt in (torch.float64, torch.float64, torch.int8))
    run = lambda: sp.bound_random_cubes(net, n_per_rank, seed=1, half=1.0 / 64, first_index=rank * n_per_rank,
                                        out=out)
    run()
    ts = []
    for _ in range(2):
        dt, _ = timed(run, torch, flush, barrier)
        ts.append(dt)
    dt, n = reduce_time_units(float(np.median(ts)), float(n_per_rank), device=coll_dev)
    return {"boxes": int(n), "boxes_per_s": n / dt, "ms": dt * 1e3, "scaling": "weak",
            "parallelism": f"contiguous first_index ranges x{world}"}


def bench_c4_sharded(torch, sp, synth, m, rank, world, coll_dev, barrier):
    """C4 sharded: every rank prunes redundantly and extracts its contiguous
    slice of the surviving blocks (spk_mesh_extract_shard), no collective
    inside; then the one gather (edge-key triangles + vertex rows, global
    sort-unique dedup on the device).  Wall time, max over ranks."""
    from paper_2202_02444_b200 import meshing
    from paper_2202_02444_b200.shard import reduce_time_units
    from paper_2202_02444_b200.spatial import AABB

    net = synth.config_net("C4")
    bounds = AABB(-np.ones(3), np.ones(3))
    meshing.extract_mesh_sharded(net, bounds, 5, rank, world, 3, sp.AFFINE_FIXED, precision="fp32")  # warm
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    part = meshing.extract_mesh_sharded(net, bounds, m, rank, world, 3, sp.AFFINE_FIXED, precision="fp32")
    torch.cuda.synchronize()
    dt, evals = reduce_time_units(time.perf_counter() - t0, float(part.point_evals), device=coll_dev)
    barrier()
    g0 = time.perf_counter()
    mesh = meshing.gather_mesh(part, device=coll_dev)
    barrier()
    return {"m": m, "seconds": dt, "point_evals": int(evals), "point_evals_per_s": evals / dt,
            "gather_ms": 1e3 * (time.perf_counter() - g0), "triangles": int(len(mesh.triangles)),
            "parallelism": f"surviving-block slices x{world}"}


def bench_frustum(torch, sp, res):
    """§8(f1): cast_frustum_image (rays.py:232-341) vs per-pixel casting on the
    reference's trained relu_sdf fixture (tests/golden/nets, 7x32), default
    camera, RayCastParams() defaults, FP32 kernels, images left on the device.
    (The random-init C3 SIREN outputs ~1e-11, so nothing certifies there and
    every frustum dissolves into per-pixel rays -- no frustum workload.)"""
    from paper_2202_02444_b200.camera import default_camera

    net = sp.load_network(Path(__file__).resolve().parent / "tests" / "golden" / "nets" / "relu_sdf.json")
    out = {"net": "relu_sdf (reference fixture, 7x32 ReLU)", "res": res}
    for pol in ("affine-fixed", "interval"):
        # warm both arms at the measured resolution (pool growth, first launches)
        sp.cast_frustum_image(net, default_camera(res), sp.RayCastParams(), pol, precision="fp32", device_output=True)
        sp.cast_camera(net, default_camera(res), sp.RayCastParams(), pol, precision="fp32")
        torch.cuda.synchronize()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        fr = sp.cast_frustum_image(net, default_camera(res), sp.RayCastParams(), pol, precision="fp32",
                                   device_output=True)
        e[1].record()
        _, _, steps, st = sp.cast_camera(net, default_camera(res), sp.RayCastParams(), pol, precision="fp32")
        e[2].record()
        torch.cuda.synchronize()
        n = res * res
        out[pol] = {"frustum_ms": e[0].elapsed_time(e[1]), "per_ray_ms": e[1].elapsed_time(e[2]),
                    "frustum_rays_per_s": n / (e[0].elapsed_time(e[1]) / 1e3),
                    "per_ray_rays_per_s": n / (e[1].elapsed_time(e[2]) / 1e3),
                    "amortised_steps_per_pixel": float(fr.steps.sum().item()) / n,
                    "per_ray_steps_per_pixel": st.ray_steps / n, **fr.stats.meta}
    return out


def bench_c4(torch, sp, synth, m):
    """C4 (reduced resolution): hierarchical marching cubes of the ELU
    3->8x512->1 net (torch-uniform, recentred) at 2^m cells per axis,
    affine-fixed prune, FP32 corner evaluation.  (1024^3 = m 10 is the
    config; it is 64x the corner evaluations of m = 8.)"""
    from paper_2202_02444_b200 import meshing
    from paper_2202_02444_b200.spatial import AABB

    net = synth.config_net("C4")
    bounds = AABB(-np.ones(3), np.ones(3))
    meshing.extract_mesh_arrays(net, bounds, 5, 3, sp.AFFINE_FIXED, precision="fp32")  # warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = meshing.extract_mesh_arrays(net, bounds, m, 3, sp.AFFINE_FIXED, precision="fp32")
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    return {"m": m, "seconds": dt, "triangles": int(len(res.triangles)), "vertices": int(len(res.vertices)),
            "surviving_blocks": res.n_blocks, "point_evals": res.point_evals, "bound_evals": res.bound_evals,
            "point_evals_per_s": res.point_evals / dt,
            "note": "wall clock through the public API incl. mesh copy to host"}


def bench_e2e_tree(torch, sp, spatial, net, bounds, args):
    """Public API, host arrays out: build_spatial_tree_arrays(to_host=True)."""
    arr = spatial.build_spatial_tree_arrays(net, bounds, policy=sp.AFFINE_FIXED, max_depth=DEPTH, to_host=True)
    ts = []
    for _ in range(max(1, min(args.steps, 3))):
        del arr  # the previous result is released outside the timed call
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        arr = spatial.build_spatial_tree_arrays(net, bounds, policy=sp.AFFINE_FIXED, max_depth=DEPTH, to_host=True)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    dt = float(np.median(ts))
    n = arr.n_nodes
    d2h = sum(l.lo.nbytes + l.hi.nbytes + l.bound_lo.nbytes + l.bound_hi.nbytes + l.label.nbytes +
              l.face.nbytes + l.parent.nbytes for l in arr.levels)
    return {"value": n / dt, "unit": UNIT, "h2d_bytes_per_step": 48, "d2h_bytes_per_step": int(d2h),
            "api": "build_spatial_tree_arrays(net, AABB([-1]*3,[1]*3), policy=AFFINE_FIXED, max_depth=18, "
                   "to_host=True)", "ms": dt * 1e3}


def bench_e2e_tree_sharded(torch, sp, spatial, net, bounds, args, rank, world, coll_dev, barrier):
    """N GPUs through the public API: build_spatial_tree_sharded on every rank,
    then gather_spatial_tree(to_host=True) -- every rank ends with the whole
    unsharded tree as host arrays.  Wall time between barriers, max over ranks."""
    from paper_2202_02444_b200.shard import reduce_time_units

    def run():
        part = spatial.build_spatial_tree_sharded(net, bounds, DEPTH, sp.AFFINE_FIXED, rank, world,
                                                  precision="fp32", to_host=False)
        return spatial.gather_spatial_tree(part, device=coll_dev, to_host=True)

    tree = run()
    ts = []
    for _ in range(max(1, min(args.steps, 3))):
        del tree
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        tree = run()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
        barrier()
    dt, _ = reduce_time_units(float(np.median(ts)), 0.0, device=coll_dev)
    n = tree.n_nodes
    d2h = sum(l.lo.nbytes + l.hi.nbytes + l.bound_lo.nbytes + l.bound_hi.nbytes + l.label.nbytes +
              l.face.nbytes + l.parent.nbytes for l in tree.levels)
    return {"value": n / dt, "unit": UNIT, "h2d_bytes_per_step": 48, "d2h_bytes_per_step": int(d2h),
            "api": f"build_spatial_tree_sharded(rank, world={world}) + gather_spatial_tree(to_host=True) on "
                   "every rank", "ms": dt * 1e3}


def cpu_reference_extras(extra):
    """The reference on the host cores for the other two CPU-comparable
    metrics (SURVEY.md §8(d) "CPU reference timing"): C1 in full (4x32,
    64^3 grid, affine-fixed) and C3 rays on a bounded sample (16x16 centre
    crop of the 256^2 default camera, interval, FP64), each beside the GPU
    number of the same workload in `extra`."""
    from paper_2202_02444_b200 import network, synth

    model, cores = cpu_info()
    kind = reference_kind()
    pool = CpuPool(cores, kind)
    out = {"kind": kind, "cores": cores, "cpu": model}
    # C1: the whole grid, 4096-box chunks per process
    doc = network.network_to_doc(synth.config_net("C1"))
    centers, axes = synth.grid_cubes(64)
    per_proc = -(-len(centers) // cores)
    pool.run(doc, centers[: cores * 64], axes[: cores * 64], 64)  # spawn + import warm-up
    boxes, busy, wall = pool.run(doc, centers, axes, per_proc)
    gpu = extra.get("C1_4x32_64cubed", {}).get("boxes_per_s")
    out["C1_4x32_64cubed"] = {"boxes": boxes, "boxes_per_s": boxes / wall, "wall_s": wall,
                              "gpu_over_cpu": (gpu / (boxes / wall)) if gpu else None}
    # C3: reference camera rays (camera.py pixel_dirs) through _march_arrays
    res, crop = 256, 16
    pos, look, up = np.array([1.6, 1.2, 2.0]), np.zeros(3), np.array([0.0, 1.0, 0.0])
    if kind == "reference":
        _ref_path()
        from spelunk.camera import Camera

        all_dirs = Camera(pos, look, up, 40.0, (res, res)).pixel_dirs()
    else:
        from oracle import spelunk_oracle as orc

        all_dirs = orc.pixel_dirs(pos, look, up, 40.0, res, res)
    doc3 = network.network_to_doc(synth.config_net("C3"))
    for policy, crop, gkey in (("interval", 16, "C3_siren_rays_interval_256sq_fp64"),
                               ("affine-truncate:16", 4, "C3_siren_rays_truncate16_128sq_fp64")):
        r0 = (res - crop) // 2
        dirs = np.ascontiguousarray(np.asarray(all_dirs)[r0:r0 + crop, r0:r0 + crop].reshape(-1, 3))
        origins = np.tile(pos, (len(dirs), 1))
        rays, ray_steps, wall = pool.run_rays(doc3, origins, dirs, policy)
        g = extra.get(gkey, {})
        gpu_steps = (g["ray_steps"] / (g["ms"] / 1e3)) if g else None
        out["C3_siren_rays_" + policy.replace("affine-", "").replace(":", "") + "_fp64"] = {
            "rays": rays, "ray_steps": ray_steps, "steps_per_ray": ray_steps / rays, "rays_per_s": rays / wall,
            "ray_steps_per_s": ray_steps / wall, "wall_s": wall,
            "sample": f"{crop}x{crop} centre crop of the {res}^2 default camera, {cores} procs, reference "
                      f"rays._march_arrays (the kernel of cast_rays), {policy}",
            "gpu_rays_per_s": g.get("rays_per_s"), "gpu_ray_steps_per_s": gpu_steps,
            "gpu_over_cpu_ray_steps": (gpu_steps / (ray_steps / wall)) if gpu_steps else None}
    pool.close()
    return out


def cpu_baseline(sp):
    from paper_2202_02444_b200 import network, synth

    net = synth.config_net("C2")
    doc = network.network_to_doc(net)
    centers, axes = level18_boxes()
    model, cores = cpu_info()
    per_proc = 2 * CHUNK
    sel = np.random.default_rng(1).permutation(len(centers))[: per_proc * cores]
    kind = reference_kind()
    pool = CpuPool(cores, kind)
    pool.run(doc, centers[sel][: cores * 64], axes[sel][: cores * 64], 64)  # spawn + import warm-up
    boxes, busy, wall = pool.run(doc, centers[sel], axes[sel], per_proc)
    pool.close()
    what = "reference spelunk.range_bound_batch (baseline/_ref)" if kind == "reference" else "oracle port"
    return {"value": boxes / wall, "unit": UNIT, "cores": cores, "kind": kind,
            "sample": f"{boxes} depth-18 boxes ({cores} procs x {per_proc}, 4096-box chunks, 1 BLAS thread each), "
                      f"affine-fixed 8x256, {what}; CPU {model}; wall {wall:.1f}s"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-rays", action="store_true", help="skip the C3 ray-casting extra")
    ap.add_argument("--no-mesh", action="store_true", help="skip the C4 mesh extra")
    ap.add_argument("--dist-backend", default="nccl", help="nccl (default) or gloo (functional checks of the "
                    "sharded path with several ranks on one GPU)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        line = run_reference(args, rank)
        if line is not None:
            print(json.dumps(line), flush=True)
        return
    if world > 1:
        import torch
        import torch.distributed as tdist

        dev = local_rank % max(1, torch.cuda.device_count())
        torch.cuda.set_device(dev)
        if args.dist_backend == "nccl":
            tdist.init_process_group("nccl", device_id=torch.device(f"cuda:{dev}"))
        else:
            tdist.init_process_group(args.dist_backend)
    line = run_ours(args, rank, world, local_rank)
    if line is not None:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as tdist

        tdist.destroy_process_group()


if __name__ == "__main__":
    main()
