"""Range-marching ray casting on the B200 (reference rays.py:30-184).

`cast_rays` / `cast_ray` keep the reference contract (lists of Ray in,
HitResult out; default policy affine-fixed).  The whole march runs in the
C-ABI (`spk_march`, K6): FP64 ray state, lock-step rounds over the compacted
active set, one point-evaluation and one bound pass per round.
`march_arrays` is the array API (NumPy or CUDA tensors) and `cast_camera`
marches every pixel of a camera with directions generated on the device.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from . import device as dv
from .camera import Camera
from .errors import InvalidParameter, InvalidRay
from .network import _precision_code, device_net
from .range_core import AFFINE_FIXED, policy_code


@dataclass(frozen=True)
class Ray:
    origin: np.ndarray
    dir: np.ndarray

    def __post_init__(self):
        p = np.asarray(self.origin, dtype=np.float64)
        r = np.asarray(self.dir, dtype=np.float64)
        if p.shape != (3,) or r.shape != (3,):
            raise InvalidRay("origin and dir must be 3-vectors")
        if not (np.all(np.isfinite(p)) and np.all(np.isfinite(r))):
            raise InvalidRay("non-finite ray")
        if abs(np.linalg.norm(r) - 1.0) > 1e-9:
            raise InvalidRay("direction must be a unit vector")
        object.__setattr__(self, "origin", p)
        object.__setattr__(self, "dir", r)


@dataclass(frozen=True)
class RayCastParams:
    """rays.py:48-71."""

    t_max: float = 10.0
    sigma0: float | None = None
    eta_plus: float = 1.5
    eta_minus: float = 0.5
    delta: float = 0.001
    safety: float = 0.98

    def __post_init__(self):
        if self.t_max <= 0.0:
            raise InvalidParameter("t_max must be positive")
        if self.sigma0 is None:
            object.__setattr__(self, "sigma0", self.t_max / 10.0)
        if self.sigma0 <= 0.0:
            raise InvalidParameter("sigma0 must be positive")
        if self.eta_plus <= 1.0:
            raise InvalidParameter("eta_plus must exceed 1")
        if not 0.0 < self.eta_minus < 1.0:
            raise InvalidParameter("eta_minus must lie in (0, 1)")
        if self.delta <= 0.0:
            raise InvalidParameter("delta must be positive")
        if not 0.0 < self.safety <= 1.0:
            raise InvalidParameter("safety must lie in (0, 1]")

    def as_array(self):
        return np.array([self.t_max, self.sigma0, self.eta_plus, self.eta_minus, self.delta, self.safety],
                        dtype=np.float64)


@dataclass(frozen=True)
class HitResult:
    hit: bool
    t: float = float("inf")

    @staticmethod
    def hit_at(t: float) -> "HitResult":
        return HitResult(True, t)

    @staticmethod
    def miss() -> "HitResult":
        return HitResult(False)


@dataclass
class MarchStats:
    rounds: int = 0
    ray_steps: int = 0
    certified_steps: int = 0
    meta: dict = field(default_factory=dict)


def march_arrays(net, origins, dirs, params: RayCastParams = RayCastParams(), policy=None,
                 t_init=None, sigma_init=None, precision: str = "fp64", shared_origin: bool = False):
    """Lock-step adaptive march of many rays (rays.py:88-138).

    origins (n, 3) (or a single (3,) origin with shared_origin=True), dirs
    (n, 3); NumPy arrays or CUDA tensors.  Returns (hit, t, steps, stats);
    hit/t/steps come back as the same kind as `dirs`.
    """
    torch = dv._torch()
    policy = AFFINE_FIXED if policy is None else policy
    pcode, n_keep = policy_code(policy)
    host = not dv.is_tensor(dirs)
    dn = device_net(net, None if host else dirs.device.index)
    dev = dn.device
    d = dv.to_device(dirs, dev).reshape(-1, 3).contiguous()
    n = d.shape[0]
    o = dv.to_device(origins, dev).reshape(-1).contiguous() if shared_origin else \
        dv.to_device(origins, dev).reshape(-1, 3).contiguous()
    hit = torch.empty(n, dtype=torch.uint8, device=d.device)
    t = torch.empty(n, dtype=torch.float64, device=d.device)
    steps = torch.empty(n, dtype=torch.float64, device=d.device)
    ti = dv.to_device(t_init, dev).contiguous() if t_init is not None else None
    si = dv.to_device(sigma_init, dev).contiguous() if sigma_init is not None else None
    p6 = params.as_array()
    stats = np.zeros(3, np.int64)
    if n:
        _lib.call(
            "spk_march", dn.ptr, pcode, n_keep, _precision_code(precision), n, o.data_ptr(),
            0 if shared_origin else 3, d.data_ptr(), ti.data_ptr() if ti is not None else None,
            si.data_ptr() if si is not None else None, p6.ctypes.data, hit.data_ptr(), t.data_ptr(),
            steps.data_ptr(), stats.ctypes.data, dv.stream_ptr(dev),
        )
    st = MarchStats(int(stats[0]), int(stats[1]), int(stats[2]))
    if host:
        return hit.cpu().numpy().astype(bool), t.cpu().numpy(), steps.cpu().numpy(), st
    return hit.bool(), t, steps, st


def last_march_rounds():
    """(active rays, host ms) per lock-step round of this thread's last march
    (spk_march_round_log): the record behind the K6 tail analysis."""
    import ctypes as C

    lib = _lib.load()
    n = lib.spk_march_round_log(None, None, 0)
    active = np.zeros(n, np.int64)
    ms = np.zeros(n, np.float64)
    lib.spk_march_round_log(active.ctypes.data_as(C.c_void_p), ms.ctypes.data_as(C.c_void_p), n)
    return active, ms


def cast_rays(net, rays, params: RayCastParams = RayCastParams(), policy=None, threads: int = 1,
              precision: str = "fp64") -> list:
    """Cast many rays; elementwise identical to cast_ray on each (rays.py:151-184).
    `threads` is accepted for API compatibility (the GPU march is batch-invariant)."""
    rays = list(rays)
    if not rays:
        return []
    origins = np.stack([r.origin for r in rays])
    dirs = np.stack([r.dir for r in rays])
    hit, t, _, _ = march_arrays(net, origins, dirs, params, policy, precision=precision)
    return [HitResult(bool(h), float(tv)) for h, tv in zip(hit, t)]


def cast_ray(net, ray: Ray, params: RayCastParams = RayCastParams(), policy=None,
             precision: str = "fp64") -> HitResult:
    return cast_rays(net, [ray], params, policy, precision=precision)[0]


def cast_camera(net, camera: Camera, params: RayCastParams = RayCastParams(), policy=None,
                precision: str = "fp64", device=None):
    """March every pixel ray of a camera; directions are generated on the
    device.  Returns (hit (H, W) bool, t (H, W), steps (H, W), stats) tensors."""
    dirs = camera.pixel_dirs_device(device)
    hit, t, steps, st = march_arrays(net, dv._torch().from_numpy(camera.position).to(dirs.device),
                                     dirs.reshape(-1, 3), params, policy, precision=precision,
                                     shared_origin=True)
    h, w = camera.height, camera.width
    return hit.reshape(h, w), t.reshape(h, w), steps.reshape(h, w), st


def cast_camera_sharded(net, camera: Camera, rank: int, world: int, params: RayCastParams = RayCastParams(),
                        policy=None, precision: str = "fp64", tile: int = 16, device=None):
    """This rank's share of a camera image: interleaved tile x tile pixel
    tiles (tile i -> rank i mod world, shard.pixel_tiles) for static load
    balance; no collective inside the march.  Returns (pixel_index tensor,
    hit, t, steps, stats) for the rank's pixels (row-major image indices)."""
    from .shard import pixel_tiles

    torch = dv._torch()
    dirs = camera.pixel_dirs_device(device).reshape(-1, 3)
    w, h = camera.width, camera.height
    idx = []
    for ty, tx in pixel_tiles(w, h, tile, rank, world):
        ys = torch.arange(ty, min(ty + tile, h), device=dirs.device)
        xs = torch.arange(tx, min(tx + tile, w), device=dirs.device)
        idx.append((ys[:, None] * w + xs[None, :]).reshape(-1))
    pix = torch.cat(idx) if idx else torch.zeros(0, dtype=torch.int64, device=dirs.device)
    sel = dirs.index_select(0, pix).contiguous()
    origin = torch.from_numpy(camera.position).to(dirs.device)
    hit, t, steps, st = march_arrays(net, origin, sel, params, policy, precision=precision, shared_origin=True)
    return pix, hit, t, steps, st


def gather_camera_image(pix, hit, t, steps, n_pixels: int, device=None):
    """Final gather of cast_camera_sharded results (one all_gather per field
    group after the march: NCCL on GPUs, gloo on CPU).  Returns full-image
    NumPy arrays (hit bool, t FP64 with inf on misses, steps int64), pixel i
    at row-major index i, on every rank.  Single process: a scatter."""
    import torch.distributed as dist

    torch = dv._torch()
    from .shard import allgather_tensor

    if device is None:
        device = pix.device if dv.is_tensor(pix) else "cpu"

    def t_(x, dtype):
        x = x if dv.is_tensor(x) else torch.from_numpy(np.ascontiguousarray(x))
        return x.to(device=device, dtype=dtype).reshape(-1)

    # the image is assembled where the collective runs (the GPU with NCCL)
    ints = torch.stack([t_(pix, torch.int64), t_(hit, torch.int64), t_(steps, torch.int64)], dim=1)
    flts = t_(t, torch.float64).reshape(-1, 1)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        ints = torch.cat(allgather_tensor(ints, device), dim=0)
        flts = torch.cat(allgather_tensor(flts, device), dim=0)
    if torch.unique(ints[:, 0]).numel() != ints.shape[0]:
        raise InvalidParameter("pixel shards overlap")
    out_hit = torch.zeros(n_pixels, dtype=torch.bool, device=device)
    out_t = torch.full((n_pixels,), float("inf"), dtype=torch.float64, device=device)
    out_steps = torch.zeros(n_pixels, dtype=torch.int64, device=device)
    out_hit[ints[:, 0]] = ints[:, 1] != 0
    out_t[ints[:, 0]] = flts[:, 0]
    out_steps[ints[:, 0]] = ints[:, 2]
    return out_hit.cpu().numpy(), out_t.cpu().numpy(), out_steps.cpu().numpy()


@dataclass
class Frustum:
    """A rectangle of pixel rays marching together (rays.py:187-209)."""

    px0: int
    px1: int
    py0: int
    py1: int
    corner_dirs: np.ndarray  # (4, 3): (px0, py1-1), (px1-1, py1-1), (px0, py0), (px1-1, py0)
    t: float = 0.0
    sigma: float = 1.0

    @property
    def n_pixels(self) -> int:
        return (self.px1 - self.px0) * (self.py1 - self.py0)

    def front_widths(self) -> tuple:
        r00, r10, r01, r11 = self.corner_dirs
        wx = max(np.linalg.norm(r10 - r00), np.linalg.norm(r11 - r01))
        wy = max(np.linalg.norm(r01 - r00), np.linalg.norm(r11 - r10))
        return self.t * wx, self.t * wy


@dataclass
class FrustumCastResult:
    """rays.py:212-220: per-pixel hit mask, hit distance (inf on miss) and
    amortised marching steps, (H, W) each.  NumPy arrays by default, CUDA
    tensors with cast_frustum_image(..., device_output=True)."""

    hit: object
    t: object
    steps: object
    stats: MarchStats = field(default_factory=MarchStats)

    def total_steps(self) -> float:
        return float(self.steps.sum())


def cast_frustum_image(net, camera: Camera, params: RayCastParams = RayCastParams(), policy=None,
                       initial_grid: int = 16, precision: str = "fp64", device_output: bool = False,
                       device=None) -> FrustumCastResult:
    """Frustum range-marching of a whole image (rays.py:232-341).

    Same contract as casting every pixel separately (identical hit mask, t
    within delta); with precision="fp64" the results are bit-identical to
    the reference's cast_frustum_image.  Runs in the C-ABI
    (spk_frustum_cast): slab-box bounds of every marching frustum per round
    in one fused bound pass, single pixels finished by the device march.
    stats.meta holds frustum_rounds / frustum_steps / pixel_handoffs /
    dissolved_frusta.  One guard is added to the reference's loop: an
    uncertified multi-pixel frustum whose sigma falls below delta * 2^-32
    dissolves into single-pixel hand-offs (the reference would loop forever
    on a frustum at t = 0 whose bound cannot resolve |f| there)."""
    from .errors import InvalidCamera

    torch = dv._torch()
    policy = AFFINE_FIXED if policy is None else policy
    pcode, n_keep = policy_code(policy)
    w, h = camera.resolution
    gw, gh = min(initial_grid, w), min(initial_grid, h)
    if initial_grid < 1 or w % gw != 0 or h % gh != 0:
        raise InvalidCamera(f"resolution {w}x{h} not divisible into a {gw}x{gh} frustum grid")
    dn = device_net(net, device)
    dev = dn.device
    hit = torch.empty((h, w), dtype=torch.uint8, device=f"cuda:{dev}")
    t = torch.empty((h, w), dtype=torch.float64, device=f"cuda:{dev}")
    steps = torch.empty((h, w), dtype=torch.float64, device=f"cuda:{dev}")
    pos = np.ascontiguousarray(camera.position, dtype=np.float64)
    frame = np.ascontiguousarray(np.concatenate(camera.frame))
    hw, hh = camera.half_extents
    p6 = params.as_array()
    stats = np.zeros(5, np.int64)
    _lib.call("spk_frustum_cast", dn.ptr, pcode, n_keep, _precision_code(precision), pos.ctypes.data,
              frame.ctypes.data, hw, hh, w, h, initial_grid, p6.ctypes.data, hit.data_ptr(), t.data_ptr(),
              steps.data_ptr(), stats.ctypes.data, dv.stream_ptr(dev))
    st = MarchStats(rounds=int(stats[0]), ray_steps=int(stats[3]),
                    meta={"frustum_rounds": int(stats[0]), "frustum_steps": int(stats[1]),
                          "pixel_handoffs": int(stats[2]), "dissolved_frusta": int(stats[4])})
    if device_output:
        return FrustumCastResult(hit.bool(), t, steps, st)
    return FrustumCastResult(hit.cpu().numpy().astype(bool), t.cpu().numpy(), steps.cpu().numpy(), st)
