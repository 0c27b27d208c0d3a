"""Image rendering from ray casts (reference render.py:1-186).

render_image keeps the reference signature and output: primary rays are
marched per pixel (`per_ray`, K6), as frusta (`frustum`, spk_frustum_cast)
or at fixed steps (`fixed_step`, the uniform-marching baseline); every hit
is refined by 48 bisections, shaded by Lambert max(0, n . l) with a
central-difference normal, and misses get the background colour.  All of
it runs in the C-ABI (spk_render_shade / spk_fixed_step_march) on the
device; only the finished (H, W, 3) uint8 image comes back.  Image,
write_image (binary P6 / PNG) and read_ppm are the reference's host-side
file I/O.
"""

from __future__ import annotations

import struct
import zlib
from dataclasses import dataclass

import numpy as np

from . import _lib
from . import device as dv
from .camera import Camera
from .errors import InvalidImage, InvalidParameter
from .network import _precision_code, device_net
from .range_core import AFFINE_FIXED, policy_code
from .rays import RayCastParams, cast_camera, cast_frustum_image

BACKGROUND = np.array([24, 28, 38], dtype=np.uint8)
LIGHT_DIR = np.array([0.35, 0.75, 0.56])
LIGHT_DIR = LIGHT_DIR / np.linalg.norm(LIGHT_DIR)
REFINE_ITERS = 48


@dataclass(frozen=True)
class Image:
    """An RGB8 raster, (height, width, 3) row-major, top row first."""

    width: int
    height: int
    pixels: np.ndarray

    def __post_init__(self):
        buf = np.asarray(self.pixels, dtype=np.uint8)
        want = (self.height, self.width, 3)
        if buf.shape != want:
            raise InvalidImage(f"pixel buffer {buf.shape} does not match {self.width}x{self.height}")
        object.__setattr__(self, "pixels", buf)


def fixed_step_march(net, camera: Camera, step: float, params: RayCastParams = RayCastParams(),
                     precision: str = "fp64", device=None):
    """Uniform-step baseline over every pixel (render.py:36-56); returns
    device (hit (H*W,) bool, t (H*W,)) tensors and the round count."""
    torch = dv._torch()
    if step is None or not step > 0.0:
        raise InvalidParameter("fixed_step mode needs a positive step")
    dirs = camera.pixel_dirs_device(device).reshape(-1, 3)
    dn = device_net(net, dirs.device.index)
    n = dirs.shape[0]
    origin = torch.from_numpy(camera.position).to(dirs.device)
    hit = torch.empty(n, dtype=torch.uint8, device=dirs.device)
    t = torch.empty(n, dtype=torch.float64, device=dirs.device)
    stats = np.zeros(2, np.int64)
    _lib.call("spk_fixed_step_march", dn.ptr, _precision_code(precision), n, origin.data_ptr(), 0, dirs.data_ptr(),
              float(step), float(params.t_max), hit.data_ptr(), t.data_ptr(), stats.ctypes.data,
              dv.stream_ptr(dn.device))
    return hit, t, int(stats[0])


def shade_hits(net, camera: Camera, dirs, hit, t, delta: float, precision: str = "fp64"):
    """Refine, normal-estimate and shade every hit pixel on the device
    (render.py:128-140).  dirs (H*W, 3), hit (H*W,), t (H*W,) CUDA tensors;
    returns the (H, W, 3) uint8 image as a CUDA tensor."""
    torch = dv._torch()
    dn = device_net(net, dirs.device.index)
    n = dirs.shape[0]
    origin = torch.from_numpy(camera.position).to(dirs.device)
    pixels = torch.empty((n, 3), dtype=torch.uint8, device=dirs.device)
    light = np.ascontiguousarray(LIGHT_DIR, dtype=np.float64)
    bg = np.ascontiguousarray(BACKGROUND)
    h8 = hit.to(torch.uint8).contiguous()
    tt = t.to(torch.float64).contiguous()
    _lib.call("spk_render_shade", dn.ptr, _precision_code(precision), n, origin.data_ptr(), 0,
              dirs.contiguous().data_ptr(), h8.data_ptr(), tt.data_ptr(), float(delta), REFINE_ITERS,
              light.ctypes.data, bg.ctypes.data, pixels.data_ptr(), None, dv.stream_ptr(dn.device))
    return pixels.reshape(camera.height, camera.width, 3)


def render_image(net, camera: Camera, params: RayCastParams = RayCastParams(), policy=AFFINE_FIXED,
                 mode: str = "per_ray", step: float | None = None, threads: int = 1,
                 precision: str = "fp64", device=None) -> Image:
    """Render primary rays with Lambert shading (render.py:91-141).

    mode: per_ray | frustum | fixed_step (needs step > 0).  `threads` is
    accepted for API compatibility (the device march is batch-invariant).
    `precision` selects the arithmetic of the march and of the shading
    passes ("fp64" = the reference's; "fp32" marches with the sound FP32
    kernels and still shades in FP64)."""
    torch = dv._torch()
    if mode == "per_ray":
        hit, t, _, _ = cast_camera(net, camera, params, policy, precision=precision, device=device)
        hit, t = hit.reshape(-1), t.reshape(-1)
    elif mode == "frustum":
        fr = cast_frustum_image(net, camera, params, policy, precision=precision, device_output=True, device=device)
        hit, t = fr.hit.reshape(-1), fr.t.reshape(-1)
    elif mode == "fixed_step":
        if step is None or step <= 0.0:
            raise InvalidParameter("fixed_step mode needs a positive step")
        hit, t, _ = fixed_step_march(net, camera, step, params, precision=precision, device=device)
    else:
        raise InvalidParameter(f"unknown render mode {mode!r}")
    dirs = camera.pixel_dirs_device(hit.device.index)
    px = shade_hits(net, camera, dirs.reshape(-1, 3), hit, t, params.delta, precision="fp64")
    return Image(camera.width, camera.height, px.cpu().numpy())


def _png_bytes(pixels: np.ndarray) -> bytes:
    h, w, _ = pixels.shape
    raw = b"".join(b"\x00" + pixels[y].tobytes() for y in range(h))

    def chunk(tag, data):
        body = tag + data
        return struct.pack(">I", len(data)) + body + struct.pack(">I", zlib.crc32(body) & 0xFFFFFFFF)

    return (b"\x89PNG\r\n\x1a\n" + chunk(b"IHDR", struct.pack(">IIBBBBB", w, h, 8, 2, 0, 0, 0))
            + chunk(b"IDAT", zlib.compress(raw, 6)) + chunk(b"IEND", b""))


def _write_ppm(img: Image, path) -> None:
    head = b"P6\n%d %d\n255\n" % (img.width, img.height)
    with open(path, "wb") as f:
        f.write(head + np.ascontiguousarray(img.pixels).tobytes())


def _write_png(img: Image, path) -> None:
    try:
        from PIL import Image as PILImage
    except ImportError:  # Pillow is optional: a minimal zlib encoder
        with open(path, "wb") as f:
            f.write(_png_bytes(img.pixels))
        return
    PILImage.fromarray(img.pixels, mode="RGB").save(path, format="PNG")


_WRITERS = {"ppm": _write_ppm, "png": _write_png}


def write_image(img: Image, path, fmt: str | None = None) -> None:
    """Binary P6 (maxval 255) or 8-bit RGB PNG (render.py:144-168); without
    `fmt` the path suffix decides."""
    if min(img.width, img.height) < 1 or img.pixels.size == 0:
        raise InvalidImage("refusing to write an empty image")
    kind = (fmt or str(path).rsplit(".", 1)[-1]).lower()
    writer = _WRITERS.get(kind)
    if writer is None:
        raise InvalidImage(f"unsupported image format {kind!r}")
    writer(img, path)


def read_ppm(path) -> Image:
    """Load a binary P6 / maxval-255 file as written by write_image
    (render.py:171-180)."""
    blob = open(path, "rb").read()
    fields = blob.split(b"\n", 3)
    ok = len(fields) == 4 and fields[0] == b"P6" and fields[2] == b"255"
    if not ok:
        raise InvalidImage(f"{path} is not a P6 file with maxval 255")
    width, height = map(int, fields[1].split())
    raster = np.frombuffer(fields[3], dtype=np.uint8, count=width * height * 3)
    return Image(width, height, raster.reshape(height, width, 3).copy())
