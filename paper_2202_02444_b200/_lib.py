"""ctypes binding of the in-tree C-ABI library (include/spelunk_b200.h).

There is no CPU fallback: if `_spk.so` is missing or cannot be loaded, every
compute entry point raises DeviceError.  Build it with
`python -m paper_2202_02444_b200.build` (or `__graft_entry__.build()`).
"""

from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

from . import errors as E

import os

# SPK_LIB_PATH overrides the in-tree library (used to A/B kernel variants)
LIB_PATH = Path(os.environ.get("SPK_LIB_PATH") or Path(__file__).resolve().parent / "_spk.so")

# status codes (spelunk_b200.h)
OK, ERR_DIM, ERR_ACT, ERR_PARAM, ERR_DEPTH, ERR_CUDA, ERR_SHAPE, ERR_OOM = range(8)
OP_DENSE, OP_RELU, OP_ELU, OP_SIN, OP_TANH, OP_IDENTITY = range(6)
POLICY_INTERVAL, POLICY_AFFINE_FIXED, POLICY_AFFINE_FULL, POLICY_AFFINE_TRUNCATE = range(4)
FP32, FP64, FP32_REFINE = 0, 1, 2

_EXC = {
    ERR_DIM: E.DimensionMismatch,
    ERR_ACT: E.UnsupportedActivation,
    ERR_PARAM: E.InvalidParameter,
    ERR_DEPTH: E.DepthOverflow,
    ERR_CUDA: E.DeviceError,
    ERR_SHAPE: E.DeviceError,
    ERR_OOM: E.DeviceError,
}

_lock = threading.Lock()
_lib = None

vp = C.c_void_p
i32 = C.c_int
i64 = C.c_int64
u64 = C.c_uint64
f64 = C.c_double

# name -> argtypes; every function returns int status unless noted
SIGNATURES = {
    "spk_last_error": ([], C.c_char_p),
    "spk_version": ([], i32),
    "spk_refine_band": ([f64, vp], i32),
    "spk_net_refine_band": ([vp, i32, vp, vp], i32),
    "spk_device_sm_count": ([], i32),
    "spk_ffma_peak": ([i32, vp, vp], i32),
    "spk_net_create": ([i32, i32, vp, vp, vp, i64, i32, vp], i32),
    "spk_net_create_ex": ([i32, i32, vp, vp, vp, i64, i32, i32, vp], i32),
    "spk_net_destroy": ([vp], i32),
    "spk_net_info": ([vp, vp, vp, vp], i32),
    "spk_net_debug_corrupt_relu": ([vp, i32], i32),
    "spk_bound_batch": ([vp, i32, i32, i32, i64, i32, vp, vp, vp, vp, vp, vp], i32),
    "spk_bound_aabb": ([vp, i32, i32, i32, i64, vp, vp, vp, vp, vp, vp], i32),
    "spk_bound_random_cubes": ([vp, i32, i32, i32, i64, i64, u64, f64, vp, vp, vp, vp], i32),
    "spk_eval_batch": ([vp, i32, i64, vp, vp, vp], i32),
    "spk_bound_batch_host": ([vp, i32, i32, i32, i64, i32, vp, vp, vp, vp, vp], i32),
    "spk_tree_build": ([vp, i32, i32, i32, i64, vp, vp, i32, i32, f64, vp, vp], i32),
    "spk_tree_build_band": ([vp, i32, i32, i32, i64, vp, vp, i32, i32, f64, f64, vp, vp], i32),
    "spk_tree_build_ex": ([vp, i32, i32, i32, i64, vp, vp, i32, i32, f64, f64, i32, vp, vp], i32),
    "spk_tree_level_host": ([vp, i32, vp, vp, vp, vp, vp, vp, vp, vp], i32),
    "spk_tree_release_device": ([vp], i32),
    "spk_tree_stats": ([vp, vp, vp], i32),
    "spk_tree_level_copy": ([vp, i32, vp, vp, vp, vp, vp, vp, vp], i32),
    "spk_march": ([vp, i32, i32, i32, i64, vp, i64, vp, vp, vp, vp, vp, vp, vp, vp, vp], i32),
    "spk_march_round_log": ([vp, vp, i32], i32),
    "spk_camera_dirs": ([vp, f64, f64, i32, i32, vp, vp], i32),
    "spk_affine_rule": ([i32, i32, i64, vp, vp, vp, vp, vp], i32),
    "spk_render_shade": ([vp, i32, i64, vp, i64, vp, vp, vp, f64, i32, vp, vp, vp, vp, vp], i32),
    "spk_fixed_step_march": ([vp, i32, i64, vp, i64, vp, f64, f64, vp, vp, vp, vp], i32),
    "spk_certified_radii": ([vp, i32, i32, i32, i64, vp, vp, f64, vp, vp, vp], i32),
    "spk_intersect": ([vp, vp, i32, i32, i32, vp, vp, f64, vp, vp, vp, vp, vp, vp, i64, vp, vp], i32),
    "spk_bisect": ([vp, i32, i64, vp, vp, i32, vp, vp], i32),
    "spk_frustum_cast": ([vp, i32, i32, i32, vp, vp, f64, f64, i32, i32, i32, vp, vp, vp, vp, vp, vp], i32),
    "spk_mesh_extract": ([vp, i32, i32, i32, vp, vp, i32, i32, i32, vp, vp, vp, vp], i32),
    "spk_mesh_extract_shard": ([vp, i32, i32, i32, vp, vp, i32, i32, i32, vp, vp, i32, i32, vp, vp], i32),
    "spk_mesh_info": ([vp, vp, vp, vp, vp, vp], i32),
    "spk_mesh_shard_info": ([vp, vp, vp], i32),
    "spk_mesh_copy": ([vp, vp, vp, vp], i32),
    "spk_mesh_destroy": ([vp], i32),
    "spk_tree_destroy": ([vp], i32),
    "spk_tree_info": ([vp, vp, vp, vp], i32),
    "spk_tree_level": ([vp, i32, vp, vp, vp, vp, vp, vp, vp, vp], i32),
}


def load():
    """Load the library once; raise DeviceError (never fall back) on failure."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise E.DeviceError(
                f"CUDA library {LIB_PATH} not built; run `python -m paper_2202_02444_b200.build`"
            )
        try:
            lib = C.CDLL(str(LIB_PATH))
        except OSError as exc:
            raise E.DeviceError(f"cannot load {LIB_PATH}: {exc}") from exc
        for name, (args, res) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
        return lib


def check(status: int, what: str = ""):
    if status == OK:
        return
    msg = load().spk_last_error().decode(errors="replace")
    raise _EXC.get(status, E.SpelunkError)(f"{what}: {msg}" if what else msg)


def call(name: str, *args):
    check(getattr(load(), name)(*args), name)
