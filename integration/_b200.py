"""B200 drop-in for the reference's bound operator (Option B).

This file is what a maintainer adds to the reference package as
`spelunk/_b200.py`; `install_shim.py` (next to it) also appends the 6-line
dispatch to `spelunk/range_core.py`, so `range_bound_batch`
(range_core.py:547) and `interval_forward_batch` (range_core.py:625) run on
the GPU through the C-ABI (include/spelunk_b200.h) when
SPELUNK_BACKEND=b200.  Every caller that imported the symbols by name picks
the dispatch up (spatial.py:183, rays.py:132, meshing.py:146, bench.py:96).

Environment:
  SPELUNK_B200_LIB        path of _spk.so (required)
  SPELUNK_B200_PRECISION  fp64 (default: the reference's own FP64 arithmetic,
                          no rounding padding -- SPK_NET_FP64_UNPADDED -- so its
                          exact and 1e-12 tests hold), fp32 (sound FP32) or
                          fp32-refine (FP32, near-certifiable UNKNOWN boxes
                          re-bounded in FP64: the reference's labels)
  SPELUNK_B200_CALLS      optional file: the number of GPU calls is written
                          there at exit (lets a test prove the GPU ran)

Only plain ctypes and NumPy: no torch, nothing from the B200 package.
"""

from __future__ import annotations

import atexit
import ctypes as C
import os
import threading
import weakref

import numpy as np

from .errors import DepthOverflow, DimensionMismatch, InvalidParameter, SpelunkError, UnsupportedActivation
from .network import DenseLayer

_lib = C.CDLL(os.environ["SPELUNK_B200_LIB"])
_vp, _i32, _i64 = C.c_void_p, C.c_int, C.c_int64
_lib.spk_net_create_ex.argtypes = [_i32, _i32, _vp, _vp, _vp, _i64, _i32, _i32, _vp]
_lib.spk_net_create_ex.restype = _i32
_lib.spk_net_destroy.argtypes = [_vp]
_lib.spk_bound_batch_host.argtypes = [_vp, _i32, _i32, _i32, _i64, _i32, _vp, _vp, _vp, _vp, _vp]
_lib.spk_bound_batch_host.restype = _i32
_lib.spk_last_error.restype = C.c_char_p

_OPS = {"relu": 1, "elu": 2, "sin": 3, "tanh": 4, "identity": 5}
_POL = {"interval": 0, "affine-fixed": 1, "affine-full": 2, "affine-truncate": 3}
_ERR = {1: DimensionMismatch, 2: UnsupportedActivation, 3: InvalidParameter, 4: DepthOverflow}
_PRECISION = {"fp32": 0, "fp64": 1, "fp32-refine": 2}[os.environ.get("SPELUNK_B200_PRECISION", "fp64")]

_handles: dict[int, tuple] = {}
# re-entrant: a weakref.finalize callback (_drop) can run from a garbage
# collection triggered inside _handle while this thread holds the lock
_lock = threading.RLock()
_calls = [0]


def _check(status: int) -> None:
    if status:
        raise _ERR.get(status, SpelunkError)(_lib.spk_last_error().decode())


def _drop(key: int) -> None:
    with _lock:
        entry = _handles.pop(key, None)
    if entry is not None:
        _lib.spk_net_destroy(entry[1])


def _handle(net):
    """Upload the net once; the device copy lives as long as the NetworkSpec
    (weakref.finalize), so a recycled id() never maps to stale weights."""
    key = id(net)
    with _lock:
        entry = _handles.get(key)
        if entry is not None:
            return entry[1]
        kinds, outs, params = [], [], []
        for layer in net.layers:
            if isinstance(layer, DenseLayer):
                kinds.append(0)
                outs.append(layer.weights.shape[0])
                params += [np.asarray(layer.weights, np.float64).ravel(), np.asarray(layer.bias, np.float64).ravel()]
            else:
                if layer.value not in _OPS:
                    raise UnsupportedActivation(f"no affine rule for {layer!r}")
                kinds.append(_OPS[layer.value])
                outs.append(0)
        k = np.array(kinds, np.int32)
        o = np.array(outs, np.int32)
        p = np.ascontiguousarray(np.concatenate(params) if params else np.zeros(0))
        h = C.c_void_p()
        # fp64: the reference's own (unpadded) FP64 arithmetic, SPK_NET_FP64_UNPADDED
        _check(_lib.spk_net_create_ex(net.input_dim, len(k), k.ctypes.data, o.ctypes.data, p.ctypes.data, p.size,
                                      0, 1 if _PRECISION == 1 else 0, C.byref(h)))
        try:
            weakref.finalize(net, _drop, key)
            _handles[key] = (None, h)
        except TypeError:  # not weak-referenceable: pin the net so its id stays unique
            _handles[key] = (net, h)
        return h


def range_bound_batch(net, centers, axes, policy):
    """range_core.range_bound_batch on the GPU: same contract (FP64 NumPy in
    and out, DimensionMismatch / UnsupportedActivation / InvalidParameter)."""
    c = np.ascontiguousarray(centers, dtype=np.float64)
    if c.ndim != 2 or c.shape[1] != net.input_dim:
        raise DimensionMismatch(f"centers must be (n, {net.input_dim})")
    n = c.shape[0]
    a = np.ascontiguousarray(axes, dtype=np.float64)
    if a.ndim != 3 or a.shape[0] != n or a.shape[2] != net.input_dim:
        raise DimensionMismatch(f"axes must be (n, s, {net.input_dim})")
    lo = np.empty(n)
    hi = np.empty(n)
    if n == 0:
        return lo, hi
    pol = _POL[policy.kind.value]
    status = _lib.spk_bound_batch_host(_handle(net), pol, int(policy.n_keep or 0), _PRECISION, n, a.shape[1],
                                       c.ctypes.data, a.ctypes.data, lo.ctypes.data, hi.ctypes.data, None)
    _check(status)
    _calls[0] += 1
    return lo, hi


def interval_forward_batch(net, centers, axes):
    from .range_core import INTERVAL_ONLY

    return range_bound_batch(net, centers, axes, INTERVAL_ONLY)


@atexit.register
def _report_calls():
    path = os.environ.get("SPELUNK_B200_CALLS")
    if path:
        with open(path, "w") as f:
            f.write(str(_calls[0]))
