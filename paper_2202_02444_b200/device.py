"""Device-buffer plumbing (torch is used only for memory, streams and
transfers; all arithmetic happens in the C-ABI kernels)."""

from __future__ import annotations

import numpy as np

from . import _lib
from .errors import DimensionMismatch


def _torch():
    import torch

    return torch


def is_tensor(x) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor)


def as_points(xs, d: int):
    if is_tensor(xs):
        t = xs
        if t.dim() != 2 or t.shape[1] != d:
            if t.numel() == 0:
                return t.reshape(0, d)
            raise DimensionMismatch(f"expected points of shape (n, {d}), got {tuple(t.shape)}")
        return t.to(dtype=_torch().float64).contiguous()
    x = np.asarray(xs, dtype=np.float64)
    if x.size == 0:
        return np.zeros((0, d))
    if x.ndim != 2 or x.shape[1] != d:
        raise DimensionMismatch(f"expected points of shape (n, {d}), got {x.shape}")
    return np.ascontiguousarray(x)


def is_empty(x) -> bool:
    return (x.numel() if is_tensor(x) else x.size) == 0


def length(x) -> int:
    return int(x.shape[0])


def device_of(x):
    if is_tensor(x) and x.is_cuda:
        return x.device.index
    return None


def empty_like_out(orig, n):
    if is_tensor(orig):
        return _torch().zeros(n, dtype=_torch().float64, device=orig.device)
    return np.zeros(n)


def stream_ptr(device=None):
    torch = _torch()
    return torch.cuda.current_stream(device).cuda_stream


def to_device(x, device):
    torch = _torch()
    if is_tensor(x):
        return x.to(device=f"cuda:{device}", dtype=torch.float64).contiguous()
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
    return t.to(device=f"cuda:{device}", non_blocking=False)


def run_eval(dn, x, prec, orig):
    torch = _torch()
    xd = to_device(x, dn.device)
    out = torch.empty(xd.shape[0], dtype=torch.float64, device=xd.device)
    _lib.call("spk_eval_batch", dn.ptr, prec, xd.shape[0], xd.data_ptr(), out.data_ptr(), stream_ptr(dn.device))
    if is_tensor(orig):
        return out
    return out.cpu().numpy()
