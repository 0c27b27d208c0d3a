"""Batched range analysis on the B200 -- the reference's `range_core`
operator boundary (range_core.py:42-201, 471-646), backed by the fused
sm_100a kernels behind the C-ABI.

`range_bound_batch(net, centers, axes, policy)` keeps the reference
signature and return types: FP64 NumPy in, FP64 NumPy out.  CUDA tensors are
accepted too and stay on the device (the throughput path).  `precision`
selects the kernel arithmetic: "fp32" (default: FP32 FFMA with directed
rounding, sound), "fp64", or "fp32-refine" (FP32, then the boxes FP32 leaves
UNKNOWN within a calibrated band of a certification re-bounded in FP64: the
labels are the reference-precision decisions at close to FP32 cost;
`refine_band`).
"""

from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass

import numpy as np

from . import _lib
from . import device as dv
from .errors import DimensionMismatch, InvalidParameter, NonOrthogonalAxes
from .network import _precision_code, device_net


class SignClass(enum.Enum):
    POSITIVE = "positive"
    NEGATIVE = "negative"
    UNKNOWN = "unknown"


@dataclass(frozen=True)
class Interval:
    lo: float | np.ndarray
    hi: float | np.ndarray

    def __post_init__(self):
        if not np.all(np.asarray(self.lo) <= np.asarray(self.hi)):
            raise InvalidParameter("interval requires lo <= hi")
        if not (np.all(np.isfinite(self.lo)) and np.all(np.isfinite(self.hi))):
            raise InvalidParameter("interval bounds must be finite")

    @property
    def width(self):
        return self.hi - self.lo

    def contains(self, value, slack: float = 0.0) -> bool:
        v = np.asarray(value)
        return bool(np.all(v >= self.lo - slack) and np.all(v <= self.hi + slack))


class PolicyKind(enum.Enum):
    INTERVAL = "interval"
    AFFINE_FIXED = "affine-fixed"
    AFFINE_FULL = "affine-full"
    AFFINE_TRUNCATE = "affine-truncate"


@dataclass(frozen=True)
class CondensationPolicy:
    """range_core.py:111-136."""

    kind: PolicyKind
    n_keep: int | None = None

    def __post_init__(self):
        if self.kind is PolicyKind.AFFINE_TRUNCATE:
            if self.n_keep is None or self.n_keep < 1:
                raise InvalidParameter("affine-truncate requires n_keep >= 1")
        elif self.n_keep is not None:
            raise InvalidParameter(f"{self.kind.value} does not take n_keep")

    def __str__(self):
        if self.kind is PolicyKind.AFFINE_TRUNCATE:
            return f"affine-truncate:{self.n_keep}"
        return self.kind.value


INTERVAL_ONLY = CondensationPolicy(PolicyKind.INTERVAL)
AFFINE_FIXED = CondensationPolicy(PolicyKind.AFFINE_FIXED)
AFFINE_FULL = CondensationPolicy(PolicyKind.AFFINE_FULL)


def affine_truncate(n_keep: int) -> CondensationPolicy:
    return CondensationPolicy(PolicyKind.AFFINE_TRUNCATE, n_keep)


def parse_policy(name: str) -> CondensationPolicy:
    """interval | affine-fixed | affine-full | affine-truncate:N (range_core.py:148-165)."""
    key = name.strip().lower()
    fixed = {"interval": INTERVAL_ONLY, "affine-fixed": AFFINE_FIXED, "affine-full": AFFINE_FULL}
    if key in fixed:
        return fixed[key]
    if key.startswith("affine-truncate"):
        _, _, arg = key.partition(":")
        if not arg:
            raise InvalidParameter("affine-truncate needs :N, e.g. affine-truncate:16")
        try:
            return affine_truncate(int(arg))
        except ValueError as exc:
            raise InvalidParameter(f"bad n_keep in {name!r}") from exc
    raise InvalidParameter(f"unknown policy {name!r}")


_POLICY_CODE = {
    "interval": _lib.POLICY_INTERVAL,
    "affine-fixed": _lib.POLICY_AFFINE_FIXED,
    "affine-full": _lib.POLICY_AFFINE_FULL,
    "affine-truncate": _lib.POLICY_AFFINE_TRUNCATE,
}


def policy_code(policy) -> tuple[int, int]:
    """(C-ABI policy code, n_keep) for a policy object, reference policy or string."""
    if isinstance(policy, str):
        policy = parse_policy(policy)
    kind = getattr(policy.kind, "value", policy.kind)
    if kind not in _POLICY_CODE:
        raise InvalidParameter(f"unknown policy {policy!r}")
    return _POLICY_CODE[kind], int(policy.n_keep or 0)


@dataclass(frozen=True)
class QueryBox:
    """s-dimensional oriented box: centre + s pairwise-orthogonal half-axes."""

    center: np.ndarray
    axes: np.ndarray

    def __post_init__(self):
        c = np.asarray(self.center, dtype=np.float64)
        a = np.asarray(self.axes, dtype=np.float64)
        if a.size == 0:
            a = a.reshape(0, c.shape[0])
        if c.ndim != 1 or a.ndim != 2 or a.shape[1] != c.shape[0]:
            raise DimensionMismatch("axes must have shape (s, d) matching center")
        if a.shape[0] > c.shape[0]:
            raise DimensionMismatch("more axes than ambient dimensions")
        norms = np.linalg.norm(a, axis=1)
        if np.any(norms == 0.0) or not np.all(np.isfinite(a)):
            raise NonOrthogonalAxes("axes must be finite and nonzero")
        gram = a @ a.T
        off = gram - np.diag(np.diag(gram))
        if np.any(np.abs(off) > 1e-6 * np.outer(norms, norms)):
            raise NonOrthogonalAxes("axes are not pairwise orthogonal")
        object.__setattr__(self, "center", c)
        object.__setattr__(self, "axes", a)

    @property
    def dim(self) -> int:
        return self.center.shape[0]

    @property
    def s(self) -> int:
        return self.axes.shape[0]


def classify(lo, hi) -> SignClass:
    if lo > 0.0:
        return SignClass.POSITIVE
    if hi < 0.0:
        return SignClass.NEGATIVE
    return SignClass.UNKNOWN


def sign_classes(lo, hi) -> list[SignClass]:
    return [classify(a, b) for a, b in zip(np.asarray(lo), np.asarray(hi))]


def _trim_axes(axes):
    """Drop trailing all-zero axis rows (padding, range_core.py:550-551)."""
    if dv.is_tensor(axes):
        nz = (axes != 0).any(dim=2).any(dim=0)
        keep = int(nz.nonzero().max().item()) + 1 if bool(nz.any()) else 0
    else:
        nz = np.any(axes != 0.0, axis=(0, 2))
        keep = int(np.flatnonzero(nz).max()) + 1 if nz.any() else 0
    return axes[:, :keep, :]


def refine_band(tau=None) -> float:
    """Get (and, given tau, set) the band of precision "fp32-refine": UNKNOWN
    boxes whose FP32 bound comes within tau * (S + w) of certifying (-lo or
    hi <= tau (S + w), S = max(1, |lo|, |hi|)) are re-bounded in FP64.
    Default ("auto", reported as -1): each net calibrates its own band on
    first use (3 x its largest FP32 excess over FP64 on 8192 random cubes).
    A float >= 0 forces a process-wide band.  Returns the previous setting."""
    prev = C.c_double(0.0)
    if tau is None:
        _lib.call("spk_refine_band", -1.0, C.byref(prev))  # query only
        return prev.value
    if isinstance(tau, str):
        if tau != "auto":
            raise InvalidParameter(f"unknown refine band {tau!r}")
        _lib.call("spk_refine_band", -2.0, C.byref(prev))
        return prev.value
    if not (float(tau) >= 0.0) or not np.isfinite(tau):
        raise InvalidParameter("refine band must be finite and >= 0")
    _lib.call("spk_refine_band", float(tau), C.byref(prev))
    return prev.value


def net_refine_band(net, policy=AFFINE_FIXED, device=None) -> float:
    """The band "fp32-refine" uses for this net and policy (calibrating the
    net's band now if no process-wide band is forced)."""
    pcode, _ = policy_code(policy)
    dn = device_net(net, device)
    out = C.c_double(0.0)
    _lib.call("spk_net_refine_band", dn.ptr, pcode, dv.stream_ptr(device), C.byref(out))
    return out.value


def range_bound_batch(net, centers, axes, policy=AFFINE_FIXED, precision: str = "fp32",
                      return_class: bool = False):
    """Bound the network over n oriented boxes (range_core.py:547-622).

    centers (n, d); axes (n, s, d), zero rows are padding.  Returns (lo, hi)
    (and the int8 sign class +1/-1/0 if return_class).  NumPy inputs go
    through the native host pipeline (copies overlap kernels); CUDA tensors
    stay on their device and run on the current stream.
    """
    pcode, n_keep = policy_code(policy)
    prec = _precision_code(precision)
    d = int(net.input_dim)
    if dv.is_tensor(centers):
        return _bound_device(net, centers, axes, pcode, n_keep, prec, return_class)
    c = np.asarray(centers, dtype=np.float64)
    if c.ndim != 2 or c.shape[1] != d:
        raise DimensionMismatch(f"centers must be (n, {d})")
    n = c.shape[0]
    a = np.asarray(axes, dtype=np.float64)
    if a.size == 0:
        a = np.zeros((n, 0, d))
    if a.ndim != 3 or a.shape[0] != n or a.shape[2] != d:
        raise DimensionMismatch(f"axes must be (n, s, {d})")
    a = _trim_axes(a)
    lo = np.empty(n)
    hi = np.empty(n)
    cls = np.empty(n, np.int8)
    if n:
        dn = device_net(net)
        c = np.ascontiguousarray(c)
        a = np.ascontiguousarray(a)
        _lib.call(
            "spk_bound_batch_host", dn.ptr, pcode, n_keep, prec, n, a.shape[1],
            c.ctypes.data, a.ctypes.data, lo.ctypes.data, hi.ctypes.data, cls.ctypes.data,
        )
    return (lo, hi, cls) if return_class else (lo, hi)


def _bound_device(net, centers, axes, pcode, n_keep, prec, return_class):
    torch = dv._torch()
    d = int(net.input_dim)
    c = centers.to(torch.float64).contiguous()
    if c.dim() != 2 or c.shape[1] != d:
        raise DimensionMismatch(f"centers must be (n, {d})")
    n = c.shape[0]
    a = axes.to(device=c.device, dtype=torch.float64)
    if a.numel() == 0:
        a = torch.zeros((n, 0, d), dtype=torch.float64, device=c.device)
    if a.dim() != 3 or a.shape[0] != n or a.shape[2] != d:
        raise DimensionMismatch(f"axes must be (n, s, {d})")
    a = a.contiguous()  # no device-side trimming: zero axis rows are harmless and a trim would sync
    lo = torch.empty(n, dtype=torch.float64, device=c.device)
    hi = torch.empty(n, dtype=torch.float64, device=c.device)
    cls = torch.empty(n, dtype=torch.int8, device=c.device)
    if n:
        dn = device_net(net, c.device.index)
        _lib.call(
            "spk_bound_batch", dn.ptr, pcode, n_keep, prec, n, a.shape[1], c.data_ptr(), a.data_ptr(),
            lo.data_ptr(), hi.data_ptr(), cls.data_ptr(), dv.stream_ptr(c.device),
        )
    return (lo, hi, cls) if return_class else (lo, hi)


def interval_forward_batch(net, centers, axes, precision: str = "fp32"):
    """Interval propagation over the boxes' axis-aligned hulls (range_core.py:625-642)."""
    return range_bound_batch(net, centers, axes, INTERVAL_ONLY, precision)


def bound_aabb(net, box_lo, box_hi, policy=AFFINE_FIXED, precision: str = "fp32"):
    """Device-side bound of axis-aligned boxes given corner tensors (n, d)
    (spatial.py:172-186).  Returns (lo, hi, cls) CUDA tensors."""
    torch = dv._torch()
    pcode, n_keep = policy_code(policy)
    lo_t = box_lo.to(torch.float64).contiguous()
    hi_t = box_hi.to(device=lo_t.device, dtype=torch.float64).contiguous()
    n = lo_t.shape[0]
    lo = torch.empty(n, dtype=torch.float64, device=lo_t.device)
    hi = torch.empty(n, dtype=torch.float64, device=lo_t.device)
    cls = torch.empty(n, dtype=torch.int8, device=lo_t.device)
    if n:
        dn = device_net(net, lo_t.device.index)
        _lib.call("spk_bound_aabb", dn.ptr, pcode, n_keep, _precision_code(precision), n,
                  lo_t.data_ptr(), hi_t.data_ptr(), lo.data_ptr(), hi.data_ptr(), cls.data_ptr(),
                  dv.stream_ptr(lo_t.device))
    return lo, hi, cls


def bound_random_cubes(net, n, seed=0, half=1.0 / 64.0, first_index=0, policy=AFFINE_FIXED,
                       precision: str = "fp32", device=None, out=None, stream=None):
    """C5 sweep: n cubes with centres U(-1,1)^3 generated on the device from
    (seed, index) and the given half-extent.  Returns (lo, hi, cls) tensors."""
    torch = dv._torch()
    pcode, n_keep = policy_code(policy)
    dev = torch.cuda.current_device() if device is None else device
    if out is None:
        out = (torch.empty(n, dtype=torch.float64, device=f"cuda:{dev}"),
               torch.empty(n, dtype=torch.float64, device=f"cuda:{dev}"),
               torch.empty(n, dtype=torch.int8, device=f"cuda:{dev}"))
    lo, hi, cls = out
    dn = device_net(net, dev)
    s = dv.stream_ptr(dev) if stream is None else stream
    _lib.call("spk_bound_random_cubes", dn.ptr, pcode, n_keep, _precision_code(precision), n,
              first_index, C.c_uint64(seed), half, lo.data_ptr(), hi.data_ptr(), cls.data_ptr(), s)
    return lo, hi, cls


def _stack_axes(axes_list, d):
    s = max((np.asarray(a).shape[0] for a in axes_list), default=0)
    out = np.zeros((len(axes_list), s, d))
    for i, a in enumerate(axes_list):
        a = np.asarray(a, dtype=np.float64)
        if a.size:
            out[i, : a.shape[0], :] = a
    return out


def _check_box(net, box: QueryBox):
    if box.dim != net.input_dim:
        raise DimensionMismatch(f"box lives in R^{box.dim}, network expects R^{net.input_dim}")


def range_bound(net, box: QueryBox, policy, precision: str = "fp32"):
    """Single-box bound + sign class (range_core.py:487-501)."""
    _check_box(net, box)
    lo, hi = range_bound_batch(net, box.center[None, :], _stack_axes([box.axes], net.input_dim), policy,
                               precision)
    lo_f, hi_f = float(lo[0]), float(hi[0])
    return Interval(lo_f, hi_f), classify(lo_f, hi_f)


def interval_forward(net, box: QueryBox, precision: str = "fp32") -> Interval:
    _check_box(net, box)
    lo, hi = interval_forward_batch(net, box.center[None, :], _stack_axes([box.axes], net.input_dim), precision)
    return Interval(float(lo[0]), float(hi[0]))


# ---------------------------------------------------------------------------
# Single-form operations (range_core.py:61-110, 369-464): the definitional
# semantics the batched kernels are tested against.  Bookkeeping on one small
# form; the activation rules come from the device (spk_affine_rule), the
# same rule code the kernels run.

_OP_CODE = {"relu": _lib.OP_RELU, "elu": _lib.OP_ELU, "sin": _lib.OP_SIN, "tanh": _lib.OP_TANH,
            "identity": _lib.OP_IDENTITY}


@dataclass(frozen=True)
class AffineForm:
    """Vector affine form x_k = base_k + sum_j coeffs_kj eps_j + [-err_k, err_k]."""

    base: np.ndarray
    coeffs: np.ndarray
    err: np.ndarray

    def __post_init__(self):
        base = np.asarray(self.base, dtype=np.float64)
        coeffs = np.asarray(self.coeffs, dtype=np.float64)
        err = np.asarray(self.err, dtype=np.float64)
        if base.ndim != 1:
            raise DimensionMismatch("base must be 1-d")
        m = base.shape[0]
        if coeffs.ndim != 2 or coeffs.shape[0] != m:
            raise DimensionMismatch(f"coeffs must have shape ({m}, n)")
        if err.shape != (m,):
            raise DimensionMismatch(f"err must have shape ({m},)")
        if np.any(err < 0.0):
            raise InvalidParameter("err must be non-negative")
        object.__setattr__(self, "base", base)
        object.__setattr__(self, "coeffs", coeffs)
        object.__setattr__(self, "err", err)

    @property
    def dim(self) -> int:
        return self.base.shape[0]

    @property
    def n_symbols(self) -> int:
        return self.coeffs.shape[1]


def interval_of(a: AffineForm) -> Interval:
    """Per-component [base - r, base + r], r = sum |coeffs| + err."""
    r = np.abs(a.coeffs).sum(axis=1) + a.err
    return Interval(a.base - r, a.base + r)


def box_to_affine(box: QueryBox) -> AffineForm:
    """One noise symbol per box axis."""
    return AffineForm(base=box.center.copy(), coeffs=box.axes.T.copy(), err=np.zeros(box.dim))


def affine_linear(a: AffineForm, layer) -> AffineForm:
    """Through a dense layer: exact, no new uncertainty."""
    w = np.asarray(layer.weights, dtype=np.float64)
    if w.shape[1] != a.dim:
        raise DimensionMismatch(f"layer expects {w.shape[1]} inputs, form has {a.dim}")
    return AffineForm(base=w @ a.base + np.asarray(layer.bias, dtype=np.float64), coeffs=w @ a.coeffs,
                      err=np.abs(w) @ a.err)


def affine_rule(kind, lo, hi, precision: str = "fp64"):
    """(alpha, beta, gamma) of an activation over per-neuron bounds, from the
    device rule code (spk_affine_rule)."""
    from .errors import UnsupportedActivation

    name = getattr(kind, "value", kind)
    if name not in _OP_CODE:
        raise UnsupportedActivation(f"no affine rule for {kind!r}")
    lo = np.ascontiguousarray(lo, dtype=np.float64)
    hi = np.ascontiguousarray(hi, dtype=np.float64)
    out = [np.empty(lo.shape) for _ in range(3)]
    _lib.call("spk_affine_rule", _OP_CODE[name], _precision_code(precision), lo.size, lo.ctypes.data, hi.ctypes.data,
              *[o.ctypes.data for o in out])
    return tuple(out)


def affine_nonlinear(a: AffineForm, kind, policy: CondensationPolicy) -> AffineForm:
    """Through an elementwise activation under a policy: rule from the current
    bounds, base/coefficients scaled by alpha, gamma folded into err (fixed)
    or appended as a diagonal block of new symbols (full / truncate)."""
    if policy.kind is PolicyKind.INTERVAL:
        raise InvalidParameter("affine_nonlinear needs an affine policy")
    b = interval_of(a)
    alpha, beta, gamma = affine_rule(kind, b.lo, b.hi)
    base = alpha * a.base + beta
    coeffs = alpha[:, None] * a.coeffs
    err = np.abs(alpha) * a.err
    if policy.kind is PolicyKind.AFFINE_FIXED:
        err = err + gamma
    else:
        coeffs = np.concatenate([coeffs, np.diag(gamma)], axis=1)
    out = AffineForm(base, coeffs, err)
    if policy.kind is PolicyKind.AFFINE_TRUNCATE and out.n_symbols > policy.n_keep:
        out = truncate(out, policy.n_keep)
    return out


def condense(a: AffineForm, indices) -> AffineForm:
    """Fold the named symbol columns into err (interval_of unchanged)."""
    from .errors import IndexOutOfRange

    idx = np.array(sorted({int(i) for i in indices}), dtype=np.intp)
    if idx.size == 0:
        return a
    if idx[0] < 0 or idx[-1] >= a.n_symbols:
        raise IndexOutOfRange(f"column index out of range 0..{a.n_symbols - 1}")
    keep = np.ones(a.n_symbols, dtype=bool)
    keep[idx] = False
    return AffineForm(a.base.copy(), a.coeffs[:, keep], a.err + np.abs(a.coeffs[:, idx]).sum(axis=1))


def truncate(a: AffineForm, n_keep: int) -> AffineForm:
    """Keep the n_keep symbols of largest L1 norm (ties to the lower index,
    kept order preserved); condense the rest."""
    if n_keep < 1:
        raise InvalidParameter("n_keep must be >= 1")
    if a.n_symbols <= n_keep:
        return a
    order = np.argsort(-np.abs(a.coeffs).sum(axis=0), kind="stable")
    return condense(a, order[n_keep:])
