"""CPU oracle for the range-analysis hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy (FP64) restatement of the reference algorithms in
`/root/reference/pkg/src/spelunk` (arXiv 2202.02444, "Spelunking the Deep").
It exists so that the CUDA path can be checked on the GPU box, where the
reference itself is absent.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import it, and only
as the checker or the timed CPU baseline -- never as a product code path.

Parity status: PINNED.  `tests/golden/make_golden.py` runs the unmodified
reference in the build container and commits its outputs under
`tests/golden/`; `tests/test_oracle_golden.py` checks this module against
every vector (bounds to 1e-12, point values bit-exact, tree labels / ray hits
/ mesh triangle sets exactly).

Layout differs from the reference on purpose: affine state is kept per box as
base (b, m), coef (b, m, n_sym), err (b, m) rather than the reference's
(n_sym, b, m) ping-pong slabs, so sums run in a different order and results
agree to the last few ulps, which the reference itself allows
(range_core.py:552-553).
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass

import numpy as np

TWO_PI = 2.0 * np.pi
ACTIVATIONS = ("relu", "elu", "sin", "tanh", "identity")


# ---------------------------------------------------------------------------
# Network  (network.py:29-116 types, :236-313 schema, :143-183 evaluation)


@dataclass
class OracleNet:
    """Flat op list: ("dense", W (out,in), b) or ("act", kind)."""

    input_dim: int
    ops: list

    @property
    def widths(self):
        out = [self.input_dim]
        for op in self.ops:
            if op[0] == "dense":
                out.append(op[1].shape[0])
        return out


def net_from_json_doc(doc: dict) -> OracleNet:
    """Weight-file schema of network.py:236-287 (validation is the package's job)."""
    ops = []
    for entry in doc["layers"]:
        if entry["type"] == "dense":
            ops.append(
                (
                    "dense",
                    np.asarray(entry["weights"], dtype=np.float64),
                    np.asarray(entry["bias"], dtype=np.float64),
                )
            )
        else:
            ops.append(("act", str(entry["kind"])))
    return OracleNet(int(doc["input_dim"]), ops)


def load_net(path) -> OracleNet:
    with open(path, "r", encoding="utf-8") as f:
        return net_from_json_doc(json.load(f))


def as_oracle_net(net) -> OracleNet:
    """Accept an OracleNet, a weight-file path/dict, or any NetworkSpec-like
    object whose .layers hold objects with .weights/.bias or enum activations."""
    if isinstance(net, OracleNet):
        return net
    if isinstance(net, dict):
        return net_from_json_doc(net)
    if isinstance(net, (str, bytes)) or hasattr(net, "__fspath__"):
        return load_net(net)
    ops = []
    for layer in net.layers:
        if hasattr(layer, "weights"):
            ops.append(
                (
                    "dense",
                    np.asarray(layer.weights, dtype=np.float64),
                    np.asarray(layer.bias, dtype=np.float64),
                )
            )
        else:
            ops.append(("act", str(getattr(layer, "value", layer))))
    return OracleNet(int(net.input_dim), ops)


def _act_value(x, kind):
    """Pointwise activations (network.py:149-160)."""
    if kind == "relu":
        return np.maximum(x, 0.0)
    if kind == "elu":
        return np.where(x >= 0.0, x, np.expm1(np.minimum(x, 0.0)))
    if kind == "sin":
        return np.sin(x)
    if kind == "tanh":
        return np.tanh(x)
    if kind == "identity":
        return x
    raise ValueError(kind)


def eval_points(net, xs) -> np.ndarray:
    """Deterministic FP64 point evaluation (network.py:163-183).

    Uses the same fixed-order einsum contraction as the reference so values
    are bit-identical to `eval_batch` (pinned by the golden test).
    """
    net = as_oracle_net(net)
    x = np.asarray(xs, dtype=np.float64)
    if x.size == 0:
        return np.zeros(0)
    for op in net.ops:
        if op[0] == "dense":
            x = np.einsum("nk,mk->nm", x, op[1], optimize=False) + op[2]
        else:
            x = _act_value(x, op[1])
    return x[:, 0]


def eval_points_blas(net, xs) -> np.ndarray:
    """BLAS forward pass (network.py:196-222); last-ulp differences allowed."""
    net = as_oracle_net(net)
    x = np.asarray(xs, dtype=np.float64)
    for op in net.ops:
        if op[0] == "dense":
            x = x @ op[1].T + op[2]
        else:
            x = _act_value(x, op[1])
    return x[:, 0]


# ---------------------------------------------------------------------------
# Linearisation rules (range_core.py:213-349).  Each affine rule returns
# (alpha, beta, gamma) with |h(x) - alpha x - beta| <= gamma on [lo, hi];
# each interval rule returns the exact image of [lo, hi].


def _relu_linear(lo, hi):
    # range_core.py:213-231: Chebyshev secant on straddling lanes
    width = hi - lo
    on = lo >= 0.0
    off = hi <= 0.0
    mixed = ~(on | off)
    slope = hi / np.where(mixed, width, 1.0)
    alpha = np.where(mixed, slope, np.where(on, 1.0, 0.0))
    beta = np.where(mixed, -slope * lo * 0.5, 0.0)
    gamma = beta.copy()
    flat = width == 0.0
    if flat.any():
        a0 = np.where(lo > 0.0, 1.0, 0.0)
        alpha = np.where(flat, a0, alpha)
        beta = np.where(flat, np.maximum(lo, 0.0) - a0 * lo, beta)
        gamma = np.where(flat, 0.0, gamma)
    return alpha, beta, gamma


def _elu_value(x):
    return np.where(x >= 0.0, x, np.expm1(np.minimum(x, 0.0)))


def _elu_linear(lo, hi):
    # range_core.py:238-264: secant slope, tangent point x* = ln(alpha)
    width = hi - lo
    flat = width == 0.0
    on = lo >= 0.0
    f_lo = _elu_value(lo)
    f_hi = _elu_value(hi)
    alpha = np.where(on, 1.0, (f_hi - f_lo) / np.where(flat, 1.0, width))
    under = alpha <= 0.0
    log_arg = np.where(under | on, 1.0, alpha)
    top = f_lo - alpha * lo
    bottom = (alpha - 1.0) - alpha * np.log(log_arg)
    beta = np.where(on, 0.0, (top + bottom) * 0.5)
    gamma = np.where(on, 0.0, (top - bottom) * 0.5)
    if under.any():
        alpha = np.where(under, 0.0, alpha)
        beta = np.where(under, (f_lo + f_hi) * 0.5, beta)
        gamma = np.where(under, (f_hi - f_lo) * 0.5, gamma)
    if flat.any():
        a0 = np.where(lo >= 0.0, 1.0, np.exp(np.minimum(lo, 0.0)))
        alpha = np.where(flat, a0, alpha)
        beta = np.where(flat, f_lo - a0 * lo, beta)
        gamma = np.where(flat, 0.0, gamma)
    return alpha, np.asarray(beta), np.maximum(gamma, 0.0)


def cos_range(lo, hi):
    """Range of cos over [lo, hi] by modular extremum detection (range_core.py:267-274)."""
    c_lo, c_hi = np.cos(lo), np.cos(hi)
    peak = np.floor(hi / TWO_PI) * TWO_PI >= lo
    trough = np.floor((hi - np.pi) / TWO_PI) * TWO_PI + np.pi >= lo
    return (
        np.where(trough, -1.0, np.minimum(c_lo, c_hi)),
        np.where(peak, 1.0, np.maximum(c_lo, c_hi)),
    )


def _sin_linear(lo, hi):
    # range_core.py:277-294: slope = mid of cos range, extremes at the ends
    # or at the first two 2pi-translates of +-arccos(alpha) at/after lo
    c_min, c_max = cos_range(lo, hi)
    alpha = (c_min + c_max) * 0.5
    e = np.arccos(np.clip(alpha, -1.0, 1.0))
    xs = [lo, hi]
    for root in (e, -e):
        first = root + TWO_PI * np.ceil((lo - root) / TWO_PI)
        xs.append(np.clip(first, lo, hi))
        xs.append(np.clip(first + TWO_PI, lo, hi))
    rem = np.stack([np.sin(x) - alpha * x for x in xs])
    top, bottom = rem.max(axis=0), rem.min(axis=0)
    return alpha, (top + bottom) * 0.5, (top - bottom) * 0.5


def _tanh_linear(lo, hi):
    # range_core.py:297-317
    width = hi - lo
    flat = width == 0.0
    f_lo, f_hi = np.tanh(lo), np.tanh(hi)
    alpha = np.where(flat, 1.0 - f_lo * f_lo, (f_hi - f_lo) / np.where(flat, 1.0, width))
    with np.errstate(divide="ignore"):
        x_star = np.arctanh(np.clip(np.sqrt(np.clip(1.0 - alpha, 0.0, 1.0)), 0.0, 1.0))
    xs = [lo, hi, np.clip(x_star, lo, hi), np.clip(-x_star, lo, hi)]
    rem = np.stack([np.tanh(x) - alpha * x for x in xs])
    top, bottom = rem.max(axis=0), rem.min(axis=0)
    beta = (top + bottom) * 0.5
    gamma = (top - bottom) * 0.5
    if flat.any():
        beta = np.where(flat, f_lo - alpha * lo, beta)
        gamma = np.where(flat, 0.0, gamma)
    return alpha, beta, np.maximum(gamma, 0.0)


def _identity_linear(lo, hi):
    return np.ones_like(lo), np.zeros_like(lo), np.zeros_like(lo)


def _sin_image(lo, hi):
    # range_core.py:338-345
    s_lo, s_hi = np.sin(lo), np.sin(hi)
    peak = np.floor((hi - 0.5 * np.pi) / TWO_PI) * TWO_PI + 0.5 * np.pi >= lo
    trough = np.floor((hi + 0.5 * np.pi) / TWO_PI) * TWO_PI - 0.5 * np.pi >= lo
    return (
        np.where(trough, -1.0, np.minimum(s_lo, s_hi)),
        np.where(peak, 1.0, np.maximum(s_lo, s_hi)),
    )


LINEAR_RULES = {
    "relu": _relu_linear,
    "elu": _elu_linear,
    "sin": _sin_linear,
    "tanh": _tanh_linear,
    "identity": _identity_linear,
}

IMAGE_RULES = {
    "relu": lambda lo, hi: (np.maximum(lo, 0.0), np.maximum(hi, 0.0)),
    "elu": lambda lo, hi: (_elu_value(lo), _elu_value(hi)),
    "sin": _sin_image,
    "tanh": lambda lo, hi: (np.tanh(lo), np.tanh(hi)),
    "identity": lambda lo, hi: (lo, hi),
}


# ---------------------------------------------------------------------------
# Policies (range_core.py:104-165)


def parse_policy(policy):
    """Return (kind, n_keep); accepts strings or CondensationPolicy-like objects."""
    if not isinstance(policy, str):
        kind = getattr(policy.kind, "value", policy.kind)
        return str(kind), getattr(policy, "n_keep", None)
    name = policy.strip().lower()
    if name.startswith("affine-truncate"):
        return "affine-truncate", int(name.partition(":")[2])
    if name in ("interval", "affine-fixed", "affine-full"):
        return name, None
    raise ValueError(f"unknown policy {policy!r}")


# ---------------------------------------------------------------------------
# Batched bound evaluation (range_core.py:547-642)


def interval_bounds(net, centers, axes):
    """Centre/radius interval propagation over the axis-aligned hull
    (range_core.py:625-642)."""
    net = as_oracle_net(net)
    c = np.asarray(centers, dtype=np.float64)
    r = np.abs(np.asarray(axes, dtype=np.float64)).sum(axis=1)
    for op in net.ops:
        if op[0] == "dense":
            w = op[1]
            c = c @ w.T + op[2]
            r = r @ np.abs(w.T)
        else:
            lo, hi = IMAGE_RULES[op[1]](c - r, c + r)
            c = (lo + hi) * 0.5
            r = (hi - lo) * 0.5
    return c[:, 0] - r[:, 0], c[:, 0] + r[:, 0]


def affine_bounds(net, centers, axes, policy="affine-fixed"):
    """Affine-arithmetic bound of the network over oriented boxes
    (range_core.py:547-622; Alg. 1 of the paper).

    centers (b, d), axes (b, s, d) with zero rows as padding.  State per box:
    base (b, m), coef (b, m, n_sym), err (b, m) >= 0.
    """
    net = as_oracle_net(net)
    kind, n_keep = parse_policy(policy)
    if kind == "interval":
        return interval_bounds(net, centers, axes)
    base = np.array(centers, dtype=np.float64)
    ax = np.asarray(axes, dtype=np.float64)
    coef = np.ascontiguousarray(np.swapaxes(ax, 1, 2))  # (b, d, s)
    err = np.zeros_like(base)
    for op in net.ops:
        if op[0] == "dense":
            w = op[1]
            base = base @ w.T + op[2]
            coef = np.matmul(w[None, :, :], coef)
            err = err @ np.abs(w.T)
            continue
        if op[1] == "identity":
            continue
        r = np.abs(coef).sum(axis=2) + err
        alpha, beta, gamma = LINEAR_RULES[op[1]](base - r, base + r)
        base = alpha * base + beta
        coef = coef * alpha[:, :, None]
        if kind == "affine-fixed":
            err = np.abs(alpha) * err + gamma
            continue
        err = np.abs(alpha) * err
        b, m = base.shape
        fresh = np.zeros((b, m, m))
        idx = np.arange(m)
        fresh[:, idx, idx] = gamma
        coef = np.concatenate([coef, fresh], axis=2)
        if kind == "affine-truncate" and coef.shape[2] > n_keep:
            coef, err = _truncate_rows(coef, err, n_keep)
    r = np.abs(coef[:, 0, :]).sum(axis=1) + err[:, 0]
    return base[:, 0] - r, base[:, 0] + r


def _truncate_rows(coef, err, n_keep):
    """Per box keep the n_keep symbols of largest L1 norm (ties -> lower
    index, kept symbols stay in order) and fold the rest into err
    (range_core.py:604-619)."""
    mag = np.abs(coef)
    norms = mag.sum(axis=1)  # (b, n)
    order = np.argsort(-norms, axis=1, kind="stable")
    keep = np.sort(order[:, :n_keep], axis=1)
    drop = np.sort(order[:, n_keep:], axis=1)
    folded = np.take_along_axis(mag, drop[:, None, :], axis=2).sum(axis=2)
    kept = np.take_along_axis(coef, keep[:, None, :], axis=2)
    return kept, err + folded


def bound_batch(net, centers, axes, policy="affine-fixed", chunk=None):
    """range_bound_batch equivalent; optional chunking like spatial.py:38."""
    centers = np.asarray(centers, dtype=np.float64)
    axes = np.asarray(axes, dtype=np.float64)
    if chunk is None or len(centers) <= chunk:
        return affine_bounds(net, centers, axes, policy)
    lo = np.empty(len(centers))
    hi = np.empty(len(centers))
    for s in range(0, len(centers), chunk):
        lo[s : s + chunk], hi[s : s + chunk] = affine_bounds(
            net, centers[s : s + chunk], axes[s : s + chunk], policy
        )
    return lo, hi


def sign_labels(lo, hi):
    """+1 POSITIVE (lo > 0), -1 NEGATIVE (hi < 0), 0 UNKNOWN (range_core.py:504-509)."""
    lo = np.asarray(lo)
    hi = np.asarray(hi)
    return np.where(lo > 0.0, 1, np.where(hi < 0.0, -1, 0)).astype(np.int8)


# ---------------------------------------------------------------------------
# k-d tree, breadth first (spatial.py:172-289)


def _cube_axes(lo, hi):
    n, d = lo.shape
    axes = np.zeros((n, d, d))
    i = np.arange(d)
    axes[:, i, i] = (hi - lo) / 2.0
    return axes


def bound_aabbs(net, los, his, policy, chunk=4096):
    """spatial.py:172-186: centres (lo+hi)/2, diagonal half-extent axes."""
    return bound_batch(net, (los + his) / 2.0, _cube_axes(los, his), policy, chunk)


def split_widest(los, his):
    """spatial.py:189-199: halve on the widest axis (ties to the lowest);
    result is [all low halves; all high halves]."""
    n = los.shape[0]
    rows = np.arange(n)
    ax = np.argmax(his - los, axis=1)
    mid = 0.5 * (los[rows, ax] + his[rows, ax])
    low_hi = his.copy()
    low_hi[rows, ax] = mid
    high_lo = los.copy()
    high_lo[rows, ax] = mid
    return np.concatenate([los, high_lo]), np.concatenate([low_hi, his])


def face_centres(los, his):
    """spatial.py:202-211: (n, 2d, d) face-centre points."""
    n, d = los.shape
    c = (los + his) / 2.0
    h = (his - los) / 2.0
    pts = np.repeat(c[:, None, :], 2 * d, axis=1)
    for i in range(d):
        pts[:, 2 * i, i] = c[:, i] - h[:, i]
        pts[:, 2 * i + 1, i] = c[:, i] + h[:, i]
    return pts


def tree_levels(net, lo, hi, policy="affine-fixed", delta=0.001, max_depth=None, start_depth=0):
    """Breadth-first k-d tree (spatial.py:214-289) as flat per-level arrays.

    Level k+1 holds the low children of level k's split nodes (in order) then
    the high children, exactly like the reference's level arrays.  Returns a
    list of dicts: lo, hi (n, d) FP64; label int8 (+1/-1/0); split bool;
    face int8 (+1/-1 annotation on tiny UNKNOWN leaves, 0 = none);
    parent int64 (index into the previous level, -1 for the root).
    """
    net = as_oracle_net(net)
    lo = np.atleast_2d(np.asarray(lo, dtype=np.float64))   # one root, or a frontier slice
    hi = np.atleast_2d(np.asarray(hi, dtype=np.float64))
    if max_depth is not None and max_depth > 60:
        raise ValueError("DepthOverflow")
    d = lo.shape[1]
    stop = delta / np.sqrt(d)
    los, his = lo.copy(), hi.copy()
    parent = np.full(len(los), -1, dtype=np.int64)
    levels = []
    depth = start_depth
    while True:
        blo, bhi = bound_aabbs(net, los, his, policy)
        label = sign_labels(blo, bhi)
        unknown = label == 0
        face = np.zeros(len(los), dtype=np.int8)
        if max_depth is not None:
            split = unknown & (depth < max_depth)
        else:
            small = unknown & (np.max(his - los, axis=1) < stop)
            split = unknown & ~small
            if small.any():
                idx = np.flatnonzero(small)
                vals = eval_points(net, face_centres(los[idx], his[idx]).reshape(-1, d))
                vals = vals.reshape(len(idx), -1)
                neg = np.any(vals < 0.0, axis=1)
                pos = np.any(vals >= 0.0, axis=1)
                face[idx] = np.where(neg & pos, 0, np.where(neg, -1, 1))
        levels.append(
            dict(lo=los, hi=his, label=label, split=split, face=face, parent=parent,
                 bound_lo=blo, bound_hi=bhi)
        )
        if not split.any():
            break
        sidx = np.flatnonzero(split)
        los, his = split_widest(los[split], his[split])
        parent = np.concatenate([sidx, sidx])
        depth += 1
    return levels


def node_keys(levels):
    """Path keys per level: root = 1, low child = 2k, high child = 2k + 1."""
    keys = [np.array([1], dtype=np.int64)]
    for lv in levels[1:]:
        k = len(lv["parent"]) // 2
        pk = keys[-1][lv["parent"]]
        bit = np.concatenate([np.zeros(k, np.int64), np.ones(k, np.int64)])
        keys.append(pk * 2 + bit)
    return keys


# ---------------------------------------------------------------------------
# Volumetric queries (spatial.py:292-684)


def certified_radii(net, points, r_start, floor, policy="affine-full"):
    """_certified_radii (spatial.py:318-343): per point, halve the cube
    half-extent from r_start until the bound is sign-definite (radius) or
    it drops below floor (0)."""
    net = as_oracle_net(net)
    pts = np.asarray(points, dtype=np.float64)
    n, d = pts.shape
    r = np.array(np.broadcast_to(np.asarray(r_start, dtype=np.float64), (n,)))
    radius = np.zeros(n)
    todo = np.flatnonzero(r >= floor)
    while todo.size:
        axes = np.zeros((todo.size, d, d))
        axes[:, np.arange(d), np.arange(d)] = r[todo][:, None]
        blo, bhi = bound_batch(net, pts[todo], axes, policy)
        ok = (blo > 0.0) | (bhi < 0.0)
        radius[todo[ok]] = r[todo[ok]]
        rest = todo[~ok]
        r[rest] /= 2.0
        todo = rest[r[rest] >= floor]
    return radius


def walk_on_spheres_stats(net, p, boundary_fn, n_walks, rng_seed=0, delta=0.001, policy="affine-full",
                          r_cap=1.0, max_rounds=10_000):
    """spatial.py:346-399: each live walk jumps to a uniform point on the
    sphere inscribed in its certified empty cube; it stops (and reads the
    boundary data) when no clearance >= 2 delta certifies."""
    net = as_oracle_net(net)
    x0 = np.asarray(p, dtype=np.float64)
    rng = np.random.default_rng(rng_seed)
    pos = np.tile(x0, (n_walks, 1))
    guess = np.full(n_walks, float(r_cap))
    vals = np.empty(n_walks)
    live = np.arange(n_walks)
    for _ in range(max_rounds):
        if not live.size:
            break
        rad = certified_radii(net, pos[live], guess[live], 2.0 * delta, policy)
        stop = rad == 0.0
        for w in live[stop]:
            vals[w] = float(boundary_fn(pos[w]))
        live, rad = live[~stop], rad[~stop]
        if not live.size:
            break
        u = rng.standard_normal((live.size, x0.shape[0]))
        u /= np.linalg.norm(u, axis=1, keepdims=True)
        pos[live] += rad[:, None] * u
        guess[live] = np.minimum(rad * 4.0, r_cap)
    se = float(vals.std(ddof=1) / np.sqrt(n_walks)) if n_walks > 1 else 0.0
    return float(vals.mean()), se


def sample_near_surface(net, lo, hi, n_samples, band, depth, policy="affine-full", rng_seed=0, max_evals=None):
    """spatial.py:402-451: band tree (split while the bound meets
    [-band, band]) to `depth`, then volume-weighted rejection sampling."""
    net = as_oracle_net(net)
    los = np.atleast_2d(np.asarray(lo, dtype=np.float64))
    his = np.atleast_2d(np.asarray(hi, dtype=np.float64))
    for level in range(depth + 1):
        blo, bhi = bound_aabbs(net, los, his, policy)
        keep = (blo <= band) & (bhi >= -band)
        if not keep.any():
            raise ValueError("EmptyBand")
        if level == depth:
            los, his = los[keep], his[keep]
            break
        los, his = split_widest(los[keep], his[keep])
    rng = np.random.default_rng(rng_seed)
    vol = np.prod(his - los, axis=1)
    w = vol / vol.sum()
    budget = max_evals if max_evals is not None else max(200 * n_samples, 100_000)
    chunk = max(1024, n_samples)
    got, total, spent = [], 0, 0
    while total < n_samples:
        if spent >= budget:
            raise ValueError("EmptyBand")
        k = int(min(chunk, budget - spent))
        pick = rng.choice(len(w), size=k, p=w)
        cand = rng.uniform(los[pick], his[pick])
        spent += k
        ok = np.abs(eval_points(net, cand)) < band
        got.append(cand[ok])
        total += int(ok.sum())
    return np.concatenate(got)[:n_samples]


def bulk_properties(net, lo, hi, depth, samples_per_unknown_node=64, rng_seed=0, policy="affine-full"):
    """spatial.py:454-541 -> (mass, mass_error_bound, centroid, inertia)."""
    net = as_oracle_net(net)
    levels = tree_levels(net, lo, hi, policy, max_depth=depth)
    neg = [(lv["lo"][lv["label"] == -1], lv["hi"][lv["label"] == -1]) for lv in levels]
    ilo = np.concatenate([a for a, _ in neg])
    ihi = np.concatenate([b for _, b in neg])
    if len(levels) == depth + 1:
        u = levels[depth]["label"] == 0
        ulo, uhi = levels[depth]["lo"][u], levels[depth]["hi"][u]
    else:
        ulo = uhi = np.zeros((0, 3))
    mass, m1, m2 = 0.0, np.zeros(3), np.zeros((3, 3))
    if len(ilo):
        ext = ihi - ilo
        vol = np.prod(ext, axis=1)
        c = (ilo + ihi) / 2.0
        mass += float(vol.sum())
        m1 += vol @ c
        m2 += np.einsum("n,ni,nj->ij", vol, c, c)
        m2 += np.diag(np.einsum("n,ni->i", vol, (ext / 2.0) ** 2) / 3.0)
    err = float(np.prod(uhi - ulo, axis=1).sum()) if len(ulo) else 0.0
    if len(ulo):
        k = max(1, round(samples_per_unknown_node ** (1.0 / 3.0)))
        rng = np.random.default_rng(rng_seed)
        sub = np.stack(np.meshgrid(*[np.arange(k)] * 3, indexing="ij"), axis=-1).reshape(-1, 3)
        ext = uhi - ulo
        vol = np.prod(ext, axis=1)
        pts = ulo[:, None, :] + (sub[None] + rng.random((len(ulo), k ** 3, 3))) * (ext / k)[:, None, :]
        ins = (eval_points(net, pts.reshape(-1, 3)) < 0.0).reshape(len(ulo), k ** 3)
        w = vol / (k ** 3)
        mass += float((w * ins.sum(axis=1)).sum())
        m1 += np.einsum("n,nsi->i", w, pts * ins[:, :, None])
        m2 += np.einsum("n,nsi,nsj->ij", w, pts * ins[:, :, None], pts)
    centroid = m1 / mass if mass > 0.0 else (np.asarray(lo, float) + np.asarray(hi, float)) / 2.0
    sc = m2 - mass * np.outer(centroid, centroid)
    inertia = np.trace(sc) * np.eye(3) - sc
    return mass, err, centroid, (inertia + inertia.T) / 2.0


def test_intersection(net_a, net_b, lo, hi, delta=0.001, policy="affine-full"):
    """spatial.py:544-588 -> ("intersecting", witness (lo, hi)) |
    ("disjoint", None) | ("inconclusive", [(lo, hi), ...])."""
    net_a, net_b = as_oracle_net(net_a), as_oracle_net(net_b)
    los = np.atleast_2d(np.asarray(lo, dtype=np.float64))
    his = np.atleast_2d(np.asarray(hi, dtype=np.float64))
    stop = delta / np.sqrt(los.shape[1])
    small = []
    while len(los):
        la, ha = bound_aabbs(net_a, los, his, policy)
        lb, hb = bound_aabbs(net_b, los, his, policy)
        live = (la <= 0.0) & (lb <= 0.0)
        inside = live & (ha < 0.0) & (hb < 0.0)
        if inside.any():
            i = int(np.flatnonzero(inside)[0])
            return "intersecting", (los[i], his[i])
        tiny = live & (np.max(his - los, axis=1) < stop)
        small += [(los[i], his[i]) for i in np.flatnonzero(tiny)]
        go = live & ~tiny
        los, his = split_widest(los[go], his[go])
    return ("inconclusive", small) if small else ("disjoint", None)


test_intersection.__test__ = False


def closest_point(net, q, lo, hi, delta=0.001, policy="affine-fixed"):
    """spatial.py:591-684: best-first descent ordered by the distance of q
    to each node; spanning nodes (face centres of both signs) report their
    centre and farthest-corner distance; a bisected surface point prunes."""
    import heapq

    net = as_oracle_net(net)
    q = np.asarray(q, dtype=np.float64)
    lo = np.asarray(lo, dtype=np.float64)
    hi = np.asarray(hi, dtype=np.float64)
    stop = delta / np.sqrt(lo.shape[0])
    near = lambda a, b: float(np.linalg.norm(np.maximum(np.maximum(a - q, q - b), 0.0)))  # noqa: E731
    far = lambda a, b: float(np.linalg.norm(np.maximum(np.abs(q - a), np.abs(q - b))))  # noqa: E731
    best, prune, best_pt, tie = np.inf, np.inf, None, 0
    heap = [(near(lo, hi), 0, lo, hi)]
    while heap:
        md, _, a, b = heapq.heappop(heap)
        if md >= min(best, prune):
            continue
        blo, bhi = bound_aabbs(net, a[None, :], b[None, :], policy)
        if blo[0] > 0.0 or bhi[0] < 0.0:
            continue
        faces = face_centres(a[None, :], b[None, :])[0]
        v = eval_points(net, faces)
        if np.any(v < 0.0) and not np.all(v < 0.0):
            fd = far(a, b)
            if fd < best:
                best, best_pt = fd, (a + b) / 2.0
            pn, pp = faces[np.argmin(v)], faces[np.argmax(v)]
            for _ in range(30):
                mid = 0.5 * (pn + pp)
                if eval_points(net, mid[None, :])[0] < 0.0:
                    pn = mid
                else:
                    pp = mid
            prune = min(prune, float(np.linalg.norm(0.5 * (pn + pp) - q)) + 1e-6)
        elif np.any(v == 0.0):
            prune = min(prune, float(np.linalg.norm(faces[np.argmin(np.abs(v))] - q)) + 1e-6)
        if np.max(b - a) < stop:
            continue
        kids = split_widest(a[None, :], b[None, :])
        for c_lo, c_hi in zip(*kids):
            cmd = near(c_lo, c_hi)
            if cmd < min(best, prune):
                tie += 1
                heapq.heappush(heap, (cmd, tie, c_lo, c_hi))
    if best_pt is None:
        raise ValueError("NoSurfaceFound")
    return best_pt, best


# ---------------------------------------------------------------------------
# Range-marching ray caster (rays.py:88-138) and pinhole camera (camera.py)


@dataclass(frozen=True)
class MarchParams:
    """rays.py:48-71 defaults."""

    t_max: float = 10.0
    sigma0: float | None = None
    eta_plus: float = 1.5
    eta_minus: float = 0.5
    delta: float = 0.001
    safety: float = 0.98

    @property
    def s0(self):
        return self.t_max / 10.0 if self.sigma0 is None else self.sigma0


def march(net, origins, dirs, params=MarchParams(), policy="affine-fixed",
          t_init=None, sigma_init=None):
    """Lock-step adaptive range-march; returns (hit bool, t FP64, steps)."""
    net = as_oracle_net(net)
    origins = np.asarray(origins, dtype=np.float64)
    dirs = np.asarray(dirs, dtype=np.float64)
    n = len(origins)
    t = np.zeros(n) if t_init is None else np.array(t_init, dtype=np.float64)
    sig = np.full(n, params.s0) if sigma_init is None else np.array(sigma_init, dtype=np.float64)
    steps = np.zeros(n)
    hit = np.zeros(n, dtype=bool)
    t_hit = np.full(n, np.inf)
    if n == 0:
        return hit, t_hit, steps
    f0 = eval_points(net, origins)
    surf = f0 == 0.0
    hit[surf] = True
    t_hit[surf] = 0.0
    inside0 = f0 < 0.0
    live = np.flatnonzero(~surf & (t < params.t_max))
    while live.size:
        p, r, tl = origins[live], dirs[live], t[live]
        probe = eval_points(net, p + (tl + params.delta)[:, None] * r)
        steps[live] += 1.0
        crossed = (probe < 0.0) != inside0[live]
        hit[live[crossed]] = True
        t_hit[live[crossed]] = t[live[crossed]]
        keep = ~crossed
        live = live[keep]
        if live.size == 0:
            break
        p, r, tl = p[keep], r[keep], tl[keep]
        sl = sig[live]
        centre = p + (tl + sl / 2.0)[:, None] * r
        axis = ((sl / 2.0)[:, None] * r)[:, None, :]
        blo, bhi = bound_batch(net, centre, axis, policy)
        ok = (blo > 0.0) | (bhi < 0.0)
        sig[live] = np.where(ok, sl * params.eta_plus, sl * params.eta_minus)
        t[live] = tl + np.maximum(params.safety * np.where(ok, sl, 0.0), params.delta)
        live = live[t[live] < params.t_max]
    return hit, t_hit, steps


def camera_frame(position, look_at, up):
    """camera.py:39-49: (forward, right, true_up)."""
    pos = np.asarray(position, dtype=np.float64)
    fwd = np.asarray(look_at, dtype=np.float64) - pos
    fwd = fwd / np.linalg.norm(fwd)
    right = np.cross(fwd, np.asarray(up, dtype=np.float64))
    right = right / np.linalg.norm(right)
    return fwd, right, np.cross(right, fwd)


def pixel_dirs(position, look_at, up, vertical_fov, width, height):
    """camera.py:68-92: unit directions (height, width, 3), row 0 on top."""
    fwd, right, tup = camera_frame(position, look_at, up)
    half_h = math.tan(math.radians(vertical_fov) / 2.0)
    half_w = half_h * width / height
    u = ((np.arange(width, dtype=np.float64) + 0.5) / width * 2.0 - 1.0) * half_w
    v = (1.0 - (np.arange(height, dtype=np.float64) + 0.5) / height * 2.0) * half_h
    d = fwd[None, None, :] + u[None, :, None] * right[None, None, :] + v[:, None, None] * tup[None, None, :]
    return d / np.linalg.norm(d, axis=2, keepdims=True)


class _PinholeRays:
    """Single-pixel directions and slab boxes (camera.py:85-135)."""

    def __init__(self, position, look_at, up, vertical_fov, width, height):
        self.pos = np.asarray(position, dtype=np.float64)
        self.fwd, self.right, self.tup = camera_frame(position, look_at, up)
        self.hh = math.tan(math.radians(vertical_fov) / 2.0)
        self.hw = self.hh * width / height
        self.w, self.h = width, height

    def u(self, i):
        return ((float(i) + 0.5) / self.w * 2.0 - 1.0) * self.hw

    def v(self, j):
        return (1.0 - (float(j) + 0.5) / self.h * 2.0) * self.hh

    def dir(self, i, j):
        d = self.fwd + self.u(i) * self.right + self.v(j) * self.tup
        return d / np.linalg.norm(d)

    def corners(self, px0, px1, py0, py1):
        return (self.dir(px0, py1 - 1), self.dir(px1 - 1, py1 - 1), self.dir(px0, py0), self.dir(px1 - 1, py0))

    def slab(self, px0, px1, py0, py1, t0, t1):
        """Hull of the 9 candidate unit directions (pixel-centre corners and
        zero-clamped midlines) scaled by t0 and t1, per frame axis."""
        u0, u1 = self.u(px0), self.u(px1 - 1)
        v0, v1 = self.v(py1 - 1), self.v(py0)
        uc = min(max(0.0, u0), u1)
        vc = min(max(0.0, v0), v1)
        ws = []
        for vv in (v0, v1, vc):
            for uu in (u0, u1, uc):
                ell = np.sqrt(1.0 + uu * uu + vv * vv)
                ws.append((1.0 / ell, uu / ell, vv / ell))
        ws = np.array(ws)
        wmin, wmax = ws.min(axis=0), ws.max(axis=0)
        lo = np.minimum(t0 * wmin, t1 * wmin)
        hi = np.maximum(t0 * wmax, t1 * wmax)
        mid, half = (lo + hi) / 2.0, (hi - lo) / 2.0
        centre = self.pos + mid[0] * self.fwd + mid[1] * self.right + mid[2] * self.tup
        axes = [half[k] * vec for k, vec in enumerate((self.fwd, self.right, self.tup)) if half[k] > 0.0]
        return centre, np.array(axes).reshape(-1, 3)


def frustum_cast(net, position, look_at, up, vertical_fov, width, height, params=MarchParams(),
                 policy="affine-fixed", initial_grid=16):
    """Frustum range-march over the pixel grid (rays.py:232-341).

    Rectangles of pixels march together while their front face is narrower
    than 2 sigma; wider ones split across the longer pixel side.  Single
    pixels finish with the per-ray march from their frustum's (t, sigma).
    Returns (hit (H, W) bool, t (H, W), steps (H, W))."""
    net = as_oracle_net(net)
    cam = _PinholeRays(position, look_at, up, vertical_fov, width, height)
    gw, gh = min(initial_grid, width), min(initial_grid, height)
    if width % gw or height % gh:
        raise ValueError("resolution not divisible into the frustum grid")
    hit = np.zeros((height, width), dtype=bool)
    t_img = np.full((height, width), np.inf)
    steps = np.zeros((height, width))
    if eval_points(net, cam.pos[None, :])[0] == 0.0:
        return np.ones_like(hit), np.zeros_like(t_img), steps
    bw, bh = width // gw, height // gh
    # frustum record: [px0, px1, py0, py1, t, sigma, corner dirs]
    live = [[bx * bw, bx * bw + bw, by * bh, by * bh + bh, 0.0, params.s0]
            for by in range(gh) for bx in range(gw)]
    singles = []
    while live:
        todo, live, batch = live, [], []
        while todo:
            f = todo.pop()
            px0, px1, py0, py1, t, sig = f
            nx, ny = px1 - px0, py1 - py0
            if nx * ny == 1:
                singles.append(f)
                continue
            if t >= params.t_max:
                continue
            r00, r10, r01, r11 = cam.corners(px0, px1, py0, py1)
            split_x = (nx >= ny and nx > 1) or ny == 1
            if split_x:
                width_w = t * max(np.linalg.norm(r10 - r00), np.linalg.norm(r11 - r01))
            else:
                width_w = t * max(np.linalg.norm(r01 - r00), np.linalg.norm(r11 - r10))
            if width_w > 2.0 * sig:
                if split_x:
                    m = px0 + nx // 2
                    todo += [[px0, m, py0, py1, t, sig], [m, px1, py0, py1, t, sig]]
                else:
                    m = py0 + ny // 2
                    todo += [[px0, px1, py0, m, t, sig], [px0, px1, m, py1, t, sig]]
                continue
            batch.append(f)
        if not batch:
            break
        slabs = [cam.slab(f[0], f[1], f[2], f[3], f[4], f[4] + f[5]) for f in batch]
        s = max(a.shape[0] for _, a in slabs)
        centres = np.array([c for c, _ in slabs])
        axes = np.zeros((len(batch), s, 3))
        for i, (_, a) in enumerate(slabs):
            axes[i, : a.shape[0]] = a
        blo, bhi = bound_batch(net, centres, axes, policy)
        for f, lo_, hi_ in zip(batch, blo, bhi):
            steps[f[2]:f[3], f[0]:f[1]] += 1.0 / ((f[1] - f[0]) * (f[3] - f[2]))
            if lo_ > 0.0 or hi_ < 0.0:
                f[4] += max(params.safety * f[5], params.delta)
                f[5] *= params.eta_plus
            else:
                f[5] *= params.eta_minus
                if f[5] < params.delta * 2.0 ** -32:
                    # product termination guard (spk_frustum.cu), absent from
                    # the reference; never reached in the golden cases
                    singles += [[x, x + 1, y, y + 1, f[4], f[5]]
                                for y in range(f[2], f[3]) for x in range(f[0], f[1])]
                    continue
            live.append(f)
    if singles:
        dirs = np.array([cam.dir(f[0], f[2]) for f in singles])
        origins = np.broadcast_to(cam.pos, dirs.shape).copy()
        h1, t1, s1 = march(net, origins, dirs, params, policy,
                           t_init=[f[4] for f in singles], sigma_init=[f[5] for f in singles])
        for f, a, b, c in zip(singles, h1, t1, s1):
            hit[f[2], f[0]] = a
            t_img[f[2], f[0]] = b
            steps[f[2], f[0]] += c
    return hit, t_img, steps


# ---------------------------------------------------------------------------
# Rendering post-process (render.py:36-141)

RENDER_BACKGROUND = np.array([24, 28, 38], dtype=np.uint8)
RENDER_LIGHT = np.array([0.35, 0.75, 0.56]) / np.linalg.norm(np.array([0.35, 0.75, 0.56]))


def fixed_step_march(net, origins, dirs, step, t_max):
    """Uniform samples at t = step, 2 step, ... (t a running FP64 sum); the
    first sign change reports a hit at the previous sample."""
    net = as_oracle_net(net)
    f0 = eval_points(net, origins)
    hit = f0 == 0.0
    t_hit = np.where(hit, 0.0, np.inf)
    inside = f0 < 0.0
    todo = np.flatnonzero(~hit)
    t = step
    while todo.size and t < t_max:
        side = eval_points(net, origins[todo] + t * dirs[todo]) < 0.0
        flipped = side != inside[todo]
        hit[todo[flipped]] = True
        t_hit[todo[flipped]] = t - step
        todo = todo[~flipped]
        t += step
    return hit, t_hit


def shade(net, origin, dirs, hit, t, delta, iters=48):
    """Bisection refine of [t, t + delta], central-difference normal
    (h = delta / 10), Lambert gray; background elsewhere.  (n, 3) uint8."""
    net = as_oracle_net(net)
    px = np.tile(RENDER_BACKGROUND, (len(dirs), 1))
    sel = np.flatnonzero(hit)
    if sel.size == 0:
        return px
    o = np.broadcast_to(origin, (sel.size, 3))
    d = dirs[sel]
    neg0 = eval_points(net, np.asarray(origin, dtype=np.float64)[None, :])[0] < 0.0
    lo, hi = t[sel].copy(), t[sel] + delta
    for _ in range(iters):
        mid = 0.5 * (lo + hi)
        cross = (eval_points(net, o + mid[:, None] * d) < 0.0) != neg0
        lo, hi = np.where(cross, lo, mid), np.where(cross, mid, hi)
    p = o + lo[:, None] * d
    h = delta / 10.0
    grad = np.stack([eval_points(net, p + h * e) - eval_points(net, p - h * e) for e in np.eye(3)], axis=1)
    length = np.linalg.norm(grad, axis=1, keepdims=True)
    length[length == 0.0] = 1.0
    lam = np.clip((grad / length) @ RENDER_LIGHT, 0.0, 1.0)
    px[sel] = np.rint(lam * 255.0).astype(np.uint8)[:, None]
    return px


def render(net, position, look_at, up, vertical_fov, width, height, params=MarchParams(),
           policy="affine-fixed", mode="per_ray", step=None):
    """render_image: march (per_ray / frustum / fixed_step) then shade;
    returns the (height, width, 3) uint8 image."""
    net = as_oracle_net(net)
    dirs = pixel_dirs(position, look_at, up, vertical_fov, width, height).reshape(-1, 3)
    pos = np.asarray(position, dtype=np.float64)
    origins = np.broadcast_to(pos, dirs.shape).copy()
    if mode == "per_ray":
        hit, t, _ = march(net, origins, dirs, params, policy)
    elif mode == "frustum":
        hit, t, _ = frustum_cast(net, position, look_at, up, vertical_fov, width, height, params, policy)
        hit, t = hit.reshape(-1), t.reshape(-1)
    else:
        hit, t = fixed_step_march(net, origins, dirs, step, params.t_max)
    return shade(net, pos, dirs, hit, t, params.delta).reshape(height, width, 3)


# ---------------------------------------------------------------------------
# Marching-cubes tables (mc_tables.py:24-105): generated, not the classic table

MC_CORNERS = np.array(
    [[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0], [0, 0, 1], [1, 0, 1], [1, 1, 1], [0, 1, 1]],
    dtype=np.int64,
)
MC_EDGES = ((0, 1), (1, 2), (2, 3), (3, 0), (4, 5), (5, 6), (6, 7), (7, 4),
            (0, 4), (1, 5), (2, 6), (3, 7))
# faces as corner cycles, counter-clockwise seen from outside
MC_FACES = ((0, 3, 2, 1), (4, 5, 6, 7), (0, 1, 5, 4), (3, 7, 6, 2), (0, 4, 7, 3), (1, 2, 6, 5))


def _edge_of(a, b):
    for e, (p, q) in enumerate(MC_EDGES):
        if (p, q) == (a, b) or (q, p) == (a, b):
            return e
    raise KeyError((a, b))


def _face_links(inside, cyc):
    """Directed isoline links (exit edge -> entry edge) on one face; an
    ambiguous face isolates each inside corner (mc_tables.py:54-69)."""
    sgn = [inside[c] for c in cyc]
    side = [_edge_of(cyc[i], cyc[(i + 1) % 4]) for i in range(4)]
    outs = [i for i in range(4) if sgn[i] and not sgn[(i + 1) % 4]]
    ins = [i for i in range(4) if not sgn[i] and sgn[(i + 1) % 4]]
    if not outs:
        return []
    if len(outs) == 1:
        return [(side[outs[0]], side[ins[0]])]
    return [(side[p], side[(p - 1) % 4]) for p in range(4) if sgn[p]]


def _case_triangles(case):
    inside = [bool((case >> i) & 1) for i in range(8)]
    succ = {}
    for cyc in MC_FACES:
        for a, b in _face_links(inside, cyc):
            succ[a] = b
    out = []
    todo = set(succ)
    while todo:
        first = min(todo)
        ring = [first]
        todo.discard(first)
        cur = succ[first]
        while cur != first:
            ring.append(cur)
            todo.discard(cur)
            cur = succ[cur]
        for i in range(1, len(ring) - 1):
            out.append((ring[0], ring[i + 1], ring[i]))  # reversed fan
    return tuple(out)


MC_TRIANGLES = tuple(_case_triangles(c) for c in range(256))


# ---------------------------------------------------------------------------
# Hierarchical marching cubes (meshing.py:23-169)


def grid_axis(lo, hi, n_cells):
    """np.linspace(lo, hi, n+1): i*step + lo, last entry forced to hi."""
    return np.linspace(lo, hi, n_cells + 1)


def edge_key(ia, ib, n_pts):
    """Global grid edge id: (linear index of the lower corner) * 3 + axis."""
    a = np.asarray(ia)
    b = np.asarray(ib)
    low = np.minimum(a, b)
    ax = int(np.flatnonzero(a != b)[0])
    lin = (int(low[0]) * n_pts + int(low[1])) * n_pts + int(low[2])
    return lin * 3 + ax


class _Builder:
    """Edge-keyed vertex dedup (meshing.py:29-66)."""

    def __init__(self, coords):
        self.coords = coords
        self.n_pts = len(coords[0])
        self.ids = {}
        self.verts = []
        self.keys = []
        self.tris = []

    def _vid(self, cell, e, vals):
        a, b = MC_EDGES[e]
        ia = tuple(int(cell[k] + MC_CORNERS[a][k]) for k in range(3))
        ib = tuple(int(cell[k] + MC_CORNERS[b][k]) for k in range(3))
        key = (ia, ib) if ia <= ib else (ib, ia)
        v = self.ids.get(key)
        if v is None:
            fa, fb = vals[a], vals[b]
            t = (0.0 - fa) / (fb - fa)
            pa = np.array([self.coords[k][ia[k]] for k in range(3)])
            pb = np.array([self.coords[k][ib[k]] for k in range(3)])
            v = len(self.verts)
            self.verts.append(pa + t * (pb - pa))
            self.keys.append(edge_key(ia, ib, self.n_pts))
            self.ids[key] = v
        return v

    def cell(self, cell, vals):
        case = sum(1 << c for c in range(8) if vals[c] < 0.0)
        for tri in MC_TRIANGLES[case]:
            self.tris.append(tuple(self._vid(cell, e, vals) for e in tri))

    def result(self):
        if not self.verts:
            return np.zeros((0, 3)), np.zeros((0, 3), np.int64), np.zeros(0, np.int64)
        return np.stack(self.verts), np.array(self.tris, np.int64), np.array(self.keys, np.int64)


def _polygonize(builder, vals, origin):
    neg = vals < 0.0
    nx, ny, nz = (s - 1 for s in vals.shape)
    case = np.zeros((nx, ny, nz), dtype=np.int32)
    for c, (dx, dy, dz) in enumerate(MC_CORNERS):
        case |= neg[dx : dx + nx, dy : dy + ny, dz : dz + nz].astype(np.int32) << c
    for i, j, k in np.argwhere((case != 0) & (case != 255)):
        cv = [vals[i + dx, j + dy, k + dz] for dx, dy, dz in MC_CORNERS]
        builder.cell((origin[0] + i, origin[1] + j, origin[2] + k), cv)


def _grid_values(net, coords, rng):
    (i0, i1), (j0, j1), (k0, k1) = rng
    g = np.stack(
        np.meshgrid(coords[0][i0 : i1 + 1], coords[1][j0 : j1 + 1], coords[2][k0 : k1 + 1],
                    indexing="ij"),
        axis=-1,
    )
    return eval_points(net, g.reshape(-1, 3)).reshape(g.shape[:3])


def mesh_blocks(net, lo, hi, m, dense_levels=3, policy="affine-fixed"):
    """Surviving index-range blocks of the hierarchical prune (meshing.py:134-163)."""
    net = as_oracle_net(net)
    n = 2 ** m
    coords = [grid_axis(lo[k], hi[k], n) for k in range(3)]

    def survivors(blocks):
        if not blocks:
            return []
        b = np.asarray(blocks, dtype=np.int64)  # (nb, 3, 2)
        wlo = np.stack([coords[k][b[:, k, 0]] for k in range(3)], axis=1)
        whi = np.stack([coords[k][b[:, k, 1]] for k in range(3)], axis=1)
        axes = _cube_axes(wlo, whi)
        blo, bhi = bound_batch(net, (wlo + whi) / 2.0, axes, policy)
        return [blk for blk, a, z in zip(blocks, blo, bhi) if a <= 0.0 <= z]

    blocks = [((0, n), (0, n), (0, n))]
    for _ in range(3 * (m - dense_levels)):
        blocks = survivors(blocks)
        nxt = []
        for blk in blocks:
            size = [blk[k][1] - blk[k][0] for k in range(3)]
            ax = int(np.argmax(size))
            cut = blk[ax][0] + size[ax] // 2
            a = list(blk)
            b = list(blk)
            a[ax] = (blk[ax][0], cut)
            b[ax] = (cut, blk[ax][1])
            nxt.extend((tuple(a), tuple(b)))
        blocks = nxt
    return survivors(blocks), coords


def mesh_extract(net, lo, hi, m, dense_levels=3, policy="affine-fixed"):
    """Hierarchical extraction; returns (vertices, triangles, vertex_edge_keys)."""
    net = as_oracle_net(net)
    blocks, coords = mesh_blocks(net, lo, hi, m, dense_levels, policy)
    builder = _Builder(coords)
    for blk in blocks:
        vals = _grid_values(net, coords, blk)
        _polygonize(builder, vals, (blk[0][0], blk[1][0], blk[2][0]))
    return builder.result()


def mesh_extract_dense(net, lo, hi, m):
    """meshing.py:100-108 brute force."""
    net = as_oracle_net(net)
    n = 2 ** m
    coords = [grid_axis(lo[k], hi[k], n) for k in range(3)]
    builder = _Builder(coords)
    _polygonize(builder, _grid_values(net, coords, ((0, n), (0, n), (0, n))), (0, 0, 0))
    return builder.result()


def triangle_key_set(triangles, vertex_keys):
    """Triangles as edge-key triples, rotated so the smallest key leads
    (winding preserved); a multiset-free canonical form for comparisons."""
    out = []
    for t in np.asarray(triangles):
        k = [int(vertex_keys[i]) for i in t]
        r = k.index(min(k))
        out.append(tuple(k[r:] + k[:r]))
    return sorted(out)
