"""Volumetric queries on the range kernels (reference spatial.py:292-720).

Same names, arguments, return types and exceptions as the reference.  The
network work runs in the C-ABI:

* `certified_radii` (spk_certified_radii) -- batched empty-cube halving, the
  inner query of `empty_box_radius` and `walk_on_spheres`;
* `sample_near_surface` / `bulk_properties` -- the K5 tree build
  (spk_tree_build_band: the band rule for sampling, the sign rule for mass
  properties) plus device point evaluation of the sample points;
* `test_intersection` (spk_intersect) -- two-network breadth-first search;
* `closest_point` -- the reference's best-first search (serial decisions)
  with speculative batched node evaluation on the device: bound,
  face-centre values and surface bisection (spk_bisect) of up to `batch`
  heap-front nodes per round trip.

Random streams (walk directions, sample positions) are drawn on the host
with numpy's Generator exactly as the reference draws them, so with FP64
kernels the results equal the reference's wherever the certification
decisions agree.  `precision` defaults to "fp64" here for that reason.
"""

from __future__ import annotations

import ctypes as C
import heapq
from dataclasses import dataclass

import numpy as np

from . import _lib
from . import device as dv
from .errors import DepthOverflow, EmptyBand, InvalidParameter, NoSurfaceFound, OnSurface
from .network import _precision_code, device_net, eval_batch, eval_scalar
from .range_core import AFFINE_FIXED, AFFINE_FULL, policy_code, range_bound_batch
from .spatial import _MAX_DEPTH, AABB, TriangleMesh, _build, _check_domain


@dataclass(frozen=True)
class BulkProperties:
    mass: float
    centroid: np.ndarray
    inertia: np.ndarray  # 3x3 about the centroid, uniform unit density
    mass_error_bound: float


@dataclass(frozen=True)
class EmptyRegion:
    radius: float
    certified: bool


@dataclass(frozen=True)
class IntersectionResult:
    kind: str  # "intersecting" | "disjoint" | "inconclusive"
    witness: AABB | None = None
    nodes: tuple = ()


# ---------------------------------------------------------------- empty cubes

def certified_radii(net, points, r_start, floor: float, policy=AFFINE_FULL, precision: str = "fp64"):
    """For every point the largest r = r_start / 2^j >= floor whose cube of
    half-extent r centred there is certified sign-definite, else 0
    (_certified_radii, spatial.py:318-343).  NumPy in, NumPy out."""
    torch = dv._torch()
    pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, net.input_dim)
    r0 = np.array(np.broadcast_to(np.asarray(r_start, dtype=np.float64), (len(pts),)))
    dn = device_net(net)
    dev = f"cuda:{dn.device}"
    out = torch.empty(len(pts), dtype=torch.float64, device=dev)
    if len(pts):
        pcode, n_keep = policy_code(policy)
        p_d = torch.from_numpy(pts).to(dev)
        r_d = torch.from_numpy(r0).to(dev)
        stats = np.zeros(2, np.int64)
        _lib.call("spk_certified_radii", dn.ptr, pcode, n_keep, _precision_code(precision), len(pts), p_d.data_ptr(),
                  r_d.data_ptr(), float(floor), out.data_ptr(), stats.ctypes.data, dv.stream_ptr(dn.device))
    return out.cpu().numpy()


def empty_box_radius(net, p, r_init: float, policy=AFFINE_FULL, delta: float = 0.001,
                     precision: str = "fp64") -> EmptyRegion:
    """Largest certified-empty cube half-extent at p by halving from r_init
    down to delta (spatial.py:292-315); 0 / not certified if none."""
    point = np.asarray(p, dtype=np.float64)
    if r_init <= 0.0:
        raise InvalidParameter("r_init must be positive")
    if eval_scalar(net, point) == 0.0:
        raise OnSurface(f"f{tuple(point)} = 0")
    r = float(certified_radii(net, point[None, :], [float(r_init)], delta, policy, precision)[0])
    return EmptyRegion(r, True) if r > 0.0 else EmptyRegion(0.0, False)


def walk_on_spheres_stats(net, p, boundary_fn, n_walks: int, rng_seed: int = 0, delta: float = 0.001,
                          policy=AFFINE_FULL, r_cap: float = 1.0, max_rounds: int = 10_000,
                          precision: str = "fp64") -> tuple:
    """Walk-on-spheres estimate of the harmonic extension of boundary_fn at
    p, with its standard error (spatial.py:346-399).  Every round the live
    walks' clearances come from one batched certified_radii call."""
    start = np.asarray(p, dtype=np.float64)
    if eval_scalar(net, start) == 0.0:
        raise OnSurface(f"f{tuple(start)} = 0")
    if n_walks < 1:
        raise InvalidParameter("n_walks must be >= 1")
    rng = np.random.default_rng(rng_seed)
    d = start.shape[0]
    pos = np.repeat(start[None, :], n_walks, axis=0)
    guess = np.full(n_walks, float(r_cap))
    values = np.empty(n_walks)
    live = np.arange(n_walks)
    for _ in range(max_rounds):
        if live.size == 0:
            break
        radii = certified_radii(net, pos[live], guess[live], 2.0 * delta, policy, precision)
        done = radii == 0.0
        for w in live[done]:
            values[w] = float(boundary_fn(pos[w]))
        live, r = live[~done], radii[~done]
        if live.size == 0:
            break
        step = rng.standard_normal((live.size, d))
        step /= np.linalg.norm(step, axis=1, keepdims=True)
        pos[live] += r[:, None] * step
        guess[live] = np.minimum(r * 4.0, r_cap)
    else:
        raise InvalidParameter("walks failed to terminate; delta too small?")
    mean = float(values.mean())
    stderr = float(values.std(ddof=1) / np.sqrt(n_walks)) if n_walks > 1 else 0.0
    return mean, stderr


def walk_on_spheres(net, p, boundary_fn, n_walks: int, rng_seed: int = 0, delta: float = 0.001,
                    policy=AFFINE_FULL, precision: str = "fp64") -> float:
    return walk_on_spheres_stats(net, p, boundary_fn, n_walks, rng_seed, delta, policy, precision=precision)[0]


# ------------------------------------------------------------ tree-based queries

def _levels(net, bounds, depth, policy, precision, band=0.0):
    return _build(net, bounds.lo[None, :], bounds.hi[None, :], 0, 0.001, policy, depth, precision, True,
                  band=band).levels


def sample_near_surface(net, bounds: AABB, n_samples: int, band: float, depth: int, policy=AFFINE_FULL,
                        rng_seed: int = 0, max_evals: int | None = None, precision: str = "fp64") -> np.ndarray:
    """n_samples points with |f| < band by rejection sampling inside the
    depth-`depth` nodes whose bound meets [-band, band] (spatial.py:402-451).
    The band tree is one device build; candidates are evaluated on the
    device in chunks."""
    _check_domain(net, bounds)
    if band <= 0.0 or depth < 1:
        raise InvalidParameter("band must be positive and depth >= 1")
    if depth > _MAX_DEPTH:
        raise DepthOverflow(f"depth {depth} exceeds {_MAX_DEPTH}")
    levels = _levels(net, bounds, depth, policy, precision, band=band)
    if len(levels) < depth + 1:
        raise EmptyBand("no node intersects the band")
    last = levels[depth]
    keep = (last.bound_lo <= band) & (last.bound_hi >= -band)
    if not np.any(keep):
        raise EmptyBand("no node intersects the band")
    los, his = last.lo[keep], last.hi[keep]
    rng = np.random.default_rng(rng_seed)
    vol = np.prod(his - los, axis=1)
    weights = vol / vol.sum()
    budget = max_evals if max_evals is not None else max(200 * n_samples, 100_000)
    chunk = max(1024, n_samples)
    found, n_found, spent = [], 0, 0
    while n_found < n_samples:
        if spent >= budget:
            raise EmptyBand(f"sample budget {budget} exhausted at {n_found} samples")
        k = int(min(chunk, budget - spent))
        pick = rng.choice(len(weights), size=k, p=weights)
        cand = rng.uniform(los[pick], his[pick])
        spent += k
        hit = np.abs(eval_batch(net, cand, precision=precision)) < band
        found.append(cand[hit])
        n_found += int(hit.sum())
    return np.concatenate(found)[:n_samples]


def bulk_properties(net, bounds: AABB, depth: int, samples_per_unknown_node: int = 64, rng_seed: int = 0,
                    policy=AFFINE_FULL, precision: str = "fp64") -> BulkProperties:
    """Mass, centroid and inertia of {f < 0} at unit density
    (spatial.py:454-541): NEGATIVE nodes of every level contribute exact box
    moments, UNKNOWN nodes of the last level stratified samples; the mass
    error bound is their total volume."""
    _check_domain(net, bounds)
    if depth < 1:
        raise InvalidParameter("depth must be >= 1")
    if depth > _MAX_DEPTH:
        raise DepthOverflow(f"depth {depth} exceeds {_MAX_DEPTH}")
    levels = _levels(net, bounds, depth, policy, precision)
    inside = [(lv.lo[lv.label == -1], lv.hi[lv.label == -1]) for lv in levels]
    in_lo = np.concatenate([a for a, _ in inside]) if inside else np.zeros((0, 3))
    in_hi = np.concatenate([b for _, b in inside]) if inside else np.zeros((0, 3))
    if len(levels) == depth + 1:
        u = levels[depth].label == 0
        un_lo, un_hi = levels[depth].lo[u], levels[depth].hi[u]
    else:
        un_lo = un_hi = np.zeros((0, 3))

    mass, first, second = 0.0, np.zeros(3), np.zeros((3, 3))
    if len(in_lo):
        ext = in_hi - in_lo
        vol = np.prod(ext, axis=1)
        c = (in_lo + in_hi) / 2.0
        h = ext / 2.0
        mass += float(vol.sum())
        first += vol @ c
        second += np.einsum("n,ni,nj->ij", vol, c, c)
        second += np.diag(np.einsum("n,ni->i", vol, h * h) / 3.0)
    err = float(np.prod(un_hi - un_lo, axis=1).sum()) if len(un_lo) else 0.0
    if len(un_lo):
        k = max(1, round(samples_per_unknown_node ** (1.0 / 3.0)))
        rng = np.random.default_rng(rng_seed)
        cells = np.stack(np.meshgrid(*[np.arange(k)] * 3, indexing="ij"), axis=-1).reshape(-1, 3)
        ext = un_hi - un_lo
        vol = np.prod(ext, axis=1)
        step = ext / k
        jitter = rng.random((len(un_lo), k ** 3, 3))
        pts = un_lo[:, None, :] + (cells[None, :, :] + jitter) * step[:, None, :]
        inside_pt = (eval_batch(net, pts.reshape(-1, 3), precision=precision) < 0.0).reshape(len(un_lo), k ** 3)
        w = vol / (k ** 3)
        mass += float((w * inside_pt.sum(axis=1)).sum())
        masked = pts * inside_pt[:, :, None]
        first += np.einsum("n,nsi->i", w, masked)
        second += np.einsum("n,nsi,nsj->ij", w, masked, pts)
    centroid = first / mass if mass > 0.0 else bounds.center
    s_c = second - mass * np.outer(centroid, centroid)
    inertia = np.trace(s_c) * np.eye(3) - s_c
    return BulkProperties(mass, centroid, (inertia + inertia.T) / 2.0, err)


def test_intersection(net_a, net_b, bounds: AABB, delta: float = 0.001, policy=AFFINE_FULL,
                      precision: str = "fp64") -> IntersectionResult:
    """Do the solids {f_a < 0} and {f_b < 0} overlap inside bounds?
    (spatial.py:544-588): simultaneous subdivision on the device."""
    _check_domain(net_a, bounds)
    _check_domain(net_b, bounds)
    pcode, n_keep = policy_code(policy)
    da, db = device_net(net_a), device_net(net_b)
    d = bounds.dim
    lo = np.ascontiguousarray(bounds.lo)
    hi = np.ascontiguousarray(bounds.hi)
    kind, n_nodes = C.c_int(), C.c_int64()
    wlo, whi = np.zeros(d), np.zeros(d)
    stats = np.zeros(2, np.int64)
    args = [da.ptr, db.ptr, pcode, n_keep, _precision_code(precision), lo.ctypes.data, hi.ctypes.data, float(delta),
            C.byref(kind), wlo.ctypes.data, whi.ctypes.data, C.byref(n_nodes)]
    cap = 4096
    nlo, nhi = np.zeros((cap, d)), np.zeros((cap, d))
    _lib.call("spk_intersect", *args, nlo.ctypes.data, nhi.ctypes.data, cap, stats.ctypes.data,
              dv.stream_ptr(da.device))
    if kind.value == 1:
        return IntersectionResult("intersecting", witness=AABB(wlo, whi))
    if kind.value == 2:
        if n_nodes.value > cap:  # rerun with room for every inconclusive node
            cap = int(n_nodes.value)
            nlo, nhi = np.zeros((cap, d)), np.zeros((cap, d))
            _lib.call("spk_intersect", *args, nlo.ctypes.data, nhi.ctypes.data, cap, stats.ctypes.data,
                      dv.stream_ptr(da.device))
        m = int(n_nodes.value)
        return IntersectionResult("inconclusive", nodes=tuple(AABB(nlo[i], nhi[i]) for i in range(m)))
    return IntersectionResult("disjoint")


test_intersection.__test__ = False  # API name, not a pytest case


def _bisect_surface(net, p_neg, p_pos, iters, precision):
    """Batched bisection on the device (spk_bisect): (n, d) pairs -> (n, d)."""
    torch = dv._torch()
    dn = device_net(net)
    dev = f"cuda:{dn.device}"
    a = torch.from_numpy(np.ascontiguousarray(p_neg, dtype=np.float64)).to(dev)
    b = torch.from_numpy(np.ascontiguousarray(p_pos, dtype=np.float64)).to(dev)
    out = torch.empty_like(a)
    _lib.call("spk_bisect", dn.ptr, _precision_code(precision), a.shape[0], a.data_ptr(), b.data_ptr(), int(iters),
              out.data_ptr(), dv.stream_ptr(dn.device))
    return out.cpu().numpy()


def _node_batch(net, boxes, policy, precision):
    """Everything closest_point needs about a batch of nodes, on the device
    in three launches: bound, face-centre values, surface bisection of the
    spanning ones.  Returns per node (definite, faces, vals, surface|None)."""
    torch = dv._torch()
    dn = device_net(net)
    dev = f"cuda:{dn.device}"
    los = np.array([b.lo for b in boxes])
    his = np.array([b.hi for b in boxes])
    n, d = los.shape
    centres = (los + his) / 2.0
    axes = np.zeros((n, d, d))
    axes[:, np.arange(d), np.arange(d)] = (his - los) / 2.0
    lo, hi = range_bound_batch(net, torch.from_numpy(centres).to(dev), torch.from_numpy(axes).to(dev), policy,
                               precision=precision)
    lo, hi = lo.cpu().numpy(), hi.cpu().numpy()
    faces = np.stack([b.face_centers() for b in boxes])
    vals = eval_batch(net, faces.reshape(-1, d), precision=precision).reshape(n, 2 * d)
    neg = vals < 0.0
    span = neg.any(axis=1) & ~neg.all(axis=1) & ~((lo > 0.0) | (hi < 0.0))
    surf = [None] * n
    idx = np.flatnonzero(span)
    if idx.size:
        rows = np.arange(idx.size)
        pn = faces[idx][rows, np.argmin(vals[idx], axis=1)]
        pp = faces[idx][rows, np.argmax(vals[idx], axis=1)]
        for k, s_pt in zip(idx, _bisect_surface(net, pn, pp, 30, precision)):
            surf[k] = s_pt
    return [((lo[k] > 0.0) | (hi[k] < 0.0), faces[k], vals[k], surf[k]) for k in range(n)]


def closest_point(net, q, bounds: AABB, delta: float = 0.001, policy=AFFINE_FIXED, precision: str = "fp64",
                  batch: int = 128):
    """Nearest level-set point by lazy best-first descent (spatial.py:591-684):
    nodes in order of their distance to q; a node whose face centres carry
    both signs spans the surface and bounds the answer by its farthest
    corner (reported) and by a bisected surface point (pruning only).

    The visiting order and every decision are the reference's; only the
    evaluation is speculative: when an unevaluated node is popped, it is
    evaluated on the device together with the next `batch - 1` cheapest
    live heap entries (results the serial walk never asks for are dropped),
    so a query costs a few dozen device round trips instead of three per
    node."""
    _check_domain(net, bounds)
    point = np.asarray(q, dtype=np.float64)
    if not np.all(np.isfinite(point)):
        raise InvalidParameter("query point must be finite")
    stop = delta / np.sqrt(bounds.dim)

    def near(box):
        return float(np.linalg.norm(np.maximum(np.maximum(box.lo - point, point - box.hi), 0.0)))

    def far(box):
        return float(np.linalg.norm(np.maximum(np.abs(point - box.lo), np.abs(point - box.hi))))

    best, prune, best_point, tie = np.inf, np.inf, None, 0
    heap = [(near(bounds), tie, bounds)]
    known = {}
    while heap:
        md, t, box = heapq.heappop(heap)
        if md >= min(best, prune):
            continue
        if t not in known:
            cut = min(best, prune)
            ahead = [e for e in heapq.nsmallest(batch - 1, heap) if e[0] < cut and e[1] not in known]
            group = [(t, box)] + [(e[1], e[2]) for e in ahead]
            for (gt, _), res in zip(group, _node_batch(net, [g for _, g in group], policy, precision)):
                known[gt] = res
        definite, faces, vals, surf = known.pop(t)
        if definite:
            continue
        neg = vals < 0.0
        if neg.any() and not neg.all():
            fd = far(box)
            if fd < best:
                best, best_point = fd, box.center
            prune = min(prune, float(np.linalg.norm(surf - point)) + 1e-6)
        elif np.any(vals == 0.0):
            witness = faces[np.argmin(np.abs(vals))]
            prune = min(prune, float(np.linalg.norm(witness - point)) + 1e-6)
        if np.max(box.extents) < stop:
            continue
        for child in box.split():
            cmd = near(child)
            if cmd < min(best, prune):
                tie += 1
                heapq.heappush(heap, (cmd, tie, child))
    if best_point is None:
        raise NoSurfaceFound("no level set found inside bounds")
    return best_point, best


# ---------------------------------------------------------------------- exports

def save_obj(mesh: TriangleMesh, path) -> None:
    """Wavefront OBJ, 1-based faces (spatial.py:690-696)."""
    lines = [f"v {x:.17g} {y:.17g} {z:.17g}\n" for x, y, z in np.asarray(mesh.vertices)]
    lines += [f"f {a + 1} {b + 1} {c + 1}\n" for a, b, c in np.asarray(mesh.triangles)]
    with open(path, "w", encoding="utf-8") as f:
        f.writelines(lines)


def save_xyz(points, path) -> None:
    """One 'x y z' line per point (spatial.py:699-703)."""
    with open(path, "w", encoding="utf-8") as f:
        f.writelines(f"{x:.17g} {y:.17g} {z:.17g}\n" for x, y, z in np.asarray(points).reshape(-1, 3))
