"""k-d bounding trees on the B200 (reference spatial.py:41-289).

`build_spatial_tree` keeps the reference contract (returns a TreeNode tree
whose nodes carry AABB, SignClass, depth, children and face_sign).  The
whole breadth-first build runs in the C-ABI (`spk_tree_build`, K5): fused
bound kernel per level, ballot/prefix-sum compaction of UNKNOWN nodes into
the next frontier, FP64 midpoint splits identical to the reference's.

`build_spatial_tree_arrays` returns the same tree as flat per-level arrays
(no Python objects) -- the throughput API for 10^5..10^7-node trees.
`build_spatial_tree_sharded` splits the frontier across ranks (one process
per GPU) with no collective on the inner loop.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from . import device as dv
from .errors import DepthOverflow, DimensionMismatch, InvalidBounds, InvalidParameter
from .network import _precision_code, device_net
from .range_core import AFFINE_FULL, SignClass, policy_code

_MAX_DEPTH = 60
_SIGN = {1: SignClass.POSITIVE, -1: SignClass.NEGATIVE, 0: SignClass.UNKNOWN}


@dataclass(frozen=True)
class AABB:
    lo: np.ndarray
    hi: np.ndarray

    def __post_init__(self):
        lo = np.asarray(self.lo, dtype=np.float64)
        hi = np.asarray(self.hi, dtype=np.float64)
        if lo.shape != hi.shape or lo.ndim != 1:
            raise InvalidBounds("corners must be 1-d points of equal dimension")
        if not (np.all(np.isfinite(lo)) and np.all(np.isfinite(hi))):
            raise InvalidBounds("non-finite bounds")
        if np.any(lo > hi):
            raise InvalidBounds("lower corner exceeds upper corner")
        object.__setattr__(self, "lo", lo)
        object.__setattr__(self, "hi", hi)

    @classmethod
    def _trusted(cls, lo, hi):
        box = object.__new__(cls)
        object.__setattr__(box, "lo", lo)
        object.__setattr__(box, "hi", hi)
        return box

    @property
    def dim(self) -> int:
        return self.lo.shape[0]

    @property
    def center(self):
        return (self.lo + self.hi) / 2.0

    @property
    def extents(self):
        return self.hi - self.lo

    @property
    def volume(self) -> float:
        return float(np.prod(self.extents))

    def split(self):
        """Halve along the widest dimension (ties to the lowest index)."""
        ax = int(np.argmax(self.extents))
        mid = 0.5 * (self.lo[ax] + self.hi[ax])
        hi_a = self.hi.copy()
        hi_a[ax] = mid
        lo_b = self.lo.copy()
        lo_b[ax] = mid
        return AABB(self.lo, hi_a), AABB(lo_b, self.hi)

    def face_centers(self):
        c = self.center
        half = self.extents / 2.0
        pts = np.repeat(c[None, :], 2 * self.dim, axis=0)
        for i in range(self.dim):
            pts[2 * i, i] = c[i] - half[i]
            pts[2 * i + 1, i] = c[i] + half[i]
        return pts


@dataclass
class TreeNode:
    aabb: AABB
    sign: SignClass
    depth: int
    children: tuple | None = None
    face_sign: int | None = None

    @property
    def is_leaf(self) -> bool:
        return self.children is None


def iter_leaves(root: TreeNode):
    stack = [root]
    while stack:
        node = stack.pop()
        if node.is_leaf:
            yield node
        else:
            stack.extend(node.children)


@dataclass(frozen=True)
class TriangleMesh:
    vertices: np.ndarray
    triangles: np.ndarray

    def __post_init__(self):
        v = np.asarray(self.vertices, dtype=np.float64).reshape(-1, 3)
        t = np.asarray(self.triangles, dtype=np.int64).reshape(-1, 3)
        if v.size and not np.all(np.isfinite(v)):
            raise InvalidParameter("mesh vertices must be finite")
        if t.size and (t.min() < 0 or t.max() >= len(v)):
            raise InvalidParameter("triangle indices out of range")
        object.__setattr__(self, "vertices", v)
        object.__setattr__(self, "triangles", t)


@dataclass
class TreeLevel:
    """One breadth-first level: AABB corners, bound, label (+1/-1/0),
    face annotation (+1/-1, 0 none), parent index into the previous level."""

    lo: object
    hi: object
    bound_lo: object
    bound_hi: object
    label: object
    face: object
    parent: object

    def __len__(self):
        return int(self.label.shape[0])


class TreeArrays:
    """Per-level arrays of a built tree.  Levels are materialised on first
    access (zero-copy CUDA views or NumPy copies), so a caller that only
    needs counts/statistics pays for no Python-side wrapping."""

    def __init__(self, levels=None, start_depth=0, bound_evals=0, launches=0, bound_ms=0.0, meta=None,
                 loader=None, n_levels=0, n_nodes=0, first_level_len=0):
        self._levels = levels
        self._loader = loader
        self.start_depth = start_depth
        self.bound_evals = bound_evals
        self.launches = launches
        self.bound_ms = bound_ms
        self.meta = meta if meta is not None else {}
        self._n_levels = n_levels if levels is None else len(levels)
        self._n_nodes = n_nodes if levels is None else sum(len(l) for l in levels)
        self._first = first_level_len if levels is None else (len(levels[0]) if levels else 0)

    @property
    def levels(self):
        if self._levels is None:
            self._levels = self._loader()
            self._loader = None
        return self._levels

    @property
    def n_levels(self) -> int:
        return self._n_levels

    @property
    def n_nodes(self) -> int:
        return self._n_nodes

    @property
    def first_level_len(self) -> int:
        return self._first

    def keys(self):
        """Path keys per level (root 1, low child 2k, high child 2k+1)."""
        out = [np.arange(1, len(self.levels[0]) + 1, dtype=np.int64)]
        for lv in self.levels[1:]:
            par = _np(lv.parent)
            k = len(par) // 2
            bit = np.concatenate([np.zeros(k, np.int64), np.ones(k, np.int64)])
            out.append(out[-1][par] * 2 + bit)
        return out


def _np(x):
    return x.cpu().numpy() if dv.is_tensor(x) else x


def _check_domain(net, bounds: AABB):
    if bounds.dim != net.input_dim:
        raise DimensionMismatch(f"bounds in R^{bounds.dim}, network expects R^{net.input_dim}")
    if np.any(bounds.extents <= 0.0):
        raise InvalidBounds("bounds must have positive extent")


class _TreeHandle:
    """Owns an spk_tree*; destroyed when the last zero-copy view dies."""

    def __init__(self, ptr):
        self.ptr = ptr

    def __del__(self):
        if self.ptr:
            try:
                _lib.load().spk_tree_destroy(self.ptr)
            except (AttributeError, TypeError):  # interpreter shutdown: module globals already gone
                pass
            self.ptr = None


class _DeviceView:
    """__cuda_array_interface__ view of library-owned device memory."""

    def __init__(self, owner, ptr, shape, typestr):
        self.owner = owner
        self.__cuda_array_interface__ = {"shape": shape, "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None, "stream": None}


def _build(net, roots_lo, roots_hi, start_depth, delta, policy, max_depth, precision, to_host, device=None,
           band: float = 0.0, level_cap: int | None = None):
    pcode, n_keep = policy_code(policy)
    dn = device_net(net, device)
    roots_lo = np.ascontiguousarray(roots_lo, dtype=np.float64)
    roots_hi = np.ascontiguousarray(roots_hi, dtype=np.float64)
    handle = C.c_void_p()
    stream = dv.stream_ptr(dn.device)
    # to_host: the library mirrors every level to host memory while the next
    # level computes (overlapped copies) and the levels are NumPy views of it
    _lib.call(
        "spk_tree_build_ex", dn.ptr, pcode, n_keep, _precision_code(precision), roots_lo.shape[0],
        roots_lo.ctypes.data, roots_hi.ctypes.data, int(start_depth),
        -1 if max_depth is None else int(max_depth), float(delta), float(band),
        (_HOST_MIRROR if to_host else 0) | (0 if level_cap is None else (int(level_cap) + 1) << 8),
        stream, C.byref(handle),
    )
    owner = _TreeHandle(handle)
    lib = _lib.load()
    nl, nn, be = C.c_int(), C.c_int64(), C.c_int64()
    _lib.check(lib.spk_tree_info(handle, C.byref(nl), C.byref(nn), C.byref(be)))
    la, ms = C.c_int64(), C.c_double()
    _lib.check(lib.spk_tree_stats(handle, C.byref(la), C.byref(ms)))
    d = net.input_dim
    n0 = C.c_int64()
    if nl.value:
        _lib.check(lib.spk_tree_level(handle, 0, C.byref(n0), None, None, None, None, None, None, None))

    def loader():
        return [_level(owner, i, d, dn.device, to_host) for i in range(nl.value)]

    arr = TreeArrays(None, int(start_depth), be.value, la.value, ms.value, loader=loader, n_levels=nl.value,
                     n_nodes=nn.value, first_level_len=n0.value)
    if to_host:
        arr.levels  # NumPy views of the host mirror; the device levels go now
        _lib.call("spk_tree_release_device", handle)
    return arr


_LEVEL_SPECS = (("lo", "<f8", 2), ("hi", "<f8", 2), ("bound_lo", "<f8", 1), ("bound_hi", "<f8", 1),
                ("label", "|i1", 1), ("face", "|i1", 1), ("parent", "<i8", 1))


_HOST_MIRROR = 1  # SPK_TREE_HOST_MIRROR


class _HostView:
    """__array_interface__ view of the library's host mirror of a level; the
    NumPy array keeps it (and so the tree) alive."""

    def __init__(self, owner, ptr, shape, typestr):
        self.owner = owner
        self.__array_interface__ = {"shape": shape, "typestr": typestr, "data": (ptr or 0, False), "version": 3}


def _level(owner, level, d, device, to_host):
    """One level as NumPy arrays over the library's host mirror (to_host) or
    zero-copy CUDA tensors; both keep the library's tree alive."""
    n = C.c_int64()
    ptrs = [C.c_void_p() for _ in range(7)]
    if to_host:
        _lib.check(_lib.load().spk_tree_level_host(owner.ptr, level, C.byref(n), *[C.byref(p) for p in ptrs]))
        n = n.value
        out = []
        for (name, ts, nd), p in zip(_LEVEL_SPECS, ptrs):
            shape = (n, d) if nd == 2 else (n,)
            out.append(np.asarray(_HostView(owner, p.value, shape, ts)) if n else np.empty(shape, np.dtype(ts)))
        return TreeLevel(*out)
    _lib.check(_lib.load().spk_tree_level(owner.ptr, level, C.byref(n), *[C.byref(p) for p in ptrs]))
    n = n.value
    torch = dv._torch()
    out = []
    for (name, ts, nd), p in zip(_LEVEL_SPECS, ptrs):
        shape = (n, d) if nd == 2 else (n,)
        out.append(torch.as_tensor(_DeviceView(owner, p.value or 0, shape, ts), device=f"cuda:{device}"))
    return TreeLevel(*out)


def build_spatial_tree_arrays(net, bounds: AABB, delta: float = 0.001, policy=AFFINE_FULL,
                              max_depth: int | None = None, precision: str = "fp32",
                              to_host: bool = True) -> TreeArrays:
    """build_spatial_tree as flat per-level arrays (see module docstring)."""
    _check_domain(net, bounds)
    if delta <= 0.0:
        raise InvalidParameter("delta must be positive")
    if max_depth is not None and max_depth > _MAX_DEPTH:
        raise DepthOverflow(f"fixed depth {max_depth} exceeds {_MAX_DEPTH}")
    return _build(net, bounds.lo[None, :], bounds.hi[None, :], 0, delta, policy, max_depth, precision, to_host)


def build_spatial_tree(net, bounds: AABB, delta: float = 0.001, policy=AFFINE_FULL,
                       max_depth: int | None = None, precision: str = "fp32") -> TreeNode:
    """Breadth-first k-d bounding tree of the level set (spatial.py:214-289)."""
    arrays = build_spatial_tree_arrays(net, bounds, delta, policy, max_depth, precision, to_host=True)
    return materialize(arrays)


class _LazyTree:
    """Host level arrays + per-level child index (split rank of each node)."""

    def __init__(self, arrays: TreeArrays):
        self.levels = [(_np(l.lo), _np(l.hi), _np(l.label), _np(l.face), _np(l.parent)) for l in arrays.levels]
        self.start_depth = arrays.start_depth
        self.split_rank = []
        for k in range(len(self.levels)):
            n = len(self.levels[k][2])
            rank = np.full(n, -1, dtype=np.int64)
            if k + 1 < len(self.levels):
                par = self.levels[k + 1][4]
                half = len(par) // 2
                rank[par[:half]] = np.arange(half)
            self.split_rank.append(rank)

    def node(self, k: int, i: int) -> "_LazyNode":
        lo, hi, lab, face, _ = self.levels[k]
        f = int(face[i])
        return _LazyNode(self, k, i, AABB._trusted(lo[i], hi[i]), _SIGN[int(lab[i])], self.start_depth + k,
                         None if f == 0 else f)


_UNSET = object()


class _LazyNode(TreeNode):
    """A TreeNode whose children are built from the level arrays on first
    access: build_spatial_tree returns at once, and a traversal pays only for
    the nodes it visits (a depth-18 build has 524,287 nodes).  Same fields,
    same values, same isinstance as an eagerly built TreeNode."""

    def __init__(self, tree, k, i, aabb, sign, depth, face_sign):  # noqa: D107 (dataclass __init__ bypassed)
        self.aabb = aabb
        self.sign = sign
        self.depth = depth
        self.face_sign = face_sign
        self._tree = tree
        self._at = (k, i)
        self._kids = _UNSET

    @property
    def children(self):
        if self._kids is _UNSET:
            k, i = self._at
            j = int(self._tree.split_rank[k][i])
            if j < 0:
                self._kids = None
            else:
                half = len(self._tree.levels[k + 1][4]) // 2
                self._kids = (self._tree.node(k + 1, j), self._tree.node(k + 1, half + j))
        return self._kids

    @children.setter
    def children(self, value):
        self._kids = value


def materialize(arrays: TreeArrays, lazy: bool = True) -> TreeNode:
    """TreeNode objects from level arrays (reference node layout).  lazy:
    children are created on first access (see _LazyNode); lazy=False builds
    every node up front."""
    if lazy:
        return _LazyTree(arrays).node(0, 0)
    prev = None
    root = None
    for depth, lv in enumerate(arrays.levels):
        lo, hi = _np(lv.lo), _np(lv.hi)
        lab, face, par = _np(lv.label), _np(lv.face), _np(lv.parent)
        nodes = [
            TreeNode(AABB._trusted(lo[i], hi[i]), _SIGN[int(lab[i])], arrays.start_depth + depth, None,
                     None if face[i] == 0 else int(face[i]))
            for i in range(len(lab))
        ]
        if prev is None:
            root = nodes[0]
        else:
            k = len(nodes) // 2
            for j in range(k):
                prev[int(par[j])].children = (nodes[j], nodes[k + j])
        prev = nodes
    return root


def build_spatial_tree_sharded(net, bounds: AABB, max_depth: int, policy, rank: int, world: int,
                               precision: str = "fp32", min_roots_per_rank: int = 64,
                               to_host: bool = False, roots: str = "contiguous") -> TreeArrays:
    """Fixed-depth build split across `world` ranks (one per GPU).

    Every rank builds the top levels redundantly until the UNKNOWN frontier
    holds >= min_roots_per_rank * world nodes (or max_depth is reached), then
    refines its share of that frontier to max_depth -- a contiguous slice
    (`roots="contiguous"`) or every world-th root (`"interleaved"`, static
    balance for builds whose depth varies over space).  No collective runs
    inside the build; the union of the ranks' levels below the cut equals the
    unsharded tree (node AABBs are bit-identical because splits are exact
    FP64 midpoints) and `gather_spatial_tree` reassembles it in the
    reference's level order.
    """
    from .shard import first_cut, interleaved_roots, split_frontier

    _check_domain(net, bounds)
    if roots not in ("contiguous", "interleaved"):
        raise InvalidParameter(f"unknown root assignment {roots!r}")
    cut = first_cut(world, min_roots_per_rank, max_depth)
    while True:
        top = build_spatial_tree_arrays(net, bounds, 1.0, policy, cut, precision, to_host=True)
        n_open = int((_np(top.levels[-1].label) == 0).sum())
        if cut >= max_depth or n_open >= min_roots_per_rank * world or n_open == 0:
            break
        cut = min(max_depth, cut + 1)
    last = top.levels[-1]
    open_idx = np.flatnonzero(_np(last.label) == 0)
    if roots == "contiguous":
        root_ids = split_frontier(np.arange(len(open_idx)), rank, world)
    else:
        root_ids = interleaved_roots(len(open_idx), rank, world)
    part = open_idx[root_ids]
    meta = dict(cut=cut, roots=int(part.size), top_nodes=top.n_nodes, top=top.levels, open_idx=open_idx,
                root_ids=np.asarray(root_ids, dtype=np.int64), rank=rank, world=world)
    if cut >= max_depth or part.size == 0:
        top.meta.update(meta)
        top.meta["own_sub"] = False
        return top
    sub = _build(net, _np(last.lo)[part], _np(last.hi)[part], cut, 1.0, policy, max_depth, precision, to_host)
    sub.meta.update(meta, top_levels=top.levels, own_sub=True)
    return sub


def build_spatial_tree_rebalanced(net, bounds: AABB, rank: int, world: int, delta: float = 0.001,
                                  policy=AFFINE_FULL, max_depth: int | None = None, precision: str = "fp32",
                                  min_roots_per_rank: int = 64, segment_levels: int = 4, imbalance: float = 1.25,
                                  device=None) -> TreeArrays:
    """Sharded build with frontier rebalancing (north-star item: NCCL over
    NVLink "only for frontier rebalancing and the final gather").  Below the
    redundant top cut every rank refines its frontier slice in segments of
    `segment_levels` levels (spk_tree_build_ex with SPK_TREE_LEVEL_CAP); after
    each segment the ranks all_gather their open-frontier sizes and, when the
    largest exceeds `imbalance` x the mean, redistribute the open nodes (AABB
    corners + order key) evenly with one all_gather -- convergence-mode
    builds refine unevenly over space, so static slices drift apart.  Node
    bounds are per node, so the tree is the unsharded one node for node;
    `gather_spatial_tree` reassembles it (order keys travel with the nodes).
    The result holds this rank's rows below the cut (meta["packed"]) and the
    rebalancing record (meta["rebalance"])."""
    from .shard import first_cut, refine_segmented, split_frontier

    _check_domain(net, bounds)
    cut = first_cut(world, min_roots_per_rank, max_depth if max_depth is not None else 60)
    while True:
        top = build_spatial_tree_arrays(net, bounds, delta, policy, cut, precision, to_host=True)
        n_open = int((_np(top.levels[-1].label) == 0).sum())
        if (max_depth is not None and cut >= max_depth) or n_open >= min_roots_per_rank * world or n_open == 0:
            break
        cut += 1
    # NOTE: the top levels were built in fixed-depth mode; in convergence mode
    # a node above the cut can be a tiny leaf, which fixed mode would split.
    last = top.levels[-1]
    open_idx = np.flatnonzero(_np(last.label) == 0)
    mine = split_frontier(np.arange(len(open_idx)), rank, world)
    lo0, hi0 = _np(last.lo)[open_idx[mine]], _np(last.hi)[open_idx[mine]]

    def segment(lo, hi, j0):
        sub = _build(net, lo, hi, cut + j0, delta, policy, max_depth, precision, True, device,
                     level_cap=segment_levels)
        return [(_np(l.lo), _np(l.hi), _np(l.bound_lo), _np(l.bound_hi), _np(l.label), _np(l.face),
                 _np(l.parent)) for l in sub.levels]

    d = net.input_dim
    stop = delta / np.sqrt(float(d))
    packed, record = refine_segmented(segment, lo0, hi0, np.asarray(mine, np.int64), len(open_idx),
                                      segment_levels, stop, cut, max_depth, rank, world, imbalance)
    meta = dict(cut=cut, top=top.levels, open_idx=open_idx, rank=rank, world=world, packed=packed,
                rebalance=record, top_nodes=top.n_nodes)
    own = int(packed[0].sum()) if len(packed[0]) else 0
    return TreeArrays(top.levels, 0, meta=meta, n_nodes=own)


def _pack_subtree(arr: TreeArrays):
    """A sharded build's own levels below the cut as (level sizes (J, 1),
    f64 rows [lo, hi, bound_lo, bound_hi], i64 rows [key, label, face])."""
    from .shard import subtree_keys

    meta = arr.meta
    if "open_idx" not in meta:
        raise InvalidParameter("not a build_spatial_tree_sharded result")
    d = _np(meta["top"][0].lo).shape[1]
    f_rows, i_rows, sizes = [], [], []
    if meta.get("own_sub"):
        lv = arr.levels
        keys = subtree_keys([_np(l.parent) for l in lv], meta["root_ids"], len(meta["open_idx"]))
        for j in range(1, len(lv)):
            l = lv[j]
            f_rows.append(np.concatenate([_np(l.lo), _np(l.hi), _np(l.bound_lo)[:, None],
                                          _np(l.bound_hi)[:, None]], axis=1))
            i_rows.append(np.stack([keys[j], _np(l.label).astype(np.int64), _np(l.face).astype(np.int64)], axis=1))
            sizes.append(len(l))
    f_all = np.concatenate(f_rows, axis=0) if f_rows else np.zeros((0, 2 * d + 2))
    i_all = np.concatenate(i_rows, axis=0) if i_rows else np.zeros((0, 3), dtype=np.int64)
    return np.asarray(sizes, dtype=np.int64).reshape(-1, 1), f_all, i_all


def _assemble(meta, packed) -> TreeArrays:
    from .shard import merge_shard_levels

    top = meta["top"]
    d = _np(top[0].lo).shape[1]
    parts = []
    for sz, fr, ir in packed:
        edges = np.cumsum(np.r_[0, sz[:, 0]]).astype(np.int64)
        parts.append([(fr[edges[j]:edges[j + 1]], ir[edges[j]:edges[j + 1]]) for j in range(len(sz))])
    levels = [TreeLevel(*[_np(getattr(l, f)) for f in ("lo", "hi", "bound_lo", "bound_hi", "label", "face",
                                                       "parent")]) for l in top]
    for f, lab, face, parent in merge_shard_levels(parts, meta["open_idx"], 2 * d + 2):
        levels.append(TreeLevel(np.ascontiguousarray(f[:, :d]), np.ascontiguousarray(f[:, d:2 * d]),
                                f[:, 2 * d].copy(), f[:, 2 * d + 1].copy(), lab, face, parent))
    return TreeArrays(levels, 0, meta={"cut": meta["cut"], "gathered_from": len(packed)})


def merge_sharded_trees(parts) -> TreeArrays:
    """The unsharded tree from every rank's build_spatial_tree_sharded result
    (held in one process); the level order is the reference's."""
    parts = list(parts)
    if not parts:
        raise InvalidParameter("no shards")
    return _assemble(parts[0].meta, [_pack_subtree(p) for p in parts])


def _pack_subtree_t(arr: TreeArrays, device):
    """_pack_subtree on torch tensors on `device` (the build's levels stay on
    the GPU: keys, row packing and the collective never touch the host)."""
    torch = dv._torch()
    from .shard import subtree_keys_t

    meta = arr.meta
    if "open_idx" not in meta:
        raise InvalidParameter("not a build_spatial_tree_sharded result")

    def t(x, dtype=None):
        x = x if dv.is_tensor(x) else torch.from_numpy(np.ascontiguousarray(x))
        return x.to(device=device, dtype=dtype) if dtype is not None else x.to(device)

    d = _np(meta["top"][0].lo).shape[1]
    f_rows, i_rows, sizes = [], [], []
    if meta.get("own_sub"):
        lv = arr.levels
        keys = subtree_keys_t([t(l.parent, torch.int64) for l in lv],
                              t(np.asarray(meta["root_ids"], np.int64)), len(meta["open_idx"]))
        for j in range(1, len(lv)):
            l = lv[j]
            f_rows.append(torch.cat([t(l.lo, torch.float64), t(l.hi, torch.float64),
                                     t(l.bound_lo, torch.float64)[:, None], t(l.bound_hi, torch.float64)[:, None]],
                                    dim=1))
            i_rows.append(torch.stack([keys[j], t(l.label, torch.int64), t(l.face, torch.int64)], dim=1))
            sizes.append(len(l))
    f_all = torch.cat(f_rows, dim=0) if f_rows else torch.zeros((0, 2 * d + 2), dtype=torch.float64, device=device)
    i_all = torch.cat(i_rows, dim=0) if i_rows else torch.zeros((0, 3), dtype=torch.int64, device=device)
    return torch.tensor(sizes, dtype=torch.int64, device=device).reshape(-1, 1), f_all, i_all


def gather_spatial_tree(arr: TreeArrays, device=None, to_host: bool = True) -> TreeArrays:
    """Final gather of a frontier-sharded build -- the one collective step,
    after the build (torch.distributed all_gather: NCCL over NVLink on GPUs,
    gloo on CPU).  Every rank receives the whole tree in the unsharded
    (reference) order: the redundant top levels, then each deeper level merged
    by order key (shard.subtree_keys).  The packing, the all_gather and the
    key merge (stable sort + searchsorted) run on `device` -- the rank's GPU
    with NCCL, so the sub-tree levels never leave HBM; "cpu" with gloo.
    to_host=False keeps the merged levels there as tensors."""
    import torch.distributed as dist

    torch = dv._torch()
    from .shard import allgather_tensor, merge_shard_levels_t

    if device is None:
        lv0 = arr.levels[0].label
        device = lv0.device if dv.is_tensor(lv0) else "cpu"
    if "packed" in arr.meta:  # rebalanced build: rows computed during the refinement
        sz, f_rows, i_rows = arr.meta["packed"]
        mine = tuple(torch.from_numpy(np.ascontiguousarray(x)).to(device)
                     for x in (np.asarray(sz, np.int64).reshape(-1, 1), f_rows, i_rows))
    else:
        mine = _pack_subtree_t(arr, device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        packed = list(zip(*[allgather_tensor(x, device) for x in mine]))
    else:
        packed = [mine]
    meta = arr.meta
    top = meta["top"]
    d = _np(top[0].lo).shape[1]
    parts = []
    for sz, fr, ir in packed:
        edges = [0]
        for v in sz[:, 0].tolist():
            edges.append(edges[-1] + int(v))
        parts.append([(fr[edges[j]:edges[j + 1]], ir[edges[j]:edges[j + 1]]) for j in range(len(edges) - 1)])
    open_idx = torch.from_numpy(np.asarray(meta["open_idx"], np.int64)).to(device)
    merged = merge_shard_levels_t(parts, open_idx)

    def out(x):
        return x.cpu().numpy() if to_host else x

    def top_field(x):
        if to_host:
            return _np(x)
        return (x if dv.is_tensor(x) else torch.from_numpy(np.ascontiguousarray(x))).to(device)

    levels = [TreeLevel(*[top_field(getattr(l, f)) for f in ("lo", "hi", "bound_lo", "bound_hi", "label", "face",
                                                              "parent")]) for l in top]
    for f, lab, face, parent in merged:
        levels.append(TreeLevel(out(f[:, :d].contiguous()), out(f[:, d:2 * d].contiguous()),
                                out(f[:, 2 * d].contiguous()), out(f[:, 2 * d + 1].contiguous()), out(lab),
                                out(face), out(parent)))
    return TreeArrays(levels, 0, meta={"cut": meta["cut"], "gathered_from": len(packed), "device": str(device)})


# The volumetric queries live in queries.py; re-exported here because the
# reference defines them in spatial.py (spatial.py:292-720).
from .queries import (  # noqa: E402
    BulkProperties,
    EmptyRegion,
    IntersectionResult,
    bulk_properties,
    certified_radii,
    closest_point,
    empty_box_radius,
    sample_near_surface,
    save_obj,
    save_xyz,
    test_intersection,
    walk_on_spheres,
    walk_on_spheres_stats,
)
