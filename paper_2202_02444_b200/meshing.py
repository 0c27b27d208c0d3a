"""Marching-cubes extraction on the B200 (reference meshing.py:100-169).

`extract_mesh` keeps the reference contract (TriangleMesh out, default
policy affine-full, output identical to `extract_mesh_dense` up to
ordering).  Everything runs in the C-ABI (`spk_mesh_extract`, K7): the
index-range prune with the fused bound kernel, per-block corner lattices
through the point-evaluation pass, case codes / emission from the
reference's generated TRI_TABLE, and edge-keyed vertex dedup with vertices
numbered in first-visit order.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from . import device as dv
from .errors import ResolutionTooSmall
from .mc_tables import flat_tables
from .network import _precision_code, device_net
from .range_core import AFFINE_FULL, policy_code
from .spatial import AABB, TriangleMesh, _check_domain

_TABLES = None


def _tables():
    global _TABLES
    if _TABLES is None:
        _TABLES = flat_tables()
    return _TABLES


@dataclass
class MeshResult:
    vertices: np.ndarray
    triangles: np.ndarray
    vertex_keys: np.ndarray  # global grid edge id per vertex
    n_blocks: int = 0
    point_evals: int = 0
    bound_evals: int = 0
    meta: dict = field(default_factory=dict)

    @property
    def mesh(self) -> TriangleMesh:
        return TriangleMesh(self.vertices, self.triangles)


def extract_mesh_arrays(net, bounds: AABB, m: int, dense_levels: int = 3, policy=AFFINE_FULL,
                        precision: str = "fp64", prune: bool = True) -> MeshResult:
    _check_domain(net, bounds)
    if m <= dense_levels:
        raise ResolutionTooSmall(f"resolution exponent {m} must exceed dense_levels {dense_levels}")
    pcode, n_keep = policy_code(policy)
    dn = device_net(net)
    table, count = _tables()
    lo = np.ascontiguousarray(bounds.lo, dtype=np.float64)
    hi = np.ascontiguousarray(bounds.hi, dtype=np.float64)
    h = C.c_void_p()
    _lib.call("spk_mesh_extract", dn.ptr, pcode, n_keep, _precision_code(precision), lo.ctypes.data, hi.ctypes.data,
              int(m), int(dense_levels), 1 if prune else 0, table.ctypes.data, count.ctypes.data,
              dv.stream_ptr(dn.device), C.byref(h))
    lib = _lib.load()
    try:
        nv, nt, nb, pe, be = (C.c_int64() for _ in range(5))
        _lib.check(lib.spk_mesh_info(h, C.byref(nv), C.byref(nt), C.byref(nb), C.byref(pe), C.byref(be)))
        verts = np.empty((nv.value, 3))
        tris = np.empty((nt.value, 3), np.int64)
        keys = np.empty(nv.value, np.uint64)
        _lib.call("spk_mesh_copy", h, verts.ctypes.data, tris.ctypes.data, keys.ctypes.data)
    finally:
        lib.spk_mesh_destroy(h)
    return MeshResult(verts, tris, keys.astype(np.int64), nb.value, pe.value, be.value)


def extract_mesh_sharded(net, bounds: AABB, m: int, rank: int, world: int, dense_levels: int = 3,
                         policy=AFFINE_FULL, precision: str = "fp64") -> MeshResult:
    """This rank's share of a hierarchical extraction (one process per GPU,
    SURVEY.md §8(e)): the prune runs redundantly, then the rank extracts its
    contiguous slice of the surviving blocks (visiting order) with no
    collective.  `gather_mesh` reassembles the reference's arrays."""
    _check_domain(net, bounds)
    if m <= dense_levels:
        raise ResolutionTooSmall(f"resolution exponent {m} must exceed dense_levels {dense_levels}")
    pcode, n_keep = policy_code(policy)
    dn = device_net(net)
    table, count = _tables()
    lo = np.ascontiguousarray(bounds.lo, dtype=np.float64)
    hi = np.ascontiguousarray(bounds.hi, dtype=np.float64)
    h = C.c_void_p()
    _lib.call("spk_mesh_extract_shard", dn.ptr, pcode, n_keep, _precision_code(precision), lo.ctypes.data,
              hi.ctypes.data, int(m), int(dense_levels), 1, table.ctypes.data, count.ctypes.data, int(rank),
              int(world), dv.stream_ptr(dn.device), C.byref(h))
    lib = _lib.load()
    try:
        nv, nt, nb, pe, be, bf, btot = (C.c_int64() for _ in range(7))
        _lib.check(lib.spk_mesh_info(h, C.byref(nv), C.byref(nt), C.byref(nb), C.byref(pe), C.byref(be)))
        _lib.check(lib.spk_mesh_shard_info(h, C.byref(bf), C.byref(btot)))
        verts = np.empty((nv.value, 3))
        tris = np.empty((nt.value, 3), np.int64)
        keys = np.empty(nv.value, np.uint64)
        _lib.call("spk_mesh_copy", h, verts.ctypes.data, tris.ctypes.data, keys.ctypes.data)
    finally:
        lib.spk_mesh_destroy(h)
    return MeshResult(verts, tris, keys.astype(np.int64), nb.value, pe.value, be.value,
                      meta={"rank": rank, "world": world, "block_first": bf.value, "blocks_total": btot.value})


def _mesh_part_t(res: MeshResult, device):
    torch = dv._torch()
    keys = torch.from_numpy(np.ascontiguousarray(res.vertex_keys, np.int64)).to(device)
    tris = torch.from_numpy(np.ascontiguousarray(res.triangles, np.int64)).to(device)
    verts = torch.from_numpy(np.ascontiguousarray(res.vertices, np.float64)).to(device)
    return keys[tris] if tris.numel() else tris.reshape(0, 3), keys, verts


def _mesh_result(vertices, triangles, vertex_keys, meta) -> MeshResult:
    return MeshResult(vertices.cpu().numpy(), triangles.cpu().numpy(), vertex_keys.cpu().numpy(), meta=meta)


def merge_sharded_meshes(parts) -> MeshResult:
    """The unsharded mesh from every rank's extract_mesh_sharded result (held
    in one process, rank order)."""
    from .shard import merge_mesh_parts_t

    parts = list(parts)
    v, t, k = merge_mesh_parts_t([_mesh_part_t(p, "cpu") for p in parts])
    return _mesh_result(v, t, k, {"merged_from": len(parts)})


def gather_mesh(res: MeshResult, device=None) -> MeshResult:
    """Final gather of a sharded extraction -- the one collective step: every
    rank all_gathers the others' triangles (as edge-key triples) and vertex
    rows (NCCL over NVLink on GPUs, gloo on CPU), then the global sort-unique
    dedup on edge keys (first occurrence) runs on `device` and every rank
    holds extract_mesh's arrays (vertices numbered in first-visit order)."""
    import torch.distributed as dist

    from .shard import allgather_tensor, merge_mesh_parts_t

    if device is None:
        torch = dv._torch()
        device = f"cuda:{torch.cuda.current_device()}" if torch.cuda.is_available() else "cpu"
    tk, vk, vp = _mesh_part_t(res, device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        parts = list(zip(allgather_tensor(tk, device), allgather_tensor(vk, device), allgather_tensor(vp, device)))
    else:
        parts = [(tk, vk, vp)]
    v, t, k = merge_mesh_parts_t(parts)
    return _mesh_result(v, t, k, {"gathered_from": len(parts)})


def extract_mesh(net, bounds: AABB, m: int, dense_levels: int = 3, policy=AFFINE_FULL,
                 precision: str = "fp64") -> TriangleMesh:
    """Hierarchical extraction at resolution 2**m (meshing.py:111-169)."""
    return extract_mesh_arrays(net, bounds, m, dense_levels, policy, precision, prune=True).mesh


def extract_mesh_dense(net, bounds: AABB, m: int, precision: str = "fp64") -> TriangleMesh:
    """Brute-force extraction over the full 2**m grid (meshing.py:100-108)."""
    _check_domain(net, bounds)
    return extract_mesh_arrays(net, bounds, m, min(3, m - 1), AFFINE_FULL, precision, prune=False).mesh


def triangle_key_set(triangles, vertex_keys):
    """Triangles as edge-key triples rotated so the smallest key leads
    (winding preserved), sorted: an order-free canonical form."""
    k = np.asarray(vertex_keys)[np.asarray(triangles)]
    r = np.argmin(k, axis=1)
    rows = np.arange(len(k))
    rot = np.stack([k[rows, r], k[rows, (r + 1) % 3], k[rows, (r + 2) % 3]], axis=1)
    return rot[np.lexsort(rot.T[::-1])]
