"""Mesh comparison rule of the north star: triangles must be
identical on every grid cell whose 8 corner signs agree between the two
evaluations.  Shared by the FP32-vs-FP64 mesh tests."""

import numpy as np

import paper_2202_02444_b200 as sp
from paper_2202_02444_b200 import meshing


def triangle_cells(tris, keys, m):
    """Grid cells a triangle can belong to: the cells containing all three of
    its vertices' grid edges (one cell, or the two sharing a face when the
    triangle lies in that face).  Returns an (n, 2) array of linear cell ids,
    -1 where there is no second cell."""
    n_pts = (1 << m) + 1
    n_cells = 1 << m
    k = keys[tris]                                  # (t, 3) edge keys
    ax = k % 3
    lin = k // 3
    low = np.stack([lin // (n_pts * n_pts), (lin // n_pts) % n_pts, lin % n_pts], axis=-1)  # (t, 3, 3)
    # candidate cells of the first edge: c[a] = low[a], c[b] in {low[b]-1, low[b]}
    cands = []
    for db in range(4):
        c = low[:, 0, :].copy()
        others = [b for b in range(3)]
        off = np.zeros_like(c)
        for t_i in range(len(c)):
            a = ax[t_i, 0]
            ob = [b for b in others if b != a]
            off[t_i, ob[0]] = -(db & 1)
            off[t_i, ob[1]] = -((db >> 1) & 1)
        cands.append(c + off)
    cands = np.stack(cands, axis=1)                 # (t, 4, 3)
    ok = np.all((cands >= 0) & (cands < n_cells), axis=-1)
    for e in range(3):
        le = low[:, e, None, :]                     # (t, 1, 3)
        a = ax[:, e]
        d = le - cands                              # (t, 4, 3)
        onaxis = np.take_along_axis(d, a[:, None, None].repeat(4, 1), axis=2)[..., 0] == 0
        inrange = np.all((d == 0) | (d == 1), axis=-1)
        ok &= onaxis & inrange
    cell_ids = (cands[..., 0] * n_cells + cands[..., 1]) * n_cells + cands[..., 2]
    out = np.full((len(k), 2), -1, np.int64)
    for i in range(len(k)):
        ids = cell_ids[i][ok[i]]
        assert 1 <= len(ids) <= 2, (i, ids)
        out[i, :len(ids)] = ids
    return out



def agreeing_triangle_sets(net, a, b, m, lo=-1.0, hi=1.0):
    """(triangles of a, triangles of b) on the cells whose corner signs agree
    between FP64 and FP32 point evaluation, as canonical edge-key sets, plus
    the counts of triangles left out and of disagreeing cells."""
    n = 1 << m
    g = np.linspace(lo, hi, n + 1)
    pts = np.stack(np.meshgrid(g, g, g, indexing="ij"), axis=-1).reshape(-1, 3)
    s64 = (sp.eval_batch(net, pts, precision="fp64") < 0.0).reshape(n + 1, n + 1, n + 1)
    s32 = (sp.eval_batch(net, pts, precision="fp32") < 0.0).reshape(n + 1, n + 1, n + 1)
    same = s64 == s32
    agree = np.ones((n, n, n), bool)
    for dx in (0, 1):
        for dy in (0, 1):
            for dz in (0, 1):
                agree &= same[dx:dx + n, dy:dy + n, dz:dz + n]
    agree = agree.reshape(-1)

    def kept(res):
        if len(res.triangles) == 0:
            return np.zeros((0, 3), np.int64), 0
        cells = triangle_cells(res.triangles, res.vertex_keys, m)
        ok = agree[cells[:, 0]] & np.where(cells[:, 1] >= 0, agree[np.maximum(cells[:, 1], 0)], True)
        return meshing.triangle_key_set(res.triangles[ok], res.vertex_keys), int((~ok).sum())

    ka, na = kept(a)
    kb, nb = kept(b)
    return ka, kb, na, nb, int((~agree).sum())
