"""Marching-cubes connectivity (reference mc_tables.py:1-105).

The reference does not use the classic Lorensen/Bourke table: it generates
its 256 cases at import time by marching squares on each cube face (inside
kept on the left seen from outside, ambiguous faces resolved by isolating
the inside corners), chaining the face segments into loops and fanning each
loop with reversed winding.  The same rule is re-derived here so the GPU
emits identical connectivity; tests compare it with the reference's table.
"""

from __future__ import annotations

import numpy as np

CORNERS = np.array(
    [[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0], [0, 0, 1], [1, 0, 1], [1, 1, 1], [0, 1, 1]],
    dtype=np.int64,
)
EDGES = ((0, 1), (1, 2), (2, 3), (3, 0), (4, 5), (5, 6), (6, 7), (7, 4), (0, 4), (1, 5), (2, 6), (3, 7))
# each face as a corner cycle, counter-clockwise seen from outside the cube
FACES = ((0, 3, 2, 1), (4, 5, 6, 7), (0, 1, 5, 4), (3, 7, 6, 2), (0, 4, 7, 3), (1, 2, 6, 5))

_EDGE_ID = {frozenset(e): i for i, e in enumerate(EDGES)}


def _segments(inside, cycle):
    """Directed isoline segments (exit edge -> entry edge) on one face."""
    flags = [inside[c] for c in cycle]
    sides = [_EDGE_ID[frozenset((cycle[i], cycle[(i + 1) % 4]))] for i in range(4)]
    leaving = [i for i in range(4) if flags[i] and not flags[(i + 1) % 4]]
    if not leaving:
        return []
    if len(leaving) == 1:
        entering = next(i for i in range(4) if not flags[i] and flags[(i + 1) % 4])
        return [(sides[leaving[0]], sides[entering])]
    # saddle face: every inside corner is cut off on its own
    return [(sides[p], sides[(p + 3) % 4]) for p in range(4) if flags[p]]


def triangles_for_case(case: int) -> tuple:
    inside = [bool(case >> c & 1) for c in range(8)]
    succ = dict(seg for cyc in FACES for seg in _segments(inside, cyc))
    tris = []
    pending = sorted(succ)
    while pending:
        start = pending[0]
        loop = [start]
        nxt = succ[start]
        while nxt != start:
            loop.append(nxt)
            nxt = succ[nxt]
        pending = [e for e in pending if e not in loop]
        tris.extend((loop[0], loop[k + 1], loop[k]) for k in range(1, len(loop) - 1))
    return tuple(tris)


TRI_TABLE = tuple(triangles_for_case(c) for c in range(256))
EDGE_TABLE = tuple(
    sum(1 << e for e, (a, b) in enumerate(EDGES) if (c >> a & 1) != (c >> b & 1)) for c in range(256)
)


def flat_tables():
    """(tri_table int8[256, 15], tri_count uint8[256]) for the C-ABI."""
    table = np.full((256, 15), -1, np.int8)
    count = np.zeros(256, np.uint8)
    for c, tris in enumerate(TRI_TABLE):
        count[c] = len(tris)
        for t, tri in enumerate(tris):
            table[c, 3 * t : 3 * t + 3] = tri
    return np.ascontiguousarray(table), count
