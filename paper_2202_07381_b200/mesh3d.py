"""Kuhn (Freudenthal) tetrahedral meshes of the unit cube and their nested
hierarchy -- BASELINE config 4 (the reference has no
3-D discretisation, F3).

Each of the n^3 cubes is split into the 6 tetrahedra along its main
diagonal: for every permutation s of the axes, the path
p0 -> p0 + e_s0 -> p0 + e_s0 + e_s1 -> p0 + (1, 1, 1).  Freudenthal's
subdivision of a Kuhn simplex is the Kuhn mesh of the doubled grid, so the
levels n0 * 2^l are nested and each is generated directly.

Numbering mirrors the 2-D meshes: vertices x-fastest, cells 6 per cube in
permutation order, edges as sorted unique vertex pairs (lexicographic); the
P2 nodes are the vertices, then the edge midpoints.
"""

from dataclasses import dataclass, field
from itertools import permutations

import numpy as np

__all__ = ["Mesh3D", "kuhn_cube", "Hierarchy3D", "build_hierarchy3d", "PERMS", "TET_EDGES",
           "locate_kuhn"]

PERMS = np.array(list(permutations(range(3))), dtype=np.int64)      # (6, 3)
TET_EDGES = np.array([(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)], dtype=np.int64)


@dataclass
class Mesh3D:
    n: int                      # cubes per direction
    vertices: np.ndarray        # (V, 3)
    cells: np.ndarray           # (C, 4) vertex ids
    edges: np.ndarray           # (E, 2) sorted vertex pairs
    cell_to_edges: np.ndarray   # (C, 6) in TET_EDGES order
    boundary_vertex_flags: np.ndarray = field(repr=False)
    boundary_edge_flags: np.ndarray = field(repr=False)
    dim: int = 3

    @property
    def num_vertices(self):
        return len(self.vertices)

    @property
    def num_edges(self):
        return len(self.edges)

    @property
    def num_cells(self):
        return len(self.cells)


def kuhn_cube(n):
    """The Kuhn mesh of an n x n x n grid of cubes on [0, 1]^3."""
    if n < 1:
        raise ValueError("n must be >= 1")
    m = n + 1
    g = np.arange(m)
    z, y, x = np.meshgrid(g, g, g, indexing="ij")
    vertices = np.column_stack([x.ravel(), y.ravel(), z.ravel()]) / float(n)

    def vid(ijk):
        return ijk[..., 0] + m * (ijk[..., 1] + m * ijk[..., 2])

    c = np.arange(n)
    cz, cy, cx = np.meshgrid(c, c, c, indexing="ij")
    corner = np.column_stack([cx.ravel(), cy.ravel(), cz.ravel()])          # (n^3, 3)
    eye = np.eye(3, dtype=np.int64)
    tets = np.empty((len(corner), 6, 4), dtype=np.int64)
    for s, perm in enumerate(PERMS):
        p = corner.copy()
        tets[:, s, 0] = vid(p)
        for k in range(3):
            p = p + eye[perm[k]]
            tets[:, s, k + 1] = vid(p)
    cells = tets.reshape(-1, 4)
    pairs = np.sort(cells[:, TET_EDGES], axis=2).reshape(-1, 2)         # (C*6, 2)
    key = pairs[:, 0] * len(vertices) + pairs[:, 1]
    ukey, inv = np.unique(key, return_inverse=True)
    edges = np.column_stack([ukey // len(vertices), ukey % len(vertices)])
    cell_to_edges = inv.reshape(-1, 6)
    on_b = np.any((vertices == 0.0) | (vertices == 1.0), axis=1)
    # an edge is on the boundary iff both ends lie on a common boundary face
    a, b = vertices[edges[:, 0]], vertices[edges[:, 1]]
    be = np.any(((a == 0.0) & (b == 0.0)) | ((a == 1.0) & (b == 1.0)), axis=1)
    return Mesh3D(n=n, vertices=vertices, cells=cells, edges=edges, cell_to_edges=cell_to_edges,
                  boundary_vertex_flags=on_b, boundary_edge_flags=be)


def locate_kuhn(n, points):
    """(cell id, barycentric coordinates (N, 4)) of points in the Kuhn mesh
    of an n^3 grid; points on shared faces get one containing cell."""
    p = np.asarray(points, dtype=np.float64) * n
    cube = np.minimum(np.floor(p).astype(np.int64), n - 1)
    u = p - cube                                                       # local coords in [0, 1]
    # descending sort of the local coordinates picks the permutation
    order = np.argsort(-u, axis=1, kind="stable")
    key = order[:, 0] * 9 + order[:, 1] * 3 + order[:, 2]
    perm_id = np.full(27, -1, dtype=np.int64)
    perm_id[PERMS[:, 0] * 9 + PERMS[:, 1] * 3 + PERMS[:, 2]] = np.arange(6)
    s = perm_id[key]
    us = np.take_along_axis(u, order, axis=1)
    lam = np.column_stack([1.0 - us[:, 0], us[:, 0] - us[:, 1], us[:, 1] - us[:, 2], us[:, 2]])
    cid = cube[:, 0] + n * (cube[:, 1] + n * cube[:, 2])
    return 6 * cid + s, lam


@dataclass
class Hierarchy3D:
    levels: list

    @property
    def num_levels(self):
        return len(self.levels)


def build_hierarchy3d(n0, level):
    """Kuhn meshes n0 * 2^l, l = 0..level (nested)."""
    return Hierarchy3D([kuhn_cube(n0 * 2 ** l) for l in range(level + 1)])
