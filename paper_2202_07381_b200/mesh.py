"""Triangle meshes of the unit square and red refinement (host-side setup).

This module produces the *inputs* of the IRK-Vanka hot path: the vertex,
edge and cell numbering from which every DoF index (and therefore every
Vanka patch index list) is derived.  DoF numbering must agree bit-for-bit
with the reference ``irkmg`` package, so the numbering rules follow it:

* edges are the sorted (min, max) vertex pairs in lexicographic order
  (reference ``/root/reference/pkg/src/irkmg/mesh.py:63-66``);
* local edge k of a cell is opposite local vertex k (``mesh.py:62-63``);
* red refinement keeps the coarse vertices and appends edge midpoints in
  edge order, vertex ``V + e`` bisecting coarse edge ``e``
  (``mesh.py:178-206``).

Two coarse grids are provided: ``diagonal_grid`` (2 right triangles per
square, the BASELINE.json configs) and ``crossed_grid``
(4 triangles per square around a centre vertex, the reference's own
``build_crossed_grid``, ``mesh.py:144-175``).
"""

from dataclasses import dataclass

import numpy as np

__all__ = [
    "Mesh2D",
    "MeshHierarchy",
    "diagonal_grid",
    "crossed_grid",
    "refine_red",
    "build_hierarchy",
]


class Mesh2D:
    """Counter-clockwise triangle mesh with derived edge / boundary data.

    Attribute names mirror the reference ``Mesh2D`` (``mesh.py:25-98``) so
    that a reference caller can hand either object to the patch builder.
    """

    def __init__(self, vertices, cells):
        verts = np.ascontiguousarray(np.asarray(vertices, dtype=np.float64))
        cells = np.ascontiguousarray(np.asarray(cells, dtype=np.int64))
        if verts.ndim != 2 or verts.shape[1] != 2:
            raise ValueError("vertices must be a (V, 2) array")
        if cells.ndim != 2 or cells.shape[1] != 3:
            raise ValueError("cells must be a (C, 3) array")
        nv = len(verts)
        if cells.size and (cells.min() < 0 or cells.max() >= nv):
            raise ValueError("cell vertex index out of range")
        if np.any(_twice_signed_area(verts, cells) <= 0.0):
            raise ValueError("all cells must be counterclockwise with positive area")

        # Local edge k joins the two cell vertices other than vertex k.
        a = cells[:, [1, 2, 0]]
        b = cells[:, [2, 0, 1]]
        lo = np.minimum(a, b).ravel()
        hi = np.maximum(a, b).ravel()
        key = lo * nv + hi
        ukey, inverse = np.unique(key, return_inverse=True)
        edges = np.column_stack([ukey // nv, ukey % nv]).astype(np.int64)
        c2e = inverse.reshape(-1, 3).astype(np.int64)

        incidence = np.bincount(inverse, minlength=len(edges))
        if np.any(incidence > 2):
            raise ValueError("edge shared by more than two cells")
        bedge = incidence == 1
        bvert = np.zeros(nv, dtype=bool)
        bvert[edges[bedge].ravel()] = True

        self.vertices = verts
        self.cells = cells
        self.edges = edges
        self.cell_to_edges = c2e
        self.boundary_vertex_flags = bvert
        self.boundary_edge_flags = bedge

    @property
    def num_vertices(self):
        return len(self.vertices)

    @property
    def num_edges(self):
        return len(self.edges)

    @property
    def num_cells(self):
        return len(self.cells)

    def cell_areas(self):
        return 0.5 * _twice_signed_area(self.vertices, self.cells)


@dataclass(frozen=True)
class MeshHierarchy:
    """Nested meshes, coarsest first, with the child->parent cell map."""

    levels: tuple
    cell_parent: tuple

    @property
    def num_levels(self):
        return len(self.levels)

    def finest(self):
        return self.levels[-1]


def _twice_signed_area(verts, cells):
    p0 = verts[cells[:, 0]]
    e1 = verts[cells[:, 1]] - p0
    e2 = verts[cells[:, 2]] - p0
    return e1[:, 0] * e2[:, 1] - e1[:, 1] * e2[:, 0]


def _grid_points(n):
    t = np.linspace(0.0, 1.0, n + 1)
    # y-major: vertex j*(n+1)+i sits at (t[i], t[j]).
    return np.column_stack([np.tile(t, n + 1), np.repeat(t, n + 1)])


def diagonal_grid(n):
    """n x n squares, each split by its lower-left -> upper-right diagonal.

    Cells per square (i, j): ``[v00, v10, v11]`` then ``[v00, v11, v01]``
    (SURVEY.md F1).  The DoF numbering depends only on the y-major vertex
    numbering and the diagonal direction, never on the cell order.
    """
    n = int(n)
    if n < 1:
        raise ValueError(f"cells-per-side must be >= 1, got {n}")
    j, i = np.divmod(np.arange(n * n), n)
    v00 = j * (n + 1) + i
    v10 = v00 + 1
    v01 = v00 + n + 1
    v11 = v01 + 1
    cells = np.empty((2 * n * n, 3), dtype=np.int64)
    cells[0::2] = np.column_stack([v00, v10, v11])
    cells[1::2] = np.column_stack([v00, v11, v01])
    return Mesh2D(_grid_points(n), cells)


def crossed_grid(n):
    """n x n squares, each cut into 4 triangles around its centre vertex.

    Same vertex order and cell order as the reference ``build_crossed_grid``
    (``mesh.py:144-175``): grid points y-major, then square centres.
    """
    n = int(n)
    if n < 1:
        raise ValueError(f"cells-per-side must be >= 1, got {n}")
    t = np.linspace(0.0, 1.0, n + 1)
    mid = 0.5 * (t[:-1] + t[1:])
    centres = np.column_stack([np.tile(mid, n), np.repeat(mid, n)])
    verts = np.vstack([_grid_points(n), centres])
    j, i = np.divmod(np.arange(n * n), n)
    v00 = j * (n + 1) + i
    v10 = v00 + 1
    v01 = v00 + n + 1
    v11 = v01 + 1
    c = (n + 1) ** 2 + j * n + i
    cells = np.empty((4 * n * n, 3), dtype=np.int64)
    cells[0::4] = np.column_stack([v00, v10, c])
    cells[1::4] = np.column_stack([v10, v11, c])
    cells[2::4] = np.column_stack([v11, v01, c])
    cells[3::4] = np.column_stack([v01, v00, c])
    return Mesh2D(verts, cells)


def refine_red(mesh):
    """Split every cell into 4 through its edge midpoints.

    Returns ``(fine, cell_parent)``.  Coarse vertices keep their indices,
    midpoint vertex ``V + e`` bisects coarse edge ``e`` and the four
    children of cell c are fine cells 4c..4c+3, in the order of the
    reference ``refine_uniform`` (``mesh.py:195-201``).
    """
    nv = mesh.num_vertices
    ev = mesh.vertices[mesh.edges]
    verts = np.vstack([mesh.vertices, 0.5 * (ev[:, 0] + ev[:, 1])])
    v = mesh.cells
    m = nv + mesh.cell_to_edges  # m[:, k] is the midpoint opposite vertex k
    kids = np.stack([
        np.column_stack([v[:, 0], m[:, 2], m[:, 1]]),
        np.column_stack([v[:, 1], m[:, 0], m[:, 2]]),
        np.column_stack([v[:, 2], m[:, 1], m[:, 0]]),
        np.column_stack([m[:, 0], m[:, 1], m[:, 2]]),
    ], axis=1).reshape(-1, 3)
    parent = np.repeat(np.arange(mesh.num_cells, dtype=np.int64), 4)
    return Mesh2D(verts, kids), parent


def build_hierarchy(n0, refinements, kind="diagonal"):
    """``refinements`` red refinements of an n0 x n0 coarse grid."""
    if refinements < 0:
        raise ValueError(f"refinement count must be >= 0, got {refinements}")
    if kind == "diagonal":
        levels = [diagonal_grid(n0)]
    elif kind == "crossed":
        levels = [crossed_grid(n0)]
    else:
        raise ValueError(f"unknown coarse grid kind {kind!r}")
    parents = []
    for _ in range(refinements):
        fine, parent = refine_red(levels[-1])
        levels.append(fine)
        parents.append(parent)
    return MeshHierarchy(tuple(levels), tuple(parents))
