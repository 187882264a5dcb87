"""Taylor-Hood P2-P1 assembly in *scalar-node* form (host-side setup).

The hot path never needs the interleaved vector-P2 matrices the reference
stores (``/root/reference/pkg/src/irkmg/fem.py:128-196``): the velocity
mass and stiffness are exactly ``M_P2 (x) I_2`` and ``K_P2 (x) I_2``
(reference ``_expand_vector``, ``fem.py:149-154``), so they
are assembled once on the scalar P2 pattern and the GPU reads each scalar
value once for both components and all s stages.  The divergence block is
stored as one (B_x, B_y) pair per (P2 node, P1 node) and the convection
Jacobian as one 2x2 block per scalar P2 pattern entry.

DoF conventions (reference ``fem.py:1-13``): P1 DoFs are the mesh
vertices; scalar P2 nodes are the vertices then the edge midpoints (node
``V + e`` on edge ``e``); vector P2 interleaves components, scalar node n
owning DoFs ``2n`` and ``2n + 1``.

Quadrature degrees are the reference's (``fem.py:45-50``): mass 4,
stiffness 2, divergence 3, convection 5.
"""

from dataclasses import dataclass
from typing import Optional

import numpy as np
import scipy.sparse as sp

from .mesh import MeshHierarchy
from .quadrature import p1_basis, p2_basis, triangle_rule

__all__ = [
    "StokesBlocks",
    "ConvectionBlocks",
    "p2_cell_nodes",
    "p2_node_coords",
    "assemble_blocks",
    "assemble_convection_jacobian",
    "assemble_convection_residual",
    "prolongation",
    "velocity_boundary_nodes",
    "velocity_boundary_dofs",
    "interpolate_velocity",
]

DEG_MASS = 4
DEG_STIFFNESS = 2
DEG_DIVERGENCE = 3
DEG_CONVECTION = 5


def p2_cell_nodes(mesh):
    """(C, 6) scalar P2 nodes per cell: vertices, then opposite-edge midpoints."""
    return np.hstack([mesh.cells, mesh.num_vertices + mesh.cell_to_edges])


def p2_node_coords(mesh):
    ev = mesh.vertices[mesh.edges]
    return np.vstack([mesh.vertices, 0.5 * (ev[:, 0] + ev[:, 1])])


def _affine(mesh):
    """Per-cell origin, inverse Jacobian (C, 2, 2) and det J."""
    p = mesh.vertices[mesh.cells]
    jac = np.stack([p[:, 1] - p[:, 0], p[:, 2] - p[:, 0]], axis=2)
    det = jac[:, 0, 0] * jac[:, 1, 1] - jac[:, 0, 1] * jac[:, 1, 0]
    inv = np.empty_like(jac)
    inv[:, 0, 0] = jac[:, 1, 1]
    inv[:, 0, 1] = -jac[:, 0, 1]
    inv[:, 1, 0] = -jac[:, 1, 0]
    inv[:, 1, 1] = jac[:, 0, 0]
    inv /= det[:, None, None]
    return p[:, 0], inv, det


def _physical_gradients(dphi, jinv):
    # G[c, a, q, d] = sum_e dphi[a, q, e] * Jinv[c, e, d]
    return np.einsum("aqe,ced->caqd", dphi, jinv)


def _coo_to_csr(rows, cols, vals, n_rows, n_cols, canonical=False):
    """Deterministic COO -> CSR: entries sorted by (row, col), duplicates
    summed in input order -- or, with ``canonical``, in ascending order of
    their values, so that equal multisets of contributions give bitwise
    equal sums wherever they occur (translation-invariant assembly).
    ``vals`` may carry trailing value axes."""
    rows = rows.reshape(-1).astype(np.int64)
    cols = cols.reshape(-1).astype(np.int64)
    vals = vals.reshape(len(rows), -1)
    key = rows * n_cols + cols
    if canonical:
        order = np.lexsort(tuple(vals[:, k] for k in range(vals.shape[1] - 1, -1, -1)) + (key,))
    else:
        order = np.argsort(key, kind="stable")
    key = key[order]
    vals = vals[order]
    first = np.flatnonzero(np.concatenate(([True], key[1:] != key[:-1])))
    summed = np.add.reduceat(vals, first, axis=0)
    ukey = key[first]
    urow = ukey // n_cols
    col = (ukey % n_cols).astype(np.int32)
    rowptr = np.concatenate(([0], np.cumsum(np.bincount(urow, minlength=n_rows)))).astype(np.int64)
    return rowptr, col, summed


@dataclass
class StokesBlocks:
    """Raw (non-eliminated) Stokes blocks on one level, scalar-node form.

    ``rowptr/col`` is the scalar P2 pattern (n_nodes x n_nodes); ``m`` and
    ``k`` are the scalar mass and (mu-scaled) stiffness values on it.
    ``b_rowptr/b_col/b_val`` hold, per scalar node, the P1 columns and the
    (B_x, B_y) coefficient pair, where B[2n + d, q] = -<psi_q, d_d phi_n>
    (reference ``assemble_divergence``, ``fem.py:182-196``).
    """

    n_nodes: int
    n_p: int
    rowptr: np.ndarray
    col: np.ndarray
    m: np.ndarray
    k: np.ndarray
    b_rowptr: np.ndarray
    b_col: np.ndarray
    b_val: np.ndarray  # (nnz_b, ncomp): (B_x, B_y) in 2-D, (B_x, B_y, B_z) in 3-D
    # optional scalar-node coordinates (vertices, then edge midpoints): only a
    # locality hint for the K1 tile plan (k1tiles.py), never part of the maths
    node_xy: np.ndarray = None

    @property
    def ncomp(self):
        """Velocity components per scalar node (2; 3 for fem3d)."""
        return int(self.b_val.shape[1])

    @property
    def n_u(self):
        return self.ncomp * self.n_nodes

    @classmethod
    def from_vector(cls, M, K, B):
        """Scalar-node blocks from the reference's interleaved vector-P2 CSR
        ``BlockSystem`` (fem.py:99-113).  Requires M = M_P2 (x) I_2 and
        K = K_P2 (x) I_2 (true for the reference's assembly, fem.py:149-154);
        the scalar pattern is the union of M's and K's stored structure."""
        M, K, B = sp.csr_matrix(M), sp.csr_matrix(K), sp.csr_matrix(B)
        n_u, n_p = B.shape
        if n_u % 2 or M.shape != (n_u, n_u) or K.shape != (n_u, n_u):
            raise ValueError("inconsistent block dimensions")
        n = n_u // 2
        # The reference sums duplicate entries of the two components in
        # independent (scipy sort) orders, so the components may differ by an
        # ulp; the x-component values are taken.
        for A in (M, K):
            scale = max(abs(A).max(), 1e-300)
            if (abs(A[1::2, 1::2] - A[0::2, 0::2]).max() > 1e-14 * scale
                    or abs(A[0::2, 1::2]).max() > 0 or abs(A[1::2, 0::2]).max() > 0):
                raise ValueError("velocity block is not (scalar P2) x I_2")
        S = _structure(M[0::2, 0::2]) + _structure(K[0::2, 0::2])
        S = sp.csr_matrix(S)
        S.sort_indices()
        rows = np.repeat(np.arange(n), np.diff(S.indptr))
        m = np.asarray(M[0::2, 0::2][rows, S.indices]).ravel()
        k = np.asarray(K[0::2, 0::2][rows, S.indices]).ravel()
        T = sp.csr_matrix(_structure(B[0::2]) + _structure(B[1::2]))
        T.sort_indices()
        brows = np.repeat(np.arange(n), np.diff(T.indptr))
        bx = np.asarray(B[0::2][brows, T.indices]).ravel()
        by = np.asarray(B[1::2][brows, T.indices]).ravel()
        return cls(n_nodes=n, n_p=n_p, rowptr=S.indptr.astype(np.int64),
                   col=S.indices.astype(np.int32), m=m, k=k,
                   b_rowptr=T.indptr.astype(np.int64), b_col=T.indices.astype(np.int32),
                   b_val=np.column_stack([bx, by]))

    # Vector-P2 views in the reference's (interleaved) layout -- used by the
    # oracle, the coarse materialisation and API parity, never by kernels.
    def scalar_matrix(self, vals):
        return sp.csr_matrix((vals, self.col, self.rowptr),
                             shape=(self.n_nodes, self.n_nodes))

    @property
    def M(self):
        return sp.kron(self.scalar_matrix(self.m), sp.identity(self.ncomp), format="csr")

    @property
    def K(self):
        return sp.kron(self.scalar_matrix(self.k), sp.identity(self.ncomp), format="csr")

    @property
    def B(self):
        nc = self.ncomp
        rows = np.repeat(np.arange(self.n_nodes), np.diff(self.b_rowptr))
        r = np.concatenate([nc * rows + d for d in range(nc)])
        c = np.concatenate([self.b_col] * nc).astype(np.int64)
        v = np.concatenate([self.b_val[:, d] for d in range(nc)])
        return sp.csr_matrix((v, (r, c)), shape=(self.n_u, self.n_p))


def _structure(A):
    """0/1 matrix with A's stored (structural, incl. explicit zero) entries."""
    A = sp.csr_matrix(A, copy=True)
    A.data[:] = 1.0
    return A


@dataclass
class ConvectionBlocks:
    """Convection Jacobian on the scalar P2 pattern: one 2x2 block per entry.

    ``val[e, d, f]`` is J[2 n + d, 2 n' + f] for pattern entry e = (n, n').
    """

    n_nodes: int
    rowptr: np.ndarray
    col: np.ndarray
    val: np.ndarray  # (nnz, 2, 2)

    @classmethod
    def from_vector(cls, J, blocks):
        """2x2 blocks of a vector-P2 Jacobian (reference ``assemble_convection``
        output) on ``blocks``' scalar pattern; entries off the pattern must be 0."""
        J = sp.csr_matrix(J)
        rows = np.repeat(np.arange(blocks.n_nodes), np.diff(blocks.rowptr))
        col = blocks.col.astype(np.int64)
        val = np.empty((len(col), 2, 2))
        for d in range(2):
            for f in range(2):
                val[:, d, f] = np.asarray(J[2 * rows + d, 2 * col + f]).ravel()
        out = cls(blocks.n_nodes, blocks.rowptr, blocks.col, val)
        if abs(out.matrix - J).max() > 0:
            raise ValueError("Jacobian has entries outside the scalar P2 pattern")
        return out

    @property
    def matrix(self):
        rows = np.repeat(np.arange(self.n_nodes), np.diff(self.rowptr))
        comp = np.arange(2)
        r = np.broadcast_to(2 * rows[:, None, None] + comp[None, :, None], self.val.shape)
        c = np.broadcast_to(2 * self.col.astype(np.int64)[:, None, None] + comp[None, None, :],
                            self.val.shape)
        n = 2 * self.n_nodes
        return sp.csr_matrix((self.val.ravel(), (r.ravel(), c.ravel())), shape=(n, n))


class _CanonicalCells:
    """The mesh with every cell's vertices rotated (cyclically, orientation
    kept) to start at its lowest-then-leftmost vertex, so congruent cells
    get bitwise-identical element matrices (exact dyadic geometry)."""

    def __init__(self, mesh):
        p = mesh.vertices[mesh.cells]
        y, x = p[:, :, 1], p[:, :, 0]
        s = np.lexsort((x.T, y.T), axis=0)[0]             # lowest y, then lowest x
        rot = (s[:, None] + np.arange(3)[None, :]) % 3
        self.cells = np.take_along_axis(mesh.cells, rot, axis=1)
        self.cell_to_edges = np.take_along_axis(mesh.cell_to_edges, rot, axis=1)
        self.vertices = mesh.vertices
        self.num_vertices = mesh.num_vertices
        self.num_edges = mesh.num_edges


def node_coordinates(mesh):
    """Coordinates of the scalar P2 nodes: vertices, then edge midpoints."""
    v = np.asarray(mesh.vertices, dtype=np.float64)
    e = np.asarray(mesh.edges)
    return np.vstack([v, 0.5 * (v[e[:, 0]] + v[e[:, 1]])])


def assemble_blocks(mesh, mu=1.0):
    """Scalar-form M, K (times mu) and B for one mesh level.

    Translation-invariant: element matrices are computed on canonically
    rotated cells and duplicates are summed in value order, so patches with
    the same local geometry get bitwise-identical matrices (patch dedup)."""
    node_xy = node_coordinates(mesh)
    mesh = _CanonicalCells(mesh)
    nodes = p2_cell_nodes(mesh)
    n_nodes = mesh.num_vertices + mesh.num_edges
    _, jinv, det = _affine(mesh)

    pts, w = triangle_rule(DEG_MASS)
    phi, _ = p2_basis(pts)
    mref = np.einsum("q,aq,bq->ab", w, phi, phi)
    mloc = det[:, None, None] * mref

    pts, w = triangle_rule(DEG_STIFFNESS)
    _, dphi = p2_basis(pts)
    g = _physical_gradients(dphi, jinv)
    kloc = mu * np.einsum("q,caqd,cbqd->cab", w, g, g) * det[:, None, None]

    rows = np.repeat(nodes[:, :, None], 6, axis=2)
    cols = np.repeat(nodes[:, None, :], 6, axis=1)
    rowptr, col, mk = _coo_to_csr(rows, cols, np.stack([mloc, kloc], axis=-1),
                                  n_nodes, n_nodes, canonical=True)

    pts, w = triangle_rule(DEG_DIVERGENCE)
    _, dphi = p2_basis(pts)
    psi, _ = p1_basis(pts)
    g = _physical_gradients(dphi, jinv)
    # bloc[c, a, b, d] = -sum_q w_q psi_b(q) G[c, a, q, d] * det
    bloc = -np.einsum("q,bq,caqd->cabd", w, psi, g) * det[:, None, None, None]
    brows = np.repeat(nodes[:, :, None], 3, axis=2)
    bcols = np.repeat(mesh.cells[:, None, :], 6, axis=1)
    b_rowptr, b_col, b_val = _coo_to_csr(brows, bcols, bloc, n_nodes, mesh.num_vertices,
                                         canonical=True)

    return StokesBlocks(n_nodes=n_nodes, n_p=mesh.num_vertices,
                        rowptr=rowptr, col=col,
                        m=np.ascontiguousarray(mk[:, 0]),
                        k=np.ascontiguousarray(mk[:, 1]),
                        b_rowptr=b_rowptr, b_col=b_col,
                        b_val=np.ascontiguousarray(b_val.reshape(-1, 2)),
                        node_xy=node_xy)


def assemble_convection_jacobian(mesh, blocks, u):
    """Jacobian of <(u . grad) u, phi> at the vector-P2 coefficients ``u``.

    Both Newton terms (reference ``assemble_convection``, ``fem.py:199-242``):
    J[(a,d),(b,f)] = <phi_a phi_b, d_f u_d> + delta_df <phi_a, u . grad phi_b>.
    The result lives on ``blocks``' scalar pattern.
    """
    u = np.asarray(u, dtype=np.float64)
    if u.shape != (2 * blocks.n_nodes,):
        raise ValueError(f"velocity coefficient vector must have length {2 * blocks.n_nodes}")
    nodes = p2_cell_nodes(mesh)
    _, jinv, det = _affine(mesh)
    pts, w = triangle_rule(DEG_CONVECTION)
    phi, dphi = p2_basis(pts)
    g = _physical_gradients(dphi, jinv)
    uloc = u.reshape(-1, 2)[nodes]                       # (C, 6, comp)
    uq = np.einsum("cad,aq->cqd", uloc, phi)             # u at quad points
    gradu = np.einsum("cad,caqe->cqde", uloc, g)         # d_e u_d
    wpp = np.einsum("q,aq,bq->abq", w, phi, phi)
    t1 = np.einsum("abq,cqde->cabde", wpp, gradu)
    adv = np.einsum("cqf,cbqf->cqb", uq, g)              # u . grad phi_b
    t2 = np.einsum("q,aq,cqb->cab", w, phi, adv, optimize=True)
    jloc = t1 + t2[:, :, :, None, None] * np.eye(2)[None, None, None]
    jloc = jloc * det[:, None, None, None, None]
    rows = np.repeat(nodes[:, :, None], 6, axis=2)
    cols = np.repeat(nodes[:, None, :], 6, axis=1)
    rowptr, col, val = _coo_to_csr(rows, cols, jloc, blocks.n_nodes, blocks.n_nodes)
    if not (np.array_equal(rowptr, blocks.rowptr) and np.array_equal(col, blocks.col)):
        raise RuntimeError("convection pattern differs from the scalar P2 pattern")
    return ConvectionBlocks(blocks.n_nodes, rowptr, col, val.reshape(-1, 2, 2))


def assemble_convection_residual(mesh, blocks, u):
    """N(u)_(a,d) = <(u . grad) u_d, phi_a> (reference ``assemble_convection``
    with need="residual", fem.py:219-227), interleaved like u."""
    u = np.asarray(u, dtype=np.float64)
    nodes = p2_cell_nodes(mesh)
    _, jinv, det = _affine(mesh)
    pts, w = triangle_rule(DEG_CONVECTION)
    phi, dphi = p2_basis(pts)
    g = _physical_gradients(dphi, jinv)
    uloc = u.reshape(-1, 2)[nodes]
    uq = np.einsum("cad,aq->cqd", uloc, phi)
    gradu = np.einsum("cad,caqe->cqde", uloc, g)
    conv = np.einsum("cqe,cqde->cqd", uq, gradu)
    nloc = np.einsum("q,aq,cqd->cad", w, phi, conv, optimize=True) * det[:, None, None]
    out = np.zeros((blocks.n_nodes, 2))
    np.add.at(out, nodes.reshape(-1), nloc.reshape(-1, 2))
    return out.reshape(-1)


def prolongation(hierarchy, level, kind):
    """Scalar nested interpolation ``level`` -> ``level + 1`` (CSR, fine x coarse).

    ``kind`` is "p2" or "p1".  Each fine node takes the coarse basis values
    of the parent of the first fine cell containing it; entries with
    |value| <= 1e-12 are dropped (reference ``prolongation``, ``fem.py:255-301``).
    """
    if not isinstance(hierarchy, MeshHierarchy):
        raise TypeError("expected a MeshHierarchy")
    if not 0 <= level < hierarchy.num_levels - 1:
        raise ValueError(f"no refinement above level {level}")
    coarse = hierarchy.levels[level]
    fine = hierarchy.levels[level + 1]
    parent = hierarchy.cell_parent[level]
    if kind == "p2":
        fnodes, cnodes = p2_cell_nodes(fine), p2_cell_nodes(coarse)
        fcoords = p2_node_coords(fine)
        nf, nc = fine.num_vertices + fine.num_edges, coarse.num_vertices + coarse.num_edges
        basis = p2_basis
    elif kind == "p1":
        fnodes, cnodes = fine.cells, coarse.cells
        fcoords = fine.vertices
        nf, nc = fine.num_vertices, coarse.num_vertices
        basis = p1_basis
    else:
        raise ValueError(f"unknown space kind {kind!r}")

    # First (cell, local slot) occurrence of every fine node.
    flat = fnodes.ravel()
    first = np.full(nf, -1, dtype=np.int64)
    order = np.argsort(flat, kind="stable")
    uniq_first = np.concatenate(([True], flat[order][1:] != flat[order][:-1]))
    first[flat[order][uniq_first]] = order[uniq_first]
    if np.any(first < 0):
        raise RuntimeError("fine node not covered by any cell")
    fcell = first // fnodes.shape[1]
    pc = parent[fcell]
    origin, jinv, _ = _affine(coarse)
    ref = np.einsum("nde,ne->nd", jinv[pc], fcoords - origin[pc])
    vals = basis(ref)[0].T                          # (nf, nb)
    cols = cnodes[pc]                                # (nf, nb)
    rows = np.repeat(np.arange(nf)[:, None], vals.shape[1], axis=1)
    keep = np.abs(vals) > 1e-12
    P = sp.csr_matrix((vals[keep], (rows[keep], cols[keep])), shape=(nf, nc))
    P.sort_indices()
    return P


def velocity_boundary_nodes(mesh):
    """Scalar P2 nodes on the boundary, ascending."""
    return np.sort(np.concatenate([
        np.flatnonzero(mesh.boundary_vertex_flags),
        mesh.num_vertices + np.flatnonzero(mesh.boundary_edge_flags),
    ])).astype(np.int64)


def velocity_boundary_dofs(mesh):
    """Both components of every boundary node (reference ``fem.py:420-427``)."""
    n = velocity_boundary_nodes(mesh)
    return np.sort(np.concatenate([2 * n, 2 * n + 1]))


def interpolate_velocity(mesh, func):
    """Nodal interpolant of ``func(points) -> (N, 2)`` as interleaved coefficients."""
    vals = np.asarray(func(p2_node_coords(mesh)), dtype=np.float64)
    if vals.shape != (mesh.num_vertices + mesh.num_edges, 2):
        raise ValueError("vector function must return (N, 2) values")
    return vals.ravel()
