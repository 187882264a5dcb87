"""Taylor-Hood P2-P1 on Kuhn tetrahedra in scalar-node form -- BASELINE
config 4 (3-D unsteady Stokes).  Host-side setup only; the hot path runs on
the same kernels as in 2-D with three velocity components per scalar node.

The reference has no 3-D discretisation, so this module
follows the 2-D conventions of ``fem.py`` (itself the reference's
``fem.py:128-196``): scalar P2 mass and (mu-scaled) stiffness on the scalar
P2 pattern (M_vec = M_P2 (x) I_3), one (B_x, B_y, B_z) triple per (P2 node,
P1 node) with B[3n + d, q] = -<psi_q, d_d phi_n>, vertices then edge
midpoints, components interleaved per node.  One collapsed Gauss-Jacobi
(conical product) rule of degree 5 serves all blocks (mass needs 4).
"""

from functools import lru_cache

import numpy as np
import scipy.sparse as sp
from scipy.special import roots_jacobi, roots_legendre

from .fem import StokesBlocks, _coo_to_csr
from .mesh3d import TET_EDGES, build_hierarchy3d, locate_kuhn

__all__ = ["tet_rule", "p1_basis3", "p2_basis3", "assemble_blocks3d", "prolongation3d",
           "velocity_boundary_nodes3d", "velocity_boundary_dofs3d", "p2_node_coords3d",
           "Discretization3D"]


@lru_cache(maxsize=None)
def tet_rule(n=3):
    """Conical product rule with n points per direction on the reference
    tetrahedron {x, y, z >= 0, x + y + z <= 1}; exact to degree 2n - 1."""
    ga, wa = roots_jacobi(n, 2, 0)
    gb, wb = roots_jacobi(n, 1, 0)
    gc, wc = roots_legendre(n)
    a, wa = 0.5 * (ga + 1.0), wa / 8.0
    b, wb = 0.5 * (gb + 1.0), wb / 4.0
    c, wc = 0.5 * (gc + 1.0), wc / 2.0
    A, B, Cc = np.meshgrid(a, b, c, indexing="ij")
    W = (wa[:, None, None] * wb[None, :, None] * wc[None, None, :]).ravel()
    A, B, Cc = A.ravel(), B.ravel(), Cc.ravel()
    x = A
    y = B * (1.0 - A)
    z = Cc * (1.0 - A) * (1.0 - B)
    pts = np.column_stack([x, y, z])
    pts.setflags(write=False)
    W.setflags(write=False)
    return pts, W


def _bary3(points):
    x, y, z = points[:, 0], points[:, 1], points[:, 2]
    lam = np.stack([1.0 - x - y - z, x, y, z])
    dlam = np.array([[-1.0, -1.0, -1.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [0.0, 0.0, 1.0]])
    return lam, dlam


def p1_basis3(points):
    """P1 values (4, Q) and gradients (4, 3)."""
    return _bary3(points)


def _p2_from_bary(lam, dlam):
    q = lam.shape[1]
    phi = np.empty((10, q))
    dphi = np.empty((10, q, dlam.shape[1]))
    for k in range(4):
        phi[k] = lam[k] * (2.0 * lam[k] - 1.0)
        dphi[k] = (4.0 * lam[k] - 1.0)[:, None] * dlam[k]
    for e, (i, j) in enumerate(TET_EDGES):
        phi[4 + e] = 4.0 * lam[i] * lam[j]
        dphi[4 + e] = 4.0 * (lam[i][:, None] * dlam[j] + lam[j][:, None] * dlam[i])
    return phi, dphi


def p2_basis3(points):
    """P2 values (10, Q) and gradients (10, Q, 3): the four vertices, then
    the edge midpoints in TET_EDGES order (the numbering behind
    ``cell_to_edges``)."""
    return _p2_from_bary(*_bary3(points))


def p2_cell_nodes3d(mesh):
    return np.hstack([mesh.cells, mesh.num_vertices + mesh.cell_to_edges])


def p2_node_coords3d(mesh):
    ev = mesh.vertices[mesh.edges]
    return np.vstack([mesh.vertices, 0.5 * (ev[:, 0] + ev[:, 1])])


def _affine3(mesh):
    p = mesh.vertices[mesh.cells]
    jac = np.stack([p[:, 1] - p[:, 0], p[:, 2] - p[:, 0], p[:, 3] - p[:, 0]], axis=2)
    det = np.linalg.det(jac)
    inv = np.linalg.inv(jac)
    return p[:, 0], inv, det


def assemble_blocks3d(mesh, mu=1.0):
    """Scalar-node Stokes blocks (M, mu K on the scalar P2 pattern; B triples)."""
    pts, w = tet_rule(3)
    phi, dphi = p2_basis3(pts)
    psi, _ = p1_basis3(pts)
    _, jinv, det = _affine3(mesh)
    vol = np.abs(det)
    nodes = p2_cell_nodes3d(mesh)                                   # (C, 10)
    C = len(nodes)
    n_nodes = mesh.num_vertices + mesh.num_edges
    # G[c, a, q, d] = sum_e dphi[a, q, e] Jinv[c, e, d]
    G = np.einsum("aqe,ced->caqd", dphi, jinv)
    mref = np.einsum("q,aq,bq->ab", w, phi, phi)
    Me = vol[:, None, None] * mref[None]
    Ke = mu * np.einsum("q,caqd,cbqd->cab", w, G, G) * vol[:, None, None]
    Be = -np.einsum("q,vq,caqd->cavd", w, psi, G) * vol[:, None, None, None]   # (C, 10, 4, 3)
    rows = np.repeat(nodes[:, :, None], 10, axis=2)
    cols = np.repeat(nodes[:, None, :], 10, axis=1)
    rowptr, col, mk = _coo_to_csr(rows, cols, np.stack([Me, Ke], axis=-1), n_nodes, n_nodes,
                                  canonical=True)
    brows = np.repeat(nodes[:, :, None], 4, axis=2)
    bcols = np.repeat(mesh.cells[:, None, :], 10, axis=1)
    b_rowptr, b_col, bv = _coo_to_csr(brows, bcols, Be, n_nodes, mesh.num_vertices,
                                      canonical=True)
    return StokesBlocks(n_nodes=n_nodes, n_p=mesh.num_vertices, rowptr=rowptr, col=col,
                        m=mk[:, 0].copy(), k=mk[:, 1].copy(), b_rowptr=b_rowptr, b_col=b_col,
                        b_val=bv.reshape(-1, 3).copy())


def prolongation3d(coarse, fine, kind):
    """Scalar nested interpolation coarse -> fine (CSR, fine x coarse): each
    fine node takes the coarse basis values at its position (|v| <= 1e-12
    dropped, as the 2-D ``fem.prolongation``)."""
    if kind == "p2":
        pts = p2_node_coords3d(fine)
        cn = p2_cell_nodes3d(coarse)
        nc = coarse.num_vertices + coarse.num_edges
    elif kind == "p1":
        pts = fine.vertices
        cn = coarse.cells
        nc = coarse.num_vertices
    else:
        raise ValueError(f"unknown space kind {kind!r}")
    cell, lam = locate_kuhn(coarse.n, pts)
    if kind == "p2":
        dl = np.eye(4)
        vals = _p2_from_bary(lam.T, dl)[0].T                    # (N, 10)
    else:
        vals = lam
    cols = cn[cell]
    rows = np.repeat(np.arange(len(pts))[:, None], vals.shape[1], axis=1)
    keep = np.abs(vals) > 1e-12
    P = sp.csr_matrix((vals[keep], (rows[keep], cols[keep])), shape=(len(pts), nc))
    P.sum_duplicates()
    P.sort_indices()
    return P


def velocity_boundary_nodes3d(mesh):
    return np.sort(np.concatenate([
        np.flatnonzero(mesh.boundary_vertex_flags),
        mesh.num_vertices + np.flatnonzero(mesh.boundary_edge_flags)])).astype(np.int64)


def velocity_boundary_dofs3d(mesh):
    n = velocity_boundary_nodes3d(mesh)
    return np.sort(np.concatenate([3 * n, 3 * n + 1, 3 * n + 2]))


class Discretization3D:
    """BASELINE config 4 setup: Kuhn meshes n0 * 2^l of the unit cube, P2-P1
    blocks, transfers; ``build_mg`` as the 2-D ``Discretization``."""

    def __init__(self, n0, level, mu=1.0):
        from .transfer import StageTransfer  # noqa: F401  (import check)
        self.hier = build_hierarchy3d(n0, level)
        self.mu = float(mu)
        self.blocks = [assemble_blocks3d(m, mu) for m in self.hier.levels]
        self.cdofs = [velocity_boundary_dofs3d(m) for m in self.hier.levels]
        self.cnodes = []
        for m, blk in zip(self.hier.levels, self.blocks):
            mask = np.zeros(blk.n_nodes, dtype=bool)
            mask[velocity_boundary_nodes3d(m)] = True
            self.cnodes.append(mask)
        self._scalar_prolong = [
            (prolongation3d(self.hier.levels[k], self.hier.levels[k + 1], "p2"),
             prolongation3d(self.hier.levels[k], self.hier.levels[k + 1], "p1"))
            for k in range(self.hier.num_levels - 1)]
        self._stage_prolong = {}

    @property
    def num_levels(self):
        return self.hier.num_levels

    @property
    def fine_mesh(self):
        return self.hier.levels[-1]

    def stage_prolong(self, level, r):
        from .transfer import StageTransfer
        key = (level, r)
        if key not in self._stage_prolong:
            p2, p1 = self._scalar_prolong[level - 1]
            self._stage_prolong[key] = StageTransfer(p2, p1, r, self.cnodes[level],
                                                     self.cnodes[level - 1], ncomp=3)
        return self._stage_prolong[key]

    def build_mg(self, tableau, dt, smoother, mg_levels=None, convection=None, use_graph=False,
                 patch_mode="auto"):
        from .discretization import Discretization
        if convection is not None:
            raise ValueError("3-D operators carry no convection")
        return Discretization.build_mg(self, tableau, dt, smoother, mg_levels=mg_levels,
                                       use_graph=use_graph, patch_mode=patch_mode)
