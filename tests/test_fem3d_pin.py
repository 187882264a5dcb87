"""Pin of the 3-D discretisation (BASELINE config 4) independent of this
repo's assembly code: ``fem3d.assemble_blocks3d`` (collapsed Gauss-Jacobi
quadrature, vectorised einsum, edge-numbered nodes) against
``oracle/fem3d_oracle.py`` (exact barycentric-monomial integrals, symbolic
P2 basis, geometric node lookup, a python loop over cells).  The reference
has no 3-D discretisation, so agreement of two independent
constructions plus exact identities of the continuous forms is the pin."""

import numpy as np
import pytest
import scipy.sparse as sp

from oracle.fem3d_oracle import exact_monomial_integral, oracle_blocks3d
from paper_2202_07381_b200.fem3d import assemble_blocks3d, p2_node_coords3d, tet_rule
from paper_2202_07381_b200.mesh3d import kuhn_cube


def _scalar(blk, vals):
    return sp.csr_matrix((vals, blk.col, blk.rowptr), shape=(blk.n_nodes, blk.n_nodes))


@pytest.mark.parametrize("n,mu", [(1, 1.0), (2, 1.0), (3, 0.37)])
def test_blocks_match_exact_cell_loop(n, mu):
    mesh = kuhn_cube(n)
    blk = assemble_blocks3d(mesh, mu)
    M, K, B = oracle_blocks3d(mesh.vertices, mesh.cells, p2_node_coords3d(mesh), mu)
    for name, got, ref in (("M", _scalar(blk, blk.m), M), ("K", _scalar(blk, blk.k), K),
                           ("B", blk.B, B)):
        d = abs(got - ref).max()
        assert d <= 1e-14 * abs(ref).max(), (name, d)
        # same structural pattern (no dropped or spurious couplings)
        s_got = sp.csr_matrix(got)
        s_got.eliminate_zeros()
        s_ref = sp.csr_matrix(ref)
        s_ref.data[np.abs(s_ref.data) < 1e-15 * abs(ref).max()] = 0
        s_ref.eliminate_zeros()
        assert (abs(s_got) > 0).nnz >= (abs(s_ref) > 0).nnz, name


def test_exact_identities_of_the_forms():
    """Properties of the continuous forms the discrete blocks must keep:
    sum of the mass = |Omega|; K annihilates constants (and linears in the
    interior); B^T of a constant field vanishes in the interior; the
    discrete divergence of a linear field integrates exactly."""
    mesh = kuhn_cube(3)
    blk = assemble_blocks3d(mesh, 1.0)
    xyz = p2_node_coords3d(mesh)
    M, K = _scalar(blk, blk.m), _scalar(blk, blk.k)
    assert abs(M.sum() - 1.0) < 1e-13
    assert abs(K @ np.ones(blk.n_nodes)).max() < 1e-12
    interior = np.flatnonzero(np.all((xyz > 1e-12) & (xyz < 1 - 1e-12), axis=1))
    lin = 0.3 * xyz[:, 0] - 1.7 * xyz[:, 1] + 0.9 * xyz[:, 2]
    assert abs((K @ lin)[interior]).max() < 1e-12
    # u = (x, 2y, -z): div u = 2, so sum_n B[:, q] . u(x_n) = -int psi_q * 2
    u = np.column_stack([xyz[:, 0], 2 * xyz[:, 1], -xyz[:, 2]]).ravel()
    Bu = blk.B.T @ u
    # int psi_q over the mesh: each tet contributes |T| / 4 to each vertex
    P = mesh.vertices[mesh.cells]
    vol = np.abs(np.linalg.det(np.stack([P[:, 1] - P[:, 0], P[:, 2] - P[:, 0],
                                         P[:, 3] - P[:, 0]], 2))) / 6
    hat = np.zeros(blk.n_p)
    np.add.at(hat, mesh.cells.ravel(), np.repeat(vol / 4, 4))
    assert np.abs(Bu + 2.0 * hat).max() < 1e-13


def test_exact_integration_formula():
    """The closed form used by the oracle against the repo's quadrature."""
    p, w = tet_rule(3)
    lam = np.stack([1 - p.sum(1), p[:, 0], p[:, 1], p[:, 2]])
    for a in [(0, 0, 0, 0), (2, 0, 0, 0), (1, 1, 1, 0), (2, 1, 0, 1), (1, 1, 1, 2)]:
        q = 6.0 * np.dot(w, np.prod([lam[i] ** a[i] for i in range(4)], axis=0))
        assert abs(q - exact_monomial_integral(a)) < 1e-15
