"""3-D extension (BASELINE config 4): Kuhn meshes, P2-P1
tetrahedral assembly, nested transfers and patch tables (CPU).  The
reference has no 3-D discretisation: these checks pin the setup
against exact properties, and the patch tables against the oracle's loop
restatement of the reference's patch construction (solvers.py:132-166)."""

import numpy as np
import pytest

from oracle.irk_vanka_oracle import OracleStageOperator, oracle_patch_indices


def test_tet_rule_and_mesh():
    from paper_2202_07381_b200.fem3d import tet_rule
    from paper_2202_07381_b200.mesh3d import kuhn_cube
    p, w = tet_rule(3)
    assert abs(w.sum() - 1 / 6) < 1e-15
    # exact to degree 5: int x^2 y z = 2! 1! 1! / 7!
    assert abs(np.dot(w, p[:, 0] ** 2 * p[:, 1] * p[:, 2]) - 2 / 5040) < 1e-17
    m = kuhn_cube(3)
    P = m.vertices[m.cells]
    vol = np.abs(np.linalg.det(np.stack([P[:, 1] - P[:, 0], P[:, 2] - P[:, 0],
                                         P[:, 3] - P[:, 0]], 2))) / 6
    assert abs(vol.sum() - 1.0) < 1e-14 and np.allclose(vol, vol[0])
    assert m.num_vertices == 64 and m.num_cells == 6 * 27
    # Euler characteristic of a ball: V - E + F - C = 1
    faces = set()
    for c in m.cells:
        for drop in range(4):
            faces.add(tuple(sorted(np.delete(c, drop))))
    assert m.num_vertices - m.num_edges + len(faces) - m.num_cells == 1


def test_blocks_and_transfers_exact():
    from paper_2202_07381_b200.fem3d import (assemble_blocks3d, p2_node_coords3d,
                                             prolongation3d)
    from paper_2202_07381_b200.mesh3d import kuhn_cube
    mc, mf = kuhn_cube(1), kuhn_cube(2)
    bf, bc = assemble_blocks3d(mf), assemble_blocks3d(mc)
    Mf, Kf = bf.scalar_matrix(bf.m), bf.scalar_matrix(bf.k)
    one = np.ones(bf.n_nodes)
    X = p2_node_coords3d(mf)
    assert abs(one @ Mf @ one - 1.0) < 1e-14
    assert abs(one @ Mf @ X[:, 0] - 0.5) < 1e-14
    assert np.abs(Kf @ one).max() < 1e-13
    # sum_q (B^T u)_q = -int div u for u = (x, 2y, -z): -(1 + 2 - 1) = -2
    u = np.column_stack([X[:, 0], 2 * X[:, 1], -X[:, 2]]).ravel()
    assert abs((bf.B.T @ u).sum() + 2.0) < 1e-13
    P2 = prolongation3d(mc, mf, "p2")
    P1 = prolongation3d(mc, mf, "p1")
    f = lambda Y: Y[:, 0] ** 2 + Y[:, 1] * Y[:, 2] - Y[:, 2]   # noqa: E731
    assert np.abs(P2 @ f(p2_node_coords3d(mc)) - f(X)).max() < 1e-14
    g = lambda Y: 1 + Y[:, 0] - 2 * Y[:, 1] + 3 * Y[:, 2]       # noqa: E731
    assert np.abs(P1 @ g(mc.vertices) - g(mf.vertices)).max() < 1e-14
    Mc = bc.scalar_matrix(bc.m)
    assert abs(P2.T @ Mf @ P2 - Mc).max() < 1e-15


@pytest.mark.parametrize("family,stages", [("radauiia", 2), ("gauss", 2)])
def test_patch_tables_match_oracle_and_operator(family, stages):
    from paper_2202_07381_b200 import tableau_lookup
    from paper_2202_07381_b200.fem3d import Discretization3D
    from paper_2202_07381_b200.patches import build_patch_tables
    from paper_2202_07381_b200.stages import StageSystem
    disc = Discretization3D(2, 1)
    tab = tableau_lookup(family, stages)
    blk, mesh = disc.blocks[1], disc.hier.levels[1]
    S = StageSystem(blk, tab, 1 / 32, disc.cdofs[1])
    t = build_patch_tables(mesh, S.n_nodes, S.n_p, S.r, S.node_constrained, ncomp=3)
    op = OracleStageOperator(blk.M, blk.K, blk.B, tab.A, 1 / 32, disc.cdofs[1])
    _, idxs = oracle_patch_indices(mesh.cells, mesh.cell_to_edges, mesh.num_vertices, op,
                                   ncomp=3)
    pos = t.patch_of_vertex()
    for v in range(mesh.num_vertices):
        assert np.array_equal(idxs[v], t.idx[t.idx_off[pos[v]]:t.idx_off[pos[v] + 1]])
    assert t.max_m == 2 * (3 * 65 + 1)          # interior vertex star: 65 P2 nodes
    x = np.random.default_rng(0).standard_normal(S.dim)
    A = S.materialize(limit=10 ** 5)
    assert np.abs(A @ x - op.matvec(x)).max() <= 1e-15 * np.abs(op.matvec(x)).max() * 100
