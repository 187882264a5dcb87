"""Host setup parity (CPU only): mesh numbering, scalar-node assembly,
transfers, boundary DoFs and the bit-exact Vanka patch index tables."""

import hashlib
import json
import os

import numpy as np
import pytest
import scipy.sparse as sp

from harness import GOLDEN, setup
from paper_2202_07381_b200 import fem
from paper_2202_07381_b200.mesh import build_hierarchy, diagonal_grid, refine_red
from paper_2202_07381_b200.patches import build_patch_tables
from paper_2202_07381_b200.stages import StageSystem
from paper_2202_07381_b200.tableaux import registry_keys, tableau_lookup


@pytest.fixture(scope="module")
def asm():
    return np.load(os.path.join(GOLDEN, "assembly.npz"))


@pytest.mark.parametrize("grid", ["diagonal", "crossed"])
def test_assembly_matches_reference(asm, grid):
    h = build_hierarchy(2, 1, grid)
    m = h.levels[1]
    blk = fem.assemble_blocks(m, mu=0.7)
    u = asm[f"{grid}_u"]
    J = fem.assemble_convection_jacobian(m, blk, u).matrix
    mats = {"M": blk.M, "K": blk.K, "B": blk.B, "J": J,
            "P2": fem.prolongation(h, 0, "p2"), "P1": fem.prolongation(h, 0, "p1")}
    for name, A in mats.items():
        ref = asm[f"{grid}_{name}"]
        assert A.shape == ref.shape
        err = np.max(np.abs(A.toarray() - ref)) / max(1e-300, np.max(np.abs(ref)))
        assert err <= 1e-14, (name, err)
    assert np.array_equal(fem.velocity_boundary_dofs(m), asm[f"{grid}_cdofs"])


def test_refinement_numbering_rules():
    m = diagonal_grid(3)
    f, parent = refine_red(m)
    # coarse vertices keep their indices, midpoint V + e bisects edge e
    assert np.array_equal(f.vertices[:m.num_vertices], m.vertices)
    mids = 0.5 * (m.vertices[m.edges[:, 0]] + m.vertices[m.edges[:, 1]])
    assert np.array_equal(f.vertices[m.num_vertices:], mids)
    assert np.array_equal(parent, np.repeat(np.arange(m.num_cells), 4))
    # edges sorted lexicographically, local edge k opposite vertex k
    assert np.all(np.diff(f.edges[:, 0] * f.num_vertices + f.edges[:, 1]) > 0)
    for c in range(0, f.num_cells, 7):
        for k in range(3):
            e = f.edges[f.cell_to_edges[c, k]]
            assert set(e) == set(np.delete(f.cells[c], k))


@pytest.mark.parametrize("name", ["cfg1", "s3", "ns", "crossed"])
def test_patch_indices_bit_exact(name):
    with open(os.path.join(GOLDEN, f"{name}.json")) as fh:
        meta = json.load(fh)
    disc, tab, conv, case = setup(name)
    for k, (mesh, blk) in enumerate(zip(disc.hier.levels, disc.blocks)):
        t = build_patch_tables(mesh, blk.n_nodes, blk.n_p, tab.r, disc.cnodes[k])
        pos = t.patch_of_vertex()
        hh = hashlib.sha256()
        for v in range(t.num_patches):
            q = pos[v]
            hh.update(t.idx[t.idx_off[q]:t.idx_off[q + 1]].astype(np.int64).tobytes())
            hh.update(b"|")
        assert hh.hexdigest() == meta["patch_index_sha256"][k]
        sizes = {str(int(m)): int(c) for m, c in zip(*np.unique(t.sizes, return_counts=True))}
        assert sizes == meta["patch_sizes"][k]
        # owner map is the exact inverse of the gather list
        assert t.dof_ptr[-1] == t.total_m
        assert np.array_equal(t.idx[t.dof_pos], np.repeat(np.arange(t.dim), np.diff(t.dof_ptr)))
        # the K3m fragment layout (modal.fragment_layout): same owner entries,
        # same per-DoF order, even-aligned patches, node-major rows
        from paper_2202_07381_b200.modal import fragment_layout
        offp, idx_f, dpos_f = fragment_layout(t, 2)
        assert np.all(offp % 2 == 0)
        assert np.array_equal(idx_f[dpos_f], t.idx[t.dof_pos])
        q = int(np.argmax(t.sizes))
        kq = int(t.node_off[q + 1] - t.node_off[q])
        seg = idx_f[offp[q]:offp[q] + t.sizes[q]]
        ref = t.idx[t.idx_off[q]:t.idx_off[q + 1]]
        blk = 2 * kq + 1
        assert seg[2 * tab.r * 3 + 1 * tab.r + 0] == ref[0 * blk + 2 * 3 + 1]   # node 3, comp 1, a 0
        assert np.array_equal(seg[2 * tab.r * kq:], ref[blk - 1::blk])          # pressures
        # group order: sizes ascending, vertices ascending within a size
        assert np.all(np.diff(t.sizes) >= 0)
        same = np.diff(t.sizes) == 0
        assert np.all(np.diff(t.order)[same] > 0)


def test_cfg1_multiplicity_histogram():
    disc, tab, conv, case = setup("cfg1")
    m, blk = disc.fine_mesh, disc.blocks[-1]
    t = build_patch_tables(m, blk.n_nodes, blk.n_p, tab.r, disc.cnodes[-1])
    hist = dict(zip(*np.unique(t.multiplicity, return_counts=True)))
    assert {int(k): int(v) for k, v in hist.items()} == {0: 1024, 1: 2178, 4: 12032, 7: 3844}


def test_cfg2_patch_sizes():
    """BASELINE config 2 fine level."""
    disc, tab, conv, case = setup("cfg2")
    m, blk = disc.fine_mesh, disc.blocks[-1]
    t = build_patch_tables(m, blk.n_nodes, blk.n_p, tab.r, disc.cnodes[-1])
    assert t.dim == 1_777_161 and t.num_patches == 66_049
    assert t.total_m == 7_635_501
    assert int(np.sum(t.sizes.astype(np.int64) ** 2)) == 888_229_449
    hist = {int(a): int(b) for a, b in zip(*np.unique(t.sizes, return_counts=True))}
    assert hist == {117: 64_009, 99: 1_012, 45: 1_016, 87: 2, 81: 2, 33: 4, 27: 2, 9: 2}
    assert len(blk.col) == 3_018_753


def test_stage_system_host_views_match_oracle():
    from oracle.irk_vanka_oracle import OracleStageOperator
    disc, tab, conv, case = setup("ns")
    k = 1
    blk = disc.blocks[k]
    S = StageSystem(blk, tab, case["dt"], disc.cdofs[k], conv[k])
    op = OracleStageOperator(blk.M, blk.K, blk.B, tab.A, case["dt"], disc.cdofs[k],
                             [J.matrix for J in conv[k]])
    A1 = S.materialize()
    A2 = op.materialize()
    assert abs(A1 - A2).max() <= 1e-15 * abs(A2).max()
    assert np.array_equal(S.constrained_stage_dofs(), op.constrained_stage_dofs())


def test_partial_node_constraint_rejected():
    disc, tab, conv, case = setup("crossed")
    c = disc.cdofs[0]
    with pytest.raises(ValueError):
        StageSystem(disc.blocks[0], tab, 0.1, c[::2])  # x components only


def test_tableaux_bitwise_equal_reference():
    """Every (family, stages) of the reference registry, including the
    non-diagonalisable DIRK-Alexander(3), with the reference's exact bits
    (tests/golden/tableaux.json, tests/golden/make_tableaux.py)."""
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "tableaux.json")) as fh:
        gold = json.load(fh)
    for key, want in gold.items():
        fam, s = key.split(":")
        t = tableau_lookup(fam, int(s))
        for k in ("A", "b", "c"):
            got = [float(v).hex() for v in np.asarray(getattr(t, k), float).ravel()]
            assert got == want[k], (key, k)
    for alias in ("alexander", "dirk3", "DIRK_Alexander"):
        assert np.array_equal(tableau_lookup(alias, 3).A, tableau_lookup("dirk-alexander", 3).A)


def test_tableaux_consistent():
    for fam, s in registry_keys():
        t = tableau_lookup(fam, s)
        assert t.r == s
        assert abs(t.b.sum() - 1.0) <= 1e-14
        assert np.max(np.abs(t.A.sum(axis=1) - t.c)) <= 1e-14
    with pytest.raises(KeyError):
        tableau_lookup("gauss", 7)


def test_coarse_tiles_reconstruct_factors():
    from paper_2202_07381_b200.solvers import tile_factor
    rng = np.random.default_rng(0)
    n = 75
    L = sp.csc_matrix(np.tril(rng.standard_normal((n, n)) * (rng.random((n, n)) < 0.2), -1)
                      + np.eye(n))
    U = sp.csc_matrix(np.triu(rng.standard_normal((n, n)) * (rng.random((n, n)) < 0.2), 1)
                      + np.diag(rng.uniform(1, 2, n)))
    for F, lower in ((L, True), (U, False)):
        colptr, row, tiles, diag, nb = tile_factor(F, lower)
        D = np.zeros((nb * 32, nb * 32))
        for K in range(nb):
            D[K * 32:(K + 1) * 32, K * 32:(K + 1) * 32] = diag[K * 1024:(K + 1) * 1024] \
                .reshape(32, 32).T
            for t in range(colptr[K], colptr[K + 1]):
                I = row[t]
                D[I * 32:(I + 1) * 32, K * 32:(K + 1) * 32] = tiles[t * 1024:(t + 1) * 1024] \
                    .reshape(32, 32).T
        Fd = F.toarray()
        if not lower:   # the upper diagonal is stored as exact reciprocals
            assert np.array_equal(np.diag(D)[:n], 1.0 / np.diag(Fd))
            D[np.arange(n), np.arange(n)] = np.diag(Fd)
        assert np.array_equal(D[:n, :n], Fd)
        assert np.array_equal(np.diag(D)[n:], np.ones(nb * 32 - n))


@pytest.mark.parametrize("grid", ["diagonal", "crossed"])
def test_blocks_from_reference_vector_matrices(asm, grid):
    """Integration path: the reference's interleaved vector CSR blocks map
    onto the scalar-node form."""
    M = sp.csr_matrix(asm[f"{grid}_M"])
    K = sp.csr_matrix(asm[f"{grid}_K"])
    B = sp.csr_matrix(asm[f"{grid}_B"])
    blk = fem.StokesBlocks.from_vector(M, K, B)
    assert abs(blk.M - M).max() <= 1e-15 * abs(M).max()
    assert abs(blk.K - K).max() <= 1e-15 * abs(K).max()
    assert abs(blk.M[0::2, 0::2] - M[0::2, 0::2]).max() == 0
    assert abs(blk.B - B).max() == 0
    J = sp.csr_matrix(asm[f"{grid}_J"])
    Jb = fem.ConvectionBlocks.from_vector(J, blk)
    assert abs(Jb.matrix - J).max() == 0


@pytest.mark.parametrize("grid", ["diagonal", "crossed"])
def test_convection_residual_matches_reference(asm, grid):
    h = build_hierarchy(2, 1, grid)
    m = h.levels[1]
    blk = fem.assemble_blocks(m, mu=0.7)
    N = fem.assemble_convection_residual(m, blk, asm[f"{grid}_u"])
    ref = asm[f"{grid}_N"]
    assert np.max(np.abs(N - ref)) <= 1e-14 * np.max(np.abs(ref))
