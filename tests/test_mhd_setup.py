"""MHD (BASELINE config 5) host setup on CPU: the vectorised assembly against
the oracle's independent cell-loop restatement of the weak form, boundary
conditions, saddle structure, vertex-star patch tables (bit-exact against
the oracle's loop construction) and transfers.  Parity is unpinned -- the
reference has no MHD (oracle/general_oracle.py)."""

import numpy as np
import pytest
import scipy.sparse as sp

from harness import MHD_CONFIGS, mhd_oracle_levels, mhd_setup
from oracle.general_oracle import oracle_mhd_apply
from paper_2202_07381_b200 import tableau_lookup
from paper_2202_07381_b200.discretization import streamfunction_velocity
from paper_2202_07381_b200.fem import p2_node_coords
from paper_2202_07381_b200.mesh import build_hierarchy
from paper_2202_07381_b200.mhd import (MHDParams, assemble_mhd, mhd_boundary_dofs,
                                       mhd_magnetic_state, mhd_prolongation)


def _unconstrained(mesh, params):
    rowptr, col, m, l, cm = assemble_mhd(mesh, params, constrained=np.zeros(0, dtype=np.int64))
    n = len(cm)
    return (sp.csr_matrix((m, col, rowptr), shape=(n, n)),
            sp.csr_matrix((l, col, rowptr), shape=(n, n)))


@pytest.mark.parametrize("grid", ["diagonal", "crossed"])
@pytest.mark.parametrize("params", [(100.0, 100.0, 1.0), (0.7, 3.0, 2.5)])
def test_assembly_matches_cell_loop_oracle(grid, params):
    mesh = build_hierarchy(4 if grid == "diagonal" else 2, 0, grid).levels[0]
    M, L = _unconstrained(mesh, MHDParams(*params))
    xy = p2_node_coords(mesh)
    rng = np.random.default_rng(3)
    for _ in range(2):
        x = rng.uniform(-1, 1, L.shape[0])
        y = oracle_mhd_apply(mesh, streamfunction_velocity(xy), mhd_magnetic_state(xy),
                             *params, x)
        assert np.linalg.norm(L @ x - y) <= 1e-13 * np.linalg.norm(y)


def test_mass_and_saddle_structure():
    mesh = build_hierarchy(4, 1).levels[-1]
    M, L = _unconstrained(mesh, MHDParams())
    nv = mesh.num_vertices
    nw = 4 * (nv + mesh.num_edges)
    # mass: M_P2 (x) I_4 on w, nothing on (r, p); total = 4 * area
    assert abs(M[nw:].sum()) == 0 and abs(M[:, nw:].sum()) == 0
    assert abs(M.sum() - 4.0) < 1e-12
    assert abs(M - M.T).max() < 1e-15
    # -(p, div v) / -(div u, q) and -(grad r, c) / -(B, grad s) are transposes
    Lw_vp = L[:nw, nw:].toarray()
    assert np.array_equal(Lw_vp, L[nw:, :nw].toarray().T)
    assert abs(L[nw:, nw:]).max() == 0
    # divergence of a constant velocity field and the gradient of a constant
    # multiplier vanish
    cu = np.zeros(L.shape[0])
    cu[0:nw:4] = 1.0
    assert abs(L[nw + nv:] @ cu).max() < 1e-13
    cr = np.zeros(L.shape[0])
    cr[nw:nw + nv] = 1.0
    assert abs(L[:nw] @ cr).max() < 1e-13


def test_boundary_conditions():
    mesh = build_hierarchy(8, 0).levels[0]
    c = mhd_boundary_dofs(mesh)
    xy = p2_node_coords(mesh)
    nn = len(xy)
    w = c[c < 4 * nn]
    node, comp = w // 4, w % 4
    onb = lambda v: (v < 1e-12) | (v > 1 - 1e-12)  # noqa: E731
    # u: both components on every boundary node (32 vertices + 32 edges)
    assert np.sum(comp == 0) == np.sum(comp == 1) == 64
    # B x n = 0: B_x fixed on y = 0, 1; B_y on x = 0, 1
    assert np.all(onb(xy[node[comp == 2], 1]))
    assert np.all(onb(xy[node[comp == 3], 0]))
    assert np.sum(comp == 2) == np.sum(comp == 3) == 2 * 17 - 0
    # r in H^1_0: every boundary vertex; p unconstrained
    rr = c[c >= 4 * nn] - 4 * nn
    assert np.array_equal(rr, np.flatnonzero(mesh.boundary_vertex_flags))


def test_patch_tables_bit_exact_against_oracle():
    disc, tab, case = mhd_setup("mhd16")
    S = disc.system(disc.num_levels - 1, tab, case["dt"])
    t = S.patch_tables(disc.fine_mesh)
    lv = mhd_oracle_levels(disc, tab, case["dt"], levels=[disc.num_levels - 1])[0]
    for k, v in enumerate(t.order):
        assert np.array_equal(t.idx[t.idx_off[k]:t.idx_off[k + 1]], lv["idxs"][v])
    # interior patch: 19 P2 nodes x 4 + r + p per stage
    assert t.max_m == case["stages"] * 78
    sizes = [m for m, _, _ in t.groups()]
    assert sizes == sorted(sizes)
    assert np.array_equal(np.bincount(t.idx, minlength=t.dim), t.multiplicity)


def test_prolongation_reproduces_fields():
    hier = build_hierarchy(4, 1)
    P = mhd_prolongation(hier, 0)
    coarse, fine = hier.levels
    xc = p2_node_coords(coarse)
    xf = p2_node_coords(fine)
    # quadratic fields are reproduced exactly on every P2 component, linear on P1
    f = lambda p: 1 + p[:, 0] ** 2 - 2 * p[:, 0] * p[:, 1]  # noqa: E731
    g = lambda p: 3 - p[:, 0] + 0.5 * p[:, 1]              # noqa: E731
    nc, nf = len(xc), len(xf)
    vc = np.zeros(P.shape[1])
    for k in range(4):
        vc[k:4 * nc:4] = (k + 1) * f(xc)
    vc[4 * nc:4 * nc + coarse.num_vertices] = g(coarse.vertices)
    vc[4 * nc + coarse.num_vertices:] = -g(coarse.vertices)
    vf = P @ vc
    for k in range(4):
        assert np.allclose(vf[k:4 * nf:4], (k + 1) * f(xf), atol=1e-13)
    assert np.allclose(vf[4 * nf:4 * nf + fine.num_vertices], g(fine.vertices), atol=1e-13)
    assert np.allclose(vf[4 * nf + fine.num_vertices:], -g(fine.vertices), atol=1e-13)


def test_stage_operator_oracle_consistency():
    """GeneralStageSystem.materialize (host) == the oracle's operator."""
    disc, tab, case = mhd_setup("mhd16")
    S = disc.system(disc.num_levels - 1, tab, case["dt"])
    lv = mhd_oracle_levels(disc, tab, case["dt"], levels=[disc.num_levels - 1])[0]
    A = S.materialize()
    x = np.random.default_rng(0).uniform(-1, 1, S.dim)
    y = lv["op"].matvec(x)
    assert np.linalg.norm(A @ x - y) <= 1e-14 * np.linalg.norm(y)
    assert S.dim == lv["op"].dim


def test_mhd_configs_are_baseline_shaped():
    c = MHD_CONFIGS["cfg5"]
    assert (c["n0"] * 2 ** c["level"], c["stages"], c["dt"], c["seed"]) == (128, 2, 1 / 128, 4)
    assert tableau_lookup(c["family"], c["stages"]).r == 2


def test_patch_vel_general_lists_p2_dofs():
    """VankaPatchSet.patch_vel on a general system: the P2 (u, B) DoFs of each
    star, consistent with the stage-0 part of patch_indices (host tables only)."""
    from paper_2202_07381_b200.general import build_general_patch_tables
    disc, tab, case = mhd_setup("mhd16")
    S = disc.system(disc.num_levels - 1, tab, case["dt"])
    t = build_general_patch_tables(disc.fine_mesh, S)
    nw = S.nc * S.n_nodes
    for k in range(0, t.num_patches, 37):
        single = t.node[t.node_off[k]:t.node_off[k + 1]]
        idx = t.idx[t.idx_off[k]:t.idx_off[k + 1]]
        assert np.array_equal(idx[:len(single)], single)
        w = single[single < nw]
        assert len(single) - len(w) in (1, 2)        # p (and r unless on the boundary)


def test_device_assembly_contribution_map():
    """The (cell, row, column) -> CSR entry map the device re-linearisation
    gathers through (MHDAssembler, K10g), summed on the host in its cell
    order, reproduces assemble_mhd for a new state -- including the
    structurally kept zeros."""
    from paper_2202_07381_b200.mhd import MHDAssembler, element_matrices
    disc, tab, case = mhd_setup("mhd16")
    mesh = disc.fine_mesh
    S = disc.system(disc.num_levels - 1, tab, case["dt"])
    asm = MHDAssembler(mesh, disc.params, S)
    n_nodes = S.n_nodes
    rng = np.random.default_rng(11)
    u1, B1 = rng.uniform(-1, 1, (n_nodes, 2)), rng.uniform(-1, 1, (n_nodes, 2))
    _, Le = element_matrices(mesh, u1, B1, disc.params)
    flat = Le.reshape(-1)[asm.entry_contrib]
    ptr = asm.entry_ptr
    got = np.array([flat[ptr[e]:ptr[e + 1]].sum() for e in range(len(ptr) - 1)])
    rowptr, col, _, l, _ = assemble_mhd(mesh, disc.params, lambda xy: u1, lambda xy: B1)
    assert np.array_equal(rowptr, S.rowptr) and np.array_equal(col, S.col)
    assert np.max(np.abs(got - l)) <= 1e-14 * np.max(np.abs(l))
    assert len(asm.sell_pos) == len(col)


def test_general_oracle_runs_through_shared_drivers():
    """The general (MHD) oracle patches plug into the shared oracle drivers
    (oracle_apply_vanka, OracleMG incl. the reversed self-floor probe) with
    the same keyword interface as the Stokes oracle."""
    from harness import oracle_mg
    from oracle.irk_vanka_oracle import oracle_apply_vanka, random_rhs
    disc, tab, case = mhd_setup("mhd16")
    lv = mhd_oracle_levels(disc, tab, case["dt"])
    op, pat = lv[-1]["op"], lv[-1]["patches"]
    b = random_rhs(op, case["seed"])
    y1 = oracle_apply_vanka(pat, op, np.zeros(op.dim), b, 0.5, threads=4)
    y2 = oracle_apply_vanka(pat, op, np.zeros(op.dim), b, 0.5)
    assert np.array_equal(y1, y2)
    z = oracle_mg(lv, dict(cheby_a=2.0), "pou").precondition(b.copy())
    zr = oracle_mg(lv, dict(cheby_a=2.0), "pou", reverse=True).precondition(b.copy())
    assert np.linalg.norm(z - zr) <= 1e-10 * np.linalg.norm(z)
