"""3-D Stokes on Kuhn tetrahedra (BASELINE config 4 family) through the C
ABI: K1 with three components per node, the large-patch K7 (global-memory
Gauss-Jordan on the transposed patch matrix, full (s b)^2 inverses or the
Kronecker eigen-blocks, b = 3k + 1 ~ 100-200), K3 full and the wide-block
K3e, K5 with ncomp = 3,
against the CPU oracle on the same host setup.  The reference has no 3-D
discretisation: parity is to this repo's oracle restatement."""

import numpy as np
import pytest

from harness import rel
from oracle.irk_vanka_oracle import (OracleMG, OraclePatches, OracleStageOperator,
                                     oracle_apply_vanka, oracle_patch_indices, random_rhs)

pytestmark = pytest.mark.gpu

_cache = {}


def _case(family="radauiia", stages=2, mode="kron"):
    key = (family, stages, mode)
    if key in _cache:
        return _cache[key]
    from paper_2202_07381_b200 import SmootherSpec, tableau_lookup
    from paper_2202_07381_b200.fem3d import Discretization3D
    disc = Discretization3D(2, 1)
    tab = tableau_lookup(family, stages)
    dt = 1 / 32
    cheb = SmootherSpec(pre=2, post=2, accel="chebyshev", cheby_a=2.0, cheby_b=8.0)
    mg, S = disc.build_mg(tab, dt, cheb, patch_mode=mode)
    lv = []
    for k in range(disc.num_levels):
        blk, mesh = disc.blocks[k], disc.hier.levels[k]
        op = OracleStageOperator(blk.M, blk.K, blk.B, tab.A, dt, disc.cdofs[k])
        vels, idxs = oracle_patch_indices(mesh.cells, mesh.cell_to_edges, mesh.num_vertices, op,
                                          ncomp=3)
        lv.append({"op": op, "patches": OraclePatches(op, vels, idxs) if k else None,
                   "prolong": disc.stage_prolong(k, tab.r).matrix if k else None, "idxs": idxs})
    _cache[key] = (disc, tab, dt, mg, S, lv)
    return _cache[key]


def test_three_stage_3d_full_patches_unsupported():
    """s = 3 gives 3-D patches of 588 unknowns: past the 512-row full K3/K7
    kernels, rejected loudly (no fallback); the eigen-split (b = 196) runs."""
    from paper_2202_07381_b200 import SmootherSpec, tableau_lookup
    from paper_2202_07381_b200._lib import IvkError
    from paper_2202_07381_b200.fem3d import Discretization3D
    disc = Discretization3D(2, 1)
    with pytest.raises(IvkError):
        disc.build_mg(tableau_lookup("radauiia", 3), 1 / 32, SmootherSpec(), patch_mode="full")


def test_three_stage_3d_kron():
    from paper_2202_07381_b200 import apply_vanka
    disc, tab, dt, mg, S, lv = _case("radauiia", 3, "kron")
    op, pat = lv[-1]["op"], lv[-1]["patches"]
    fine = mg.levels[-1].patches
    assert fine.mode == "kron" and fine.tables.max_m == 588
    b = random_rhs(op, 4)
    x = np.random.default_rng(2).uniform(-1, 1, S.dim)
    x[S.constrained_stage_dofs()] = 0.0
    w = pat.pou_weights(op.dim)
    assert rel(apply_vanka(fine, S, x, b, omega=0.4, weights="pou"),
               oracle_apply_vanka(pat, op, x, b, 0.4, weights=w)) <= 1e-12


@pytest.mark.parametrize("mode", ["kron", "full", "modal"])
@pytest.mark.parametrize("fam", [("radauiia", 2), ("gauss", 2), ("lobattoiiic", 2)])
def test_matvec_and_sweep_3d(fam, mode):
    disc, tab, dt, mg, S, lv = _case(*fam, mode=mode)
    op, pat = lv[-1]["op"], lv[-1]["patches"]
    fine = mg.levels[-1].patches
    assert fine.mode == mode
    x = np.random.default_rng(1).uniform(-1, 1, S.dim)
    x[S.constrained_stage_dofs()] = 0.0
    assert rel(S.matvec(x), op.matvec(x)) <= 1e-13
    b = random_rhs(op, 3)
    from paper_2202_07381_b200 import apply_vanka
    assert rel(apply_vanka(fine, S, x, b, omega=0.4), oracle_apply_vanka(pat, op, x, b, 0.4)) \
        <= 1e-12
    w = pat.pou_weights(op.dim)
    assert rel(apply_vanka(fine, S, x, b, omega=0.4, weights="pou"),
               oracle_apply_vanka(pat, op, x, b, 0.4, weights=w)) <= 1e-12


@pytest.mark.parametrize("mode", ["kron", "full", "modal"])
def test_large_patch_inverses_3d(mode):
    """K7 (global Gauss-Jordan, d up to 392 / eigen-blocks b up to 196)
    against np.linalg.inv."""
    disc, tab, dt, mg, S, lv = _case(mode=mode)
    fine = mg.levels[-1].patches
    for (idx_d, inv_d), (idx_o, inv_o) in zip(fine.groups, lv[-1]["patches"].groups):
        assert np.array_equal(np.asarray(idx_d), idx_o)
        assert rel(np.asarray(inv_d), inv_o) <= 1e-12


@pytest.mark.parametrize("pmode", ["kron", "full", "modal"])
@pytest.mark.parametrize("mode", ["cheb", "pou"])
def test_vcycle_3d(mode, pmode):
    from paper_2202_07381_b200 import MGHierarchyOp, MGLevel, SmootherSpec
    disc, tab, dt, mg, S, lv = _case(mode=pmode)
    if mode == "pou":
        sm = SmootherSpec(pre=2, post=2, accel="richardson", omega=0.4, weighting="pou")
        mg = MGHierarchyOp([MGLevel(l.system, l.patches, sm, l.prolong) for l in mg.levels],
                           mg.coarse)
        osm = dict(pre=2, post=2, accel="richardson", omega=0.4, weights="pou")
    else:
        osm = dict(pre=2, post=2, accel="chebyshev", a=2.0, b=8.0, omega=1.0, weights=None)
    omg = OracleMG(lv, osm)
    b = random_rhs(lv[-1]["op"], 5)
    assert rel(mg.precondition(b), omg.precondition(b.copy())) <= 1e-11


@pytest.mark.parametrize("smoother", ["pou", "cheb"])
def test_fgmres_3d(smoother):
    """BASELINE config 4's smoother is PoU-weighted Vanka damped by 0.4 (the
    weighted spectrum here lies in [0, 1.7]); unweighted additive Vanka in
    3-D has eigenvalues up to ~17 (15 patches share a vertex DoF), so the
    Chebyshev interval scales to [4, 17] (2-D: [2, 8])."""
    from paper_2202_07381_b200 import MGHierarchyOp, MGLevel, SmootherSpec, fgmres
    disc, tab, dt, mg, S, lv = _case()
    if smoother == "pou":
        sm = SmootherSpec(pre=2, post=2, accel="richardson", omega=0.4, weighting="pou")
    else:
        sm = SmootherSpec(pre=2, post=2, accel="chebyshev", cheby_a=4.0, cheby_b=17.0)
    h = MGHierarchyOp([MGLevel(l.system, l.patches, sm, l.prolong) for l in mg.levels],
                      mg.coarse)
    b = random_rhs(lv[-1]["op"], 3)
    _, st = fgmres(S.matvec, b, precond=h.precondition, rtol=1e-8, maxiter=100, restart=50)
    assert st.converged and st.iterations <= (25 if smoother == "pou" else 40)
