"""Breadth of the device path against the CPU oracle (GPU): every Butcher
tableau family of the reference registry (tableaux.py:114-123) including a
non-diagonalisable DIRK (no eigen-split: modal or full formulations), GMRES-
accelerated smoothing (solvers.py:321-332), partial hierarchies
(bench.py:212-216) and singular-patch detection (solvers.py:176-183)."""

import numpy as np
import pytest

from harness import oracle_levels, rel
from oracle.irk_vanka_oracle import OracleMG, oracle_apply_vanka, random_rhs

pytestmark = pytest.mark.gpu

TABLEAUX = [("gauss", 1), ("gauss", 2), ("gauss", 3), ("radauiia", 1), ("radauiia", 2),
            ("radauiia", 3), ("lobattoiiic", 2), ("lobattoiiic", 3), ("backwardeuler", 1),
            ("dirk-pareschirusso", 2), ("dirk-alexander", 3)]


def _disc(grid="diagonal", n0=4, level=1, mu=1.0):
    from paper_2202_07381_b200 import Discretization
    return Discretization(n0, level, mu=mu, grid=grid)


@pytest.mark.parametrize("family,stages", TABLEAUX)
def test_sweep_and_vcycle_every_tableau(family, stages):
    from paper_2202_07381_b200 import SmootherSpec, apply_vanka, tableau_lookup
    disc = _disc()
    tab = tableau_lookup(family, stages)
    dt = 1.0 / 16
    sm = SmootherSpec()
    mg, S = disc.build_mg(tab, dt, sm)
    fine = mg.levels[-1].patches
    if family.startswith("dirk-"):
        # repeated eigenvalue (PareschiRusso(2), Alexander(3) -- a single
        # Jordan block): no eigen-split, the modal split needs none
        assert fine.mode in ("modal", "dedup")
    lv = oracle_levels(disc, tab, dt, None)
    op, pat = lv[-1]["op"], lv[-1]["patches"]
    b = random_rhs(op, 3)
    x0 = np.random.default_rng(4).uniform(-1, 1, op.dim)
    x0[op.constrained_stage_dofs()] = 0.0
    got = apply_vanka(fine, S, x0, b, omega=0.5)
    assert rel(got, oracle_apply_vanka(pat, op, x0, b, 0.5)) <= 1e-12
    omg = OracleMG(lv, dict(pre=2, post=2, accel="chebyshev", a=2.0, b=8.0, omega=1.0,
                            weights=None))
    assert rel(mg.precondition(b), omg.precondition(b.copy())) <= 1e-11


def test_gmres_accelerated_smoothing_matches_oracle():
    from paper_2202_07381_b200 import SmootherSpec, fgmres, tableau_lookup
    disc = _disc(grid="crossed", n0=2, level=1)
    tab = tableau_lookup("radauiia", 2)
    sm = SmootherSpec(accel="gmres")
    mg, S = disc.build_mg(tab, 0.1, sm)
    lv = oracle_levels(disc, tab, 0.1, None)
    omg = OracleMG(lv, dict(pre=2, post=2, accel="gmres", omega=1.0, weights=None))
    b = random_rhs(lv[-1]["op"], 12)
    assert rel(mg.precondition(b), omg.precondition(b.copy())) <= 1e-10
    # reference test_gmres_accelerated_smoothing (test_solvers.py:321-334)
    xs = np.random.default_rng(12).standard_normal(S.dim)
    xs[S.constrained_stage_dofs()] = 0.0
    xs = S.project_pressure_means(xs)
    _, st = fgmres(S.matvec, S.matvec(xs), precond=mg.precondition, rtol=1e-8, maxiter=60,
                   restart=30)
    assert st.converged and st.iterations <= 30


def test_partial_hierarchy():
    from paper_2202_07381_b200 import ConfigError, SmootherSpec, tableau_lookup
    disc = _disc(n0=4, level=2)
    tab = tableau_lookup("radauiia", 2)
    mg, S = disc.build_mg(tab, 1 / 16, SmootherSpec(), mg_levels=2)
    assert len(mg.levels) == 2 and mg.levels[0].system.dim == disc.blocks[1].n_u * 0 + \
        tab.r * (disc.blocks[1].n_u + disc.blocks[1].n_p)
    lv = oracle_levels(disc, tab, 1 / 16, None, levels=[1, 2])
    lv[0]["prolong"] = None
    omg = OracleMG(lv, dict(pre=2, post=2, accel="chebyshev", a=2.0, b=8.0, omega=1.0,
                            weights=None))
    b = random_rhs(lv[-1]["op"], 5)
    assert rel(mg.precondition(b), omg.precondition(b.copy())) <= 1e-11
    with pytest.raises(ConfigError):
        disc.build_mg(tab, 1 / 16, SmootherSpec(), mg_levels=7)


def test_singular_patch_detected():
    from paper_2202_07381_b200 import PatchSingularError, VankaPatchSet, tableau_lookup
    from paper_2202_07381_b200.stages import StageSystem
    disc = _disc(n0=2, level=0)
    tab = tableau_lookup("backwardeuler", 1)
    # dt = 0: the patch pressure rows vanish -> every patch matrix is singular
    S = StageSystem(disc.blocks[0], tab, 0.0, disc.cdofs[0])
    for mode in ("full", "kron", "modal"):
        with pytest.raises(PatchSingularError) as ei:
            VankaPatchSet(S, disc.hier.levels[0], mode=mode)
        assert 0 <= ei.value.vertex < disc.hier.levels[0].num_vertices


def test_invalid_arguments_raise():
    from paper_2202_07381_b200 import SmootherSpec, apply_vanka, tableau_lookup
    disc = _disc(n0=2, level=1)
    mg, S = disc.build_mg(tableau_lookup("radauiia", 2), 0.1, SmootherSpec())
    with pytest.raises(ValueError):
        S.matvec(np.zeros(S.dim + 1))
    with pytest.raises(ValueError):
        apply_vanka(mg.levels[-1].patches, S, np.zeros(3), np.zeros(S.dim))


@pytest.mark.parametrize("name", ["crossed", "cfg1", "s3", "ns"])
def test_coarse_methods_against_superlu(name):
    """K6 in both forms against the reference's own solve (solvers.py:284-287):
    x = P lu.solve(P b), P = I - Z Z^T."""
    import torch
    from harness import setup
    from paper_2202_07381_b200.solvers import CoarseSolver
    from paper_2202_07381_b200.stages import StageSystem
    disc, tab, conv, case = setup(name)
    S0 = StageSystem(disc.blocks[0], tab, case["dt"], disc.cdofs[0],
                     None if conv is None else conv[0])
    A = S0.materialize()
    b = np.random.default_rng(5).standard_normal(S0.dim)
    for method in ("dense", "lu"):
        cs = CoarseSolver(S0, method)
        Z = cs.Z
        pb = b - Z @ (Z.T @ b)
        ref = cs.lu.solve(pb)
        ref -= Z @ (Z.T @ ref)
        x = torch.empty(S0.dim, dtype=torch.float64, device="cuda")
        got = cs.solve_into(torch.from_numpy(b).cuda(), x).cpu().numpy()
        tol = 1e-12 if name in ("crossed", "cfg1") else 1e-7
        assert rel(got, ref) <= tol, method
        be = np.linalg.norm(A @ got - pb) / np.linalg.norm(pb)
        be_ref = np.linalg.norm(A @ ref - pb) / np.linalg.norm(pb)
        assert be <= max(10 * be_ref, 1e-13), method


@pytest.mark.parametrize("name", ["crossed", "s3", "ns"])
def test_residual_in_place_matches(name):
    """K1 with out aliasing b (the residual r = b - A x written over b) equals
    the out-of-place result bitwise (every row computed exactly once)."""
    import torch
    from harness import setup
    from paper_2202_07381_b200 import _lib
    from paper_2202_07381_b200._device import ptr, stream
    from paper_2202_07381_b200.stages import StageSystem
    disc, tab, conv, case = setup(name)
    k = disc.num_levels - 1
    S = StageSystem(disc.blocks[k], tab, case["dt"], disc.cdofs[k],
                    None if conv is None else conv[k])
    rng = np.random.default_rng(2)
    x = torch.from_numpy(rng.standard_normal(S.dim)).cuda()
    b = torch.from_numpy(rng.standard_normal(S.dim)).cuda()
    r = torch.empty_like(b)
    L = _lib.lib()
    _lib.check(L.ivk_stage_apply(S.desc, ptr(x), ptr(b), ptr(r), stream()), "K1")
    bb = b.clone()
    _lib.check(L.ivk_stage_apply(S.desc, ptr(x), ptr(bb), ptr(bb), stream()), "K1")
    assert torch.equal(r, bb)
    assert rel(r.cpu().numpy(), b.cpu().numpy() - S.matvec(x.cpu().numpy())) <= 1e-13


@pytest.mark.parametrize("family,stages", [("dirk-pareschirusso", 2), ("dirk-alexander", 3),
                                           ("lobattoiiic", 3),
                                           ("backwardeuler", 1), ("gauss", 3)])
def test_modal_any_tableau(family, stages):
    """The modal split needs no eigen-split of A: non-diagonalisable DIRK
    tableaux run through it too (sweep parity against the full inverses)."""
    import torch
    from paper_2202_07381_b200 import SmootherSpec, VankaPatchSet, apply_vanka, tableau_lookup
    disc = _disc()
    tab = tableau_lookup(family, stages)
    mg, S = disc.build_mg(tab, 1.0 / 16, SmootherSpec(), patch_mode="modal")
    fine = mg.levels[-1].patches
    assert fine.mode == "modal"
    full = VankaPatchSet(S, disc.fine_mesh, mode="full")
    b = torch.from_numpy(np.random.default_rng(3).uniform(-1, 1, S.dim)).cuda()
    x0 = torch.zeros_like(b)
    ym = apply_vanka(fine, S, x0, b, omega=0.5, weights="pou")
    yf = apply_vanka(full, S, x0, b, omega=0.5, weights="pou")
    assert float(torch.linalg.vector_norm(ym - yf)) <= 1e-12 * float(torch.linalg.vector_norm(yf))
