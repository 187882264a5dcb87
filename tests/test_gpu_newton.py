"""End-to-end Navier--Stokes IRK Newton step on the device (newton.py,
SURVEY.md §8(f) #3) against a host restatement of the reference's inner
Newton loop (bench.py:373-424, newton.py:60-115) on the same seeded state:
the same Newton iteration count, residual histories that agree, and stage
vectors that agree to the Newton tolerance."""

import numpy as np
import pytest

from harness import rel
from oracle.irk_vanka_oracle import (OracleMG, OraclePatches, OracleStageOperator,
                                     oracle_fgmres, oracle_patch_indices)

pytestmark = pytest.mark.gpu

MU, DT = 0.01, 1.0 / 32


def _setup():
    from paper_2202_07381_b200 import Discretization, SmootherSpec, tableau_lookup, fem
    from paper_2202_07381_b200.discretization import streamfunction_velocity
    disc = Discretization(8, 1, mu=MU, grid="diagonal")
    tab = tableau_lookup("gauss", 2)
    sm = SmootherSpec(pre=2, post=2, accel="chebyshev", cheby_a=1.5, cheby_b=8.0)
    mesh = disc.fine_mesh
    u_n = 0.8 * fem.interpolate_velocity(mesh, streamfunction_velocity)
    p_n = np.random.default_rng(7).uniform(-1, 1, mesh.num_vertices)
    return disc, tab, sm, u_n, p_n


def host_newton(disc, tab, u_n, p_n, config, maxiter=200, restart=50):
    """The reference's inner Newton loop with numpy/scipy pieces."""
    from paper_2202_07381_b200 import fem
    from paper_2202_07381_b200.newton import ew_forcing
    A, s = np.asarray(tab.A), tab.r
    blk = disc.blocks[-1]
    mesh = disc.fine_mesh
    op0 = OracleStageOperator(blk.M, blk.K, blk.B, A, DT, disc.cdofs[-1])
    n_u = op0.n_u
    cu = op0.K @ u_n + op0.B @ p_n
    cu[op0.constrained] = 0.0
    c = np.tile(np.concatenate([cu, op0.BT @ u_n]), s)

    def stages(k):
        ku = k.reshape(s, -1)[:, :n_u]
        return u_n[None, :] + DT * (A @ ku)

    def residual(k):
        F = op0.matvec(k) + c
        us = stages(k)
        Fv = F.reshape(s, -1)
        for i in range(s):
            N = fem.assemble_convection_residual(mesh, blk, us[i])
            N[op0.constrained] = 0.0
            Fv[i, :n_u] += N
        return F

    def jacobian(k):
        us = stages(k)
        levels = []
        for lv in range(disc.num_levels):
            b_l, m_l = disc.blocks[lv], disc.hier.levels[lv]
            n = 2 * b_l.n_nodes
            Js = [fem.assemble_convection_jacobian(m_l, b_l, us[i, :n]).matrix for i in range(s)]
            op = OracleStageOperator(b_l.M, b_l.K, b_l.B, A, DT, disc.cdofs[lv], convection=Js)
            vels, idxs = oracle_patch_indices(m_l.cells, m_l.cell_to_edges, m_l.num_vertices, op)
            levels.append({"op": op, "patches": OraclePatches(op, vels, idxs) if lv else None,
                           "prolong": disc.stage_prolong(lv, s).matrix if lv else None})
        sm = dict(pre=2, post=2, accel="chebyshev", a=1.5, b=8.0, omega=1.0, weights=None)
        return levels[-1]["op"], OracleMG(levels, sm)

    k = np.zeros(op0.dim)
    F = residual(k)
    norms = [np.linalg.norm(F)]
    eta, its = config.eta0, 0
    while norms[-1] > config.atol:
        op, mg = jacobian(k)
        dx, _ = oracle_fgmres(op.matvec, -F, precond=mg.precondition, rtol=eta,
                              atol=0.1 * config.atol, maxiter=maxiter, restart=restart)
        k = k + dx
        its += 1
        F = residual(k)
        norms.append(np.linalg.norm(F))
        eta = ew_forcing(eta, norms[-1], norms[-2], config)
        assert its <= config.maxit
    return k, its, norms


def test_ns_newton_step_matches_host():
    from paper_2202_07381_b200.newton import NewtonConfig, NSStageNewton
    disc, tab, sm, u_n, p_n = _setup()
    cfg = NewtonConfig(atol=1e-9)
    solver = NSStageNewton(disc, tab, DT, sm)
    k, st = solver.solve(u_n, p_n, config=cfg)
    kh, its, norms = host_newton(disc, tab, u_n, p_n, cfg)
    assert st.converged and its >= 2
    assert st.iterations == its
    # the first residual is exact arithmetic on identical inputs
    assert abs(st.residual_norms[0] - norms[0]) <= 1e-12 * norms[0]
    # both iterates satisfy F(k) <= atol; they agree to that scale
    assert rel(k.cpu().numpy(), kh) <= 1e-6
    # the device residual at the host solution is the host's own residual
    import torch
    Fd = solver.residual(torch.from_numpy(kh).cuda(), torch.from_numpy(u_n).cuda(),
                         solver.constant(u_n, p_n))
    assert float(torch.linalg.vector_norm(Fd)) <= 10 * cfg.atol


def test_newton_jacobian_is_the_residual_derivative():
    """J dk (the relinearised stage operator) equals the directional
    derivative of the device residual (central difference)."""
    import torch
    from paper_2202_07381_b200.newton import NSStageNewton
    disc, tab, sm, u_n, p_n = _setup()
    solver = NSStageNewton(disc, tab, DT, sm)
    rng = np.random.default_rng(3)
    S = solver.S0
    k = torch.from_numpy(rng.uniform(-1, 1, S.dim)).cuda()
    k[torch.from_numpy(S.constrained_stage_dofs()).cuda()] = 0.0
    dk = torch.from_numpy(rng.uniform(-1, 1, S.dim)).cuda()
    dk[torch.from_numpy(S.constrained_stage_dofs()).cuda()] = 0.0
    ud = torch.from_numpy(u_n).cuda()
    c = solver.constant(u_n, p_n)
    solver.relinearize(k, ud)
    Jdk = solver.S.matvec(dk)
    h = 1e-6
    fd = (solver.residual(k + h * dk, ud, c) - solver.residual(k - h * dk, ud, c)) / (2 * h)
    assert float(torch.linalg.vector_norm(Jdk - fd)) <= 1e-7 * float(torch.linalg.vector_norm(fd))
