"""Inexact Newton for one IRK step of Navier--Stokes, on the device.

The reference's Navier--Stokes driver (``bench.run_ns_taylor_green``,
/root/reference/pkg/src/irkmg/bench.py:373-424) solves the stage equations

    Fu_i = M ku_i + K us_i + N(us_i) + B ps_i,   Fp_i = B^T us_i,
    us_i = u_n + dt sum_j a_ij ku_j,   ps_i = p_n + dt sum_j a_ij kp_j,

with inexact Newton and Eisenstat--Walker forcing (newton.py:60-115),
rebuilding the per-stage convection Jacobians J_N(us_i) on every grid level
and all Vanka patch inverses at each iteration.  Here every piece runs on the
GPU: the residual is K1 on the Stokes stage operator plus a per-step constant
plus the convection residual of K10; the Jacobian update is K10 per stage and
level written straight into the operators' device buffers, K7 refactorises
every level's patches in place, and FGMRES + the V-cycle solve for the
direction.  Only the coarsest level's SuperLU factorisation (the reference's
own coarse solver) and the Newton scalars stay on the host.

Dirichlet data are homogeneous (u_n = 0 on the boundary, zero stage boundary
values -- the BASELINE configurations' setting); the constrained rows are
then exactly ``Fu_i[c] = ku_i[c]``, which the stage operator's identity rows
produce.
"""

from dataclasses import dataclass, field

import numpy as np

from .fem import ConvectionBlocks
from .solvers import CoarseSolver, fgmres
from .stages import assemble_stage_operator

__all__ = ["NewtonConfig", "NewtonStats", "NewtonError", "ew_forcing", "NSStageNewton"]

ETA_FLOOR = 1e-12


@dataclass
class NewtonConfig:
    """Reference ``NewtonConfig`` (newton.py:19-33)."""

    atol: float = 1e-10
    maxit: int = 20
    ew_gamma: float = 0.9
    ew_alpha: float = 2.0
    eta0: float = 0.5
    eta_max: float = 0.9
    safeguard: bool = True

    def __post_init__(self):
        if not 0.0 <= self.eta0 < 1.0 or not 0.0 < self.eta_max < 1.0:
            raise ValueError("forcing terms must lie in [0, 1)")
        if self.atol <= 0.0:
            raise ValueError("tolerance must be positive")


@dataclass
class NewtonStats:
    iterations: int = 0
    residual_norms: list = field(default_factory=list)
    linear_stats: list = field(default_factory=list)
    converged: bool = False


class NewtonError(RuntimeError):
    pass


def ew_forcing(eta_prev, norm_k, norm_prev, config):
    """Eisenstat--Walker "Choice 2" with the safeguard (newton.py:46-56)."""
    if norm_prev <= 0.0:
        raise ValueError("previous residual norm must be positive")
    eta = config.ew_gamma * (norm_k / norm_prev) ** config.ew_alpha
    if config.safeguard:
        stale = config.ew_gamma * eta_prev ** config.ew_alpha
        if stale > 0.1:
            eta = max(eta, stale)
    return float(np.clip(eta, ETA_FLOOR, config.eta_max))


class NSStageNewton:
    """One IRK step of Navier--Stokes: ``solve(u_n, p_n)`` -> (k, stats).

    ``disc`` is a ``Discretization`` (its ``mu`` is 1/Re); the V-cycle runs
    the full per-patch inverses (per-stage Jacobians differ, so the
    Butcher eigen-split does not apply, solvers.py:169-212)."""

    def __init__(self, disc, tableau, dt, smoother, mg_levels=None, maxiter=200, restart=50):
        import torch
        self.disc, self.tab, self.dt = disc, tableau, float(dt)
        self.s = tableau.r
        self.maxiter, self.restart = int(maxiter), int(restart)
        # distinct per-stage Jacobian slots on every level (filled at relinearize)
        conv = []
        for blk in disc.blocks:
            z = np.zeros((len(blk.col), 2, 2))
            conv.append([ConvectionBlocks(blk.n_nodes, blk.rowptr, blk.col, z.copy())
                         for _ in range(self.s)])
        self.mg, self.S = disc.build_mg(tableau, dt, smoother, mg_levels=mg_levels,
                                        convection=conv, patch_mode="full")
        # the Stokes stage operator for the residual (K1 without convection)
        self.S0 = assemble_stage_operator(disc.blocks[-1], tableau, dt,
                                          constrained=disc.cdofs[-1])
        self.asm = disc.convection_assemblers()
        self.start = disc.num_levels - len(self.mg.levels)
        self._A = torch.from_numpy(np.asarray(tableau.A, dtype=np.float64))
        self._cmask = None
        self._host_kb = None

    # -- pieces ---------------------------------------------------------------

    def _velocities(self, k, u_n):
        """Stage velocities us_i = u_n + dt sum_j a_ij ku_j, (s, n_u) device."""
        S = self.S0
        ku = k.view(self.s, S.stage_dim)[:, :S.n_u]
        return u_n[None, :] + self.dt * (self._A.to(k.device) @ ku)

    def constant(self, u_n, p_n):
        """Per-step part of the residual: [K u_n + B p_n ; B^T u_n] (eliminated,
        host scipy, once per time step), as a device stage vector."""
        import torch
        S = self.S0
        un = np.asarray(u_n, dtype=np.float64)
        pn = np.asarray(p_n, dtype=np.float64)
        if self._host_kb is None:
            # the vector-form scipy blocks are rebuilt from the scalar ones on
            # every property access (a second per step at cfg3): keep them
            self._host_kb = (S.K, S.B, S.BT)
        K, B, BT = self._host_kb
        cu = K @ un + B @ pn
        cu[S.constrained] = 0.0
        cp = BT @ un
        c = np.tile(np.concatenate([cu, cp]), self.s)
        return torch.from_numpy(c).cuda()

    def residual(self, k, u_n, c):
        """F(k) on the device (bench.py:393-403)."""
        import torch
        S = self.S0
        F = torch.empty_like(k)
        S.apply_into(k, None, F)                        # (I (x) M + dt A (x) S) k, k[c] on c
        F += c
        if self._cmask is None:
            self._cmask = S.device_data()["cmask_dofs"]
        us = self._velocities(k, u_n)
        Fv = F.view(self.s, S.stage_dim)
        for i in range(self.s):
            _, N = self.asm[-1].jacobian(us[i].contiguous(), residual=True)
            N[self._cmask] = 0.0
            Fv[i, :S.n_u] += N
        return F

    def relinearize(self, k, u_n):
        """J_N(us_i) for every stage on every level (nodal injection, as the
        reference's ``disc.inject_velocity``), patches refactorised in place,
        coarse SuperLU rebuilt (bench.py:405-417)."""
        us = self._velocities(k, u_n)
        for lv, lev in enumerate(self.mg.levels):
            asm = self.asm[self.start + lv]
            n = 2 * lev.system.n_nodes
            for i in range(self.s):
                asm.assemble_stage(lev.system, i, us[i, :n].contiguous())
            if lv > 0:
                lev.patches.factor()
                lev.system.mark_host_stale()
        s0 = self.mg.levels[0].system
        if getattr(self.mg.coarse, "method", "dense") == "dense":
            # the coarse operator straight from the re-assembled device operator
            # (the host route -- download, materialize, SuperLU, n solves --
            # cost 0.3 s per Newton iteration at cfg3, most of the step)
            s0.mark_host_stale()
            self.mg.coarse = CoarseSolver.from_device_operator(s0)
        else:
            s0.download_convection()
            self.mg.coarse = CoarseSolver(s0, self.mg.coarse.method)
        self.mg._graph = None
        self.mg._bufs = None

    # -- the Newton loop (newton.py:60-115) --------------------------------------

    def solve(self, u_n, p_n, k0=None, config=None):
        import torch
        config = config or NewtonConfig()
        S = self.S0
        u_d = torch.as_tensor(np.asarray(u_n, dtype=np.float64)).cuda()
        c = self.constant(u_n, p_n)
        k = torch.zeros(S.dim, dtype=torch.float64, device="cuda") if k0 is None else \
            torch.as_tensor(np.asarray(k0, dtype=np.float64)).cuda().clone()
        stats = NewtonStats()
        F = self.residual(k, u_d, c)
        norm = float(torch.linalg.vector_norm(F))
        stats.residual_norms.append(norm)
        eta = config.eta0
        while norm > config.atol:
            if stats.iterations >= config.maxit:
                raise NewtonError(f"Newton failed to converge in {config.maxit} iterations "
                                  f"(residual {norm:.3e}, tolerance {config.atol:.3e})")
            self.relinearize(k, u_d)
            dx, lin = fgmres(self.S.matvec, -F, precond=self.mg.precondition, rtol=eta,
                             atol=0.1 * config.atol, maxiter=self.maxiter, restart=self.restart)
            if lin.final_residual > max(eta * norm, config.atol) * (1.0 + 1e-8):
                raise NewtonError(f"inner solve violated the forcing bound: "
                                  f"{lin.final_residual:.3e} > {eta * norm:.3e}")
            stats.linear_stats.append(lin)
            k += dx
            stats.iterations += 1
            F = self.residual(k, u_d, c)
            prev = norm
            norm = float(torch.linalg.vector_norm(F))
            stats.residual_norms.append(norm)
            eta = ew_forcing(eta, norm, prev, config)
        stats.converged = True
        return k, stats
