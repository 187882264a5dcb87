"""Per-level setup bundle: meshes, scalar-node Stokes blocks, transfers, and
the V-cycle constructor (mirror of the reference ``bench.Discretization``,
/root/reference/pkg/src/irkmg/bench.py:157-228).

Host-side setup only: it produces the hot path's inputs and wires the
device objects together.  ``grid`` selects the coarse grid: "crossed" is
the reference's own (``mesh.py:144-175``), "diagonal" the BASELINE.json
right-triangle grids.
"""

import numpy as np

from . import fem
from .mesh import build_hierarchy
from .solvers import MGHierarchyOp, MGLevel, VankaPatchSet, coarse_direct_solve
from .stages import assemble_stage_operator
from .transfer import StageTransfer

__all__ = ["Discretization", "ConfigError", "oseen_convection", "streamfunction_velocity"]


class ConfigError(ValueError):
    pass


class Discretization:
    def __init__(self, n0, level, mu=1.0, grid="crossed"):
        self.hier = build_hierarchy(n0, level, grid)
        self.mu = float(mu)
        self.blocks = [fem.assemble_blocks(m, mu=mu) for m in self.hier.levels]
        self.cdofs = [fem.velocity_boundary_dofs(m) for m in self.hier.levels]
        self.cnodes = []
        for m, blk in zip(self.hier.levels, self.blocks):
            mask = np.zeros(blk.n_nodes, dtype=bool)
            mask[fem.velocity_boundary_nodes(m)] = True
            self.cnodes.append(mask)
        self._scalar_prolong = [
            (fem.prolongation(self.hier, k, "p2"), fem.prolongation(self.hier, k, "p1"))
            for k in range(self.hier.num_levels - 1)
        ]
        self._stage_prolong = {}

    @property
    def num_levels(self):
        return self.hier.num_levels

    @property
    def fine_mesh(self):
        return self.hier.levels[-1]

    def stage_prolong(self, level, r):
        """Transfer level-1 -> level for r stages (bench.py:187-194)."""
        key = (level, r)
        if key not in self._stage_prolong:
            p2, p1 = self._scalar_prolong[level - 1]
            self._stage_prolong[key] = StageTransfer(p2, p1, r, self.cnodes[level],
                                                     self.cnodes[level - 1])
        return self._stage_prolong[key]

    def build_mg(self, tableau, dt, smoother, mg_levels=None, convection=None, use_graph=False,
                 patch_mode="auto"):
        """Stage systems on every level, GPU-factorised Vanka patches and the
        V-cycle (bench.py:206-228).  Returns (MGHierarchyOp, finest system)."""
        total = self.num_levels
        depth = total if mg_levels is None else int(mg_levels)
        if not 1 <= depth <= total:
            raise ConfigError(f"mg.levels must lie in [1, {total}]")
        start = total - depth
        levels = []
        for k in range(start, total):
            conv_k = None if convection is None else convection[k]
            system = assemble_stage_operator(self.blocks[k], tableau, dt,
                                             constrained=self.cdofs[k], convection=conv_k)
            # The coarsest level's patches are never used (direct solve); the
            # reference builds them anyway (bench.py:224) -- we skip the
            # factorisation there.
            patches = VankaPatchSet(system, self.hier.levels[k], factor=(k > start),
                                    mode=patch_mode)
            P = self.stage_prolong(k, tableau.r) if k > start else None
            levels.append(MGLevel(system, patches, smoother, P))
        coarse = coarse_direct_solve(levels[0].system)
        return MGHierarchyOp(levels, coarse, use_graph=use_graph), levels[-1].system


    def convection_assemblers(self):
        """One device ConvectionAssembler per level (MGHierarchyOp.relinearize)."""
        from .assembly import ConvectionAssembler
        if not hasattr(self, "_assemblers"):
            self._assemblers = [ConvectionAssembler(m, b, cm) for m, b, cm in
                                zip(self.hier.levels, self.blocks, self.cnodes)]
        return self._assemblers


def streamfunction_velocity(points):
    """w = (d psi/dy, -d psi/dx) / pi for psi = sin^2(pi x) sin^2(pi y);
    max |w| = 1 (BASELINE config 3 / SURVEY.md §8(d))."""
    x, y = points[:, 0], points[:, 1]
    sx, sy = np.sin(np.pi * x), np.sin(np.pi * y)
    return np.column_stack([sx * sx * np.sin(2 * np.pi * y),
                            -np.sin(2 * np.pi * x) * sy * sy])


def oseen_convection(disc, stages, velocity=streamfunction_velocity):
    """Frozen-velocity Newton Jacobians J_N(w_l) on every level, shared by
    all stages: ``convection[l] = [J_l] * stages``."""
    out = []
    for mesh, blk in zip(disc.hier.levels, disc.blocks):
        w = fem.interpolate_velocity(mesh, velocity)
        J = fem.assemble_convection_jacobian(mesh, blk, w)
        out.append([J] * stages)
    return out
