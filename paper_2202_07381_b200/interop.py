"""Object-level interop with hierarchies built by the reference package.

A reference user holding ``irkmg`` objects can hand them over as they are:

* ``GpuStage(system)`` -- wraps a reference ``irkmg.stages.StageSystem``
  (duck-typed: ``.blocks`` with the vector-P2 CSR ``M``, ``K``, ``B``;
  ``.tableau``, ``.dt``, ``.constrained``, ``.convection`` = the eliminated
  per-stage vector Jacobians or None; stages.py:63-88) into the device
  ``StageSystem``; its ``matvec`` replaces stages.py:110-126.
* ``as_transfer(P, fine, coarse)`` -- a reference stage prolongation (scipy
  CSR, fine x coarse: ``Discretization.stage_prolong``, bench.py:187-194,
  used as ``P.T @ r`` / ``P @ e`` with constrained rows zeroed,
  solvers.py:340-346) as a device transfer (K5g over the full stage-level
  CSR).  ``MGHierarchyOp`` applies it automatically to any level whose
  ``prolong`` is a scipy matrix.
* ``from_reference_hierarchy(mg, meshes)`` -- a reference ``MGHierarchyOp``
  (levels of ``system, patches, smoother, prolong``) rebuilt on the device:
  stage systems via ``GpuStage``, Vanka patches factorised by K7 on the same
  meshes (patch tables bit-exact with the reference's ``_build``), the
  reference's scipy prolongations kept as they are.
"""

import numpy as np
import scipy.sparse as sp

__all__ = ["GpuStage", "as_transfer", "from_reference_hierarchy"]


def GpuStage(system):
    """Device ``StageSystem`` equivalent to a reference ``StageSystem``."""
    from .fem import ConvectionBlocks, StokesBlocks
    from .stages import StageSystem
    if isinstance(system, StageSystem):
        return system
    blk = system.blocks
    blocks = StokesBlocks.from_vector(blk.M, blk.K, blk.B)
    conv = None
    if getattr(system, "convection", None) is not None:
        # elimination is idempotent (D J D), so the reference's eliminated
        # Jacobians are valid raw input
        conv = [ConvectionBlocks.from_vector(J, blocks) for J in system.convection]
    return StageSystem(blocks, system.tableau, system.dt, np.asarray(system.constrained),
                       conv)


def _cmask(system):
    m = np.zeros(system.dim, dtype=bool)
    m[system.constrained_stage_dofs()] = True
    return m


def as_transfer(P, fine, coarse):
    """Device transfer for a stage-level scipy prolongation ``P``."""
    from .general import GeneralTransfer
    P = sp.csr_matrix(P)
    if P.shape != (fine.dim, coarse.dim):
        raise ValueError(f"prolongation shape {P.shape} does not match the level dims "
                         f"({fine.dim}, {coarse.dim})")
    return GeneralTransfer(P, 1, _cmask(fine), _cmask(coarse))


def is_matrix(P):
    return sp.issparse(P) or isinstance(P, np.ndarray)


def from_reference_hierarchy(mg, meshes, patch_mode="auto", use_graph=False):
    """Rebuild a reference ``MGHierarchyOp`` on the device.

    ``meshes``: the level meshes, coarsest first (``cells``,
    ``cell_to_edges``, ``num_vertices`` -- the reference ``Mesh2D`` works)."""
    from .solvers import MGHierarchyOp, MGLevel, SmootherSpec, VankaPatchSet, \
        coarse_direct_solve
    if len(meshes) != len(mg.levels):
        raise ValueError("one mesh per level required")
    levels = []
    for k, (lev, mesh) in enumerate(zip(mg.levels, meshes)):
        S = GpuStage(lev.system)
        sm = lev.smoother
        spec = SmootherSpec(pre=sm.pre, post=sm.post, accel=sm.accel, cheby_a=sm.cheby_a,
                            cheby_b=sm.cheby_b, omega=sm.omega)
        pat = VankaPatchSet(S, mesh, omega=getattr(lev.patches, "omega", 1.0), factor=k > 0,
                            mode=patch_mode)
        levels.append(MGLevel(S, pat, spec, lev.prolong if k > 0 else None))
    return MGHierarchyOp(levels, coarse_direct_solve(levels[0].system), use_graph=use_graph)
