"""B200-native IRK-Vanka: additive vertex-star Vanka relaxation for
fully-implicit Runge-Kutta stage-coupled Taylor-Hood systems, applied on
every level of a monolithic geometric V-cycle (arXiv:2202.07381), as
hand-written sm_100a CUDA kernels behind the reference ``irkmg`` Python API.
"""

from . import fem, mesh, quadrature, tableaux
from ._lib import IvkError
from .discretization import (ConfigError, Discretization, oseen_convection,
                             streamfunction_velocity)
from .fem import assemble_blocks, assemble_convection_jacobian, prolongation
from .mesh import Mesh2D, MeshHierarchy, build_hierarchy, crossed_grid, diagonal_grid
from .solvers import (CoarseSolver, KrylovStats, MGHierarchyOp, MGLevel, PatchSingularError,
                      SmootherSpec, VankaPatchSet, apply_vanka, build_vanka_patches,
                      chebyshev_smooth, coarse_direct_solve, fgmres, vcycle)
from .general import GeneralStageSystem, GeneralTransfer
from .mhd import MHDDiscretization, MHDParams
from .stages import StageSystem, assemble_stage_operator
from .tableaux import ButcherTableau, tableau_lookup

__version__ = "0.1.0"
