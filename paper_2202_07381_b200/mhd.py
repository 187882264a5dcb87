"""2-D incompressible resistive MHD, Newton-linearised (BASELINE config 5).

The paper (PAPER.md, "Magnetohydrodynamics", eq. MHD semi-discrete) solves
single-fluid visco-resistive MHD in the formulation of its [scottmhd]
reference with a monolithic IRK-Vanka multigrid; the reference package
implements only Stokes / Navier--Stokes, so this module is
new host setup feeding the same device path.  BASELINE config 5 fixes the
discretisation: velocity u and magnetic field B in vector P2, pressure p
and magnetic Lagrange multiplier r in P1, on the right-triangle grids.

Linearisation about a frozen state (u0, B0), trial (u, B, r, p), test
(v, c, s, q), 2-D curls j(B) = d_x B_y - d_y B_x, X x Y = X_x Y_y - X_y Y_x,
z^ x X = (-X_y, X_x):

    (u_t, v) + (2/Re)(eps(u), eps(v)) + ((u0.grad)u + (u.grad)u0, v)
        - S (j(B) z^ x B0 + j(B0) z^ x B, v) - (p, div v)
    (B_t, c) + (1/Rm)(j(B), j(c)) - (u x B0 + u0 x B, j(c)) - (grad r, c)
    -(div u, q)
    -(B, grad s)

with u = 0 and B x n = 0 on the boundary of the unit square (u fully,
the tangential B component per side) and r in H^1_0 (r = 0 on boundary
vertices); p has the constant null space (mean-zero pressure).  Every
stage shares the frozen state, so the stage system is
``I_s (x) M + dt A (x) L`` with one single-stage operator L (and mass M on
u, B) -- the general operator path (``general.py``, kernels ``ivk_general_*``).

Single-stage DoF layout: ``[w | r | p]`` where w interleaves
(u_x, u_y, B_x, B_y) per scalar P2 node (node n owns w DoFs 4n .. 4n+3),
then one r and one p per vertex.  All forms are integrated with the
degree-5 triangle rule, exact for every term (the highest is degree 5:
P2 state x P1 gradient x P2 test).
"""

import numpy as np
import scipy.sparse as sp

from . import _lib, fem
from .fem import _affine, _coo_to_csr, _physical_gradients, p2_cell_nodes, p2_node_coords
from .discretization import ConfigError, streamfunction_velocity
from .mesh import build_hierarchy
from .quadrature import p1_basis, p2_basis, triangle_rule

__all__ = ["MHDParams", "MHDDiscretization", "assemble_mhd", "mhd_boundary_dofs",
           "mhd_prolongation", "mhd_magnetic_state", "MHDAssembler", "NCOMP_W"]

NCOMP_W = 4          # (u_x, u_y, B_x, B_y) per scalar P2 node
DEG_MHD = 5


class MHDParams:
    def __init__(self, Re=100.0, Rm=100.0, S=1.0):
        if Re <= 0 or Rm <= 0:
            raise ValueError("Reynolds numbers must be positive")
        self.Re, self.Rm, self.S = float(Re), float(Rm), float(S)


def mhd_magnetic_state(points):
    """B0 = (1, 0) + 0.1 curl(sin(2 pi x) sin(2 pi y)), curl f = (d_y f, -d_x f)
    (BASELINE config 5)."""
    x, y = points[:, 0], points[:, 1]
    tp = 2.0 * np.pi
    return np.column_stack([1.0 + 0.1 * tp * np.sin(tp * x) * np.cos(tp * y),
                            -0.1 * tp * np.cos(tp * x) * np.sin(tp * y)])


def _layout(mesh):
    nv = mesh.num_vertices
    n_nodes = nv + mesh.num_edges
    return n_nodes, nv, NCOMP_W * n_nodes + 2 * nv


def cell_dofs(mesh):
    """(C, 30) single-stage DoFs of each cell: w (6 nodes x 4 comps), r (3), p (3)."""
    n_nodes, nv, _ = _layout(mesh)
    nodes = p2_cell_nodes(mesh)
    w = (NCOMP_W * nodes[:, :, None] + np.arange(NCOMP_W)[None, None, :]).reshape(-1, 24)
    r = NCOMP_W * n_nodes + mesh.cells
    p = NCOMP_W * n_nodes + nv + mesh.cells
    return np.hstack([w, r, p]).astype(np.int64)


def element_matrices(mesh, u0, B0, params):
    """Element mass and linearised operator, each (C, 30, 30), local order of
    ``cell_dofs``.  ``u0``, ``B0``: (n_nodes, 2) nodal P2 values."""
    nodes = p2_cell_nodes(mesh)
    _, jinv, det = _affine(mesh)
    C = len(nodes)
    pts, w = triangle_rule(DEG_MHD)
    phi, dphi = p2_basis(pts)                       # (6, Q), (6, Q, 2)
    psi, dpsi = p1_basis(pts)                       # (3, Q), (3, 2)
    G = _physical_gradients(dphi, jinv)             # (C, 6, Q, 2)
    gpsi = np.einsum("ie,ced->cid", dpsi, jinv)     # (C, 3, 2)
    wq = w[None, :] * det[:, None]                  # (C, Q)
    u0c, B0c = u0[nodes], B0[nodes]                 # (C, 6, 2)
    u0q = np.einsum("cad,aq->cqd", u0c, phi)
    B0q = np.einsum("cad,aq->cqd", B0c, phi)
    gu0 = np.einsum("cad,caqe->cqde", u0c, G)       # d_e u0_d
    gB0 = np.einsum("cad,caqe->cqde", B0c, G)
    j0 = gB0[:, :, 1, 0] - gB0[:, :, 0, 1]          # d_x B0_y - d_y B0_x
    jc = np.stack([-G[..., 1], G[..., 0]], axis=-1)  # j(phi_a e_g) = jc[c, a, q, g]
    Re, Rm, S = params.Re, params.Rm, params.S

    mass = np.einsum("cq,aq,bq->cab", wq, phi, phi)
    lap = np.einsum("cq,caqd,cbqd->cab", wq, G, G)
    gg = np.einsum("cq,caqf,cbqd->cabfd", wq, G, G)              # d_f phi_a d_d phi_b
    adv = np.einsum("cq,aq,cqe,cbqe->cab", wq, phi, u0q, G, optimize=True)
    cu = np.einsum("cq,aq,bq,cqde->cabde", wq, phi, phi, gu0, optimize=True)
    eye2 = np.eye(2)

    Me = np.zeros((C, 30, 30))
    Le = np.zeros((C, 30, 30))
    uu = np.zeros((C, 6, 2, 6, 2))       # test (a, d), trial (b, f)
    uB = np.zeros((C, 6, 2, 6, 2))       # test (a, d), trial (b, g)
    Bu = np.zeros((C, 6, 2, 6, 2))       # test (a, h), trial (b, f)
    BB = np.zeros((C, 6, 2, 6, 2))       # test (a, h), trial (b, g)

    # (2/Re)(eps(u), eps(v)) = (1/Re)[delta_df grad.grad + d_f phi_a d_d phi_b]
    uu += (1.0 / Re) * (lap[:, :, None, :, None] * eye2[None, None, :, None, :]
                        + np.transpose(gg, (0, 1, 4, 2, 3)))
    # ((u0.grad)u + (u.grad)u0, v): delta_df phi_a (u0.grad phi_b) + phi_a phi_b d_f u0_d
    uu += adv[:, :, None, :, None] * eye2[None, None, :, None, :]
    uu += np.transpose(cu, (0, 1, 3, 2, 4))
    # -S (j(B) z^xB0 + j(B0) z^xB, v)
    zB0 = np.stack([-B0q[..., 1], B0q[..., 0]], axis=-1)          # (C, Q, 2) index d
    Z = np.array([[0.0, 1.0], [-1.0, 0.0]])                        # (z^ x e_g)_d = Z[g, d]
    uB += -S * np.einsum("cq,aq,cqd,cbqg->cadbg", wq, phi, zB0, jc, optimize=True)
    uB += -S * np.einsum("cq,aq,bq,cq,gd->cadbg", wq, phi, phi, j0, Z, optimize=True)
    # -(u x B0, j(c)):  (e_f x B0) = (B0_y, -B0_x)[f]
    cB0 = np.stack([B0q[..., 1], -B0q[..., 0]], axis=-1)
    Bu += -np.einsum("cq,bq,cqf,caqh->cahbf", wq, phi, cB0, jc, optimize=True)
    # -(u0 x B, j(c)):  (u0 x e_g) = (-u0_y, u0_x)[g];  + (1/Rm)(j(B), j(c))
    cu0 = np.stack([-u0q[..., 1], u0q[..., 0]], axis=-1)
    BB += -np.einsum("cq,bq,cqg,caqh->cahbg", wq, phi, cu0, jc, optimize=True)
    BB += (1.0 / Rm) * np.einsum("cq,cbqg,caqh->cahbg", wq, jc, jc, optimize=True)

    def put(dst, blk, r0, c0):
        # blk (C, 6, 2, 6, 2) -> rows 4a + r0 + d, cols 4b + c0 + f
        for d in range(2):
            for f in range(2):
                dst[:, r0 + d:24:4, c0 + f:24:4] += blk[:, :, d, :, f]

    put(Le, uu, 0, 0)
    put(Le, uB, 0, 2)
    put(Le, Bu, 2, 0)
    put(Le, BB, 2, 2)
    for k in range(NCOMP_W):
        Me[:, k:24:4, k:24:4] = mass
    # pressure: -(p, div v) and -(div u, q)
    bp = -np.einsum("cq,iq,caqd->cadi", wq, psi, G)                # (C, 6, 2, 3)
    # multiplier: -(grad r, c) and -(B, grad s)
    br = -np.einsum("cq,aq,cih->cahi", wq, phi, gpsi)              # (C, 6, 2, 3)
    for d in range(2):
        Le[:, d:24:4, 27:30] = bp[:, :, d, :]
        Le[:, 27:30, d:24:4] = np.transpose(bp[:, :, d, :], (0, 2, 1))
        Le[:, 2 + d:24:4, 24:27] = br[:, :, d, :]
        Le[:, 24:27, 2 + d:24:4] = np.transpose(br[:, :, d, :], (0, 2, 1))
    return Me, Le


def mhd_boundary_dofs(mesh, tol=1e-12):
    """Constrained single-stage DoFs: u (both components) on boundary nodes,
    the tangential B component per side of the unit square (B_y on x = 0, 1;
    B_x on y = 0, 1; both at corners), r on boundary vertices."""
    n_nodes, nv, _ = _layout(mesh)
    bnodes = fem.velocity_boundary_nodes(mesh)
    xy = p2_node_coords(mesh)[bnodes]
    on_x = (np.abs(xy[:, 0]) < tol) | (np.abs(xy[:, 0] - 1.0) < tol)
    on_y = (np.abs(xy[:, 1]) < tol) | (np.abs(xy[:, 1] - 1.0) < tol)
    if not np.all(on_x | on_y):
        raise ValueError("MHD boundary conditions assume the unit square")
    out = [NCOMP_W * bnodes, NCOMP_W * bnodes + 1,
           NCOMP_W * bnodes[on_y] + 2, NCOMP_W * bnodes[on_x] + 3,
           NCOMP_W * n_nodes + np.flatnonzero(mesh.boundary_vertex_flags)]
    return np.unique(np.concatenate(out)).astype(np.int64)


def element_structure():
    """(30, 30) bool: the element couplings the linearised MHD form can make
    nonzero for any state (u, B among themselves; u-p and B-r saddle pairs)."""
    st = np.zeros((30, 30), dtype=bool)
    st[:24, :24] = True
    uu = np.arange(24)[np.arange(24) % 4 < 2]
    bb = np.arange(24)[np.arange(24) % 4 >= 2]
    st[np.ix_(uu, np.arange(27, 30))] = True
    st[np.ix_(np.arange(27, 30), uu)] = True
    st[np.ix_(bb, np.arange(24, 27))] = True
    st[np.ix_(np.arange(24, 27), bb)] = True
    return st


def assemble_mhd(mesh, params, u0_func=streamfunction_velocity, B0_func=mhd_magnetic_state,
                 constrained=None):
    """Single-stage CSR (rowptr, col, m, l) of the mass and the linearised
    operator on one shared pattern, Dirichlet-eliminated (constrained rows
    and columns dropped; the stage operator puts identity rows there).  The
    pattern is structural (``element_structure``), not value-dependent, so a
    device re-linearisation (``MHDAssembler``) fills the same entries."""
    n_nodes, nv, n1 = _layout(mesh)
    xy = p2_node_coords(mesh)
    u0 = np.asarray(u0_func(xy), dtype=np.float64)
    B0 = np.asarray(B0_func(xy), dtype=np.float64)
    Me, Le = element_matrices(mesh, u0, B0, params)
    dofs = cell_dofs(mesh)
    rows = np.repeat(dofs[:, :, None], 30, axis=2)
    cols = np.repeat(dofs[:, None, :], 30, axis=1)
    nzr = np.broadcast_to(element_structure(), Me.shape)
    rowptr, col, ml = _coo_to_csr(rows[nzr], cols[nzr], np.stack([Me[nzr], Le[nzr]], axis=-1),
                                  n1, n1)
    if constrained is None:
        constrained = mhd_boundary_dofs(mesh)
    cmask = np.zeros(n1, dtype=bool)
    cmask[constrained] = True
    r_of = np.repeat(np.arange(n1), np.diff(rowptr))
    keep = ~(cmask[r_of] | cmask[col])
    counts = np.bincount(r_of[keep], minlength=n1)
    rowptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    return rowptr, col[keep], np.ascontiguousarray(ml[keep, 0]), \
        np.ascontiguousarray(ml[keep, 1]), cmask


class MHDAssembler:
    """Device re-linearisation of one level's operator L at a new frozen state
    (K10g, ``ivk_mhd_assemble``): element rows by the formulas of
    ``element_matrices``, then a deterministic per-entry gather (cell order,
    the order ``assemble_mhd`` sums in) into the l half of the system's CSR
    and SELL-32 (m, l) pairs.  The mass half and every index table of the
    stage system, patches and transfers stay as they are."""

    def __init__(self, mesh, params, system):
        self.params = params
        nodes = p2_cell_nodes(mesh)
        _, jinv, det = _affine(mesh)
        self.cell_nodes = nodes
        self.cell_geo = np.column_stack([jinv.reshape(-1, 4), det])
        C_ = len(nodes)
        n1 = system.n1
        cmask = system.cmask
        dofs = cell_dofs(mesh)
        ii, jj = np.nonzero(element_structure())
        r, c = dofs[:, ii], dofs[:, jj]
        contrib = np.arange(C_, dtype=np.int64)[:, None] * 900 + (ii * 30 + jj)[None, :]
        keep = ~(cmask[r] | cmask[c])
        key = (r.astype(np.int64) * n1 + c)[keep]
        contrib = contrib[keep]
        order = np.argsort(key, kind="stable")        # cell-ascending within an entry
        rows = np.repeat(np.arange(n1), np.diff(system.rowptr))
        pkey = rows.astype(np.int64) * n1 + system.col
        if not np.array_equal(np.unique(key), pkey):
            raise ValueError("cell connectivity does not match the operator pattern")
        counts = np.bincount(np.searchsorted(pkey, key[order]), minlength=len(pkey))
        self.entry_ptr = np.concatenate([[0], np.cumsum(counts)])
        self.entry_contrib = contrib[order]
        if self.entry_contrib.max(initial=0) >= 2 ** 31:
            raise ValueError("level too large for 32-bit contribution indices")
        self.sell_pos = system.sell_pos()
        self.n_cells, self.nnz = C_, len(pkey)
        self.n_nodes = system.n_nodes
        pts, w = triangle_rule(DEG_MHD)
        phi, dphi = p2_basis(pts)
        psi, dpsi = p1_basis(pts)
        d = _lib.MHDDesc()
        d.n_cells, d.nnz, d.nq = C_, len(pkey), len(w)
        if d.nq > _lib.IVK_MAX_QUAD:
            raise ValueError("quadrature rule too large")
        d.Re, d.Rm, d.S = params.Re, params.Rm, params.S
        for q in range(d.nq):
            d.w[q] = w[q]
            for a in range(6):
                d.phi[q * 6 + a] = phi[a, q]
                d.dphi[(q * 6 + a) * 2] = dphi[a, q, 0]
                d.dphi[(q * 6 + a) * 2 + 1] = dphi[a, q, 1]
            for v in range(3):
                d.psi[q * 3 + v] = psi[v, q]
        for v in range(3):
            d.dpsi[2 * v], d.dpsi[2 * v + 1] = dpsi[v, 0], dpsi[v, 1]
        self.desc = d
        self._dev = None

    def _device(self):
        if self._dev is None:
            import torch
            from ._device import upload
            t = {"cell_geo": upload(self.cell_geo, np.float64),
                 "cell_nodes": upload(self.cell_nodes, np.int32),
                 "entry_ptr": upload(self.entry_ptr, np.int32),
                 "entry_contrib": upload(self.entry_contrib, np.int32),
                 "sell_pos": upload(self.sell_pos, np.int32)}
            t["scratch"] = torch.empty(self.n_cells * 900, dtype=torch.float64,
                                       device=t["cell_geo"].device)
            d = self.desc
            d.cell_geo, d.cell_nodes = t["cell_geo"].data_ptr(), t["cell_nodes"].data_ptr()
            d.entry_ptr = t["entry_ptr"].data_ptr()
            d.entry_contrib = t["entry_contrib"].data_ptr()
            d.sell_pos = t["sell_pos"].data_ptr()
            self._dev = t
        return self._dev

    def assemble_into_system(self, system, u0, B0):
        """Overwrite ``system``'s device l values (CSR and SELL) with the
        operator linearised about device nodal states u0, B0 ((n_nodes, 2) or
        flat, this level's nodes)."""
        from ._device import ptr, stream
        t = self._device()
        sd = system.device_data()["tensors"]
        u0 = u0.reshape(-1)[:2 * self.n_nodes].contiguous()
        B0 = B0.reshape(-1)[:2 * self.n_nodes].contiguous()
        _lib.check(_lib.lib().ivk_mhd_assemble(self.desc, ptr(u0), ptr(B0), ptr(t["scratch"]),
                                               ptr(sd["ml"]), ptr(sd["sml"]), stream()),
                   "mhd_assemble")


def mhd_prolongation(hier, level):
    """Single-stage nested interpolation level -> level + 1 in the [w | r | p]
    layout: blockdiag(P_P2 (x) I_4, P_P1, P_P1)."""
    p2 = fem.prolongation(hier, level, "p2")
    p1 = fem.prolongation(hier, level, "p1")
    return sp.block_diag([sp.kron(p2, sp.identity(NCOMP_W)), p1, p1], format="csr")


class MHDDiscretization:
    """Per-level MHD setup and the V-cycle constructor (the config-5 analogue
    of ``Discretization.build_mg``, reference bench.py:206-228)."""

    def __init__(self, n0, level, params=None, grid="diagonal",
                 u0_func=streamfunction_velocity, B0_func=mhd_magnetic_state):
        self.params = params if params is not None else MHDParams()
        self.hier = build_hierarchy(n0, level, grid)
        self.ops = []
        for m in self.hier.levels:
            rowptr, col, mv, lv, cmask = assemble_mhd(m, self.params, u0_func, B0_func)
            self.ops.append(dict(rowptr=rowptr, col=col, m=mv, l=lv, cmask=cmask,
                                 layout=_layout(m)))
        self._prolong = [mhd_prolongation(self.hier, k) for k in range(self.hier.num_levels - 1)]
        self._stage_prolong = {}
        self._assemblers = {}

    @property
    def num_levels(self):
        return self.hier.num_levels

    @property
    def fine_mesh(self):
        return self.hier.levels[-1]

    def system(self, level, tableau, dt):
        from .general import GeneralStageSystem
        o = self.ops[level]
        n_nodes, nv, n1 = o["layout"]
        return GeneralStageSystem(o["rowptr"], o["col"], o["m"], o["l"], o["cmask"], tableau, dt,
                                  n_nodes=n_nodes, ncomp=NCOMP_W, n_vertex_fields=2,
                                  pressure_offset=n1 - nv)

    def stage_prolong(self, level, r):
        from .general import GeneralTransfer
        key = (level, r)
        if key not in self._stage_prolong:
            self._stage_prolong[key] = GeneralTransfer(self._prolong[level - 1], r,
                                                       self.ops[level]["cmask"],
                                                       self.ops[level - 1]["cmask"])
        return self._stage_prolong[key]

    def build_mg(self, tableau, dt, smoother, mg_levels=None, convection=None, use_graph=False,
                 patch_mode="auto"):
        """(MGHierarchyOp, finest GeneralStageSystem); the frozen linearisation
        state is part of the operator, so ``convection`` must be None."""
        from .solvers import MGHierarchyOp, MGLevel, VankaPatchSet, coarse_direct_solve
        if convection is not None:
            raise ConfigError("the MHD operator carries its own linearisation state")
        total = self.num_levels
        depth = total if mg_levels is None else int(mg_levels)
        if not 1 <= depth <= total:
            raise ConfigError(f"mg.levels must lie in [1, {total}]")
        start = total - depth
        levels = []
        for k in range(start, total):
            system = self.system(k, tableau, dt)
            patches = VankaPatchSet(system, self.hier.levels[k], factor=(k > start),
                                    mode=patch_mode)
            P = self.stage_prolong(k, tableau.r) if k > start else None
            levels.append(MGLevel(system, patches, smoother, P))
        coarse = coarse_direct_solve(levels[0].system)
        return MGHierarchyOp(levels, coarse, use_graph=use_graph), levels[-1].system

    def assembler(self, level, system):
        """The level's device assembler (its maps depend only on the level's
        operator pattern, shared by every stage system built on it)."""
        if level not in self._assemblers:
            self._assemblers[level] = MHDAssembler(self.hier.levels[level], self.params, system)
        return self._assemblers[level]

    def relinearize(self, mg, u0, B0):
        """Re-linearise every level of ``mg`` about the fine-level device state
        (u0, B0) -- (n_nodes, 2) nodal P2 values, injected to coarser levels as
        the nodal prefix (nested P2 node numbering, as the reference's
        ``inject_velocity``) -- then refactorise the smoothed levels' patches in
        place (K7g) and re-form the coarse operator (on the device for the dense
        coarse method): the Newton-cadence update of config 5."""
        from .solvers import coarse_direct_solve
        start = self.num_levels - len(mg.levels)
        for lv, lev in enumerate(mg.levels):
            self.assembler(start + lv, lev.system).assemble_into_system(lev.system, u0, B0)
            if lv > 0:
                lev.patches.factor()
                lev.system.mark_host_stale()
        s0 = mg.levels[0].system
        if getattr(mg.coarse, "method", "dense") == "dense":
            # coarse operator straight from the re-assembled device operator
            from .solvers import CoarseSolver
            s0.mark_host_stale()
            mg.coarse = CoarseSolver.from_device_operator(s0)
        else:
            s0.download_operator()
            mg.coarse = coarse_direct_solve(s0, mg.coarse.method)
        mg._graph = None
        mg._bufs = None
