"""The general stage-coupled operator path (host side of ``ivk_general_*``).

``StageSystem`` (stages.py) is the reference's Taylor--Hood structure
(``[[M + dt a K, dt a B], [dt a B^T, 0]]``, stages.py:63-126) stored in
scalar-node form.  Multi-field systems -- BASELINE config 5, resistive MHD
with (u, B) in vector P2 and (p, r) in P1 (mhd.py) -- have a spatial operator
L coupling every field, so this module keeps the same duck-typed API
(``dim``, ``matvec``, ``residual``, ``apply_into``, ``materialize``,
``pressure_nullspace``, ``project_pressure_means``, ...) over a general
single-stage CSR of (m, l) pairs shared by all stages:

    A_stage = I_s (x) M + dt A (x) L,   identity on constrained DoFs.

Patches are the vertex stars of the paper's Vanka relaxation (PAPER.md
"Vanka relaxation": every DoF on the closure of the cells around a vertex,
P1 fields only at the vertex itself), for every stage; ``VankaPatchSet``,
``MGHierarchyOp``, ``fgmres`` and ``CoarseSolver`` run on these objects
unchanged.  Kernels: K1g (apply), K7g (patch factor), K5g (transfers),
K8g (constrained seeding); K3/K3e and K4 are shared with the Stokes path.
"""

import numpy as np
import scipy.sparse as sp

from . import _lib
from .patches import PatchTables, star_closure_nodes
from .stages import to_sell

__all__ = ["GeneralStageSystem", "GeneralTransfer", "build_general_patch_tables"]


class GeneralStageSystem:
    """Stage system over a general single-stage operator.

    Parameters
    ----------
    rowptr, col, m, l : single-stage CSR (columns sorted per row) of the mass
        and the spatial operator on one pattern, already Dirichlet-eliminated.
    cmask : (n,) bool, constrained single-stage DoFs (identity rows).
    tableau, dt : Butcher tableau (``.A``, ``.r``) and time step.
    n_nodes, ncomp : scalar P2 nodes and the P2 components per node (the
        first ``ncomp * n_nodes`` DoFs interleave them per node).
    n_vertex_fields : P1 fields following the P2 block, one per vertex each.
    pressure_offset : start of the mean-free pressure block, which runs to
        the end of the stage vector (``project_pressure_means``).
    """

    _ivk_device_native = True   # takes / returns device tensors as well as numpy

    general = True
    convection = None

    def __init__(self, rowptr, col, m, l, cmask, tableau, dt, n_nodes, ncomp, n_vertex_fields,
                 pressure_offset):
        if dt < 0.0:
            raise ValueError("timestep must be nonnegative")
        self.rowptr = np.asarray(rowptr, dtype=np.int64)
        self.col = np.asarray(col, dtype=np.int32)
        self.m = np.asarray(m, dtype=np.float64)
        self.l = np.asarray(l, dtype=np.float64)
        self.cmask = np.asarray(cmask, dtype=bool)
        self.n1 = len(self.cmask)
        if len(self.rowptr) != self.n1 + 1 or self.rowptr[-1] != len(self.col):
            raise ValueError("inconsistent CSR arrays")
        self.tableau = tableau
        self.dt = float(dt)
        self.r = tableau.r
        if not 1 <= self.r <= _lib.IVK_MAX_STAGES:
            raise ValueError(f"{self.r} stages unsupported (max {_lib.IVK_MAX_STAGES})")
        self.n_nodes = int(n_nodes)
        self.nc = int(ncomp)
        self.n_vertex_fields = int(n_vertex_fields)
        self.n_vertices = (self.n1 - self.nc * self.n_nodes) // max(self.n_vertex_fields, 1)
        if self.nc * self.n_nodes + self.n_vertex_fields * self.n_vertices != self.n1:
            raise ValueError("layout does not match the operator size")
        self.n_u = int(pressure_offset)
        self.n_p = self.n1 - self.n_u
        self.constrained = np.flatnonzero(self.cmask).astype(np.int64)
        self._dev = None

    # -- layout helpers (stages.py:92-106, 169-186) -------------------------

    @property
    def stage_dim(self):
        return self.n1

    @property
    def dim(self):
        return self.r * self.n1

    def constrained_stage_dofs(self):
        offs = np.arange(self.r) * self.n1
        return (offs[:, None] + self.constrained[None, :]).ravel()

    def project_pressure_means(self, x):
        """Remove the per-stage mean of the pressure block in place; returns x.
        Always libivk: a numpy ``x`` is projected on the device and written
        back into the same array."""
        from ._device import is_device, ptr, stream, upload
        if not is_device(x):
            arr = np.asarray(x)
            if arr.dtype != np.float64 or arr.shape != (self.dim,):
                raise ValueError(f"expected a float64 vector of length {self.dim}")
            xd = upload(arr, np.float64)
            self.project_pressure_means(xd)
            arr[...] = xd.cpu().numpy()
            return x
        scratch = self.device_data()["tensors"]["proj_scratch"]
        _lib.check(_lib.lib().ivk_project_pressure_means(
            self.r, self.n_u, self.n_p, ptr(x), ptr(scratch), stream()), "project_pressure_means")
        return x

    def pressure_nullspace(self):
        Z = np.zeros((self.dim, self.r))
        for i in range(self.r):
            lo = i * self.n1 + self.n_u
            Z[lo:lo + self.n_p, i] = 1.0 / np.sqrt(self.n_p)
        return Z

    @property
    def M(self):
        return sp.csr_matrix((self.m, self.col, self.rowptr), shape=(self.n1, self.n1))

    def mark_host_stale(self):
        """The device operator was re-linearised; ``l`` is refreshed lazily."""
        self._host_stale = True

    def _sync_host(self):
        if getattr(self, "_host_stale", False):
            self.download_operator()

    @property
    def L(self):
        self._sync_host()
        return sp.csr_matrix((self.l, self.col, self.rowptr), shape=(self.n1, self.n1))

    def materialize(self, limit=200_000):
        """Explicit sparse stage matrix (stages.py:139-167): small systems only."""
        if self.dim > limit:
            raise ValueError(f"refusing to materialize {self.dim} stage dofs")
        A = np.asarray(self.tableau.A, dtype=np.float64)
        out = sp.kron(sp.identity(self.r), self.M) + self.dt * sp.kron(A, self.L)
        ones = np.zeros(self.dim)
        ones[self.constrained_stage_dofs()] = 1.0
        return (out + sp.diags(ones)).tocsr()

    # -- device data --------------------------------------------------------

    def device_data(self):
        if self._dev is not None:
            return self._dev
        from ._device import upload
        t = {}
        ml = np.column_stack([self.m, self.l])
        t["rowptr"] = upload(self.rowptr, np.int32)
        t["col"] = upload(self.col, np.int32)
        t["ml"] = upload(ml, np.float64)
        sptr, scol, sml = to_sell(self.rowptr, self.col, ml, self.n1, C=32)
        t["sptr"], t["scol"], t["sml"] = (upload(sptr, np.int32), upload(scol, np.int32),
                                          upload(sml, np.float64))
        t["cmask"] = upload(self.cmask.astype(np.uint8), np.uint8)
        import torch
        t["proj_scratch"] = torch.zeros(_lib.PROJECT_BLOCKS * self.r, dtype=torch.float64,
                                        device=t["cmask"].device)
        d = _lib.GeneralDesc()
        d.stages = self.r
        d.n = self.n1
        d.nnz = len(self.col)
        d.dt = self.dt
        A = np.asarray(self.tableau.A, dtype=np.float64)
        for i in range(self.r):
            for j in range(self.r):
                d.butcher_a[i * self.r + j] = A[i, j]
        d.rowptr, d.col, d.ml = t["rowptr"].data_ptr(), t["col"].data_ptr(), t["ml"].data_ptr()
        d.sptr, d.scol, d.sml = t["sptr"].data_ptr(), t["scol"].data_ptr(), t["sml"].data_ptr()
        d.constrained = t["cmask"].data_ptr()
        self._dev = {"tensors": t, "desc": d, "sell_entries": len(scol)}
        return self._dev

    @property
    def desc(self):
        return self.device_data()["desc"]

    def sell_pos(self):
        """Position of every CSR entry in the SELL-32 copy (``to_sell``)."""
        from .stages import sell_positions
        return sell_positions(self.rowptr, self.n1, C=32)[1]

    def download_operator(self):
        """Refresh the host ``l`` from the device CSR after a device
        re-linearisation (the coarse direct solve factorises on the host)."""
        self._host_stale = False
        if self._dev is not None:
            self.l = self._dev["tensors"]["ml"][:, 1].cpu().numpy().copy()

    def apply_into(self, x, b, out):
        """Device: out = b - A x (b is not None) or out = A x (K1g)."""
        from ._device import ptr, stream
        _lib.check(_lib.lib().ivk_general_apply(self.desc, ptr(x), ptr(b), ptr(out), stream()),
                   "general_apply")
        return out

    def matvec(self, x):
        from ._device import as_device_vector, to_host
        import torch
        xd, host = as_device_vector(x, self.dim)
        y = torch.empty_like(xd)
        self.apply_into(xd, None, y)
        return to_host(y) if host else y

    def residual(self, x, b):
        from ._device import as_device_vector, to_host
        import torch
        xd, host = as_device_vector(x, self.dim)
        bd, _ = as_device_vector(b, self.dim)
        r = torch.empty_like(xd)
        self.apply_into(xd, bd, r)
        return to_host(r) if host else r

    def seed_constrained_into(self, r, z):
        """Device: z = 0 except z[cd] = r[cd] (solvers.py:352-354)."""
        from ._device import ptr, stream
        _lib.check(_lib.lib().ivk_general_seed_constrained(self.desc, ptr(r), ptr(z), stream()),
                   "general_seed_constrained")
        return z

    # -- patches -------------------------------------------------------------

    def patch_tables(self, mesh, vertices=None):
        return build_general_patch_tables(mesh, self, vertices=vertices)

    def factor_patches(self, patch_desc, flag):
        """K7g on a patch descriptor; ``flag`` receives the smallest singular vertex."""
        from ._device import ptr, stream
        _lib.check(_lib.lib().ivk_general_patch_factor(self.desc, patch_desc, ptr(flag), stream()),
                   "general_patch_factor")

    def vanka_sweep(self, patch_desc, x, b, omega, w, r, local, out):
        from ._device import ptr, stream
        _lib.check(_lib.lib().ivk_general_vanka_sweep(self.desc, patch_desc, ptr(x), ptr(b),
                                                      float(omega), ptr(w), ptr(r), ptr(local),
                                                      ptr(out), stream()), "general_vanka_sweep")
        return out


def build_general_patch_tables(mesh, system, vertices=None):
    """Vertex-star patch tables of a general stage system (the layout of
    ``patches.build_patch_tables``: stage-major local lists, groups by size
    ascending then vertex ascending, solvers.py:132-175).

    Patch v holds, for every stage, the unconstrained single-stage DoFs of
    every P2 component on the closure of star(v) and of every P1 field at v,
    ascending.  ``node``/``node_off`` hold the stage-0 (single-stage) lists."""
    nv = mesh.num_vertices
    n_nodes, nc, nf, n1 = system.n_nodes, system.nc, system.n_vertex_fields, system.n1
    if n_nodes != nv + mesh.num_edges or system.n_vertices != nv:
        raise ValueError("mesh does not match the system layout")
    stages = system.r
    dim = stages * n1
    starts, nodes = star_closure_nodes(mesh)
    owner = np.repeat(np.arange(nv), np.diff(starts))
    # P2 DoFs of each (vertex, node) pair, then the vertex's P1 DoFs
    w_dofs = (nc * nodes[:, None] + np.arange(nc)[None, :]).ravel()
    w_own = np.repeat(owner, nc)
    base = nc * n_nodes
    v_dofs = (base + np.arange(nf)[None, :] * nv + np.arange(nv)[:, None]).ravel()
    v_own = np.repeat(np.arange(nv), nf)
    own = np.concatenate([w_own, v_own])
    dofs = np.concatenate([w_dofs, v_dofs])
    keep = ~system.cmask[dofs]
    own, dofs = own[keep], dofs[keep]
    order_ = np.lexsort((dofs, own))
    own, dofs = own[order_], dofs[order_]
    cnt = np.bincount(own, minlength=nv)
    size_of_v = stages * cnt
    order = np.argsort(size_of_v, kind="stable")
    if vertices is not None:
        sel = np.zeros(nv, dtype=bool)
        sel[np.asarray(vertices, dtype=np.int64)] = True
        order = order[sel[order]]
    sizes = size_of_v[order]
    bb = cnt[order]
    vstart = np.concatenate([[0], np.cumsum(cnt)])
    from .patches import _ranges
    single = dofs[_ranges(vstart[order], bb)]                     # stage-0 lists, flat
    node_off = np.concatenate([[0], np.cumsum(bb)]).astype(np.int64)
    idx_off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    total_m = int(idx_off[-1])
    idx = np.empty(total_m, dtype=np.int64)
    P = len(order)
    slot = np.repeat(np.arange(P), bb)
    k = np.arange(len(single)) - node_off[slot]
    for s in range(stages):
        idx[idx_off[slot] + s * bb[slot] + k] = s * n1 + single
    ld = (sizes + 3) & ~3
    inv_off = np.concatenate([[0], np.cumsum(sizes.astype(np.int64) * ld)]).astype(np.int64)
    mult = np.bincount(idx, minlength=dim)
    dof_pos = np.argsort(idx, kind="stable")
    dof_ptr = np.concatenate([[0], np.cumsum(mult)]).astype(np.int64)
    return PatchTables(num_patches=P, dim=dim, stages=stages, order=order, sizes=sizes,
                       idx_off=idx_off, idx=idx, node_off=node_off, node=single,
                       inv_off=inv_off[:-1], inv_size=int(inv_off[-1]),
                       dof_ptr=dof_ptr, dof_pos=dof_pos, multiplicity=mult)


class GeneralTransfer:
    """I_s (x) P for a single-stage CSR transfer P (fine x coarse), with its
    transpose stored explicitly (bench.py:187-194; solvers.py:340-346)."""

    def __init__(self, P, stages, fine_cmask, coarse_cmask):
        self.P = sp.csr_matrix(P)
        self.P.sort_indices()
        self.stages = int(stages)
        self.nf, self.nc = self.P.shape
        self.fine_cm = np.asarray(fine_cmask, dtype=bool)
        self.coarse_cm = np.asarray(coarse_cmask, dtype=bool)
        if len(self.fine_cm) != self.nf or len(self.coarse_cm) != self.nc:
            raise ValueError("constrained masks do not match the transfer")
        self._dev = None

    @property
    def shape(self):
        return (self.stages * self.nf, self.stages * self.nc)

    @property
    def matrix(self):
        return sp.kron(sp.identity(self.stages), self.P, format="csr")

    def device_data(self):
        if self._dev is not None:
            return self._dev
        from ._device import upload
        t = {}
        PT = self.P.T.tocsr()
        PT.sort_indices()
        for name, m in (("p", self.P), ("pt", PT)):
            t[name + "_rowptr"] = upload(m.indptr, np.int32)
            t[name + "_col"] = upload(m.indices, np.int32)
            t[name + "_val"] = upload(m.data, np.float64)
        t["fcm"] = upload(self.fine_cm.astype(np.uint8), np.uint8)
        t["ccm"] = upload(self.coarse_cm.astype(np.uint8), np.uint8)
        d = _lib.GeneralTransferDesc()
        d.stages, d.nf, d.nc = self.stages, self.nf, self.nc
        for name in ("p", "pt"):
            for f in ("rowptr", "col", "val"):
                setattr(d, f"{name}_{f}", t[f"{name}_{f}"].data_ptr())
        d.fine_constrained = t["fcm"].data_ptr()
        d.coarse_constrained = t["ccm"].data_ptr()
        self._dev = {"tensors": t, "desc": d}
        return self._dev

    def restrict_into(self, rf, rc):
        from ._device import ptr, stream
        _lib.check(_lib.lib().ivk_general_restrict(self.device_data()["desc"], ptr(rf), ptr(rc),
                                                   stream()), "general_restrict")
        return rc

    def prolong_add(self, ec, xf):
        from ._device import ptr, stream
        _lib.check(_lib.lib().ivk_general_prolong_add(self.device_data()["desc"], ptr(ec), ptr(xf),
                                                      stream()), "general_prolong_add")
        return xf
