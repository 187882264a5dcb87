"""The stage-coupled saddle-point operator (host mirror of the reference
``StageSystem``, /root/reference/pkg/src/irkmg/stages.py:47-186).

    [ I_s (x) diag(M, 0)  +  dt A (x) [[K, B], [B^T, 0]] ] k = F

Vectors are stage-major ``[(u_1, p_1), ..., (u_s, p_s)]``.  The operator
apply (``matvec``) and the residual run in libivk (kernel K1); this class
owns the eliminated scalar-node data on the device and keeps the
reference's layout helpers on the host.
"""

import ctypes as C
import os

import numpy as np
import scipy.sparse as sp

from . import _lib
from .fem import ConvectionBlocks, StokesBlocks
from .k1tiles import build_k1_tiles

__all__ = ["StageSystem", "assemble_stage_operator", "to_sell"]


def sell_positions(rowptr, n_rows, C=32):
    """(sptr, pos): the SELL-C slice pointers of ``to_sell`` and the position
    of every CSR entry in the SELL arrays."""
    rowptr = np.asarray(rowptr, dtype=np.int64)
    lens = np.diff(rowptr)
    nsl = (n_rows + C - 1) // C
    padded = np.zeros(nsl * C, dtype=np.int64)
    padded[:n_rows] = lens
    width = padded.reshape(nsl, C).max(axis=1)
    sptr = np.concatenate([[0], np.cumsum(width * C)])
    rows = np.repeat(np.arange(n_rows), lens)
    ent = np.arange(len(rows)) - rowptr[rows]
    return sptr, sptr[rows // C] + ent * C + rows % C


def to_sell(rowptr, col, vals, n_rows, pad_col=None, C=32):
    """CSR -> SELL-C (slices of C rows, entry e of a slice's lane-th row at
    ptr[slice] + C e + lane).  Padding entries get zero values and a valid
    column (the row itself, or ``pad_col``)."""
    rowptr = np.asarray(rowptr, dtype=np.int64)
    lens = np.diff(rowptr)
    nsl = (n_rows + C - 1) // C
    padded = np.zeros(nsl * C, dtype=np.int64)
    padded[:n_rows] = lens
    width = padded.reshape(nsl, C).max(axis=1)
    sptr = np.concatenate([[0], np.cumsum(width * C)])
    total = int(sptr[-1])
    rows = np.repeat(np.arange(n_rows), lens)
    ent = np.arange(len(rows)) - rowptr[rows]
    pos = sptr[rows // C] + ent * C + rows % C
    fill_rows = np.repeat(np.arange(nsl * C), np.repeat(width, C))
    scol = (np.minimum(fill_rows, n_rows - 1) if pad_col is None
            else np.full(total, pad_col)).astype(np.int32)
    scol[pos] = col
    vals = np.asarray(vals)
    sval = np.zeros((total,) + vals.shape[1:], dtype=vals.dtype)
    sval[pos] = vals
    return sptr.astype(np.int32), scol, sval


class StageSystem:
    """Drop-in for the reference ``StageSystem`` (stages.py:47-88).

    Parameters
    ----------
    blocks : StokesBlocks
        Raw (non-eliminated) scalar-node M, K, B.
    tableau : ButcherTableau (needs ``.A`` and ``.r``)
    dt : float
    constrained : int array of constrained velocity DoFs (interleaved);
        both components of a node must be constrained together, which is
        what ``velocity_boundary_dofs`` produces (fem.py:420-427).
    convection : optional list of s ConvectionBlocks (row-stage Jacobians
        J_N(u_i), stages.py:118-123); the same object repeated means one
        shared Jacobian.
    """

    _ivk_device_native = True   # takes / returns device tensors as well as numpy

    def __init__(self, blocks, tableau, dt, constrained=None, convection=None):
        if dt < 0.0:
            raise ValueError("timestep must be nonnegative")
        if not isinstance(blocks, StokesBlocks):
            raise TypeError("blocks must be a StokesBlocks (scalar-node form)")
        self.blocks = blocks
        self.tableau = tableau
        self.dt = float(dt)
        self.n_nodes = blocks.n_nodes
        self.nc = blocks.ncomp          # velocity components per scalar node (2; 3 in 3-D)
        self.n_u = blocks.n_u
        self.n_p = blocks.n_p
        self.r = tableau.r
        if not 1 <= self.r <= _lib.IVK_MAX_STAGES:
            raise ValueError(f"{self.r} stages unsupported (max {_lib.IVK_MAX_STAGES})")
        self.constrained = np.asarray(constrained if constrained is not None else [],
                                      dtype=np.int64)
        if convection is not None and len(convection) != self.r:
            raise ValueError("one convection Jacobian per stage required")
        if convection is not None and self.nc != 2:
            raise ValueError("convection is implemented for 2-D operators only")

        c = self.constrained
        node_mask = np.zeros(self.n_nodes, dtype=bool)
        if len(c):
            if c.min() < 0 or c.max() >= self.n_u:
                raise ValueError("constrained DoF out of range")
            nc = self.nc
            nodes = np.unique(c // nc)
            full = np.sort(np.concatenate([nc * nodes + d for d in range(nc)]))
            if not np.array_equal(full, np.unique(c)):
                raise ValueError("both velocity components of a constrained node must be "
                                 "constrained (node-level Dirichlet elimination)")
            node_mask[nodes] = True
        self.node_constrained = node_mask
        self._cmask = np.repeat(node_mask, self.nc)

        # Elimination D A D / D B (stages.py:77-85, fem.py:304-315), on the
        # scalar pattern: zero every entry touching a constrained node.
        rows = np.repeat(np.arange(self.n_nodes), np.diff(blocks.rowptr))
        keep = ~(node_mask[rows] | node_mask[blocks.col])
        self._m = np.where(keep, blocks.m, 0.0)
        self._k = np.where(keep, blocks.k, 0.0)
        brows = np.repeat(np.arange(self.n_nodes), np.diff(blocks.b_rowptr))
        self._b = np.where(node_mask[brows][:, None], 0.0, blocks.b_val)
        self._brows = brows

        self.convection = None
        self._conv_vals = None
        if convection is not None:
            for J in convection:
                if not isinstance(J, ConvectionBlocks):
                    raise TypeError("convection entries must be ConvectionBlocks")
                if not (np.array_equal(J.rowptr, blocks.rowptr) and np.array_equal(J.col, blocks.col)):
                    raise ValueError("convection Jacobian is not on the scalar P2 pattern")
            shared = all(J is convection[0] for J in convection)
            uniq = [convection[0]] if shared else list(convection)
            self._conv_vals = [np.where(keep[:, None, None], J.val, 0.0) for J in uniq]
            self.convection = list(convection)
        self._dev = None

    # -- layout helpers (stages.py:92-106, 169-186) -------------------------

    @property
    def stage_dim(self):
        return self.n_u + self.n_p

    @property
    def dim(self):
        return self.r * self.stage_dim

    def split(self, x):
        blocks = np.asarray(x).reshape(self.r, self.stage_dim)
        return blocks[:, :self.n_u], blocks[:, self.n_u:]

    def join(self, u, p):
        return np.hstack([u, p]).ravel()

    def constrained_stage_dofs(self):
        offs = np.arange(self.r) * self.stage_dim
        return (offs[:, None] + self.constrained[None, :]).ravel()

    def project_pressure_means(self, x):
        """Remove the per-stage constant pressure in place; returns ``x``
        (stages.py:174-178).  Always libivk (K8): a numpy ``x`` is copied to
        the device, projected there and written back into the same array."""
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
            lo = i * self.stage_dim + self.n_u
            Z[lo:lo + self.n_p, i] = 1.0 / np.sqrt(self.n_p)
        return Z

    # -- eliminated vector-P2 views (reference layout, host) -----------------

    def _scalar(self, vals):
        b = self.blocks
        return sp.csr_matrix((vals, b.col, b.rowptr), shape=(self.n_nodes, self.n_nodes))

    @property
    def M(self):
        return sp.kron(self._scalar(self._m), sp.identity(self.nc), format="csr")

    @property
    def K(self):
        return sp.kron(self._scalar(self._k), sp.identity(self.nc), format="csr")

    @property
    def B(self):
        nc = self.nc
        r = np.concatenate([nc * self._brows + d for d in range(nc)])
        c = np.concatenate([self.blocks.b_col] * nc).astype(np.int64)
        v = np.concatenate([self._b[:, d] for d in range(nc)])
        return sp.csr_matrix((v, (r, c)), shape=(self.n_u, self.n_p))

    @property
    def BT(self):
        return self.B.T.tocsr()

    def mark_host_stale(self):
        """The device convection was re-assembled (``relinearize``); the host
        copy is refreshed lazily, on the next host-side use."""
        self._host_stale = True

    def _sync_host(self):
        if getattr(self, "_host_stale", False):
            self.download_convection()

    def convection_matrices(self):
        """Eliminated per-stage vector Jacobians (reference ``self.convection``)."""
        if self.convection is None:
            return None
        self._sync_host()
        mats = []
        for v in self._conv_vals:
            J = ConvectionBlocks(self.n_nodes, self.blocks.rowptr, self.blocks.col, v)
            mats.append(J.matrix)
        return mats * self.r if len(mats) == 1 else mats

    def materialize(self, raw=False, limit=10_000):
        """Explicit sparse stage matrix (stages.py:139-167); small systems only."""
        if self.dim > limit:
            raise ValueError(f"refusing to materialize {self.dim} stage dofs")
        if raw:
            M, K, B = self.blocks.M, self.blocks.K, self.blocks.B
        else:
            M, K, B = self.M, self.K, self.B
        saddle = sp.bmat([[K, B], [B.T, None]], format="csr")
        massd = sp.block_diag([M, sp.csr_matrix((self.n_p, self.n_p))], format="csr")
        A = self.tableau.A
        out = (sp.kron(sp.identity(self.r), massd) + self.dt * sp.kron(A, saddle)).tolil()
        if self.convection is not None:
            if raw:
                raise ValueError("raw materialization is not defined with convection")
            conv = self.convection_matrices()
            sd = self.stage_dim
            for i in range(self.r):
                for j in range(self.r):
                    out[i * sd:i * sd + self.n_u, j * sd:j * sd + self.n_u] += \
                        self.dt * A[i, j] * conv[i]
        out = out.tocsr()
        if not raw and len(self.constrained):
            ones = np.zeros(self.dim)
            ones[self.constrained_stage_dofs()] = 1.0
            out = out + sp.diags(ones)
        return out.tocsr()

    # -- device data and the K1 apply ---------------------------------------

    def device_data(self):
        """Upload the eliminated operator once; returns the descriptor."""
        if self._dev is not None:
            return self._dev
        from ._device import upload
        import torch
        b = self.blocks
        t = {}
        t["p2_rowptr"] = upload(b.rowptr, np.int32)
        t["p2_col"] = upload(b.col, np.int32)
        t["p2_mk"] = upload(np.column_stack([self._m, self._k]), np.float64)
        t["b_rowptr"] = upload(b.b_rowptr, np.int32)
        t["b_col"] = upload(b.b_col, np.int32)
        t["b_val"] = upload(self._b, np.float64)
        # B^T rows per P1 node with (B_x, B_y) pairs -- the eliminated B (so
        # constrained velocities drop out, stages.py:81,125).
        order = np.lexsort((self._brows, b.b_col))
        bt_rowptr = np.concatenate([[0], np.cumsum(np.bincount(b.b_col, minlength=self.n_p))])
        t["bt_rowptr"] = upload(bt_rowptr, np.int32)
        t["bt_col"] = upload(self._brows[order], np.int32)
        t["bt_val"] = upload(self._b[order], np.float64)
        t["cmask"] = upload(self.node_constrained.astype(np.uint8), np.uint8)
        t["proj_scratch"] = torch.zeros(_lib.PROJECT_BLOCKS * self.r, dtype=torch.float64,
                                        device=t["cmask"].device)
        n_conv = 0
        if self._conv_vals is not None:
            t["conv"] = upload(np.stack(self._conv_vals).reshape(len(self._conv_vals), -1, 4),
                               np.float64)
            n_conv = len(self._conv_vals)
        # SELL copies for the K1 apply (coalesced entry loads): velocity rows
        # in slices of 16 nodes (2-D: lane pairs per node) or 32 (3-D: one
        # thread per node), pressure rows in slices of 32.
        cv = 16 if self.nc == 2 else 32
        sptr, scol, smk = to_sell(b.rowptr, b.col, np.column_stack([self._m, self._k]),
                                  self.n_nodes, C=cv)
        t["p2_sptr"], t["p2_scol"] = upload(sptr, np.int32), upload(scol, np.int32)
        t["p2_smk"] = upload(smk, np.float64)
        nnz_s = len(scol)
        if self._conv_vals is not None:
            cs = [to_sell(b.rowptr, b.col, v.reshape(-1, 4), self.n_nodes, C=16)[2]
                  for v in self._conv_vals]
            t["conv_s"] = upload(np.stack(cs), np.float64)
        sptr, scol, sval = to_sell(b.b_rowptr, b.b_col, self._b, self.n_nodes, pad_col=0, C=cv)
        t["b_sptr"], t["b_scol"], t["b_sval"] = (upload(sptr, np.int32), upload(scol, np.int32),
                                                 upload(sval, np.float64))
        sptr, scol, sval = to_sell(bt_rowptr, self._brows[order], self._b[order], self.n_p,
                                   pad_col=0)
        t["bt_sptr"], t["bt_scol"], t["bt_sval"] = (upload(sptr, np.int32), upload(scol, np.int32),
                                                    upload(sval, np.float64))
        desc = _lib.OperatorDesc()
        desc.stages = self.r
        desc.n_nodes = self.n_nodes
        desc.n_p = self.n_p
        desc.n_conv = n_conv
        desc.nnz = len(b.col)
        desc.dt = self.dt
        A = np.asarray(self.tableau.A, dtype=np.float64)
        for i in range(self.r):
            for j in range(self.r):
                desc.butcher_a[i * self.r + j] = A[i, j]
        desc.p2_rowptr = t["p2_rowptr"].data_ptr()
        desc.p2_col = t["p2_col"].data_ptr()
        desc.p2_mk = t["p2_mk"].data_ptr()
        desc.conv = t["conv"].data_ptr() if "conv" in t else None
        desc.b_rowptr = t["b_rowptr"].data_ptr()
        desc.b_col = t["b_col"].data_ptr()
        desc.b_val = t["b_val"].data_ptr()
        desc.bt_rowptr = t["bt_rowptr"].data_ptr()
        desc.bt_col = t["bt_col"].data_ptr()
        desc.bt_val = t["bt_val"].data_ptr()
        desc.node_constrained = t["cmask"].data_ptr()
        for k in ("p2_sptr", "p2_scol", "p2_smk", "b_sptr", "b_scol", "b_sval", "bt_sptr",
                  "bt_scol", "bt_sval"):
            setattr(desc, k, t[k].data_ptr())
        desc.conv_s = t["conv_s"].data_ptr() if "conv_s" in t else None
        desc.nnz_s = nnz_s
        desc.ncomp = self.nc
        # locality order of the SELL slices (2-D, coordinates known): pressure
        # slices first (long rows), both kinds along a Hilbert curve through
        # the slice centroids, so a CTA's eight slices gather overlapping x
        xy = getattr(b, "node_xy", None)
        if self.nc == 2 and xy is not None and os.environ.get("IVK_K1_ORDER", "0") != "0":
            from .k1tiles import hilbert_key

            def centroid_order(pts, width):
                n = len(pts)
                sl = np.arange(n) // width
                cnt = np.bincount(sl)
                c = np.column_stack([np.bincount(sl, weights=pts[:, d]) / cnt for d in range(2)])
                return np.argsort(hilbert_key(c), kind="stable")
            nsv = (self.n_nodes + 15) // 16
            ordv = centroid_order(xy[:self.n_nodes], 16)
            ordp = centroid_order(xy[:self.n_p], 32) + nsv
            t["k1_order"] = upload(np.concatenate([ordp, ordv]), np.int32)
            desc.k1_order = t["k1_order"].data_ptr()
            desc.k1_order_n = len(ordp) + len(ordv)
        tiles = None
        tile_rows = int(os.environ.get("IVK_K1_TILES", "0"))
        if tile_rows > 0 and self.nc == 2 and n_conv == 0:
            # K1 tile plan (k1tiles.py): rows in Hilbert-curve tiles, x staged
            # in shared memory; the SELL copies above stay for row-list applies
            # (shard.py) and as the A/B reference (IVK_K1_TILES=0).
            plan = build_k1_tiles(b.rowptr, b.col, np.column_stack([self._m, self._k]),
                                  b.b_rowptr, b.b_col, self._b, bt_rowptr, self._brows[order],
                                  self._b[order], self.node_constrained,
                                  xy=getattr(b, "node_xy", None), tile_rows=tile_rows)
            tiles = _lib.K1Tiles()
            for k in ("n_tiles", "max_u", "max_p", "max_ent", "max_slices", "max_blob"):
                setattr(tiles, k, int(plan[k]))
            for k, dt_ in (("tile_rec", np.int32), ("blob", np.int32), ("ecol", np.uint16),
                           ("eval", np.float64)):
                t["k1t_" + k] = upload(plan[k], dt_)
                setattr(tiles, k, t["k1t_" + k].data_ptr())
            desc.k1_tiles = C.pointer(tiles)
            self.k1_plan_stats = {k: int(plan[k]) for k in
                                  ("n_tiles", "n_slices", "max_u", "max_p", "max_ent", "max_slices",
                                   "n_entries", "tile_rows")}
        self._dev = {"tensors": t, "desc": desc, "k1_tiles": tiles,
                     "cmask_dofs": torch.from_numpy(self._cmask).to(t["cmask"].device)}
        return self._dev

    def sell_pos(self):
        """Position of every CSR pattern entry in the SELL-16 copy."""
        b = self.blocks
        lens = np.diff(b.rowptr)
        C_ = 16
        nsl = (self.n_nodes + C_ - 1) // C_
        padded = np.zeros(nsl * C_, dtype=np.int64)
        padded[:self.n_nodes] = lens
        width = padded.reshape(nsl, C_).max(axis=1)
        sptr = np.concatenate([[0], np.cumsum(width * C_)])
        rows = np.repeat(np.arange(self.n_nodes), lens)
        ent = np.arange(len(rows)) - b.rowptr[rows]
        return sptr[rows // C_] + ent * C_ + rows % C_

    def download_convection(self):
        """Refresh the host copy of the device convection (one shared Jacobian
        or one per stage)."""
        self._host_stale = False
        if self._dev is None or "conv" not in self._dev["tensors"]:
            return
        conv = self._dev["tensors"]["conv"]
        vals = [conv[i].reshape(-1, 2, 2).cpu().numpy() for i in range(conv.shape[0])]
        self._conv_vals = vals
        Js = [ConvectionBlocks(self.n_nodes, self.blocks.rowptr, self.blocks.col, v) for v in vals]
        self.convection = Js * self.r if len(Js) == 1 else Js

    @property
    def desc(self):
        return self.device_data()["desc"]

    def apply_into(self, x, b, out):
        """Device: out = b - A x (b is not None) or out = A x."""
        from ._device import ptr, stream
        _lib.check(_lib.lib().ivk_stage_apply(self.desc, ptr(x), ptr(b), ptr(out), stream()),
                   "stage_apply")
        return out

    def matvec(self, x):
        """Eliminated operator apply (stages.py:110-126) on the GPU.

        numpy in -> numpy out (host edge); a CUDA tensor stays on the device."""
        from ._device import as_device_vector, to_host
        import torch
        xd, host = as_device_vector(x, self.dim)
        y = torch.empty_like(xd)
        self.apply_into(xd, None, y)
        return to_host(y) if host else y

    def residual(self, x, b):
        """b - A x on the GPU (same host/device convention as ``matvec``)."""
        from ._device import as_device_vector, to_host
        import torch
        xd, host = as_device_vector(x, self.dim)
        bd, _ = as_device_vector(b, self.dim)
        r = torch.empty_like(xd)
        self.apply_into(xd, bd, r)
        return to_host(r) if host else r


def assemble_stage_operator(blocks, tableau, dt, constrained=None, convection=None):
    """Stage operator with Dirichlet stage constraints (stages.py:189-194)."""
    if blocks.b_rowptr[-1] == 0 and blocks.n_p:
        raise ValueError("inconsistent block dimensions")
    return StageSystem(blocks, tableau, dt, constrained=constrained, convection=convection)
