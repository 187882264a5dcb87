"""Device convection linearisation (kernel K10) for Newton-cadence updates.

The reference rebuilds every level's convection Jacobian and all Vanka
patch inverses on every Newton iteration (bench.py:403-417 via
``Discretization.build_mg``).  Here the Jacobian of a device velocity field
is assembled on the GPU straight into the operator's CSR/SELL buffers and the
patches are refactorised in place (K7), reusing every index table.
"""

import ctypes as C

import numpy as np

from . import _lib
from .fem import DEG_CONVECTION, _affine, p2_cell_nodes
from .quadrature import p2_basis, triangle_rule

__all__ = ["ConvectionAssembler"]


class ConvectionAssembler:
    """Convection Jacobian / residual of one level on the device.

    ``system`` must carry one shared convection Jacobian (n_conv = 1); its
    device buffers are overwritten by :meth:`assemble_into_system`."""

    def __init__(self, mesh, blocks, node_constrained):
        self.mesh = mesh
        self.blocks = blocks
        self.n_nodes = blocks.n_nodes
        nodes = p2_cell_nodes(mesh)
        _, jinv, det = _affine(mesh)
        self.cell_nodes = nodes
        self.cell_geo = np.column_stack([jinv.reshape(-1, 4), det])
        C_ = len(nodes)
        N = blocks.n_nodes
        # pattern entry of every (cell, a, b) contribution, cell-ascending
        key = (np.repeat(nodes[:, :, None], 6, axis=2).astype(np.int64) * N
               + np.repeat(nodes[:, None, :], 6, axis=1)).reshape(-1)
        order = np.argsort(key, kind="stable")
        rows = np.repeat(np.arange(N), np.diff(blocks.rowptr))
        pkey = rows.astype(np.int64) * N + blocks.col
        counts = np.bincount(np.searchsorted(pkey, key[order]), minlength=len(pkey))
        if not np.array_equal(np.unique(key), pkey):
            raise ValueError("cell connectivity does not match the scalar P2 pattern")
        self.entry_ptr = np.concatenate([[0], np.cumsum(counts)])
        self.entry_contrib = order  # cell*36 + a*6 + b
        self.row_of = rows
        self.col = blocks.col
        self.node_constrained = np.asarray(node_constrained, dtype=bool)
        norder = np.argsort(nodes.reshape(-1), kind="stable")
        self.node_ptr = np.concatenate([[0], np.cumsum(np.bincount(nodes.reshape(-1),
                                                                   minlength=N))])
        self.node_contrib = norder  # cell*6 + a
        pts, w = triangle_rule(DEG_CONVECTION)
        phi, dphi = p2_basis(pts)
        q = _lib.QuadTable()
        q.nq = len(w)
        if q.nq > _lib.IVK_MAX_QUAD:
            raise ValueError("quadrature rule too large")
        for i in range(q.nq):
            q.w[i] = w[i]
            for a in range(6):
                q.phi[i * 6 + a] = phi[a, i]
                q.dphi[(i * 6 + a) * 2] = dphi[a, i, 0]
                q.dphi[(i * 6 + a) * 2 + 1] = dphi[a, i, 1]
        self.quad = q
        self.n_cells = C_
        self._dev = None

    def device_data(self, sell_pos=None):
        """``sell_pos``: a callable returning the CSR -> SELL position map of
        the system being written (evaluated once: it is a host pass over every
        pattern entry, far dearer than the assembly kernel itself)."""
        if self._dev is not None:
            if sell_pos is not None and "sell_pos" not in self._dev["tensors"]:
                from ._device import upload
                self._dev["tensors"]["sell_pos"] = upload(sell_pos(), np.int32)
                self._dev["desc"].sell_pos = self._dev["tensors"]["sell_pos"].data_ptr()
            return self._dev
        import torch
        from ._device import upload
        t = {
            "cell_nodes": upload(self.cell_nodes, np.int32),
            "cell_geo": upload(self.cell_geo, np.float64),
            "entry_ptr": upload(self.entry_ptr, np.int32),
            "entry_contrib": upload(self.entry_contrib, np.int32),
            "row_of": upload(self.row_of, np.int32),
            "col": upload(self.col, np.int32),
            "cmask": upload(self.node_constrained.astype(np.uint8), np.uint8),
            "node_ptr": upload(self.node_ptr, np.int32),
            "node_contrib": upload(self.node_contrib, np.int32),
        }
        t["scratch"] = torch.empty(self.n_cells * 156, dtype=torch.float64,
                                   device=t["cell_geo"].device)
        if sell_pos is not None:
            t["sell_pos"] = upload(sell_pos(), np.int32)
        d = _lib.ConvectionDesc()
        d.n_cells, d.n_nodes, d.nnz = self.n_cells, self.n_nodes, len(self.col)
        d.quad = C.pointer(self.quad)
        d.cell_nodes = t["cell_nodes"].data_ptr()
        d.cell_geo = t["cell_geo"].data_ptr()
        d.entry_ptr = t["entry_ptr"].data_ptr()
        d.entry_contrib = t["entry_contrib"].data_ptr()
        d.row_of = t["row_of"].data_ptr()
        d.col = t["col"].data_ptr()
        d.node_constrained = t["cmask"].data_ptr()
        d.sell_pos = t["sell_pos"].data_ptr() if "sell_pos" in t else None
        d.node_ptr = t["node_ptr"].data_ptr()
        d.node_contrib = t["node_contrib"].data_ptr()
        self._dev = {"tensors": t, "desc": d}
        return self._dev

    def jacobian(self, u, residual=False):
        """Device (J values (nnz, 4) eliminated, N(u) or None) for a device
        velocity vector u (2 n_nodes, interleaved)."""
        import torch
        from ._device import ptr, stream
        dev = self.device_data()
        J = torch.empty(len(self.col), 4, dtype=torch.float64, device=u.device)
        N = torch.empty(2 * self.n_nodes, dtype=torch.float64, device=u.device) if residual \
            else None
        _lib.check(_lib.lib().ivk_convection_assemble(dev["desc"], ptr(u),
                                                      ptr(dev["tensors"]["scratch"]), ptr(J),
                                                      None, ptr(N), stream()),
                   "convection_assemble")
        return J, N

    def assemble_into_system(self, system, u):
        """Overwrite ``system``'s device convection (CSR and SELL copies)."""
        from ._device import ptr, stream
        sdev = system.device_data()
        if system._conv_vals is None or len(system._conv_vals) != 1:
            raise ValueError("system needs one shared convection Jacobian")
        dev = self.device_data(sell_pos=system.sell_pos)
        t = sdev["tensors"]
        _lib.check(_lib.lib().ivk_convection_assemble(dev["desc"], ptr(u),
                                                      ptr(dev["tensors"]["scratch"]),
                                                      ptr(t["conv"]), ptr(t["conv_s"]), None,
                                                      stream()), "convection_assemble")

    def assemble_stage(self, system, stage, u):
        """Overwrite stage ``stage``'s device Jacobian of a system carrying one
        convection Jacobian per stage (n_conv = s, stages.py:118-123)."""
        from ._device import ptr, stream
        sdev = system.device_data()
        if system._conv_vals is None or len(system._conv_vals) != system.r:
            raise ValueError("system needs one convection Jacobian per stage")
        if not 0 <= stage < system.r:
            raise ValueError("stage out of range")
        dev = self.device_data(sell_pos=system.sell_pos)
        t = sdev["tensors"]
        conv, conv_s = t["conv"], t["conv_s"]
        _lib.check(_lib.lib().ivk_convection_assemble(
            dev["desc"], ptr(u), ptr(dev["tensors"]["scratch"]),
            conv[stage].data_ptr(), conv_s[stage].data_ptr(), None, stream()),
            "convection_assemble")
