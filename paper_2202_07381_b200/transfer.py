"""Stage prolongation I_s (x) blockdiag(P_P2 (x) I_d, P_P1) on the device (d = 2, or 3 in 3-D).

Mirror of the reference ``Discretization.stage_prolong`` (bench.py:187-194)
with the restriction ``P^T r`` and the constrained-row zeroing of
``MGHierarchyOp.vcycle`` (solvers.py:341-346) fused into kernel K5.
The scalar P2 and P1 interpolation matrices are stored once (the vector
and stage Kronecker factors are implicit), with explicit transposes so both
directions are deterministic row gathers.
"""

import numpy as np
import scipy.sparse as sp

from . import _lib

__all__ = ["StageTransfer"]


class StageTransfer:
    def __init__(self, p2, p1, stages, fine_node_constrained, coarse_node_constrained, ncomp=2):
        self.p2 = sp.csr_matrix(p2)
        self.p1 = sp.csr_matrix(p1)
        self.p2.sort_indices()
        self.p1.sort_indices()
        self.stages = int(stages)
        self.ncomp = int(ncomp)
        self.nf_nodes, self.nc_nodes = self.p2.shape
        self.nf_p, self.nc_p = self.p1.shape
        self.fine_cm = np.asarray(fine_node_constrained, dtype=bool)
        self.coarse_cm = np.asarray(coarse_node_constrained, dtype=bool)
        self._dev = None

    @property
    def shape(self):
        sf = self.ncomp * self.nf_nodes + self.nf_p
        sc = self.ncomp * self.nc_nodes + self.nc_p
        return (self.stages * sf, self.stages * sc)

    @property
    def matrix(self):
        """Reference-layout CSR (bench.py:187-194), for the oracle / API."""
        P = sp.block_diag([sp.kron(self.p2, sp.identity(self.ncomp)), self.p1]).tocsr()
        return sp.kron(sp.identity(self.stages), P, format="csr")

    def device_data(self):
        if self._dev is not None:
            return self._dev
        from ._device import upload
        t = {}

        def put(name, m):
            m = sp.csr_matrix(m)
            m.sort_indices()
            t[name + "_rowptr"] = upload(m.indptr, np.int32)
            t[name + "_col"] = upload(m.indices, np.int32)
            t[name + "_val"] = upload(m.data, np.float64)

        put("p2", self.p2)
        put("p2t", self.p2.T.tocsr())
        put("p1", self.p1)
        put("p1t", self.p1.T.tocsr())
        t["fcm"] = upload(self.fine_cm.astype(np.uint8), np.uint8)
        t["ccm"] = upload(self.coarse_cm.astype(np.uint8), np.uint8)
        d = _lib.TransferDesc()
        d.stages = self.stages
        d.nf_nodes, d.nf_p, d.nc_nodes, d.nc_p = self.nf_nodes, self.nf_p, self.nc_nodes, self.nc_p
        for name in ("p2", "p2t", "p1", "p1t"):
            for f in ("rowptr", "col", "val"):
                setattr(d, f"{name}_{f}", t[f"{name}_{f}"].data_ptr())
        d.fine_constrained = t["fcm"].data_ptr()
        d.coarse_constrained = t["ccm"].data_ptr()
        d.ncomp = self.ncomp
        self._dev = {"tensors": t, "desc": d}
        return self._dev

    def restrict_into(self, rf, rc):
        """rc = P^T rf with constrained coarse rows zeroed (device)."""
        from ._device import ptr, stream
        _lib.check(_lib.lib().ivk_restrict(self.device_data()["desc"], ptr(rf), ptr(rc), stream()),
                   "restrict")
        return rc

    def prolong_add(self, ec, xf):
        """xf += P ec on unconstrained fine rows (device)."""
        from ._device import ptr, stream
        _lib.check(_lib.lib().ivk_prolong_add(self.device_data()["desc"], ptr(ec), ptr(xf),
                                              stream()), "prolong_add")
        return xf
