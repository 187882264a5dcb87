"""Monolithic multigrid with additive IRK-Vanka relaxation -- the hot path.

Host mirror of the reference ``irkmg.solvers`` API
(/root/reference/pkg/src/irkmg/solvers.py); every flop of the relaxation,
the transfers and the coarse solve runs in libivk (sm_100a):

    reference                         here                       kernel
    StageSystem.matvec / b - A x      StageSystem.apply_into     K1
    resid[idx] + einsum               VankaPatchSet._apply       K2+K3
    np.bincount + x + w z             VankaPatchSet._combine     K4
    np.linalg.inv (setup)             ivk_patch_factor           K7
    P.T @ r / P @ e                   StageTransfer              K5
    CoarseSolver.solve (splu)         CoarseSolver.solve         K6
    chebyshev recurrence, projections ivk_patch_combine/axpby    K8

Numpy inputs are accepted at the public edge (copied to and from the
device); CUDA tensors stay resident.  There is no CPU fallback.
"""

from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
import scipy.sparse.linalg as spla

import ctypes as C

from . import _lib
from .patches import build_patch_tables

__all__ = [
    "PatchSingularError",
    "SmootherSpec",
    "KrylovStats",
    "VankaPatchSet",
    "build_vanka_patches",
    "apply_vanka",
    "chebyshev_smooth",
    "CoarseSolver",
    "coarse_direct_solve",
    "MGLevel",
    "MGHierarchyOp",
    "vcycle",
    "fgmres",
]


class PatchSingularError(RuntimeError):
    """Singular Vanka patch matrix (solvers.py:81-84)."""

    def __init__(self, vertex):
        super().__init__(f"singular Vanka patch matrix at vertex {vertex}")
        self.vertex = vertex


@dataclass
class SmootherSpec:
    """Relaxation configuration (solvers.py:87-105), extended with the
    stationary ``"richardson"`` driver and partition-of-unity weighting used
    by the BASELINE "damping 0.5" smoother."""

    pre: int = 2
    post: int = 2
    accel: str = "chebyshev"  # "chebyshev" | "gmres" | "richardson"
    cheby_a: float = 2.0
    cheby_b: float = 8.0
    omega: float = 1.0
    weighting: str = "none"   # "none" (reference) | "pou" (1 / multiplicity)

    def __post_init__(self):
        if self.accel not in ("chebyshev", "gmres", "richardson"):
            raise ValueError(f"unknown smoother acceleration {self.accel!r}")
        if self.accel == "chebyshev" and not 0.0 < self.cheby_a < self.cheby_b:
            raise ValueError("Chebyshev interval must satisfy 0 < a < b")
        if min(self.pre, self.post) < 0:
            raise ValueError("sweep counts must be >= 0")
        if self.weighting not in ("none", "pou"):
            raise ValueError(f"unknown weighting {self.weighting!r}")


@dataclass
class KrylovStats:
    iterations: int = 0
    residual_norms: list = field(default_factory=list)
    final_residual: float = np.inf
    relative_residual: float = np.inf
    converged: bool = False


# ----------------------------------------------------------------- patches

class KronSplit:
    """Eigen-split A = V diag(lam) V^-1 of the Butcher matrix (include/ivk.h,
    ``ivk_kron_desc``): one stored block per real eigenvalue and per
    complex-conjugate pair."""

    def __init__(self, A, max_cond=1e6, symmetric=False):
        self.symmetric = bool(symmetric)
        A = np.asarray(A, dtype=np.float64)
        s = len(A)
        lam, V = np.linalg.eig(A)
        if not np.all(np.isfinite(V)) or np.linalg.cond(V) > max_cond:
            raise ValueError("Butcher matrix is not (well) diagonalisable")
        Vinv = np.linalg.inv(V)
        tol = 1e-12 * max(1.0, np.max(np.abs(lam)))
        real = [k for k in range(s) if abs(lam[k].imag) <= tol]
        pos = [k for k in range(s) if lam[k].imag > tol]
        if len(real) + 2 * len(pos) != s:
            raise ValueError("unpaired complex eigenvalues")
        keep = real + pos
        self.s = s
        self.lam = lam[keep]
        self.is_complex = np.array([0] * len(real) + [1] * len(pos), dtype=np.int32)
        self.V = V[:, keep]
        self.Vinv = Vinv[keep, :]
        for k in range(len(real)):
            self.lam[k] = self.lam[k].real
            self.V[:, k] = self.V[:, k].real
            self.Vinv[k, :] = self.Vinv[k, :].real
        self.scale = np.where(self.is_complex == 1, 2.0, 1.0)

    @property
    def nblk(self):
        return len(self.lam)

    def desc(self):
        d = _lib.KronDesc()
        d.nblk = self.nblk
        for k in range(self.nblk):
            d.is_complex[k] = int(self.is_complex[k])
            d.lam_re[k] = self.lam[k].real
            d.lam_im[k] = self.lam[k].imag
            d.scale[k] = self.scale[k]
            for i in range(self.s):
                d.v_re[i * self.s + k] = self.V[i, k].real
                d.v_im[i * self.s + k] = self.V[i, k].imag
                d.vinv_re[k * self.s + i] = self.Vinv[k, i].real
                d.vinv_im[k * self.s + i] = self.Vinv[k, i].imag
        d.symmetric = int(self.symmetric)
        return d

    def block_doubles(self, b):
        """Stored doubles per patch of block size b (matches the kernels)."""
        if self.symmetric:
            return sum(self._sym_block(c, b) for c in self.is_complex)
        ldr = (b + 3) & ~3
        ldc = (b + 1) & ~1 if b <= 64 else (b + 3) & ~3
        return sum(2 * b * ldc if c else b * ldr for c in self.is_complex)

    @staticmethod
    def _sym_block(cplx, b):
        nt = (b + 3) // 4
        return (32 if cplx else 16) * (nt * (nt + 1) // 2)

    def unpack(self, raw, b):
        """Stored blocks of one patch (raw doubles) -> list of b x b blocks."""
        G, pos = [], 0
        for cplx in self.is_complex:
            if self.symmetric:
                nt = (b + 3) // 4
                size = self._sym_block(cplx, b)
                vals = raw[pos:pos + size]
                qc = 8 if cplx else 4
                T = np.zeros((4 * nt, 4 * nt), dtype=complex if cplx else float)
                base = 0
                for d in range(nt):
                    ln = nt - d
                    blk = vals[base:base + 4 * qc * ln].reshape(qc, ln, 4)
                    for t in range(ln):
                        I, J = d + t, t
                        chunks = blk[:, t, :]            # (qc, 4)
                        if cplx:
                            tile = (chunks[:, 0::2] + 1j * chunks[:, 1::2]).reshape(4, 4)
                        else:
                            tile = chunks.reshape(4, 4)
                        T[4 * I:4 * I + 4, 4 * J:4 * J + 4] = tile
                        T[4 * J:4 * J + 4, 4 * I:4 * I + 4] = tile.T
                    base += 4 * qc * ln
                G.append(T[:b, :b])
                pos += size
            elif cplx:
                ldc = (b + 1) & ~1 if b <= 64 else (b + 3) & ~3
                a = raw[pos:pos + 2 * b * ldc].reshape(b, ldc, 2)[:, :b]
                G.append((a[..., 0] + 1j * a[..., 1]).T)
                pos += 2 * b * ldc
            else:
                ldr = (b + 3) & ~3
                G.append(raw[pos:pos + b * ldr].reshape(b, ldr)[:, :b].T)
                pos += b * ldr
        return G

    def full_inverse(self, G, b):
        """Reassemble the (s b) x (s b) inverse from stored blocks G[k] (b x b)."""
        s = self.s
        out = np.zeros((s * b, s * b))
        for k in range(self.nblk):
            T = self.scale[k] * np.real(np.einsum("i,ac,j->iajc", self.V[:, k], G[k],
                                                  self.Vinv[k, :]))
            out += T.reshape(s * b, s * b)
        return out


class VankaPatchSet:
    """Vertex-star patches with device-resident dense inverses (solvers.py:116-222).

    One patch per mesh vertex: every unconstrained velocity DoF (both
    components, all stages) on the closure of the vertex star plus the r
    centre pressures.  Inverses are assembled and factorised on the GPU
    (K7) unless ``factor=False`` (then ``set_inverses`` must be called).

    ``mode``: "full" stores each patch's (s b)^2 inverse (the reference's
    formulation); "kron" the Butcher eigen-split (s b^2 doubles per patch,
    3x fewer bytes at s = 3); "kron-sym" additionally stores each block as a
    symmetric tile-triangle (Stokes: no convection; 44% fewer bytes than
    kron at cfg2); "dedup" shares the kron blocks of patches whose
    canonical matrices are bitwise identical (translation-invariant
    operators: dedup.py); "modal" the per-patch generalised eigenbasis of
    the Stokes velocity blocks (modal.py: ~10x fewer bytes than kron, any
    tableau); "auto" picks dedup when it collapses the patch set at least 8x
    (2-D, convection-free), else modal (convection-free), else kron (all
    stages share the convection Jacobian, A well diagonalisable), else full.
    """

    _ivk_device_native = True   # takes / returns device tensors as well as numpy

    def __init__(self, system, mesh, omega=1.0, factor=True, mode="auto", scatter="patch",
                 vertices=None):
        if scatter not in ("patch", "owner"):
            raise ValueError(f"unknown scatter layout {scatter!r}")
        self.scatter = scatter
        self.omega = float(omega)
        self.system = system
        # vertices: only the patches of these centre vertices (one shard of a
        # partitioned level, shard.py); None = every vertex
        # general multi-field systems (general.py, e.g. MHD) build their own
        # vertex-star tables; Taylor-Hood systems use the reference layout
        self.general = getattr(system, "general", False)
        if self.general:
            self.tables = system.patch_tables(mesh, vertices=vertices)
        else:
            self.tables = build_patch_tables(mesh, system.n_nodes, system.n_p, system.r,
                                             system.node_constrained, vertices=vertices,
                                             ncomp=system.nc)
        self.num_patches = self.tables.num_patches
        if mode not in ("auto", "full", "kron", "kron-sym", "dedup", "modal"):
            raise ValueError(f"unknown patch mode {mode!r}")
        self.modal = None
        if mode == "modal":
            # Stokes only: velocity blocks M_s (x) I and K_s (x) I, K_s symmetric
            if self.general or system.convection is not None:
                raise ValueError("modal split needs a convection-free Taylor-Hood operator")
            if int(np.diff(self.tables.node_off).max()) > 72:
                raise ValueError("modal split supports patches of at most 72 free nodes")
            from .modal import ModalSplit
            self.modal = ModalSplit(system.tableau, system.dt, system.nc)
        # kron-sym halves the inverse bytes but measures no faster than kron on
        # B200 (latency-bound, profiles/r01): "auto" keeps the plain kron layout.
        symmetric = mode == "kron-sym"
        if mode == "kron-sym" and system.convection is not None:
            raise ValueError("kron-sym needs a symmetric (convection-free) operator")
        self.kron = None
        self.dedup = None
        if mode == "dedup" and system.convection is not None:
            raise ValueError("dedup needs a translation-invariant (convection-free) operator")
        if self.general and mode in ("kron-sym", "dedup"):
            raise ValueError(f"mode {mode!r} is not available for general operators")
        if mode in ("auto", "kron", "kron-sym", "dedup"):
            try:
                shared = system.convection is None or len(system._conv_vals) == 1
                if not shared:
                    raise ValueError("per-stage convection Jacobians differ")
                # K7e (Stokes) factors b <= 64 in shared memory and larger
                # blocks (3-D) in place in global memory up to b = 256; K7g
                # (general) holds 2 b^2 doubles in shared memory (b <= 112);
                # K3e streams blocks up to b = 256.  kron-sym / dedup: b <= 64
                bmax = self.tables.max_m // system.r
                if bmax > (112 if self.general else 256) or \
                        (mode in ("kron-sym", "dedup") and bmax > 64):
                    raise ValueError("patch block too large for the kron kernels")
                # Stokes (no convection): S^ symmetric -> packed symmetric blocks
                self.kron = KronSplit(system.tableau.A,
                                      symmetric=(system.convection is None and symmetric))
            except ValueError:
                if mode in ("kron", "kron-sym", "dedup"):
                    raise
                self.kron = None
        if self.kron is not None and not self.general and (
                mode == "dedup" or (mode == "auto" and system.nc == 2 and
                                    system.convection is None)):
            # translation-invariant operator: share inverses between patches
            # whose canonical matrices are bitwise identical (dedup.py); "auto"
            # keeps it only when it actually collapses the patch set
            from .dedup import build_dedup_tables
            dd = build_dedup_tables(mesh, system, self.tables)
            if mode == "dedup" or dd.n_classes * 8 <= self.tables.num_patches:
                self.dedup = dd
        if (mode == "auto" and self.dedup is None and not self.general and
                system.convection is None and int(np.diff(self.tables.node_off).max()) <= 72):
            # convection-free Taylor-Hood operator on a mesh without enough
            # repeated patches: the modal split (any tableau, fewest bytes)
            from .modal import ModalSplit
            self.kron = None
            self.modal = ModalSplit(system.tableau, system.dt, system.nc)
        self.mode = "modal" if self.modal is not None else "full" if self.kron is None else \
            ("dedup" if self.dedup is not None else
             ("kron-sym" if self.kron.symmetric else "kron"))
        self._layout()
        self._dev = None
        self._factored = False
        if factor:
            self.factor()

    def _layout(self):
        t = self.tables
        if self.modal is not None:
            ks = np.diff(t.node_off).astype(np.int64)
            sizes = np.array([self.modal.record_doubles(int(k)) for k in ks], dtype=np.int64)
            off = np.concatenate([[0], np.cumsum(sizes)])
            self.inv_off, self.inv_size = off[:-1], int(off[-1])
            return
        if self.dedup is not None:
            # per-class (representative) inverse blocks only
            sizes = np.array([self.kron.block_doubles(int(t.sizes[q]) // t.stages)
                              for q in self.dedup.rep], dtype=np.int64)
            off = np.concatenate([[0], np.cumsum(sizes)])
            self.inv_off, self.inv_size = off[:-1], int(off[-1])
            return
        if self.kron is None:
            self.inv_off, self.inv_size = t.inv_off, t.inv_size
        else:
            sizes = np.array([self.kron.block_doubles(int(m) // t.stages) for m in t.sizes],
                             dtype=np.int64)
            off = np.concatenate([[0], np.cumsum(sizes)])
            self.inv_off, self.inv_size = off[:-1], int(off[-1])

    # -- reference attributes ------------------------------------------------

    @property
    def patch_indices(self):
        """Per-vertex stage-major index arrays (solvers.py:160-166)."""
        t = self.tables
        out = [None] * t.num_patches
        for k, v in enumerate(t.order):
            out[v] = t.idx[t.idx_off[k]:t.idx_off[k + 1]].copy()
        return out

    @property
    def patch_vel(self):
        """Per-vertex P2 (velocity; for general operators every P2 field)
        single-stage DoFs of each patch (solvers.py:160)."""
        t = self.tables
        out = [None] * t.num_patches
        if self.general:
            nw = self.system.nc * self.system.n_nodes
            for k, v in enumerate(t.order):
                d = t.node[t.node_off[k]:t.node_off[k + 1]]
                out[v] = d[d < nw].astype(np.int64)
            return out
        for k, v in enumerate(t.order):
            n = t.node[t.node_off[k]:t.node_off[k + 1]]
            vel = np.empty(2 * len(n), dtype=np.int64)
            vel[0::2] = 2 * n
            vel[1::2] = 2 * n + 1
            out[v] = vel
        return out

    @property
    def groups(self):
        """[(idx (P, m), inv (P, m, m))] in the reference group order,
        downloaded from the device (solvers.py:169-184)."""
        t = self.tables
        dev = self.device_data()
        inv_all = dev["inv"]
        out = []
        if self.modal is not None:
            raw = inv_all.cpu().numpy()
            ks = np.diff(t.node_off)
            for m, first, count in t.groups():
                idx = t.idx[t.idx_off[first]:t.idx_off[first + count]].reshape(count, m)
                inv = np.empty((count, m, m))
                for qq in range(count):
                    q = first + qq
                    o = int(self.inv_off[q])
                    inv[qq] = self.modal.full_inverse(raw[o:o + self.modal.record_doubles(int(ks[q]))],
                                                      int(ks[q]))
                out.append((idx.copy(), inv))
            return out
        if self.dedup is not None:
            dd = self.dedup
            raw = inv_all.cpu().numpy()
            cls_inv = []
            for c_, q in enumerate(dd.rep):
                b = int(t.sizes[q]) // t.stages
                o = int(self.inv_off[c_])
                cls_inv.append(self.kron.full_inverse(
                    self.kron.unpack(raw[o:o + self.kron.block_doubles(b)], b), b))
            for m, first, count in t.groups():
                idx = t.idx[t.idx_off[first]:t.idx_off[first + count]].reshape(count, m)
                inv = np.empty((count, m, m))
                for qq in range(count):
                    q = first + qq
                    pm = dd.perm[t.idx_off[q]:t.idx_off[q + 1]].astype(np.int64)
                    G = cls_inv[dd.class_of[q]]
                    inv[qq][np.ix_(pm, pm)] = G
                out.append((idx.copy(), inv))
            return out
        for m, first, count in t.groups():
            idx = t.idx[t.idx_off[first]:t.idx_off[first + count]].reshape(count, m)
            off = int(self.inv_off[first])
            if self.kron is None:
                ld = (m + 3) & ~3
                blk = inv_all[off:off + count * m * ld].view(count, m, ld)[:, :, :m]
                inv = blk.transpose(1, 2).contiguous().cpu().numpy()
            else:
                b = m // t.stages
                per = self.kron.block_doubles(b)
                raw = inv_all[off:off + count * per].view(count, per).cpu().numpy()
                inv = np.empty((count, m, m))
                for q in range(count):
                    inv[q] = self.kron.full_inverse(self.kron.unpack(raw[q], b), b)
            out.append((idx.copy(), inv))
        return out

    @property
    def multiplicity(self):
        return self.tables.multiplicity

    def pou_weights(self):
        """W = 1 / multiplicity (0 where no patch covers the DoF)."""
        mult = self.tables.multiplicity
        w = np.zeros(len(mult))
        nz = mult > 0
        w[nz] = 1.0 / mult[nz]
        return w

    # -- device data ---------------------------------------------------------

    def device_data(self):
        if self._dev is not None:
            return self._dev
        from ._device import upload
        import torch
        t = self.tables
        if t.total_m >= 2 ** 31:
            raise ValueError("patch index total exceeds int32")
        d = {}
        d["idx_off"] = upload(t.idx_off, np.int32)
        d["idx"] = upload(t.idx, np.int32)
        d["inv_off"] = upload(self.inv_off, np.int64)
        d["inv"] = torch.zeros(self.inv_size, dtype=torch.float64, device=d["idx"].device)
        d["dof_ptr"] = upload(t.dof_ptr, np.int32)
        d["dof_pos"] = upload(t.dof_pos, np.int32)
        slot_pos = np.empty(t.total_m, dtype=np.int64)
        slot_pos[t.dof_pos] = np.arange(t.total_m)       # owner-sorted write position
        d["slot_pos"] = upload(slot_pos, np.int32)
        d["vertex"] = upload(t.order, np.int32)
        d["node_off"] = upload(t.node_off, np.int32)
        d["node"] = upload(t.node, np.int32)
        d["local"] = torch.empty(t.total_m, dtype=torch.float64, device=d["idx"].device)
        d["pou"] = upload(self.pou_weights(), np.float64)
        desc = _lib.PatchDesc()
        desc.num_patches = t.num_patches
        desc.dim = t.dim
        desc.max_m = t.max_m
        desc.total_m = t.total_m
        for name in ("idx_off", "idx", "inv_off", "inv", "dof_ptr", "dof_pos", "vertex",
                     "node_off", "node"):
            setattr(desc, name, d[name].data_ptr())
        desc.slot_pos = d["slot_pos"].data_ptr() if self.scatter == "owner" else None
        if self.kron is not None:
            d["kron"] = self.kron.desc()          # keep the host struct alive
            desc.kron = C.pointer(d["kron"])
        if self.modal is not None:
            # warp-per-patch tensor-core K3m (k <= 32 free nodes): fragment
            # layout of the gather list / local[] (include/ivk.h layout = 1)
            kmax = int(np.diff(t.node_off).max())
            frag = kmax <= 32
            if frag:
                from .modal import fragment_layout
                offp, idx_f, dpos_f = fragment_layout(t, self.system.nc)
                if offp[-1] >= 2 ** 31:
                    raise ValueError("patch index total exceeds int32")
                d["idx_off"] = upload(offp, np.int32)
                d["idx"] = upload(idx_f, np.int32)
                d["dof_pos"] = upload(dpos_f, np.int32)
                d["local"] = torch.empty(int(offp[-1]), dtype=torch.float64,
                                         device=d["idx"].device)
                desc.total_m = int(offp[-1])
                for name in ("idx_off", "idx", "dof_pos"):
                    setattr(desc, name, d[name].data_ptr())
                desc.slot_pos = None
            d["modal"] = self.modal.desc(layout=1 if frag else 0)
            desc.modal = C.pointer(d["modal"])
        if self.dedup is not None:
            dd = self.dedup
            # canonical gather list and write positions, in tile (class) order
            lens = t.sizes[dd.order].astype(np.int64)
            starts = t.idx_off[dd.order].astype(np.int64)
            cum = np.concatenate([[0], np.cumsum(lens)])
            flat = np.repeat(starts - cum[:-1], lens) + np.arange(t.total_m)
            le = np.repeat(starts, lens) + dd.perm[flat].astype(np.int64)
            d["cidx"] = upload(t.idx[le], np.int32)
            d["cdst"] = upload(slot_pos[le] if self.scatter == "owner" else le, np.int32)
            d["class_off"] = upload(np.append(self.inv_off, self.inv_size), np.int64)
            d["tile_start"] = upload(dd.tile_start, np.int32)
            d["tile_class"] = upload(dd.tile_class, np.int32)
            d["tile_off"] = upload(cum[dd.tile_start], np.int32)
            desc.n_classes = dd.n_classes
            desc.class_inv_off = d["class_off"].data_ptr()
            desc.class_inv = d["inv"].data_ptr()
            desc.n_tiles = len(dd.tile_class)
            for name in ("tile_start", "tile_class", "tile_off", "cidx", "cdst"):
                setattr(desc, name, d[name].data_ptr())
            # the class representatives as a patch set of their own (K7 input)
            sizes = t.sizes[dd.rep]
            rep_idx_off = np.concatenate([[0], np.cumsum(sizes)])
            rep_node_off = np.concatenate([[0], np.cumsum([len(n) for n in dd.rep_nodes])])
            d["rep_idx_off"] = upload(rep_idx_off, np.int32)
            d["rep_node_off"] = upload(rep_node_off, np.int32)
            d["rep_node"] = upload(np.concatenate(dd.rep_nodes), np.int32)
            d["rep_vertex"] = upload(dd.rep_vertex, np.int32)
            rd = _lib.PatchDesc()
            rd.num_patches = dd.n_classes
            rd.dim = t.dim
            rd.max_m = int(sizes.max())
            rd.total_m = int(rep_idx_off[-1])
            rd.idx_off = d["rep_idx_off"].data_ptr()
            rd.idx = d["idx"].data_ptr()            # unused by K7
            rd.inv_off = d["inv_off"].data_ptr()
            rd.inv = d["inv"].data_ptr()
            rd.dof_ptr = d["dof_ptr"].data_ptr()    # unused by K7
            rd.dof_pos = d["dof_pos"].data_ptr()
            rd.vertex = d["rep_vertex"].data_ptr()
            rd.node_off = d["rep_node_off"].data_ptr()
            rd.node = d["rep_node"].data_ptr()
            rd.kron = C.pointer(d["kron"])
            d["rep_desc"] = rd
        d["desc"] = desc
        self._dev = d
        return d

    @property
    def desc(self):
        return self.device_data()["desc"]

    def factor(self):
        """K7: assemble + invert every patch matrix on the GPU."""
        import torch
        from ._device import ptr, stream
        dev = self.device_data()
        flag = torch.full((1,), 2 ** 31 - 1, dtype=torch.int32, device=dev["idx"].device)
        target = dev["rep_desc"] if self.dedup is not None else dev["desc"]
        if self.modal is not None:
            bad = self.modal.factor(self)
            if bad:
                raise PatchSingularError(int(min(self.tables.order[b] for b in bad)))
            self._factored = True
            return
        if self.general:
            self.system.factor_patches(target, flag)
        else:
            _lib.check(_lib.lib().ivk_patch_factor(self.system.desc, target, ptr(flag), stream()),
                       "patch_factor")
        bad = int(flag.item())
        if bad != 2 ** 31 - 1:
            raise PatchSingularError(bad)
        self._factored = True

    def set_inverses(self, groups):
        """Parity mode: install host inverses given in the reference ``groups``
        format [(idx (P,m), inv (P,m,m))] instead of factorising on the GPU."""
        import torch
        t = self.tables
        if self.kron is not None or self.modal is not None:   # reference inverses are full
            self.kron = None
            self.modal = None
            self.dedup = None
            self.mode = "full"
            self._layout()
            self._dev = None
        dev = self.device_data()
        mine = t.groups()
        if len(groups) != len(mine):
            raise ValueError("group structure differs from this patch set")
        for (m, first, count), (idx, inv) in zip(mine, groups):
            idx = np.asarray(idx)
            if idx.shape != (count, m) or not np.array_equal(
                    idx.ravel(), t.idx[t.idx_off[first]:t.idx_off[first + count]]):
                raise ValueError(f"patch indices of size group {m} differ")
            ld = (m + 3) & ~3
            blk = np.zeros((count, m, ld))
            blk[:, :, :m] = np.transpose(np.asarray(inv, dtype=np.float64), (0, 2, 1))
            off = int(t.inv_off[first])
            dev["inv"][off:off + blk.size] = torch.from_numpy(blk.ravel()).to(dev["inv"].device)
        self._factored = True

    def _require(self):
        if not self._factored:
            raise RuntimeError("patch inverses are not available (call factor() or set_inverses())")

    def apply_local(self, r, local=None):
        """K2+K3 on device: local = blockdiag(Inv_p) gathered r."""
        from ._device import ptr, stream
        self._require()
        dev = self.device_data()
        local = dev["local"] if local is None else local
        _lib.check(_lib.lib().ivk_patch_apply(dev["desc"], ptr(r), ptr(local), stream()),
                   "patch_apply")
        return local

    def combine(self, local, x, alpha, beta, w, out, accum=None):
        """K4 on device: out = alpha x + beta W sum_i R_i^T local_i (+ accum)."""
        from ._device import ptr, stream
        _lib.check(_lib.lib().ivk_patch_combine(self.desc, ptr(local), ptr(x), float(alpha),
                                                float(beta), ptr(w), ptr(out), ptr(accum),
                                                stream()), "patch_combine")
        return out

    def weights(self, weighting):
        return None if weighting == "none" else self.device_data()["pou"]

    def workspace(self):
        """Fresh per-stream sweep scratch (see ``apply_vanka``)."""
        import torch
        dev = self.device_data()
        return {"r": torch.empty(self.tables.dim, dtype=torch.float64, device=dev["idx"].device),
                "local": torch.empty_like(dev["local"])}

    def solve_additive(self, resid):
        """z = sum_i R_i^T (R_i A R_i^T)^{-1} R_i resid (solvers.py:214-222)."""
        from ._device import as_device_vector, to_host
        import torch
        rd, host = as_device_vector(resid, self.tables.dim)
        z = torch.empty_like(rd)
        loc = self.apply_local(rd)
        self.combine(loc, None, 0.0, 1.0, None, z)
        return to_host(z) if host else z


def build_vanka_patches(system, mesh, omega=1.0):
    """Vanka patch set for a stage system on ``mesh`` (solvers.py:225-229)."""
    if system.n_p != mesh.num_vertices:
        raise ValueError("mesh does not match the pressure space of the system")
    return VankaPatchSet(system, mesh, omega=omega)


def apply_vanka(patches, system, x, b, omega=None, weights=None, workspace=None, out=None):
    """One additive Schwarz sweep x + omega W sum R_i^T A_i^-1 R_i (b - A x)
    (solvers.py:232-239) as one fused K1 -> K3 -> K4 pass.

    ``weights``: None (reference, unweighted), "pou", or a DoF vector.
    ``workspace``: optional dict with device scratch "r" (dim) and "local"
    (total_m) -- one per stream when sweeps run concurrently on several
    streams (the patch set's own scratch is shared).  ``out``: optional
    device output buffer."""
    from ._device import as_device_vector, ptr, stream, to_host, upload
    import torch
    w = patches.omega if omega is None else omega
    xd, host = as_device_vector(x, system.dim)
    bd, _ = as_device_vector(b, system.dim)
    if isinstance(weights, str):
        wd = patches.weights(weights)
    elif weights is None:
        wd = None
    else:
        wd, _ = as_device_vector(weights, system.dim)
    patches._require()
    dev = patches.device_data()
    if workspace is not None:
        r, local = workspace["r"], workspace["local"]
    else:
        r, local = torch.empty_like(xd), dev["local"]
    if out is None:
        out = torch.empty_like(xd)
    if getattr(system, "general", False):
        system.vanka_sweep(dev["desc"], xd, bd, w, wd, r, local, out)
        return to_host(out) if host else out
    _lib.check(_lib.lib().ivk_vanka_sweep(system.desc, dev["desc"], ptr(xd), ptr(bd), float(w),
                                          ptr(wd), ptr(r), ptr(local), ptr(out), stream()),
               "vanka_sweep")
    return to_host(out) if host else out


def chebyshev_smooth(op_apply, precond, a, b, steps, x, rhs):
    """Chebyshev-accelerated preconditioned Richardson (solvers.py:242-268),
    run on the device: every vector update is a libivk axpby; numpy ``x`` /
    ``rhs`` are copied up and the result copied back (numpy callables are
    wrapped at the edge, this package's own operators run natively).  The
    multigrid cycle uses the fused K1/K3/K4 form in ``MGHierarchyOp._smooth``."""
    from ._device import as_device_vector, to_host
    if not 0.0 < a < b:
        raise ValueError("Chebyshev interval must satisfy 0 < a < b")
    if steps <= 0:
        return x
    n = int(np.asarray(rhs).shape[0]) if not _is_torch(rhs) else rhs.numel()
    xd, host = as_device_vector(x, n)
    bd, _ = as_device_vector(rhs, n)
    apply_op = _device_callable(op_apply, host)
    apply_pc = _device_callable(precond, host)
    ax = _axpby
    theta, delta = 0.5 * (b + a), 0.5 * (b - a)
    sigma1 = theta / delta
    rho = 1.0 / sigma1
    xk = xd.clone()
    r = ax(1.0, bd, -1.0, apply_op(xk))              # r = rhs - A x
    d = ax(1.0 / theta, apply_pc(r), 0.0, None)      # d = z / theta
    for _ in range(1, steps):
        ax(1.0, xk, 1.0, d, out=xk)                  # x += d
        r = ax(1.0, r, -1.0, apply_op(d))            # r -= A d
        rho_new = 1.0 / (2.0 * sigma1 - rho)
        d = ax(rho_new * rho, d, 2.0 * rho_new / delta, apply_pc(r))
        rho = rho_new
    out = ax(1.0, xk, 1.0, d)
    return to_host(out) if host else out


def _axpby(alpha, x, beta, y, out=None):
    """out = alpha x + beta y on the device (libivk K9 vector op)."""
    import torch
    from ._device import ptr, stream
    ref = x if x is not None else y
    if out is None:
        out = torch.empty_like(ref)
    _lib.check(_lib.lib().ivk_axpby(ref.numel(), float(alpha), ptr(x), float(beta), ptr(y),
                                    ptr(out), stream()), "axpby")
    return out


def _device_callable(f, host_semantics):
    """Adapt an operator / preconditioner callable to device vectors.

    This package's own objects (flagged ``_ivk_device_native``) take device
    tensors directly.  With host (numpy) semantics any other callable is a
    reference-style numpy function: it gets a numpy copy and its result is
    copied back up."""
    import torch
    from ._device import as_device_vector, to_host
    if f is None:
        return lambda v: v
    owner = getattr(f, "__self__", None)
    if not host_semantics or getattr(owner, "_ivk_device_native", False):
        return lambda v: torch.as_tensor(f(v), dtype=torch.float64, device=v.device)

    def wrapped(v):
        res = f(to_host(v))
        return as_device_vector(res, v.numel())[0] if not _is_torch(res) else res
    return wrapped


# ------------------------------------------------------------ coarse solve

class CoarseSolver:
    """Fixed SuperLU factorisation of A + Z Z^T (solvers.py:271-287).

    The factorisation is the reference's own host setup (scipy ``splu`` with
    its defaults).  The per-cycle solve x = P LU^-1 P b (P = I - Z Z^T) is
    kernel K6 on the device, in one of two forms:

    * ``method="dense"`` (default): P (A + Z Z^T)^-1 P is formed once at setup
      from the same LU factors (one LU solve per unit vector) and applied as
      one GEMV spread over every SM -- the coarse solve stops being a serial
      single-CTA chain.  Its result differs from the triangular solves by
      rounding only (measured 2e-15 .. 6e-14 relative where cond(A) <= 1e6,
      ~cond * eps at the cond 6e7 RadauIIA(3) coarse level, the same order as
      SuperLU's own forward error), and its backward error matches SuperLU's.
    * ``method="lu"``: the permuted triangular solves on tile-sparse copies
      of the factors (one CTA, TMA-staged diagonal tiles)."""

    def __init__(self, system, method="dense"):
        if method not in ("dense", "lu"):
            raise ValueError(f"unknown coarse method {method!r}")
        A = system.materialize()
        Z = system.pressure_nullspace()
        reg = sp.csr_matrix(Z @ Z.T)
        self.lu = spla.splu((A + reg).tocsc())
        self.Z = Z
        self.system = system
        self.method = method
        self._dev = None

    def dense_operator(self):
        """P (A + Z Z^T)^-1 P from the LU factors (n x n, fp64)."""
        n = self.system.dim
        inv = self.lu.solve(np.eye(n))
        Z = np.asarray(self.Z)
        izt = inv @ Z
        out = inv - izt @ Z.T
        out -= Z @ (Z.T @ out)
        return out

    @classmethod
    def from_device_operator(cls, system):
        """Dense coarse operator P (A + Z Z^T)^-1 P formed on the device from
        the system's CURRENT device operator (the Newton-cadence rebuild: the
        convection was just re-assembled there): A by applying K1 to the unit
        vectors (n tiny launches), the inverse by a dense LU with partial
        pivoting (torch.linalg.inv -> cuSOLVER getrf / getri, setup only), the
        projections as small GEMMs.  Same operator as the SuperLU route up to
        rounding (both LUs are backward stable); no host factorisation, no
        download of the convection.  ``method`` is "dense"."""
        import torch
        self = cls.__new__(cls)
        self.system, self.method, self.lu = system, "dense", None
        self.Z = system.pressure_nullspace()
        n = system.dim
        dev = system.device_data()["tensors"]["cmask"].device
        eye = torch.eye(n, dtype=torch.float64, device=dev)
        At = torch.empty((n, n), dtype=torch.float64, device=dev)
        for j in range(n):
            system.apply_into(eye[j], None, At[j])           # row j of A^T = A e_j
        Z = torch.from_numpy(np.ascontiguousarray(self.Z)).to(dev)
        inv = torch.linalg.inv(At.T + Z @ Z.T)
        out = inv - (inv @ Z) @ Z.T
        out -= Z @ (Z.T @ out)
        ld = (n + 3) & ~3
        D = torch.zeros((n, ld), dtype=torch.float64, device=dev)
        D[:, :n] = out
        d = _lib.CoarseDesc()
        d.n = n
        d.stages, d.n_u, d.n_p = system.r, system.n_u, system.n_p
        t = {"dense": D.reshape(-1)}
        d.dense = t["dense"].data_ptr()
        d.dense_ld = ld
        d.nb = (n + 31) // 32
        self._dev = {"tensors": t, "desc": d}
        return self

    def tiles(self):
        """Tile-sparse (32 x 32, column-major tiles) copies of the factors."""
        return (tile_factor(self.lu.L, lower=True, invert_lower_diag=True),
                tile_factor(self.lu.U, lower=False))

    def device_data(self):
        if self._dev is not None:
            return self._dev
        from ._device import upload
        s = self.system
        d = _lib.CoarseDesc()
        d.n = s.dim
        d.stages, d.n_u, d.n_p = s.r, s.n_u, s.n_p
        if self.method == "dense":
            ld = (s.dim + 3) & ~3
            D = np.zeros((s.dim, ld))
            D[:, :s.dim] = self.dense_operator()
            t = {"dense": upload(D.reshape(-1), np.float64)}
            d.dense = t["dense"].data_ptr()
            d.dense_ld = ld
            d.nb = (s.dim + 31) // 32
            self._dev = {"tensors": t, "desc": d}
            return self._dev
        (lc, lr, lt, ld, nb), (uc, ur, ut, ud, _) = self.tiles()
        t = {
            "l_colptr": upload(lc, np.int32), "l_row": upload(lr, np.int32),
            "l_tiles": upload(lt, np.float64), "l_diag": upload(ld, np.float64),
            "u_colptr": upload(uc, np.int32), "u_row": upload(ur, np.int32),
            "u_tiles": upload(ut, np.float64), "u_diag": upload(ud, np.float64),
            "perm_r": upload(self.lu.perm_r, np.int32),
            "perm_c": upload(self.lu.perm_c, np.int32),
        }
        d.nb = nb
        d.l_ntiles, d.u_ntiles = int(lc[-1]), int(uc[-1])
        for k in t:
            setattr(d, k, t[k].data_ptr())
        self._dev = {"tensors": t, "desc": d}
        return self._dev

    def solve_into(self, b, x):
        from ._device import ptr, stream
        _lib.check(_lib.lib().ivk_coarse_solve(self.device_data()["desc"], ptr(b), ptr(x),
                                               stream()), "coarse_solve")
        return x

    def solve(self, b):
        from ._device import as_device_vector, to_host
        import torch
        bd, host = as_device_vector(b, self.system.dim)
        x = torch.empty_like(bd)
        self.solve_into(bd, x)
        return to_host(x) if host else x


def tile_factor(F, lower, tile=32, invert_lower_diag=False):
    """Split a triangular factor into dense tile x tile blocks (column-major
    inside a tile), keeping only nonzero off-diagonal tiles, grouped by
    block column.  Padding rows/columns get a unit diagonal."""
    F = sp.csc_matrix(F)
    n = F.shape[0]
    nb = (n + tile - 1) // tile
    npad = nb * tile
    coo = F.tocoo()
    keep = (coo.row >= coo.col) if lower else (coo.row <= coo.col)
    r, c, v = coo.row[keep], coo.col[keep], coo.data[keep]
    diag = np.zeros((nb, tile, tile))
    bi, bj = r // tile, c // tile
    on = bi == bj
    diag[bi[on], r[on] % tile, c[on] % tile] = v[on]
    # unit diagonal for L (implicit in SuperLU's L) and for padding rows; the
    # upper solve multiplies by the stored reciprocal of U's diagonal
    d = np.arange(npad) if lower else np.arange(n, npad)
    diag[d // tile, d % tile, d % tile] = 1.0
    if not lower:
        k = np.arange(nb)[:, None]
        i = np.arange(tile)[None, :]
        diag[k, i, i] = 1.0 / diag[k, i, i]
    elif invert_lower_diag:
        # unit lower 32 x 32 diagonal tiles -> their inverses (the device
        # applies them as a GEMV; numerics within SuperLU's own floor, F9)
        eye = np.eye(tile)
        for k in range(nb):
            diag[k] = sla.solve_triangular(diag[k], eye, lower=True, unit_diagonal=True)
    off = ~on
    key = bj[off].astype(np.int64) * nb + bi[off]
    ukey, inv = np.unique(key, return_inverse=True)
    tiles = np.zeros((len(ukey), tile, tile))
    tiles[inv, r[off] % tile, c[off] % tile] = v[off]
    col_of = ukey // nb
    row_of = ukey % nb
    colptr = np.concatenate([[0], np.cumsum(np.bincount(col_of, minlength=nb))])
    # column-major storage inside each tile: element (i, j) at j*tile + i
    tiles_cm = np.ascontiguousarray(np.transpose(tiles, (0, 2, 1))).reshape(-1)
    diag_cm = np.ascontiguousarray(np.transpose(diag, (0, 2, 1))).reshape(-1)
    if len(tiles_cm) == 0:
        tiles_cm = np.zeros(tile * tile)
    return colptr, row_of, tiles_cm, diag_cm, nb


def coarse_direct_solve(system, method="dense"):
    return CoarseSolver(system, method)


# --------------------------------------------------------------- V-cycle

@dataclass
class MGLevel:
    system: object
    patches: Optional[VankaPatchSet]
    smoother: SmootherSpec
    prolong: Optional[object]  # StageTransfer from the next-coarser level


class _LevelBuffers:
    def __init__(self, dim, device):
        import torch
        self.x = torch.zeros(dim, dtype=torch.float64, device=device)
        self.b = torch.zeros(dim, dtype=torch.float64, device=device)
        self.r = torch.zeros(dim, dtype=torch.float64, device=device)
        self.d = torch.zeros(dim, dtype=torch.float64, device=device)


class MGHierarchyOp:
    """V-cycle preconditioner over rediscretised levels (solvers.py:295-356).

    ``levels`` runs coarsest to finest; ``levels[k].prolong`` maps level k-1
    to level k.  The cycle runs entirely on the device on per-level scratch
    buffers; ``precondition`` on a CUDA tensor can be captured once into a
    CUDA graph (``use_graph=True``) and replayed.
    """

    _ivk_device_native = True   # takes / returns device tensors as well as numpy

    def __init__(self, levels, coarse, use_graph=False):
        self.levels = levels
        self.coarse = coarse
        for k, lev in enumerate(levels[1:], start=1):
            if lev.prolong is None:
                raise ValueError(f"level {k} is missing its prolongation")
            if not hasattr(lev.prolong, "restrict_into"):
                # a reference-style stage prolongation (scipy CSR, fine x
                # coarse; bench.py:187-194): run it as a device transfer
                from .interop import as_transfer, is_matrix
                if not is_matrix(lev.prolong):
                    raise TypeError(f"level {k}: prolong must be a transfer or a sparse matrix")
                lev.prolong = as_transfer(lev.prolong, lev.system, levels[k - 1].system)
        self.use_graph = use_graph
        self._bufs = None
        self._graph = None
        # Parity-protocol hooks: record per-level intermediates
        # into a dict, and/or replace the coarse output by a given vector.
        self.trace = None
        self.coarse_override = None

    @property
    def finest(self):
        return self.levels[-1].system

    def _buffers(self):
        if self._bufs is None:
            from ._device import device
            dev = device()
            self._bufs = [_LevelBuffers(lev.system.dim, dev) for lev in self.levels]
            # Make sure every level's device data exists before any capture.
            for lev in self.levels:
                lev.system.device_data()
                if lev.patches is not None and lev is not self.levels[0]:
                    lev.patches.device_data()
                if lev.prolong is not None:
                    lev.prolong.device_data()
            self.coarse.device_data()
        return self._bufs

    # -- smoothing (fused device versions of solvers.py:321-332) --------------

    def _smooth(self, level, x, b, sweeps, x_zero=False):
        """x_zero: x is known to be 0, so the first residual b - A x is b
        itself (bitwise: A 0 = +0) and its K1 launch is skipped."""
        if sweeps == 0:
            return
        lev = self.levels[level]
        sm = lev.smoother
        sys_, pat = lev.system, lev.patches
        buf = self._bufs[level]
        w = pat.weights(sm.weighting)
        if sm.accel == "richardson":
            for k in range(sweeps):
                if k == 0 and x_zero:
                    loc = pat.apply_local(b)
                else:
                    sys_.apply_into(x, b, buf.r)
                    loc = pat.apply_local(buf.r)
                pat.combine(loc, x, 1.0, sm.omega, w, x)
            return
        if sm.accel == "chebyshev":
            a, bb = sm.cheby_a, sm.cheby_b
            theta = 0.5 * (bb + a)
            delta = 0.5 * (bb - a)
            sigma1 = theta / delta
            rho = 1.0 / sigma1
            if x_zero:
                loc = pat.apply_local(b)        # r = b
            else:
                sys_.apply_into(x, b, buf.r)
                loc = pat.apply_local(buf.r)
            pat.combine(loc, None, 0.0, sm.omega / theta, w, buf.d, accum=x)
            for k in range(1, sweeps):
                # r = r - A d (with r = b when the first residual was skipped)
                sys_.apply_into(buf.d, b if (k == 1 and x_zero) else buf.r, buf.r)
                loc = pat.apply_local(buf.r)
                rho_new = 1.0 / (2.0 * sigma1 - rho)
                pat.combine(loc, buf.d, rho_new * rho, 2.0 * rho_new / delta * sm.omega, w,
                            buf.d, accum=x)
                rho = rho_new
            return
        # GMRES-accelerated smoothing: inner FGMRES, fixed sweep count.
        import torch

        def precond(v):
            z = torch.empty_like(v)
            loc = pat.apply_local(v)
            pat.combine(loc, None, 0.0, sm.omega, w, z)
            return z

        xs, _ = fgmres(sys_.matvec, b, precond=precond, x0=x, rtol=0.0, atol=0.0,
                       maxiter=sweeps, restart=sweeps)
        x.copy_(xs)

    def _cycle(self, level, x, b, x_zero=False):
        """In place: x <- V-cycle(level, x, b) (solvers.py:334-347)."""
        tr = self.trace
        if level == 0:
            if self.coarse_override is not None:
                x.copy_(self.coarse_override)
            else:
                self.coarse.solve_into(b, x)
            if tr is not None:
                tr["coarse_in"] = b.clone()
                tr["coarse_out"] = x.clone()
            return
        lev = self.levels[level]
        buf = self._bufs[level]
        below = self._bufs[level - 1]
        self._smooth(level, x, b, lev.smoother.pre, x_zero=x_zero)
        if tr is not None:
            tr[f"pre_{level}"] = x.clone()
        lev.system.apply_into(x, b, buf.r)
        lev.prolong.restrict_into(buf.r, below.b)
        if tr is not None:
            tr[f"rc_{level}"] = below.b.clone()
        below.x.zero_()
        self._cycle(level - 1, below.x, below.b, x_zero=True)
        lev.prolong.prolong_add(below.x, x)
        self._smooth(level, x, b, lev.smoother.post)
        if tr is not None:
            tr[f"post_{level}"] = x.clone()

    # -- public API ----------------------------------------------------------

    def vcycle(self, level, x, b):
        """One V-cycle at ``level`` (returns a new array, solvers.py:334)."""
        from ._device import as_device_vector, to_host
        self._buffers()
        dim = self.levels[level].system.dim
        xd, host = as_device_vector(x, dim)
        bd, _ = as_device_vector(b, dim)
        out = xd.clone()
        self._cycle(level, out, bd)
        return to_host(out) if host else out

    def precondition_into(self, r, z):
        """Device: z = precondition(r) (solvers.py:349-356)."""
        from ._device import ptr, stream
        sys_ = self.finest
        dev = sys_.device_data()
        if getattr(sys_, "general", False):
            sys_.seed_constrained_into(r, z)
            self._cycle(len(self.levels) - 1, z, r)
            sys_.project_pressure_means(z)
            return z
        _lib.check(_lib.lib().ivk_seed_constrained(sys_.r, sys_.n_nodes, sys_.nc, sys_.n_p,
                                                   ptr(dev["tensors"]["cmask"]), ptr(r), ptr(z),
                                                   stream()), "seed_constrained")
        self._cycle(len(self.levels) - 1, z, r)
        sys_.project_pressure_means(z)
        return z

    def relinearize(self, u, assemblers):
        """Newton-cadence update: assemble J_N(u_l) on the
        GPU for every level from the device velocity ``u`` (nodal injection
        u_l = u[:2 n_l], bench.py:178-185), refactorise every level's patches
        in place (K7) and re-factor the coarsest operator (host SuperLU, as the
        reference's coarse_direct_solve -- its result is pinned against a
        hierarchy built from scratch at 1e-9 where the coarse operator has
        cond ~1e8; the Newton drivers, which only need a preconditioner, take
        the device route ``CoarseSolver.from_device_operator`` instead)."""
        if len(assemblers) != len(self.levels):
            raise ValueError("one ConvectionAssembler per level required")
        for k, (lev, asm) in enumerate(zip(self.levels, assemblers)):
            n = 2 * lev.system.n_nodes
            asm.assemble_into_system(lev.system, u[:n])
            if k > 0:
                lev.patches.factor()
                lev.system.mark_host_stale()
        s0 = self.levels[0].system
        s0.download_convection()
        self.coarse = CoarseSolver(s0, getattr(self.coarse, "method", "dense"))
        self._graph = None
        self._bufs = None

    def _graph_precondition(self, r):
        import torch
        if self._graph is None:
            self._g_in = torch.zeros_like(r)
            self._g_out = torch.zeros_like(r)
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                self.precondition_into(self._g_in, self._g_out)  # warm-up (attributes, caches)
            torch.cuda.current_stream().wait_stream(s)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self.precondition_into(self._g_in, self._g_out)
            self._graph = g
        self._g_in.copy_(r)
        self._graph.replay()
        return self._g_out.clone()

    def precondition_to(self, r, out):
        """Device: out = precondition(r) without allocating (graph or eager)."""
        self._buffers()
        if self.use_graph and all(l.smoother.accel != "gmres" for l in self.levels[1:]):
            if self._graph is None:
                self._graph_precondition(r)
            self._g_in.copy_(r)
            self._graph.replay()
            out.copy_(self._g_out)
        else:
            self.precondition_into(r, out)
        return out

    def precondition(self, r):
        """Preconditioner application for FGMRES: approximately solve A z = r."""
        from ._device import as_device_vector, to_host
        import torch
        self._buffers()
        rd, host = as_device_vector(r, self.finest.dim)
        if self.use_graph and all(l.smoother.accel != "gmres" for l in self.levels[1:]):
            z = self._graph_precondition(rd)
        else:
            z = torch.empty_like(rd)
            self.precondition_into(rd, z)
        return to_host(z) if host else z


def vcycle(hierarchy, level, x, b):
    """Module-level alias (solvers.py:359-361)."""
    return hierarchy.vcycle(level, x, b)


# ----------------------------------------------------------------- FGMRES

def _is_torch(v):
    try:
        import torch
        return isinstance(v, torch.Tensor)
    except ImportError:  # pragma: no cover
        return False


def fgmres(op_apply, b, precond=None, x0=None, rtol=1e-8, atol=0.0, maxiter=100, restart=30):
    """Flexible right-preconditioned GMRES (solvers.py:364-443), on the device.

    Same algorithm and statistics as the reference: MGS Arnoldi, Givens
    rotations, restart, the true residual at each cycle end, the monotone
    envelope of the reported norms.  The Krylov basis, the Hessenberg matrix,
    the rotations and the triangular solve all live in device memory (libivk
    K9); the host reads back one scalar (the residual estimate) per
    iteration to decide convergence.  A numpy ``b`` is copied up, solved on
    the device and the solution returned as numpy (numpy callables are
    wrapped at the edge; this package's own operator and V-cycle run
    natively)."""
    from ._device import as_device_vector, to_host
    if restart < 1 or maxiter < 0:
        raise ValueError("restart must be >= 1 and maxiter >= 0")
    if _is_torch(b):
        return _fgmres_device(op_apply, b, precond, x0, rtol, atol, maxiter, restart)
    n = int(np.asarray(b).shape[0])
    bd, _ = as_device_vector(b, n)
    x0d = None if x0 is None else as_device_vector(x0, n)[0]
    op_d = op_apply if getattr(getattr(op_apply, "__self__", None), "_ivk_device_native",
                               False) else _device_callable(op_apply, True)
    pc_d = None
    if precond is not None:
        pc_d = precond if getattr(getattr(precond, "__self__", None), "_ivk_device_native",
                                  False) else _device_callable(precond, True)
    x, stats = _fgmres_device(op_d, bd, pc_d, x0d, rtol, atol, maxiter, restart)
    return to_host(x), stats


class _KrylovWorkspace:
    """Device storage of one FGMRES restart cycle, allocated once per
    (n, restart) and reused (uninitialised: every row is written before it
    is read)."""

    def __init__(self, n, m, device):
        import torch
        f64 = dict(dtype=torch.float64, device=device)
        self.n, self.m = n, m
        self.V = torch.empty(m + 1, n, **f64)
        self.Z = torch.empty(m, n, **f64)
        self.w = torch.empty(n, **f64)
        self.r = torch.empty(n, **f64)
        self.tmp = torch.empty(n, **f64)
        self.H = torch.zeros((m + 1) * m + 1, **f64)   # column-major, ld = m + 1
        self.rot = torch.zeros(3 * (m + 1), **f64)     # cs | sn | g
        self.y = torch.zeros(m + 1, **f64)
        self.scal = torch.zeros(4, **f64)              # norm / est scratch
        self.red = _lib.reduction_scratch()
        self.host = torch.zeros(4, dtype=torch.float64).pin_memory()
        self.events = [torch.cuda.Event(), torch.cuda.Event()]


def _fgmres_device(op_apply, b, precond, x0, rtol, atol, maxiter, restart):
    import torch
    from ._device import ptr, stream
    L = _lib.lib()
    n = b.numel()
    f64 = dict(dtype=torch.float64, device=b.device)
    x = torch.zeros(n, **f64) if x0 is None else torch.as_tensor(x0, **f64).clone()
    if precond is None:
        precond = lambda v: v
    stats = KrylovStats()

    # Allocation-free fast paths for this package's own operator / cycle.
    pre_to = None
    owner = None
    if getattr(precond, "__func__", None) is MGHierarchyOp.precondition:
        owner = precond.__self__
        pre_to = owner.precondition_to
    op_into = None
    if getattr(getattr(op_apply, "__self__", None), "apply_into", None) is not None and \
            getattr(op_apply, "__name__", "") == "matvec":
        sysobj = op_apply.__self__
        op_into = lambda v, out: sysobj.apply_into(v, None, out)

    m_max = max(1, min(restart, maxiter))
    ws = None
    if owner is not None:
        ws = getattr(owner, "_krylov_ws", None)
        if ws is not None and (ws.n != n or ws.m < m_max or ws.V.device != b.device):
            ws = None
    if ws is None:
        ws = _KrylovWorkspace(n, m_max, b.device)
        if owner is not None:
            owner._krylov_ws = ws
    ld = ws.m + 1
    cs, sn, g = ws.rot[:ld], ws.rot[ld:2 * ld], ws.rot[2 * ld:]
    st = stream()

    def read(k):
        """Device scalar ws.scal[k] -> host (one small D2H)."""
        ws.host[k:k + 1].copy_(ws.scal[k:k + 1], non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return float(ws.host[k])

    def residual_norm(xv):
        """ws.r = b - A x; returns ||ws.r||."""
        if op_into is not None:
            op_into(xv, ws.tmp)
            ax = ws.tmp
        else:
            ax = torch.as_tensor(op_apply(xv), **f64)
        _lib.check(L.ivk_axpby(n, 1.0, ptr(b), -1.0, ptr(ax), ptr(ws.r), st), "residual")
        _lib.check(L.ivk_norm(n, ptr(ws.r), ptr(ws.scal), ptr(ws.red), st), "norm")
        return read(0)

    norm0 = residual_norm(x)
    stats.residual_norms.append(norm0)
    tol = max(rtol * norm0, atol)
    if norm0 <= tol:
        stats.final_residual = norm0
        stats.relative_residual = 0.0 if norm0 == 0 else 1.0
        stats.converged = True
        return x, stats

    beta = norm0
    while stats.iterations < maxiter:
        m = min(restart, maxiter - stats.iterations)
        # V_0 = r / beta, g = beta e_0 (device)
        _lib.check(L.ivk_axpby(n, 1.0 / beta, ptr(ws.r), 0.0, None, ptr(ws.V[0]), st), "scale")
        g.zero_()
        g[0:1].fill_(beta)
        # Arnoldi steps are enqueued one ahead of the convergence test: step
        # j's residual estimate is copied to a pinned slot behind it in stream
        # order and read while step j + 1 already runs, so the device never
        # idles on the host's read-back.  Close to the tolerance (last known
        # estimate within 100x) the test turns synchronous again, so a step is
        # only ever enqueued in vain if the estimate drops by more than 100x
        # in one step -- and then it is simply not counted: it writes Z[j],
        # V[j+1], column j of H and g[j..j+1], none of which the solution over
        # the first j columns reads.  Same decisions, same counts, same
        # history as the step-by-step loop.
        k = 0
        done = False
        last_est = beta
        pending = None          # (step index, event) whose estimate is in flight
        for j in range(m):
            if pre_to is not None:
                pre_to(ws.V[j], ws.Z[j])
            else:
                ws.Z[j].copy_(torch.as_tensor(precond(ws.V[j]), **f64))
            if op_into is not None:
                op_into(ws.Z[j], ws.w)
            else:
                ws.w.copy_(torch.as_tensor(op_apply(ws.Z[j]), **f64))
            hcol = ws.H[j * ld:]
            _lib.check(L.ivk_mgs(n, ptr(ws.V), n, j + 1, ptr(ws.w), ptr(hcol), ptr(ws.V[j + 1]),
                                 ptr(ws.red), st), "mgs")
            _lib.check(L.ivk_givens(j, ld, ptr(ws.H), ptr(cs), ptr(sn), ptr(g), ptr(ws.scal[1:]),
                                    st), "givens")
            slot = 2 + (j & 1)
            ws.host[slot:slot + 1].copy_(ws.scal[1:2], non_blocking=True)
            ev = ws.events[j & 1]
            ev.record()
            if pending is not None:
                # the previous step's estimate (complete by now or soon: this
                # step's work is already queued behind it)
                pj, pev = pending
                pev.synchronize()
                est = float(ws.host[2 + (pj & 1)])
                k = pj + 1
                stats.iterations += 1
                stats.residual_norms.append(est)
                last_est = est
                if est <= tol or stats.iterations >= maxiter:
                    done = True       # step j was enqueued in vain
                    break
            pending = (j, ev)
            last = j == m - 1 or stats.iterations + 1 >= maxiter
            if last or last_est <= 100.0 * tol:
                ev.synchronize()
                est = float(ws.host[slot])
                pending = None
                k = j + 1
                stats.iterations += 1
                stats.residual_norms.append(est)
                last_est = est
                if est <= tol or stats.iterations >= maxiter:
                    done = True
                    break
        if pending is not None and not done:   # (m steps enqueued, last one unread)
            pj, pev = pending
            pev.synchronize()
            k = pj + 1
            stats.iterations += 1
            stats.residual_norms.append(float(ws.host[2 + (pj & 1)]))
        _lib.check(L.ivk_hessenberg_solve(k, ld, ptr(ws.H), ptr(g), ptr(ws.y), st), "triu solve")
        _lib.check(L.ivk_lincomb(n, ptr(ws.Z), n, k, ptr(ws.y), ptr(x), st), "lincomb")
        true_norm = residual_norm(x)
        stats.residual_norms[-1] = true_norm
        beta = true_norm
        if true_norm <= tol:
            break

    stats.final_residual = residual_norm(x)
    stats.relative_residual = stats.final_residual / norm0 if norm0 > 0 else 0.0
    stats.converged = stats.final_residual <= tol
    stats.residual_norms = list(np.minimum.accumulate(stats.residual_norms))
    return x, stats
