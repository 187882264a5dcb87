"""Strip-partitioned fine-level IRK-Vanka sweep over N ranks.

Patches are independent given the residual, so a level shards by centre
vertex: rank p owns the patches of the vertices in its strip (vertices sorted
by (y, x), cut into N equal runs).  Per sweep, rank p

  1. computes the residual on the rows its patches read (K1 on a slice list,
     ``ivk_stage_apply_slices``) -- this needs x on a distance-2 halo;
  2. solves its own patches (K3, a ``VankaPatchSet`` over its vertices) and
     sums their contributions per DoF (K4 on its DoF list,
     ``ivk_patch_combine_list``);
  3. exchanges the partial sums of the DoFs it shares with its neighbours
     (the only reduction of the sweep), adding the partials in ascending rank
     order, so every rank holding a shared DoF computes the same bits;
  4. updates x on its DoFs (x + w W z, ``ivk_index_update``);
  5. exchanges x on the halo (each halo DoF comes from the lowest other rank
     whose patches cover it).

Both exchanges are NCCL point-to-point (``batch_isend_irecv``) of packed
buffers (``ivk_index_copy``) -- a few hundred KB per neighbour at cfg2, so they
are latency-bound and sized for NVLink launch latency, not bandwidth.  The
result equals the single-GPU sweep (solvers.py:232-239) up to the summation
order at the shared DoFs.  Coarse levels and the coarse solve stay replicated
(SURVEY.md §8(e)); this module shards the fine-level sweep, the unit the
north-star metric counts.

The plan (``shard_plans``) is host logic built identically on every rank from
the global tables; the per-rank ``ShardedSweep`` runs its local steps through
a backend (``DeviceBackend``: the ivk kernels; tests substitute a CPU oracle
backend to run the exchange logic over gloo) and its exchanges through a comm
(``DistComm`` over torch.distributed, or ``LoopbackGroup`` driving several
shards in one process).
"""

from dataclasses import dataclass, field

import numpy as np

from .patches import _ranges, build_patch_tables

__all__ = ["StripPartition", "ShardPlan", "shard_plans", "ShardedSweep", "DeviceBackend",
           "DistComm", "LoopbackGroup", "PeerShard", "PeerLoopback", "SymmetricPeers",
           "peer_holders"]


class StripPartition:
    """Vertices sorted by (y, x) and cut into ``nparts`` equal runs."""

    def __init__(self, mesh, nparts):
        if nparts < 1:
            raise ValueError("nparts must be >= 1")
        v = np.asarray(mesh.vertices)
        nv = len(v)
        if nparts > nv:
            raise ValueError("more parts than vertices")
        key = np.lexsort((v[:, 0], v[:, 1]))
        self.part = np.empty(nv, dtype=np.int64)
        self.part[key] = (np.arange(nv) * nparts) // nv
        self.nparts = nparts


@dataclass
class ShardPlan:
    rank: int
    nparts: int
    vertices: np.ndarray                  # own patch centres
    dofs: np.ndarray                      # sorted stage DoFs of the own patches
    slices: np.ndarray                    # K1 warp slices covering the rows in `dofs`
    shared: dict = field(default_factory=dict)     # q -> sorted DoFs shared with q
    halo_recv: dict = field(default_factory=dict)  # q -> sorted halo DoFs provided by q
    halo_send: dict = field(default_factory=dict)  # q -> sorted own DoFs q needs from us

    @property
    def neighbours(self):
        return sorted(set(self.shared) | set(self.halo_recv) | set(self.halo_send))


def _node_dofs(system, nodes, pres):
    """All stage DoFs (both components) of scalar P2 nodes and P1 nodes."""
    sd, n_u = system.stage_dim, system.n_u
    out = []
    for s in range(system.r):
        out.append(s * sd + 2 * nodes)
        out.append(s * sd + 2 * nodes + 1)
        out.append(s * sd + n_u + pres)
    return np.unique(np.concatenate(out))


def shard_plans(system, mesh, partition):
    """Every rank's plan (identical on all ranks: pure function of the global
    tables)."""
    if system.nc != 2:
        raise ValueError("the sharded sweep is implemented for 2-D levels")
    t = build_patch_tables(mesh, system.n_nodes, system.n_p, system.r, system.node_constrained)
    part = partition.part
    N = partition.nparts
    sd, n_u, dim = system.stage_dim, system.n_u, system.dim
    slot_part = part[t.order]
    entry_part = np.repeat(slot_part, t.sizes)
    # (dof, part) incidence, unique
    pairs = np.unique(t.idx.astype(np.int64) * N + entry_part)
    pd_dof, pd_part = pairs // N, pairs % N
    dofs_of = [pd_dof[pd_part == p] for p in range(N)]
    # lowest part covering each DoF (halo provider), -1 if none (constrained)
    first = np.full(dim, -1, dtype=np.int64)
    # pairs are sorted by dof then part: the first occurrence per dof is the min part
    u, iu = np.unique(pd_dof, return_index=True)
    first[u] = pd_part[iu]
    # DoFs covered by >= 2 parts
    counts = np.bincount(pd_dof, minlength=dim)
    nsl_v = (system.n_nodes + 15) >> 4
    blk = system.blocks
    rowptr, col = np.asarray(blk.rowptr), np.asarray(blk.col)
    brow, bcol = np.asarray(blk.b_rowptr), np.asarray(blk.b_col)
    # B^T pattern: pressure q -> nodes
    bt_nodes = np.repeat(np.arange(system.n_nodes), np.diff(brow))
    bt_order = np.argsort(bcol, kind="stable")
    bt_ptr = np.concatenate([[0], np.cumsum(np.bincount(bcol, minlength=system.n_p))])
    bt_col = bt_nodes[bt_order]
    plans = []
    for p in range(N):
        D = dofs_of[p]
        loc = D % sd
        vel = loc < n_u
        rnodes = np.unique(loc[vel] // 2)
        rpres = np.unique(loc[~vel] - n_u)
        slices = np.unique(np.concatenate([rnodes // 16, nsl_v + rpres // 32])).astype(np.int64)
        # columns the rows in D read: P2 pattern + B (velocity rows), B^T (pressure rows)
        nodes = np.unique(np.concatenate([
            rnodes, col[_ranges(rowptr[rnodes], rowptr[rnodes + 1] - rowptr[rnodes])],
            bt_col[_ranges(bt_ptr[rpres], bt_ptr[rpres + 1] - bt_ptr[rpres])]]))
        pres = np.unique(np.concatenate([
            rpres, bcol[_ranges(brow[rnodes], brow[rnodes + 1] - brow[rnodes])]]))
        need = _node_dofs(system, nodes, pres)
        halo = np.setdiff1d(need, D, assume_unique=True)
        halo = halo[first[halo] >= 0]          # constrained DoFs never change
        plan = ShardPlan(rank=p, nparts=N, vertices=np.flatnonzero(part == p), dofs=D,
                         slices=slices)
        prov = first[halo]
        for q in np.unique(prov):
            plan.halo_recv[int(q)] = halo[prov == q]
        plans.append(plan)
    # shared DoFs and halo send lists
    multi = np.flatnonzero(counts >= 2)
    sel = np.isin(pd_dof, multi)
    md, mp = pd_dof[sel], pd_part[sel]
    for p in range(N):
        mine = md[mp == p]
        for q in range(N):
            if q == p:
                continue
            s = np.intersect1d(mine, md[mp == q], assume_unique=True)
            if len(s):
                plans[p].shared[q] = s
        for q in range(N):
            if q != p and p in plans[q].halo_recv:
                plans[p].halo_send[q] = plans[q].halo_recv[p]
    return plans


class DeviceBackend:
    """The ivk kernels on CUDA tensors (the product path)."""

    def __init__(self, system, mesh, plan, mode="auto", weights=None):
        import torch
        from . import _lib
        from ._device import require_cuda, upload
        from .solvers import VankaPatchSet
        require_cuda()
        self.system = system
        self.patches = VankaPatchSet(system, mesh, mode=mode, vertices=plan.vertices)
        self.lib = _lib.lib()
        self.check = _lib.check
        self.dofs = upload(plan.dofs, np.int32)
        self.slices = upload(plan.slices, np.int32)
        self.w = None if weights is None else upload(weights, np.float64)
        self.dim = system.dim
        self._torch = torch

    def index(self, a):
        from ._device import upload
        return upload(np.asarray(a), np.int32)

    def empty(self, n):
        # zero-filled: the ordered partial sums zero their target by 0 * old
        return self._torch.zeros(n, dtype=self._torch.float64, device="cuda")

    def residual(self, x, b, r):
        from ._device import ptr, stream
        self.check(self.lib.ivk_stage_apply_slices(self.system.desc, ptr(self.slices),
                                                   len(self.slices), ptr(x), ptr(b), ptr(r),
                                                   stream()), "stage_apply_slices")

    def own_patch_sum(self, r, z):
        from ._device import ptr, stream
        local = self.patches.apply_local(r)
        self.check(self.lib.ivk_patch_combine_list(self.patches.desc, ptr(self.dofs),
                                                   len(self.dofs), ptr(local), None, 0.0, 1.0,
                                                   None, ptr(z), None, stream()),
                   "patch_combine_list")

    def index_copy(self, n, src_idx, src, dst_idx, dst, beta):
        from ._device import ptr, stream
        self.check(self.lib.ivk_index_copy(n, ptr(src_idx), ptr(src), ptr(dst_idx), ptr(dst),
                                           float(beta), stream()), "index_copy")

    def update(self, x, omega, z):
        """x[d] = x[d] + omega W[d] z[d] on the own DoFs."""
        from ._device import ptr, stream
        self.check(self.lib.ivk_index_update(len(self.dofs), ptr(self.dofs), 1.0, ptr(x),
                                             float(omega), ptr(self.w), ptr(z), ptr(x),
                                             stream()), "index_update")

    def zero(self, z):
        from ._device import ptr, stream
        self.check(self.lib.ivk_index_update(len(self.dofs), ptr(self.dofs), 0.0, None, 0.0,
                                             None, ptr(z), ptr(z), stream()), "index_update")


class ShardedSweep:
    """One rank's part of ``apply_vanka`` over a strip partition.

    ``sweep(x, b, comm)`` updates the full-length ``x`` in place on this
    rank's DoFs and halo (other entries are stale by design)."""

    def __init__(self, plan, backend, omega=0.5):
        self.plan = plan
        self.be = backend
        self.omega = float(omega)
        n = backend.dim
        self.r = backend.empty(n)
        self.z = backend.empty(n)
        self.zt = backend.empty(n)
        self.idx = {"dofs": backend.index(plan.dofs)}
        self.sh = {q: backend.index(s) for q, s in plan.shared.items()}
        self.hr = {q: backend.index(s) for q, s in plan.halo_recv.items()}
        self.hs = {q: backend.index(s) for q, s in plan.halo_send.items()}
        self.zsend = {q: backend.empty(len(s)) for q, s in plan.shared.items()}
        self.zrecv = {q: backend.empty(len(s)) for q, s in plan.shared.items()}
        self.xsend = {q: backend.empty(len(s)) for q, s in plan.halo_send.items()}
        self.xrecv = {q: backend.empty(len(s)) for q, s in plan.halo_recv.items()}

    # phases (LoopbackGroup interleaves them across shards)
    def local(self, x, b):
        be = self.be
        be.residual(x, b, self.r)
        be.own_patch_sum(self.r, self.z)
        for q, buf in self.zsend.items():
            be.index_copy(len(buf), self.sh[q], self.z, None, buf, 0.0)
        return self.zsend, self.zrecv

    def reduce_update(self, x):
        be = self.be
        be.zero(self.zt)
        me = self.plan.rank
        d = self.idx["dofs"]
        for q in sorted(set(self.sh) | {me}):
            if q == me:
                be.index_copy(len(self.plan.dofs), d, self.z, d, self.zt, 1.0)
            else:
                be.index_copy(len(self.zrecv[q]), None, self.zrecv[q], self.sh[q], self.zt, 1.0)
        be.update(x, self.omega, self.zt)
        for q, buf in self.xsend.items():
            be.index_copy(len(buf), self.hs[q], x, None, buf, 0.0)
        return self.xsend, self.xrecv

    def halo(self, x):
        for q, buf in self.xrecv.items():
            self.be.index_copy(len(buf), None, buf, self.hr[q], x, 0.0)

    def sweep(self, x, b, comm):
        comm.exchange(*self.local(x, b))
        comm.exchange(*self.reduce_update(x))
        self.halo(x)
        return x


class DistComm:
    """Point-to-point exchange over torch.distributed (NCCL on CUDA tensors,
    gloo on CPU tensors)."""

    def exchange(self, sends, recvs):
        import torch.distributed as dist
        ops = [dist.P2POp(dist.isend, t, q) for q, t in sorted(sends.items())]
        ops += [dist.P2POp(dist.irecv, t, q) for q, t in sorted(recvs.items())]
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()


class LoopbackGroup:
    """Drives several shards in one process (tests): the exchanges become
    buffer copies between the shards, phase by phase."""

    def __init__(self, shards):
        self.shards = shards

    def _deliver(self, outs):
        for p, (sends, _) in enumerate(outs):
            for q, buf in sends.items():
                outs[q][1][p].copy_(buf)

    def sweep(self, xs, b):
        self._deliver([s.local(x, b) for s, x in zip(self.shards, xs)])
        self._deliver([s.reduce_update(x) for s, x in zip(self.shards, xs)])
        for s, x in zip(self.shards, xs):
            s.halo(x)
        return xs


# ------------------------------------------------- fused exchange over peers

def peer_holders(plan):
    """CSR (ptr, ranks) over the plan's own DoFs: the ranks whose patches
    contain each DoF, ascending (the fused kernel's summation order)."""
    n = len(plan.dofs)
    cols = [np.full(n, plan.rank, dtype=np.int64)]
    rows = [np.arange(n)]
    for q, dd in plan.shared.items():
        cols.append(np.full(len(dd), q, dtype=np.int64))
        rows.append(np.searchsorted(plan.dofs, dd))
    rows, cols = np.concatenate(rows), np.concatenate(cols)
    order = np.lexsort((cols, rows))
    ptr = np.concatenate([[0], np.cumsum(np.bincount(rows, minlength=n))])
    return ptr.astype(np.int64), cols[order]


class PeerShard:
    """One rank's sweep with the exchange fused into the update kernel
    (``ivk_peer_combine_update``): after K1 + K3 on its patches, the rank sums
    every own DoF's contributions from ALL ranks holding it -- reading their
    patch outputs through peer pointers (NVLink P2P loads) in ascending rank
    order -- and updates x, then pulls its halo straight from the owners' x.
    No packed buffers, no send/recv: 2 kernels + 1 copy kernel per provider.

    The peer table (``set_peers``) maps rank -> (dof_ptr, dof_pos, local, x)
    device pointers: in-process shards in tests (``PeerLoopback``), symmetric
    memory mapped over NVLink across processes (``SymmetricPeers``)."""

    def __init__(self, plan, backend, omega=0.5, local=None):
        import torch
        from ._device import upload
        self.plan = plan
        self.be = backend
        self.omega = float(omega)
        self.r = backend.empty(backend.dim)
        dev = backend.patches.device_data()
        self.local = dev["local"] if local is None else local
        self.dof_ptr, self.dof_pos = dev["dof_ptr"], dev["dof_pos"]
        hp, hr = peer_holders(plan)
        self.holder_ptr = upload(hp, np.int32)
        self.holder_rank = upload(hr, np.int32)
        self.dofs = backend.dofs
        self.hr = {q: backend.index(s_) for q, s_ in plan.halo_recv.items()}
        self.peers_dev = None
        self.peer_x = {}
        self._torch = torch

    def view(self):
        """(dof_ptr, dof_pos, local) device pointers of this rank."""
        return (self.dof_ptr.data_ptr(), self.dof_pos.data_ptr(), self.local.data_ptr())

    def set_peers(self, views, x_ptrs):
        """views[q] = (dof_ptr, dof_pos, local) and x_ptrs[q] = x of rank q, as
        device addresses valid on this rank."""
        tbl = np.asarray(views, dtype=np.uint64).reshape(-1, 3).view(np.int64)
        self.peers_dev = self._torch.from_numpy(tbl.copy()).cuda()
        self.peer_x = dict(enumerate(x_ptrs))

    def local_phase(self, x, b):
        self.be.residual(x, b, self.r)
        self.be.patches.apply_local(self.r, self.local)

    def combine_phase(self, x):
        from ._device import ptr, stream
        from . import _lib
        _lib.check(_lib.lib().ivk_peer_combine_update(
            len(self.plan.dofs), ptr(self.dofs), ptr(self.holder_ptr), ptr(self.holder_rank),
            ptr(self.peers_dev), self.omega, ptr(self.be.w), ptr(x), stream()),
            "peer_combine_update")

    def halo_phase(self, x):
        from ._device import ptr, stream
        from . import _lib
        for q, idx in self.hr.items():
            # x[idx] = x_q[idx]: a gather over NVLink from the owner's iterate
            _lib.check(_lib.lib().ivk_index_copy(len(idx), ptr(idx), self.peer_x[q], ptr(idx),
                                                 ptr(x), 0.0, stream()), "index_copy(peer)")


class PeerLoopback:
    """All ranks' shards in one process (the 1-GPU emulation of the peer
    path: every phase runs for all shards before the next phase, so no kernel
    ever waits on another)."""

    def __init__(self, shards, xs):
        self.shards = shards
        views = [s.view() for s in shards]
        x_ptrs = [x.data_ptr() for x in xs]
        for s in shards:
            s.set_peers(views, x_ptrs)

    def sweep(self, xs, b):
        for s, x in zip(self.shards, xs):
            s.local_phase(x, b)
        for s, x in zip(self.shards, xs):
            s.combine_phase(x)
        for s, x in zip(self.shards, xs):
            s.halo_phase(x)
        return xs


class SymmetricPeers:
    """Multi-process wiring of ``PeerShard`` (one rank per GPU): the patch
    outputs, DoF tables and iterate live in torch symmetric memory, whose
    rendezvous maps every peer's buffer into this rank's address space over
    NVLink; the phases are separated by process-group barriers (host-side:
    no kernel waits on another rank).  Not exercised here -- the environment
    has one GPU; the kernel and the phase logic are the ones PeerLoopback
    tests."""

    def __init__(self, plan, backend, x, omega=0.5, group=None):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm
        self.group = group if group is not None else dist.group.WORLD
        dev = backend.patches.device_data()
        world = dist.get_world_size(self.group)

        def symmetric(src):
            n = torch.tensor([src.numel()], device=src.device)
            dist.all_reduce(n, op=dist.ReduceOp.MAX, group=self.group)
            t = symm.empty(int(n.item()), dtype=src.dtype, device=src.device)
            t[:src.numel()].copy_(src)
            return t, symm.rendezvous(t, self.group)

        self.local, hl = symmetric(dev["local"])
        self.dof_ptr, hp = symmetric(dev["dof_ptr"])
        self.dof_pos, hq = symmetric(dev["dof_pos"])
        self.x, hx = symmetric(x)
        self.shard = PeerShard(plan, backend, omega, local=self.local[:dev["local"].numel()])
        views = [(hp.buffer_ptrs[q], hq.buffer_ptrs[q], hl.buffer_ptrs[q]) for q in range(world)]
        self.shard.set_peers(views, [hx.buffer_ptrs[q] for q in range(world)])

    def sweep(self, b):
        import torch.distributed as dist
        x = self.x[:self.shard.be.dim]
        self.shard.local_phase(x, b)
        dist.barrier(group=self.group)
        self.shard.combine_phase(x)
        dist.barrier(group=self.group)
        self.shard.halo_phase(x)
        dist.barrier(group=self.group)
        return x
