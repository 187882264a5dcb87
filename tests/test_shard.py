"""Strip-sharded fine-level sweep (shard.py).

CPU: plan invariants, and the full exchange logic over a 2-rank gloo group
with the local steps done by the CPU oracle (``OracleBackend`` -- test
infrastructure, the product backend is the ivk kernels).  GPU: the device
backend, several shards driven in one process (``LoopbackGroup``), against
the single-GPU sweep."""

import os
import socket

import numpy as np
import pytest

from harness import oracle_levels, rel, setup
from oracle.irk_vanka_oracle import OraclePatches, oracle_apply_vanka, random_rhs


def _problem(name="s3"):
    from paper_2202_07381_b200.stages import StageSystem
    disc, tab, conv, case = setup(name)
    k = disc.num_levels - 1
    S = StageSystem(disc.blocks[k], tab, case["dt"], disc.cdofs[k],
                    None if conv is None else conv[k])
    return disc, tab, conv, case, S, disc.hier.levels[k]


@pytest.mark.parametrize("nparts", [2, 3, 5])
def test_plan_invariants(nparts):
    from paper_2202_07381_b200.patches import build_patch_tables
    from paper_2202_07381_b200.shard import StripPartition, shard_plans
    disc, tab, conv, case, S, mesh = _problem()
    plans = shard_plans(S, mesh, StripPartition(mesh, nparts))
    t = build_patch_tables(mesh, S.n_nodes, S.n_p, S.r, S.node_constrained)
    free = np.flatnonzero(t.multiplicity > 0)
    # the shards' patches partition the vertices; their DoFs cover every free DoF
    assert np.array_equal(np.sort(np.concatenate([p.vertices for p in plans])),
                          np.arange(mesh.num_vertices))
    assert np.array_equal(np.unique(np.concatenate([p.dofs for p in plans])), free)
    nsl_v = (S.n_nodes + 15) >> 4
    for p in plans:
        # shared lists are symmetric and are exactly the intersections
        for q, s in p.shared.items():
            assert np.array_equal(s, plans[q].shared[p.rank])
            assert np.array_equal(s, np.intersect1d(p.dofs, plans[q].dofs))
        # halo DoFs come from a shard that owns them, are not own, send == recv
        for q, h in p.halo_recv.items():
            assert np.all(np.isin(h, plans[q].dofs)) and not np.any(np.isin(h, p.dofs))
            assert np.array_equal(plans[q].halo_send[p.rank], h)
        # K1 slices cover every own row
        loc = p.dofs % S.stage_dim
        vel = loc < S.n_u
        rows = np.concatenate([(loc[vel] // 2) // 16, nsl_v + (loc[~vel] - S.n_u) // 32])
        assert np.all(np.isin(rows, p.slices))
        # the halo closes the residual: every column an own row reads is own,
        # halo or constrained (A materialised on this small level)
    A = S.materialize(limit=10 ** 6).tocsr()
    cons = np.setdiff1d(np.arange(S.dim), free)
    for p in plans:
        cols = np.unique(A[p.dofs].indices)
        have = np.concatenate([p.dofs, cons] + list(p.halo_recv.values()))
        assert np.all(np.isin(cols, have))


class OracleBackend:
    """CPU stand-in for the device backend (tests only): numpy restatement of
    the reference sweep steps on torch CPU tensors (so gloo can send them)."""

    def __init__(self, op, vels, idxs, plan, weights=None):
        self.op = op
        self.dim = op.dim
        self.pat = OraclePatches(op, vels, idxs, members=plan.vertices)
        self.dofs = plan.dofs
        self.w = weights

    def index(self, a):
        return None if a is None else np.asarray(a, dtype=np.int64)

    def empty(self, n):
        import torch
        return torch.zeros(n, dtype=torch.float64)

    def residual(self, x, b, r):
        r.numpy()[:] = b.numpy() - self.op.matvec(x.numpy())

    def own_patch_sum(self, r, z):
        z.numpy()[self.dofs] = self.pat.solve_additive(r.numpy())[self.dofs]

    def index_copy(self, n, src_idx, src, dst_idx, dst, beta):
        s = src.numpy()
        d = dst.numpy()
        v = s[src_idx] if src_idx is not None else s[:n]
        if dst_idx is None:
            d[:n] = v + beta * d[:n] if beta else v
        else:
            d[dst_idx] = v + beta * d[dst_idx] if beta else v

    def update(self, x, omega, z):
        d = self.dofs
        w = 1.0 if self.w is None else self.w[d]
        x.numpy()[d] = x.numpy()[d] + omega * w * z.numpy()[d]

    def zero(self, z):
        z.numpy()[self.dofs] = 0.0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from paper_2202_07381_b200.shard import DistComm, ShardedSweep, StripPartition, shard_plans
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    disc, tab, conv, case, S, mesh = _problem()
    lv = oracle_levels(disc, tab, case["dt"], None, levels=[disc.num_levels - 1])[0]
    op = lv["op"]
    from oracle.irk_vanka_oracle import oracle_patch_indices
    vels, idxs = oracle_patch_indices(mesh.cells, mesh.cell_to_edges, mesh.num_vertices, op)
    plans = shard_plans(S, mesh, StripPartition(mesh, world))
    plan = plans[rank]
    w = lv["patches"].pou_weights(op.dim)
    sw = ShardedSweep(plan, OracleBackend(op, vels, idxs, plan, weights=w), omega=0.5)
    b = torch.from_numpy(random_rhs(op, 3))
    x0 = np.random.default_rng(4).uniform(-1, 1, op.dim)
    x0[op.constrained_stage_dofs()] = 0.0
    x = torch.from_numpy(x0.copy())
    comm = DistComm()
    for _ in range(2):
        sw.sweep(x, b, comm)
    q.put((rank, plan.dofs, x.numpy()[plan.dofs].copy()))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_sweep_two_ranks_gloo(monkeypatch):
    import multiprocessing as mp
    # two BLAS-threaded workers on a shared host thrash: one thread each
    for v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        monkeypatch.setenv(v, "1")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=300) for _ in procs), key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    disc, tab, conv, case, S, mesh = _problem()
    lv = oracle_levels(disc, tab, case["dt"], None, levels=[disc.num_levels - 1])[0]
    op, pat = lv["op"], lv["patches"]
    b = random_rhs(op, 3)
    x = np.random.default_rng(4).uniform(-1, 1, op.dim)
    x[op.constrained_stage_dofs()] = 0.0
    w = pat.pou_weights(op.dim)
    for _ in range(2):
        x = oracle_apply_vanka(pat, op, x, b, 0.5, weights=w)
    got = x.copy()
    for _, dofs, vals in res:
        got[dofs] = vals
    assert rel(got, x) <= 1e-13
    # the shared DoFs agree bitwise between the two ranks
    shared = np.intersect1d(res[0][1], res[1][1])
    a = dict(zip(res[0][1], res[0][2]))
    c = dict(zip(res[1][1], res[1][2]))
    assert all(a[d] == c[d] for d in shared)


@pytest.mark.gpu
@pytest.mark.parametrize("name,nparts,mode", [("s3", 2, "auto"), ("s3", 3, "kron"),
                                              ("ns", 4, "auto"), ("crossed", 2, "full"),
                                              ("s3", 2, "modal"), ("crossed", 3, "modal")])
def test_sharded_sweep_device_loopback(name, nparts, mode):
    import torch
    from paper_2202_07381_b200 import VankaPatchSet, apply_vanka
    from paper_2202_07381_b200.shard import (DeviceBackend, LoopbackGroup, ShardedSweep,
                                             StripPartition, shard_plans)
    disc, tab, conv, case, S, mesh = _problem(name)
    full = VankaPatchSet(S, mesh, mode=mode)
    w = full.pou_weights()
    plans = shard_plans(S, mesh, StripPartition(mesh, nparts))
    shards = [ShardedSweep(p, DeviceBackend(S, mesh, p, mode=mode, weights=w), omega=0.5)
              for p in plans]
    rng = np.random.default_rng(11)
    b = rng.uniform(-1, 1, S.dim)
    x0 = rng.uniform(-1, 1, S.dim)
    cd = S.constrained_stage_dofs()
    b[cd] = 0.0
    x0[cd] = 0.0
    bd = torch.from_numpy(b).cuda()
    xs = [torch.from_numpy(x0.copy()).cuda() for _ in plans]
    ref = torch.from_numpy(x0.copy()).cuda()
    grp = LoopbackGroup(shards)
    for _ in range(3):
        grp.sweep(xs, bd)
        ref = apply_vanka(full, S, ref, bd, omega=0.5, weights="pou")
    got = ref.clone()
    for p, x in zip(plans, xs):
        idx = torch.from_numpy(p.dofs).cuda()
        got[idx] = x[idx]
    assert rel(got.cpu().numpy(), ref.cpu().numpy()) <= 1e-12
    for p, x in zip(plans, xs):
        for q, s in p.shared.items():
            idx = torch.from_numpy(s).cuda()
            assert torch.equal(x[idx], xs[q][idx])


@pytest.mark.gpu
@pytest.mark.parametrize("name,nparts,mode", [("s3", 2, "modal"), ("s3", 3, "kron"),
                                              ("ns", 4, "auto"), ("crossed", 3, "full")])
def test_peer_fused_sweep_loopback(name, nparts, mode):
    """The fused exchange (ivk_peer_combine_update reading the other shards'
    patch outputs through peer pointers, halo pulled from the owners' x) equals
    the single-GPU sweep, and shared DoFs carry the same bits on every shard.
    Phases run for all shards in turn (one kernel never waits on another)."""
    import torch
    from paper_2202_07381_b200 import VankaPatchSet, apply_vanka
    from paper_2202_07381_b200.shard import (DeviceBackend, PeerLoopback, PeerShard,
                                             StripPartition, shard_plans)
    disc, tab, conv, case, S, mesh = _problem(name)
    full = VankaPatchSet(S, mesh, mode=mode)
    w = full.pou_weights()
    plans = shard_plans(S, mesh, StripPartition(mesh, nparts))
    shards = [PeerShard(p, DeviceBackend(S, mesh, p, mode=mode, weights=w), omega=0.5)
              for p in plans]
    rng = np.random.default_rng(12)
    b = rng.uniform(-1, 1, S.dim)
    x0 = rng.uniform(-1, 1, S.dim)
    cd = S.constrained_stage_dofs()
    b[cd] = 0.0
    x0[cd] = 0.0
    bd = torch.from_numpy(b).cuda()
    xs = [torch.from_numpy(x0.copy()).cuda() for _ in plans]
    ref = torch.from_numpy(x0.copy()).cuda()
    grp = PeerLoopback(shards, xs)
    for _ in range(3):
        grp.sweep(xs, bd)
        ref = apply_vanka(full, S, ref, bd, omega=0.5, weights="pou")
    got = ref.clone()
    for p, x in zip(plans, xs):
        idx = torch.from_numpy(p.dofs).cuda()
        got[idx] = x[idx]
    assert rel(got.cpu().numpy(), ref.cpu().numpy()) <= 1e-12
    for p, x in zip(plans, xs):
        for q, s in p.shared.items():
            idx = torch.from_numpy(s).cuda()
            assert torch.equal(x[idx], xs[q][idx])


def test_peer_holders_cover_every_contribution():
    """CPU: the fused kernel's holder lists name, for every own DoF, exactly
    the ranks whose patches contain it, ascending; summed over ranks the
    holder counts reproduce the global patch multiplicity's support."""
    from paper_2202_07381_b200.patches import build_patch_tables
    from paper_2202_07381_b200.shard import StripPartition, peer_holders, shard_plans
    disc, tab, conv, case, S, mesh = _problem("s3")
    plans = shard_plans(S, mesh, StripPartition(mesh, 3))
    t = build_patch_tables(mesh, S.n_nodes, S.n_p, S.r, S.node_constrained)
    part = StripPartition(mesh, 3).part
    owner_of_entry = np.repeat(part[t.order], t.sizes)
    for p in plans:
        ptr, ranks = peer_holders(p)
        assert len(ptr) == len(p.dofs) + 1
        for i in range(0, len(p.dofs), 97):
            d = p.dofs[i]
            expect = np.unique(owner_of_entry[t.idx == d])
            got = ranks[ptr[i]:ptr[i + 1]]
            assert np.array_equal(got, expect) and p.rank in got
