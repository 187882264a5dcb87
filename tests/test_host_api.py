"""The reference-compatible numpy entry points of FGMRES and the Chebyshev
driver (mirroring test_solvers.py of the reference; they run on the device
-- numpy in, numpy out -- so those tests are GPU tests), SmootherSpec
validation, the no-fallback contract, and the replica/timing plumbing of
bench.py under a 2-rank gloo process group (CPU)."""

import os
import socket

import numpy as np
import pytest

from paper_2202_07381_b200 import SmootherSpec, chebyshev_smooth, fgmres


@pytest.mark.gpu
def test_fgmres_small_dense_exact():
    rng = np.random.default_rng(5)
    A = rng.standard_normal((5, 5)) + 5 * np.eye(5)
    b = rng.standard_normal(5)
    x, st = fgmres(lambda v: A @ v, b, rtol=1e-12, maxiter=10)
    assert st.converged and st.iterations <= 5
    assert np.linalg.norm(A @ x - b) < 1e-10


@pytest.mark.gpu
def test_fgmres_identity_one_iteration():
    b = np.arange(1.0, 6.0)
    x, st = fgmres(lambda v: v, b, rtol=1e-12)
    assert st.iterations == 1 and np.allclose(x, b)


@pytest.mark.gpu
def test_fgmres_monotone_and_restart():
    rng = np.random.default_rng(6)
    A = rng.standard_normal((40, 40)) + 8 * np.eye(40)
    b = rng.standard_normal(40)
    _, st = fgmres(lambda v: A @ v, b, rtol=1e-10, restart=10, maxiter=60)
    assert st.iterations == 60 and st.relative_residual < 1e-8
    assert np.all(np.diff(st.residual_norms) <= 1e-12)


@pytest.mark.gpu
def test_fgmres_absolute_tolerance_and_flexible():
    rng = np.random.default_rng(8)
    A = rng.standard_normal((30, 30)) + 10 * np.eye(30)
    b = rng.standard_normal(30)
    state = {"k": 0}

    def precond(v):
        state["k"] += 1
        return v / (1.0 + 0.1 * (state["k"] % 3))

    x, st = fgmres(lambda v: A @ v, b, precond=precond, rtol=0.0, atol=1e-9, maxiter=60,
                   restart=15)
    assert st.converged and st.final_residual <= 1e-9


@pytest.mark.gpu
def test_fgmres_matches_oracle_history():
    from oracle.irk_vanka_oracle import oracle_fgmres
    rng = np.random.default_rng(9)
    A = rng.standard_normal((60, 60)) + 6 * np.eye(60)
    b = rng.standard_normal(60)
    x1, st = fgmres(lambda v: A @ v, b, rtol=1e-10, restart=7, maxiter=80)
    x2, (its, norms, ok) = oracle_fgmres(lambda v: A @ v, b, rtol=1e-10, restart=7, maxiter=80)
    assert st.iterations == its
    assert np.linalg.norm(x1 - x2) <= 1e-12 * np.linalg.norm(x2)
    assert np.allclose(st.residual_norms, norms, rtol=1e-9, atol=0)


def test_numpy_entry_points_have_no_cpu_fallback():
    """Without a CUDA device the numpy entry points raise instead of running
    the reference's algorithm on the host."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("needs a host without a CUDA device")
    from paper_2202_07381_b200 import IvkError
    A = np.eye(4) * 2.0
    with pytest.raises(IvkError):
        fgmres(lambda v: A @ v, np.ones(4))
    with pytest.raises(IvkError):
        chebyshev_smooth(lambda v: A @ v, lambda v: v, 2.0, 8.0, 2, np.zeros(4), np.ones(4))


@pytest.mark.gpu
def test_chebyshev_polynomial_oracle():
    lams = np.linspace(2.0, 8.0, 7)
    rng = np.random.default_rng(3)
    x0 = rng.standard_normal(7)
    xs = rng.standard_normal(7)
    for k in (1, 2, 3, 4):
        xk = chebyshev_smooth(lambda v: lams * v, lambda v: v, 2.0, 8.0, k, x0.copy(), lams * xs)
        arg = (5.0 - lams) / 3.0
        poly = np.cos(k * np.arccos(np.clip(arg, -1, 1))) / np.cosh(k * np.arccosh(5.0 / 3.0))
        assert np.max(np.abs(xk - (xs + poly * (x0 - xs)))) < 1e-12


def test_smoother_spec_validation():
    for bad in (dict(accel="jacobi"), dict(cheby_a=5.0, cheby_b=2.0), dict(pre=-1),
                dict(weighting="lumped")):
        with pytest.raises(ValueError):
            SmootherSpec(**bad)
    SmootherSpec(accel="richardson", omega=0.5, weighting="pou")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _replica_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import bench
    from harness import oracle_levels, setup
    from oracle.irk_vanka_oracle import oracle_apply_vanka, random_rhs
    r, w, _ = bench.dist_init()
    disc, tab, conv, case = setup("crossed")
    lv = oracle_levels(disc, tab, case["dt"], None, levels=[disc.num_levels - 1])[0]
    b = random_rhs(lv["op"], case["seed"])
    y = oracle_apply_vanka(lv["patches"], lv["op"], np.zeros(lv["op"].dim), b, 0.5)
    t = bench.max_over_ranks(float(rank + 1), w)
    bench.barrier(w)
    q.put((r, w, t, float(np.linalg.norm(y))))
    dist.destroy_process_group()


def test_replicas_two_ranks_gloo():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_replica_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[0] for r in res] == [0, 1]
    assert all(r[1] == 2 for r in res)
    assert all(r[2] == 2.0 for r in res)          # max over ranks
    assert res[0][3] == res[1][3]                # replicas agree bitwise


def test_patch_mode_validation_on_host():
    """Formulation choices are validated before any device work (CPU): the
    modal split needs a convection-free Taylor-Hood operator, kron-sym / dedup
    a symmetric translation-invariant one, general operators run kron / full."""
    from paper_2202_07381_b200 import VankaPatchSet, tableau_lookup
    from paper_2202_07381_b200.mhd import MHDDiscretization
    from harness import setup
    disc, tab, conv, case = setup("ns")
    from paper_2202_07381_b200.stages import assemble_stage_operator
    S = assemble_stage_operator(disc.blocks[-1], tab, case["dt"], constrained=disc.cdofs[-1],
                                convection=conv[-1])
    for mode in ("modal", "kron-sym", "dedup", "bogus"):
        with pytest.raises(ValueError):
            VankaPatchSet(S, disc.fine_mesh, mode=mode, factor=False)
    md = MHDDiscretization(4, 1)
    G = md.system(1, tableau_lookup("radauiia", 2), 0.01)
    for mode in ("modal", "kron-sym", "dedup"):
        with pytest.raises(ValueError):
            VankaPatchSet(G, md.fine_mesh, mode=mode, factor=False)


def _run_bench(*args, timeout=600):
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    env["CUDA_VISIBLE_DEVICES"] = ""   # CPU ranks (gloo) in this test
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), *args],
                         capture_output=True, text=True, timeout=timeout, env=env, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    return lines


def test_bench_launcher_spawns_ranks_gloo():
    """bench.py --gpus 2 without a torchrun environment re-launches itself as
    two ranks (torch.distributed.run, 127.0.0.1); the ranks all-reduce and
    rank 0 alone prints."""
    lines = _run_bench("--gpus", "2", "--impl", "probe")
    assert len(lines) == 1
    assert lines[0]["n_gpus"] == 2 and lines[0]["max_over_ranks"] == 2.0


def test_bench_reference_arm_two_ranks_gloo():
    """The reference arm under the 2-rank launch: rank 0 times the CPU
    oracle over every patch (no extrapolation), the other rank exits."""
    lines = _run_bench("--gpus", "2", "--impl", "reference", "--config", "cfg1", "--steps", "2",
                       "--warmup", "1", "--no-cpu-cycles")
    assert len(lines) == 1
    ln = lines[0]
    assert ln["impl"] == "reference" and ln["n_gpus"] == 2 and ln["value"] > 0
    assert "all 1089 patch solves" in ln["cpu_baseline"]["sample"]
    assert ln["e2e"]["h2d_bytes_per_step"] == 0
