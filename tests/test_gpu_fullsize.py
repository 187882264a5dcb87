"""Full BASELINE-size checks on the GPU (configs 2 and 3), through the C ABI.

At full size the oracle cannot run every patch in seconds, so parity is
checked through size-independent properties and sampled oracles:
  * fine-level patch indices bit-exact (sha256 of the reference's own
    ``patch_indices`` at full size, tests/golden/full_counts.json);
  * FGMRES iteration counts within +-1 of the reference's (both smoothers),
    final relative residual <= 1e-8;
  * a sampled sweep: at 48 random DoFs the device sweep equals
    x + w * sum_{p owns d} (A_p^-1 r_p)_d computed by the oracle with
    np.linalg.inv on exactly those owning patches (rel <= 1e-12);
  * fixed point at an exact solution, linearity and bitwise determinism of
    the patch solve, and agreement of the two patch formulations.
"""

import hashlib
import json
import os

import numpy as np
import pytest

from harness import GOLDEN, setup

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

with open(os.path.join(GOLDEN, "full_counts.json")) as fh:
    FULL = json.load(fh)

_cache = {}


def build(name):
    if name in _cache:
        return _cache[name]
    _cache.clear()
    import torch
    from paper_2202_07381_b200 import MGHierarchyOp, MGLevel, SmootherSpec
    disc, tab, conv, case = setup(name)
    cheb = SmootherSpec(pre=2, post=2, accel="chebyshev", cheby_a=case["cheby_a"], cheby_b=8.0)
    mg, S = disc.build_mg(tab, case["dt"], cheb, convection=conv, use_graph=True)
    pou = SmootherSpec(pre=2, post=2, accel="richardson", omega=0.5, weighting="pou")
    mg_pou = MGHierarchyOp([MGLevel(l.system, l.patches, pou, l.prolong) for l in mg.levels],
                           mg.coarse, use_graph=True)
    b = np.random.default_rng(case["seed"]).uniform(-1.0, 1.0, S.dim)
    b[S.constrained_stage_dofs()] = 0.0
    S.project_pressure_means(b)
    _cache[name] = (disc, tab, conv, case, mg, mg_pou, S, torch.from_numpy(b).cuda())
    return _cache[name]


@pytest.fixture(params=["cfg2", "cfg3"])
def full(request):
    return build(request.param), request.param


def test_fine_patch_indices_bit_exact(full):
    (disc, tab, conv, case, mg, mg_pou, S, b), name = full
    t = mg.levels[-1].patches.tables
    pos = t.patch_of_vertex()
    hh = hashlib.sha256()
    for v in range(t.num_patches):
        q = pos[v]
        hh.update(t.idx[t.idx_off[q]:t.idx_off[q + 1]].astype(np.int64).tobytes())
        hh.update(b"|")
    assert hh.hexdigest() == FULL[name]["patch_index_sha256_fine"]
    assert S.dim == FULL[name]["dim"]


@pytest.mark.parametrize("smoother", ["cheb", "pou"])
def test_fgmres_counts_full_size(full, smoother):
    from paper_2202_07381_b200 import fgmres
    (disc, tab, conv, case, mg, mg_pou, S, b), name = full
    h = mg if smoother == "cheb" else mg_pou
    _, st = fgmres(S.matvec, b, precond=h.precondition, rtol=1e-8, maxiter=200, restart=50)
    assert st.converged and st.relative_residual <= 1e-8
    assert abs(st.iterations - FULL[name][f"fgmres_its_{smoother}"]) <= 1


def test_sampled_sweep_against_oracle(full):
    """Oracle patch solves (np.linalg.inv) on the patches owning 48 random DoFs."""
    import torch
    from oracle.irk_vanka_oracle import OraclePatches, OracleStageOperator
    from paper_2202_07381_b200 import apply_vanka
    (disc, tab, conv, case, mg, mg_pou, S, b), name = full
    k = disc.num_levels - 1
    cm = None if conv is None else [J.matrix for J in conv[k]]
    op = OracleStageOperator(disc.blocks[k].M, disc.blocks[k].K, disc.blocks[k].B, tab.A,
                             case["dt"], disc.cdofs[k], convection=cm)
    pat = mg.levels[-1].patches
    t = pat.tables
    rng = np.random.default_rng(7)
    x = rng.uniform(-1.0, 1.0, S.dim)
    x[S.constrained_stage_dofs()] = 0.0
    bh = b.cpu().numpy()
    got = apply_vanka(pat, S, torch.from_numpy(x).cuda(), b, omega=0.5).cpu().numpy()
    r = bh - op.matvec(x)
    free = np.flatnonzero(t.multiplicity > 0)
    dofs = np.sort(rng.choice(free, 48, replace=False))
    owners = set()
    for d in dofs:
        for pos in t.dof_pos[t.dof_ptr[d]:t.dof_ptr[d + 1]]:
            owners.add(int(t.order[np.searchsorted(t.idx_off, pos, side="right") - 1]))
    owners = sorted(owners)
    idxs = {v: t.idx[t.idx_off[q]:t.idx_off[q + 1]] for v, q in
            zip(owners, t.patch_of_vertex()[owners])}
    vels = {}
    for v in owners:
        ix = idxs[v]
        n_u, sd = S.n_u, S.stage_dim
        vels[v] = ix[(ix < sd) & (ix < n_u)]
    z = np.zeros(S.dim)
    for v in owners:
        mats = OraclePatches.patch_matrices(op, [vels[v]], [v])
        z[idxs[v]] += np.linalg.inv(mats[0]) @ r[idxs[v]]
    ref = x[dofs] + 0.5 * z[dofs]
    assert np.linalg.norm(got[dofs] - ref) <= 1e-12 * np.linalg.norm(ref)


def test_fixed_point_linearity_determinism(full):
    import torch
    from paper_2202_07381_b200 import apply_vanka
    (disc, tab, conv, case, mg, mg_pou, S, b), name = full
    pat = mg.levels[-1].patches
    xs = torch.from_numpy(np.random.default_rng(3).uniform(-1, 1, S.dim)).cuda()
    bs = S.matvec(xs)
    y = apply_vanka(pat, S, xs, bs, omega=1.0)
    assert float((y - xs).abs().max()) <= 1e-12 * float(xs.abs().max())
    r1 = b
    r2 = torch.roll(b, 12345)
    z1 = pat.solve_additive(r1)
    z2 = pat.solve_additive(r2)
    z12 = pat.solve_additive(2.0 * r1 - 3.0 * r2)
    assert float(torch.linalg.vector_norm(z12 - (2.0 * z1 - 3.0 * z2))) <= \
        1e-13 * float(torch.linalg.vector_norm(z12))
    assert torch.equal(pat.solve_additive(r1), z1)
    p1 = mg.precondition(b)
    p2 = mg.precondition(b)
    assert torch.equal(p1, p2)


def test_patch_formulations_agree(full):
    import torch
    from paper_2202_07381_b200 import VankaPatchSet, apply_vanka
    (disc, tab, conv, case, mg, mg_pou, S, b), name = full
    kron = mg.levels[-1].patches
    assert kron.mode == ("kron" if conv is not None else "dedup")
    x0 = torch.zeros_like(b)
    yk = apply_vanka(kron, S, x0, b, omega=0.5, weights="pou")
    for mode in (["full"] if conv is not None else ["full", "kron", "kron-sym", "modal"]):
        other = VankaPatchSet(S, disc.fine_mesh, mode=mode)
        yo = apply_vanka(other, S, x0, b, omega=0.5, weights="pou")
        del other
        torch.cuda.empty_cache()
        assert float(torch.linalg.vector_norm(yk - yo)) <= \
            1e-12 * float(torch.linalg.vector_norm(yo)), mode
