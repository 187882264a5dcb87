"""Guard-band checks of the device kernels (the stand-in for compute-sanitizer,
which is closed on this GPU pool: profiles/r02/sanitizer_closed_on_pool.log).

Every vector a kernel reads or writes is carved out of a larger buffer whose
surroundings hold NaN sentinels, so
  * an out-of-bounds WRITE to a neighbouring element changes a guard word
    (checked bit for bit), and
  * an out-of-bounds READ of a neighbouring element that reaches the result
    poisons it with NaN -- the result must be finite and bitwise equal to the
    run on plain, unguarded buffers.
The inverse / record store and the patch-local scratch get the same guards
(the K3 kernels stream them with wide vector loads; K3m reads whole records
by TMA bulk copies).  Covered: K1, K3 full / kron / kron-sym
/ dedup / modal, K4, the fused sweep, K5, K6 (dense and tile-LU), K7 / K7e /
K7m (factorisation writes into a guarded store), K8, K9 and the V-cycle.
"""

import numpy as np
import pytest

from harness import setup

pytestmark = pytest.mark.gpu

GUARD = 2048


def guarded(n, fill=None, dtype=None):
    """(whole buffer, view of n elements in its middle), guards = NaN."""
    import torch
    dtype = dtype or torch.float64
    whole = torch.full((n + 2 * GUARD,), float("nan"), dtype=dtype, device="cuda")
    view = whole[GUARD:GUARD + n]
    if fill is not None:
        view.copy_(fill)
    return whole, view


def guards_intact(whole, n):
    import torch
    a = whole[:GUARD].view(torch.int64)
    b = whole[GUARD + n:].view(torch.int64)
    ref = torch.full((1,), float("nan"), dtype=torch.float64, device="cuda").view(torch.int64)
    return bool((a == ref).all()) and bool((b == ref).all())


def same_bits(a, b):
    import torch
    return bool((a.contiguous().view(torch.int64) == b.contiguous().view(torch.int64)).all())


def build(name, mode):
    from paper_2202_07381_b200 import SmootherSpec
    disc, tab, conv, case = setup(name)
    sm = SmootherSpec(pre=2, post=2, accel="chebyshev", cheby_a=case["cheby_a"], cheby_b=8.0)
    mg, S = disc.build_mg(tab, case["dt"], sm, convection=conv, patch_mode=mode)
    return disc, tab, case, mg, S


CASES = [("crossed", "full"), ("crossed", "modal"), ("crossed", "kron"), ("s3", "modal"),
         ("s3", "dedup"), ("s3", "kron-sym"), ("s3", "kron"), ("ns", "kron"), ("ns", "full")]


@pytest.mark.parametrize("name,mode", CASES, ids=[f"{n}-{m}" for n, m in CASES])
def test_sweep_kernels_stay_in_bounds(name, mode):
    import torch
    from paper_2202_07381_b200 import apply_vanka
    disc, tab, case, mg, S = build(name, mode)
    pat = mg.levels[-1].patches
    dim = S.dim
    rng = np.random.default_rng(case["seed"])
    x0 = torch.from_numpy(rng.uniform(-1, 1, dim)).cuda()
    b0 = torch.from_numpy(rng.uniform(-1, 1, dim)).cuda()

    # plain run (reference bits)
    r_ref = torch.empty_like(x0)
    S.apply_into(x0, b0, r_ref)
    loc_ref = pat.apply_local(r_ref).clone()
    z_ref = torch.empty_like(x0)
    pat.combine(loc_ref, x0, 1.0, 0.5, pat.weights("pou"), z_ref)
    y_ref = apply_vanka(pat, S, x0, b0, omega=0.5, weights="pou")
    assert torch.isfinite(y_ref).all()

    # guarded vectors
    xw, x = guarded(dim, x0)
    bw, b = guarded(dim, b0)
    rw, r = guarded(dim)
    S.apply_into(x, b, r)                                   # K1
    assert guards_intact(rw, dim) and guards_intact(xw, dim) and guards_intact(bw, dim)
    assert same_bits(r, r_ref)

    nloc = loc_ref.numel()
    lw, loc = guarded(nloc, torch.zeros(nloc, dtype=torch.float64, device="cuda"))
    loc_ref = pat.apply_local(r_ref, local=torch.zeros_like(loc)).clone()   # (pad slots stay 0)
    pat.apply_local(r, local=loc)                           # K2 + K3
    assert guards_intact(lw, nloc) and guards_intact(rw, dim)
    assert same_bits(loc, loc_ref)

    zw, z = guarded(dim)
    pat.combine(loc, x, 1.0, 0.5, pat.weights("pou"), z)    # K4
    assert guards_intact(zw, dim) and guards_intact(lw, nloc) and guards_intact(xw, dim)
    assert same_bits(z, z_ref)

    yw, y = guarded(dim)                                    # fused sweep, guarded scratch
    r2w, r2 = guarded(dim)
    l2w, l2 = guarded(nloc, torch.zeros(nloc, dtype=torch.float64, device="cuda"))
    apply_vanka(pat, S, x, b, omega=0.5, weights="pou", workspace={"r": r2, "local": l2}, out=y)
    for w, n in ((yw, dim), (r2w, dim), (l2w, nloc), (xw, dim), (bw, dim)):
        assert guards_intact(w, n)
    assert same_bits(y, y_ref)


@pytest.mark.parametrize("name,mode", [("crossed", "full"), ("crossed", "modal"), ("s3", "kron"),
                                       ("s3", "modal"), ("ns", "kron"), ("ns", "full")],
                         ids=lambda v: str(v))
def test_factorisation_stays_inside_the_store(name, mode):
    """K7 / K7e / K7m write their inverses / records into a store whose
    surroundings are NaN guards; the refactorised store equals the first one."""
    import torch
    disc, tab, case, mg, S = build(name, mode)
    pat = mg.levels[-1].patches
    dev = pat.device_data()
    inv0 = dev["inv"]
    n = inv0.numel()
    want = inv0.clone()
    whole, view = guarded(n)
    view.zero_()
    # point the descriptor at the guarded store and refactorise in place
    desc = dev["desc"]
    old = desc.inv
    desc.inv = view.data_ptr()
    dev["inv"] = view
    try:
        pat.factor()
        torch.cuda.synchronize()
        assert guards_intact(whole, n)
        assert same_bits(view, want)
        # and the apply reads only the store
        rng = np.random.default_rng(1)
        r = torch.from_numpy(rng.uniform(-1, 1, S.dim)).cuda()
        a = pat.apply_local(r).clone()
        assert torch.isfinite(a).all()
    finally:
        desc.inv = old
        dev["inv"] = inv0
    b = pat.apply_local(r).clone()
    assert same_bits(a, b)


@pytest.mark.parametrize("name", ["crossed", "s3", "ns"])
def test_cycle_kernels_stay_in_bounds(name):
    """K5 restrict / prolong, K6 coarse solve (both methods), K8 projection /
    constrained seeding and the whole V-cycle on guarded vectors."""
    import torch
    from paper_2202_07381_b200.solvers import CoarseSolver
    disc, tab, case, mg, S = build(name, "auto")
    rng = np.random.default_rng(case["seed"] + 1)
    fine, coarse = mg.levels[-1], mg.levels[-2]
    nf, nc = fine.system.dim, coarse.system.dim
    rf0 = torch.from_numpy(rng.uniform(-1, 1, nf)).cuda()
    ec0 = torch.from_numpy(rng.uniform(-1, 1, nc)).cuda()
    P = fine.prolong

    rc_ref = torch.empty(nc, dtype=torch.float64, device="cuda")
    P.restrict_into(rf0, rc_ref)
    rfw, rf = guarded(nf, rf0)
    rcw, rc = guarded(nc)
    P.restrict_into(rf, rc)                                 # K5 restrict
    assert guards_intact(rcw, nc) and guards_intact(rfw, nf) and same_bits(rc, rc_ref)

    xf_ref = rf0.clone()
    P.prolong_add(ec0, xf_ref)
    ecw, ec = guarded(nc, ec0)
    xfw, xf = guarded(nf, rf0)
    P.prolong_add(ec, xf)                                   # K5 prolong
    assert guards_intact(xfw, nf) and guards_intact(ecw, nc) and same_bits(xf, xf_ref)

    s0 = mg.levels[0].system
    n0 = s0.dim
    b00 = torch.from_numpy(rng.uniform(-1, 1, n0)).cuda()
    for method in ("dense", "lu"):                          # K6
        cs = CoarseSolver(s0, method)
        ref = torch.empty(n0, dtype=torch.float64, device="cuda")
        cs.solve_into(b00, ref)
        bw, b = guarded(n0, b00)
        xw, x = guarded(n0)
        cs.solve_into(b, x)
        assert guards_intact(xw, n0) and guards_intact(bw, n0)
        assert torch.isfinite(x).all() and same_bits(x, ref)

    z_ref = mg.precondition(rf0)                            # V-cycle (K1-K8)
    zw, z = guarded(nf)
    mg.precondition_to(rf, z)
    assert guards_intact(zw, nf) and guards_intact(rfw, nf)
    assert torch.isfinite(z).all() and same_bits(z, z_ref)


def test_krylov_kernels_stay_in_bounds():
    """K9: dot / norm / MGS / lincomb on guarded vectors through FGMRES."""
    import torch
    from paper_2202_07381_b200 import fgmres
    disc, tab, case, mg, S = build("crossed", "auto")
    rng = np.random.default_rng(3)
    b0 = torch.from_numpy(rng.uniform(-1, 1, S.dim)).cuda()
    x_ref, st_ref = fgmres(S.matvec, b0, precond=mg.precondition, rtol=1e-8, maxiter=60)
    bw, b = guarded(S.dim, b0)
    x, st = fgmres(S.matvec, b, precond=mg.precondition, rtol=1e-8, maxiter=60)
    assert guards_intact(bw, S.dim)
    assert st.iterations == st_ref.iterations and torch.isfinite(x).all()
    assert same_bits(x, x_ref)
