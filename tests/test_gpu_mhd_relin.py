"""Device re-linearisation of the MHD operator (K10g, ``ivk_mhd_assemble``;
the Newton-cadence update of BASELINE config 5): the device L at a new
frozen state against the host assembly (mhd.assemble_mhd, itself pinned to
the oracle's cell loop in test_mhd_setup.py), and a whole re-linearised
hierarchy (every level's L, K7g patch refactorisation, coarse solve)
against one built from scratch on the host at that state."""

import numpy as np
import pytest

from harness import mhd_setup, rel

pytestmark = pytest.mark.gpu


def _state(disc, seed, amp=0.2):
    from paper_2202_07381_b200.fem import p2_node_coords
    from paper_2202_07381_b200.discretization import streamfunction_velocity
    from paper_2202_07381_b200.mhd import mhd_magnetic_state
    xy = p2_node_coords(disc.fine_mesh)
    rng = np.random.default_rng(seed)
    # smooth fields plus a perturbation: a plausible Newton iterate
    u = 0.7 * streamfunction_velocity(xy) + amp * rng.uniform(-1, 1, xy.shape)
    B = mhd_magnetic_state(xy) + amp * rng.uniform(-1, 1, xy.shape)
    return u, B


def _prefix_funcs(u, B):
    return (lambda xy: u[:len(xy)]), (lambda xy: B[:len(xy)])


@pytest.mark.parametrize("name", ["mhd16", "mhd32"])
def test_device_operator_matches_host(name):
    import torch
    from paper_2202_07381_b200.mhd import MHDAssembler, assemble_mhd
    disc, tab, case = mhd_setup(name)
    u, B = _state(disc, 5)
    for k in range(disc.num_levels):
        mesh = disc.hier.levels[k]
        S = disc.system(k, tab, case["dt"])
        n = S.n_nodes
        asm = MHDAssembler(mesh, disc.params, S)
        asm.assemble_into_system(S, torch.from_numpy(u).cuda(), torch.from_numpy(B).cuda())
        dev = S.device_data()["tensors"]
        l_dev = dev["ml"][:, 1].cpu().numpy()
        _, _, m_h, l_h, _ = assemble_mhd(mesh, disc.params, *_prefix_funcs(u[:n], B[:n]))
        assert np.max(np.abs(l_dev - l_h)) <= 1e-13 * np.max(np.abs(l_h))
        assert np.array_equal(dev["ml"][:, 0].cpu().numpy(), m_h)   # mass untouched
        # the SELL copy carries the same values: K1g against the host matrix
        S.download_operator()
        x = np.random.default_rng(k).uniform(-1, 1, S.dim)
        y = S.matvec(torch.from_numpy(x).cuda()).cpu().numpy()
        assert rel(y, S.materialize() @ x) <= 1e-13


@pytest.mark.parametrize("mode", ["kron", "full"])
def test_relinearized_hierarchy_matches_fresh_build(mode):
    import torch
    from paper_2202_07381_b200 import SmootherSpec, fgmres
    from paper_2202_07381_b200.mhd import MHDDiscretization
    disc, tab, case = mhd_setup("mhd32")
    sm = SmootherSpec(pre=2, post=2, accel="chebyshev", cheby_a=2.0, cheby_b=8.0)
    mg, S = disc.build_mg(tab, case["dt"], sm, patch_mode=mode)
    u, B = _state(disc, 9, amp=0.02)
    disc.relinearize(mg, torch.from_numpy(u).cuda(), torch.from_numpy(B).cuda())
    fresh = MHDDiscretization(case["n0"], case["level"], disc.params,
                              u0_func=_prefix_funcs(u, B)[0], B0_func=_prefix_funcs(u, B)[1])
    mg2, S2 = fresh.build_mg(tab, case["dt"], sm, patch_mode=mode)
    rng = np.random.default_rng(2)
    b = torch.from_numpy(rng.uniform(-1, 1, S.dim)).cuda()
    b[torch.from_numpy(S.constrained_stage_dofs()).cuda()] = 0.0
    S.project_pressure_means(b)          # consistent with the pressure null space
    assert rel(S.matvec(b).cpu().numpy(), S2.matvec(b).cpu().numpy()) <= 1e-13
    v1 = mg.precondition(b).cpu().numpy()
    v2 = mg2.precondition(b).cpu().numpy()
    assert rel(v1, v2) <= 1e-10
    x1, st1 = fgmres(S.matvec, b, precond=mg.precondition, rtol=1e-8, maxiter=200)
    x2, st2 = fgmres(S2.matvec, b, precond=mg2.precondition, rtol=1e-8, maxiter=200)
    n = min(len(st1.residual_norms), len(st2.residual_norms))
    h1, h2 = np.array(st1.residual_norms[:n]), np.array(st2.residual_norms[:n])
    assert np.all(np.abs(h1 - h2) <= 1e-6 * h1[0])
    assert st1.converged and abs(st1.iterations - st2.iterations) <= 1

