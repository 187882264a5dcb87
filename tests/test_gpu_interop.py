"""Object-level drop-in: reference-shaped objects handed
to the device path.

The reference package cannot travel to the GPU box, so its objects are
stood in for by duck-typed namespaces carrying exactly the attributes the
reference defines (stages.py:63-88: ``blocks.M/K/B`` vector CSR, ``tableau``,
``dt``, ``constrained``, ``convection``; solvers.py:295-300: ``MGLevel``
fields with a scipy ``prolong``), built from the same host setup."""

from types import SimpleNamespace

import numpy as np
import pytest

from harness import load_golden, oracle_levels, oracle_mg, rel, setup

pytestmark = pytest.mark.gpu


def _ref_system(disc, tab, dt, k, conv=None):
    blk = disc.blocks[k]
    ns = SimpleNamespace(blocks=SimpleNamespace(M=blk.M, K=blk.K, B=blk.B), tableau=tab, dt=dt,
                         constrained=np.asarray(disc.cdofs[k]), convection=None)
    if conv is not None:
        from oracle.irk_vanka_oracle import OracleStageOperator
        op = OracleStageOperator(blk.M, blk.K, blk.B, tab.A, dt, disc.cdofs[k],
                                 convection=[J.matrix for J in conv[k]])
        ns.convection = op.convection            # the reference stores them eliminated
    return ns


@pytest.mark.parametrize("name", ["cfg1", "ns"])
def test_gpu_stage_wraps_reference_system(name):
    from paper_2202_07381_b200.interop import GpuStage
    disc, tab, conv, case = setup(name)
    g, _ = load_golden(name)
    k = disc.num_levels - 1
    S = GpuStage(_ref_system(disc, tab, case["dt"], k, conv))
    lv = oracle_levels(disc, tab, case["dt"], conv, levels=[k])[0]
    y = S.matvec(g["x_rand"])
    assert rel(y, lv["op"].matvec(g["x_rand"])) <= 1e-13
    assert rel(y, g["matvec_xr"]) <= 1e-13


def test_scipy_prolong_levels_match_native_transfers():
    """MGLevel.prolong given as the reference's scipy stage CSR."""
    import torch
    from paper_2202_07381_b200 import MGHierarchyOp, MGLevel, SmootherSpec
    disc, tab, conv, case = setup("cfg1")
    g, _ = load_golden("cfg1")
    sm = SmootherSpec(pre=2, post=2, accel="chebyshev", cheby_a=2.0, cheby_b=8.0)
    mg, S = disc.build_mg(tab, case["dt"], sm)
    mg_sp = MGHierarchyOp([MGLevel(l.system, l.patches, l.smoother,
                                   None if l.prolong is None else l.prolong.matrix)
                           for l in mg.levels], mg.coarse)
    b = torch.from_numpy(g["b"]).cuda()
    z0 = mg.precondition(b).cpu().numpy()
    z1 = mg_sp.precondition(b).cpu().numpy()
    assert rel(z1, z0) <= 1e-14
    zo = oracle_mg(oracle_levels(disc, tab, case["dt"], None), case, "cheb").precondition(
        g["b"].copy())
    assert rel(z1, zo) <= 1e-12
    with pytest.raises(ValueError):
        MGHierarchyOp([mg.levels[0], MGLevel(S, mg.levels[-1].patches, sm,
                                             mg.levels[1].prolong.matrix)], mg.coarse)


def test_from_reference_hierarchy():
    """A reference-shaped MGHierarchyOp (duck-typed levels, scipy prolongs)
    rebuilt on the device: V-cycle and FGMRES against the oracle/golden."""
    from paper_2202_07381_b200 import fgmres
    from paper_2202_07381_b200.interop import from_reference_hierarchy
    disc, tab, conv, case = setup("cfg1")
    g, meta = load_golden("cfg1")
    spec = SimpleNamespace(pre=2, post=2, accel="chebyshev", cheby_a=2.0, cheby_b=8.0,
                           omega=1.0)
    levels = []
    for k in range(disc.num_levels):
        levels.append(SimpleNamespace(
            system=_ref_system(disc, tab, case["dt"], k), patches=SimpleNamespace(omega=1.0),
            smoother=spec, prolong=disc.stage_prolong(k, tab.r).matrix if k else None))
    mg = from_reference_hierarchy(SimpleNamespace(levels=levels), disc.hier.levels)
    zo = oracle_mg(oracle_levels(disc, tab, case["dt"], None), case, "cheb").precondition(
        g["b"].copy())
    z = mg.precondition(g["b"])
    assert isinstance(z, np.ndarray)
    assert rel(z, zo) <= 1e-12
    assert rel(z, g["precond_cheb"]) <= 1e-12
    S = mg.levels[-1].system
    _, st = fgmres(S.matvec, g["b"], precond=mg.precondition, rtol=1e-8, maxiter=200, restart=50)
    assert st.converged and abs(st.iterations - meta["fgmres_its_cheb"]) <= 1
