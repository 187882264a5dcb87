"""GPU parity: the sm_100a path (through libivk's C ABI) against the CPU
oracle on identical seeded inputs, and against the reference goldens.

Gates (BASELINE.json north_star):
  * K1 operator apply: rel l2 <= 1e-13
  * one relaxation sweep (W = I and PoU, from 0 and from a random x): <= 1e-12
  * V-cycle (mg.precondition): the F9 decomposed protocol everywhere --
    down-leg intermediates <= 1e-12, up-leg with the oracle's coarse output
    injected <= 1e-12, coarse backward error no worse than SuperLU's own
    (x10) -- and end to end <= 1e-12 where the coarse solve is well
    conditioned (cfg1, ns, crossed), else <= 10x the reference's self-floor
    (oracle vs oracle with reversed reduction order, measured in the test;
    ~5e-10 on the RadauIIA(3) case s3)
  * FGMRES iteration counts within +-1 of the reference's
"""

import numpy as np
import pytest

from harness import load_golden, oracle_levels, oracle_mg, rel, setup
from oracle.irk_vanka_oracle import oracle_apply_vanka, oracle_fgmres

pytestmark = pytest.mark.gpu

CASES = ["cfg1", "s3", "ns", "crossed"]
WELL_CONDITIONED = {"cfg1", "ns", "crossed"}


class Case:
    def __init__(self, name, mode):
        import torch
        from paper_2202_07381_b200 import MGHierarchyOp, MGLevel, SmootherSpec
        self.name = name
        self.golden, self.meta = load_golden(name)
        self.disc, self.tab, self.conv, self.case = setup(name)
        c = self.case
        cheb = SmootherSpec(pre=2, post=2, accel="chebyshev", cheby_a=c["cheby_a"], cheby_b=8.0)
        self.mode = mode
        self.mg, self.S = self.disc.build_mg(self.tab, c["dt"], cheb, convection=self.conv,
                                             patch_mode=mode)
        expect = mode if mode != "auto" else \
            ("kron" if c["conv"] else "modal" if name == "crossed" else "dedup")
        assert self.mg.levels[-1].patches.mode == expect
        pou = SmootherSpec(pre=2, post=2, accel="richardson", omega=0.5, weighting="pou")
        self.mg_pou = MGHierarchyOp([MGLevel(l.system, l.patches, pou, l.prolong)
                                     for l in self.mg.levels], self.mg.coarse)
        self.oracle = oracle_levels(self.disc, self.tab, c["dt"], self.conv)
        self.dev = torch.device("cuda")


_cache = {}


@pytest.fixture(params=[(n, m) for n in CASES
                        for m in ("auto", "kron-sym", "dedup", "full", "modal")],
                ids=lambda p: f"{p[0]}-{p[1]}")
def case(request):
    if request.param in (("ns", "kron-sym"), ("ns", "dedup"), ("ns", "modal")):
        pytest.skip("kron-sym / dedup / modal need a convection-free operator")
    if request.param not in _cache:
        _cache.clear()   # one case resident at a time
        _cache[request.param] = Case(*request.param)
    return _cache[request.param]


def d(x):
    import torch
    return torch.as_tensor(np.asarray(x), dtype=torch.float64, device="cuda")


def h(t):
    return t.detach().cpu().numpy()


def test_patch_indices_match_reference_digest(case):
    import hashlib
    for lev, digest in zip(case.mg.levels, case.meta["patch_index_sha256"]):
        hh = hashlib.sha256()
        for ix in lev.patches.patch_indices:
            hh.update(np.asarray(ix, dtype=np.int64).tobytes())
            hh.update(b"|")
        assert hh.hexdigest() == digest


def test_operator_apply(case):
    g = case.golden
    op = case.oracle[-1]["op"]
    y = case.S.matvec(g["x_rand"])
    assert rel(y, op.matvec(g["x_rand"])) <= 1e-13
    assert rel(y, g["matvec_xr"]) <= 1e-13
    # device-resident call and residual form
    r = h(case.S.residual(d(g["x_rand"]), d(g["b"])))
    assert rel(r, g["b"] - op.matvec(g["x_rand"])) <= 1e-13


def test_patch_inverses_invert_patch_matrices(case):
    fine = case.mg.levels[-1].patches
    opat = case.oracle[-1]["patches"]
    for (idx_g, inv_g), (idx_o, inv_o) in zip(fine.groups, opat.groups):
        assert np.array_equal(idx_g, idx_o)
        # same inverse up to the patch conditioning (<= 1e7 * eps)
        err = np.linalg.norm(inv_g - inv_o, axis=(1, 2)) / np.linalg.norm(inv_o, axis=(1, 2))
        assert err.max() <= 1e-8


@pytest.mark.parametrize("start", ["zero", "random"])
def test_sweep_matches_oracle(case, start):
    from paper_2202_07381_b200 import apply_vanka
    g = case.golden
    op = case.oracle[-1]["op"]
    opat = case.oracle[-1]["patches"]
    x0 = np.zeros(op.dim) if start == "zero" else g["x_rand"]
    ref = oracle_apply_vanka(opat, op, x0, g["b"], 0.5)
    got = apply_vanka(case.mg.levels[-1].patches, case.S, x0, g["b"], omega=0.5)
    assert rel(got, ref) <= 1e-12
    gold = g["sweep0"] if start == "zero" else g["sweep_rand"]
    assert rel(got, gold) <= 1e-12


def test_pou_sweep_matches_oracle(case):
    from paper_2202_07381_b200 import apply_vanka
    g = case.golden
    op = case.oracle[-1]["op"]
    opat = case.oracle[-1]["patches"]
    w = opat.pou_weights(op.dim)
    ref = oracle_apply_vanka(opat, op, np.zeros(op.dim), g["b"], 0.5, w)
    got = apply_vanka(case.mg.levels[-1].patches, case.S, np.zeros(op.dim), g["b"], omega=0.5,
                      weights="pou")
    assert rel(got, ref) <= 1e-12
    assert rel(got, g["sweep_pou"]) <= 1e-12


def test_sweep_with_reference_inverses(case):
    """Parity mode: the oracle's (np.linalg.inv) inverses installed in the
    device store; only the summation order differs then."""
    from paper_2202_07381_b200 import VankaPatchSet, apply_vanka
    g = case.golden
    op = case.oracle[-1]["op"]
    opat = case.oracle[-1]["patches"]
    pat = VankaPatchSet(case.S, case.disc.fine_mesh, factor=False)
    pat.set_inverses(opat.groups)
    got = apply_vanka(pat, case.S, g["x_rand"], g["b"], omega=0.5)
    assert rel(got, oracle_apply_vanka(opat, op, g["x_rand"], g["b"], 0.5)) <= 1e-14


def test_solve_additive_linear_and_deterministic(case):
    g = case.golden
    pat = case.mg.levels[-1].patches
    r1, r2 = d(g["b"]), d(g["x_rand"])
    z1 = pat.solve_additive(r1)
    z2 = pat.solve_additive(r2)
    z12 = pat.solve_additive(2.0 * r1 - 3.0 * r2)
    assert rel(h(z12), h(2.0 * z1 - 3.0 * z2)) <= 1e-13
    assert np.array_equal(h(pat.solve_additive(r1)), h(z1))  # bitwise repeatable
    assert rel(h(z1), g["solve_additive_b"]) <= 1e-12


@pytest.mark.parametrize("mode", ["cheb", "pou"])
def test_vcycle_protocol(case, mode):
    g = case.golden
    mg = case.mg if mode == "cheb" else case.mg_pou
    omg = oracle_mg(case.oracle, case.case, mode)
    b = g["b"]
    otrace = []
    zo = omg.precondition(b.copy(), otrace)
    otr = dict(otrace)
    # the reference's self-floor: the oracle against itself
    # with every solve_additive's reduction order reversed
    floor = rel(oracle_mg(case.oracle, case.case, mode, reverse=True).precondition(b.copy()), zo)
    mg.trace = {}
    try:
        z = h(mg.precondition(d(b)))
        tr = {k: h(v) for k, v in mg.trace.items()}
    finally:
        mg.trace = None
    gate = max(1e-12, 10.0 * floor)
    # golden (reference run) agrees with the oracle
    assert rel(zo, g["precond_" + mode]) <= gate
    # down-leg intermediates
    for k in tr:
        if k.startswith("pre_") or k.startswith("rc_") or k == "coarse_in":
            assert rel(tr[k], otr[k]) <= 1e-12, k
    # coarse: backward error of the device solve vs SuperLU's own
    A0 = case.oracle[0]["op"].materialize()
    cin = tr["coarse_in"]
    be_dev = np.linalg.norm(A0 @ tr["coarse_out"] - cin) / np.linalg.norm(cin)
    be_ref = np.linalg.norm(A0 @ otr["coarse_out"] - cin) / np.linalg.norm(cin)
    assert be_dev <= max(10 * be_ref, 1e-13)
    # up-leg with the oracle's coarse output injected
    mg.coarse_override = d(otr["coarse_out"])
    try:
        zi = h(mg.precondition(d(b)))
    finally:
        mg.coarse_override = None
    assert rel(zi, zo) <= 1e-12
    # end to end: 1e-12, or 10x the reference's own self-floor where the
    # coarse solve amplifies rounding (s3: floor ~5e-10)
    assert rel(z, zo) <= gate
    if case.name in WELL_CONDITIONED:
        assert rel(z, zo) <= 1e-12


@pytest.mark.parametrize("mode", ["cheb", "pou"])
def test_fgmres_iterations(case, mode):
    from paper_2202_07381_b200 import fgmres
    g = case.golden
    mg = case.mg if mode == "cheb" else case.mg_pou
    x, st = fgmres(case.S.matvec, d(g["b"]), precond=mg.precondition, rtol=1e-8, maxiter=200,
                   restart=50)
    assert st.converged
    assert abs(st.iterations - case.meta["fgmres_its_" + mode]) <= 1
    assert np.all(np.diff(st.residual_norms) <= 1e-12)


def test_graph_precondition_matches_eager(case):
    mg = case.mg
    r = d(case.golden["b"])
    z_eager = h(mg.precondition(r))
    mg.use_graph = True
    try:
        z1 = h(mg.precondition(r))
        z2 = h(mg.precondition(d(case.golden["x_rand"])))
        z3 = h(mg.precondition(r))
    finally:
        mg.use_graph = False
    assert np.array_equal(z1, z_eager)
    assert np.array_equal(z3, z_eager)
    assert not np.array_equal(z2, z1)


def test_fixed_point_at_exact_solution(case):
    from paper_2202_07381_b200 import apply_vanka
    xs = case.golden["x_rand"]
    b = case.S.matvec(xs)
    y = apply_vanka(case.mg.levels[-1].patches, case.S, xs, b, omega=1.0)
    assert np.max(np.abs(y - xs)) <= 1e-12 * max(1.0, np.max(np.abs(xs)))
