"""Full-vector parity at the BASELINE headline sizes (configs 2 and 3).

The CPU oracle (oracle/irk_vanka_oracle.py, pinned to the reference's own
outputs by tests/test_oracle_golden.py) is built over EVERY patch of every
level -- 66,049 fine patches at cfg2, 263,169 at cfg3 -- with the batched
inversions spread over the host threads.  Against it, on identical seeded
inputs (BASELINE RHS convention, x_rand = default_rng(seed + 100)):

  * one fine-level sweep, whole vector, rel l2 <= 1e-12: W = I and PoU, from
    x = 0 and from x_rand, for every device formulation that applies
    (cfg2: modal -- the benched one --, dedup, kron, full; cfg3: kron, full);
  * the V-cycle (mg.precondition, both smoothers) by the decomposed protocol
    of SURVEY.md F9 / BASELINE.md §4: down-leg intermediates <= 1e-12, coarse
    backward error <= 10x SuperLU's own, up-leg with the oracle's coarse
    output injected <= 1e-12, end to end <= max(1e-12, 10 x self-floor) where
    the self-floor is the oracle against itself with the reduction order of
    every solve_additive reversed, measured here in the same run;
  * FGMRES iteration counts of the benched hierarchy within +-1 of the
    reference's (tests/golden/full_counts.json).

Every measured number is printed and, with IVK_PARITY_LOG=<file>, appended
to that file as JSON lines (profiles/r02/parity_fullsize.jsonl).
"""

import json
import os

import numpy as np
import pytest

from harness import GOLDEN, host_threads, oracle_levels, oracle_mg, rel, setup
from oracle.irk_vanka_oracle import oracle_apply_vanka

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

with open(os.path.join(GOLDEN, "full_counts.json")) as fh:
    FULL = json.load(fh)

MODES = {"cfg2": ["modal", "dedup", "kron", "full"], "cfg3": ["kron", "full"]}
CYCLE_MODES = {"cfg2": ["modal", "dedup"], "cfg3": ["kron"]}


def record(**kw):
    line = json.dumps(kw)
    print(line)
    path = os.environ.get("IVK_PARITY_LOG")
    if path:
        with open(path, "a") as fh:
            fh.write(line + "\n")


class Full:
    def __init__(self, name):
        self.name = name
        self.disc, self.tab, self.conv, self.case = setup(name)
        self.threads = host_threads()
        self.oracle = oracle_levels(self.disc, self.tab, self.case["dt"], self.conv,
                                    threads=self.threads)
        op = self.oracle[-1]["op"]
        b = np.random.default_rng(self.case["seed"]).uniform(-1.0, 1.0, op.dim)
        b[op.constrained_stage_dofs()] = 0.0
        self.b = op.project_pressure_means(b)
        x = np.random.default_rng(self.case["seed"] + 100).uniform(-1.0, 1.0, op.dim)
        x[op.constrained_stage_dofs()] = 0.0
        self.x_rand = x
        pat = self.oracle[-1]["patches"]
        self.w = pat.pou_weights(op.dim)
        self.ref = {}
        for start, x0 in (("zero", np.zeros(op.dim)), ("random", x)):
            for wname, w in (("I", None), ("pou", self.w)):
                self.ref[(start, wname)] = oracle_apply_vanka(pat, op, x0, self.b, 0.5, w,
                                                              threads=self.threads)
        self._oracle_cycles = {}
        self.mgs = {}
        self.S = None

    def hierarchy(self, mode, smoother):
        from paper_2202_07381_b200 import MGHierarchyOp, MGLevel, SmootherSpec
        if mode not in self.mgs:
            c = self.case
            cheb = SmootherSpec(pre=2, post=2, accel="chebyshev", cheby_a=c["cheby_a"],
                                cheby_b=8.0)
            mg, S = self.disc.build_mg(self.tab, c["dt"], cheb, convection=self.conv,
                                       patch_mode=mode)
            assert mg.levels[-1].patches.mode == mode
            pou = SmootherSpec(pre=2, post=2, accel="richardson", omega=0.5, weighting="pou")
            mg_pou = MGHierarchyOp([MGLevel(l.system, l.patches, pou, l.prolong)
                                    for l in mg.levels], mg.coarse)
            self.mgs[mode] = (mg, mg_pou)
            self.S = S
        mg, mg_pou = self.mgs[mode]
        return mg if smoother == "cheb" else mg_pou

    def oracle_cycle(self, smoother):
        """(z, trace dict, self-floor) of the oracle precondition(b)."""
        if smoother not in self._oracle_cycles:
            tr = []
            z = oracle_mg(self.oracle, self.case, smoother,
                          threads=self.threads).precondition(self.b.copy(), tr)
            zr = oracle_mg(self.oracle, self.case, smoother, threads=self.threads,
                           reverse=True).precondition(self.b.copy())
            self._oracle_cycles[smoother] = (z, dict(tr), rel(zr, z))
        return self._oracle_cycles[smoother]


_cache = {}


def get(name):
    if name not in _cache:
        _cache.clear()
        import gc
        gc.collect()
        _cache[name] = Full(name)
    return _cache[name]


SWEEP_CASES = [(n, m) for n in ("cfg2", "cfg3") for m in MODES[n]]


@pytest.mark.parametrize("name,mode", SWEEP_CASES, ids=[f"{n}-{m}" for n, m in SWEEP_CASES])
def test_full_sweep_parity(name, mode):
    """Whole-vector sweep parity, every patch, four (start, weighting) cases."""
    import torch
    from paper_2202_07381_b200 import VankaPatchSet, apply_vanka
    f = get(name)
    owned = mode not in CYCLE_MODES[name]
    if owned:
        f.hierarchy(CYCLE_MODES[name][0], "cheb")
        pat = VankaPatchSet(f.S, f.disc.fine_mesh, mode=mode)
    else:
        pat = f.hierarchy(mode, "cheb").levels[-1].patches
    S = f.S
    assert pat.mode == mode
    bd = torch.from_numpy(f.b).cuda()
    worst = 0.0
    for (start, wname), ref in f.ref.items():
        x0 = torch.zeros_like(bd) if start == "zero" else torch.from_numpy(f.x_rand).cuda()
        got = apply_vanka(pat, S, x0, bd, omega=0.5,
                          weights=None if wname == "I" else "pou").cpu().numpy()
        e = rel(got, ref)
        record(test="sweep", config=name, mode=mode, start=start, weights=wname, rel=e)
        worst = max(worst, e)
        assert e <= 1e-12, (start, wname, e)
    if owned:
        del pat
        torch.cuda.empty_cache()


CYCLE_CASES = [(n, m, s) for n in ("cfg2", "cfg3") for m in CYCLE_MODES[n]
               for s in ("cheb", "pou")]


@pytest.mark.parametrize("name,mode,smoother", CYCLE_CASES,
                         ids=[f"{n}-{m}-{s}" for n, m, s in CYCLE_CASES])
def test_full_vcycle_protocol(name, mode, smoother):
    import torch
    f = get(name)
    mg = f.hierarchy(mode, smoother)
    zo, otr, floor = f.oracle_cycle(smoother)
    bd = torch.from_numpy(f.b).cuda()
    mg.trace = {}
    try:
        z = mg.precondition(bd).cpu().numpy()
        tr = {k: v.cpu().numpy() for k, v in mg.trace.items()}
    finally:
        mg.trace = None
    down = {k: rel(tr[k], otr[k]) for k in tr
            if k.startswith("pre_") or k.startswith("rc_") or k == "coarse_in"}
    A0 = f.oracle[0]["op"].materialize()
    cin = tr["coarse_in"]
    be_dev = float(np.linalg.norm(A0 @ tr["coarse_out"] - cin) / np.linalg.norm(cin))
    be_ref = float(np.linalg.norm(A0 @ otr["coarse_out"] - cin) / np.linalg.norm(cin))
    mg.coarse_override = torch.from_numpy(otr["coarse_out"]).cuda()
    try:
        zi = mg.precondition(bd).cpu().numpy()
    finally:
        mg.coarse_override = None
    up = rel(zi, zo)
    e2e = rel(z, zo)
    gate = max(1e-12, 10.0 * floor)
    record(test="vcycle", config=name, mode=mode, smoother=smoother,
           down_leg_max=max(down.values()), down_leg=down, coarse_backward_error=be_dev,
           coarse_backward_error_superlu=be_ref, up_leg_injected=up, end_to_end=e2e,
           self_floor=floor, end_to_end_gate=gate)
    for k, e in down.items():
        assert e <= 1e-12, (k, e)
    assert be_dev <= max(10.0 * be_ref, 1e-13)
    assert up <= 1e-12
    assert e2e <= gate


@pytest.mark.parametrize("name,mode,smoother", CYCLE_CASES,
                         ids=[f"{n}-{m}-{s}" for n, m, s in CYCLE_CASES])
def test_full_fgmres_counts(name, mode, smoother):
    import torch
    from paper_2202_07381_b200 import fgmres
    f = get(name)
    mg = f.hierarchy(mode, smoother)
    bd = torch.from_numpy(f.b).cuda()
    _, st = fgmres(f.S.matvec, bd, precond=mg.precondition, rtol=1e-8, maxiter=200,
                   restart=50)
    ref = FULL[name][f"fgmres_its_{smoother}"]
    record(test="fgmres", config=name, mode=mode, smoother=smoother, iterations=st.iterations,
           reference_iterations=ref, relative_residual=st.relative_residual)
    assert st.converged and st.relative_residual <= 1e-8
    assert abs(st.iterations - ref) <= 1
