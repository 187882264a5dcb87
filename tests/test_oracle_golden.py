"""Pin the CPU oracle against golden vectors produced by the reference
package itself (tests/golden/make_golden.py) -- CPU only.

The oracle runs on this repo's host setup (mesh, assembly, patch tables);
the goldens come from the reference's own setup and solvers, so these
tests pin both the oracle restatement and the setup it shares with the
device path.  Tolerances follow SURVEY.md F5/F9: sweeps 1e-12; V-cycles
1e-12 where the coarse solve is well conditioned, else the decomposed
protocol (down-leg 1e-12, coarse-injected up-leg 1e-12, end to end 1e-8).
"""

import numpy as np
import pytest

from harness import load_golden, oracle_levels, oracle_mg, rel, setup
from oracle.irk_vanka_oracle import oracle_apply_vanka, oracle_fgmres, random_rhs

CASES = ["cfg1", "s3", "ns", "crossed"]
WELL_CONDITIONED = {"cfg1", "ns", "crossed"}
_cache = {}


def _case(name):
    if name not in _cache:
        g, meta = load_golden(name)
        disc, tab, conv, case = setup(name)
        _cache[name] = (g, meta, disc, tab, conv, case,
                        oracle_levels(disc, tab, case["dt"], conv))
    return _cache[name]


@pytest.mark.parametrize("name", CASES)
def test_rhs_and_operator(name):
    g, meta, disc, tab, conv, case, L = _case(name)
    op = L[-1]["op"]
    assert op.dim == meta["dim"]
    assert np.array_equal(random_rhs(op, case["seed"]), g["b"])
    assert rel(op.matvec(g["x_rand"]), g["matvec_xr"]) <= 1e-13


@pytest.mark.parametrize("name", CASES)
def test_sweeps(name):
    g, meta, disc, tab, conv, case, L = _case(name)
    op, pat = L[-1]["op"], L[-1]["patches"]
    b = g["b"]
    assert rel(oracle_apply_vanka(pat, op, np.zeros(op.dim), b, 0.5), g["sweep0"]) <= 1e-12
    assert rel(oracle_apply_vanka(pat, op, g["x_rand"], b, 0.5), g["sweep_rand"]) <= 1e-12
    w = pat.pou_weights(op.dim)
    assert np.array_equal(w, g["pou_w"])
    assert rel(oracle_apply_vanka(pat, op, np.zeros(op.dim), b, 0.5, w), g["sweep_pou"]) <= 1e-12
    assert rel(pat.solve_additive(b), g["solve_additive_b"]) <= 1e-12


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("mode", ["cheb", "pou"])
def test_vcycle(name, mode):
    g, meta, disc, tab, conv, case, L = _case(name)
    mg = oracle_mg(L, case, mode)
    trace = []
    z = mg.precondition(g["b"].copy(), trace)
    tr = dict(trace)
    for k, v in tr.items():
        if k.startswith("pre_") or k.startswith("rc_") or k == "coarse_in":
            assert rel(v, g[f"{mode}_{k}"]) <= 1e-12, k
    mg.coarse_hook = lambda rhs: g[f"{mode}_coarse_out"].copy()
    zi = mg.precondition(g["b"].copy())
    mg.coarse_hook = None
    assert rel(zi, g[f"precond_{mode}"]) <= 1e-12
    tol = 1e-12 if name in WELL_CONDITIONED else 1e-8
    assert rel(z, g[f"precond_{mode}"]) <= tol


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("mode", ["cheb", "pou"])
def test_fgmres_counts(name, mode):
    g, meta, disc, tab, conv, case, L = _case(name)
    op = L[-1]["op"]
    mg = oracle_mg(L, case, mode)
    _, (its, norms, ok) = oracle_fgmres(op.matvec, g["b"], mg.precondition, rtol=1e-8,
                                        maxiter=200, restart=50)
    assert ok
    assert abs(its - meta[f"fgmres_its_{mode}"]) <= 1
    assert np.all(np.diff(norms) <= 1e-12)
