"""Test/bench harness: BASELINE configurations, seeded inputs and the CPU
oracle built on the same host setup the device path uses."""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from oracle.irk_vanka_oracle import (OracleMG, OraclePatches, OracleStageOperator,  # noqa: E402
                                     oracle_patch_indices)
from paper_2202_07381_b200 import Discretization, tableau_lookup  # noqa: E402
from paper_2202_07381_b200.discretization import oseen_convection  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")

# BASELINE.json configs, diagonal grids with an 8x8 base.
CONFIGS = {
    "cfg1": dict(grid="diagonal", n0=8, level=2, mu=1.0, family="radauiia", stages=2,
                 dt=1 / 32, seed=0, cheby_a=2.0, conv=False),
    "cfg2": dict(grid="diagonal", n0=8, level=5, mu=1.0, family="radauiia", stages=3,
                 dt=1 / 256, seed=1, cheby_a=2.0, conv=False),
    "cfg3": dict(grid="diagonal", n0=8, level=6, mu=0.01, family="gauss", stages=2,
                 dt=1 / 512, seed=2, cheby_a=1.5, conv=True),
    # reduced-grid parity cases with the cfg2 / cfg3 schemes (tests/golden/*.npz)
    "s3": dict(grid="diagonal", n0=8, level=2, mu=1.0, family="radauiia", stages=3,
               dt=1 / 256, seed=1, cheby_a=2.0, conv=False),
    "ns": dict(grid="diagonal", n0=8, level=2, mu=0.01, family="gauss", stages=2,
               dt=1 / 512, seed=2, cheby_a=1.5, conv=True),
    "crossed": dict(grid="crossed", n0=2, level=1, mu=1.0, family="radauiia", stages=2,
                    dt=0.1, seed=10, cheby_a=2.0, conv=False),
}


def setup(name):
    """(disc, tableau, convection-or-None, case) for a named configuration."""
    case = CONFIGS[name]
    disc = Discretization(case["n0"], case["level"], mu=case["mu"], grid=case["grid"])
    tab = tableau_lookup(case["family"], case["stages"])
    conv = oseen_convection(disc, case["stages"]) if case["conv"] else None
    return disc, tab, conv, case


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def oracle_levels(disc, tab, dt, conv, levels=None, threads=1):
    """Oracle operators / patches / stage prolongations on every level
    (``threads``: host threads for the batched patch inversions)."""
    out = []
    ks = range(disc.num_levels) if levels is None else levels
    for k in ks:
        blk = disc.blocks[k]
        cm = None if conv is None else [J.matrix for J in conv[k]]
        op = OracleStageOperator(blk.M, blk.K, blk.B, tab.A, dt, disc.cdofs[k], convection=cm)
        mesh = disc.hier.levels[k]
        vels, idxs = oracle_patch_indices(mesh.cells, mesh.cell_to_edges, mesh.num_vertices, op)
        pat = OraclePatches(op, vels, idxs, threads=threads) if k > 0 else None
        P = disc.stage_prolong(k, tab.r).matrix if k > 0 else None
        out.append({"op": op, "patches": pat, "prolong": P, "idxs": idxs})
    return out


def oracle_mg(levels, case, mode, threads=1, reverse=False):
    if mode == "cheb":
        sm = dict(pre=2, post=2, accel="chebyshev", a=case["cheby_a"], b=8.0, omega=1.0,
                  weights=None)
    else:
        sm = dict(pre=2, post=2, accel="richardson", omega=0.5, weights="pou")
    return OracleMG(levels, sm, threads=threads, reverse=reverse)


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def load_golden(name):
    import json
    data = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    with open(os.path.join(GOLDEN, f"{name}.json")) as fh:
        meta = json.load(fh)
    return data, meta


# BASELINE config 5 (2-D resistive MHD, mhd.py) and reduced parity cases with
# its scheme.  No reference implementation exists: parity is against the
# oracle restatement only (oracle/general_oracle.py, "parity unpinned").
MHD_CONFIGS = {
    "cfg5": dict(n0=8, level=4, Re=100.0, Rm=100.0, S=1.0, family="radauiia", stages=2,
                 dt=1 / 128, seed=4),
    "mhd16": dict(n0=8, level=1, Re=100.0, Rm=100.0, S=1.0, family="radauiia", stages=2,
                  dt=1 / 128, seed=4),
    "mhd32": dict(n0=8, level=2, Re=100.0, Rm=100.0, S=1.0, family="radauiia", stages=2,
                  dt=1 / 128, seed=4),
    "mhd16s3": dict(n0=8, level=1, Re=100.0, Rm=100.0, S=1.0, family="radauiia", stages=3,
                    dt=1 / 128, seed=5),
}


def mhd_setup(name):
    from paper_2202_07381_b200.mhd import MHDDiscretization, MHDParams
    case = MHD_CONFIGS[name]
    disc = MHDDiscretization(case["n0"], case["level"],
                             MHDParams(case["Re"], case["Rm"], case["S"]))
    return disc, tableau_lookup(case["family"], case["stages"]), case


def mhd_oracle_levels(disc, tab, dt, levels=None, patches=True):
    """Oracle operators / patches / stage prolongations on every MHD level."""
    import scipy.sparse as sp
    from oracle.general_oracle import (OracleGeneralOperator, OracleGeneralPatches,
                                       oracle_general_patch_indices)
    out = []
    ks = range(disc.num_levels) if levels is None else levels
    for k in ks:
        o = disc.ops[k]
        n_nodes, nv, n1 = o["layout"]
        M = sp.csr_matrix((o["m"], o["col"], o["rowptr"]), shape=(n1, n1))
        L = sp.csr_matrix((o["l"], o["col"], o["rowptr"]), shape=(n1, n1))
        op = OracleGeneralOperator(M, L, tab.A, dt, np.flatnonzero(o["cmask"]), n1 - nv)
        mesh = disc.hier.levels[k]
        idxs = oracle_general_patch_indices(mesh.cells, mesh.cell_to_edges, mesh.num_vertices,
                                            op, 4, 2)
        pat = OracleGeneralPatches(op, idxs) if (k > 0 and patches) else None
        P = disc.stage_prolong(k, tab.r).matrix if k > 0 else None
        out.append({"op": op, "patches": pat, "prolong": P, "idxs": idxs})
    return out
