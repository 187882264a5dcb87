"""Phase breakdown of the device Navier-Stokes Newton step (cfg3 or a
smaller grid): K10 assembly, K7 refactor per level, coarse rebuild, FGMRES,
residual -- host-clocked with a device synchronize around every phase.

    python scripts/time_newton.py [cfg3|ns] [runs]
"""
import json
import os
import sys
import time
from collections import defaultdict

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from harness import setup  # noqa: E402
from paper_2202_07381_b200 import SmootherSpec, fem, newton, solvers  # noqa: E402
from paper_2202_07381_b200.discretization import streamfunction_velocity  # noqa: E402

T = defaultdict(float)
N = defaultdict(int)


def timed(name, fn):
    def w(*a, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = fn(*a, **k)
        torch.cuda.synchronize()
        T[name] += time.perf_counter() - t0
        N[name] += 1
        return out
    return w


def main(name="cfg3", runs=2):
    disc, tab, conv, case = setup(name)
    cheb = SmootherSpec(pre=2, post=2, accel="chebyshev", cheby_a=case["cheby_a"], cheby_b=8.0)
    t0 = time.perf_counter()
    nsn = newton.NSStageNewton(disc, tab, case["dt"], cheb)
    torch.cuda.synchronize()
    build = time.perf_counter() - t0
    # instrument the phases
    for lev in nsn.mg.levels[1:]:
        k = lev.system.n_nodes
        lev.patches.factor = timed(f"K7 factor (n_nodes {k}, {lev.patches.num_patches} patches)",
                                   lev.patches.factor)
    for a in nsn.asm:
        a.assemble_stage = timed("K10 assemble_stage", a.assemble_stage)
    solvers.CoarseSolver.from_device_operator = staticmethod(
        timed("coarse operator rebuild (device)",
              solvers.CoarseSolver.from_device_operator))
    newton.fgmres = timed("fgmres", solvers.fgmres)
    nsn.residual = timed("residual", nsn.residual)
    nsn.relinearize = timed("relinearize (total)", nsn.relinearize)
    u_n = fem.interpolate_velocity(disc.fine_mesh, streamfunction_velocity)
    p_n = np.zeros(disc.fine_mesh.num_vertices)
    out = []
    for r in range(runs):
        T.clear()
        N.clear()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, st = nsn.solve(u_n, p_n, config=newton.NewtonConfig(atol=1e-8))
        torch.cuda.synchronize()
        tot = time.perf_counter() - t0
        out.append({"run": r, "seconds": tot, "newton_iterations": st.iterations,
                    "linear_iterations": [l.iterations for l in st.linear_stats],
                    "phases_s": {k: round(v, 4) for k, v in T.items()},
                    "calls": dict(N)})
    print(json.dumps({"config": name, "build_s": build, "runs": out}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "cfg3", int(sys.argv[2]) if len(sys.argv) > 2 else 2)
