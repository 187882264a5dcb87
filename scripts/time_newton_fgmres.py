"""Where a Newton iteration's linear solve spends its time at cfg3 (after one
relinearisation): first / later V-cycles, the per-stage-Jacobian matvec, the
FGMRES call.  python scripts/time_newton_fgmres.py"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from harness import setup  # noqa: E402
from paper_2202_07381_b200 import SmootherSpec, fem, newton, solvers  # noqa: E402
from paper_2202_07381_b200.discretization import streamfunction_velocity  # noqa: E402


def clock(label, fn, reps=1):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        out = fn()
    torch.cuda.synchronize()
    print(f"{label:40s} {1e3 * (time.perf_counter() - t0) / reps:9.2f} ms")
    return out


disc, tab, conv, case = setup(sys.argv[1] if len(sys.argv) > 1 else "cfg3")
cheb = SmootherSpec(pre=2, post=2, accel="chebyshev", cheby_a=case["cheby_a"], cheby_b=8.0)
nsn = newton.NSStageNewton(disc, tab, case["dt"], cheb)
u_n = torch.from_numpy(fem.interpolate_velocity(disc.fine_mesh, streamfunction_velocity)).cuda()
k = torch.zeros(nsn.S0.dim, dtype=torch.float64, device="cuda")
clock("relinearize (cold)", lambda: nsn.relinearize(k, u_n))
clock("relinearize (warm)", lambda: nsn.relinearize(k, u_n))
b = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, nsn.S0.dim)).cuda()
clock("first precondition after relinearize", lambda: nsn.mg.precondition(b))
clock("precondition", lambda: nsn.mg.precondition(b), 5)
clock("matvec (per-stage Jacobians)", lambda: nsn.S.matvec(b), 5)
clock("fgmres rtol 1e-2", lambda: solvers.fgmres(nsn.S.matvec, b, precond=nsn.mg.precondition,
                                                  rtol=1e-2, maxiter=50, restart=50))
x, st = solvers.fgmres(nsn.S.matvec, b, precond=nsn.mg.precondition, rtol=1e-2, maxiter=50,
                       restart=50)
print("iterations", st.iterations)
