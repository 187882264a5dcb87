"""Small fixed workload for ncu: cfg2 setup, 3 fine sweeps (K1->K3->K4),
then one eager V-cycle per smoother.  Usage: python scripts/prof_workload.py [cfg]"""

import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from harness import setup  # noqa: E402
from paper_2202_07381_b200 import MGHierarchyOp, MGLevel, SmootherSpec, apply_vanka  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    disc, tab, conv, case = setup(name)
    cheb = SmootherSpec(pre=2, post=2, accel="chebyshev", cheby_a=case["cheby_a"], cheby_b=8.0)
    mg, S = disc.build_mg(tab, case["dt"], cheb, convection=conv)
    pou = SmootherSpec(pre=2, post=2, accel="richardson", omega=0.5, weighting="pou")
    mg_pou = MGHierarchyOp([MGLevel(l.system, l.patches, pou, l.prolong) for l in mg.levels],
                           mg.coarse)
    b = np.random.default_rng(case["seed"]).uniform(-1, 1, S.dim)
    b[S.constrained_stage_dofs()] = 0.0
    S.project_pressure_means(b)
    bd = torch.from_numpy(b).cuda()
    x = torch.zeros_like(bd)
    fine = mg.levels[-1].patches
    for _ in range(3):
        x = apply_vanka(fine, S, x, bd, omega=0.5, weights="pou")
    torch.cuda.synchronize()
    z1 = mg.precondition(bd)
    z2 = mg_pou.precondition(bd)
    torch.cuda.synchronize()
    print("ok", float(torch.linalg.vector_norm(x)), float(torch.linalg.vector_norm(z1)),
          float(torch.linalg.vector_norm(z2)))


if __name__ == "__main__":
    main()
