"""Host-side profile of the cfg2 setup (Discretization + build_mg, modal):
python scripts/prof_setup.py [cfg2]"""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402
from harness import CONFIGS  # noqa: E402
from paper_2202_07381_b200 import Discretization, SmootherSpec, tableau_lookup  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
case = CONFIGS[name]
torch.zeros(1).cuda()
for rep in range(2):
    pr = cProfile.Profile()
    t0 = time.perf_counter()
    pr.enable()
    disc = Discretization(case["n0"], case["level"], mu=case["mu"], grid=case["grid"])
    t1 = time.perf_counter()
    tab = tableau_lookup(case["family"], case["stages"])
    mg, S = disc.build_mg(tab, case["dt"], SmootherSpec(), patch_mode="modal")
    torch.cuda.synchronize()
    pr.disable()
    t2 = time.perf_counter()
    print(f"rep {rep}: discretization {t1 - t0:.2f} s, build_mg {t2 - t1:.2f} s")
pstats.Stats(pr).sort_stats("cumulative").print_stats(45)
