"""Where the modal setup time goes (cfg4 fine level): gather + each batched
torch.linalg step for the largest k group.  python scripts/time_modal_setup.py cfg4"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2202_07381_b200 import VankaPatchSet  # noqa: E402
from paper_2202_07381_b200.stages import assemble_stage_operator  # noqa: E402


def main(name):
    cfg = bench.CONFIGS[name]
    disc, tab, conv = bench.make_disc(cfg)
    S = assemble_stage_operator(disc.blocks[-1], tab, cfg["dt"], constrained=disc.cdofs[-1])
    t0 = time.perf_counter()
    pat = VankaPatchSet(S, disc.fine_mesh, mode="modal", factor=False)
    pat.device_data()
    torch.cuda.synchronize()
    print(f"tables+upload {time.perf_counter() - t0:.2f} s")
    n = 4096
    for k in (19, 65):
        for step in ("chol", "trsm", "eigh", "inv"):
            X = torch.randn(n, k, k, dtype=torch.float64, device="cuda")
            A = X @ X.mT + k * torch.eye(k, dtype=torch.float64, device="cuda")
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if step == "chol":
                torch.linalg.cholesky_ex(A)
            elif step == "trsm":
                torch.linalg.solve_triangular(A.tril(), A, upper=False)
            elif step == "eigh":
                torch.linalg.eigh(A)
            else:
                torch.linalg.inv(A)
            torch.cuda.synchronize()
            print(f"k={k} {step}: {time.perf_counter() - t0:.3f} s per {n}")
    t0 = time.perf_counter()
    pat.factor()
    torch.cuda.synchronize()
    print(f"factor {time.perf_counter() - t0:.2f} s for {pat.num_patches} patches")


if __name__ == "__main__":
    main(sys.argv[1])
