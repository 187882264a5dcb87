"""K7 timing: CUDA-event time of the patch factorisation (assemble + invert
+ store) on every level of a bench config's hierarchy, per formulation.

    python scripts/time_k7.py [cfg3|cfg2|cfg1|ns] [full,kron] [reps]

Prints one JSON object: per level and mode the median milliseconds, the
Gauss-Jordan flops (2 d^3 per real matrix, 8 b^3 per complex eigen-block) and
the implied FP64 rate.  IVK_K7_SMEM=1 selects the previous shared-memory
elimination for the A/B.
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from harness import setup  # noqa: E402
from paper_2202_07381_b200 import SmootherSpec  # noqa: E402


def flops(pat, mode, tab):
    m = np.asarray(pat.tables.sizes, dtype=np.float64)
    s = tab.A.shape[0]
    if mode == "full":
        return float((2.0 * m ** 3).sum())
    b = m / s
    lam = np.linalg.eigvals(tab.A)
    n_real = int(np.sum(np.abs(lam.imag) < 1e-12))
    n_pair = (s - n_real) // 2
    return float(((2.0 * n_real + 8.0 * n_pair) * b ** 3).sum())


def main(name="cfg3", modes="full,kron", reps=5):
    disc, tab, conv, case = setup(name)
    sm = SmootherSpec(pre=2, post=2, accel="chebyshev", cheby_a=case["cheby_a"], cheby_b=8.0)
    out = {"config": name, "smem_path": bool(os.environ.get("IVK_K7_SMEM")), "levels": []}
    for mode in modes.split(","):
        mg, _ = disc.build_mg(tab, case["dt"], sm, convection=conv, patch_mode=mode)
        for lev in mg.levels[1:]:
            pat = lev.patches
            ts = []
            for _ in range(reps):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                a.record()
                pat.factor()
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            ms = float(np.median(ts))
            fl = flops(pat, pat.mode, tab)
            out["levels"].append({"mode": pat.mode, "patches": int(pat.num_patches),
                                  "max_m": int(pat.tables.sizes.max()), "ms": round(ms, 4),
                                  "gflop": round(fl / 1e9, 3),
                                  "tflops": round(fl / ms / 1e9, 3)})
        del mg
        torch.cuda.empty_cache()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    a = sys.argv[1:]
    main(a[0] if a else "cfg3", a[1] if len(a) > 1 else "full,kron", int(a[2]) if len(a) > 2 else 5)
