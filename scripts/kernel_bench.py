"""Per-kernel CUDA-event timings on cfg2 (K1, K3 in both formulations and
both scatter layouts, K4).  python scripts/kernel_bench.py [reps]"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from harness import setup  # noqa: E402
from paper_2202_07381_b200 import VankaPatchSet, _lib  # noqa: E402
from paper_2202_07381_b200._device import ptr, stream  # noqa: E402
from paper_2202_07381_b200.stages import StageSystem  # noqa: E402


def timeit(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3  # us


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
    name = sys.argv[2] if len(sys.argv) > 2 else "cfg2"
    disc, tab, conv, case = setup(name)
    k = disc.num_levels - 1
    S = StageSystem(disc.blocks[k], tab, case["dt"], disc.cdofs[k],
                    None if conv is None else conv[k])
    L = _lib.lib()
    x = torch.randn(S.dim, dtype=torch.float64, device="cuda")
    b = torch.randn_like(x)
    r = torch.empty_like(x)
    out = {"dim": S.dim}
    out["K1_us"] = timeit(lambda: L.ivk_stage_apply(S.desc, ptr(x), ptr(b), ptr(r), stream()), reps)
    from paper_2202_07381_b200.solvers import CoarseSolver
    S0 = StageSystem(disc.blocks[0], tab, case["dt"], disc.cdofs[0],
                     None if conv is None else conv[0])
    cs = CoarseSolver(S0)
    b0 = torch.randn(S0.dim, dtype=torch.float64, device="cuda")
    x0 = torch.empty_like(b0)
    out["coarse_us"] = timeit(lambda: cs.solve_into(b0, x0), reps)
    cl = CoarseSolver(S0, "lu")
    out["coarse_lu_us"] = timeit(lambda: cl.solve_into(b0, x0), reps)
    modes = sys.argv[3].split(",") if len(sys.argv) > 3 else \
        (["kron", "dedup", "kron-sym", "full"] if conv is None else ["kron", "full"])
    for mode in modes:
        for scatter in (os.environ.get("KB_SCATTER", "patch").split(",")):
            pat = VankaPatchSet(S, disc.fine_mesh, mode=mode, scatter=scatter)
            dev = pat.device_data()
            w = pat.weights("pou")
            k3 = timeit(lambda: L.ivk_patch_apply(dev["desc"], ptr(r), ptr(dev["local"]),
                                                  stream()), reps)
            k4 = timeit(lambda: L.ivk_patch_combine(dev["desc"], ptr(dev["local"]), ptr(x), 1.0,
                                                    0.5, ptr(w), ptr(b), None, stream()), reps)

            def sweep():
                L.ivk_stage_apply(S.desc, ptr(x), ptr(b), ptr(r), stream())
                L.ivk_patch_apply(dev["desc"], ptr(r), ptr(dev["local"]), stream())
                L.ivk_patch_combine(dev["desc"], ptr(dev["local"]), ptr(x), 1.0, 0.5, ptr(w),
                                    ptr(x), None, stream())
            sw = timeit(sweep, reps)
            out[f"{mode}_{scatter}"] = {"K3_us": k3, "K4_us": k4, "sweep_us": sw,
                                        "inverse_GB": 8 * pat.inv_size / 1e9}
            del pat, dev
            torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
