"""K3/K4 timings for the two scatter layouts (patch order vs owner-sorted
slot_pos) of one patch formulation on a bench config.
    python scripts/kbench_scatter.py cfg2 modal"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2202_07381_b200 import SmootherSpec, VankaPatchSet, _lib  # noqa: E402
from paper_2202_07381_b200._device import ptr, stream  # noqa: E402


def main(name, mode):
    cfg = bench.CONFIGS[name]
    disc, tab, conv = bench.make_disc(cfg)
    mg, S = disc.build_mg(tab, cfg["dt"], SmootherSpec(), convection=conv, patch_mode=mode)
    b = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, S.dim)).cuda()
    L = _lib.lib()
    for scatter in ("patch", "owner"):
        pat = VankaPatchSet(S, disc.fine_mesh, mode=mode, scatter=scatter)
        dev = pat.device_data()
        x, r = torch.zeros_like(b), torch.zeros_like(b)
        w = pat.weights("pou")
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        t = np.zeros(3)
        n = 30
        for it in range(n):
            st = stream()
            ev[0].record()
            _lib.check(L.ivk_stage_apply(S.desc, ptr(x), ptr(b), ptr(r), st), "K1")
            ev[1].record()
            _lib.check(L.ivk_patch_apply(dev["desc"], ptr(r), ptr(dev["local"]), st), "K3")
            ev[2].record()
            _lib.check(L.ivk_patch_combine(dev["desc"], ptr(dev["local"]), ptr(x), 1.0, 0.5,
                                           ptr(w), ptr(x), None, st), "K4")
            ev[3].record()
            torch.cuda.synchronize()
            if it >= 5:
                t += [ev[k].elapsed_time(ev[k + 1]) for k in range(3)]
        t /= n - 5
        print(f"{name} {mode} scatter={scatter}: K1 {1e3 * t[0]:.1f} us, K3 {1e3 * t[1]:.1f} us, "
              f"K4 {1e3 * t[2]:.1f} us, sum {1e3 * t.sum():.1f} us")
        del pat
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "modal")
