"""Profiling workload for the cfg4 / cfg5 fine-level sweep: build the
hierarchy exactly as bench.py does (patch_mode="kron"), then run N sweeps
K1 (K1g for MHD) -> K3e (wide) -> K4 with CUDA-event timings printed.

    python scripts/prof_general.py cfg5 [sweeps] [patch_mode]
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2202_07381_b200 import SmootherSpec, _lib  # noqa: E402
from paper_2202_07381_b200._device import ptr, stream  # noqa: E402


def main(name, n, mode="kron"):
    cfg = bench.CONFIGS[name]
    disc, tab, conv = bench.make_disc(cfg)
    mg, S = disc.build_mg(tab, cfg["dt"], SmootherSpec(), convection=conv, patch_mode=mode)
    pat = mg.levels[-1].patches
    dev = pat.device_data()
    if os.environ.get("IVK_EXP_SHARE_RECORDS") and pat.mode == "modal":
        # experiment: patches with bitwise identical records read one copy
        from paper_2202_07381_b200.modal import _bitwise_classes
        ks = np.diff(pat.tables.node_off)
        off = np.asarray(pat.inv_off, dtype=np.int64).copy()
        ncls = 0
        for k in np.unique(ks):
            sel = np.flatnonzero(ks == k)
            rec = pat.modal.record_doubles(int(k))
            first, count = int(sel[0]), len(sel)
            o0 = int(off[first])
            recs = dev["inv"][o0:o0 + count * rec].view(count, rec)
            rep, inv = _bitwise_classes(recs)
            ncls += len(rep)
            off[first:first + count] = o0 + rep.cpu().numpy()[inv.cpu().numpy()] * rec
        dev["inv_off"].copy_(torch.from_numpy(off).to(dev["inv_off"].device))
        print(f"shared records: {ncls} classes for {pat.num_patches} patches")
    b_h = np.random.default_rng(cfg["seed"]).uniform(-1, 1, S.dim)
    b_h[S.constrained_stage_dofs()] = 0.0
    S.project_pressure_means(b_h)
    b = torch.from_numpy(b_h).cuda()
    x, r = torch.zeros_like(b), torch.zeros_like(b)
    w = pat.weights("pou")
    L = _lib.lib()
    k1 = L.ivk_general_apply if getattr(S, "general", False) else L.ivk_stage_apply
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    t = np.zeros(3)
    for it in range(n):
        st = stream()
        ev[0].record()
        _lib.check(k1(S.desc, ptr(x), ptr(b), ptr(r), st), "K1")
        ev[1].record()
        _lib.check(L.ivk_patch_apply(dev["desc"], ptr(r), ptr(dev["local"]), st), "K3")
        ev[2].record()
        _lib.check(L.ivk_patch_combine(dev["desc"], ptr(dev["local"]), ptr(x), 1.0,
                                       cfg.get("omega", 0.5), ptr(w), ptr(x), None, st), "K4")
        ev[3].record()
        torch.cuda.synchronize()
        if it >= 2:
            t += [ev[k].elapsed_time(ev[k + 1]) for k in range(3)]
    t /= max(n - 2, 1)
    print(f"{name}: mode {pat.mode}, K1 {1e3 * t[0]:.1f} us, K3 {1e3 * t[1]:.1f} us, "
          f"K4 {1e3 * t[2]:.1f} us, inverse store {8 * pat.inv_size / 1e9:.3f} GB, "
          f"finite {bool(torch.isfinite(x).all())}, r checksum {float(r.abs().sum())!r}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 6,
         sys.argv[3] if len(sys.argv) > 3 else "kron")
