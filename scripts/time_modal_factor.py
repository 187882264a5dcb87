"""Modal setup A/B at a bench config's fine level: K7m (ivk_modal_factor, a
warp per patch) against the batched torch.linalg / cuSOLVER route
(IVK_MODAL_SETUP=cusolver), host-clocked with synchronisation, plus the
record-level agreement of the two (patch inverses rebuilt from the records).

    python scripts/time_modal_factor.py [cfg2|cfg1] [reps]
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from harness import setup  # noqa: E402
from paper_2202_07381_b200 import VankaPatchSet  # noqa: E402
from paper_2202_07381_b200.stages import assemble_stage_operator  # noqa: E402


def main(name="cfg2", reps=3):
    disc, tab, conv, case = setup(name)
    S = assemble_stage_operator(disc.blocks[-1], tab, case["dt"], constrained=disc.cdofs[-1])
    pat = VankaPatchSet(S, disc.fine_mesh, mode="modal", factor=False)
    pat.device_data()
    out = {"config": name, "patches": int(pat.num_patches)}
    stores = {}
    for how in ("k7m", "cusolver"):
        os.environ["IVK_MODAL_SETUP"] = "" if how == "k7m" else "cusolver"
        ts = []
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            pat.factor()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        out[how + "_ms"] = round(1e3 * float(np.median(ts)), 3)
        stores[how] = pat.device_data()["inv"].clone()
    # agreement: the exact patch inverse rebuilt from each route's record
    t = pat.tables
    ks = np.diff(t.node_off)
    rng = np.random.default_rng(0)
    worst = 0.0
    for slot in rng.choice(pat.num_patches, size=24, replace=False):
        k = int(ks[slot])
        rec = pat.modal.record_doubles(k)
        off = int(pat.inv_off[slot])
        a = pat.modal.full_inverse(stores["k7m"][off:off + rec].cpu().numpy(), k)
        b = pat.modal.full_inverse(stores["cusolver"][off:off + rec].cpu().numpy(), k)
        worst = max(worst, float(np.linalg.norm(a - b) / np.linalg.norm(b)))
    out["inverse_rel_diff_max_24_patches"] = worst
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "cfg2", int(sys.argv[2]) if len(sys.argv) > 2 else 3)
