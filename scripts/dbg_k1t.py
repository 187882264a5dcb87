import os, sys, numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from harness import setup
from paper_2202_07381_b200 import StageSystem
name, tr = sys.argv[1], sys.argv[2]
disc, tab, conv, case = setup(name)
k = disc.num_levels - 1
os.environ["IVK_K1_TILES"] = tr
St = StageSystem(disc.blocks[k], tab, case["dt"], disc.cdofs[k]); St.device_data()
os.environ["IVK_K1_TILES"] = "0"
Ss = StageSystem(disc.blocks[k], tab, case["dt"], disc.cdofs[k]); Ss.device_data()
rng = np.random.default_rng(5)
x = torch.from_numpy(rng.standard_normal(St.dim)).cuda()
b = torch.from_numpy(rng.standard_normal(St.dim)).cuda()
print(St.k1_plan_stats)
for rhs in (None, b):
    yt = torch.full_like(x, float("nan")); ys = torch.full_like(x, float("nan"))
    St.apply_into(x, rhs, yt); Ss.apply_into(x, rhs, ys)
    torch.cuda.synchronize()
    d = (yt - ys).abs()
    bad = torch.nonzero(~(yt == ys)).ravel().cpu().numpy()
    sd = St.stage_dim
    print("rhs", rhs is not None, "nan", int(torch.isnan(yt).sum()), "nbad", len(bad), "maxdiff", float(d[~torch.isnan(d)].max()) if len(bad) else 0.0)
    for i in bad[:20]:
        loc = i % sd
        print("  idx", i, "stage", i // sd, "vel node" if loc < St.n_u else "p", loc // 2 if loc < St.n_u else loc - St.n_u, float(yt[i]), float(ys[i]))
