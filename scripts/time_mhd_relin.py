"""Time the device re-linearisation of the cfg5 hierarchy (K10g on every
level + K7g refactorisation + coarse rebuild) against the host rebuild."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2202_07381_b200 import SmootherSpec, tableau_lookup
from paper_2202_07381_b200.mhd import MHDDiscretization, MHDParams
from paper_2202_07381_b200.fem import p2_node_coords

t0 = time.perf_counter()
disc = MHDDiscretization(8, 4, MHDParams())
tab = tableau_lookup("radauiia", 2)
sm = SmootherSpec(pre=2, post=2, accel="chebyshev", cheby_a=2.0, cheby_b=8.0)
mg, S = disc.build_mg(tab, 1 / 128, sm, patch_mode="kron")
torch.cuda.synchronize()
host = time.perf_counter() - t0
xy = p2_node_coords(disc.fine_mesh)
rng = np.random.default_rng(0)
u = torch.from_numpy(rng.uniform(-1, 1, xy.shape)).cuda()
B = torch.from_numpy(rng.uniform(-1, 1, xy.shape)).cuda()
disc.relinearize(mg, u, B)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    disc.relinearize(mg, u, B)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
fine = mg.levels[-1]
asm = disc.assembler(disc.num_levels - 1, fine.system)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    asm.assemble_into_system(fine.system, u, B)
e1.record(); torch.cuda.synchronize()
k10 = e0.elapsed_time(e1) / 10
e0.record()
for _ in range(10):
    fine.patches.factor()
e1.record(); torch.cuda.synchronize()
k7 = e0.elapsed_time(e1) / 10
print(f"host build (disc + build_mg): {host:.2f} s; device relinearize: "
      f"median {1e3 * sorted(ts)[2]:.1f} ms; fine K10g {k10:.3f} ms, fine K7g {k7:.3f} ms")
