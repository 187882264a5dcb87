"""Generate the golden fixtures by running the REFERENCE package itself.

Runs only in the build container (it imports /root/reference/pkg/src);
the committed .npz / .json outputs travel, this script's inputs do not.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py          # small cases
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py --full   # cfg1-3 FGMRES counts

Cases (BASELINE.json configs on the diagonal-split grids of SURVEY.md F1,
plus the reference's own crossed-grid two-level fixture):
  cfg1     32x32 diag, RadauIIA(2), dt=1/32, 3 levels, seed 0  (BASELINE config 1, full size)
  s3       32x32 diag, RadauIIA(3), dt=1/256, 3 levels, seed 1 (config-2 scheme, reduced grid)
  ns       32x32 diag, Gauss(2), dt=1/512, mu=0.01, frozen Oseen convection, 3 levels, seed 2
           (config-3 scheme, reduced grid), Chebyshev a=1.5
  crossed  crossed n0=2, 1 refinement, RadauIIA(2), dt=0.1, seed 10 (test_solvers.py:246-251)
The reference's own RHS pattern with BASELINE uniform draws.
"""

import hashlib
import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.dont_write_bytecode = True

import irkmg.bench as rbench  # noqa: E402
import irkmg.fem as rfem  # noqa: E402
import irkmg.mesh as rmesh  # noqa: E402
from irkmg.solvers import MGHierarchyOp, SmootherSpec, apply_vanka, fgmres  # noqa: E402
from irkmg.tableaux import tableau_lookup  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def diag_grid(n):
    j, i = np.divmod(np.arange(n * n), n)
    v00 = j * (n + 1) + i
    v10, v01 = v00 + 1, v00 + n + 1
    v11 = v01 + 1
    cells = np.empty((2 * n * n, 3), dtype=np.int64)
    cells[0::2] = np.column_stack([v00, v10, v11])
    cells[1::2] = np.column_stack([v00, v11, v01])
    t = np.linspace(0.0, 1.0, n + 1)
    pts = np.column_stack([np.tile(t, n + 1), np.repeat(t, n + 1)])
    return rmesh.Mesh2D(pts, cells)


def diag_hierarchy(n0, l):
    levels = [diag_grid(n0)]
    pe, cp = [], []
    for _ in range(l):
        f, e, c = rmesh.refine_uniform(levels[-1])
        levels.append(f)
        pe.append(e)
        cp.append(c)
    return rmesh.MeshHierarchy(tuple(levels), tuple(pe), tuple(cp))


def make_disc(n0, level, mu, grid):
    if grid == "crossed":
        return rbench.Discretization(n0, level, mu=mu)
    saved = rbench.meshmod.build_hierarchy
    rbench.meshmod.build_hierarchy = diag_hierarchy
    try:
        return rbench.Discretization(n0, level, mu=mu)
    finally:
        rbench.meshmod.build_hierarchy = saved


def oseen(disc, stages):
    def w(points):
        x, y = points[:, 0], points[:, 1]
        sx, sy = np.sin(np.pi * x), np.sin(np.pi * y)
        return np.column_stack([sx * sx * np.sin(2 * np.pi * y), -np.sin(2 * np.pi * x) * sy * sy])
    conv = []
    for k in range(disc.num_levels):
        wl = rfem.interpolate(disc.vel[k], w)
        _, J = rfem.assemble_convection(disc.hier.levels[k], disc.vel[k], wl, need="jacobian")
        conv.append([J] * stages)
    return conv


class PoUHierarchy(MGHierarchyOp):
    """Reference V-cycle with the BASELINE smoother: stationary
    x += 0.5 W sum R_i^T A_i^-1 R_i (b - A x), W = 1/multiplicity."""

    omega = 0.5

    def _smooth(self, lev, x, b, sweeps):
        if not hasattr(lev, "_w"):
            n = lev.system.dim
            mult = np.zeros(n)
            for idx, _ in lev.patches.groups:
                mult += np.bincount(idx.ravel(), minlength=n)
            lev._w = np.where(mult > 0, 1.0 / np.maximum(mult, 1.0), 0.0)
        for _ in range(sweeps):
            x = x + self.omega * lev._w * lev.patches.solve_additive(b - lev.system.matvec(x))
        return x


def pou_hier(mg):
    return PoUHierarchy(mg.levels, mg.coarse)


def rhs(system, seed):
    b = np.random.default_rng(seed).uniform(-1.0, 1.0, system.dim)
    b[system.constrained_stage_dofs()] = 0.0
    return system.project_pressure_means(b)


def index_digest(patches):
    h = hashlib.sha256()
    for ix in patches.patch_indices:
        h.update(np.asarray(ix, dtype=np.int64).tobytes())
        h.update(b"|")
    return h.hexdigest()


class Tracer:
    """Record per-level intermediates of one reference V-cycle."""

    def __init__(self, mg):
        self.mg = mg
        self.items = {}

    def run(self, r):
        mg = self.mg
        orig_vcycle = mg.vcycle
        orig_coarse = mg.coarse.solve
        items = self.items

        def coarse_solve(b):
            out = orig_coarse(b)
            items["coarse_in"] = b.copy()
            items["coarse_out"] = out.copy()
            return out

        def vcycle(level, x, b):
            if level == 0:
                return mg.coarse.solve(b)
            lev = mg.levels[level]
            below = mg.levels[level - 1].system
            x = mg._smooth(lev, x, b, lev.smoother.pre)
            items[f"pre_{level}"] = x.copy()
            rr = b - lev.system.matvec(x)
            rc = lev.prolong.T @ rr
            rc[below.constrained_stage_dofs()] = 0.0
            items[f"rc_{level}"] = rc.copy()
            ec = vcycle(level - 1, np.zeros_like(rc), rc)
            corr = lev.prolong @ ec
            corr[lev.system.constrained_stage_dofs()] = 0.0
            x = x + corr
            x = mg._smooth(lev, x, b, lev.smoother.post)
            items[f"post_{level}"] = x.copy()
            return x

        mg.vcycle = vcycle
        mg.coarse.solve = coarse_solve
        try:
            z = mg.precondition(r)
        finally:
            mg.vcycle = orig_vcycle
            mg.coarse.solve = orig_coarse
        return z


CASES = {
    "cfg1": dict(grid="diagonal", n0=8, level=2, mu=1.0, family="radauiia", stages=2,
                 dt=1 / 32, seed=0, cheby_a=2.0, conv=False),
    "s3": dict(grid="diagonal", n0=8, level=2, mu=1.0, family="radauiia", stages=3,
               dt=1 / 256, seed=1, cheby_a=2.0, conv=False),
    "ns": dict(grid="diagonal", n0=8, level=2, mu=0.01, family="gauss", stages=2,
               dt=1 / 512, seed=2, cheby_a=1.5, conv=True),
    "crossed": dict(grid="crossed", n0=2, level=1, mu=1.0, family="radauiia", stages=2,
                    dt=0.1, seed=10, cheby_a=2.0, conv=False),
}

FULL = {
    "cfg1": dict(grid="diagonal", n0=8, level=2, mu=1.0, family="radauiia", stages=2,
                 dt=1 / 32, seed=0, cheby_a=2.0, conv=False),
    "cfg2": dict(grid="diagonal", n0=8, level=5, mu=1.0, family="radauiia", stages=3,
                 dt=1 / 256, seed=1, cheby_a=2.0, conv=False),
    "cfg3": dict(grid="diagonal", n0=8, level=6, mu=0.01, family="gauss", stages=2,
                 dt=1 / 512, seed=2, cheby_a=1.5, conv=True),
}


def build(case):
    disc = make_disc(case["n0"], case["level"], case["mu"], case["grid"])
    tab = tableau_lookup(case["family"], case["stages"])
    sm = SmootherSpec(pre=2, post=2, accel="chebyshev", cheby_a=case["cheby_a"], cheby_b=8.0)
    conv = oseen(disc, case["stages"]) if case["conv"] else None
    mg, system = disc.build_mg(tab, case["dt"], sm, convection=conv)
    return disc, tab, mg, system


def small_case(name, case):
    t0 = time.perf_counter()
    disc, tab, mg, S = build(case)
    fine = mg.levels[-1]
    seed = case["seed"]
    b = rhs(S, seed)
    rng = np.random.default_rng(seed + 100)
    xr = rng.uniform(-1.0, 1.0, S.dim)
    xr[S.constrained_stage_dofs()] = 0.0
    out = {"b": b, "x_rand": xr, "matvec_xr": S.matvec(xr)}
    out["sweep0"] = apply_vanka(fine.patches, S, np.zeros(S.dim), b, omega=0.5)
    out["sweep_rand"] = apply_vanka(fine.patches, S, xr, b, omega=0.5)
    out["solve_additive_b"] = fine.patches.solve_additive(b)
    pmg = pou_hier(mg)
    pmg._smooth(fine, np.zeros(S.dim), b, 0)  # builds the weights
    w = fine._w
    out["pou_w"] = w
    out["sweep_pou"] = np.zeros(S.dim) + 0.5 * w * fine.patches.solve_additive(b)
    tr = Tracer(mg)
    out["precond_cheb"] = tr.run(b.copy())
    for k, v in tr.items.items():
        out["cheb_" + k] = v
    trp = Tracer(pmg)
    out["precond_pou"] = trp.run(b.copy())
    for k, v in trp.items.items():
        out["pou_" + k] = v
    _, st_c = fgmres(S.matvec, b, precond=mg.precondition, rtol=1e-8, maxiter=200, restart=50)
    _, st_p = fgmres(S.matvec, b, precond=pmg.precondition, rtol=1e-8, maxiter=200, restart=50)
    out["fgmres_norms_cheb"] = np.array(st_c.residual_norms)
    out["fgmres_norms_pou"] = np.array(st_p.residual_norms)
    meta = {
        "case": case, "dim": int(S.dim), "n_u": int(S.n_u), "n_p": int(S.n_p),
        "fgmres_its_cheb": st_c.iterations, "fgmres_its_pou": st_p.iterations,
        "patch_index_sha256": [index_digest(l.patches) for l in mg.levels],
        "patch_sizes": [{str(int(m)): int(c) for m, c in zip(*np.unique(
            [len(ix) for ix in l.patches.patch_indices], return_counts=True))} for l in mg.levels],
        "seconds": time.perf_counter() - t0,
    }
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **out)
    with open(os.path.join(OUT, f"{name}.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print(name, meta["fgmres_its_cheb"], meta["fgmres_its_pou"], f"{meta['seconds']:.1f}s",
          flush=True)


def assembly_golden():
    """Reference M, K, B, J and prolongations on a 2-level 2x2 diagonal hierarchy."""
    out = {}
    for grid in ("diagonal", "crossed"):
        disc = make_disc(2, 1, 0.7, grid)
        m = disc.hier.levels[1]
        blk = disc.blocks[1]
        u = np.random.default_rng(5).standard_normal(blk.n_u)
        N, J = rfem.assemble_convection(m, disc.vel[1], u, need="both")
        out[f"{grid}_N"] = N
        for name, A in (("M", blk.M), ("K", blk.K), ("B", blk.B), ("J", J),
                        ("P2", rfem.prolongation(disc.hier, 0, "p2")),
                        ("P1", rfem.prolongation(disc.hier, 0, "p1"))):
            out[f"{grid}_{name}"] = A.toarray()
        out[f"{grid}_u"] = u
        out[f"{grid}_cdofs"] = rfem.velocity_boundary_dofs(m)
    np.savez_compressed(os.path.join(OUT, "assembly.npz"), **out)


def full_counts():
    res = {}
    path = os.path.join(OUT, "full_counts.json")
    if os.path.exists(path):
        res = json.load(open(path))
    for name, case in FULL.items():
        if name in res:
            continue
        t0 = time.perf_counter()
        disc, tab, mg, S = build(case)
        t_setup = time.perf_counter() - t0
        b = rhs(S, case["seed"])
        t0 = time.perf_counter()
        _, st_c = fgmres(S.matvec, b, precond=mg.precondition, rtol=1e-8, maxiter=200, restart=50)
        t_c = time.perf_counter() - t0
        t0 = time.perf_counter()
        _, st_p = fgmres(S.matvec, b, precond=pou_hier(mg).precondition, rtol=1e-8, maxiter=200,
                         restart=50)
        t_p = time.perf_counter() - t0
        res[name] = {"dim": int(S.dim), "fgmres_its_cheb": st_c.iterations,
                     "fgmres_its_pou": st_p.iterations, "setup_s": t_setup,
                     "solve_cheb_s": t_c, "solve_pou_s": t_p,
                     "final_rel_cheb": st_c.relative_residual,
                     "final_rel_pou": st_p.relative_residual,
                     "patch_index_sha256_fine": index_digest(mg.levels[-1].patches),
                     "nproc": os.cpu_count()}
        print(name, res[name], flush=True)
        with open(path, "w") as fh:
            json.dump(res, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    if "--full" in sys.argv:
        full_counts()
    else:
        assembly_golden()
        for name, case in CASES.items():
            small_case(name, case)
