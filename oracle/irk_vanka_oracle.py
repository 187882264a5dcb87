"""CPU ORACLE for the IRK-Vanka hot path -- TEST INFRASTRUCTURE ONLY.

A plain numpy/scipy restatement of the reference ``irkmg`` algorithm on
the relaxation / cycle path, used as the checker for the CUDA path.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg
(``cpu_baseline`` and ``--impl reference``) may import it; the product
package never does.

Pinning: the oracle is checked against golden vectors produced by running
the reference package itself (``tests/golden/make_golden.py`` imports
/root/reference/pkg/src in the build container) on the BASELINE-shaped
diagonal-grid configurations: ``tests/test_oracle_golden.py``.

The reference's arithmetic lives in third-party numerics absent from
/root/reference (numpy >= 1.24 ``einsum``/``bincount``/``linalg.inv``,
scipy >= 1.10 CSR matvec and SuperLU ``splu``; unpinned in
pkg/pyproject.toml:5-10).  This restatement calls the same published
routines (here numpy 2.3.5, scipy 1.18.1).

Every function cites the reference file:line it restates (paths relative
to /root/reference/pkg/src/irkmg/).
"""

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

__all__ = [
    "OracleStageOperator",
    "oracle_patch_indices",
    "OraclePatches",
    "oracle_apply_vanka",
    "oracle_chebyshev",
    "OracleCoarse",
    "OracleMG",
    "oracle_fgmres",
    "random_rhs",
]


def _eliminate(A, idx, square):
    """D A D (square) or D A (fem.py:304-315, unit_diagonal=False)."""
    mask = np.ones(A.shape[0])
    mask[idx] = 0.0
    D = sp.diags(mask)
    return (D @ A @ D).tocsr() if square else (D @ A).tocsr()


class OracleStageOperator:
    """Eliminated stage operator (stages.py:63-126).

    ``M, K, B`` are the raw vector-P2 CSR blocks (n_u x n_u, n_u x n_p),
    ``convection`` an optional list of s raw vector Jacobians."""

    def __init__(self, M, K, B, A, dt, constrained, convection=None):
        self.A = np.asarray(A, dtype=float)
        self.r = len(self.A)
        self.dt = float(dt)
        self.n_u, self.n_p = B.shape
        self.constrained = np.asarray(constrained, dtype=np.int64)
        c = self.constrained
        self.M = _eliminate(sp.csr_matrix(M), c, True)
        self.K = _eliminate(sp.csr_matrix(K), c, True)
        self.B = _eliminate(sp.csr_matrix(B), c, False)
        self.BT = self.B.T.tocsr()
        self.convection = None
        if convection is not None:
            self.convection = [_eliminate(sp.csr_matrix(J), c, True) for J in convection]
        self._cmask = np.zeros(self.n_u, dtype=bool)
        self._cmask[c] = True

    @property
    def stage_dim(self):
        return self.n_u + self.n_p

    @property
    def dim(self):
        return self.r * self.stage_dim

    def split(self, x):
        b = np.asarray(x).reshape(self.r, self.stage_dim)
        return b[:, :self.n_u], b[:, self.n_u:]

    def matvec(self, x):
        """stages.py:110-126."""
        u, p = self.split(x)
        A = self.A
        Ku = np.stack([self.K @ u[j] for j in range(self.r)])
        Bp = np.stack([self.B @ p[j] for j in range(self.r)])
        yu = np.stack([self.M @ u[i] for i in range(self.r)])
        yu += self.dt * (A @ (Ku + Bp))
        if self.convection is not None:
            for i in range(self.r):
                yu[i] += self.dt * (self.convection[i] @ (A[i] @ u))
        yu[:, self._cmask] = u[:, self._cmask]
        yp = self.dt * (A @ np.stack([self.BT @ u[j] for j in range(self.r)]))
        return np.hstack([yu, yp]).ravel()

    def constrained_stage_dofs(self):
        """stages.py:169-172."""
        offs = np.arange(self.r) * self.stage_dim
        return (offs[:, None] + self.constrained[None, :]).ravel()

    def project_pressure_means(self, x):
        """stages.py:174-178 (in place, returns x)."""
        _, p = self.split(x)
        p -= p.mean(axis=1, keepdims=True)
        return x

    def pressure_nullspace(self):
        """stages.py:180-186."""
        Z = np.zeros((self.dim, self.r))
        for i in range(self.r):
            lo = i * self.stage_dim + self.n_u
            Z[lo:lo + self.n_p, i] = 1.0 / np.sqrt(self.n_p)
        return Z

    def materialize(self):
        """stages.py:139-167 (eliminated)."""
        saddle = sp.bmat([[self.K, self.B], [self.BT, None]], format="csr")
        massd = sp.block_diag([self.M, sp.csr_matrix((self.n_p, self.n_p))], format="csr")
        out = (sp.kron(sp.identity(self.r), massd) + self.dt * sp.kron(self.A, saddle)).tolil()
        if self.convection is not None:
            sd = self.stage_dim
            for i in range(self.r):
                for j in range(self.r):
                    out[i * sd:i * sd + self.n_u, j * sd:j * sd + self.n_u] += \
                        self.dt * self.A[i, j] * self.convection[i]
        out = out.tocsr()
        ones = np.zeros(self.dim)
        ones[self.constrained_stage_dofs()] = 1.0
        return (out + sp.diags(ones)).tocsr()


def oracle_patch_indices(cells, cell_to_edges, num_vertices, op, ncomp=2):
    """Per-vertex patch index lists (solvers.py:132-166), loop form
    (``ncomp`` = 3 for the 3-D tetrahedral extension)."""
    V = num_vertices
    cell_nodes = np.hstack([cells, V + cell_to_edges])
    closure = [set() for _ in range(V)]
    for c in range(len(cells)):
        for v in cells[c]:
            closure[v].update(int(n) for n in cell_nodes[c])
    cmask = np.zeros(op.n_u, dtype=bool)
    cmask[op.constrained] = True
    sd, n_u = op.stage_dim, op.n_u
    vels, idxs = [], []
    for v in range(V):
        sn = np.array(sorted(closure[v]), dtype=np.int64)
        vel = np.empty(ncomp * len(sn), dtype=np.int64)
        for d in range(ncomp):
            vel[d::ncomp] = ncomp * sn + d
        vel = vel[~cmask[vel]]
        vels.append(vel)
        idxs.append(np.concatenate([np.concatenate([s * sd + vel, [s * sd + n_u + v]])
                                    for s in range(op.r)]))
    return vels, idxs


class OraclePatches:
    """Grouped patch inverses and the additive solve (solvers.py:169-222).

    ``members``: restrict to a subset of vertices (a bounded sample for
    timing or spot checks); default all."""

    def __init__(self, op, vels, idxs, members=None):
        self.op = op
        sizes = np.array([len(ix) for ix in idxs])
        allowed = np.ones(len(idxs), dtype=bool)
        if members is not None:
            allowed[:] = False
            allowed[np.asarray(members)] = True
        self.groups = []
        self.members = []
        for m in np.unique(sizes[allowed]):
            mem = np.flatnonzero((sizes == m) & allowed)
            idx = np.stack([idxs[p] for p in mem])
            mats = self.patch_matrices(op, [vels[p] for p in mem], mem)
            self.groups.append((idx, np.linalg.inv(mats)))
            self.members.append(mem)

    @staticmethod
    def patch_matrices(op, vels, verts):
        """Dense stage-coupled patch matrices (solvers.py:186-212)."""
        A, dt, r = op.A, op.dt, op.r
        m = len(vels[0])
        d = r * (m + 1)
        mats = np.zeros((len(vels), d, d))
        for q, (vel, v) in enumerate(zip(vels, verts)):
            Ml = op.M[vel][:, vel].toarray()
            Kl = op.K[vel][:, vel].toarray()
            bcol = op.B[vel][:, [v]].toarray().ravel()
            Cl = None
            if op.convection is not None:
                Cl = [op.convection[i][vel][:, vel].toarray() for i in range(r)]
            for i in range(r):
                for j in range(r):
                    Kij = dt * A[i, j] * Kl
                    if Cl is not None:
                        Kij = Kij + dt * A[i, j] * Cl[i]
                    if i == j:
                        Kij = Kij + Ml
                    r0, c0 = i * (m + 1), j * (m + 1)
                    mats[q, r0:r0 + m, c0:c0 + m] = Kij
                    mats[q, r0:r0 + m, c0 + m] = dt * A[i, j] * bcol
                    mats[q, r0 + m, c0:c0 + m] = dt * A[i, j] * bcol
        return mats

    def solve_additive(self, resid):
        """solvers.py:214-222."""
        z = np.zeros_like(resid)
        n = len(resid)
        for idx, inv in self.groups:
            local = np.einsum("pij,pj->pi", inv, resid[idx])
            z += np.bincount(idx.ravel(), weights=local.ravel(), minlength=n)
        return z

    def multiplicity(self, n):
        mult = np.zeros(n)
        for idx, _ in self.groups:
            mult += np.bincount(idx.ravel(), minlength=n)
        return mult

    def pou_weights(self, n):
        """BASELINE partition-of-unity weights."""
        mult = self.multiplicity(n)
        return np.where(mult > 0, 1.0 / np.maximum(mult, 1.0), 0.0)


def oracle_apply_vanka(patches, op, x, b, omega, weights=None):
    """solvers.py:232-239 (+ optional PoU weight vector)."""
    z = patches.solve_additive(b - op.matvec(x))
    if weights is not None:
        z = weights * z
    return x + omega * z


def oracle_chebyshev(op_apply, precond, a, b, steps, x, rhs):
    """solvers.py:242-268."""
    if steps <= 0:
        return x
    theta = 0.5 * (b + a)
    delta = 0.5 * (b - a)
    sigma1 = theta / delta
    rho = 1.0 / sigma1
    x = x.copy()
    r = rhs - op_apply(x)
    z = precond(r)
    d = z / theta
    for _ in range(1, steps):
        x += d
        r = r - op_apply(d)
        z = precond(r)
        rho_new = 1.0 / (2.0 * sigma1 - rho)
        d = rho_new * rho * d + (2.0 * rho_new / delta) * z
        rho = rho_new
    return x + d


class OracleCoarse:
    """splu(A + Z Z^T) and the projected solve (solvers.py:271-287)."""

    def __init__(self, op):
        A = op.materialize()
        Z = op.pressure_nullspace()
        self.lu = spla.splu((A + sp.csr_matrix(Z @ Z.T)).tocsc())
        self.Z = Z

    def solve(self, b):
        b = b - self.Z @ (self.Z.T @ b)
        x = self.lu.solve(b)
        return x - self.Z @ (self.Z.T @ x)


class OracleMG:
    """V-cycle / precondition (solvers.py:303-356).

    levels: list (coarsest first) of dicts with keys ``op``, ``patches``,
    ``prolong`` (scipy stage prolongation from the level below, or None).
    smoother: dict(pre, post, accel in {"chebyshev","richardson","gmres"},
    a, b, omega, weights in {None, "pou"})."""

    def __init__(self, levels, smoother, coarse=None):
        self.levels = levels
        self.sm = dict(smoother)
        self.coarse = coarse if coarse is not None else OracleCoarse(levels[0]["op"])
        self.coarse_hook = None  # optional override: f(level0_rhs) -> solution

    def _smooth(self, lev, x, b, sweeps):
        if sweeps == 0:
            return x
        op, pat, sm = lev["op"], lev["patches"], self.sm
        w = pat.pou_weights(op.dim) if sm.get("weights") == "pou" else None

        def precond(r):
            z = sm["omega"] * pat.solve_additive(r)
            return z if w is None else w * z

        if sm["accel"] == "chebyshev":
            return oracle_chebyshev(op.matvec, precond, sm["a"], sm["b"], sweeps, x, b)
        if sm["accel"] == "richardson":
            for _ in range(sweeps):
                x = x + precond(b - op.matvec(x))
            return x
        x, _ = oracle_fgmres(op.matvec, b, precond=precond, x0=x, rtol=0.0, atol=0.0,
                             maxiter=sweeps, restart=sweeps)
        return x

    def vcycle(self, level, x, b, trace=None):
        """solvers.py:334-347; ``trace`` (a list) collects intermediates."""
        if level == 0:
            out = self.coarse.solve(b) if self.coarse_hook is None else self.coarse_hook(b)
            if trace is not None:
                trace.append(("coarse_in", b.copy()))
                trace.append(("coarse_out", out.copy()))
            return out
        lev = self.levels[level]
        below = self.levels[level - 1]["op"]
        x = self._smooth(lev, x, b, self.sm["pre"])
        r = b - lev["op"].matvec(x)
        rc = lev["prolong"].T @ r
        rc[below.constrained_stage_dofs()] = 0.0
        if trace is not None:
            trace.append((f"pre_{level}", x.copy()))
            trace.append((f"rc_{level}", rc.copy()))
        ec = self.vcycle(level - 1, np.zeros_like(rc), rc, trace)
        corr = lev["prolong"] @ ec
        corr[lev["op"].constrained_stage_dofs()] = 0.0
        x = x + corr
        x = self._smooth(lev, x, b, self.sm["post"])
        if trace is not None:
            trace.append((f"post_{level}", x.copy()))
        return x

    def precondition(self, r, trace=None):
        """solvers.py:349-356."""
        op = self.levels[-1]["op"]
        z = np.zeros_like(r)
        cd = op.constrained_stage_dofs()
        z[cd] = r[cd]
        z = self.vcycle(len(self.levels) - 1, z, r, trace)
        return op.project_pressure_means(z)


def oracle_fgmres(op_apply, b, precond=None, x0=None, rtol=1e-8, atol=0.0, maxiter=100,
                  restart=30):
    """Flexible GMRES (solvers.py:364-443). Returns (x, iterations, norms, converged)."""
    n = len(b)
    x = np.zeros(n) if x0 is None else np.asarray(x0, dtype=float).copy()
    if precond is None:
        precond = lambda v: v
    its = 0
    norms = []
    r = b - op_apply(x)
    norm0 = np.linalg.norm(r)
    norms.append(norm0)
    tol = max(rtol * norm0, atol)
    if norm0 <= tol:
        return x, (0, norms, True)
    while its < maxiter:
        m = min(restart, maxiter - its)
        V = np.zeros((m + 1, n))
        Z = np.zeros((m, n))
        H = np.zeros((m + 1, m))
        cs = np.zeros(m)
        sn = np.zeros(m)
        g = np.zeros(m + 1)
        beta = np.linalg.norm(r)
        V[0] = r / beta
        g[0] = beta
        k = 0
        for j in range(m):
            Z[j] = precond(V[j])
            w = np.array(op_apply(Z[j]), dtype=float)
            for i in range(j + 1):
                H[i, j] = w @ V[i]
                w -= H[i, j] * V[i]
            H[j + 1, j] = np.linalg.norm(w)
            if H[j + 1, j] > 1e-300:
                V[j + 1] = w / H[j + 1, j]
            for i in range(j):
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            denom = np.hypot(H[j, j], H[j + 1, j])
            cs[j] = H[j, j] / denom
            sn[j] = H[j + 1, j] / denom
            H[j, j] = denom
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            k = j + 1
            its += 1
            est = abs(g[j + 1])
            norms.append(est)
            if est <= tol or its >= maxiter:
                break
        y = np.linalg.solve(np.triu(H[:k, :k]), g[:k])
        x = x + y @ Z[:k]
        r = b - op_apply(x)
        norms[-1] = np.linalg.norm(r)
        if norms[-1] <= tol:
            break
    final = float(np.linalg.norm(b - op_apply(x)))
    return x, (its, list(np.minimum.accumulate(norms)), final <= tol)


def random_rhs(op, seed):
    """BASELINE RHS convention: uniform[-1, 1], constrained
    entries zeroed, per-stage pressure mean removed."""
    b = np.random.default_rng(seed).uniform(-1.0, 1.0, op.dim)
    b[op.constrained_stage_dofs()] = 0.0
    return op.project_pressure_means(b)
