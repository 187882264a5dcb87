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


def _gather_dense(A, rows):
    """Dense submatrices A[rows_p, rows_p] for a batch of ascending index
    sets, (P, m) -> (P, m, m): one pass over the CSR arrays, each stored
    column located in its patch's sorted row set by a searchsorted over
    offset-disambiguated keys (solvers.py:33-59)."""
    A = sp.csr_matrix(A)
    P, m = rows.shape
    n = A.shape[1]
    flat = rows.ravel()
    start = A.indptr[flat]
    cnt = A.indptr[flat + 1] - start
    off = np.concatenate(([0], np.cumsum(cnt)))
    pos = np.repeat(start - off[:-1], cnt) + np.arange(off[-1])
    cols, vals = A.indices[pos], A.data[pos]
    row_of = np.repeat(np.arange(P * m), cnt)
    patch = row_of // m
    keys = (rows + np.arange(P, dtype=np.int64)[:, None] * n).ravel()
    query = cols + patch * n
    loc = np.minimum(np.searchsorted(keys, query), P * m - 1)
    hit = keys[loc] == query
    out = np.zeros((P, m, m))
    out[patch[hit], row_of[hit] % m, loc[hit] - patch[hit] * m] = vals[hit]
    return out


def _gather_columns(B, rows, col_of_patch):
    """B[rows_p, col_p] per patch, (P, m) (solvers.py:62-78)."""
    B = sp.csr_matrix(B)
    P, m = rows.shape
    flat = rows.ravel()
    start = B.indptr[flat]
    cnt = B.indptr[flat + 1] - start
    off = np.concatenate(([0], np.cumsum(cnt)))
    pos = np.repeat(start - off[:-1], cnt) + np.arange(off[-1])
    cols, vals = B.indices[pos], B.data[pos]
    row_of = np.repeat(np.arange(P * m), cnt)
    patch = row_of // m
    hit = cols == np.asarray(col_of_patch)[patch]
    out = np.zeros((P, m))
    out[patch[hit], row_of[hit] % m] = vals[hit]
    return out


def _chunks(n, k):
    cuts = [(i * n) // k for i in range(k + 1)]
    return [(a, b) for a, b in zip(cuts[:-1], cuts[1:]) if b > a]


def _pool_map(fn, items, threads):
    """Map over host threads with BLAS pinned to one thread each (numpy's
    batched LAPACK / einsum release the GIL; nested OpenBLAS threading in
    every worker would oversubscribe the cores)."""
    if threads <= 1 or len(items) <= 1:
        return [fn(it) for it in items]
    from concurrent.futures import ThreadPoolExecutor
    from threadpoolctl import threadpool_limits
    with threadpool_limits(1), ThreadPoolExecutor(threads) as ex:
        return list(ex.map(fn, items))


class OraclePatches:
    """Grouped patch inverses and the additive solve (solvers.py:169-222).

    ``members``: restrict to a subset of vertices (a bounded sample for
    timing or spot checks); default all.  ``threads``: host threads for the
    batched ``np.linalg.inv`` of each size group (the reference calls it on
    the whole group at once; splitting the batch does not change any
    patch's inverse)."""

    def __init__(self, op, vels, idxs, members=None, threads=1):
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
            vel = np.stack([vels[p] for p in mem])
            d = len(idx[0])
            inv = np.empty((len(mem), d, d))
            parts = _chunks(len(mem), max(1, len(mem) // 1024))

            def work(ab, mem=mem, vel=vel, inv=inv):
                # gather + inversion of one slice of the group: every patch's
                # matrix and inverse are the same as the whole-group call's
                a, b = ab
                inv[a:b] = np.linalg.inv(self.patch_matrices(op, vel[a:b], mem[a:b]))
            _pool_map(work, parts, threads)
            self.groups.append((idx, inv))
            self.members.append(mem)

    @staticmethod
    def patch_matrices(op, vels, verts):
        """Dense stage-coupled patch matrices of one size group
        (solvers.py:186-212): per stage block (i, j)
        [M d_ij + dt a_ij (K + C_i) | dt a_ij b] over [dt a_ij b^T | 0]."""
        A, dt, r = op.A, op.dt, op.r
        vel = np.stack([np.asarray(v, dtype=np.int64) for v in vels])
        P, m = vel.shape
        Ml = _gather_dense(op.M, vel)
        Kl = _gather_dense(op.K, vel)
        bcol = _gather_columns(op.B, vel, np.asarray(verts))
        Cl = None
        if op.convection is not None:
            Cl = [_gather_dense(op.convection[i], vel) for i in range(r)]
        d = r * (m + 1)
        mats = np.zeros((P, d, d))
        for i in range(r):
            for j in range(r):
                Kij = dt * A[i, j] * Kl
                if Cl is not None:
                    Kij = Kij + dt * A[i, j] * Cl[i]
                if i == j:
                    Kij = Kij + Ml
                r0, c0 = i * (m + 1), j * (m + 1)
                mats[:, r0:r0 + m, c0:c0 + m] = Kij
                mats[:, r0:r0 + m, c0 + m] = dt * A[i, j] * bcol
                mats[:, r0 + m, c0:c0 + m] = dt * A[i, j] * bcol
        return mats

    def solve_additive(self, resid, threads=1, reverse=False):
        """solvers.py:214-222: per size group einsum("pij,pj->pi") and a
        bincount scatter, groups summed in order.  ``threads`` > 1 splits each
        group's patches into chunks whose bincounts are added in chunk order
        (a different, fixed summation order: ~1e-16 relative).  ``reverse``
        runs the groups and the patches inside each group in the opposite
        order -- the reference's self-floor probe."""
        z = np.zeros_like(resid)
        n = len(resid)
        groups = self.groups[::-1] if reverse else self.groups
        for idx, inv in groups:
            if reverse:
                idx, inv = idx[::-1], inv[::-1]
            if threads <= 1:
                local = np.einsum("pij,pj->pi", inv, resid[idx])
                z += np.bincount(idx.ravel(), weights=local.ravel(), minlength=n)
                continue

            def part(ab, idx=idx, inv=inv):
                ix = idx[ab[0]:ab[1]]
                loc = np.einsum("pij,pj->pi", inv[ab[0]:ab[1]], resid[ix])
                return np.bincount(ix.ravel(), weights=loc.ravel(), minlength=n)
            for zz in _pool_map(part, _chunks(len(idx), max(1, min(threads, len(idx) // 16))),
                                threads):
                z += zz
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


def oracle_apply_vanka(patches, op, x, b, omega, weights=None, threads=1):
    """solvers.py:232-239 (+ optional PoU weight vector)."""
    z = patches.solve_additive(b - op.matvec(x), threads=threads)
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
    a, b, omega, weights in {None, "pou"}).  ``threads`` / ``reverse`` are
    passed to every ``solve_additive`` (reverse = the F9 self-floor probe)."""

    def __init__(self, levels, smoother, coarse=None, threads=1, reverse=False):
        self.levels = levels
        self.sm = dict(smoother)
        self.coarse = coarse if coarse is not None else OracleCoarse(levels[0]["op"])
        self.coarse_hook = None  # optional override: f(level0_rhs) -> solution
        self.threads = threads
        self.reverse = reverse
        self._w = {}

    def _smooth(self, lev, x, b, sweeps):
        if sweeps == 0:
            return x
        op, pat, sm = lev["op"], lev["patches"], self.sm
        w = None
        if sm.get("weights") == "pou":
            if id(pat) not in self._w:
                self._w[id(pat)] = pat.pou_weights(op.dim)
            w = self._w[id(pat)]

        def precond(r):
            z = sm["omega"] * pat.solve_additive(r, threads=self.threads, reverse=self.reverse)
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
