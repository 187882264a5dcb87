"""CPU ORACLE for the general (multi-field) IRK-Vanka path -- TEST
INFRASTRUCTURE ONLY (tests/, smoke(), bench.py's CPU legs).

PARITY UNPINNED: the reference package implements Stokes / Navier--Stokes
only; BASELINE config 5 (2-D resistive MHD) has no reference
implementation, no golden vectors and no fixture to pin against.  This
module restates the reference ALGORITHM on the general stage system
I_s (x) M + dt A (x) L, independently of the CUDA path's data structures:

* ``OracleGeneralOperator.matvec`` -- stages.py:110-126 (stage loop of
  scipy CSR products; identity rows on constrained DoFs);
* ``oracle_general_patch_indices`` -- solvers.py:132-166 in loop form over
  cells, with the paper's Vanka patch (PAPER.md "Vanka relaxation": all DoFs
  on the closure of the vertex star, P1 fields only at the vertex);
* ``OracleGeneralPatches`` -- solvers.py:169-222: dense R_i A R_i^T sliced
  from the materialised stage operator, ``np.linalg.inv`` per size group,
  einsum + bincount;
* ``oracle_mhd_apply`` -- the linearised MHD operator of mhd.py evaluated
  cell by cell with scalar loops over quadrature points (an independent
  restatement of the weak form in PAPER.md eq. "MHD semi-discrete"),
  checking the vectorised assembly.

``OracleMG`` / ``oracle_fgmres`` / ``oracle_apply_vanka`` of
irk_vanka_oracle.py run on these objects unchanged.
"""

import numpy as np
import scipy.sparse as sp

__all__ = ["OracleGeneralOperator", "oracle_general_patch_indices", "OracleGeneralPatches",
           "oracle_mhd_apply"]


class OracleGeneralOperator:
    """I_s (x) M + dt A (x) L with identity rows on constrained DoFs
    (stages.py:63-126 generalised); L, M eliminated scipy matrices."""

    def __init__(self, M, L, A, dt, constrained, pressure_offset):
        self.A = np.asarray(A, dtype=float)
        self.r = len(self.A)
        self.dt = float(dt)
        self.M = sp.csr_matrix(M)
        self.L = sp.csr_matrix(L)
        self.n1 = self.M.shape[0]
        self.constrained = np.asarray(constrained, dtype=np.int64)
        self._cmask = np.zeros(self.n1, dtype=bool)
        self._cmask[self.constrained] = True
        self.n_u = int(pressure_offset)
        self.n_p = self.n1 - self.n_u

    @property
    def stage_dim(self):
        return self.n1

    @property
    def dim(self):
        return self.r * self.n1

    def matvec(self, x):
        X = np.asarray(x).reshape(self.r, self.n1)
        LX = np.stack([self.L @ X[j] for j in range(self.r)])
        Y = np.stack([self.M @ X[i] for i in range(self.r)]) + self.dt * (self.A @ LX)
        Y[:, self._cmask] = X[:, self._cmask]
        return Y.ravel()

    def constrained_stage_dofs(self):
        offs = np.arange(self.r) * self.n1
        return (offs[:, None] + self.constrained[None, :]).ravel()

    def project_pressure_means(self, x):
        p = np.asarray(x).reshape(self.r, self.n1)[:, self.n_u:]
        p -= p.mean(axis=1, keepdims=True)
        return x

    def pressure_nullspace(self):
        Z = np.zeros((self.dim, self.r))
        for i in range(self.r):
            lo = i * self.n1 + self.n_u
            Z[lo:lo + self.n_p, i] = 1.0 / np.sqrt(self.n_p)
        return Z

    def materialize(self):
        out = sp.kron(sp.identity(self.r), self.M) + self.dt * sp.kron(self.A, self.L)
        ones = np.zeros(self.dim)
        ones[self.constrained_stage_dofs()] = 1.0
        return (out + sp.diags(ones)).tocsr()


def oracle_general_patch_indices(cells, cell_to_edges, num_vertices, op, ncomp, n_vertex_fields):
    """Per-vertex stage-major patch index lists, loop form: P2 components
    interleaved per node (ncomp per node), then ``n_vertex_fields`` P1 blocks
    of one DoF per vertex; constrained DoFs removed."""
    V = num_vertices
    cell_nodes = np.hstack([cells, V + cell_to_edges])
    n_nodes = V + int(cell_to_edges.max()) + 1
    closure = [set() for _ in range(V)]
    for c in range(len(cells)):
        for v in cells[c]:
            closure[v].update(int(n) for n in cell_nodes[c])
    idxs = []
    for v in range(V):
        single = []
        for n in sorted(closure[v]):
            single.extend(ncomp * n + d for d in range(ncomp))
        single.extend(ncomp * n_nodes + f * V + v for f in range(n_vertex_fields))
        single = np.array([d for d in single if not op._cmask[d]], dtype=np.int64)
        idxs.append(np.concatenate([s * op.n1 + single for s in range(op.r)]))
    return idxs


class OracleGeneralPatches:
    """Grouped patch inverses and the additive solve (solvers.py:169-222)."""

    def __init__(self, op, idxs, members=None):
        self.op = op
        A = op.materialize().tocsr()
        sizes = np.array([len(ix) for ix in idxs])
        allowed = np.ones(len(idxs), dtype=bool)
        if members is not None:
            allowed[:] = False
            allowed[np.asarray(members)] = True
        self.groups = []
        for m in np.unique(sizes[allowed]):
            mem = np.flatnonzero((sizes == m) & allowed)
            idx = np.stack([idxs[p] for p in mem])
            mats = np.stack([A[ix][:, ix].toarray() for ix in idx])
            self.groups.append((idx, np.linalg.inv(mats)))

    def solve_additive(self, resid, threads=1, reverse=False):
        """``threads`` is accepted for interface parity with ``OraclePatches``
        (the general oracle runs single-threaded); ``reverse`` runs groups and
        patches in the opposite order (the F9 self-floor probe)."""
        z = np.zeros_like(resid)
        n = len(resid)
        for idx, inv in (self.groups[::-1] if reverse else self.groups):
            if reverse:
                idx, inv = idx[::-1], inv[::-1]
            local = np.einsum("pij,pj->pi", inv, resid[idx])
            z += np.bincount(idx.ravel(), weights=local.ravel(), minlength=n)
        return z

    def multiplicity(self, n):
        mult = np.zeros(n)
        for idx, _ in self.groups:
            mult += np.bincount(idx.ravel(), minlength=n)
        return mult

    def pou_weights(self, n):
        mult = self.multiplicity(n)
        return np.where(mult > 0, 1.0 / np.maximum(mult, 1.0), 0.0)


# ---------------------------------------------------------------- MHD form

def _p2_local(lx, ly):
    """P2 values and reference gradients at one point (vertices, then the
    midpoint of the edge opposite vertex k)."""
    lam = [1.0 - lx - ly, lx, ly]
    dlam = [(-1.0, -1.0), (1.0, 0.0), (0.0, 1.0)]
    val, grad = [0.0] * 6, [(0.0, 0.0)] * 6
    for k in range(3):
        val[k] = lam[k] * (2.0 * lam[k] - 1.0)
        grad[k] = ((4.0 * lam[k] - 1.0) * dlam[k][0], (4.0 * lam[k] - 1.0) * dlam[k][1])
        a, b = (k + 1) % 3, (k + 2) % 3
        val[3 + k] = 4.0 * lam[a] * lam[b]
        grad[3 + k] = (4.0 * (lam[a] * dlam[b][0] + lam[b] * dlam[a][0]),
                       4.0 * (lam[a] * dlam[b][1] + lam[b] * dlam[a][1]))
    return val, grad, lam, dlam


def _strang_fix_rule():
    """Degree-6 (12-point) symmetric triangle rule (weights sum to 1/2):
    a different rule from the product (Duffy) rule the assembly uses, exact
    for the degree-5 integrands of the form."""
    out = []
    groups = [(0.063089014491502, 0.050844906370207),
              (0.249286745170910, 0.116786275726379)]
    for a, w in groups:
        b = 1.0 - 2.0 * a
        for p in ((a, a), (a, b), (b, a)):
            out.append((p[0], p[1], 0.5 * w))
    a, b, w = 0.053145049844817, 0.310352451033784, 0.082851075618374
    c = 1.0 - a - b
    for p in ((a, b), (b, a), (a, c), (c, a), (b, c), (c, b)):
        out.append((p[0], p[1], 0.5 * w))
    return out


def oracle_mhd_apply(mesh, u0, B0, Re, Rm, S, x):
    """y = L x for the unconstrained single-stage linearised MHD operator
    (layout [w | r | p], w = (u_x, u_y, B_x, B_y) per P2 node), by scalar
    loops over cells and quadrature points."""
    V = mesh.num_vertices
    n_nodes = V + mesh.num_edges
    y = np.zeros_like(x)
    rule = _strang_fix_rule()
    for c in range(mesh.num_cells):
        vid = mesh.cells[c]
        nodes = list(vid) + [V + e for e in mesh.cell_to_edges[c]]
        p0, p1, p2 = (mesh.vertices[v] for v in vid)
        J = np.array([[p1[0] - p0[0], p2[0] - p0[0]], [p1[1] - p0[1], p2[1] - p0[1]]])
        det = J[0, 0] * J[1, 1] - J[0, 1] * J[1, 0]
        Ji = np.linalg.inv(J)
        for (lx, ly, wq) in rule:
            val, gref, lam, dlam = _p2_local(lx, ly)
            g = [(gr[0] * Ji[0, 0] + gr[1] * Ji[1, 0], gr[0] * Ji[0, 1] + gr[1] * Ji[1, 1])
                 for gr in gref]
            gp = [(d[0] * Ji[0, 0] + d[1] * Ji[1, 0], d[0] * Ji[0, 1] + d[1] * Ji[1, 1])
                  for d in dlam]
            W = wq * det

            def field(vals, comp):
                return sum(vals[4 * nodes[a] + comp] * val[a] for a in range(6))

            def fgrad(vals, comp):
                return (sum(vals[4 * nodes[a] + comp] * g[a][0] for a in range(6)),
                        sum(vals[4 * nodes[a] + comp] * g[a][1] for a in range(6)))

            def state(arr, comp):
                return sum(arr[nodes[a], comp] * val[a] for a in range(6))

            def sgrad(arr, comp):
                return (sum(arr[nodes[a], comp] * g[a][0] for a in range(6)),
                        sum(arr[nodes[a], comp] * g[a][1] for a in range(6)))

            u = (field(x, 0), field(x, 1))
            B = (field(x, 2), field(x, 3))
            gu = (fgrad(x, 0), fgrad(x, 1))            # gu[d][e] = d_e u_d
            gB = (fgrad(x, 2), fgrad(x, 3))
            r = sum(x[4 * n_nodes + vid[i]] * lam[i] for i in range(3))
            gr = (sum(x[4 * n_nodes + vid[i]] * gp[i][0] for i in range(3)),
                  sum(x[4 * n_nodes + vid[i]] * gp[i][1] for i in range(3)))
            p = sum(x[4 * n_nodes + V + vid[i]] * lam[i] for i in range(3))
            U0 = (state(u0, 0), state(u0, 1))
            Bs = (state(B0, 0), state(B0, 1))
            gU0 = (sgrad(u0, 0), sgrad(u0, 1))
            gBs = (sgrad(B0, 0), sgrad(B0, 1))
            eps = [[0.5 * (gu[d][e] + gu[e][d]) for e in range(2)] for d in range(2)]
            jB = gB[1][0] - gB[0][1]
            j0 = gBs[1][0] - gBs[0][1]
            conv = [U0[0] * gu[d][0] + U0[1] * gu[d][1] + u[0] * gU0[d][0] + u[1] * gU0[d][1]
                    for d in range(2)]
            lor = [-S * (jB * (-Bs[1]) + j0 * (-B[1])), -S * (jB * Bs[0] + j0 * B[0])]
            emf = (u[0] * Bs[1] - u[1] * Bs[0]) + (U0[0] * B[1] - U0[1] * B[0])
            divu = gu[0][0] + gu[1][1]
            for a in range(6):
                n = nodes[a]
                for d in range(2):
                    # test v = phi_a e_d: eps(v)_{ke} = (delta_kd g_e + delta_ed g_k)/2
                    ev = sum(eps[d][e] * g[a][e] for e in range(2))
                    y[4 * n + d] += W * ((2.0 / Re) * ev + conv[d] * val[a] + lor[d] * val[a]
                                         - p * g[a][d])
                # test c = phi_a e_h: j(c) = (-d_y phi_a, d_x phi_a)[h]
                jc = (-g[a][1], g[a][0])
                for h in range(2):
                    y[4 * n + 2 + h] += W * ((1.0 / Rm) * jB * jc[h] - emf * jc[h]
                                             - gr[h] * val[a])
            for i in range(3):
                y[4 * n_nodes + vid[i]] += W * (-(B[0] * gp[i][0] + B[1] * gp[i][1]))
                y[4 * n_nodes + V + vid[i]] += W * (-divu * lam[i])
    return y
