"""TEST INFRASTRUCTURE ONLY (tests/ may import it; the product path never
does).  Independent cell-by-cell restatement of the 3-D Taylor-Hood P2-P1
Stokes weak form (BASELINE config 4) -- the pin for ``fem3d.assemble_blocks3d``.

The reference has no 3-D discretisation (/root/reference
SPEC.md:8,92), so there is no golden vector to pin config 4 against.  This
module recomputes the same bilinear forms by a different method, so that an
agreement to rounding level is evidence for both:

* integrals are EXACT: every integrand is a polynomial in the barycentric
  coordinates, integrated with the closed form
  ``int_T l0^a l1^b l2^c l3^d = |T| 3! a! b! c! d! / (a+b+c+d+3)!``
  (no quadrature rule, unlike ``fem3d.tet_rule``'s conical product);
* the P2 basis is built as barycentric polynomials (dicts of monomials) and
  differentiated symbolically; gradients of the barycentrics come from the
  cell's vertex coordinates by solving the 4x4 affine system per cell;
* global node identity comes from GEOMETRY: every P2 node is located by its
  coordinates (vertex or edge midpoint) in a coordinate table, not through
  the mesh's edge numbering;
* one python loop over cells, dense per-cell element matrices accumulated
  entry by entry.

Forms (the 2-D reference conventions, ``fem.py:128-196`` of the reference):
M[n, m] = int phi_n phi_m, K[n, m] = mu int grad phi_n . grad phi_m,
B[3 n + d, q] = -int psi_q d_d phi_n (psi: P1 hat functions).
"""

from itertools import product
from math import factorial

import numpy as np
import scipy.sparse as sp

__all__ = ["p2_barycentric_basis", "exact_monomial_integral", "oracle_blocks3d"]

_EDGES = [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)]


def _mono(**kw):
    e = [0, 0, 0, 0]
    for k, v in kw.items():
        e[int(k[1])] += v
    return tuple(e)


def _mul(p, q):
    out = {}
    for a, ca in p.items():
        for b, cb in q.items():
            k = tuple(x + y for x, y in zip(a, b))
            out[k] = out.get(k, 0.0) + ca * cb
    return out


def _dlam(p, k):
    """d p / d lambda_k of a barycentric polynomial."""
    out = {}
    for a, c in p.items():
        if a[k] > 0:
            b = list(a)
            b[k] -= 1
            out[tuple(b)] = out.get(tuple(b), 0.0) + c * a[k]
    return out


def p2_barycentric_basis():
    """The 10 P2 shape functions on a tetrahedron as barycentric polynomials:
    vertices l_k (2 l_k - 1), then edge midpoints 4 l_i l_j (edges (0,1),
    (0,2), (0,3), (1,2), (1,3), (2,3))."""
    basis = []
    for k in range(4):
        e2 = [0, 0, 0, 0]
        e2[k] = 2
        e1 = [0, 0, 0, 0]
        e1[k] = 1
        basis.append({tuple(e2): 2.0, tuple(e1): -1.0})
    for i, j in _EDGES:
        e = [0, 0, 0, 0]
        e[i] += 1
        e[j] += 1
        basis.append({tuple(e): 4.0})
    return basis


def exact_monomial_integral(a):
    """int over the reference-volume-normalised tet of l^a, times 1/|T|."""
    s = sum(a)
    return factorial(3) * np.prod([factorial(x) for x in a]) / factorial(s + 3)


def _integrate(p):
    return sum(c * exact_monomial_integral(a) for a, c in p.items())


def _reference_tables():
    """Cell-independent exact integrals:
    mass[n, m] = int phi_n phi_m / |T|,
    stiff[n, m, k, l] = int d_k phi_n d_l phi_m / |T|,
    div[n, q, k] = int l_q d_k phi_n / |T|."""
    phi = p2_barycentric_basis()
    dphi = [[_dlam(f, k) for k in range(4)] for f in phi]
    lam = [{tuple(int(i == q) for i in range(4)): 1.0} for q in range(4)]
    mass = np.array([[_integrate(_mul(a, b)) for b in phi] for a in phi])
    stiff = np.zeros((10, 10, 4, 4))
    for n, m, k, l in product(range(10), range(10), range(4), range(4)):
        stiff[n, m, k, l] = _integrate(_mul(dphi[n][k], dphi[m][l]))
    div = np.zeros((10, 4, 4))
    for n, q, k in product(range(10), range(4), range(4)):
        div[n, q, k] = _integrate(_mul(lam[q], dphi[n][k]))
    return mass, stiff, div


def oracle_blocks3d(vertices, cells, node_coords, mu=1.0):
    """Assemble M, mu K (n x n) and B (3n x nv) by a loop over ``cells``
    ((C, 4) vertex ids into ``vertices``).  ``node_coords`` (n, 3) gives the
    global P2 node positions; each cell's nodes are found by coordinate
    lookup.  Returns scipy CSR (M, K, B)."""
    mass, stiff, div = _reference_tables()
    key = lambda x: tuple(np.round(np.asarray(x) * (1 << 20)).astype(np.int64))  # noqa: E731
    where = {key(x): i for i, x in enumerate(node_coords)}
    n = len(node_coords)
    nv = len(vertices)
    Mr, Mc, Mv, Kv, Br, Bc, Bv = [], [], [], [], [], [], []
    for c in cells:
        P = vertices[c]                                      # (4, 3)
        # barycentric gradients: [1 x y z] rows, lambda = T^{-1} [1; x]
        T = np.vstack([np.ones(4), P.T])                     # (4, 4)
        Tinv = np.linalg.inv(T)                              # lambda_k = Tinv[k] . [1, x, y, z]
        g = Tinv[:, 1:]                                      # (4, 3): grad lambda_k
        vol = abs(np.linalg.det(T)) / 6.0
        pos = list(P) + [0.5 * (P[i] + P[j]) for i, j in _EDGES]
        nodes = [where[key(x)] for x in pos]
        G = g @ g.T                                          # grad l_k . grad l_l
        for a in range(10):
            for b in range(10):
                Mr.append(nodes[a])
                Mc.append(nodes[b])
                Mv.append(vol * mass[a, b])
                Kv.append(mu * vol * float(np.sum(stiff[a, b] * G)))
            for q in range(4):
                for d in range(3):
                    Br.append(3 * nodes[a] + d)
                    Bc.append(c[q])
                    Bv.append(-vol * float(np.dot(div[a, q], g[:, d])))
    M = sp.csr_matrix((Mv, (Mr, Mc)), shape=(n, n))
    K = sp.csr_matrix((Kv, (Mr, Mc)), shape=(n, n))
    B = sp.csr_matrix((Bv, (Br, Bc)), shape=(3 * n, nv))
    for A in (M, K, B):
        A.sum_duplicates()
    return M, K, B
