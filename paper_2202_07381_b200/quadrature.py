"""Reference-triangle quadrature and Lagrange bases (host-side setup).

The rule is the collapsed (Duffy) product of an n-point Gauss-Legendre
rule in the collapsed coordinate and an n-point Gauss-Jacobi(1, 0) rule in
the other, n = max(1, (degree + 2) // 2); it integrates every polynomial of
total degree ``degree`` exactly.  The same construction (and the same
SciPy node generators) as the reference ``quadrature.py:18-44`` is used so
that assembled matrices agree with the reference to rounding.
"""

from functools import lru_cache

import numpy as np
from scipy.special import roots_jacobi, roots_legendre

__all__ = ["triangle_rule", "p1_basis", "p2_basis"]


@lru_cache(maxsize=None)
def triangle_rule(degree):
    """(points (Q, 2), weights (Q,)) on {x, y >= 0, x + y <= 1}."""
    if degree < 0:
        raise ValueError("quadrature degree must be >= 0")
    n = max(1, (degree + 2) // 2)
    gl_x, gl_w = roots_legendre(n)
    gj_x, gj_w = roots_jacobi(n, 1, 0)
    s = 0.5 * (gl_x + 1.0)          # collapsed coordinate in [0, 1]
    ws = 0.5 * gl_w
    t = 0.5 * (gj_x + 1.0)          # y in [0, 1], weight (1 - t) built in
    wt = 0.25 * gj_w
    x = (s[:, None] * (1.0 - t[None, :])).ravel()
    y = np.broadcast_to(t[None, :], (n, n)).ravel()
    w = (ws[:, None] * wt[None, :]).ravel()
    pts = np.column_stack([x, y])
    pts.setflags(write=False)
    w.setflags(write=False)
    return pts, w


def _barycentric(points):
    x, y = points[:, 0], points[:, 1]
    lam = np.stack([1.0 - x - y, x, y])
    dlam = np.array([[-1.0, -1.0], [1.0, 0.0], [0.0, 1.0]])
    return lam, dlam


def p1_basis(points):
    """P1 values (3, Q) and constant gradients (3, 2)."""
    lam, dlam = _barycentric(points)
    return lam, dlam


def p2_basis(points):
    """P2 values (6, Q) and gradients (6, Q, 2).

    Nodes: the three vertices, then the midpoint of the edge opposite
    vertex k for k = 0, 1, 2 (the numbering behind ``cell_to_edges``).
    """
    lam, dlam = _barycentric(points)
    q = lam.shape[1]
    phi = np.empty((6, q))
    dphi = np.empty((6, q, 2))
    for k in range(3):
        phi[k] = lam[k] * (2.0 * lam[k] - 1.0)
        dphi[k] = (4.0 * lam[k] - 1.0)[:, None] * dlam[k]
        a, b = (k + 1) % 3, (k + 2) % 3
        phi[3 + k] = 4.0 * lam[a] * lam[b]
        dphi[3 + k] = 4.0 * (lam[a][:, None] * dlam[b] + lam[b][:, None] * dlam[a])
    return phi, dphi
