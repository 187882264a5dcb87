"""Modal split of Stokes patches (modal.py, K3m's algebra) on CPU: the
record's apply equals the inverse of the stage-coupled patch matrix
(solvers.py:186-212) for every tableau family, including non-diagonalisable
ones, and patch sizes of 2-D and 3-D Taylor-Hood stars."""

import numpy as np
import pytest

from paper_2202_07381_b200 import tableau_lookup
from paper_2202_07381_b200.modal import ModalSplit


def patch_matrix(Ms, Ks, c, A, dt, nc):
    """[M d_ab + dt a_ab K | dt a_ab b ; dt a_ab b^T | 0] in the reference's
    stage-major local layout (vel DoFs node-major, then the pressure)."""
    k = len(Ms)
    M = np.kron(Ms, np.eye(nc))
    K = np.kron(Ks, np.eye(nc))
    b = np.asarray(c).reshape(-1)
    s = len(A)
    blk = nc * k + 1
    P = np.zeros((s * blk, s * blk))
    for a in range(s):
        for bb in range(s):
            f = dt * A[a, bb]
            r0, c0 = a * blk, bb * blk
            P[r0:r0 + nc * k, c0:c0 + nc * k] = f * K + (M if a == bb else 0.0)
            P[r0:r0 + nc * k, c0 + nc * k] = f * b
            P[r0 + nc * k, c0:c0 + nc * k] = f * b
    return P


def spd(rng, k, scale):
    X = rng.standard_normal((k, k))
    return scale * (X @ X.T / k + np.eye(k))


@pytest.mark.parametrize("fam", [("radauiia", 3), ("radauiia", 2), ("gauss", 2),
                                 ("lobattoiiic", 2), ("backwardeuler", 1), ("gauss", 3)])
@pytest.mark.parametrize("k,nc", [(19, 2), (7, 2), (30, 3)])
def test_modal_record_inverts_patch_matrix(fam, k, nc):
    tab = tableau_lookup(*fam)
    dt = 1 / 256
    rng = np.random.default_rng(k + nc)
    Ms = spd(rng, k, 1e-3)
    Ks = spd(rng, k, 1.0)
    c = rng.standard_normal(k * nc) * 1e-2
    ms = ModalSplit(tab, dt, nc)
    rec = ms.record_host(Ms, Ks, c)
    P = patch_matrix(Ms, Ks, c, tab.A, dt, nc)
    Pinv = np.linalg.inv(P)
    G = ms.full_inverse(rec, k)
    assert np.linalg.norm(G - Pinv) <= 1e-11 * np.linalg.norm(Pinv)
    R = rng.standard_normal((len(P), 3))
    assert np.linalg.norm(ms.apply_host(rec, k, R) - Pinv @ R) <= 1e-11 * np.linalg.norm(Pinv @ R)
    assert len(rec) == ms.record_doubles(k) and ms.record_doubles(k) % 4 == 0
