"""Device Krylov kernels (K9: ivk_dot / ivk_norm / ivk_mgs / ivk_lincomb) and
the device FGMRES path against the host (reference-algorithm) FGMRES."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _t(a):
    import torch
    return torch.as_tensor(a, dtype=torch.float64, device="cuda")


def test_dot_norm_deterministic():
    import torch
    from paper_2202_07381_b200 import _lib
    from paper_2202_07381_b200._device import ptr, stream
    L = _lib.lib()
    rng = np.random.default_rng(0)
    for n in (1, 1000, 1_777_161):
        x, y = rng.standard_normal(n), rng.standard_normal(n)
        xd, yd = _t(x), _t(y)
        out = torch.zeros(2, dtype=torch.float64, device="cuda")
        _lib.check(L.ivk_dot(n, ptr(xd), ptr(yd), ptr(out[0:1]), stream()))
        _lib.check(L.ivk_norm(n, ptr(xd), ptr(out[1:2]), stream()))
        d, nr = out.cpu().numpy()
        assert abs(d - x @ y) <= 1e-12 * np.sqrt(n) * np.linalg.norm(x) * np.linalg.norm(y)
        assert abs(nr - np.linalg.norm(x)) <= 1e-13 * np.linalg.norm(x)
        out2 = torch.zeros(1, dtype=torch.float64, device="cuda")
        _lib.check(L.ivk_dot(n, ptr(xd), ptr(yd), ptr(out2), stream()))
        assert float(out2.item()) == d  # bitwise repeatable


def test_mgs_matches_host_mgs():
    import torch
    from paper_2202_07381_b200 import _lib
    from paper_2202_07381_b200._device import ptr, stream
    rng = np.random.default_rng(1)
    n, k = 50_000, 7
    Q, _ = np.linalg.qr(rng.standard_normal((n, k)))
    V = Q.T.copy()
    w = rng.standard_normal(n)
    h_ref = np.zeros(k + 1)
    wr = w.copy()
    for i in range(k):
        h_ref[i] = wr @ V[i]
        wr -= h_ref[i] * V[i]
    h_ref[k] = np.linalg.norm(wr)
    Vd = torch.zeros(k + 1, n, dtype=torch.float64, device="cuda")
    Vd[:k] = _t(V)
    wd = _t(w)
    hd = torch.zeros(k + 1, dtype=torch.float64, device="cuda")
    _lib.check(_lib.lib().ivk_mgs(n, ptr(Vd), n, k, ptr(wd), ptr(hd), ptr(Vd[k]), stream()))
    h = hd.cpu().numpy()
    assert np.max(np.abs(h - h_ref)) <= 1e-12 * np.max(np.abs(h_ref))
    assert np.max(np.abs(Vd[k].cpu().numpy() - wr / h_ref[k])) <= 1e-12


def test_device_fgmres_matches_host():
    import torch
    from paper_2202_07381_b200 import fgmres
    rng = np.random.default_rng(8)
    n = 300
    A = rng.standard_normal((n, n)) / np.sqrt(n) + 3 * np.eye(n)
    b = rng.standard_normal(n)
    Ad = _t(A)
    x_h, st_h = fgmres(lambda v: A @ v, b, rtol=1e-10, restart=12, maxiter=80)
    x_d, st_d = fgmres(lambda v: Ad @ v, _t(b), rtol=1e-10, restart=12, maxiter=80)
    assert st_d.converged and st_h.converged
    assert st_d.iterations == st_h.iterations
    assert np.linalg.norm(x_d.cpu().numpy() - x_h) <= 1e-9 * np.linalg.norm(x_h)
    assert np.all(np.diff(st_d.residual_norms) <= 1e-12)
