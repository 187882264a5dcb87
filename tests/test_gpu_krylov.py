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
        red = _lib.reduction_scratch()
        _lib.check(L.ivk_dot(n, ptr(xd), ptr(yd), ptr(out[0:1]), ptr(red), stream()))
        _lib.check(L.ivk_norm(n, ptr(xd), ptr(out[1:2]), ptr(red), stream()))
        d, nr = out.cpu().numpy()
        assert abs(d - x @ y) <= 1e-12 * np.sqrt(n) * np.linalg.norm(x) * np.linalg.norm(y)
        assert abs(nr - np.linalg.norm(x)) <= 1e-13 * np.linalg.norm(x)
        out2 = torch.zeros(1, dtype=torch.float64, device="cuda")
        _lib.check(L.ivk_dot(n, ptr(xd), ptr(yd), ptr(out2), ptr(red), stream()))
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
    _lib.check(_lib.lib().ivk_mgs(n, ptr(Vd), n, k, ptr(wd), ptr(hd), ptr(Vd[k]),
                                  ptr(_lib.reduction_scratch()), stream()))
    h = hd.cpu().numpy()
    assert np.max(np.abs(h - h_ref)) <= 1e-12 * np.max(np.abs(h_ref))
    assert np.max(np.abs(Vd[k].cpu().numpy() - wr / h_ref[k])) <= 1e-12


def test_device_fgmres_matches_oracle():
    """Device FGMRES (device Hessenberg, Givens and triangular solve) against
    the oracle's host restatement of solvers.py:364-443: same iteration
    count and history, same solution; numpy-in / numpy-out and device-in /
    device-out entry points agree; several restarts."""
    import torch
    from oracle.irk_vanka_oracle import oracle_fgmres
    from paper_2202_07381_b200 import fgmres
    rng = np.random.default_rng(8)
    n = 300
    A = rng.standard_normal((n, n)) / np.sqrt(n) + 3 * np.eye(n)
    b = rng.standard_normal(n)
    Ad = _t(A)
    x_o, (its_o, norms_o, conv_o) = oracle_fgmres(lambda v: A @ v, b, rtol=1e-10, restart=12,
                                                  maxiter=80)
    x_h, st_h = fgmres(lambda v: A @ v, b, rtol=1e-10, restart=12, maxiter=80)
    x_d, st_d = fgmres(lambda v: Ad @ v, _t(b), rtol=1e-10, restart=12, maxiter=80)
    assert isinstance(x_h, np.ndarray)
    assert st_d.converged and st_h.converged and conv_o
    assert st_d.iterations == st_h.iterations == its_o
    # the histories agree to rounding: relative 1e-8 of the initial norm
    # (the last entries are ~1e-10 of it, where rounding of the reductions shows)
    assert np.allclose(st_d.residual_norms, norms_o, rtol=1e-8, atol=1e-12 * norms_o[0])
    assert np.linalg.norm(x_d.cpu().numpy() - x_o) <= 1e-9 * np.linalg.norm(x_o)
    assert np.linalg.norm(x_h - x_o) <= 1e-9 * np.linalg.norm(x_o)
    assert np.all(np.diff(st_d.residual_norms) <= 1e-12)


def test_concurrent_reductions_on_two_streams():
    """Per-call reduction scratch: two FGMRES-style norm streams interleaved
    on different CUDA streams stay exact (shared scratch)."""
    import torch
    from paper_2202_07381_b200 import _lib
    from paper_2202_07381_b200._device import ptr
    L = _lib.lib()
    n = 1_000_000
    x = torch.randn(n, dtype=torch.float64, device="cuda")
    y = torch.randn(n, dtype=torch.float64, device="cuda")
    ref = (float(torch.linalg.vector_norm(x)), float(torch.linalg.vector_norm(y)))
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    r1, r2 = _lib.reduction_scratch(), _lib.reduction_scratch()
    o = torch.zeros(2 * 64, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    for k in range(64):
        _lib.check(L.ivk_norm(n, ptr(x), ptr(o[k:]), ptr(r1), s1.cuda_stream))
        _lib.check(L.ivk_norm(n, ptr(y), ptr(o[64 + k:]), ptr(r2), s2.cuda_stream))
    torch.cuda.synchronize()
    oh = o.cpu().numpy()
    assert np.all(np.abs(oh[:64] - ref[0]) <= 1e-12 * ref[0])
    assert np.all(np.abs(oh[64:] - ref[1]) <= 1e-12 * ref[1])
    assert len(set(oh[:64])) == 1 and len(set(oh[64:])) == 1
