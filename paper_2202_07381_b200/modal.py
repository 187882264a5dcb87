"""Modal split of Taylor-Hood (Stokes) Vanka patches (``ivk_modal_desc``).

The reference forms every stage-coupled patch matrix
``[M_l d_ab + dt a_ab K_l | dt a_ab b ; dt a_ab b^T | 0]`` and inverts it
(solvers.py:169-212).  For convection-free operators its velocity blocks are
``M_s (x) I_nc`` and ``K_s (x) I_nc`` on the patch's k free scalar nodes
 with M_s symmetric positive definite and K_s symmetric, so the
generalised eigendecomposition ``K_s W = M_s W Theta``, ``W^T M_s W = I``
turns every stage/eigen block diagonal at once.  The exact inverse is then
carried by ``W_s`` (k x k), ``theta`` (k), ``c^ = (W_s (x) I)^T b`` (k nc) and
the s x s inverse of the pressure Schur complement
``H = dt^2 A (sum_id c^_id^2 (I + dt theta_i A)^-1) A`` -- for the cfg2
interior patch 446 doubles instead of 4,563 (kron) or 13,689 (full), for any
Butcher tableau.  Setup (kernels ``ivk_patch_gather_blocks`` + K7m
``ivk_modal_factor``: Cholesky, Jacobi eigensolver and record assembly, a
warp per patch; patches with more than 32 nodes: batched torch.linalg calls)
replaces ``np.linalg.inv``; the apply is kernel K3m (``ivk_patch_apply`` with
``pd->modal``).
"""

import os

import numpy as np

from . import _lib

__all__ = ["ModalSplit", "modal_ld"]


def modal_ld(k):
    """Leading dimension of W_s in a record: k rounded up to 4 (mod 8), so the
    K3m tensor-core A-fragment loads are bank-conflict free (ivk_patches.cu
    modal_ld)."""
    return ((k + 3) // 8) * 8 + 4


def _bitwise_classes(rows):
    """(rep, inverse): indices of one representative per class of bitwise
    identical rows and each row's class.  A 64-bit multiplicative hash of the
    bit patterns groups rows; every row is then compared with its class
    representative and any mismatch (a hash collision) becomes its own class."""
    import torch
    bits = rows.contiguous().view(torch.int64)
    g = torch.Generator(device="cpu").manual_seed(12345)
    mult = (torch.randint(1, 2 ** 62, (bits.shape[1],), generator=g, dtype=torch.int64) | 1)
    h = (bits * mult.to(bits.device)).sum(dim=1)
    _, first_inv = torch.unique(h, return_inverse=True)
    n = len(h)
    order = torch.arange(n, device=h.device)
    first = torch.full((int(first_inv.max()) + 1,), n, dtype=torch.int64, device=h.device)
    first = first.scatter_reduce(0, first_inv, order, reduce="amin")
    cand = first[first_inv]
    same = (bits == bits[cand]).all(dim=1)
    cls = torch.where(same, cand, order)                    # colliding rows stand alone
    rep, inverse = torch.unique(cls, return_inverse=True)
    return rep, inverse


def fragment_layout(tables, ncomp):
    """The K3m fragment layout (``ivk_modal_desc.layout`` = 1) of a patch
    table: (offsets (P+1), gather list, dof_pos) with patch entry
    ``node*(nc s) + comp*s + a`` / pressures ``nc s k + a`` and every patch
    padded to an even length.  ``perm`` maps each reference position
    (a*(nc k+1) + nc*node + comp, pressure a*(nc k+1) + nc k) to its
    fragment position; dof_pos keeps the reference per-DoF owner order."""
    t = tables
    S, nc = t.stages, int(ncomp)
    na = nc * S
    m = t.sizes.astype(np.int64)
    k = np.diff(t.node_off).astype(np.int64)
    if not np.array_equal(m, S * (nc * k + 1)):
        raise ValueError("patch sizes do not match the Taylor-Hood layout")
    mpad = m + (m & 1)
    offp = np.concatenate([[0], np.cumsum(mpad)])
    pid = np.repeat(np.arange(len(m)), m)
    e = np.arange(t.total_m, dtype=np.int64) - np.repeat(t.idx_off[:-1].astype(np.int64), m)
    blk = nc * k[pid] + 1
    a = e // blk
    rem = e - a * blk
    vel = rem < nc * k[pid]
    al, dd = rem // nc, rem % nc
    f = np.where(vel, al * na + dd * S + a, na * k[pid] + a)
    perm = offp[:-1][pid] + f
    idx_f = np.zeros(int(offp[-1]), dtype=np.int64)
    idx_f[perm] = t.idx
    return offp, idx_f, perm[t.dof_pos]


class ModalSplit:
    def __init__(self, tableau, dt, ncomp):
        self.A = np.asarray(tableau.A, dtype=np.float64)
        self.s = len(self.A)
        self.dt = float(dt)
        self.nc = int(ncomp)

    def record_doubles(self, k):
        return (k * modal_ld(k) + k + self.nc * k + self.s * self.s + 3) & ~3

    def _pack(self, W, theta, chat, Hinv, lib):
        """Records (count, record_doubles(k)): W_s rows padded to the
        leading dimension ``modal_ld(k)`` (the kernel's shared-memory layout)."""
        count, k = W.shape[0], W.shape[1]
        ld = modal_ld(k)
        if ld != k:
            W = lib.cat([W, W.new_zeros((count, k, ld - k))], dim=2) if hasattr(lib, "cat") \
                else np.concatenate([W, np.zeros((count, k, ld - k))], axis=2)
        parts = [W.reshape(count, -1), theta.reshape(count, -1), chat.reshape(count, -1),
                 Hinv.reshape(count, -1)]
        body = lib.cat(parts, dim=1) if hasattr(lib, "cat") else np.concatenate(parts, axis=1)
        rec = self.record_doubles(k)
        if body.shape[1] < rec:
            pad = (body.new_zeros((count, rec - body.shape[1])) if hasattr(body, "new_zeros")
                   else np.zeros((count, rec - body.shape[1])))
            body = lib.cat([body, pad], dim=1) if hasattr(lib, "cat") else \
                np.concatenate([body, pad], axis=1)
        return body

    def desc(self, layout=0):
        d = _lib.ModalDesc()
        d.stages, d.ncomp, d.dt = self.s, self.nc, self.dt
        d.layout = int(layout)
        for i in range(self.s):
            for j in range(self.s):
                d.butcher_a[i * self.s + j] = self.A[i, j]
        return d

    # -- setup (device) -------------------------------------------------------

    def factor(self, patches):
        """Fill the patch set's store with modal records; returns the flat
        slots whose patch matrix is singular (empty when all are fine)."""
        import torch
        from ._device import ptr, stream
        t = patches.tables
        dev = patches.device_data()
        ks = np.diff(t.node_off).astype(np.int64)
        kmax = int(ks.max())
        P = t.num_patches
        tdev = dev["inv"].device
        Ms = torch.zeros((P, kmax, kmax), dtype=torch.float64, device=tdev)
        Ks = torch.zeros_like(Ms)
        Cb = torch.zeros((P, kmax, self.nc), dtype=torch.float64, device=tdev)
        _lib.check(_lib.lib().ivk_patch_gather_blocks(patches.system.desc, dev["desc"], kmax,
                                                      ptr(Ms), ptr(Ks), ptr(Cb), stream()),
                   "patch_gather_blocks")
        if kmax <= 32 and os.environ.get("IVK_MODAL_SETUP", "") != "cusolver":
            # K7m: Cholesky + Jacobi eigensolver + record assembly in one kernel,
            # a warp per patch (ivk_modal_factor); larger patches (3-D, k = 65)
            # and IVK_MODAL_SETUP=cusolver (the A/B) take the batched
            # torch.linalg route below
            flag = torch.full((1,), 2 ** 31 - 1, dtype=torch.int32, device=tdev)
            _lib.check(_lib.lib().ivk_modal_factor(dev["desc"], kmax, ptr(Ms), ptr(Ks), ptr(Cb),
                                                   ptr(flag), stream()), "modal_factor")
            v = int(flag.item())
            bad = np.flatnonzero(ks == 0).tolist()
            if v != 2 ** 31 - 1:
                bad.extend(np.flatnonzero(np.asarray(t.order) == v).tolist())
            return bad
        A = torch.from_numpy(self.A).to(tdev)
        s, nc, dt = self.s, self.nc, self.dt
        eye = torch.eye(s, dtype=torch.float64, device=tdev)
        bad = []
        for k in np.unique(ks):
            sel = np.flatnonzero(ks == k)
            first, count = int(sel[0]), len(sel)
            if k == 0 or not np.array_equal(sel, np.arange(first, first + count)):
                bad.extend(sel.tolist())
                continue
            Mk = Ms[first:first + count, :k, :k]
            Kk = Ks[first:first + count, :k, :k]
            Ck = Cb[first:first + count, :k, :]
            # the eigenbasis depends on (M_s, K_s) only: patches whose blocks are
            # bitwise identical (translation-invariant stars) share one
            # decomposition -- found by a hash, then confirmed bit for bit
            rep, inv = _bitwise_classes(torch.cat([Mk.reshape(count, -1),
                                                   Kk.reshape(count, -1)], dim=1))
            L, info = torch.linalg.cholesky_ex(Mk[rep])
            X = torch.linalg.solve_triangular(L, Kk[rep], upper=False)         # L^-1 K
            Cm = torch.linalg.solve_triangular(L, X.mT, upper=False)           # L^-1 K L^-T
            Cm = 0.5 * (Cm + Cm.mT)
            # cuSOLVER's batched eigensolver takes bounded batches
            parts = [torch.linalg.eigh(Cm[i:i + 4096]) for i in range(0, len(rep), 4096)]
            theta = torch.cat([q[0] for q in parts])[inv]
            Q = torch.cat([q[1] for q in parts])
            W = torch.linalg.solve_triangular(L.mT, Q, upper=True)[inv]       # L^-T Q
            info = info[inv]
            chat = W.mT @ Ck                                                   # (P, k, nc)
            E = torch.linalg.inv(eye + dt * theta[..., None, None] * A)        # (P, k, s, s)
            wsum = torch.einsum("pi,piab->pab", (chat * chat).sum(-1), E)
            H = dt * dt * (A @ wsum @ A)
            Hinv, hinfo = torch.linalg.inv_ex(H)
            # 1-norm condition number (exact for the s x s Schur complement;
            # an SVD per patch would cost more than the factorisation)
            cond = torch.linalg.matrix_norm(H, ord=1) * torch.linalg.matrix_norm(Hinv, ord=1)
            ok = (info == 0) & (hinfo == 0) & torch.isfinite(Hinv).flatten(1).all(1) & \
                (cond < 1e14)
            rec = self.record_doubles(int(k))
            body = self._pack(W, theta, chat, Hinv, torch)
            off = int(patches.inv_off[first])
            dev["inv"][off:off + count * rec] = body.reshape(-1)
            bad.extend((first + np.flatnonzero(~ok.cpu().numpy())).tolist())
        return bad

    # -- host algebra (API parity: ``VankaPatchSet.groups``; tests) ------------

    def record_host(self, Ms, Ks, c):
        """One patch's record from its scalar blocks and pressure column
        (scipy generalised eigh; the device setup's host twin)."""
        import scipy.linalg as sla
        k = len(Ms)
        theta, W = sla.eigh(Ks, Ms)
        chat = W.T @ np.asarray(c, dtype=np.float64).reshape(k, self.nc)
        E = np.linalg.inv(np.eye(self.s) + self.dt * theta[:, None, None] * self.A)
        H = self.dt ** 2 * (self.A @ np.einsum("i,iab->ab", (chat ** 2).sum(1), E) @ self.A)
        return self._pack(W[None], theta[None], chat[None], np.linalg.inv(H)[None], np)[0]

    def unpack(self, raw, k):
        nc, s, ld = self.nc, self.s, modal_ld(k)
        o = k * ld
        W = raw[:o].reshape(k, ld)[:, :k]
        th = raw[o:o + k]
        ch = raw[o + k:o + k + nc * k].reshape(k, nc)
        Hi = raw[o + k + nc * k:o + k + nc * k + s * s].reshape(s, s)
        return W, th, ch, Hi

    def apply_host(self, raw, k, R):
        """Y = P^-1 R for one patch (R: (m, ncols), stage-major local layout)."""
        W, th, ch, Hi = self.unpack(raw, k)
        s, nc, dt, A = self.s, self.nc, self.dt, self.A
        blk = nc * k + 1
        R = np.asarray(R, dtype=np.float64).reshape(s, blk, -1)
        ru = R[:, :nc * k].reshape(s, k, nc, -1)
        rp = R[:, nc * k]                                            # (s, n)
        t = np.einsum("ai,sadn->sidn", W, ru)
        E = np.linalg.inv(np.eye(s) + dt * th[:, None, None] * A)   # (k, s, s)
        w = np.einsum("iab,bidn->aidn", E, t)
        g = np.einsum("id,aidn->an", ch, w)
        p = Hi @ (dt * (A @ g) - rp)
        Ap = A @ p
        v = w - dt * ch[None, :, :, None] * np.einsum("iab,bn->ain", E, Ap)[:, :, None, :]
        u = np.einsum("ai,sidn->sadn", W, v).reshape(s, nc * k, -1)
        return np.concatenate([u, p[:, None, :]], axis=1).reshape(s * blk, -1)

    def full_inverse(self, raw, k):
        m = self.s * (self.nc * k + 1)
        return self.apply_host(raw, k, np.eye(m))
