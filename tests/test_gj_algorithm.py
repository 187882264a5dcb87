"""CPU restatement of the K7 elimination (csrc/ivk_gj.cuh) -- the algorithm,
not the kernel: Gauss-Jordan with IMPLICIT partial pivoting (rows are never
swapped), the pivot chosen by the 32-bit key the kernel reduces with
redux.sync (top 25 bits of |re| + |im| above 127 - row), the uniform update
a <- a' - c r with a' zero in the pivot row and column, c_pivot = -1 and
r_k = 1 / pivot, and the final unscrambling  Inv[step(i)][order(j)] = slot
(i, j)  written transposed with leading dimension ldo.  Checked against
np.linalg.inv on the matrix kinds the kernel sees (saddle-point patch
matrices with zero diagonal blocks, complex eigen-blocks, near-tie pivots).
"""

import numpy as np
import pytest


def pivot_key(mag, row):
    """The kernel's search key: high 32 bits of the double, >> 6 << 7, | (127 - row)."""
    hi = (np.float64(mag).view(np.uint64) >> np.uint64(32)).astype(np.uint32)
    return (int(hi) >> 6 << 7) | (127 - row)


def gj_invert_implicit(A, ldo=None):
    """Returns (T, order): T[j * ldo + i] = Inv[i][j] as the kernel leaves it in
    shared memory, or raises ZeroDivisionError for a singular matrix."""
    A = np.array(A, dtype=np.complex128 if np.iscomplexobj(A) else np.float64)
    d = len(A)
    ldo = d if ldo is None else ldo
    used = np.zeros(d, dtype=bool)
    order = np.zeros(d, dtype=int)
    step = np.zeros(d, dtype=int)
    for k in range(d):
        col = A[:, k].copy()
        A[:, k] = 0.0                                   # a' = 0 in the pivot column
        mag = np.abs(col.real) + np.abs(col.imag)
        keys = [0 if used[i] else pivot_key(mag[i], i) for i in range(d)]
        key = max(keys)
        prow = 127 - (key & 127)
        piv = col[prow]
        if key == 0 or not np.isfinite(piv) or piv == 0:
            raise ZeroDivisionError("singular")
        inv = 1.0 / piv
        row = A[prow].copy() * inv                      # scaled pivot row ...
        row[k] = inv                                    # ... slot k: 1 / pivot
        A[prow] = 0.0                                   # a' = 0 in the pivot row
        col[prow] = -1.0
        A -= np.outer(col, row)                         # the uniform update
        used[prow] = True
        order[k] = prow
        step[prow] = k
    T = np.zeros(d * ldo, dtype=A.dtype)
    for i in range(d):
        for j in range(d):
            T[order[j] * ldo + step[i]] = A[i, j]       # slot (i, j) = Inv[step(i)][order(j)]
    return T, order


def saddle(rng, nv, s):
    """A stage-coupled saddle-point patch matrix: SPD velocity blocks, a
    pressure column, zero pressure diagonal (solvers.py:186-212)."""
    X = rng.standard_normal((nv, nv))
    M = X @ X.T + nv * np.eye(nv)
    K = rng.standard_normal((nv, nv))
    K = K @ K.T
    b = rng.standard_normal(nv)
    Ab = np.tril(rng.uniform(0.1, 1.0, (s, s)))
    blk = nv + 1
    out = np.zeros((s * blk, s * blk))
    for a in range(s):
        for c in range(s):
            f = 0.01 * Ab[a, c]
            out[a * blk:a * blk + nv, c * blk:c * blk + nv] = (a == c) * M + f * K
            out[a * blk:a * blk + nv, c * blk + nv] = f * b
            out[a * blk + nv, c * blk:c * blk + nv] = f * b
    return out


@pytest.mark.parametrize("d,ldo", [(1, 4), (7, 8), (39, 40), (78, 80), (117, 120)])
def test_real_inverse_and_layout(d, ldo):
    rng = np.random.default_rng(d)
    A = rng.standard_normal((d, d)) + np.diag(rng.uniform(-3, 3, d))
    T, _ = gj_invert_implicit(A, ldo)
    Inv = T.reshape(d, ldo)[:, :d].T                    # T is Inv^T with leading dimension ldo
    assert np.allclose(Inv @ A, np.eye(d), atol=1e-9)
    assert np.linalg.norm(Inv - np.linalg.inv(A)) <= 1e-10 * np.linalg.norm(Inv)
    assert not T.reshape(d, ldo)[:, d:].any()           # padding rows stay zero


@pytest.mark.parametrize("nv,s", [(6, 1), (9, 2), (12, 3)])
def test_saddle_point_patch_needs_pivoting(nv, s):
    rng = np.random.default_rng(10 * nv + s)
    A = saddle(rng, nv, s)
    T, order = gj_invert_implicit(A)
    Inv = T.reshape(len(A), len(A)).T
    assert np.linalg.norm(Inv - np.linalg.inv(A)) <= 1e-9 * np.linalg.norm(Inv)
    assert sorted(order) == list(range(len(A)))         # every row pivots exactly once


def test_complex_eigen_block():
    rng = np.random.default_rng(3)
    b = 39
    X = rng.standard_normal((b, b))
    M = X @ X.T + b * np.eye(b)
    S = rng.standard_normal((b, b))
    A = M + 0.01 * (2.0 + 1.5j) * S
    T, _ = gj_invert_implicit(A, 40)
    Inv = T.reshape(b, 40)[:, :b].T
    assert np.linalg.norm(Inv - np.linalg.inv(A)) <= 1e-10 * np.linalg.norm(Inv)


def test_permutation_rows_and_near_ties():
    """A scaled permutation (every step needs an off-diagonal pivot) and a
    column of near-equal entries (the 25-bit key picks the first of them)."""
    rng = np.random.default_rng(5)
    d = 16
    P = np.eye(d)[rng.permutation(d)] * rng.uniform(0.5, 2.0, d)
    T, order = gj_invert_implicit(P)
    assert np.allclose(T.reshape(d, d).T, np.linalg.inv(P))
    A = rng.standard_normal((d, d))
    A[:, 0] = 1.55 + 1e-7 * rng.standard_normal(d)      # equal in the key's 25 bits
    T, order = gj_invert_implicit(A)
    assert order[0] == 0                                # the first of the tied rows
    assert np.linalg.norm(T.reshape(d, d).T - np.linalg.inv(A)) <= 1e-8 * np.linalg.norm(T)


def test_singular_is_reported():
    A = np.ones((5, 5))
    with pytest.raises(ZeroDivisionError):
        gj_invert_implicit(A)
    B = np.eye(4)
    B[2, 2] = np.nan
    with pytest.raises(ZeroDivisionError):
        gj_invert_implicit(B)
