"""K1 tile plan (k1tiles.py): the plan reproduces the stage operator
(StageSystem.matvec, reference stages.py:110-126) on the host, and the tiled
kernel equals the SELL kernel bit for bit and the oracle to <= 1e-13."""

import dataclasses

import numpy as np
import pytest

from harness import oracle_levels, rel, setup
from paper_2202_07381_b200 import StageSystem
from paper_2202_07381_b200.k1tiles import apply_tiles_host, build_k1_tiles, hilbert_key


def _plan(S, xy, tile_rows):
    b = S.blocks
    order = np.lexsort((S._brows, b.b_col))
    bt_rowptr = np.concatenate([[0], np.cumsum(np.bincount(b.b_col, minlength=S.n_p))])
    return build_k1_tiles(b.rowptr, b.col, np.column_stack([S._m, S._k]), b.b_rowptr, b.b_col,
                          S._b, bt_rowptr, S._brows[order], S._b[order], S.node_constrained,
                          xy=xy, tile_rows=tile_rows)


def test_hilbert_key_is_a_bijection_on_a_grid():
    g = np.stack(np.meshgrid(np.arange(16), np.arange(16)), axis=-1).reshape(-1, 2)
    k = hilbert_key(g, bits=4)
    assert sorted(k) == list(range(256))
    o = g[np.argsort(k)]
    # consecutive curve points are grid neighbours
    assert np.all(np.abs(np.diff(o, axis=0)).sum(axis=1) == 1)


@pytest.mark.parametrize("name,coords", [("crossed", True), ("crossed", False), ("cfg1", True),
                                         ("cfg1", False), ("s3", True)])
def test_plan_reproduces_operator(name, coords):
    disc, tab, conv, case = setup(name)
    k = disc.num_levels - 1 if name == "crossed" else 1
    S = StageSystem(disc.blocks[k], tab, case["dt"], disc.cdofs[k])
    plan = _plan(S, S.blocks.node_xy if coords else None, 64)
    assert plan["n_tiles"] == -(-S.n_nodes // 64)
    # every live row appears exactly once
    rows = plan["rows"].reshape(-1, 32)
    kind = plan["slices"][:, 3]
    v = rows[kind == 0].ravel()
    v = np.where(v < -1, -(v + 2), v)
    assert sorted(v[v >= 0]) == list(range(S.n_nodes))
    p = rows[kind == 1].ravel()
    assert sorted(p[p >= 0]) == list(range(S.n_p))
    x = np.random.default_rng(3).standard_normal(S.dim)
    y = apply_tiles_host(plan, S.r, tab.A, S.dt, S.n_nodes, S.n_p, x)
    yr = S.materialize(limit=10 ** 7) @ x
    assert rel(y, yr) <= 1e-14


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["crossed", "cfg1", "s3"])
@pytest.mark.parametrize("variant", ["coords-64", "coords-256", "pseudo-128"])
def test_tiled_kernel_matches_sell_and_oracle(name, variant, monkeypatch):
    import torch
    disc, tab, conv, case = setup(name)
    k = disc.num_levels - 1
    kind, tr = variant.split("-")
    blk = disc.blocks[k]
    if kind == "pseudo":
        blk = dataclasses.replace(blk, node_xy=None)
    monkeypatch.setenv("IVK_K1_TILES", tr)
    St = StageSystem(blk, tab, case["dt"], disc.cdofs[k])
    assert St.device_data()["k1_tiles"] is not None
    monkeypatch.setenv("IVK_K1_TILES", "0")
    Ss = StageSystem(blk, tab, case["dt"], disc.cdofs[k])
    assert Ss.device_data()["k1_tiles"] is None
    rng = np.random.default_rng(5)
    x = torch.from_numpy(rng.standard_normal(St.dim)).cuda()
    b = torch.from_numpy(rng.standard_normal(St.dim)).cuda()
    for rhs in (None, b):
        yt = torch.full_like(x, float("nan"))
        ys = torch.full_like(x, float("nan"))
        St.apply_into(x, rhs, yt)
        Ss.apply_into(x, rhs, ys)
        assert torch.equal(yt, ys)          # same sums in the same order
    # in place: out == b (the Chebyshev residual update)
    r = b.clone()
    St.apply_into(x, r, r)
    assert torch.equal(r, ys)
    op = oracle_levels(disc, tab, case["dt"], None, levels=[k])[0]["op"]
    assert rel(St.matvec(x.cpu().numpy()), op.matvec(x.cpu().numpy())) <= 1e-13
