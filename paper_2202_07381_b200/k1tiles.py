"""Tile plan of the K1 stage apply (host setup, numpy).

The stage operator ``StageSystem.matvec`` (reference stages.py:110-126) is a
gather SpMV on the reference's hierarchical node numbering (coarse vertices
first, then edge midpoints level by level, mesh.py:178-206), so neighbouring
rows share almost no cache lines of ``x``.  The plan groups the rows into
geometrically compact *tiles* (runs of a Hilbert curve through the node
coordinates): each tile lists the scalar P2 nodes and P1 nodes its rows read
(``ulist`` / ``plist``), the kernel stages those values of all s stages in
shared memory once, and the operator entries carry 16-bit *local* columns
into the staged lists.  Vectors stay in the reference layout; only the order
in which rows are processed changes.

A tile's rows form slices of 32 (one warp each), longest rows first:
velocity slices (one thread per scalar node: both components, all stages;
``wa`` scalar P2 entries with (m, k) values, then ``wb`` B entries with
(B_x, B_y)), then pressure slices (one thread per P1 node, ``wa`` B^T
entries).  Entry e of lane l sits at ``ent_off + 32 e + l``; the entries of
a row keep their CSR order, so every row sums exactly as the SELL kernel
does.  Padding entries carry a zero value and a column of the row's own
stencil.
"""

import numpy as np

__all__ = ["hilbert_key", "pseudo_coordinates", "build_k1_tiles", "apply_tiles_host"]

LANES = 32
KIND_VELOCITY, KIND_PRESSURE = 0, 1


def hilbert_key(xy, bits=15):
    """Hilbert-curve index of 2-D points (quantised to ``bits`` per axis)."""
    xy = np.asarray(xy, dtype=np.float64)
    lo = xy.min(axis=0)
    span = np.maximum(xy.max(axis=0) - lo, 1e-300)
    n = 1 << bits
    q = np.minimum(((xy - lo) / span.max() * (n - 1) + 0.5).astype(np.int64), n - 1)
    x, y = q[:, 0].copy(), q[:, 1].copy()
    d = np.zeros(len(x), dtype=np.int64)
    s = n >> 1
    while s > 0:
        rx = (x & s) > 0
        ry = (y & s) > 0
        d += s * s * ((3 * rx.astype(np.int64)) ^ ry.astype(np.int64))
        flip = (~ry) & rx
        x = np.where(flip, n - 1 - x, x)
        y = np.where(flip, n - 1 - y, y)
        swap = ~ry
        x, y = np.where(swap, y, x), np.where(swap, x, y)
        s >>= 1
    return d


def pseudo_coordinates(rowptr, col, n):
    """2-D landmark embedding of the pattern graph by breadth-first distances
    (for operators that arrive without node coordinates, e.g. built from the
    reference's vector CSR blocks)."""
    import scipy.sparse as sp
    from scipy.sparse.csgraph import dijkstra
    G = sp.csr_matrix((np.ones(len(col), dtype=np.int8), col, rowptr), shape=(n, n))

    def dist(src):
        d = dijkstra(G, unweighted=True, indices=int(src))
        fin = np.isfinite(d)
        d[~fin] = (d[fin].max() if fin.any() else 0.0) + 1.0
        return d

    b = int(np.argmax(dist(0)))
    db = dist(b)
    c = int(np.argmax(db))
    dc = dist(c)
    e = int(np.argmax(db + dc))
    de = dist(e)
    f = int(np.argmax(de))
    df = dist(f)
    return np.column_stack([db - dc, de - df])


def _group_slices(tile_of_row, sort_len, n_tiles):
    """Order rows by (tile, length descending, row id) and cut every tile's
    run into slices of 32.  Returns (rows padded with -1, slice tile ids)."""
    n = len(tile_of_row)
    order = np.lexsort((np.arange(n), -sort_len, tile_of_row))
    cnt = np.bincount(tile_of_row, minlength=n_tiles)
    nsl = (cnt + LANES - 1) // LANES
    s0 = np.concatenate([[0], np.cumsum(nsl)])
    start = np.concatenate([[0], np.cumsum(cnt)])
    t = tile_of_row[order]
    within = np.arange(n) - start[t]
    rows = np.full(int(s0[-1]) * LANES, -1, dtype=np.int64)
    rows[s0[t] * LANES + within] = order
    return rows, np.repeat(np.arange(n_tiles), nsl)


def _fill_entries(rows, lens, rowptr, ent_off, width, total_lanes):
    """Positions (in the flat entry arrays) of the CSR entries of the padded
    row list: entry e of lane l of slice s -> ent_off[s] + 32 e + l."""
    live = np.flatnonzero((rows >= 0) & (lens > 0))
    r = rows[live]
    ln = lens[live]
    rep = np.repeat(np.arange(len(live)), ln)
    e = np.arange(int(ln.sum())) - np.repeat(np.concatenate([[0], np.cumsum(ln)[:-1]]), ln)
    src = rowptr[r][rep] + e
    sl = live // LANES
    pos = ent_off[sl][rep] + e * LANES + (live % LANES)[rep]
    return src, pos, live


def build_k1_tiles(rowptr, col, mk, b_rowptr, b_col, b_val, bt_rowptr, bt_col, bt_val,
                   node_fixed, xy=None, tile_rows=256):
    """Build the tile plan.  ``mk`` is (nnz, 2), ``b_val`` / ``bt_val`` are
    (nnz_b, 2); all values eliminated.  Returns a dict of numpy arrays."""
    rowptr = np.asarray(rowptr, dtype=np.int64)
    b_rowptr = np.asarray(b_rowptr, dtype=np.int64)
    bt_rowptr = np.asarray(bt_rowptr, dtype=np.int64)
    col = np.asarray(col, dtype=np.int64)
    b_col = np.asarray(b_col, dtype=np.int64)
    bt_col = np.asarray(bt_col, dtype=np.int64)
    n = len(rowptr) - 1
    n_p = len(bt_rowptr) - 1
    fixed = np.asarray(node_fixed, dtype=bool)
    if xy is None:
        xy = pseudo_coordinates(rowptr, col, n)
    key = hilbert_key(np.asarray(xy)[:, :2])
    perm = np.lexsort((np.arange(n), key))
    n_tiles = (n + tile_rows - 1) // tile_rows
    tile_of_node = np.empty(n, dtype=np.int64)
    tile_of_node[perm] = np.arange(n) // tile_rows

    len_a = np.diff(rowptr)
    len_b = np.diff(b_rowptr)
    len_bt = np.diff(bt_rowptr)
    # a P1 row goes to the tile of the B^T column with the widest P2 stencil
    # (the coincident vertex node, whose stencil is the whole star)
    tile_of_p = np.zeros(n_p, dtype=np.int64)
    has = len_bt > 0
    if has.any():
        w = len_a[bt_col]
        rowid = np.repeat(np.arange(n_p), len_bt)
        best = np.lexsort((np.arange(len(w)), -w, rowid))
        first = bt_rowptr[:-1][has]
        tile_of_p[has] = tile_of_node[bt_col[best[first]]]

    # velocity slices (fixed rows carry no entries: identity rows)
    la = np.where(fixed, 0, len_a)
    lb = np.where(fixed, 0, len_b)
    vrows, vtile = _group_slices(tile_of_node, la + lb, n_tiles)
    prows, ptile = _group_slices(tile_of_p, len_bt, n_tiles)
    nv, npz = len(vtile), len(ptile)

    def widths(rows, lens):
        l = np.where(rows >= 0, lens[np.maximum(rows, 0)], 0)
        return l, l.reshape(-1, LANES).max(axis=1)

    va, wa = widths(vrows, la)
    vb, wb = widths(vrows, lb)
    pa, wp = widths(prows, len_bt)

    # interleave: per tile its velocity slices, then its pressure slices
    s_tile = np.concatenate([vtile, ptile])
    s_kind = np.concatenate([np.zeros(nv, np.int64), np.ones(npz, np.int64)])
    s_wa = np.concatenate([wa, wp])
    s_wb = np.concatenate([wb, np.zeros(npz, np.int64)])
    s_rows = np.concatenate([vrows.reshape(-1, LANES), prows.reshape(-1, LANES)])
    order = np.lexsort((np.arange(nv + npz), s_kind, s_tile))
    s_tile, s_kind, s_wa, s_wb, s_rows = (a[order] for a in (s_tile, s_kind, s_wa, s_wb, s_rows))
    n_slices = nv + npz
    tile_s0 = np.searchsorted(s_tile, np.arange(n_tiles + 1))
    ent_off = np.concatenate([[0], np.cumsum((s_wa + s_wb) * LANES)])
    n_ent = int(ent_off[-1])

    flat_rows = s_rows.ravel()
    kind_lane = np.repeat(s_kind, LANES)
    tile_lane = np.repeat(s_tile, LANES)
    is_v = (kind_lane == KIND_VELOCITY) & (flat_rows >= 0)
    is_p = (kind_lane == KIND_PRESSURE) & (flat_rows >= 0)
    vr = np.where(is_v, flat_rows, -1)
    pr = np.where(is_p, flat_rows, -1)

    la_l = np.where(vr >= 0, la[np.maximum(vr, 0)], 0)
    lb_l = np.where(vr >= 0, lb[np.maximum(vr, 0)], 0)
    lp_l = np.where(pr >= 0, len_bt[np.maximum(pr, 0)], 0)
    srcA, posA, liveA = _fill_entries(vr, la_l, rowptr, ent_off[:-1], s_wa, len(flat_rows))
    srcB, posB, liveB = _fill_entries(vr, lb_l, b_rowptr, ent_off[:-1] + s_wa * LANES, s_wb,
                                      len(flat_rows))
    srcP, posP, liveP = _fill_entries(pr, lp_l, bt_rowptr, ent_off[:-1], s_wa, len(flat_rows))

    # staged node lists: every velocity node a tile's entries read
    tA = np.repeat(tile_lane[liveA], la_l[liveA])
    tP = np.repeat(tile_lane[liveP], lp_l[liveP])
    ukeys = np.concatenate([tA * n + col[srcA], tP * n + bt_col[srcP]])
    uu, uinv = np.unique(ukeys, return_inverse=True)
    tile_u0 = np.searchsorted(uu // n, np.arange(n_tiles + 1))
    ulist = uu % n
    ulocal = uinv - tile_u0[uu[uinv] // n]
    tB = np.repeat(tile_lane[liveB], lb_l[liveB])
    pkeys = tB * max(n_p, 1) + b_col[srcB]
    pu, pinv = np.unique(pkeys, return_inverse=True)
    tile_p0 = np.searchsorted(pu // max(n_p, 1), np.arange(n_tiles + 1))
    plist = pu % max(n_p, 1)
    plocal = pinv - tile_p0[pu[pinv] // max(n_p, 1)]
    max_u = int(np.diff(tile_u0).max()) if n_tiles else 0
    max_p = int(np.diff(tile_p0).max()) if n_tiles else 0
    if max_u > 0xFFFF or max_p > 0xFFFF:
        raise ValueError("tile too large for 16-bit local columns")

    ecol = np.zeros(n_ent, dtype=np.uint16)
    eval_ = np.zeros((n_ent, 2), dtype=np.float64)
    # padding columns: a valid entry of the same row / section (zero value)
    def pad_cols(live, lens_l, local, base_off, width):
        if len(live) == 0:
            return
        firsts = np.concatenate([[0], np.cumsum(lens_l[live])[:-1]])
        first_local = local[firsts]
        sl = live // LANES
        w = width[sl]
        npad = w - lens_l[live]
        rep = np.repeat(np.arange(len(live)), npad)
        e = np.arange(int(npad.sum())) - np.repeat(np.concatenate([[0], np.cumsum(npad)[:-1]]), npad)
        pos = base_off[sl][rep] + (lens_l[live][rep] + e) * LANES + (live % LANES)[rep]
        ecol[pos] = first_local[rep]

    mk = np.asarray(mk, dtype=np.float64).reshape(-1, 2)
    nA, nP = len(srcA), len(srcP)
    ecol[posA] = ulocal[:nA]
    eval_[posA] = mk[srcA]
    ecol[posP] = ulocal[nA:nA + nP]
    eval_[posP] = np.asarray(bt_val, dtype=np.float64).reshape(-1, 2)[srcP]
    ecol[posB] = plocal
    eval_[posB] = np.asarray(b_val, dtype=np.float64).reshape(-1, 2)[srcB]
    pad_cols(liveA, la_l, ulocal[:nA], ent_off[:-1], s_wa)
    pad_cols(liveP, lp_l, ulocal[nA:nA + nP], ent_off[:-1], s_wa)
    pad_cols(liveB, lb_l, plocal, ent_off[:-1] + s_wa * LANES, s_wb)

    # rows: id, -1 = padding lane, -(id + 2) = fixed velocity row (identity)
    rows_enc = flat_rows.copy()
    fx = is_v & fixed[np.maximum(flat_rows, 0)]
    rows_enc[fx] = -(flat_rows[fx] + 2)
    slices = np.column_stack([ent_off[:-1], s_wa, s_wb, s_kind]).astype(np.int32)
    tile_ent = np.diff(ent_off[tile_s0])
    blob, tile_rec = _pack_blobs(n_tiles, tile_u0, tile_p0, tile_s0, ent_off, ulist, plist,
                                 slices, rows_enc)
    return {
        "blob": blob, "tile_rec": tile_rec, "max_blob": int(tile_rec[:, 1].max()) if n_tiles else 0,
        "n_tiles": n_tiles, "n_slices": n_slices, "max_u": max_u, "max_p": max_p,
        "max_ent": int(tile_ent.max()) if n_tiles else 0,
        "max_slices": int(np.diff(tile_s0).max()) if n_tiles else 0,
        "n_entries": n_ent, "tile_rows": tile_rows,
        "tile_u0": tile_u0.astype(np.int32), "tile_p0": tile_p0.astype(np.int32),
        "tile_s0": tile_s0.astype(np.int32),
        "ulist": ulist.astype(np.int32), "plist": plist.astype(np.int32),
        "slices": slices, "rows": rows_enc.astype(np.int32),
        "ecol": ecol, "eval": eval_,
    }


def _pack_blobs(n_tiles, tile_u0, tile_p0, tile_s0, ent_off, ulist, plist, slices, rows):
    """Per-tile metadata blobs (int32 words, one TMA bulk copy each):
    header (nu, np, ns, n_ent, 0, 0, 0, 0) | ulist | plist | pad to 4 words |
    slices (ns x 4, entry offsets relative to the tile) | rows (ns x 32).
    tile_rec[t] = (blob offset, blob words, entry offset, entries, nu, np, ns, 0)."""
    nu = np.diff(tile_u0).astype(np.int64)
    npp = np.diff(tile_p0).astype(np.int64)
    ns = np.diff(tile_s0).astype(np.int64)
    e0 = ent_off[tile_s0[:-1]].astype(np.int64)
    ne = np.diff(ent_off[tile_s0]).astype(np.int64)
    o_sl = (8 + nu + npp + 3) // 4 * 4
    words = o_sl + 36 * ns
    boff = np.concatenate([[0], np.cumsum(words)])
    blob = np.zeros(int(boff[-1]), dtype=np.int32)
    b0 = boff[:-1]
    blob[b0], blob[b0 + 1], blob[b0 + 2], blob[b0 + 3] = nu, npp, ns, ne

    def scatter(dst0, cnt, src):
        rep = np.repeat(np.arange(n_tiles), cnt)
        within = np.arange(int(cnt.sum())) - np.repeat(np.concatenate([[0], np.cumsum(cnt)[:-1]]), cnt)
        blob[dst0[rep] + within] = src

    scatter(b0 + 8, nu, ulist)
    scatter(b0 + 8 + nu, npp, plist)
    sl = slices.astype(np.int64).copy()
    sl[:, 0] -= np.repeat(e0, ns)
    scatter(b0 + o_sl, 4 * ns, sl.ravel())
    scatter(b0 + o_sl + 4 * ns, 32 * ns, rows)
    rec = np.column_stack([b0, words, e0, ne, nu, npp, ns, np.zeros(n_tiles, np.int64)])
    return blob, rec.astype(np.int32)


def apply_tiles_host(plan, S, A, dt, n_nodes, n_p, x, b=None):
    """Numpy walk of the tile plan, mirroring the kernel (tests only: checks
    the plan against the CSR operator without a GPU)."""
    nu = 2 * n_nodes
    sd = nu + n_p
    x = np.asarray(x, dtype=np.float64).reshape(S, sd)
    out = np.full((S, sd), np.nan)
    A = np.asarray(A, dtype=np.float64)
    for t in range(plan["n_tiles"]):
        ul = plan["ulist"][plan["tile_u0"][t]:plan["tile_u0"][t + 1]]
        pl = plan["plist"][plan["tile_p0"][t]:plan["tile_p0"][t + 1]]
        xs = x[:, :nu].reshape(S, n_nodes, 2)[:, ul, :]          # (S, nu_t, 2)
        ps = x[:, nu:][:, pl]                                    # (S, np_t)
        for s in range(plan["tile_s0"][t], plan["tile_s0"][t + 1]):
            off, wa, wb, kind = plan["slices"][s]
            rows = plan["rows"][s * LANES:(s + 1) * LANES]
            for lane in range(LANES):
                r = rows[lane]
                if r == -1:
                    continue
                if kind == KIND_VELOCITY:
                    if r <= -2:
                        node = -r - 2
                        y = x[:, 2 * node:2 * node + 2].copy()
                    else:
                        node = r
                        mu = np.zeros((S, 2))
                        ku = np.zeros((S, 2))
                        for e in range(wa):
                            c = plan["ecol"][off + e * LANES + lane]
                            m, k = plan["eval"][off + e * LANES + lane]
                            mu += m * xs[:, c, :]
                            ku += k * xs[:, c, :]
                        for e in range(wa, wa + wb):
                            c = plan["ecol"][off + e * LANES + lane]
                            bx, by = plan["eval"][off + e * LANES + lane]
                            ku[:, 0] += bx * ps[:, c]
                            ku[:, 1] += by * ps[:, c]
                        y = mu + dt * (A @ ku)
                    o = slice(2 * node, 2 * node + 2)
                else:
                    btu = np.zeros(S)
                    for e in range(wa):
                        c = plan["ecol"][off + e * LANES + lane]
                        bx, by = plan["eval"][off + e * LANES + lane]
                        btu += bx * xs[:, c, 0] + by * xs[:, c, 1]
                    y = dt * (A @ btu)
                    o = nu + r
                out[:, o] = y
    out = out.ravel()
    return out if b is None else np.asarray(b) - out
