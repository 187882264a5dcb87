"""Translation-invariant patch dedup (host setup) for the "dedup" patch mode.

On a uniform mesh with constant coefficients (Stokes, cfg1/cfg2) almost all
vertex-star patches have the same local geometry, so their stage-coupled
matrices are *bitwise* identical once the patch DoFs are put in a canonical
order -- the assembly is translation-invariant (fem.assemble_blocks rotates
cells canonically and sums duplicates in value order).  Patches are grouped
into classes of bitwise-identical canonical matrices; one set of eigen-split
inverse blocks is factorised per class (K7) and every patch applies its
class's blocks through its own canonical permutation (K3d).  The result is
the per-patch inverse of the reference (solvers.py:169-184) up to summation
order -- nothing is approximated: patches are merged only on exact equality.
"""

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from .fem import p2_node_coords

__all__ = ["DedupTables", "build_dedup_tables"]


@dataclass
class DedupTables:
    n_classes: int
    class_of: np.ndarray      # (P,) class of every flat patch slot
    perm: np.ndarray          # (total_m,) uint8: canonical position -> local position
    order: np.ndarray         # (P,) processing order: by class, then slot
    rep: np.ndarray           # (n_classes,) flat slot of each class representative
    rep_nodes: list           # canonical free-node list of each representative
    rep_vertex: np.ndarray    # (n_classes,) centre vertex of each representative
    tile_start: np.ndarray    # (n_tiles + 1,) tiles of <= CLASS_TILE same-class patches
    tile_class: np.ndarray    # (n_tiles,)    over `order`


CLASS_TILE = 32               # kClassTile in ivk_patches.cu


def _as_u8(perm):
    if perm.size and int(perm.max()) > 255:
        raise ValueError("patch too large for uint8 permutations")
    return perm.astype(np.uint8)


def build_dedup_tables(mesh, system, tables):
    """Classes of bitwise-identical canonical patch matrices for ``tables``."""
    if system.convection is not None:
        raise ValueError("dedup needs a translation-invariant (convection-free) operator")
    if system.nc != 2:
        raise ValueError("dedup is implemented for 2-D levels")
    t = tables
    P = t.num_patches
    S = t.stages
    coords = p2_node_coords(mesh)
    vcoords = mesh.vertices
    kk = np.diff(t.node_off).astype(np.int64)
    if int(t.sizes.max()) > 256:
        # perm holds stage-major local positions 0 .. m-1 of the whole patch
        raise ValueError("patch too large for uint8 permutations (m > 256)")
    slot_of = np.repeat(np.arange(P), kk)
    # canonical node order inside each patch: by (dy, dx) offset from the vertex
    off = coords[t.node] - vcoords[t.order[slot_of]]
    canon = np.lexsort((off[:, 0], off[:, 1], slot_of))      # grouped by slot
    cn = t.node[canon]                                       # canonical node lists
    alpha = np.arange(len(t.node)) - t.node_off[slot_of]     # local index (reference order)
    alpha_c = alpha[canon]                                   # local index of canonical node
    # permutation of the full stage-major local DoF list
    perm = np.empty(t.total_m, dtype=np.int64)
    blk = 2 * kk + 1
    pos_c = np.arange(len(cn)) - t.node_off[slot_of]         # canonical index
    for s in range(S):
        base = t.idx_off[:-1] + s * blk
        for c in range(2):
            perm[base[slot_of] + 2 * pos_c + c] = s * blk[slot_of] + 2 * alpha_c + c
        perm[base + 2 * kk] = s * blk + 2 * kk
    # signature: geometry offsets + scalar M, K among canonical nodes + B(node, v)
    Ms = sp.csr_matrix((system._m, system.blocks.col, system.blocks.rowptr),
                       shape=(system.n_nodes, system.n_nodes))
    Ks = sp.csr_matrix((system._k, system.blocks.col, system.blocks.rowptr),
                       shape=(system.n_nodes, system.n_nodes))
    Bx = sp.csr_matrix((system._b[:, 0], system.blocks.b_col, system.blocks.b_rowptr),
                       shape=(system.n_nodes, system.n_p))
    By = sp.csr_matrix((system._b[:, 1], system.blocks.b_col, system.blocks.b_rowptr),
                       shape=(system.n_nodes, system.n_p))
    class_of = np.empty(P, dtype=np.int64)
    n_classes = 0
    reps = []
    for k in np.unique(kk):
        slots = np.flatnonzero(kk == k)
        starts = t.node_off[slots]
        nodes = cn[starts[:, None] + np.arange(k)[None, :]]           # (n, k)
        v = t.order[slots]
        rr = np.repeat(nodes, k, axis=1).reshape(-1)
        cc = np.tile(nodes, (1, k)).reshape(-1)
        mvals = np.asarray(Ms[rr, cc]).reshape(len(slots), -1)
        kvals = np.asarray(Ks[rr, cc]).reshape(len(slots), -1)
        vv = np.repeat(v, k)
        bx = np.asarray(Bx[nodes.reshape(-1), vv]).reshape(len(slots), -1)
        by = np.asarray(By[nodes.reshape(-1), vv]).reshape(len(slots), -1)
        geo = (coords[nodes] - vcoords[v][:, None, :]).reshape(len(slots), -1)
        sig = np.ascontiguousarray(np.hstack([geo, mvals, kvals, bx, by]))
        view = sig.view(np.dtype((np.void, sig.dtype.itemsize * sig.shape[1]))).ravel()
        _, first, inv = np.unique(view, return_index=True, return_inverse=True)
        # class ids in order of first appearance (deterministic)
        rank = np.empty(len(first), dtype=np.int64)
        rank[np.argsort(first)] = np.arange(len(first))
        class_of[slots] = n_classes + rank[inv]
        for f in np.sort(first):
            reps.append(slots[f])
        n_classes += len(first)
    rep = np.array(reps, dtype=np.int64)
    order = np.lexsort((np.arange(P), class_of))
    rep_nodes = [cn[t.node_off[q]:t.node_off[q + 1]] for q in rep]
    cstart = np.concatenate([[0], np.cumsum(np.bincount(class_of, minlength=n_classes))])
    starts, classes = [], []
    for c in range(n_classes):
        s = np.arange(cstart[c], cstart[c + 1], CLASS_TILE)
        starts.append(s)
        classes.append(np.full(len(s), c))
    tile_start = np.concatenate(starts + [[P]]).astype(np.int64)
    return DedupTables(n_classes=n_classes, class_of=class_of,
                       perm=_as_u8(perm), order=order, rep=rep,
                       rep_nodes=rep_nodes, rep_vertex=t.order[rep],
                       tile_start=tile_start, tile_class=np.concatenate(classes))
