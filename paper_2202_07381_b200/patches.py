"""Vertex-star Vanka patch tables (host setup) and the device patch set.

Index construction follows the reference ``VankaPatchSet._build`` /
``_group`` (/root/reference/pkg/src/irkmg/solvers.py:132-175) exactly:

* patch v holds the sorted unique scalar P2 nodes of every cell touching
  vertex v (the closure of its star), minus constrained nodes; each node n
  contributes velocity DoFs ``2n, 2n+1`` (interleaved);
* the local layout is stage-major: ``[s*sd + vel..., s*sd + n_u + v]`` for
  s = 0..r-1 (solvers.py:160-165);
* groups are the distinct patch sizes ascending, members by ascending
  vertex (solvers.py:169-175).

The device layout flattens the groups in that order; the inverse store,
the gather list and the DoF-owner map are built once here.
"""

from dataclasses import dataclass

import numpy as np

__all__ = ["PatchTables", "build_patch_tables"]


@dataclass
class PatchTables:
    num_patches: int
    dim: int
    stages: int
    order: np.ndarray       # (P,) vertex of flat patch slot k (group order)
    sizes: np.ndarray       # (P,) patch size m in flat order
    idx_off: np.ndarray     # (P+1,) int64
    idx: np.ndarray         # (total_m,) int64 global stage-major DoFs
    node_off: np.ndarray    # (P+1,)
    node: np.ndarray        # free scalar nodes per patch (sorted)
    inv_off: np.ndarray     # (P,) int64 offsets (doubles) into the inverse store
    inv_size: int           # total doubles in the inverse store
    dof_ptr: np.ndarray     # (dim+1,)
    dof_pos: np.ndarray     # (total_m,) positions into idx/local, ascending per DoF
    multiplicity: np.ndarray  # (dim,) number of patches containing each DoF

    @property
    def total_m(self):
        return int(self.idx_off[-1])

    @property
    def max_m(self):
        return int(self.sizes.max())

    def groups(self):
        """[(m, first flat slot, count)] in the reference's group order."""
        out = []
        ms, first, counts = np.unique(self.sizes, return_index=True, return_counts=True)
        for m, f, c in zip(ms, first, counts):
            out.append((int(m), int(f), int(c)))
        return out

    def patch_of_vertex(self):
        """Inverse of ``order``: flat slot of each vertex's patch."""
        inv = np.empty(self.num_patches, dtype=np.int64)
        inv[self.order] = np.arange(self.num_patches)
        return inv


def star_closure_nodes(mesh):
    """CSR (starts, nodes): sorted unique scalar P2 nodes of the cells around
    each vertex (solvers.py:135-145); triangles or tetrahedra."""
    nv = mesh.num_vertices
    n_nodes = nv + mesh.num_edges
    cell_nodes = np.hstack([mesh.cells, nv + mesh.cell_to_edges])          # (C, 6 or 10)
    nvc, nnc = mesh.cells.shape[1], cell_nodes.shape[1]
    centre = np.repeat(mesh.cells, nnc, axis=1).reshape(-1)
    nodes = np.tile(cell_nodes, (1, nvc)).reshape(-1)
    key = np.unique(centre.astype(np.int64) * n_nodes + nodes)
    v = key // n_nodes
    starts = np.concatenate([[0], np.cumsum(np.bincount(v, minlength=nv))])
    return starts, (key % n_nodes).astype(np.int64)


def build_patch_tables(mesh, n_nodes, n_p, stages, node_constrained, vertices=None, ncomp=2):
    """All host-side tables of the vertex-star patch set for one level
    (``vertices``: only those centre vertices' patches, in the same relative
    group order)."""
    nv = mesh.num_vertices
    if n_p != nv:
        raise ValueError("mesh does not match the pressure space of the system")
    if n_nodes != nv + mesh.num_edges:
        raise ValueError("mesh does not match the velocity space of the system")
    nc = int(ncomp)
    n_u = nc * n_nodes
    sd = n_u + n_p
    dim = stages * sd
    starts, nodes = star_closure_nodes(mesh)
    owner = np.repeat(np.arange(nv), np.diff(starts))
    free = ~node_constrained[nodes]
    nodes, owner = nodes[free], owner[free]
    k_of_v = np.bincount(owner, minlength=nv)                   # free nodes per vertex
    size_of_v = stages * (nc * k_of_v + 1)

    # Group order: size ascending, vertex ascending (stable sort on size).
    order = np.argsort(size_of_v, kind="stable")
    if vertices is not None:
        keep = np.zeros(nv, dtype=bool)
        keep[np.asarray(vertices, dtype=np.int64)] = True
        order = order[keep[order]]
    sizes = size_of_v[order]
    kk = k_of_v[order]
    vstart = np.concatenate([[0], np.cumsum(k_of_v)])          # per-vertex node offsets
    # Node lists in flat patch order.
    node_off = np.concatenate([[0], np.cumsum(kk)])
    gather = _ranges(vstart[order], kk)
    pnodes = nodes[gather]

    idx_off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    total_m = int(idx_off[-1])
    idx = np.empty(total_m, dtype=np.int64)
    blk = nc * kk + 1                                           # per-stage block length
    P = len(order)
    slot_of_node = np.repeat(np.arange(P), kk)                 # patch slot of each listed node
    alpha = np.arange(len(pnodes)) - node_off[slot_of_node]    # local node index
    for s in range(stages):
        base = idx_off[:-1] + s * blk                          # start of stage block s
        pos = base[slot_of_node] + nc * alpha
        for d in range(nc):
            idx[pos + d] = s * sd + nc * pnodes + d
        idx[base + nc * kk] = s * sd + n_u + order
    ld = (sizes + 3) & ~3
    blocks = sizes.astype(np.int64) * ld
    inv_off = np.concatenate([[0], np.cumsum(blocks)]).astype(np.int64)
    mult = np.bincount(idx, minlength=dim)
    dof_pos = np.argsort(idx, kind="stable")
    dof_ptr = np.concatenate([[0], np.cumsum(mult)]).astype(np.int64)
    return PatchTables(num_patches=P, dim=dim, stages=stages, order=order, sizes=sizes,
                       idx_off=idx_off, idx=idx, node_off=node_off.astype(np.int64),
                       node=pnodes, inv_off=inv_off[:-1], inv_size=int(inv_off[-1]),
                       dof_ptr=dof_ptr, dof_pos=dof_pos, multiplicity=mult)


def _ranges(starts, lengths):
    """Concatenation of arange(s, s + l) for each (s, l), vectorised."""
    lengths = np.asarray(lengths, dtype=np.int64)
    total = int(lengths.sum())
    if total == 0:
        return np.zeros(0, dtype=np.int64)
    offs = np.concatenate([[0], np.cumsum(lengths)[:-1]])
    rep_start = np.repeat(np.asarray(starts, dtype=np.int64) - offs, lengths)
    return rep_start + np.arange(total)
