"""K1 gather locality on the host: distinct 128-byte lines and 32-byte sectors
touched per warp-wide x gather of the SELL-16 kernel (16 rows, entry slot e)
at the cfg2 fine level, under the reference node numbering and under two
mesh-level vertex renumberings (lexicographic, Hilbert; edges follow as the
sorted vertex pairs).  python scripts/k1_gather_lines.py"""
import os
import sys

import numpy as np
import scipy.sparse as sp

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2202_07381_b200.mesh import build_hierarchy, Mesh2D
from paper_2202_07381_b200.fem import p2_cell_nodes
from paper_2202_07381_b200.k1tiles import hilbert_key
h = build_hierarchy(8, 5, "diagonal")
fine = h.levels[-1]
def pattern(mesh):
    nodes = p2_cell_nodes(mesh)
    N = mesh.num_vertices + mesh.num_edges
    r = np.repeat(nodes, 6, axis=1).ravel(); c = np.tile(nodes, (1,6)).ravel()
    A = sp.csr_matrix((np.ones(len(r)), (r, c)), shape=(N,N)); A.sum_duplicates(); A.sort_indices()
    return A.indptr, A.indices, N
def lines(rowptr, col, N):
    lens = np.diff(rowptr); nsl=(N+15)//16
    pad=np.zeros(nsl*16,dtype=int); pad[:N]=lens; maxw=pad.max()
    C=-np.ones((nsl*16,maxw),dtype=np.int64)
    rows=np.repeat(np.arange(N),lens); ent=np.arange(len(col))-rowptr[rows]; C[rows,ent]=col
    C=C.reshape(nsl,16,maxw); ln=0; rq=0; sc=0
    for e in range(maxw):
        c=C[:,:,e]; valid=c>=0; has=valid.any(1)
        for gran, acc in ((128,'l'),(32,'s')):
            s=np.sort(np.where(valid,(c*16)//gran,-1),axis=1)
            d=(s[:,1:]!=s[:,:-1]).sum(1)+1-(~valid).any(1)
            if acc=='l': ln+=d[has].sum()
            else: sc+=d[has].sum()
        rq+=has.sum()
    return ln/rq, sc/rq
rp,cl,N = pattern(fine); print('reference numbering: lines, sectors per request', lines(rp,cl,N))
def renumber(mesh, key):
    order = np.argsort(key, kind='stable')       # new id -> old id
    new_of_old = np.empty(len(order), dtype=np.int64); new_of_old[order] = np.arange(len(order))
    return Mesh2D(mesh.vertices[order], new_of_old[mesh.cells])
v = fine.vertices
for name, key in (('lexicographic (y,x)', np.round(v[:,1]*1e6)*1e7 + np.round(v[:,0]*1e6)),
                  ('hilbert', hilbert_key(v))):
    m2 = renumber(fine, key)
    rp,cl,N = pattern(m2)
    print(name, lines(rp,cl,N))
