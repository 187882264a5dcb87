/*
 * ivk.h -- C ABI of the B200-native IRK-Vanka hot path (libivk.so, sm_100a).
 *
 * The reference (`irkmg`, /root/reference/pkg/src/irkmg) is pure Python on
 * numpy/scipy and has no FFI; its "operator interface" is the duck-typed
 * Python API of stages.py / solvers.py.  Each entry point below replaces one
 * reference call site on that path (cited file:line, paths relative to
 * /root/reference/pkg/src/irkmg/).  The Python host layer
 * (paper_2202_07381_b200/) binds these with ctypes and keeps the reference's
 * Python signatures; INTEGRATION.md shows the binding.
 *
 * Conventions
 *  - All pointers except descriptors are DEVICE pointers owned by the caller
 *    (torch allocations); the library never allocates or frees them.
 *  - Every call is asynchronous on `stream` (a cudaStream_t, passed as void*;
 *    NULL = legacy default stream) and returns 0 or a negative IVK_E* code;
 *    ivk_last_error() gives a message (thread-local).
 *  - fp64 values, int32 indices, int64 offsets into the patch-inverse store.
 *  - Vectors are in the reference's stage-major layout
 *    [(u_1, p_1), ..., (u_s, p_s)], u interleaving the two velocity
 *    components per scalar P2 node (stages.py:100-106, fem.py:9-13).
 *  - Not thread-safe per descriptor; descriptors are plain structs.
 */
#ifndef IVK_H
#define IVK_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IVK_OK 0
#define IVK_EINVAL (-1)
#define IVK_ECUDA (-2)
#define IVK_ESINGULAR (-3)
#define IVK_EUNSUPPORTED (-4)

#define IVK_MAX_STAGES 3
#define IVK_MAX_QUAD 16

/* Stage-coupled operator  I_s (x) diag(M, 0) + dt A (x) [[K, B], [B^T, 0]]
 * (+ dt a_ij J_i on the velocity block), with identity rows on constrained
 * velocity DoFs.  Replaces StageSystem.__init__/matvec (stages.py:63-126).
 * M, K, J are stored on the scalar P2 pattern already eliminated (zero in
 * constrained rows/columns, stages.py:77-85); B rows are per scalar node with
 * (B_x, B_y) pairs, B^T rows per P1 node -- both eliminated. */
/* Tile plan of the K1 apply (k1tiles.py; 2-D Stokes operators, n_conv == 0).
 * Rows are grouped into geometrically compact tiles (one CTA each).  A tile
 * stages, for all s stages, the velocity values of the scalar nodes in its
 * ulist and the pressures of the P1 nodes in its plist in shared memory, then
 * runs its row slices (32 rows, one warp each) against its entry stream.
 * tile_rec[8t .. 8t+7] = (blob offset, blob words, entry offset, entries,
 * nu, np, ns, 0).  The tile's blob (int32 words, one TMA bulk copy) is
 *   header (nu, np, ns, entries, 0, 0, 0, 0) | ulist (nu) | plist (np) |
 *   pad to 4 words | slices (ns x 4) | rows (ns x 32)
 * with slice = (entry offset within the tile, wa, wb, kind): kind 0 =
 * velocity rows (one thread per scalar node: wa scalar-P2 entries with (m, k)
 * values, then wb B entries with (B_x, B_y)); kind 1 = pressure rows (wa B^T
 * entries).  Entry e of lane l sits at offset + 32 e + l in ecol (16-bit
 * column, local to the staged lists) and eval; a row id is the scalar node /
 * P1 node, -1 for a padding lane, -(node + 2) for a constrained (identity)
 * velocity row.  Every row keeps its CSR entry order, so the sums are the
 * SELL kernel's bit for bit.  All arrays are device pointers; the struct
 * itself lives on the host. */
typedef struct ivk_k1_tiles {
  int32_t n_tiles;
  int32_t max_u;           /* longest staged velocity-node list           */
  int32_t max_p;           /* longest staged P1-node list                 */
  int32_t max_ent;         /* most entries (with padding) of one tile     */
  int32_t max_slices;      /* most slices of one tile                     */
  int32_t max_blob;        /* longest blob (words)                        */
  const int32_t* tile_rec; /* n_tiles * 8                                 */
  const int32_t* blob;
  const uint16_t* ecol;
  const double* eval;      /* 2 per entry                                 */
} ivk_k1_tiles;

typedef struct ivk_operator_desc {
  int32_t stages;          /* s, 1..IVK_MAX_STAGES                        */
  int32_t n_nodes;         /* scalar P2 nodes; n_u = 2 * n_nodes          */
  int32_t n_p;             /* P1 pressure nodes                           */
  int32_t n_conv;          /* 0: Stokes; 1: one J for all stages; s: J_i  */
  int32_t nnz;             /* scalar P2 pattern entries                   */
  double dt;
  double butcher_a[IVK_MAX_STAGES * IVK_MAX_STAGES]; /* row-major s x s   */
  const int32_t* p2_rowptr; /* n_nodes + 1                                 */
  const int32_t* p2_col;    /* nnz                                         */
  const double* p2_mk;      /* nnz * 2: (m, k) per entry                   */
  const double* conv;       /* n_conv * nnz * 4: (Jxx, Jxy, Jyx, Jyy)      */
  const int32_t* b_rowptr;  /* n_nodes + 1                                 */
  const int32_t* b_col;     /* nnz_b (P1 node)                             */
  const double* b_val;      /* nnz_b * 2: (B_x, B_y)                       */
  const int32_t* bt_rowptr; /* n_p + 1                                     */
  const int32_t* bt_col;    /* nnz_b (scalar P2 node)                      */
  const double* bt_val;     /* nnz_b * 2                                   */
  const uint8_t* node_constrained; /* n_nodes: 1 = both components fixed   */
  /* The same operator in sliced-ELL form for the K1 apply: velocity rows
   * (p2_*, conv_s, b_*) in SELL-16, pressure rows (bt_*) in SELL-32; entry
   * e of a slice's j-th row at ptr[slice] + H e + j, padding entries carry
   * zero values.  The CSR arrays above serve the patch assembly (K7). */
  const int32_t* p2_sptr;   /* ceil(n_nodes/16) + 1                        */
  const int32_t* p2_scol;
  const double* p2_smk;     /* (m, k) per entry                            */
  const double* conv_s;     /* n_conv blocks of (Jxx, Jxy, Jyx, Jyy)       */
  int32_t nnz_s;            /* SELL entries per operand (conv stride)      */
  const int32_t* b_sptr;
  const int32_t* b_scol;
  const double* b_sval;
  const int32_t* bt_sptr;   /* ceil(n_p/32) + 1                            */
  const int32_t* bt_scol;
  const double* bt_sval;
  /* Velocity components per scalar node: 0 or 2 (2-D, as above), or 3 (3-D
   * Kuhn tetrahedra, fem3d.py: n_u = 3 n_nodes, B/B^T values are (B_x, B_y,
   * B_z) triples, velocity rows in SELL-32 with one thread per node; no
   * convection). */
  int32_t ncomp;
  /* Optional tile plan of the K1 apply (HOST pointer, or NULL: SELL kernel). */
  const struct ivk_k1_tiles* k1_tiles;
  /* Optional processing order of the SELL kernel's slices (device pointer,
   * k1_order_n = all of them: velocity slices 0 .. ceil(n_nodes/16)-1, then
   * ceil(n_nodes/16) + pressure slice): warp w of the grid runs slice
   * k1_order[w], so the eight slices of a CTA can be chosen close together in
   * space (L1 reuse of the gathered x).  NULL: memory order. */
  const int32_t* k1_order;
  int32_t k1_order_n;
} ivk_operator_desc;

/* Vanka vertex-star patch set (solvers.py:116-222).  Patches are laid out
 * in the reference's group order (size ascending, vertex ascending within a
 * size, solvers.py:169-175).  Patch p owns idx[idx_off[p] .. idx_off[p+1])
 * (its stage-major local DoF list, solvers.py:160-165) and an m x ld block
 * of the inverse store at inv_off[p], holding Inv^T (inv[j*ld + i] =
 * Inv[i][j]), ld = (m + 3) & ~3.  dof_ptr/dof_pos is the inverse map
 * global DoF -> positions in the flat local[] array, ascending. */
typedef struct ivk_patch_desc {
  int32_t num_patches;
  int32_t dim;             /* stage-system dimension                      */
  int32_t max_m;
  int32_t total_m;         /* sum of patch sizes                          */
  const int32_t* idx_off;  /* num_patches + 1                             */
  const int32_t* idx;      /* total_m                                     */
  const int64_t* inv_off;  /* num_patches                                 */
  double* inv;             /* inverse store                               */
  const int32_t* dof_ptr;  /* dim + 1                                     */
  const int32_t* dof_pos;  /* total_m                                     */
  const int32_t* vertex;   /* num_patches: centre vertex                  */
  const int32_t* node_off; /* num_patches + 1                             */
  const int32_t* node;     /* free scalar P2 nodes of each patch, sorted  */
  const int32_t* slot_pos; /* total_m or NULL: where patch slot k is written
                              in local[] (owner-sorted, so the scatter reads
                              local[dof_ptr[d] .. dof_ptr[d+1]) contiguously);
                              NULL = patch order, scatter gathers via dof_pos */
  const struct ivk_kron_desc* kron; /* HOST pointer; NULL = full inverses */
  /* Dedup (kron only; n_classes == 0: per-patch inverses).  Patches whose
   * canonical stage-coupled matrices are bitwise identical share one set of
   * inverse blocks (class_inv + class_inv_off[c]); ivk_patch_factor on a
   * descriptor of the class representatives (canonical node lists) fills
   * class_inv.  The apply runs over tiles of <= 32 same-class patches, in
   * class order: tile t holds tile_start[t+1] - tile_start[t] patches of
   * class tile_class[t]; its patches' DoFs, each patch in the class's
   * canonical order, are cidx[tile_off[t] .. tile_off[t+1]) (gather indices
   * into r) and cdst[...] (write positions in local[]). */
  int32_t n_classes;
  const int64_t* class_inv_off; /* n_classes + 1 */
  const double* class_inv;
  int32_t n_tiles;
  const int32_t* tile_start;    /* n_tiles + 1 */
  const int32_t* tile_class;    /* n_tiles     */
  const int32_t* tile_off;      /* n_tiles + 1 */
  const int32_t* cidx;          /* total_m     */
  const int32_t* cdst;          /* total_m     */
  /* Modal store (non-NULL, HOST pointer; kron must be NULL): see
   * ivk_modal_desc.  Patch p holds k = node_off[p+1] - node_off[p] free
   * nodes and its record at inv_off[p]. */
  const struct ivk_modal_desc* modal;
} ivk_patch_desc;

/* Modal split of Taylor-Hood (Stokes) patches.  The velocity blocks are
 * M_s (x) I_nc and K_s (x) I_nc on the patch's k free scalar nodes,
 * M_s symmetric positive definite, K_s symmetric, so one generalised
 * eigendecomposition K_s W = M_s W Theta, W^T M_s W = I, diagonalises every
 * stage and eigen-block at once.  With W = W_s (x) I_nc, c the patch's
 * pressure column (B[vel, v]) and c^ = W^T c, the stage-coupled patch system
 *   sum_b [delta_ab M + dt A_ab K] u_b + dt A_ab c p_b = r_a,
 *   sum_b dt A_ab c^T u_b = q_a
 * becomes, per mode (i, d) with E_i = (I_s + dt theta_i A)^-1 (s x s):
 *   t = W^T r,  w_id = E_i t_id,  g = sum_id c^_id w_id,
 *   p = H^-1 (dt A g - q),  H = dt^2 A (sum_id c^_id^2 E_i) A,
 *   v_id = w_id - dt c^_id E_i A p,  u = W v.
 * Exactly the inverse of R_i A R_i^T (solvers.py:186-212; any tableau).
 * Record of a patch (doubles, padded to a multiple of 4):
 *   W_s[alpha][i] row-major (k x k) | theta (k) | c^[i][d] (k x nc) | H^-1 (s x s). */
typedef struct ivk_modal_desc {
  int32_t stages;
  int32_t ncomp;
  double dt;
  double butcher_a[IVK_MAX_STAGES * IVK_MAX_STAGES];
  /* Layout of the patch gather list / local[] (and so of idx_off, idx,
   * dof_pos, total_m in the patch descriptor):
   *   0 = reference: patch entry a*(nc k+1) + nc*node + comp, pressures at
   *       a*(nc k+1) + nc k (solvers.py:160-166) -- the CTA kernel (k > 32);
   *   1 = fragment: entry node*(nc s) + comp*s + a, then the s pressures at
   *       nc s k + a, each patch padded to an even length -- the warp-per-
   *       patch tensor-core kernel (k <= 32): r lands in its shared-memory
   *       rows and the DMMA output fragments store as 16-byte pairs without
   *       index decode.  dof_pos addresses the same local[] entries, in the
   *       reference's per-DoF summation order, under either layout. */
  int32_t layout;
} ivk_modal_desc;

/* Kronecker eigen-split of the patch matrices.  With all stages sharing one
 * convection Jacobian the stage-coupled patch matrix is
 *   P = I_s (x) M^ + dt A (x) S^,   M^ = [[M_l,0],[0,0]],  S^ = [[K_l+J_l, b],[b^T, 0]]
 * (solvers.py:196-211), so with A = V diag(lam) V^-1:
 *   P^-1 = (V (x) I) blockdiag_k (M^ + dt lam_k S^)^-1 (V^-1 (x) I).
 * One block is stored per real eigenvalue and one per complex-conjugate pair
 * (the conjugate block is its complex conjugate).  Per patch, block k is
 * G_k^T (b = m / s rows): real blocks b x ldr doubles (ldr = (b+3)&~3),
 * complex blocks b x 2*ldc doubles, (re, im) interleaved (ldc = (b+1)&~1 for
 * b <= 64, else (b+3)&~3 so every column starts on a 64-byte DRAM granule).
 * Back-transform: z_i = sum_k scale_k Re(V[i][k] z~_k), scale 1 (real) or 2
 * (pair).  Inverse bytes per patch drop from (s b)^2 to s b^2 doubles. */
typedef struct ivk_kron_desc {
  int32_t nblk;                       /* stored eigen-blocks              */
  int32_t is_complex[IVK_MAX_STAGES];
  double lam_re[IVK_MAX_STAGES], lam_im[IVK_MAX_STAGES];
  double v_re[IVK_MAX_STAGES * IVK_MAX_STAGES];    /* V[i][k], row-major    */
  double v_im[IVK_MAX_STAGES * IVK_MAX_STAGES];
  double vinv_re[IVK_MAX_STAGES * IVK_MAX_STAGES]; /* V^-1[k][i]           */
  double vinv_im[IVK_MAX_STAGES * IVK_MAX_STAGES];
  double scale[IVK_MAX_STAGES];
  /* symmetric != 0 (Stokes: S^ symmetric, so every block and its inverse is
   * complex-symmetric): each block is stored as the lower tile-triangle of
   * 4 x 4 tiles -- tile (I, J), J <= I < nt = ceil(b/4), at index
   * I(I+1)/2 + J, row-major inside the tile, 16 doubles real / 32 complex
   * (re, im interleaved), zero padding past b; a patch's blocks are
   * contiguous. */
  int32_t symmetric;
} ivk_kron_desc;

/* Nested P2/P1 transfer I_s (x) blockdiag(P_P2 (x) I_2, P_P1)
 * (bench.py:187-194, fem.py:255-301), fine <- coarse, plus its transpose. */
typedef struct ivk_transfer_desc {
  int32_t stages;
  int32_t nf_nodes, nf_p;  /* fine scalar P2 nodes, fine P1 nodes        */
  int32_t nc_nodes, nc_p;  /* coarse                                     */
  const int32_t *p2_rowptr, *p2_col; const double* p2_val;    /* nf rows */
  const int32_t *p2t_rowptr, *p2t_col; const double* p2t_val; /* nc rows */
  const int32_t *p1_rowptr, *p1_col; const double* p1_val;
  const int32_t *p1t_rowptr, *p1t_col; const double* p1t_val;
  const uint8_t* fine_constrained;   /* per fine scalar node            */
  const uint8_t* coarse_constrained; /* per coarse scalar node          */
  int32_t ncomp;                     /* velocity components (0/2, or 3) */
} ivk_transfer_desc;

/* Coarsest-level direct solve with fixed LU factors (CoarseSolver,
 * solvers.py:271-292): P_r (A + Z Z^T) P_c = L U, L unit lower.  The
 * factors are stored tile-sparse: 32 x 32 tiles, column-major inside a tile
 * (tile[j*32 + i] = F[32I + i][32K + j]), only nonzero off-diagonal tiles,
 * grouped by block column K (l_colptr: tiles (I > K) of L in column K;
 * u_colptr: tiles (I < K) of U in column K), plus all diagonal tiles.
 * Solve: project pressure means, x = P_c U^-1 L^-1 P_r b, project again. */
typedef struct ivk_coarse_desc {
  int32_t n;               /* = stages * (n_u + n_p)                      */
  int32_t nb;              /* ceil(n / 32) block columns                  */
  int32_t l_ntiles, u_ntiles; /* off-diagonal tile counts                 */
  int32_t stages, n_u, n_p;
  const int32_t* l_colptr; /* nb + 1                                      */
  const int32_t* l_row;    /* block row I of each off-diagonal L tile     */
  const double* l_tiles;   /* 1024 doubles per tile                       */
  const double* l_diag;    /* nb tiles (unit lower; padding = identity)   */
  const int32_t* u_colptr;
  const int32_t* u_row;
  const double* u_tiles;
  const double* u_diag;    /* nb tiles (upper; padding diagonal = 1)      */
  const int32_t* perm_r;   /* (P_r b)[perm_r[i]] = b[i]                   */
  const int32_t* perm_c;   /* x[i] = y[perm_c[i]]                         */
  /* Dense alternative (non-NULL: the tile fields may be NULL): the n x n
   * operator P (A + Z Z^T)^-1 P, P = I - Z Z^T, formed at setup from the same
   * SuperLU factors, row-major with leading dimension dense_ld (multiple of
   * 4); the solve is then one GEMV spread over every SM. */
  const double* dense;
  int32_t dense_ld;
} ivk_coarse_desc;

const char* ivk_last_error(void);
int ivk_version(void);
/* Number of kernels this library launched since load (for gpu_launches). */
int64_t ivk_launch_count(void);

/* out = b - A x  (b != NULL), or out = A x (b == NULL).  out may alias b.
 * Replaces StageSystem.matvec (stages.py:110-126) and the residuals at
 * solvers.py:238,258,263,340. */
int ivk_stage_apply(const ivk_operator_desc* op, const double* x, const double* b,
                    double* out, void* stream);

/* local[slot_pos[idx_off[p] + i]] = sum_j Inv_p[i][j] * r[idx[idx_off[p] + j]]
 * (gather + batched patch solve: einsum at solvers.py:219-220). */
int ivk_patch_apply(const ivk_patch_desc* pd, const double* r, double* local, void* stream);

/* Deterministic scatter (bincount at solvers.py:221) fused with the update:
 * z_d = sum_{k = dof_ptr[d]}^{dof_ptr[d+1]-1} local[k] (contributions in the
 * reference's group/patch order); out_d = alpha * x_d + beta * w_d * z_d
 * (x == NULL -> 0, w == NULL -> 1); if accum != NULL also accum_d += out_d.
 * out may alias x. */
int ivk_patch_combine(const ivk_patch_desc* pd, const double* local, const double* x,
                      double alpha, double beta, const double* w, double* out,
                      double* accum, void* stream);

/* Sharded sweep (shard.py): the same three kernels
 * restricted to one rank's part of the fine level.
 * ivk_stage_apply_slices: K1 on the listed warp slices only (velocity slice
 *   s < ceil(n_nodes/16) covers nodes 16s..16s+15, pressure slice
 *   ceil(n_nodes/16) + t covers P1 nodes 32t..32t+31); other rows of out
 *   are untouched.
 * ivk_patch_combine_list: K4 on the listed DoFs only.
 * ivk_index_copy: dst[dst_idx[i]] = src[src_idx[i]] + beta * dst[dst_idx[i]]
 *   (NULL index = identity) -- halo pack / unpack.
 * ivk_index_update: out[d] = alpha x[d] + beta w[d] z[d] for d in idx. */
int ivk_stage_apply_slices(const ivk_operator_desc* op, const int32_t* slices, int32_t n_slices,
                           const double* x, const double* b, double* out, void* stream);
int ivk_patch_combine_list(const ivk_patch_desc* pd, const int32_t* dofs, int32_t n_dofs,
                           const double* local, const double* x, double alpha, double beta,
                           const double* w, double* out, double* accum, void* stream);
int ivk_index_copy(int64_t n, const int32_t* src_idx, const double* src, const int32_t* dst_idx,
                   double* dst, double beta, void* stream);
int ivk_index_update(int64_t n, const int32_t* idx, double alpha, const double* x, double beta,
                     const double* w, const double* z, double* out, void* stream);

/* Modal-split setup input: for every patch p the k x k scalar blocks
 * Ms[p][alpha][beta] = M_s, Ks[p][alpha][beta] = K_s (zero padded to kmax x
 * kmax) and C[p][alpha][d] = B[nc alpha + d, vertex] (kmax x nc), gathered
 * from the eliminated operator (solvers.py:190-194).  Stokes only (n_conv = 0). */
int ivk_patch_gather_blocks(const ivk_operator_desc* op, const ivk_patch_desc* pd, int32_t kmax,
                            double* Ms, double* Ks, double* C, void* stream);

/* K7m: fill the modal store (pd->modal != NULL) from the gathered blocks, one
 * warp per patch, k <= kmax <= 32 free nodes: Cholesky of M_s, cyclic Jacobi
 * eigendecomposition of L^-1 K_s L^-T, W = L^-T V, c^, the s x s Schur
 * inverse, written as the records described at ivk_modal_desc -- the device
 * twin of scipy.linalg.eigh(K_s, M_s) + np.linalg.inv per patch, replacing
 * np.linalg.inv of the stage-coupled matrix (solvers.py:169-184).
 * singular_dev receives the smallest vertex id whose patch is singular (M_s
 * not positive definite, H not finite or cond_1(H) >= 1e14), else untouched. */
int ivk_modal_factor(const ivk_patch_desc* pd, int32_t kmax, const double* Ms, const double* Ks,
                     const double* C, int32_t* singular_dev, void* stream);

/* Sharded sweep over peer memory: the partial-sum
 * exchange + ordered reduction + x update of a strip-sharded sweep fused into
 * one kernel that reads the other ranks' patch outputs directly (NVLink P2P
 * loads through mapped peer pointers; in-process shards in tests).  For
 * own DoF d = dofs[i]: z = sum over the ranks holding d (holder_rank[
 * holder_ptr[i] .. holder_ptr[i+1]), ascending) of sum_k local_q[dof_pos_q[k]],
 * k in [dof_ptr_q[d], dof_ptr_q[d+1]); x[d] += omega * w[d] * z.  Every rank
 * holding d adds the same terms in the same order: the same bits. */
typedef struct ivk_peer_view {
  const int32_t* dof_ptr;  /* that rank's patch-set tables (global DoF index) */
  const int32_t* dof_pos;
  const double* local;     /* that rank's patch outputs (K3)                  */
} ivk_peer_view;

int ivk_peer_combine_update(int32_t n, const int32_t* dofs, const int32_t* holder_ptr,
                            const int32_t* holder_rank, const ivk_peer_view* peers_dev,
                            double omega, const double* w, double* x, void* stream);

/* Assemble every patch matrix from the operator (solvers.py:186-212) and
 * invert it in place into pd->inv (np.linalg.inv, solvers.py:177) by
 * Gauss-Jordan with partial pivoting.  *singular_dev (device int32, set to
 * INT32_MAX by the caller) receives the smallest singular patch vertex. */
int ivk_patch_factor(const ivk_operator_desc* op, const ivk_patch_desc* pd,
                     int32_t* singular_dev, void* stream);

/* One additive Vanka sweep x_out = x + omega * W * sum_i R_i^T A_i^-1 R_i (b - A x)
 * (apply_vanka, solvers.py:232-239); r and local are caller scratch
 * (dim and total_m doubles).  w == NULL is the reference's unweighted sweep. */
int ivk_vanka_sweep(const ivk_operator_desc* op, const ivk_patch_desc* pd,
                    const double* x, const double* b, double omega, const double* w,
                    double* r, double* local, double* x_out, void* stream);

/* rc = (I_s (x) P)^T rf, constrained coarse rows zeroed (solvers.py:341-342). */
int ivk_restrict(const ivk_transfer_desc* t, const double* rf, double* rc, void* stream);
/* xf += (I_s (x) P) ec on unconstrained fine rows (solvers.py:343-346). */
int ivk_prolong_add(const ivk_transfer_desc* t, const double* ec, double* xf, void* stream);

/* x = CoarseSolver.solve(b) (solvers.py:284-287): tile triangular solves, or
 * one GEMV with c->dense when set; b and x must not alias. */
int ivk_coarse_solve(const ivk_coarse_desc* c, const double* b, double* x, void* stream);

/* Per-stage pressure-mean removal in place (stages.py:174-178): two
 * launches over (IVK_PROJECT_BLOCKS x stages) CTAs -- block partial sums,
 * then every CTA re-adds its stage's partials in block order (deterministic,
 * identical on every CTA) and subtracts the mean from its slice.  `scratch`:
 * caller-owned device memory of IVK_PROJECT_BLOCKS * stages doubles (no
 * initialisation needed). */
#define IVK_PROJECT_BLOCKS 64
int ivk_project_pressure_means(int32_t stages, int32_t n_u, int32_t n_p, double* x,
                               double* scratch, void* stream);
/* out = alpha * x + beta * y (x or y may be NULL -> 0); out may alias. */
int ivk_axpby(int64_t n, double alpha, const double* x, double beta, const double* y,
              double* out, void* stream);
/* out = 0 except out[d] = src[d] on constrained velocity DoFs (the z[cd] = r[cd]
 * seeding of MGHierarchyOp.precondition, solvers.py:352-354). */
int ivk_seed_constrained(int32_t stages, int32_t n_nodes, int32_t ncomp, int32_t n_p,
                         const uint8_t* node_constrained, const double* src,
                         double* out, void* stream);

/* ---- Convection linearisation at Newton cadence (fem.py:199-242) ----------
 * Reference-triangle quadrature (points in the collapsed degree-5 rule) with
 * the P2 basis values and reference gradients at each point. */
typedef struct ivk_quad_table {
  int32_t nq;
  double w[IVK_MAX_QUAD];
  double phi[IVK_MAX_QUAD * 6];       /* [q][a]                             */
  double dphi[IVK_MAX_QUAD * 6 * 2];  /* [q][a][e]                          */
} ivk_quad_table;

typedef struct ivk_convection_desc {
  int32_t n_cells, n_nodes, nnz;
  const ivk_quad_table* quad;  /* HOST pointer                            */
  const int32_t* cell_nodes;   /* C x 6 scalar P2 nodes                    */
  const double* cell_geo;      /* C x 5: Jinv (row-major [e][d]), det J    */
  const int32_t* entry_ptr;    /* nnz + 1                                  */
  const int32_t* entry_contrib;/* cell*36 + a*6 + b, cell-ascending        */
  const int32_t* row_of;       /* nnz: row node of each pattern entry      */
  const int32_t* col;          /* nnz: column node                         */
  const uint8_t* node_constrained; /* eliminated rows/columns -> 0         */
  const int32_t* sell_pos;     /* nnz: position in the SELL-16 copy        */
  const int32_t* node_ptr;     /* n_nodes + 1 (residual map)               */
  const int32_t* node_contrib; /* cell*6 + a                               */
} ivk_convection_desc;

/* Convection Jacobian J_N(u) of the velocity u (interleaved, 2*n_nodes) on
 * the scalar P2 pattern, eliminated, written as (Jxx,Jxy,Jyx,Jyy) per entry
 * to conv (CSR order) and/or conv_s (SELL order); if residual != NULL also
 * N(u) (interleaved).  elem_scratch: C*144 (+ C*12 with residual) doubles. */
int ivk_convection_assemble(const ivk_convection_desc* d, const double* u, double* elem_scratch,
                            double* conv, double* conv_s, double* residual, void* stream);

/* ---- Krylov vector work of FGMRES (solvers.py:388-430), deterministic ----
 * Reductions use a fixed grid of block partials summed in block order by
 * the last block to finish.  `scratch` is caller-owned device memory of
 * ivk_reduction_scratch_bytes() bytes, ZEROED once before first use; the
 * library allocates nothing (graph-capture safe).  Calls sharing one scratch
 * must be stream-ordered: give every concurrent stream its own scratch. */
size_t ivk_reduction_scratch_bytes(void);
/* *result = <x, y> (device scalar). */
int ivk_dot(int64_t n, const double* x, const double* y, double* result, void* scratch,
            void* stream);
/* *result = ||x||_2 (device scalar). */
int ivk_norm(int64_t n, const double* x, double* result, void* scratch, void* stream);
/* Modified Gram-Schmidt of w against V_0..V_{k-1} (rows of V, stride ldv):
 * h[i] = <w, V_i>; w -= h[i] V_i (i ascending); h[k] = ||w||; if v_next:
 * v_next = w / h[k] when h[k] > 1e-300 (solvers.py:401-408).  h is device. */
int ivk_mgs(int64_t n, const double* V, int64_t ldv, int32_t k, double* w, double* h,
            double* v_next, void* scratch, void* stream);
/* FGMRES Givens step on Hessenberg column j (solvers.py:409-421), all on the
 * device: apply rotations 0..j-1 to H[:, j], form rotation j, rotate g, and
 * *est = |g[j+1]|.  H column-major, leading dimension ldh >= j + 2. */
int ivk_givens(int32_t j, int32_t ldh, double* H, double* cs, double* sn, double* g, double* est,
               void* stream);
/* y = triu(H[:k, :k])^-1 g[:k] (back substitution; solvers.py:430). */
int ivk_hessenberg_solve(int32_t k, int32_t ldh, const double* H, const double* g, double* y,
                         void* stream);
/* out = x / coef[k] when coef[k] > 1e-300, else 0 (coef device). */
int ivk_scale(int64_t n, const double* x, const double* coef, int32_t k, double* out,
              void* stream);
/* x += sum_i y[i] Z_i, i ascending (solvers.py:432); y device. */
int ivk_lincomb(int64_t n, const double* Z, int64_t ldz, int32_t k, const double* y, double* x,
                void* stream);

/* ---- General stage-coupled operator (multi-field systems: BASELINE config 5
 * MHD, mhd.py / general.py) -------------------------------------------------
 * The stage system of any spatial operator shared by all stages,
 *   I_s (x) M + dt A (x) L,
 * with M and L given on ONE single-stage CSR pattern as (m, l) pairs, and
 * identity rows on constrained single-stage DoFs (whose rows and columns the
 * caller has already zeroed -- Dirichlet elimination as stages.py:77-85).
 * This is StageSystem.matvec (stages.py:110-126) with the reference's
 * [[M + dt a K, dt a B], [dt a B^T, 0]] structure replaced by a general L.
 * Vectors are stage-major [x_1, ..., x_s], x_i of length n. */
typedef struct ivk_general_desc {
  int32_t stages;
  int32_t n;                /* single-stage DoFs                            */
  int32_t nnz;              /* CSR entries                                  */
  double dt;
  double butcher_a[IVK_MAX_STAGES * IVK_MAX_STAGES];
  const int32_t* rowptr;    /* n + 1, columns sorted per row (K7g)          */
  const int32_t* col;
  const double* ml;         /* nnz * 2: (m, l)                              */
  const int32_t* sptr;      /* SELL-32 copy for K1g: ceil(n/32) + 1         */
  const int32_t* scol;      /* padding: column = the row, values 0          */
  const double* sml;
  const uint8_t* constrained; /* n                                          */
} ivk_general_desc;

/* Single-stage transfer P (fine x coarse CSR) and its explicit transpose,
 * applied as I_s (x) P (bench.py:187-194 generalised to any field layout). */
typedef struct ivk_general_transfer_desc {
  int32_t stages;
  int32_t nf, nc;           /* single-stage fine / coarse DoFs              */
  const int32_t *p_rowptr, *p_col; const double* p_val;     /* nf rows      */
  const int32_t *pt_rowptr, *pt_col; const double* pt_val;  /* nc rows      */
  const uint8_t* fine_constrained;   /* nf                                  */
  const uint8_t* coarse_constrained; /* nc                                  */
} ivk_general_transfer_desc;

/* Device re-linearisation of the 2-D resistive MHD operator (mhd.py, K10g):
 * the element matrices of L at a new frozen state (u0, B0: (n_nodes, 2) nodal
 * P2 values each), one thread per (cell, element row), at the degree-5
 * triangle rule; then every CSR entry sums its (cell, row, column)
 * contributions in cell order (deterministic) into the l half of op->ml and,
 * through sell_pos, of op->sml.  The mass half is state-independent. */
#define IVK_MHD_MAX_QUAD 16
typedef struct ivk_mhd_desc {
  int32_t n_cells, nnz, nq;
  double Re, Rm, S;
  double w[IVK_MHD_MAX_QUAD];
  double phi[IVK_MHD_MAX_QUAD * 6];       /* [q][a]                          */
  double dphi[IVK_MHD_MAX_QUAD * 12];     /* [q][a][e] reference gradients   */
  double psi[IVK_MHD_MAX_QUAD * 3];       /* [q][v]                          */
  double dpsi[6];                         /* [v][e]                          */
  const double* cell_geo;      /* C x 5: Jinv row-major [e][d], det J        */
  const int32_t* cell_nodes;   /* C x 6 scalar P2 nodes                      */
  const int32_t* entry_ptr;    /* nnz + 1                                    */
  const int32_t* entry_contrib;/* cell * 900 + i * 30 + j, cell-ascending    */
  const int32_t* sell_pos;     /* nnz: SELL-32 position of each CSR entry    */
} ivk_mhd_desc;

int ivk_mhd_assemble(const ivk_mhd_desc* d, const double* u0, const double* B0,
                     double* elem_scratch, double* ml, double* sml, void* stream);

/* out = b - A x (b != NULL) or A x; out may alias b.  K1g. */
int ivk_general_apply(const ivk_general_desc* op, const double* x, const double* b, double* out,
                      void* stream);
/* K7g: assemble every patch matrix R_i A R_i^T from the single-stage CSR
 * (the stage-0 block of each patch's idx list is its sorted single-stage DoF
 * list, the same for every stage) and invert it: full (s b)^2 inverses, or
 * the Kronecker eigen-blocks when pd->kron is set (non-symmetric layout).
 * Replaces _patch_matrices + np.linalg.inv (solvers.py:169-212). */
int ivk_general_patch_factor(const ivk_general_desc* op, const ivk_patch_desc* pd,
                             int32_t* singular_dev, void* stream);
/* K1g -> K3 -> K4: x_out = x + omega W sum_i R_i^T A_i^-1 R_i (b - A x). */
int ivk_general_vanka_sweep(const ivk_general_desc* op, const ivk_patch_desc* pd,
                            const double* x, const double* b, double omega, const double* w,
                            double* r, double* local, double* x_out, void* stream);
/* out = 0 except out = src on constrained DoFs of every stage
 * (MGHierarchyOp.precondition z[cd] = r[cd], solvers.py:352-354). */
int ivk_general_seed_constrained(const ivk_general_desc* op, const double* src, double* out,
                                 void* stream);
/* rc = (I_s (x) P)^T rf with constrained coarse rows zeroed; xf += (I_s (x) P) ec
 * on unconstrained fine rows (solvers.py:340-346). */
int ivk_general_restrict(const ivk_general_transfer_desc* t, const double* rf, double* rc,
                         void* stream);
int ivk_general_prolong_add(const ivk_general_transfer_desc* t, const double* ec, double* xf,
                            void* stream);

#ifdef __cplusplus
}
#endif
#endif /* IVK_H */
