// K2-K4 and K7: the vertex-star Vanka patch set on sm_100a, fp64.
//
//  K2+K3 ivk_patch_apply   gather r at each patch's DoFs and apply the stored
//                          dense inverse (solvers.py:218-220).  HBM-bound: the
//                          inverse store is streamed exactly once per sweep
//                          with 256-bit evict-first loads; r stays in L2.
//  K4    ivk_patch_combine deterministic owner-computes scatter-add
//                          (np.bincount, solvers.py:221) fused with the sweep
//                          update x + omega * W * z (solvers.py:239).
//  K7    ivk_patch_factor  assemble each stage-coupled patch matrix from the
//                          scalar operator (solvers.py:186-212) and invert it
//                          by Gauss-Jordan with partial pivoting in shared
//                          memory (replaces np.linalg.inv, solvers.py:177).

#include <climits>
#include <cstdlib>

#include "ivk_common.cuh"
#include "ivk_gj.cuh"

namespace ivk {

int validate_op(const ivk_operator_desc* d);         // ivk_operator.cu
int validate_general(const ivk_general_desc* d);     // ivk_general.cu

struct PatchParams {
  int num_patches, dim, max_m, total_m;
  const int32_t* __restrict__ idx_off;
  const int32_t* __restrict__ idx;
  const int64_t* __restrict__ inv_off;
  double* inv;
  const int32_t* __restrict__ dof_ptr;
  const int32_t* __restrict__ dof_pos;
  const int32_t* __restrict__ vertex;
  const int32_t* __restrict__ node_off;
  const int32_t* __restrict__ node;
  const int32_t* __restrict__ slot_pos;
};

// dedup tables (kept out of PatchParams: the per-patch kernels' register
// allocation is sensitive to their parameter block)
struct DedupParams {
  int n_classes, n_tiles;
  const int64_t* __restrict__ class_inv_off;
  const double* __restrict__ class_inv;
  const int32_t* __restrict__ tile_start;
  const int32_t* __restrict__ tile_class;
  const int32_t* __restrict__ tile_off;
  const int32_t* __restrict__ cidx;
  const int32_t* __restrict__ cdst;
};

static PatchParams make_patch_params(const ivk_patch_desc* d) {
  PatchParams p;
  p.num_patches = d->num_patches;
  p.dim = d->dim;
  p.max_m = d->max_m;
  p.total_m = d->total_m;
  p.idx_off = d->idx_off;
  p.idx = d->idx;
  p.inv_off = d->inv_off;
  p.inv = d->inv;
  p.dof_ptr = d->dof_ptr;
  p.dof_pos = d->dof_pos;
  p.vertex = d->vertex;
  p.node_off = d->node_off;
  p.node = d->node;
  p.slot_pos = d->slot_pos;
  return p;
}

static int validate_patches(const ivk_patch_desc* d) {
  IVK_REQUIRE(d != nullptr, "patch descriptor is NULL");
  IVK_REQUIRE(d->num_patches > 0 && d->dim > 0 && d->max_m > 0, "empty patch set");
  IVK_REQUIRE(d->idx_off && d->idx && d->inv_off && d->inv && d->dof_ptr &&
                  (d->slot_pos || d->dof_pos),
              "patch descriptor has a NULL array");
  return IVK_OK;
}

// ------------------------------------------------------------------ K2+K3
//
// One warp per patch.  Lane t owns output rows 4t..4t+3 of a 128-row chunk;
// for each column j it issues one 256-bit streaming load of Inv^T[j][4t..4t+3]
// (a warp reads 1 KB contiguous per j) and broadcasts r_p[j] from shared
// memory.  Patches wider than 128 loop over row chunks.
constexpr int kApplyWarps = 8;
constexpr int kRowsPerWarp = 128;
constexpr int kUnroll = 4;  // 4 x 32 B in flight per lane; ~48 regs -> 40 warps/SM

// Patch-local results are re-read by the scatter right after: keep them in L2.
__device__ __forceinline__ void st_keep(double* p, double v) {
  asm volatile(
      "{\n\t.reg .b64 pol;\n\t"
      "createpolicy.fractional.L2::evict_last.b64 pol, 1.0;\n\t"
      "st.global.L1::no_allocate.L2::cache_hint.f64 [%0], %1, pol;\n\t}"
      :: "l"(p), "d"(v) : "memory");
}

__device__ __forceinline__ void ld_stream4(const double* p, double& a, double& b, double& c,
                                           double& d) {
  asm volatile("ld.global.L1::no_allocate.L2::evict_first.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(a), "=d"(b), "=d"(c), "=d"(d)
               : "l"(p));
}

template <int MAXM>
__global__ void __launch_bounds__(kApplyWarps * 32) patch_apply_kernel(PatchParams pd,
                                                                       const double* __restrict__ r,
                                                                       double* __restrict__ local) {
  __shared__ __align__(16) double rs_all[kApplyWarps][MAXM];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* rs = rs_all[warp];
  const int stride = gridDim.x * kApplyWarps;
  for (int p = blockIdx.x * kApplyWarps + warp; p < pd.num_patches; p += stride) {
    const int off = pd.idx_off[p];
    const int m = pd.idx_off[p + 1] - off;
    const int ld = (m + 3) & ~3;
    for (int j = lane; j < m; j += 32) rs[j] = __ldg(r + pd.idx[off + j]);
    __syncwarp();
    const double* inv = pd.inv + pd.inv_off[p];
    for (int row0 = 0; row0 < m; row0 += kRowsPerWarp) {
      const int i0 = row0 + 4 * lane;
      if (i0 < ld) {
        double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
        const double* col = inv + i0;
        int j = 0;
#pragma unroll 1
        for (; j + kUnroll <= m; j += kUnroll) {
          double v[kUnroll][4];
#pragma unroll
          for (int u = 0; u < kUnroll; ++u)
            ld_stream4(col + (long)(j + u) * ld, v[u][0], v[u][1], v[u][2], v[u][3]);
#pragma unroll
          for (int u = 0; u < kUnroll; ++u) {
            const double rj = rs[j + u];
            acc0 = fma(v[u][0], rj, acc0);
            acc1 = fma(v[u][1], rj, acc1);
            acc2 = fma(v[u][2], rj, acc2);
            acc3 = fma(v[u][3], rj, acc3);
          }
        }
        for (; j < m; ++j) {
          double v0, v1, v2, v3;
          ld_stream4(col + (long)j * ld, v0, v1, v2, v3);
          const double rj = rs[j];
          acc0 = fma(v0, rj, acc0);
          acc1 = fma(v1, rj, acc1);
          acc2 = fma(v2, rj, acc2);
          acc3 = fma(v3, rj, acc3);
        }
        if (pd.slot_pos) {
          const int32_t* sp = pd.slot_pos + off + i0;
          if (i0 + 0 < m) st_keep(local + sp[0], acc0);
          if (i0 + 1 < m) st_keep(local + sp[1], acc1);
          if (i0 + 2 < m) st_keep(local + sp[2], acc2);
          if (i0 + 3 < m) st_keep(local + sp[3], acc3);
        } else {
          double* out = local + off + i0;
          if (i0 + 0 < m) st_keep(out + 0, acc0);
          if (i0 + 1 < m) st_keep(out + 1, acc1);
          if (i0 + 2 < m) st_keep(out + 2, acc2);
          if (i0 + 3 < m) st_keep(out + 3, acc3);
        }
      }
    }
    __syncwarp();
  }
}

// -------------------------------------------------------------------- K4

// dofs != NULL: only the listed DoFs (a shard's patch DoFs, shard.py).
__global__ void patch_combine_kernel(PatchParams pd, const double* __restrict__ local,
                                     const double* x, double alpha, double beta,
                                     const double* __restrict__ w, double* out, double* accum,
                                     const int32_t* __restrict__ dofs, int n_dofs) {
  const int n = dofs ? n_dofs : pd.dim;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int d = dofs ? dofs[i] : i;
    const int k0 = pd.dof_ptr[d], k1 = pd.dof_ptr[d + 1];
    double z = 0.0;
    if (pd.slot_pos) {
      for (int k = k0; k < k1; ++k) z += local[k];
    } else {
      // up to 8 contributions per round: all position loads, then all value
      // loads in flight (a 2-D vertex DoF has 7: one round trip pair instead
      // of a batch of 4 plus 3 dependent singles); summed in slot order
      constexpr int U = 8;
      for (int k = k0; k < k1; k += U) {
        int pp[U];
        double v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) pp[u] = k + u < k1 ? __ldg(pd.dof_pos + k + u) : -1;
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = pp[u] >= 0 ? local[pp[u]] : 0.0;
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (pp[u] >= 0) z += v[u];
      }
    }
    double v = beta * (w ? w[d] : 1.0) * z;
    if (x) v = alpha * x[d] + v;
    out[d] = v;
    if (accum) accum[d] += v;
  }
}

// K4p: the sharded sweep's exchange + ordered reduction + update in one
// kernel over peer memory (ivk_peer_combine_update).
__global__ void peer_combine_update_kernel(int n, const int32_t* __restrict__ dofs,
                                           const int32_t* __restrict__ holder_ptr,
                                           const int32_t* __restrict__ holder_rank,
                                           const ivk_peer_view* __restrict__ peers,
                                           double omega, const double* __restrict__ w,
                                           double* __restrict__ x) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int d = dofs[i];
    double z = 0.0;
    for (int h = holder_ptr[i]; h < holder_ptr[i + 1]; ++h) {
      const ivk_peer_view pv = peers[holder_rank[h]];
      const int k0 = pv.dof_ptr[d], k1 = pv.dof_ptr[d + 1];
      for (int k = k0; k < k1; ++k) z += pv.local[pv.dof_pos[k]];
    }
    x[d] = fma(omega * (w ? w[d] : 1.0), z, x[d]);
  }
}

// -------------------------------------------------------------------- K7

struct FactorParams {
  int n_nodes, n_p, n_conv, nnz, S;
  double dt;
  double a[IVK_MAX_STAGES * IVK_MAX_STAGES];
  const int32_t* __restrict__ p2_rowptr;
  const int32_t* __restrict__ p2_col;
  const double2* __restrict__ p2_mk;
  const double4* __restrict__ conv;
  const int32_t* __restrict__ b_rowptr;
  const int32_t* __restrict__ b_col;
  const double2* __restrict__ b_val;
  const double* __restrict__ b_raw;  // ncomp values per entry
  int ncomp;
};

static FactorParams make_factor_params(const ivk_operator_desc* op) {
  FactorParams f;
  f.n_nodes = op->n_nodes;
  f.n_p = op->n_p;
  f.n_conv = op->n_conv;
  f.nnz = op->nnz;
  f.S = op->stages;
  f.dt = op->dt;
  for (int i = 0; i < IVK_MAX_STAGES * IVK_MAX_STAGES; ++i) f.a[i] = op->butcher_a[i];
  f.p2_rowptr = op->p2_rowptr;
  f.p2_col = op->p2_col;
  f.p2_mk = reinterpret_cast<const double2*>(op->p2_mk);
  f.conv = reinterpret_cast<const double4*>(op->conv);
  f.b_rowptr = op->b_rowptr;
  f.b_col = op->b_col;
  f.b_val = reinterpret_cast<const double2*>(op->b_val);
  f.b_raw = op->b_val;
  f.ncomp = op->ncomp == 3 ? 3 : 2;
  return f;
}

// Position of `col` in the sorted CSR row [lo, hi), or -1.
__device__ __forceinline__ int find_col(const int32_t* __restrict__ cols, int lo, int hi, int col) {
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    const int c = cols[mid];
    if (c == col) return mid;
    if (c < col) lo = mid + 1; else hi = mid;
  }
  return -1;
}

constexpr int kFactorThreads = 512;

// Assemble the stage-coupled d x d patch matrix (row-major, leading dimension
// d) into shared memory.  Local layout (solvers.py:160-165, 196-211): stage
// block a occupies rows a*(mv+1) .. a*(mv+1)+mv, velocity DoFs 2*alpha + c
// for the patch's free nodes, then the vertex pressure.  Ends with a barrier.
__device__ __forceinline__ void assemble_full_patch(const FactorParams& op, double* A,
                                                    const int* __restrict__ nodes, int nk, int v) {
  const int S = op.S;
  const int mv = 2 * nk, blk = mv + 1, d = S * blk;
  const int tid = threadIdx.x;
  for (int e = tid; e < d * d; e += blockDim.x) A[e] = 0.0;
  __syncthreads();

  // Velocity-velocity blocks: M delta_ab + dt a_ab (K + J_a).
  for (int pr = tid; pr < nk * nk; pr += blockDim.x) {
    const int al = pr / nk, be = pr % nk;
    const int row = nodes[al];
    const int pos = find_col(op.p2_col, op.p2_rowptr[row], op.p2_rowptr[row + 1], nodes[be]);
    if (pos < 0) continue;  // not coupled: zero block
    const double2 mk = op.p2_mk[pos];
    for (int a = 0; a < S; ++a) {
      double4 J = make_double4(0.0, 0.0, 0.0, 0.0);
      if (op.n_conv == 1) J = op.conv[pos];
      else if (op.n_conv > 1) J = op.conv[(long)a * op.nnz + pos];
      for (int b = 0; b < S; ++b) {
        const double f = op.dt * op.a[a * S + b];
        const double diag = (a == b ? mk.x : 0.0) + f * mk.y;
        double* base = A + (long)(a * blk + 2 * al) * d + b * blk + 2 * be;
        base[0] = diag + f * J.x;
        base[1] = f * J.y;
        base[d] = f * J.z;
        base[d + 1] = diag + f * J.w;
      }
    }
  }
  // Velocity-pressure couplings with the patch vertex: dt a_ab B[vel, v].
  for (int al = tid; al < nk; al += blockDim.x) {
    const int row = nodes[al];
    const int pos = find_col(op.b_col, op.b_rowptr[row], op.b_rowptr[row + 1], v);
    const double2 bv = pos >= 0 ? op.b_val[pos] : make_double2(0.0, 0.0);
    for (int a = 0; a < S; ++a)
      for (int b = 0; b < S; ++b) {
        const double f = op.dt * op.a[a * S + b];
        const int r0 = a * blk + 2 * al, c0 = b * blk + 2 * al;
        A[(long)r0 * d + b * blk + mv] = f * bv.x;
        A[(long)(r0 + 1) * d + b * blk + mv] = f * bv.y;
        A[(long)(a * blk + mv) * d + c0] = f * bv.x;
        A[(long)(a * blk + mv) * d + c0 + 1] = f * bv.y;
      }
  }
  __syncthreads();
}

// K7 (d <= 16 RT, TX CT): one CTA of 16 TX threads per patch; the matrix is
// assembled in dynamic shared memory (d x ld doubles), inverted in registers
// (ivk_gj.cuh), which leaves Inv^T with leading dimension ld there, and copied out.
template <int TX, int RT, int CT, int MINB>
__global__ void __launch_bounds__(16 * TX, MINB) patch_factor_reg_kernel(FactorParams op, PatchParams pd,
                                                                         int32_t* singular) {
  extern __shared__ __align__(16) double A[];
  __shared__ GjScratch<false, 16 * RT, TX * CT> gj;
  const int p = blockIdx.x;
  const int n0 = pd.node_off[p], nk = pd.node_off[p + 1] - n0;
  const int v = pd.vertex[p];
  const int d = op.S * (2 * nk + 1);
  const int tid = threadIdx.x;
  assemble_full_patch(op, A, pd.node + n0, nk, v);
  const int ld = (d + 3) & ~3;
  if (!gj_invert_registers<false, TX, RT, CT>(A, nullptr, d, ld, gj)) {
    if (tid == 0) atomicMin(singular, v);
    return;
  }
  // A now holds Inv^T with leading dimension ld: a straight 16-byte copy
  double2* out = reinterpret_cast<double2*>(pd.inv + pd.inv_off[p]);
  const double2* src = reinterpret_cast<const double2*>(A);
  for (int e = tid; e < d * ld / 2; e += blockDim.x) out[e] = src[e];
}

// One CTA per patch (d > 128); the d x d matrix lives in dynamic shared memory
// (row-major, leading dimension d) through the whole elimination.
__global__ void __launch_bounds__(kFactorThreads) patch_factor_kernel(FactorParams op, PatchParams pd,
                                                                      int32_t* singular) {
  extern __shared__ __align__(16) double A[];
  __shared__ int piv[512];
  __shared__ double colk[512];
  __shared__ int s_prow;
  __shared__ int s_bad;
  const int p = blockIdx.x;
  const int S = op.S;
  const int n0 = pd.node_off[p], nk = pd.node_off[p + 1] - n0;
  const int v = pd.vertex[p];
  const int mv = 2 * nk, blk = mv + 1, d = S * blk;
  const int tid = threadIdx.x;
  if (tid == 0) s_bad = 0;
  assemble_full_patch(op, A, pd.node + n0, nk, v);

  // In-place Gauss-Jordan inverse with row pivoting (first max |pivot|, as
  // LAPACK idamax); columns are unscrambled at the end.
  for (int k = 0; k < d; ++k) {
    if (tid < 32) {
      double best = -1.0;
      int bi = k;
      for (int i = k + tid; i < d; i += 32) {
        const double a = fabs(A[(long)i * d + k]);
        if (a > best) { best = a; bi = i; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_down_sync(0xffffffffu, best, o);
        const int oi = __shfl_down_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      if (tid == 0) {
        s_prow = bi;
        piv[k] = bi;
        if (!(best > 0.0)) s_bad = 1;
      }
    }
    __syncthreads();
    if (s_bad) break;
    const int pr = s_prow;
    if (pr != k) {
      for (int j = tid; j < d; j += blockDim.x) {
        const double t = A[(long)k * d + j];
        A[(long)k * d + j] = A[(long)pr * d + j];
        A[(long)pr * d + j] = t;
      }
      __syncthreads();
    }
    const double pinv = 1.0 / A[(long)k * d + k];
    for (int i = tid; i < d; i += blockDim.x) colk[i] = (i == k) ? 0.0 : A[(long)i * d + k];
    __syncthreads();
    for (int j = tid; j < d; j += blockDim.x)
      A[(long)k * d + j] = (j == k) ? pinv : A[(long)k * d + j] * pinv;
    __syncthreads();
    for (int e = tid; e < d * d; e += blockDim.x) {
      const int i = e / d, j = e - i * d;
      if (i == k) continue;
      const double f = colk[i];
      const double base = (j == k) ? 0.0 : A[e];
      A[e] = base - f * A[(long)k * d + j];
    }
    __syncthreads();
  }
  if (s_bad) {
    if (tid == 0) atomicMin(singular, v);
    return;
  }
  for (int k = d - 1; k >= 0; --k) {
    const int pk = piv[k];
    if (pk != k) {
      for (int i = tid; i < d; i += blockDim.x) {
        const double t = A[(long)i * d + k];
        A[(long)i * d + k] = A[(long)i * d + pk];
        A[(long)i * d + pk] = t;
      }
      __syncthreads();
    }
  }
  // Store Inv^T with leading dimension ld: inv[j*ld + i] = Inv[i][j].
  const int ld = (d + 3) & ~3;
  double* out = pd.inv + pd.inv_off[p];
  for (int e = tid; e < d * ld; e += blockDim.x) {
    const int j = e / ld, i = e - j * ld;
    out[e] = (i < d) ? A[(long)i * d + j] : 0.0;
  }
}


// Patches too large for shared memory (3-D: d = s (3k + 1) ~ 400): one CTA
// per patch (persistent), the matrix held in its own slot of the inverse
// store.  The TRANSPOSE A^T is assembled (row-major, leading dimension ld)
// and inverted in place by Gauss-Jordan with row pivoting -- (A^T)^-1 =
// (A^-1)^T is exactly the Inv^T layout K3 streams, so no scratch and no
// final transpose.  Pivot row and multiplier column are staged in shared
// memory each step; the d x d update streams through L2.
constexpr int kFactorGlobalThreads = 1024;

template <int NC>
__global__ void __launch_bounds__(kFactorGlobalThreads) patch_factor_global_kernel(
    FactorParams op, PatchParams pd, int32_t* singular) {
  __shared__ double prow[512];
  __shared__ double colk[512];
  __shared__ int piv[512];
  __shared__ int s_prow, s_bad;
  const int tid = threadIdx.x;
  const int S = op.S;
  for (int p = blockIdx.x; p < pd.num_patches; p += gridDim.x) {
    const int n0 = pd.node_off[p], nk = pd.node_off[p + 1] - n0;
    const int* nodes = pd.node + n0;
    const int v = pd.vertex[p];
    const int mv = NC * nk, blk = mv + 1, d = S * blk;
    const int ld = (d + 3) & ~3;
    double* B = pd.inv + pd.inv_off[p];  // B[r * ld + c] = A[c][r]
    for (int e = tid; e < d * ld; e += blockDim.x) B[e] = 0.0;
    if (tid == 0) s_bad = 0;
    __syncthreads();
    for (int pr = tid; pr < nk * nk; pr += blockDim.x) {
      const int al = pr / nk, be = pr % nk;
      const int row = nodes[al];
      const int pos = find_col(op.p2_col, op.p2_rowptr[row], op.p2_rowptr[row + 1], nodes[be]);
      if (pos < 0) continue;
      const double2 mk = op.p2_mk[pos];
      for (int a = 0; a < S; ++a)
        for (int b = 0; b < S; ++b) {
          const double f = op.dt * op.a[a * S + b];
          const double val = (a == b ? mk.x : 0.0) + f * mk.y;
          for (int cc = 0; cc < NC; ++cc) {
            const int r = a * blk + NC * al + cc, col = b * blk + NC * be + cc;
            B[(long)col * ld + r] = val;
          }
        }
    }
    for (int al = tid; al < nk; al += blockDim.x) {
      const int row = nodes[al];
      const int pos = find_col(op.b_col, op.b_rowptr[row], op.b_rowptr[row + 1], v);
      for (int cc = 0; cc < NC; ++cc) {
        const double bv = pos >= 0 ? op.b_raw[(long)pos * NC + cc] : 0.0;
        for (int a = 0; a < S; ++a)
          for (int b = 0; b < S; ++b) {
            const double f = op.dt * op.a[a * S + b];
            const int r = a * blk + NC * al + cc;
            B[(long)(b * blk + mv) * ld + r] = f * bv;   // A[r][b*blk + mv]
            B[(long)(b * blk + NC * al + cc) * ld + a * blk + mv] = f * bv;  // A[a*blk+mv][.]
          }
      }
    }
    __syncthreads();
    for (int k = 0; k < d; ++k) {
      if (tid < 32) {
        double best = -1.0;
        int bi = k;
        for (int i = k + tid; i < d; i += 32) {
          const double a = fabs(B[(long)i * ld + k]);
          if (a > best) { best = a; bi = i; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double ob = __shfl_down_sync(0xffffffffu, best, o);
          const int oi = __shfl_down_sync(0xffffffffu, bi, o);
          if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
        }
        if (tid == 0) {
          s_prow = bi;
          piv[k] = bi;
          if (!(best > 0.0)) s_bad = 1;
        }
      }
      __syncthreads();
      if (s_bad) break;
      const int pr = s_prow;
      // pivot row (swapped in) scaled, and the multiplier column
      const double pinv = 1.0 / B[(long)pr * ld + k];
      for (int j = tid; j < d; j += blockDim.x) {
        const double t = B[(long)pr * ld + j];
        prow[j] = (j == k) ? pinv : t * pinv;
      }
      for (int i = tid; i < d; i += blockDim.x)
        colk[i] = (i == pr) ? B[(long)k * ld + k] : B[(long)i * ld + k];
      __syncthreads();
      // row pr <- old row k (the swap); then every row i != k updated
      if (pr != k)
        for (int j = tid; j < d; j += blockDim.x) B[(long)pr * ld + j] = B[(long)k * ld + j];
      __syncthreads();
      {
        const int warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5;
        for (int i = warp; i < d; i += nw) {
          double* arow = B + (long)i * ld;
          const double f = colk[i];
          if (i == k) {
            for (int j = lane; j < d; j += 32) arow[j] = prow[j];
          } else {
            for (int j = lane; j < d; j += 32) {
              const double base = (j == k) ? 0.0 : arow[j];
              arow[j] = base - f * prow[j];
            }
          }
        }
      }
      __syncthreads();
    }
    if (s_bad) {
      if (tid == 0) atomicMin(singular, v);
      __syncthreads();
      continue;
    }
    for (int k = d - 1; k >= 0; --k) {
      const int pk = piv[k];
      if (pk != k) {
        for (int i = tid; i < d; i += blockDim.x) {
          const double t = B[(long)i * ld + k];
          B[(long)i * ld + k] = B[(long)i * ld + pk];
          B[(long)i * ld + pk] = t;
        }
      }
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------- Kronecker split
//
// K7e / K3e: the eigen-split formulation (include/ivk.h, ivk_kron_desc).

struct KronParams {
  int nblk, S;
  int is_complex[IVK_MAX_STAGES];
  double lam_re[IVK_MAX_STAGES], lam_im[IVK_MAX_STAGES];
  double v_re[IVK_MAX_STAGES * IVK_MAX_STAGES], v_im[IVK_MAX_STAGES * IVK_MAX_STAGES];
  double vinv_re[IVK_MAX_STAGES * IVK_MAX_STAGES], vinv_im[IVK_MAX_STAGES * IVK_MAX_STAGES];
  double scale[IVK_MAX_STAGES];
  int symmetric;
};

static KronParams make_kron(const ivk_kron_desc* k, int S) {
  KronParams p;
  p.nblk = k->nblk;
  p.S = S;
  p.symmetric = k->symmetric;
  for (int i = 0; i < IVK_MAX_STAGES; ++i) {
    p.is_complex[i] = k->is_complex[i];
    p.lam_re[i] = k->lam_re[i];
    p.lam_im[i] = k->lam_im[i];
    p.scale[i] = k->scale[i];
  }
  for (int i = 0; i < IVK_MAX_STAGES * IVK_MAX_STAGES; ++i) {
    p.v_re[i] = k->v_re[i];
    p.v_im[i] = k->v_im[i];
    p.vinv_re[i] = k->vinv_re[i];
    p.vinv_im[i] = k->vinv_im[i];
  }
  return p;
}

__host__ __device__ __forceinline__ int kron_ldr(int b) { return (b + 3) & ~3; }
// Complex columns: even length up to b = 64 (the narrow K3e / K3d layout the
// cfg2 kernels are tuned on), then padded to 64-byte DRAM granules (b > 64:
// MHD b = 78 -> 80, 3-D b = 176) so no granule straddles two columns.
__host__ __device__ __forceinline__ int kron_ldc_narrow(int b) { return (b + 1) & ~1; }
__host__ __device__ __forceinline__ int kron_ldc(int b) {
  return b <= 64 ? kron_ldc_narrow(b) : (b + 3) & ~3;
}
// symmetric storage: the lower tile-triangle of 4x4 tiles (I >= J, nt =
// ceil(b/4)), ordered by tile diagonal d = I - J and, inside a diagonal,
// chunk-major: the q-th 32-byte chunk of tile (d + t, t) at
// base_d + 4 (q (nt - d) + t), base_d = 4 QC sum_{d' < d} (nt - d'), QC = 4
// (real: chunk q = tile row q) or 8 (complex: row q/2, columns 2(q%2)..+1,
// (re, im) interleaved).  Zero padding past b.
__host__ __device__ __forceinline__ int kron_sym_block(bool cplx, int b) {
  const int nt = (b + 3) >> 2;
  return (cplx ? 32 : 16) * (nt * (nt + 1) / 2);
}
__host__ __device__ __forceinline__ int kron_sym_doubles(const KronParams& kp, int b) {
  int n = 0;
  for (int k = 0; k < kp.nblk; ++k) n += kron_sym_block(kp.is_complex[k] != 0, b);
  return n;
}

// In-place Gauss-Jordan inverse (row pivoting, first max of |re|+|im|) of a
// d x d matrix held as separate re/im arrays in shared memory.
template <bool CPLX>
__device__ bool gauss_jordan(double* Are, double* Aim, int d, int* piv, double* colre,
                             double* colim, int* s_prow, int* s_bad) {
  const int tid = threadIdx.x;
  for (int k = 0; k < d; ++k) {
    if (tid < 32) {
      double best = -1.0;
      int bi = k;
      for (int i = k + tid; i < d; i += 32) {
        double a = fabs(Are[i * d + k]);
        if (CPLX) a += fabs(Aim[i * d + k]);
        if (a > best) { best = a; bi = i; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_down_sync(0xffffffffu, best, o);
        const int oi = __shfl_down_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      if (tid == 0) {
        *s_prow = bi;
        piv[k] = bi;
        if (!(best > 0.0)) *s_bad = 1;
      }
    }
    __syncthreads();
    if (*s_bad) return false;
    const int pr = *s_prow;
    if (pr != k) {
      for (int j = tid; j < d; j += blockDim.x) {
        double t = Are[k * d + j]; Are[k * d + j] = Are[pr * d + j]; Are[pr * d + j] = t;
        if (CPLX) { t = Aim[k * d + j]; Aim[k * d + j] = Aim[pr * d + j]; Aim[pr * d + j] = t; }
      }
      __syncthreads();
    }
    double pr_re = Are[k * d + k], pr_im = CPLX ? Aim[k * d + k] : 0.0;
    double inv_re, inv_im = 0.0;
    if (CPLX) {
      const double den = pr_re * pr_re + pr_im * pr_im;
      inv_re = pr_re / den;
      inv_im = -pr_im / den;
    } else {
      inv_re = 1.0 / pr_re;
    }
    for (int i = tid; i < d; i += blockDim.x) {
      colre[i] = (i == k) ? 0.0 : Are[i * d + k];
      if (CPLX) colim[i] = (i == k) ? 0.0 : Aim[i * d + k];
    }
    __syncthreads();
    for (int j = tid; j < d; j += blockDim.x) {
      if (j == k) {
        Are[k * d + k] = inv_re;
        if (CPLX) Aim[k * d + k] = inv_im;
      } else if (CPLX) {
        const double a = Are[k * d + j], b = Aim[k * d + j];
        Are[k * d + j] = a * inv_re - b * inv_im;
        Aim[k * d + j] = a * inv_im + b * inv_re;
      } else {
        Are[k * d + j] *= inv_re;
      }
    }
    __syncthreads();
    for (int e = tid; e < d * d; e += blockDim.x) {
      const int i = e / d, j = e - i * d;
      if (i == k) continue;
      const double fr = colre[i];
      const double br = (j == k) ? 0.0 : Are[e];
      const double pr2 = Are[k * d + j];
      if (CPLX) {
        const double fi = colim[i];
        const double bi = (j == k) ? 0.0 : Aim[e];
        const double pi2 = Aim[k * d + j];
        Are[e] = br - (fr * pr2 - fi * pi2);
        Aim[e] = bi - (fr * pi2 + fi * pr2);
      } else {
        Are[e] = br - fr * pr2;
      }
    }
    __syncthreads();
  }
  for (int k = d - 1; k >= 0; --k) {
    const int pk = piv[k];
    if (pk != k) {
      for (int i = tid; i < d; i += blockDim.x) {
        double t = Are[i * d + k]; Are[i * d + k] = Are[i * d + pk]; Are[i * d + pk] = t;
        if (CPLX) { t = Aim[i * d + k]; Aim[i * d + k] = Aim[i * d + pk]; Aim[i * d + pk] = t; }
      }
      __syncthreads();
    }
  }
  return true;
}

constexpr int kKronFactorThreads = 256;

// One CTA per patch; for every stored eigen-block assemble M^ + dt lam S^
// (b x b) and invert it.  Dynamic smem: 2 * bmax^2 doubles.
template <int RT, int CT, int MINB>
__global__ void __launch_bounds__(kKronFactorThreads, MINB) patch_factor_kron_kernel(
    FactorParams op, PatchParams pd, KronParams kp, int32_t* singular) {
  extern __shared__ __align__(16) double sm[];
  __shared__ GjScratch<true, 16 * RT, 16 * CT> gj;
  const int p = blockIdx.x;
  const int n0 = pd.node_off[p], nk = pd.node_off[p + 1] - n0;
  const int* nodes = pd.node + n0;
  const int v = pd.vertex[p];
  const int mv = 2 * nk, b = mv + 1;
  const int tid = threadIdx.x;
  double* Are = sm;
  double* Aim = sm + b * kron_ldr(b);
  double* out = pd.inv + pd.inv_off[p];
  for (int k = 0; k < kp.nblk; ++k) {
    const bool cplx = kp.is_complex[k] != 0;
    const double fre = op.dt * kp.lam_re[k], fim = op.dt * kp.lam_im[k];
    for (int e = tid; e < b * b; e += blockDim.x) { Are[e] = 0.0; Aim[e] = 0.0; }
    __syncthreads();
    for (int pr = tid; pr < nk * nk; pr += blockDim.x) {
      const int al = pr / nk, be = pr % nk;
      const int row = nodes[al];
      const int pos = find_col(op.p2_col, op.p2_rowptr[row], op.p2_rowptr[row + 1], nodes[be]);
      if (pos < 0) continue;
      const double2 mk = op.p2_mk[pos];
      double4 J = make_double4(0.0, 0.0, 0.0, 0.0);
      if (op.n_conv >= 1) J = op.conv[pos];
      // S^ entries of the 2x2 node block, then M^ + dt lam S^
      const double s00 = mk.y + J.x, s01 = J.y, s10 = J.z, s11 = mk.y + J.w;
      const int r0 = 2 * al, c0 = 2 * be;
      Are[r0 * b + c0] = mk.x + fre * s00;
      Are[r0 * b + c0 + 1] = fre * s01;
      Are[(r0 + 1) * b + c0] = fre * s10;
      Are[(r0 + 1) * b + c0 + 1] = mk.x + fre * s11;
      Aim[r0 * b + c0] = fim * s00;
      Aim[r0 * b + c0 + 1] = fim * s01;
      Aim[(r0 + 1) * b + c0] = fim * s10;
      Aim[(r0 + 1) * b + c0 + 1] = fim * s11;
    }
    for (int al = tid; al < nk; al += blockDim.x) {
      const int row = nodes[al];
      const int pos = find_col(op.b_col, op.b_rowptr[row], op.b_rowptr[row + 1], v);
      const double2 bv = pos >= 0 ? op.b_val[pos] : make_double2(0.0, 0.0);
      const int r0 = 2 * al;
      Are[r0 * b + mv] = fre * bv.x;
      Are[(r0 + 1) * b + mv] = fre * bv.y;
      Are[mv * b + r0] = fre * bv.x;
      Are[mv * b + r0 + 1] = fre * bv.y;
      Aim[r0 * b + mv] = fim * bv.x;
      Aim[(r0 + 1) * b + mv] = fim * bv.y;
      Aim[mv * b + r0] = fim * bv.x;
      Aim[mv * b + r0 + 1] = fim * bv.y;
    }
    __syncthreads();
    // leaves G^T in Are / Aim with the leading dimension of the stored block
    const int ldo = kp.symmetric ? b : (cplx ? kron_ldc(b) : kron_ldr(b));
    const bool ok = cplx ? gj_invert_registers<true, 16, RT, CT>(Are, Aim, b, ldo, gj)
                         : gj_invert_registers<false, 16, RT, CT>(Are, Aim, b, ldo, gj);
    if (!ok) {
      if (tid == 0) atomicMin(singular, v);
      return;
    }
    // store G^T, or the lower tile-triangle of (G + G^T) / 2 (diagonal order)
    if (kp.symmetric) {
      const int nt = (b + 3) >> 2;
      const int qc = cplx ? 8 : 4;
      const int total = kron_sym_block(cplx, b);
      for (int e = tid; e < total; e += blockDim.x) {
        // e -> (d, q, t, w): w = element within the 4-double chunk
        int d = 0, base = 0;
        while (base + 4 * qc * (nt - d) <= e) { base += 4 * qc * (nt - d); ++d; }
        const int rem = e - base, len = nt - d;
        const int q = rem / (4 * len), t = (rem / 4) % len, w = rem & 3;
        const int I = d + t, J = t;
        int i, j;
        bool im = false;
        if (cplx) {
          i = 4 * I + (q >> 1);
          j = 4 * J + 2 * (q & 1) + (w >> 1);
          im = (w & 1) != 0;
        } else {
          i = 4 * I + q;
          j = 4 * J + w;
        }
        double v = 0.0;
        if (i < b && j < b)
          v = im ? 0.5 * (Aim[i * b + j] + Aim[j * b + i]) : 0.5 * (Are[i * b + j] + Are[j * b + i]);
        out[e] = v;
      }
      out += kron_sym_block(cplx, b);
    } else if (cplx) {
      double2* o2 = reinterpret_cast<double2*>(out);
      for (int e = tid; e < b * ldo; e += blockDim.x) o2[e] = make_double2(Are[e], Aim[e]);
      out += 2 * b * ldo;
    } else {
      for (int e = tid; e < b * ldo; e += blockDim.x) out[e] = Are[e];
      out += b * ldo;
    }
    __syncthreads();
  }
}

// Kronecker eigen-blocks too large for shared memory (3-D: b = 3k + 1 ~ 176):
// persistent CTAs, each block assembled TRANSPOSED straight into its own
// slot of the inverse store -- complex blocks as interleaved (re, im) with
// leading dimension ldc, real blocks with ldr -- and inverted in place by
// Gauss-Jordan with row pivoting: (A^T)^-1 = (A^-1)^T = G^T, exactly the K3e
// layout, so no scratch and no final transpose (cf. patch_factor_global_kernel).
template <int NC>
__global__ void __launch_bounds__(kFactorGlobalThreads) patch_factor_kron_global_kernel(
    FactorParams op, PatchParams pd, KronParams kp, int32_t* singular) {
  __shared__ double prow[2 * 512];
  __shared__ double colk[2 * 512];
  __shared__ int piv[512];
  __shared__ int s_prow, s_bad;
  const int tid = threadIdx.x;
  for (int p = blockIdx.x; p < pd.num_patches; p += gridDim.x) {
    const int n0 = pd.node_off[p], nk = pd.node_off[p + 1] - n0;
    const int* nodes = pd.node + n0;
    const int v = pd.vertex[p];
    const int mv = NC * nk, b = mv + 1;
    double* out = pd.inv + pd.inv_off[p];
    bool bad = false;
    for (int k = 0; k < kp.nblk && !bad; ++k) {
      const bool cplx = kp.is_complex[k] != 0;
      const double fre = op.dt * kp.lam_re[k], fim = op.dt * kp.lam_im[k];
      const int ld = cplx ? kron_ldc(b) : kron_ldr(b);
      const int w = cplx ? 2 : 1;  // doubles per element
      double* B = out;             // B[(c * ld + r) * w] = A[r][c]
      for (int e = tid; e < b * ld * w; e += blockDim.x) B[e] = 0.0;
      if (tid == 0) s_bad = 0;
      __syncthreads();
      for (int pr = tid; pr < nk * nk; pr += blockDim.x) {
        const int al = pr / nk, be = pr % nk;
        const int row = nodes[al];
        const int pos = find_col(op.p2_col, op.p2_rowptr[row], op.p2_rowptr[row + 1], nodes[be]);
        if (pos < 0) continue;
        const double2 mk = op.p2_mk[pos];
        for (int cc = 0; cc < NC; ++cc) {
          const long e = (long)(NC * be + cc) * ld + NC * al + cc;  // A[NC al + cc][NC be + cc]
          B[e * w] = mk.x + fre * mk.y;
          if (cplx) B[e * w + 1] = fim * mk.y;
        }
      }
      for (int al = tid; al < nk; al += blockDim.x) {
        const int row = nodes[al];
        const int pos = find_col(op.b_col, op.b_rowptr[row], op.b_rowptr[row + 1], v);
        for (int cc = 0; cc < NC; ++cc) {
          const double bv = pos >= 0 ? op.b_raw[(long)pos * NC + cc] : 0.0;
          const long e1 = (long)mv * ld + NC * al + cc;      // A[NC al + cc][mv]
          const long e2 = (long)(NC * al + cc) * ld + mv;    // A[mv][NC al + cc]
          B[e1 * w] = fre * bv;
          B[e2 * w] = fre * bv;
          if (cplx) {
            B[e1 * w + 1] = fim * bv;
            B[e2 * w + 1] = fim * bv;
          }
        }
      }
      __syncthreads();
      for (int kk = 0; kk < b; ++kk) {
        if (tid < 32) {
          double best = -1.0;
          int bi = kk;
          for (int i = kk + tid; i < b; i += 32) {
            const long e = ((long)i * ld + kk) * w;
            double a = fabs(B[e]);
            if (cplx) a += fabs(B[e + 1]);
            if (a > best) { best = a; bi = i; }
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const double ob = __shfl_down_sync(0xffffffffu, best, o);
            const int oi = __shfl_down_sync(0xffffffffu, bi, o);
            if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
          }
          if (tid == 0) {
            s_prow = bi;
            piv[kk] = bi;
            if (!(best > 0.0)) s_bad = 1;
          }
        }
        __syncthreads();
        if (s_bad) break;
        const int pr = s_prow;
        const long pe = ((long)pr * ld + kk) * w;
        double ir, ii = 0.0;
        if (cplx) {
          const double xr = B[pe], xi = B[pe + 1], den = xr * xr + xi * xi;
          ir = xr / den;
          ii = -xi / den;
        } else {
          ir = 1.0 / B[pe];
        }
        // scaled pivot row (swapped in) and the multiplier column
        for (int j = tid; j < b; j += blockDim.x) {
          const long e = ((long)pr * ld + j) * w;
          if (j == kk) {
            prow[w * j] = ir;
            if (cplx) prow[w * j + 1] = ii;
          } else if (cplx) {
            const double xr = B[e], xi = B[e + 1];
            prow[2 * j] = xr * ir - xi * ii;
            prow[2 * j + 1] = xr * ii + xi * ir;
          } else {
            prow[j] = B[e] * ir;
          }
        }
        for (int i = tid; i < b; i += blockDim.x) {
          const long e = ((long)(i == pr ? kk : i) * ld + kk) * w;
          colk[w * i] = B[e];
          if (cplx) colk[w * i + 1] = B[e + 1];
        }
        __syncthreads();
        if (pr != kk)
          for (int j = tid; j < b * w; j += blockDim.x)
            B[(long)pr * ld * w + j] = B[(long)kk * ld * w + j];
        __syncthreads();
        {
          const int wp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5;
          for (int i = wp; i < b; i += nw) {
            double* arow = B + (long)i * ld * w;
            if (i == kk) {
              for (int j = lane; j < b * w; j += 32) arow[j] = prow[j];
            } else if (cplx) {
              const double fr = colk[2 * i], fi = colk[2 * i + 1];
              for (int j = lane; j < b; j += 32) {
                const double br = (j == kk) ? 0.0 : arow[2 * j];
                const double bi = (j == kk) ? 0.0 : arow[2 * j + 1];
                const double pr2 = prow[2 * j], pi2 = prow[2 * j + 1];
                arow[2 * j] = br - (fr * pr2 - fi * pi2);
                arow[2 * j + 1] = bi - (fr * pi2 + fi * pr2);
              }
            } else {
              const double f = colk[i];
              for (int j = lane; j < b; j += 32) {
                const double base = (j == kk) ? 0.0 : arow[j];
                arow[j] = base - f * prow[j];
              }
            }
          }
        }
        __syncthreads();
      }
      if (s_bad) {
        if (tid == 0) atomicMin(singular, v);
        bad = true;
        __syncthreads();
        break;
      }
      for (int kk = b - 1; kk >= 0; --kk) {
        const int pk = piv[kk];
        if (pk != kk) {
          for (int i = tid; i < b; i += blockDim.x) {
            const long e1 = ((long)i * ld + kk) * w, e2 = ((long)i * ld + pk) * w;
            double t = B[e1]; B[e1] = B[e2]; B[e2] = t;
            if (cplx) { t = B[e1 + 1]; B[e1 + 1] = B[e2 + 1]; B[e2 + 1] = t; }
          }
        }
        __syncthreads();
      }
      out += (long)b * ld * w;
    }
  }
}

// ------------------------------------------------------------ modal split
//
// K7m input (ivk_patch_gather_blocks): the scalar M_s, K_s blocks and the
// pressure column of every patch, gathered from the eliminated operator on
// the patch's free nodes (the same lookups as K7); the generalised
// eigendecomposition itself runs at setup on the device (solvers.py
// ModalSplit).  K3m (patch_apply_modal_kernel): warp per patch, the record
// W_s | theta | c^ | H^-1 staged in shared memory (W_s with an odd leading
// dimension, so both W^T r and W v read it conflict-free), r_p gathered once;
// t = W^T r, per-mode s x s solves, one warp reduction for the pressure
// Schur complement, u = W v.  Bytes per patch: (k^2 + (1 + nc) k + s^2)
// doubles instead of s b^2 (kron) or (s b)^2 (full).

struct ModalParams {
  int S, NC;
  double dt;
  double a[IVK_MAX_STAGES * IVK_MAX_STAGES];
};

// record: W_s rows with leading dimension modal_ld(k) = 4 (mod 8) (the
// shared-memory layout, so one TMA bulk copy lands it ready to use: the
// tensor-core A fragments -- lane (g, q) reading row q, column g or the
// transpose -- then hit 16 distinct 8-byte banks per half-warp), theta, c^,
// H^-1; 32-byte padded
__host__ __device__ __forceinline__ int modal_ld(int k) { return ((k + 3) >> 3) * 8 + 4; }
__host__ __device__ __forceinline__ int modal_rec(int S, int NC, int k) {
  return (k * modal_ld(k) + k + NC * k + S * S + 3) & ~3;
}
template <int NC>
__global__ void __launch_bounds__(128) patch_gather_blocks_kernel(FactorParams op, PatchParams pd,
                                                                  int kmax, double* __restrict__ Ms,
                                                                  double* __restrict__ Ks,
                                                                  double* __restrict__ Cb) {
  const int p = blockIdx.x;
  const int n0 = pd.node_off[p], nk = pd.node_off[p + 1] - n0;
  const int* nodes = pd.node + n0;
  const int v = pd.vertex[p];
  double* ms = Ms + (long)p * kmax * kmax;
  double* ks = Ks + (long)p * kmax * kmax;
  double* cb = Cb + (long)p * kmax * NC;
  for (int e = threadIdx.x; e < kmax * kmax; e += blockDim.x) {
    const int al = e / kmax, be = e - al * kmax;
    double m = 0.0, k = 0.0;
    if (al < nk && be < nk) {
      const int row = nodes[al];
      const int pos = find_col(op.p2_col, op.p2_rowptr[row], op.p2_rowptr[row + 1], nodes[be]);
      if (pos >= 0) {
        const double2 mk = op.p2_mk[pos];
        m = mk.x;
        k = mk.y;
      }
    }
    ms[e] = m;
    ks[e] = k;
  }
  for (int al = threadIdx.x; al < kmax; al += blockDim.x) {
    int pos = -1;
    if (al < nk) {
      const int row = nodes[al];
      pos = find_col(op.b_col, op.b_rowptr[row], op.b_rowptr[row + 1], v);
    }
    for (int d = 0; d < NC; ++d) cb[al * NC + d] = pos >= 0 ? op.b_raw[(long)pos * NC + d] : 0.0;
  }
}

// E = (I + f A)^-1 for s <= 3 (explicit adjugate: I + f A is well
// conditioned for f = dt theta >= 0 and A with eigenvalues in the right
// half plane -- every tableau the library builds).
// 1 / x: hardware approximation + two Newton steps (relative error at
// rounding level; the mode matrices I + dt theta A are far from singular).
__device__ __forceinline__ double rcp_nr(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}

template <int S>
__device__ __forceinline__ void modal_small_inv(const double* A, double f, double* E) {
  double m[S * S];
#pragma unroll
  for (int i = 0; i < S; ++i)
#pragma unroll
    for (int j = 0; j < S; ++j) m[i * S + j] = (i == j ? 1.0 : 0.0) + f * A[i * S + j];
  if constexpr (S == 1) {
    E[0] = rcp_nr(m[0]);
  } else if constexpr (S == 2) {
    const double id = rcp_nr(m[0] * m[3] - m[1] * m[2]);
    E[0] = m[3] * id;
    E[1] = -m[1] * id;
    E[2] = -m[2] * id;
    E[3] = m[0] * id;
  } else {
    const double c00 = m[4] * m[8] - m[5] * m[7];
    const double c01 = m[5] * m[6] - m[3] * m[8];
    const double c02 = m[3] * m[7] - m[4] * m[6];
    const double id = rcp_nr(m[0] * c00 + m[1] * c01 + m[2] * c02);
    E[0] = c00 * id;
    E[1] = (m[2] * m[7] - m[1] * m[8]) * id;
    E[2] = (m[1] * m[5] - m[2] * m[4]) * id;
    E[3] = c01 * id;
    E[4] = (m[0] * m[8] - m[2] * m[6]) * id;
    E[5] = (m[2] * m[3] - m[0] * m[5]) * id;
    E[6] = c02 * id;
    E[7] = (m[1] * m[6] - m[0] * m[7]) * id;
    E[8] = (m[0] * m[4] - m[1] * m[3]) * id;
  }
}

// K7m: the modal record of every patch with k <= 32 free nodes, one warp per
// patch, straight from the gathered scalar blocks (ivk_patch_gather_blocks):
//   M_s = L L^T (Cholesky),  C = L^-1 K_s L^-T,
//   C = V Theta V^T by cyclic two-sided Jacobi rotations (stopping rule
//   |c_pq| <= eps sqrt(c_pp c_qq): eigenvalues of the positive definite C to
//   high relative accuracy, V orthogonal to rounding),  W = L^-T V,
//   c^ = W^T c,  E_i = (I + dt theta_i A)^-1,  H = dt^2 A (sum_i |c^_i|^2 E_i) A,
// and the record W | theta | c^ | H^-1 written where K3m streams it.
// Replaces the batched Cholesky / eigh / inverse calls into cuSOLVER (setup).
// Work arrays per warp in shared memory, row stride ks = kmax | 1 (column
// walks -- lane j at row j -- hit distinct banks).  Every lane computes the
// rotation angle from the same three broadcast entries, so all agree.
// A patch is flagged singular when M_s is not positive definite, when H or
// H^-1 is not finite, or when cond_1(H) >= 1e14.
constexpr int kModalSetupWarps = 4;

template <int S, int NC>
__global__ void __launch_bounds__(kModalSetupWarps * 32) modal_factor_kernel(
    PatchParams pd, ModalParams mp, int kmax, const double* __restrict__ Ms,
    const double* __restrict__ Ks, const double* __restrict__ Cb, int32_t* singular) {
  extern __shared__ __align__(16) double msm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int p = blockIdx.x * kModalSetupWarps + warp;
  if (p >= pd.num_patches) return;
  const int k = pd.node_off[p + 1] - pd.node_off[p];
  const int ks = kmax | 1;
  double* L = msm + (long)warp * 3 * kmax * ks;
  double* C = L + kmax * ks;
  double* V = C + kmax * ks;
  const double* Mg = Ms + (long)p * kmax * kmax;
  const double* Kg = Ks + (long)p * kmax * kmax;
  for (int e = lane; e < k * k; e += 32) {
    const int i = e / k, j = e - i * k;
    L[i * ks + j] = Mg[i * kmax + j];
    C[i * ks + j] = Kg[i * kmax + j];
    V[i * ks + j] = i == j ? 1.0 : 0.0;
  }
  __syncwarp();
  bool bad = k < 1;
  // Cholesky, right-looking; lane i owns row i
  for (int j = 0; j < k && !bad; ++j) {
    const double djj = L[j * ks + j];
    if (!(djj > 0.0) || !(djj < 1.79e308)) { bad = true; break; }   // uniform: broadcast read
    const double ljj = sqrt(djj);
    __syncwarp();
    if (lane == j) L[j * ks + j] = ljj;
    if (lane > j && lane < k) L[lane * ks + j] /= ljj;
    __syncwarp();
    if (lane > j && lane < k) {
      const double lij = L[lane * ks + j];
      for (int t = j + 1; t <= lane; ++t) L[lane * ks + t] -= lij * L[t * ks + j];
    }
    __syncwarp();
  }
  if (bad) {
    if (lane == 0) atomicMin(singular, pd.vertex[p]);
    return;
  }
  // X = L^-1 K (lane c solves column c), then C = L^-1 X^T (lane r solves row r)
  if (lane < k) {
    for (int i = 0; i < k; ++i) {
      double x = C[i * ks + lane];
      for (int t = 0; t < i; ++t) x -= L[i * ks + t] * C[t * ks + lane];
      C[i * ks + lane] = x / L[i * ks + i];
    }
  }
  __syncwarp();
  if (lane < k) {
    for (int i = 0; i < k; ++i) {
      double x = C[lane * ks + i];
      for (int t = 0; t < i; ++t) x -= L[i * ks + t] * C[lane * ks + t];
      C[lane * ks + i] = x / L[i * ks + i];
    }
  }
  __syncwarp();
  // symmetrise (pairs i < j, each handled once)
  for (int e = lane; e < k * k; e += 32) {
    const int i = e / k, j = e - i * k;
    if (i < j) {
      const double m = 0.5 * (C[i * ks + j] + C[j * ks + i]);
      C[i * ks + j] = m;
      C[j * ks + i] = m;
    }
  }
  __syncwarp();
  // cyclic Jacobi
  for (int sweep = 0; sweep < 40; ++sweep) {
    bool rotated = false;
    for (int pp = 0; pp < k - 1; ++pp)
      for (int qq = pp + 1; qq < k; ++qq) {
        const double apq = C[pp * ks + qq];
        const double app = C[pp * ks + pp], aqq = C[qq * ks + qq];
        if (!(fabs(apq) > 2.220446049250313e-16 * sqrt(fabs(app * aqq)))) continue;
        rotated = true;
        const double tau = (aqq - app) / (2.0 * apq);
        const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
        const double c = 1.0 / sqrt(1.0 + t * t), sn = t * c;
        __syncwarp();   // the broadcast reads above precede the updates
        if (lane < k) {   // columns pp, qq (lane = row), and V's
          const double cjp = C[lane * ks + pp], cjq = C[lane * ks + qq];
          C[lane * ks + pp] = c * cjp - sn * cjq;
          C[lane * ks + qq] = sn * cjp + c * cjq;
          const double vjp = V[lane * ks + pp], vjq = V[lane * ks + qq];
          V[lane * ks + pp] = c * vjp - sn * vjq;
          V[lane * ks + qq] = sn * vjp + c * vjq;
        }
        __syncwarp();
        if (lane < k) {   // rows pp, qq (lane = column)
          const double cpj = C[pp * ks + lane], cqj = C[qq * ks + lane];
          C[pp * ks + lane] = c * cpj - sn * cqj;
          C[qq * ks + lane] = sn * cpj + c * cqj;
        }
        __syncwarp();
        if (lane == 0) {
          C[pp * ks + qq] = 0.0;
          C[qq * ks + pp] = 0.0;
        }
        __syncwarp();
      }
    if (!rotated) break;
  }
  // W = L^-T V (lane c back-substitutes column c, in place)
  if (lane < k) {
    for (int i = k - 1; i >= 0; --i) {
      double x = V[i * ks + lane];
      for (int t = i + 1; t < k; ++t) x -= L[t * ks + i] * V[t * ks + lane];
      V[i * ks + lane] = x / L[i * ks + i];
    }
  }
  __syncwarp();
  // record
  const int ld = modal_ld(k);
  double* rec = pd.inv + pd.inv_off[p];
  double* th = rec + k * ld;
  double* ch = th + k;
  double* hi = ch + NC * k;
  const int reclen = modal_rec(S, NC, k);
  for (int e = lane; e < k * ld; e += 32) {
    const int i = e / ld, j = e - i * ld;
    rec[e] = j < k ? V[i * ks + j] : 0.0;
  }
  double ws[S * S];
#pragma unroll
  for (int a = 0; a < S * S; ++a) ws[a] = 0.0;
  if (lane < k) {
    const double theta = C[lane * ks + lane];
    th[lane] = theta;
    double c2 = 0.0;
    const double* cg = Cb + (long)p * kmax * NC;
#pragma unroll
    for (int d = 0; d < NC; ++d) {
      double acc = 0.0;
      for (int a = 0; a < k; ++a) acc = fma(V[a * ks + lane], cg[a * NC + d], acc);
      ch[lane * NC + d] = acc;
      c2 = fma(acc, acc, c2);
    }
    double E[S * S];
    modal_small_inv<S>(mp.a, mp.dt * theta, E);
#pragma unroll
    for (int a = 0; a < S * S; ++a) ws[a] = c2 * E[a];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int a = 0; a < S * S; ++a) ws[a] += __shfl_xor_sync(0xffffffffu, ws[a], o);
  // H = dt^2 A ws A and its inverse (every lane the same bits)
  double H[S * S], T1[S * S], Hi[S * S];
#pragma unroll
  for (int a = 0; a < S; ++a)
#pragma unroll
    for (int b = 0; b < S; ++b) {
      double acc = 0.0;
#pragma unroll
      for (int c = 0; c < S; ++c) acc = fma(mp.a[a * S + c], ws[c * S + b], acc);
      T1[a * S + b] = acc;
    }
#pragma unroll
  for (int a = 0; a < S; ++a)
#pragma unroll
    for (int b = 0; b < S; ++b) {
      double acc = 0.0;
#pragma unroll
      for (int c = 0; c < S; ++c) acc = fma(T1[a * S + c], mp.a[c * S + b], acc);
      H[a * S + b] = mp.dt * mp.dt * acc;
    }
  if constexpr (S == 1) {
    Hi[0] = 1.0 / H[0];
  } else if constexpr (S == 2) {
    const double det = H[0] * H[3] - H[1] * H[2];
    Hi[0] = H[3] / det;
    Hi[1] = -H[1] / det;
    Hi[2] = -H[2] / det;
    Hi[3] = H[0] / det;
  } else {
    const double c00 = H[4] * H[8] - H[5] * H[7];
    const double c01 = H[5] * H[6] - H[3] * H[8];
    const double c02 = H[3] * H[7] - H[4] * H[6];
    const double det = H[0] * c00 + H[1] * c01 + H[2] * c02;
    Hi[0] = c00 / det;
    Hi[1] = (H[2] * H[7] - H[1] * H[8]) / det;
    Hi[2] = (H[1] * H[5] - H[2] * H[4]) / det;
    Hi[3] = c01 / det;
    Hi[4] = (H[0] * H[8] - H[2] * H[6]) / det;
    Hi[5] = (H[2] * H[3] - H[0] * H[5]) / det;
    Hi[6] = c02 / det;
    Hi[7] = (H[1] * H[6] - H[0] * H[7]) / det;
    Hi[8] = (H[0] * H[4] - H[1] * H[3]) / det;
  }
  double nh = 0.0, ni = 0.0;   // 1-norms (max column sum)
  bool finite = true;
#pragma unroll
  for (int b = 0; b < S; ++b) {
    double sh = 0.0, si = 0.0;
#pragma unroll
    for (int a = 0; a < S; ++a) {
      sh += fabs(H[a * S + b]);
      si += fabs(Hi[a * S + b]);
    }
    nh = fmax(nh, sh);
    ni = fmax(ni, si);
    finite = finite && sh < 1.79e308 && si < 1.79e308;   // false for inf / NaN
  }
  if (lane < S * S) {
    double v = Hi[0];
#pragma unroll
    for (int a = 1; a < S * S; ++a)
      if (lane == a) v = Hi[a];
    hi[lane] = v;
  }
  for (int e = k * ld + k + NC * k + S * S + lane; e < reclen; e += 32) rec[e] = 0.0;
  if (lane == 0 && (!finite || !(nh * ni < 1e14))) atomicMin(singular, pd.vertex[p]);
}

template <int N>
__device__ __forceinline__ void lds_vec(const double* p, double (&v)[N]) {
  if constexpr (N % 2 == 0) {
#pragma unroll
    for (int q = 0; q < N; q += 2) {
      const double2 x = *reinterpret_cast<const double2*>(p + q);
      v[q] = x.x;
      v[q + 1] = x.y;
    }
  } else {
#pragma unroll
    for (int q = 0; q < N; ++q) v[q] = p[q];
  }
}

// K3m on the FP64 tensor cores (DMMA.8x8x4), for patches with k <= KP nodes:
// T = W^T R and U = W V as 8x8x4 tiles (M = modes / nodes, N = the NA
// (component, stage) columns padded to 8, K = nodes / modes), zero padding
// by predication on the compact record (no extra HBM bytes); everything else
// as patch_apply_modal_kernel.
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// R and T row layout.  Up to 8 (component, stage) columns (IVK_K3M_SWZ, the
// default): rows of 8 doubles with the column XOR-swizzled by
// sw(row) = (row bit 1) << 2 | (row bit 2) << 1 | (row bit 3), which makes every
// access pattern of the kernel conflict-free: the lane-per-mode phase (lane i
// reads / writes row i, one column: the eight even rows of a half-warp get
// eight distinct sw, odd rows sit in the other 64 bytes), the tensor-core B
// loads (lanes (n, k) = (lane / 4, lane % 4) read row k0 + k, column n: rows
// two apart differ in sw bit 2, so their four columns fall in different
// halves of the row) and the D fragment stores (a 16-byte pair per lane).
// Wider rows keep the earlier odd stride NA | 1 (conflict-free per-mode
// phase, two-way conflicts on the B loads); there the B loads read the padded
// columns NA..NW-1 past the row end (finite values of the next row or the NW
// slack, multiplied into output columns that are dropped).
#ifndef IVK_K3M_SWZ
#define IVK_K3M_SWZ 1
#endif
__host__ __device__ __forceinline__ constexpr bool modal_tc_swz(int NA) {
  return IVK_K3M_SWZ && NA <= 8;
}
__host__ __device__ __forceinline__ constexpr int modal_tc_ts(int NA) {
  return modal_tc_swz(NA) ? 8 : (NA | 1);
}
__host__ __device__ __forceinline__ int modal_tc_tbuf(int S, int NC, int KP) {
  return KP * modal_tc_ts(NC * S) + 8 * ((NC * S + 7) / 8);
}
__device__ __forceinline__ int modal_sw(int row) {
  return ((row << 1) & 4) | ((row >> 1) & 2) | ((row >> 3) & 1);
}
// element (row, col) of an R / T buffer
template <int NA>
__device__ __forceinline__ int modal_tpos(int row, int col) {
  if constexpr (modal_tc_swz(NA)) return row * 8 + (col ^ modal_sw(row));
  else return row * (NA | 1) + col;
}
// per warp: two record buffers (TMA), two R buffers (cp.async gathers one
// patch ahead; the one in use turns into the T / w / v buffer after the T
// GEMM), two sets of 4 pressure slots
__host__ __device__ __forceinline__ int modal_tc_seg(int S, int NC, int kmax, int KP) {
  return (2 * modal_rec(S, NC, kmax) + 2 * modal_tc_tbuf(S, NC, KP) + 2 * 4 + 3) & ~3;
}

// Ampere-style asynchronous 8-byte global -> shared copy (LDGSTS): the r
// gathers land straight in the R rows, no register staging.
__device__ __forceinline__ void cp_async8(uint32_t dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait1() {
  asm volatile("cp.async.wait_group 1;" ::: "memory");
}

// L2 evict-last policy for the patch-local results (the scatter re-reads
// them right after), created once per thread.
__device__ __forceinline__ uint64_t keep_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void st_keep_pol(double* p, double v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v),
               "l"(pol)
               : "memory");
}
__device__ __forceinline__ void st_keep_pol2(double* p, double v0, double v1, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p),
               "d"(v0), "d"(v1), "l"(pol)
               : "memory");
}

// Land gathered value v of fragment-layout entry j (include/ivk.h layout 1:
// node*NA + q, then the S pressures) in the R rows (stride TS) / pressures.
// shared address of fragment-layout entry j (include/ivk.h layout 1:
// node*NA + q, then the S pressures) in the R rows (stride TS) / pressures
template <int NA>
__device__ __forceinline__ uint32_t modal_slot(uint32_t R, uint32_t Rp, int j, int nak) {
  const int al = j / NA;   // NA is a compile-time constant: a multiply-shift
  return j < nak ? R + 8u * modal_tpos<NA>(al, j - al * NA) : Rp + 8u * (j - nak);
}

// KTX = ceil(kmax / 4) K-steps of 4 nodes run for every patch, branch-free:
// rows of R / T past a patch's k are exact zeros, so smaller patches simply
// multiply zeros (no divergent DMMA regions, loads pipelined across steps).
// A/B knob: -DIVK_K3M_CH=2 splits each GEMM row tile's K steps into two
// independent accumulator chains (measured below).
#ifndef IVK_K3M_CH
#define IVK_K3M_CH 1
#endif
// A/B knob: -DIVK_K3M_MAXT=160 -DIVK_K3M_MINB=4 caps the kernel at 96 registers
// (20 warps/SM): measured slower than the uncapped 98 (16 warps/SM), DESIGN §9.
// (An explicit minBlocks of 1 is NOT neutral: ptxas then spends 138 registers.)
#ifdef IVK_K3M_MAXT
#define IVK_K3M_BOUNDS __launch_bounds__(IVK_K3M_MAXT, IVK_K3M_MINB)
#else
#define IVK_K3M_MAXT (kApplyWarps * 32)
#define IVK_K3M_BOUNDS __launch_bounds__(kApplyWarps * 32)
#endif
template <int S, int NC, int KP, int KTX>
__global__ void IVK_K3M_BOUNDS patch_apply_modal_tc_kernel(
    PatchParams pd, ModalParams mp, const double* __restrict__ r, double* __restrict__ local,
    int kmax) {
  extern __shared__ __align__(16) double modal_sm[];
  __shared__ __align__(8) uint64_t bars[kApplyWarps][2];
  constexpr int NA = NC * S;
  constexpr int NT = (NA + 7) / 8;   // 8-column N tiles
  constexpr int NW = 8 * NT;         // padded row width of R / T
  constexpr int MT = KP / 8;
  constexpr int TS = modal_tc_ts(NA);           // row stride of R and T
  constexpr bool SWZ = modal_tc_swz(NA);
  static_assert(KP <= 32, "one mode per lane");
  static_assert(4 * KTX <= KP, "K steps exceed the padded node count");
  constexpr int TBUF = KP * TS + NW;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int gq = lane >> 2, gk = lane & 3;
  const int recmax = modal_rec(S, NC, kmax);
  double* buf0 = modal_sm + (long)warp * modal_tc_seg(S, NC, kmax, KP);
  double* buf1 = buf0 + recmax;
  // R[2]: [alpha][TS] with zero rows past k, double-buffered: patch i+1's r
  // values are gathered (cp.async) while patch i computes
  double* rsT0 = buf1 + recmax;
  double* rsP = rsT0 + 2 * TBUF;     // the s pressures, two buffers of 4
  const uint32_t rsT0_u = smem_u32(rsT0), rsP_u = smem_u32(rsP);
  // zero the whole segment once: the tensor-core A loads below are not
  // predicated, so they read (finite) record tails, the other buffer and
  // stale rows past k -- every such value meets an exact zero in B
  for (int e = lane; e < modal_tc_seg(S, NC, kmax, KP); e += 32) buf0[e] = 0.0;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // before TMA overwrites
  if (lane == 0) {
    mbar_init(&bars[warp][0], 1);
    mbar_init(&bars[warp][1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const uint64_t pol = keep_policy();
  const double dt = mp.dt;
  // each CTA walks a contiguous run of patches (neighbouring vertex stars:
  // their r gathers and local[] writes share cache lines), warps interleaved
  const int stride = nw;
  const int chunk = (pd.num_patches + gridDim.x - 1) / gridDim.x;
  const int pbeg = blockIdx.x * chunk;
  const int pend = min(pd.num_patches, pbeg + chunk);
  int p = pbeg + warp;
  // byte offset, inside an R buffer, of fragment-layout entry lane + 32 u (a
  // velocity entry: node*NA + q); the same for every patch
  uint32_t lslot[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int j = lane + 32 * u, al = j / NA;
    lslot[u] = 8u * modal_tpos<NA>(al, j - al * NA);
  }
  int rz0 = 0, rz1 = 0;   // leading rows of R[0] / R[1] a gather may have left non-zero
  if (lane == 0 && p < pend) {
    const int k0 = pd.node_off[p + 1] - pd.node_off[p];
    bulk_load(buf0, pd.inv + pd.inv_off[p], modal_rec(S, NC, k0) * 8, &bars[warp][0]);
  }
  if (p < pend) {
    const int off0 = pd.idx_off[p];
    const int k0 = pd.node_off[p + 1] - pd.node_off[p];
    for (int j = lane; j < S * (NC * k0 + 1); j += 32)
      cp_async8(modal_slot<NA>(rsT0_u, rsP_u, j, NA * k0), r + __ldg(pd.idx + off0 + j));
    rz0 = k0;
  }
  cp_async_commit();
  // gather indices of the next patch (one patch ahead of its r gathers)
  int pf_idx[4];
  int pn_off = 0, pn_k = 0, pn_m = 0;
  {
    const int pn = p + stride;
    if (pn < pend) {
      pn_off = pd.idx_off[pn];
      pn_k = pd.node_off[pn + 1] - pd.node_off[pn];
      pn_m = S * (NC * pn_k + 1);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = lane + 32 * u;
      pf_idx[u] = j < pn_m ? __ldg(pd.idx + pn_off + j) : -1;
    }
  }
  uint32_t phase = 0;
  for (int it = 0; p < pend; ++it, p += stride) {
    const int slot = it & 1;
    const int pn = p + stride;
    if (lane == 0 && pn < pend) {
      const int kn = pd.node_off[pn + 1] - pd.node_off[pn];
      bulk_load(slot ? buf0 : buf1, pd.inv + pd.inv_off[pn], modal_rec(S, NC, kn) * 8,
                &bars[warp][slot ^ 1]);
    }
    // gather the next patch's r into the other R buffer (cp.async); clear
    // rows an earlier, larger patch left there first (rare: sizes ascend)
    {
      double* RN = rsT0 + (slot ^ 1) * TBUF;
      const uint32_t RN_u = rsT0_u + 8u * ((slot ^ 1) * TBUF);
      const uint32_t RPN_u = rsP_u + 8u * (4 * (slot ^ 1));
      int& rzn = slot ? rz0 : rz1;
      if (pn_k < rzn)
        for (int e = pn_k * TS + lane; e < rzn * TS; e += 32) RN[e] = 0.0;
      const int nak = NA * pn_k;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (pf_idx[u] >= 0) {
          const int j = lane + 32 * u;
          cp_async8(j < nak ? RN_u + lslot[u] : RPN_u + 8u * (j - nak), r + pf_idx[u]);
        }
      for (int j = 128 + lane; j < pn_m; j += 32)
        cp_async8(modal_slot<NA>(RN_u, RPN_u, j, nak), r + __ldg(pd.idx + pn_off + j));
      cp_async_commit();
      rzn = pn_k;
    }
    // indices of the patch after next
    {
      const int pnn = pn + stride;
      pn_off = pn_k = pn_m = 0;
      if (pnn < pend) {
        pn_off = pd.idx_off[pnn];
        pn_k = pd.node_off[pnn + 1] - pd.node_off[pnn];
        pn_m = S * (NC * pn_k + 1);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = lane + 32 * u;
        pf_idx[u] = j < pn_m ? __ldg(pd.idx + pn_off + j) : -1;
      }
    }
    const int off = pd.idx_off[p];
    const int k = pd.node_off[p + 1] - pd.node_off[p];
    const int ld = modal_ld(k);
    double* t = rsT0 + slot * TBUF;    // R, then (after the T GEMM) T / w / v
    const double* R = t;
    const double* Rp = rsP + 4 * slot;
    mbar_wait(&bars[warp][slot], (phase >> slot) & 1u);
    phase ^= 1u << slot;
    cp_async_wait1();   // this patch's gathers (all but the newest group) landed
    __syncwarp();
    const double* W = slot ? buf1 : buf0;
    const double* th = W + k * ld;
    const double* ch = th + k;
    const double* hi = ch + NC * k;
    // T = W^T R
    {
      double d[MT][NT][2];
#pragma unroll
      for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int n = 0; n < NT; ++n) d[m][n][0] = d[m][n][1] = 0.0;
#if IVK_K3M_CH > 1
      double d2[MT][NT][2];   // second accumulator chain (odd K steps)
#pragma unroll
      for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int n = 0; n < NT; ++n) d2[m][n][0] = d2[m][n][1] = 0.0;
#endif
#pragma unroll
      for (int kt = 0; kt < KTX; ++kt) {
        const int al = 4 * kt + gk;
        double b[NT];
#pragma unroll
        for (int n = 0; n < NT; ++n) b[n] = R[modal_tpos<NA>(al, 8 * n + gq)];
#pragma unroll
        for (int m = 0; m < MT; ++m) {
          const double a = W[al * ld + 8 * m + gq];   // rows al >= k meet R's zero rows
#pragma unroll
          for (int n = 0; n < NT; ++n) {
#if IVK_K3M_CH > 1
            if (kt & 1) dmma884(d2[m][n][0], d2[m][n][1], a, b[n]);
            else
#endif
            dmma884(d[m][n][0], d[m][n][1], a, b[n]);
          }
        }
      }
#if IVK_K3M_CH > 1
#pragma unroll
      for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          d[m][n][0] += d2[m][n][0];
          d[m][n][1] += d2[m][n][1];
        }
#endif
      __syncwarp();   // every lane's R reads are done: T overwrites R in place
#pragma unroll
      for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          const int q0 = 8 * n + 2 * gk;
          // rows past k (their A columns were record tails: finite garbage)
          // are stored as the exact zeros the U GEMM's unpredicated A
          // columns must meet
          const bool live = 8 * m + gq < k;
          const double t0 = live ? d[m][n][0] : 0.0, t1 = live ? d[m][n][1] : 0.0;
          if constexpr (SWZ && NA % 2 == 0) {
            // the pair (q0, q0 + 1) stays one aligned 16-byte slot, swapped
            // where sw(row) is odd
            const int row = 8 * m + gq, sw = modal_sw(row);
            if (q0 < NA)
              *reinterpret_cast<double2*>(t + row * 8 + ((q0 ^ sw) & ~1)) =
                  (sw & 1) ? make_double2(t1, t0) : make_double2(t0, t1);
          } else {
            if (q0 < NA) t[modal_tpos<NA>(8 * m + gq, q0)] = t0;
            if (q0 + 1 < NA) t[modal_tpos<NA>(8 * m + gq, q0 + 1)] = t1;
          }
        }
    }
    __syncwarp();
    // lane per mode i (k <= KP <= 32: one mode per lane): w_i = E_i t_i,
    // g += c^ w; E_i, w_i and c^_i stay in registers across the reduction
    const int im = lane;
    const bool act = im < k;
    double E[S * S], wv[NA], cc[NC];
    double g[S];
#pragma unroll
    for (int a = 0; a < S; ++a) g[a] = 0.0;
    if (act) {
      double acc[NA];
#pragma unroll
      for (int q = 0; q < NA; ++q) acc[q] = t[modal_tpos<NA>(im, q)];
      modal_small_inv<S>(mp.a, dt * th[im], E);
#pragma unroll
      for (int dd = 0; dd < NC; ++dd) {
        cc[dd] = ch[im * NC + dd];
#pragma unroll
        for (int a = 0; a < S; ++a) {
          double w = 0.0;
#pragma unroll
          for (int b = 0; b < S; ++b) w = fma(E[a * S + b], acc[dd * S + b], w);
          wv[dd * S + a] = w;
          g[a] = fma(cc[dd], w, g[a]);
        }
      }
    }
    // butterfly: x + y is commutative, so every lane ends with the same bits
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int a = 0; a < S; ++a) g[a] += __shfl_xor_sync(0xffffffffu, g[a], o);
    double rhs[S], pv[S], Ap[S];
#pragma unroll
    for (int a = 0; a < S; ++a) {
      double s_ = 0.0;
#pragma unroll
      for (int b = 0; b < S; ++b) s_ = fma(mp.a[a * S + b], g[b], s_);
      rhs[a] = dt * s_ - Rp[a];
    }
#pragma unroll
    for (int a = 0; a < S; ++a) {
      double s_ = 0.0;
#pragma unroll
      for (int b = 0; b < S; ++b) s_ = fma(hi[a * S + b], rhs[b], s_);
      pv[a] = s_;
    }
#pragma unroll
    for (int a = 0; a < S; ++a) {
      double s_ = 0.0;
#pragma unroll
      for (int b = 0; b < S; ++b) s_ = fma(mp.a[a * S + b], pv[b], s_);
      Ap[a] = s_;
    }
    if (act) {
      double e[S];
#pragma unroll
      for (int a = 0; a < S; ++a) {
        double s_ = 0.0;
#pragma unroll
        for (int b = 0; b < S; ++b) s_ = fma(E[a * S + b], Ap[b], s_);
        e[a] = s_;
      }
#pragma unroll
      for (int dd = 0; dd < NC; ++dd)
#pragma unroll
        for (int a = 0; a < S; ++a)
          t[modal_tpos<NA>(im, dd * S + a)] = fma(-dt * cc[dd], e[a], wv[dd * S + a]);
    }   // (rows past k already hold the zeros the T store wrote)
    __syncwarp();
    // U = W V; each lane stores its D fragment entries (node 8m+gq, columns
    // 8n+2gk, +1) straight to their fragment-layout slots
    {
      double d[MT][NT][2];
#pragma unroll
      for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int n = 0; n < NT; ++n) d[m][n][0] = d[m][n][1] = 0.0;
#if IVK_K3M_CH > 1
      double d2[MT][NT][2];
#pragma unroll
      for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int n = 0; n < NT; ++n) d2[m][n][0] = d2[m][n][1] = 0.0;
#endif
#pragma unroll
      for (int kt = 0; kt < KTX; ++kt) {
        const int i = 4 * kt + gk;
        double b[NT];
#pragma unroll
        for (int n = 0; n < NT; ++n) b[n] = t[modal_tpos<NA>(i, 8 * n + gq)];
#pragma unroll
        for (int m = 0; m < MT; ++m) {
          const double a = W[(8 * m + gq) * ld + i];   // columns i >= k meet t's zero rows
#pragma unroll
          for (int n = 0; n < NT; ++n) {
#if IVK_K3M_CH > 1
            if (kt & 1) dmma884(d2[m][n][0], d2[m][n][1], a, b[n]);
            else
#endif
            dmma884(d[m][n][0], d[m][n][1], a, b[n]);
          }
        }
      }
#if IVK_K3M_CH > 1
#pragma unroll
      for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          d[m][n][0] += d2[m][n][0];
          d[m][n][1] += d2[m][n][1];
        }
#endif
      double* lp = local + off;
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        const int al = 8 * m + gq;
        if (al < k) {
#pragma unroll
          for (int n = 0; n < NT; ++n) {
            const int q = 8 * n + 2 * gk;
            if constexpr (NA % 2 == 0) {
              // off, al*NA and q are even: a 16-byte aligned pair
              if (q < NA) st_keep_pol2(lp + al * NA + q, d[m][n][0], d[m][n][1], pol);
            } else {
              if (q < NA) st_keep_pol(lp + al * NA + q, d[m][n][0], pol);
              if (q + 1 < NA) st_keep_pol(lp + al * NA + q + 1, d[m][n][1], pol);
            }
          }
        }
      }
    }
    // the buffer now holds v in rows < k (zeros past k)
    if (slot) rz1 = k; else rz0 = k;
    if (lane < S) {
      double pl = pv[0];
#pragma unroll
      for (int a = 1; a < S; ++a)
        if (lane == a) pl = pv[a];
      st_keep_pol(local + off + NA * k + lane, pl, pol);
    }
    __syncwarp();
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// K3m for large patches (3-D: k = 65 nodes, W_s 34 KB): one CTA of
// kModalCtaWarps warps per patch (persistent over patches, 2 CTAs per SM), the
// record double-buffered by TMA bulk copies, the two GEMMs on the FP64 tensor cores
// with the 8-row tiles split over the warps, the per-mode work thread per
// mode, the pressure Schur solve by thread 0 after a fixed-order CTA reduction.
constexpr int kModalCtaWarps = 16;

__host__ __device__ __forceinline__ int modal_cta_smem(int S, int NC, int kmax, int KP) {
  const int NW = 8 * ((NC * S + 7) / 8);
  return (2 * modal_rec(S, NC, kmax) + 2 * KP * NW + 8 + KP * NW + KP * S * S +
          kModalCtaWarps * 4 + 8 + 3) & ~3;
}

template <int S, int NC, int KP>
__global__ void __launch_bounds__(kModalCtaWarps * 32) patch_apply_modal_cta_kernel(
    PatchParams pd, ModalParams mp, const double* __restrict__ r, double* __restrict__ local,
    int kmax) {
  extern __shared__ __align__(16) double modal_sm[];
  __shared__ __align__(8) uint64_t bars[2];
  constexpr int NA = NC * S;
  constexpr int NT = (NA + 7) / 8;
  constexpr int NW = 8 * NT;
  constexpr int MT = KP / 8, KT = KP / 4;
  constexpr int NTH = kModalCtaWarps * 32;
  constexpr int PF = 4;             // prefetched r values per thread (m <= 512)
#ifndef IVK_MODAL_CTA_CH
#define IVK_MODAL_CTA_CH 3
#endif
  constexpr int CH = IVK_MODAL_CTA_CH;   // accumulator chains per GEMM row tile
  static_assert(KT % CH == 0, "the K steps must split evenly into the chains");
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gq = lane >> 2, gk = lane & 3;
  const int recmax = modal_rec(S, NC, kmax);
  double* buf0 = modal_sm;
  double* buf1 = buf0 + recmax;
  double* R0 = buf1 + recmax;
  double* R1 = R0 + KP * NW;
  double* Rp = R1 + KP * NW;        // 2 x 4 pressures
  double* t = Rp + 8;
  double* Es = t + KP * NW;
  double* gred = Es + KP * S * S;   // kModalCtaWarps x 4 partial sums
  double* pAp = gred + kModalCtaWarps * 4;  // p (4) and A p (4)
  // zero the whole segment once: the tensor-core A loads below are not
  // predicated, so they read (finite) record tails and the buffers behind
  // them -- every such value meets an exact zero row of R / t
  for (int e = tid; e < modal_cta_smem(S, NC, kmax, KP); e += NTH) modal_sm[e] = 0.0;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // before TMA overwrites
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const double dt = mp.dt;
  int p = blockIdx.x;
  if (tid == 0 && p < pd.num_patches) {
    const int k0 = pd.node_off[p + 1] - pd.node_off[p];
    bulk_load(buf0, pd.inv + pd.inv_off[p], modal_rec(S, NC, k0) * 8, &bars[0]);
  }
  if (p < pd.num_patches) {
    const int off0 = pd.idx_off[p];
    const int k0 = pd.node_off[p + 1] - pd.node_off[p];
    const int blk0 = NC * k0 + 1;
    for (int j = tid; j < S * blk0; j += NTH) {
      const int a = (j >= blk0) + (S > 2 && j >= 2 * blk0);
      const int e = j - a * blk0;
      const double v = __ldg(r + pd.idx[off0 + j]);
      if (e < NC * k0) {
        const int al = e / NC, d = e - al * NC;
        R0[al * NW + d * S + a] = v;
      } else {
        Rp[a] = v;
      }
    }
  }
  __syncthreads();
  uint32_t phase = 0;
  for (int it = 0; p < pd.num_patches; ++it, p += gridDim.x) {
    const int slot = it & 1;
    const int pn = p + gridDim.x;
    if (tid == 0 && pn < pd.num_patches) {
      const int kn = pd.node_off[pn + 1] - pd.node_off[pn];
      bulk_load(slot ? buf0 : buf1, pd.inv + pd.inv_off[pn], modal_rec(S, NC, kn) * 8,
                &bars[slot ^ 1]);
    }
    const int off = pd.idx_off[p];
    const int k = pd.node_off[p + 1] - pd.node_off[p];
    const int blk = NC * k + 1;
    const int ld = modal_ld(k);
    const double* R = slot ? R1 : R0;
    const double* Rpc = Rp + 4 * slot;
    int pf_idx[PF];
    int pn_off = 0, pn_k = 0, pn_blk = 0;
    if (pn < pd.num_patches) {
      pn_off = pd.idx_off[pn];
      pn_k = pd.node_off[pn + 1] - pd.node_off[pn];
      pn_blk = NC * pn_k + 1;
    }
#pragma unroll
    for (int u = 0; u < PF; ++u) {
      const int j = tid + NTH * u;
      pf_idx[u] = (pn < pd.num_patches && j < S * pn_blk) ? __ldg(pd.idx + pn_off + j) : -1;
    }
    // t rows this patch's T store will not reach (a larger patch may have left
    // values there) must be the zeros the U GEMM's unpredicated A columns meet;
    // every thread is past the previous patch's reads of t (barrier at the
    // loop end), and two barriers separate this from the U GEMM
    for (int e = ((k + 7) & ~7) * NW + tid; e < KP * NW; e += NTH) t[e] = 0.0;
    mbar_wait(&bars[slot], (phase >> slot) & 1u);
    phase ^= 1u << slot;
    const double* W = slot ? buf1 : buf0;
    const double* th = W + k * ld;
    const double* ch = th + k;
    const double* hi = ch + NC * k;
    // T = W^T R: warp w takes mode tiles w, w + 4, ...
    for (int m = warp; m < MT; m += kModalCtaWarps) {
      if (8 * m >= k) break;
      // CH independent accumulator chains over the K steps (one chain of
      // KT = 18 dependent DMMAs is latency-bound: 584 -> 513 us at cfg4),
      // summed in a fixed order
      double dc[CH][NT][2];
#pragma unroll
      for (int c = 0; c < CH; ++c)
#pragma unroll
        for (int n = 0; n < NT; ++n) dc[c][n][0] = dc[c][n][1] = 0.0;
      const int i = 8 * m + gq;
      for (int kt0 = 0; kt0 < KT && 4 * kt0 < k; kt0 += CH) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
          const int al = 4 * (kt0 + c) + gk;      // < KP: KT is a multiple of CH
          const double a = W[al * ld + i];        // rows al >= k meet R's zero rows
#pragma unroll
          for (int n = 0; n < NT; ++n)
            dmma884(dc[c][n][0], dc[c][n][1], a, R[al * NW + 8 * n + gq]);
        }
      }
      double d[NT][2];
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        d[n][0] = dc[0][n][0];
        d[n][1] = dc[0][n][1];
#pragma unroll
        for (int c = 1; c < CH; ++c) {
          d[n][0] += dc[c][n][0];
          d[n][1] += dc[c][n][1];
        }
      }
      // mode rows past k (their A columns were record tails) are stored as the
      // exact zeros the U GEMM's unpredicated A columns must meet
      const bool live = i < k;
#pragma unroll
      for (int n = 0; n < NT; ++n)
        *reinterpret_cast<double2*>(t + i * NW + 8 * n + 2 * gk) =
            live ? make_double2(d[n][0], d[n][1]) : make_double2(0.0, 0.0);
    }
    double pf_val[PF];
#pragma unroll
    for (int u = 0; u < PF; ++u) pf_val[u] = pf_idx[u] >= 0 ? __ldg(r + pf_idx[u]) : 0.0;
    __syncthreads();
    // thread per mode: w_i = E_i t_i, g += c^ w
    double g[S];
#pragma unroll
    for (int a = 0; a < S; ++a) g[a] = 0.0;
    for (int i = tid; i < k; i += NTH) {
      double acc[NA];
      lds_vec<NA>(t + i * NW, acc);
      double E[S * S];
      modal_small_inv<S>(mp.a, dt * th[i], E);
#pragma unroll
      for (int e = 0; e < S * S; ++e) Es[i * S * S + e] = E[e];
#pragma unroll
      for (int dd = 0; dd < NC; ++dd) {
        const double c = ch[i * NC + dd];
#pragma unroll
        for (int a = 0; a < S; ++a) {
          double w = 0.0;
#pragma unroll
          for (int b = 0; b < S; ++b) w = fma(E[a * S + b], acc[dd * S + b], w);
          t[i * NW + dd * S + a] = w;
          g[a] = fma(c, w, g[a]);
        }
      }
    }
#pragma unroll
    for (int a = 0; a < S; ++a) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) g[a] += __shfl_down_sync(0xffffffffu, g[a], o);
    }
    if (lane == 0) {
#pragma unroll
      for (int a = 0; a < S; ++a) gred[warp * 4 + a] = g[a];
    }
    __syncthreads();
    if (tid == 0) {
      double gg[S], rhs[S], pv[S];
#pragma unroll
      for (int a = 0; a < S; ++a) {
        gg[a] = gred[a];
        for (int w = 1; w < kModalCtaWarps; ++w) gg[a] += gred[w * 4 + a];
      }
#pragma unroll
      for (int a = 0; a < S; ++a) {
        double s_ = 0.0;
#pragma unroll
        for (int b = 0; b < S; ++b) s_ = fma(mp.a[a * S + b], gg[b], s_);
        rhs[a] = dt * s_ - Rpc[a];
      }
#pragma unroll
      for (int a = 0; a < S; ++a) {
        double s_ = 0.0;
#pragma unroll
        for (int b = 0; b < S; ++b) s_ = fma(hi[a * S + b], rhs[b], s_);
        pv[a] = s_;
        pAp[a] = s_;
      }
#pragma unroll
      for (int a = 0; a < S; ++a) {
        double s_ = 0.0;
#pragma unroll
        for (int b = 0; b < S; ++b) s_ = fma(mp.a[a * S + b], pv[b], s_);
        pAp[4 + a] = s_;
      }
    }
    __syncthreads();
    for (int i = tid; i < k; i += NTH) {
      double e[S];
#pragma unroll
      for (int a = 0; a < S; ++a) {
        double s_ = 0.0;
#pragma unroll
        for (int b = 0; b < S; ++b) s_ = fma(Es[i * S * S + a * S + b], pAp[4 + b], s_);
        e[a] = s_;
      }
#pragma unroll
      for (int dd = 0; dd < NC; ++dd) {
        const double c = dt * ch[i * NC + dd];
#pragma unroll
        for (int a = 0; a < S; ++a) t[i * NW + dd * S + a] = fma(-c, e[a], t[i * NW + dd * S + a]);
      }
    }
    __syncthreads();
    // U = W V: warp w takes node tiles w, w + 4, ...
    for (int m = warp; m < MT; m += kModalCtaWarps) {
      if (8 * m >= k) break;
      double dc[CH][NT][2];
#pragma unroll
      for (int c = 0; c < CH; ++c)
#pragma unroll
        for (int n = 0; n < NT; ++n) dc[c][n][0] = dc[c][n][1] = 0.0;
      const int al = 8 * m + gq;
      for (int kt0 = 0; kt0 < KT && 4 * kt0 < k; kt0 += CH) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
          const int i = 4 * (kt0 + c) + gk;
          const double a = W[al * ld + i];        // columns i >= k meet t's zero rows
#pragma unroll
          for (int n = 0; n < NT; ++n)
            dmma884(dc[c][n][0], dc[c][n][1], a, t[i * NW + 8 * n + gq]);
        }
      }
      double d[NT][2];
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        d[n][0] = dc[0][n][0];
        d[n][1] = dc[0][n][1];
#pragma unroll
        for (int c = 1; c < CH; ++c) {
          d[n][0] += dc[c][n][0];
          d[n][1] += dc[c][n][1];
        }
      }
      if (al < k) {
#pragma unroll
        for (int n = 0; n < NT; ++n)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int q = 8 * n + 2 * gk + h;
            if (q < NA) {
              const int dd = q / S, a = q - dd * S;
              const int pos = off + a * blk + NC * al + dd;
              st_keep(local + (pd.slot_pos ? pd.slot_pos[pos] : pos), d[n][h]);
            }
          }
      }
    }
    if (tid < S) {
      const int pos = off + tid * blk + NC * k;
      st_keep(local + (pd.slot_pos ? pd.slot_pos[pos] : pos), pAp[tid]);
    }
    // clear t rows this patch wrote (the next patch may be smaller) and land
    // the next patch's r
    {
      double* RN = slot ? R0 : R1;
      double* RPN = Rp + 4 * (slot ^ 1);
      for (int e = pn_k * NW + tid; e < KP * NW; e += NTH) RN[e] = 0.0;

#pragma unroll
      for (int u = 0; u < PF; ++u) {
        const int j = tid + NTH * u;
        if (pf_idx[u] >= 0) {
          const int a = (j >= pn_blk) + (S > 2 && j >= 2 * pn_blk);
          const int e = j - a * pn_blk;
          if (e < NC * pn_k) {
            const int al = e / NC, dd = e - al * NC;
            RN[al * NW + dd * S + a] = pf_val[u];
          } else {
            RPN[a] = pf_val[u];
          }
        }
      }
      for (int j = PF * NTH + tid; pn < pd.num_patches && j < S * pn_blk; j += NTH) {
        const int a = (j >= pn_blk) + (S > 2 && j >= 2 * pn_blk);
        const int e = j - a * pn_blk;
        const double v = __ldg(r + pd.idx[pn_off + j]);
        if (e < NC * pn_k) {
          const int al = e / NC, dd = e - al * NC;
          RN[al * NW + dd * S + a] = v;
        } else {
          RPN[a] = v;
        }
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------- K7g (general path)
//
// One CTA per patch of a general stage operator I_s (x) M + dt A (x) L
// (ivk_general_desc).  The stage-0 block of the patch's idx list is its
// sorted single-stage DoF list (b = m / s entries, identical for every
// stage); a warp per local row walks that row of the single-stage CSR and
// binary-searches each column in the list, so the patch matrix R_i A R_i^T
// is assembled straight into shared memory.  full: the (s b)^2 stage-coupled
// matrix, Gauss-Jordan, Inv^T stored with ld = (m + 3) & ~3 (the K3 layout);
// kron: one (complex) b x b block M^ + dt lam_k L^ per stored eigenvalue,
// stored as G^T in the K3e layout.
struct GenFactorParams {
  int S;
  double dt;
  double a[IVK_MAX_STAGES * IVK_MAX_STAGES];
  const int32_t* __restrict__ rowptr;
  const int32_t* __restrict__ col;
  const double2* __restrict__ ml;
};

constexpr int kGenFactorThreads = 256;
constexpr int kGenMaxD = 512;

__device__ __forceinline__ int find_sorted(const int* a, int n, int v) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    const int c = a[mid];
    if (c == v) return mid;
    if (c < v) lo = mid + 1; else hi = mid;
  }
  return -1;
}

// RT > 0: every matrix of the launch fits the 16 RT x 16 CT register tile
// (ivk_gj.cuh); RT == 0: elimination in shared memory (gauss_jordan above).
// RT > 0 (ivk_gj.cuh): Are / Aim end up holding the TRANSPOSED inverse with
// leading dimension ldo (they must hold d * ldo doubles); RT == 0
// (gauss_jordan above): the inverse itself, leading dimension d.
template <bool CPLX, int RT, int CT, class Scratch>
__device__ __forceinline__ bool general_invert(double* Are, double* Aim, int d, int ldo,
                                               Scratch& gj, int* piv, double* colre,
                                               double* colim, int* s_prow, int* s_bad) {
  if constexpr (RT > 0) return gj_invert_registers<CPLX, 16, RT, CT>(Are, Aim, d, ldo, gj);
  else return gauss_jordan<CPLX>(Are, Aim, d, piv, colre, colim, s_prow, s_bad);
}

template <int RT, int CT>
__global__ void __launch_bounds__(kGenFactorThreads) general_factor_kernel(
    GenFactorParams g, PatchParams pd, KronParams kp, int use_kron, int32_t* singular) {
  extern __shared__ __align__(16) double sm[];
  constexpr bool kReg = RT > 0;
  constexpr int kOld = kReg ? 1 : kGenMaxD;  // the shared-memory path's scratch
  __shared__ int piv[kOld];
  __shared__ double colre[kOld], colim[kOld];
  __shared__ int dofs[kGenMaxD];
  __shared__ int s_prow, s_bad;
  __shared__ GjScratch<true, kReg ? 16 * RT : 1, kReg ? 16 * CT : 1> gj;
  const int p = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5;
  const int off = pd.idx_off[p], m = pd.idx_off[p + 1] - off, S = g.S, b = m / S;
  for (int i = tid; i < b; i += blockDim.x) dofs[i] = pd.idx[off + i];
  if (tid == 0) s_bad = 0;
  __syncthreads();
  if (!use_kron) {
    double* A = sm;
    const int d = m;
    const int ld = (d + 3) & ~3;
    for (int e = tid; e < d * d; e += blockDim.x) A[e] = 0.0;
    __syncthreads();
    for (int i = warp; i < b; i += nw) {
      const int row = dofs[i];
      for (int e = g.rowptr[row] + lane; e < g.rowptr[row + 1]; e += 32) {
        const int j = find_sorted(dofs, b, g.col[e]);
        if (j < 0) continue;
        const double2 v = g.ml[e];
        for (int x = 0; x < S; ++x)
          for (int y = 0; y < S; ++y)
            A[(long)(x * b + i) * d + y * b + j] = (x == y ? v.x : 0.0) + g.dt * g.a[x * S + y] * v.y;
      }
    }
    __syncthreads();
    if (!general_invert<false, RT, CT>(A, nullptr, d, ld, gj, piv, colre, colim, &s_prow, &s_bad)) {
      if (tid == 0) atomicMin(singular, pd.vertex[p]);
      return;
    }
    double* out = pd.inv + pd.inv_off[p];
    for (int e = tid; e < d * ld; e += blockDim.x) {
      if constexpr (kReg) {
        out[e] = A[e];
      } else {
        const int j = e / ld, i = e - j * ld;
        out[e] = (i < d) ? A[(long)i * d + j] : 0.0;
      }
    }
    return;
  }
  double* Are = sm;
  double* Aim = sm + b * kron_ldr(b);
  double* out = pd.inv + pd.inv_off[p];
  for (int k = 0; k < kp.nblk; ++k) {
    const bool cplx = kp.is_complex[k] != 0;
    const double fre = g.dt * kp.lam_re[k], fim = g.dt * kp.lam_im[k];
    for (int e = tid; e < b * b; e += blockDim.x) { Are[e] = 0.0; Aim[e] = 0.0; }
    __syncthreads();
    for (int i = warp; i < b; i += nw) {
      const int row = dofs[i];
      for (int e = g.rowptr[row] + lane; e < g.rowptr[row + 1]; e += 32) {
        const int j = find_sorted(dofs, b, g.col[e]);
        if (j < 0) continue;
        const double2 v = g.ml[e];
        Are[i * b + j] = v.x + fre * v.y;
        Aim[i * b + j] = fim * v.y;
      }
    }
    __syncthreads();
    const int ldo = cplx ? kron_ldc(b) : kron_ldr(b);
    const bool ok =
        cplx ? general_invert<true, RT, CT>(Are, Aim, b, ldo, gj, piv, colre, colim, &s_prow, &s_bad)
             : general_invert<false, RT, CT>(Are, Aim, b, ldo, gj, piv, colre, colim, &s_prow, &s_bad);
    if (!ok) {
      if (tid == 0) atomicMin(singular, pd.vertex[p]);
      return;
    }
    if (cplx) {
      double2* o2 = reinterpret_cast<double2*>(out);
      for (int e = tid; e < b * ldo; e += blockDim.x) {
        if constexpr (kReg) {
          o2[e] = make_double2(Are[e], Aim[e]);
        } else {
          const int j = e / ldo, i = e - j * ldo;
          o2[e] = i < b ? make_double2(Are[i * b + j], Aim[i * b + j]) : make_double2(0.0, 0.0);
        }
      }
      out += 2 * b * ldo;
    } else {
      for (int e = tid; e < b * ldo; e += blockDim.x) {
        if constexpr (kReg) {
          out[e] = Are[e];
        } else {
          const int j = e / ldo, i = e - j * ldo;
          out[e] = (i < b) ? Are[i * b + j] : 0.0;
        }
      }
      out += b * ldo;
    }
    __syncthreads();
  }
}

// Warp per patch.  Gather r_p, transform to the eigenbasis, one streamed
// GEMV per stored block (lanes split into G groups of CPC lanes; each lane
// owns a 32-byte row chunk, groups take interleaved columns), back-transform.
template <int MAXB>
__global__ void __launch_bounds__(kApplyWarps * 32) patch_apply_kron_kernel(
    PatchParams pd, KronParams kp, const double* __restrict__ r, double* __restrict__ local) {
  constexpr int MAXM = IVK_MAX_STAGES * MAXB;
  __shared__ __align__(16) double rs_all[kApplyWarps][MAXM];
  __shared__ __align__(16) double rt_all[kApplyWarps][IVK_MAX_STAGES][2 * MAXB];
  __shared__ __align__(16) double red_all[kApplyWarps][32 * 4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* rs = rs_all[warp];
  double* red = red_all[warp];
  const int S = kp.S;
  const int stride = gridDim.x * kApplyWarps;
  for (int p = blockIdx.x * kApplyWarps + warp; p < pd.num_patches; p += stride) {
    const int off = pd.idx_off[p];
    const int m = pd.idx_off[p + 1] - off;
    const int b = m / S;
    for (int j = lane; j < m; j += 32) rs[j] = __ldg(r + pd.idx[off + j]);
    __syncwarp();
    // r~_k[a] = sum_i Vinv[k][i] r[i][a]
    for (int e = lane; e < kp.nblk * b; e += 32) {
      const int k = e / b, a = e - k * b;
      double re = 0.0, im = 0.0;
      for (int i = 0; i < S; ++i) {
        const double x = rs[i * b + a];
        re = fma(kp.vinv_re[k * S + i], x, re);
        im = fma(kp.vinv_im[k * S + i], x, im);
      }
      rt_all[warp][k][2 * a] = re;
      rt_all[warp][k][2 * a + 1] = im;
    }
    __syncwarp();
    const double* G = pd.inv + pd.inv_off[p];
    for (int k = 0; k < kp.nblk; ++k) {
      double* rt = rt_all[warp][k];
      const bool cplx = kp.is_complex[k] != 0;
      const int ldd = cplx ? 2 * kron_ldc_narrow(b) : kron_ldr(b);  // doubles per column
      const int cpc = ldd >> 2;                               // 32-byte chunks per column
      const int groups = 32 / cpc;
      const int g = lane / cpc, c = lane - g * cpc;
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      if (g < groups) {
        const double* col = G + 4 * c;
        int j = g;
        if (cplx) {
          for (; j + 3 * groups < b; j += 4 * groups) {
            double v[4][4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
              ld_stream4(col + (long)(j + u * groups) * ldd, v[u][0], v[u][1], v[u][2], v[u][3]);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const double xr = rt[2 * (j + u * groups)], xi = rt[2 * (j + u * groups) + 1];
              a0 = fma(v[u][0], xr, fma(-v[u][1], xi, a0));
              a1 = fma(v[u][0], xi, fma(v[u][1], xr, a1));
              a2 = fma(v[u][2], xr, fma(-v[u][3], xi, a2));
              a3 = fma(v[u][2], xi, fma(v[u][3], xr, a3));
            }
          }
          for (; j < b; j += groups) {
            double v0, v1, v2, v3;
            ld_stream4(col + (long)j * ldd, v0, v1, v2, v3);
            const double xr = rt[2 * j], xi = rt[2 * j + 1];
            a0 = fma(v0, xr, fma(-v1, xi, a0));
            a1 = fma(v0, xi, fma(v1, xr, a1));
            a2 = fma(v2, xr, fma(-v3, xi, a2));
            a3 = fma(v2, xi, fma(v3, xr, a3));
          }
        } else {
          for (; j + 3 * groups < b; j += 4 * groups) {
            double v[4][4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
              ld_stream4(col + (long)(j + u * groups) * ldd, v[u][0], v[u][1], v[u][2], v[u][3]);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const double x = rt[2 * (j + u * groups)];
              a0 = fma(v[u][0], x, a0);
              a1 = fma(v[u][1], x, a1);
              a2 = fma(v[u][2], x, a2);
              a3 = fma(v[u][3], x, a3);
            }
          }
          for (; j < b; j += groups) {
            double v0, v1, v2, v3;
            ld_stream4(col + (long)j * ldd, v0, v1, v2, v3);
            const double x = rt[2 * j];
            a0 = fma(v0, x, a0);
            a1 = fma(v1, x, a1);
            a2 = fma(v2, x, a2);
            a3 = fma(v3, x, a3);
          }
        }
      }
      red[4 * lane + 0] = a0;
      red[4 * lane + 1] = a1;
      red[4 * lane + 2] = a2;
      red[4 * lane + 3] = a3;
      __syncwarp();
      // z~_k[a] = sum over groups; overwrite rt[k] (no longer needed)
      if (cplx) {
        for (int a = lane; a < b; a += 32) {
          const int ch = a >> 1, q = (a & 1) * 2;
          double re = 0.0, im = 0.0;
          for (int gg = 0; gg < groups; ++gg) {
            re += red[4 * (gg * cpc + ch) + q];
            im += red[4 * (gg * cpc + ch) + q + 1];
          }
          rt[2 * a] = re;
          rt[2 * a + 1] = im;
        }
        G += 2L * b * kron_ldc_narrow(b);
      } else {
        for (int a = lane; a < b; a += 32) {
          const int ch = a >> 2, q = a & 3;
          double re = 0.0;
          for (int gg = 0; gg < groups; ++gg) re += red[4 * (gg * cpc + ch) + q];
          rt[2 * a] = re;
          rt[2 * a + 1] = 0.0;
        }
        G += (long)b * kron_ldr(b);
      }
      __syncwarp();
    }
    // z[i][a] = sum_k scale_k Re(V[i][k] z~_k[a])
    for (int e = lane; e < m; e += 32) {
      const int i = e / b, a = e - i * b;
      double acc = 0.0;
      for (int k = 0; k < kp.nblk; ++k) {
        const double zr = rt_all[warp][k][2 * a], zi = rt_all[warp][k][2 * a + 1];
        acc += kp.scale[k] * (kp.v_re[i * S + k] * zr - kp.v_im[i * S + k] * zi);
      }
      st_keep(local + (pd.slot_pos ? pd.slot_pos[off + e] : off + e), acc);
    }
    __syncwarp();
  }
}

// Blocks up to b = 256 (MHD: b = 78, 3-D Stokes: b = 176): the same algorithm with
// per-warp buffers in dynamic shared memory; complex blocks wider than 64
// rows (more than 32 chunks per column) take a multi-pass column walk.
// Dynamic shared memory: per warp S*bmax (r_p) + nblk*2*bmax (eigenbasis
// vectors) + 2*bmax + 128 (partials) doubles.
__host__ __device__ __forceinline__ int kron_apply_seg(int S, int nblk, int bmax) {
  return S * bmax + nblk * 2 * bmax + 128 + 2 * bmax + 8;
}

__global__ void __launch_bounds__(kApplyWarps * 32, 4) patch_apply_kron_wide_kernel(
    PatchParams pd, KronParams kp, const double* __restrict__ r, double* __restrict__ local,
    int bmax) {
  extern __shared__ __align__(16) double kron_sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = kp.S;
  double* rs = kron_sm + (long)warp * kron_apply_seg(S, kp.nblk, bmax);
  double* rtb = rs + S * bmax;                 // block k: rtb + k * 2 * bmax
  double* red = rtb + kp.nblk * 2 * bmax;      // 128 partials
  double* zt = red + 128;                      // block result, chunk layout
  const int stride = gridDim.x * kApplyWarps;
  for (int p = blockIdx.x * kApplyWarps + warp; p < pd.num_patches; p += stride) {
    const int off = pd.idx_off[p];
    const int m = pd.idx_off[p + 1] - off;
    const int b = m / S;
    for (int j = lane; j < m; j += 32) rs[j] = __ldg(r + pd.idx[off + j]);
    __syncwarp();
    // r~_k[a] = sum_i Vinv[k][i] r[i][a]
    for (int e = lane; e < kp.nblk * b; e += 32) {
      const int k = e / b, a = e - k * b;
      double re = 0.0, im = 0.0;
      for (int i = 0; i < S; ++i) {
        const double x = rs[i * b + a];
        re = fma(kp.vinv_re[k * S + i], x, re);
        im = fma(kp.vinv_im[k * S + i], x, im);
      }
      rtb[k * 2 * bmax + 2 * a] = re;
      rtb[k * 2 * bmax + 2 * a + 1] = im;
    }
    __syncwarp();
    const double* G = pd.inv + pd.inv_off[p];
    for (int k = 0; k < kp.nblk; ++k) {
      double* rt = rtb + k * 2 * bmax;
      const bool cplx = kp.is_complex[k] != 0;
      const int ldd = cplx ? 2 * kron_ldc(b) : kron_ldr(b);  // doubles per column
      const int cpc = ldd >> 2;                               // 32-byte chunks per column
      // passes of <= 32 chunks; inside a pass the lanes split into
      // groups = 32 / cc groups of cc lanes (one 32-byte row chunk each) that
      // take interleaved columns, so a 39-chunk complex column (b = 78) runs
      // as 32 chunks x 1 group, then 7 chunks x 4 groups
      for (int c0 = 0; c0 < cpc; c0 += 32) {
        const int cc = min(32, cpc - c0);
        const int groups = 32 / cc;
        const int g = lane / cc, c = c0 + lane - g * cc;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        if (g < groups) {
          const double* col = G + 4 * c;
          int j = g;
          for (; j + 3 * groups < b; j += 4 * groups) {
            double v[4][4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
              ld_stream4(col + (long)(j + u * groups) * ldd, v[u][0], v[u][1], v[u][2], v[u][3]);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const double xr = rt[2 * (j + u * groups)], xi = rt[2 * (j + u * groups) + 1];
              if (cplx) {
                a0 = fma(v[u][0], xr, fma(-v[u][1], xi, a0));
                a1 = fma(v[u][0], xi, fma(v[u][1], xr, a1));
                a2 = fma(v[u][2], xr, fma(-v[u][3], xi, a2));
                a3 = fma(v[u][2], xi, fma(v[u][3], xr, a3));
              } else {
                a0 = fma(v[u][0], xr, a0);
                a1 = fma(v[u][1], xr, a1);
                a2 = fma(v[u][2], xr, a2);
                a3 = fma(v[u][3], xr, a3);
              }
            }
          }
          for (; j < b; j += groups) {
            double v0, v1, v2, v3;
            ld_stream4(col + (long)j * ldd, v0, v1, v2, v3);
            const double xr = rt[2 * j], xi = rt[2 * j + 1];
            if (cplx) {
              a0 = fma(v0, xr, fma(-v1, xi, a0));
              a1 = fma(v0, xi, fma(v1, xr, a1));
              a2 = fma(v2, xr, fma(-v3, xi, a2));
              a3 = fma(v2, xi, fma(v3, xr, a3));
            } else {
              a0 = fma(v0, xr, a0);
              a1 = fma(v1, xr, a1);
              a2 = fma(v2, xr, a2);
              a3 = fma(v3, xr, a3);
            }
          }
        }
        red[4 * lane + 0] = a0;
        red[4 * lane + 1] = a1;
        red[4 * lane + 2] = a2;
        red[4 * lane + 3] = a3;
        __syncwarp();
        // fixed-order sum over the groups -> zt[4 c .. 4 c + 3]
        for (int e = lane; e < 4 * cc; e += 32) {
          const int ch = e >> 2, q = e & 3;
          double acc = 0.0;
          for (int gg = 0; gg < groups; ++gg) acc += red[4 * (gg * cc + ch) + q];
          zt[4 * (c0 + ch) + q] = acc;
        }
        __syncwarp();
      }
      // z~_k: complex chunks hold (re, im) interleaved rows, real chunks 4 rows
      for (int a = lane; a < b; a += 32) {
        if (cplx) {
          rt[2 * a] = zt[2 * a];
          rt[2 * a + 1] = zt[2 * a + 1];
        } else {
          rt[2 * a] = zt[a];
          rt[2 * a + 1] = 0.0;
        }
      }
      G += cplx ? 2L * b * kron_ldc(b) : (long)b * kron_ldr(b);
      __syncwarp();
    }
    // z[i][a] = sum_k scale_k Re(V[i][k] z~_k[a])
    for (int e = lane; e < m; e += 32) {
      const int i = e / b, a = e - i * b;
      double acc = 0.0;
      for (int k = 0; k < kp.nblk; ++k) {
        const double zr = rtb[k * 2 * bmax + 2 * a], zi = rtb[k * 2 * bmax + 2 * a + 1];
        acc += kp.scale[k] * (kp.v_re[i * S + k] * zr - kp.v_im[i * S + k] * zi);
      }
      st_keep(local + (pd.slot_pos ? pd.slot_pos[off + e] : off + e), acc);
    }
    __syncwarp();
  }
}

// K3d: dedup -- class-batched eigen-block GEMM.  Patches of one class share
// their blocks, so a tile of up to kClassTile same-class patches is one small
// GEMM per block, Z_k = G_k R_k (b x b times b x T), with G_k staged once in
// shared memory and reused across the tile from registers: each lane owns a
// 2-row x 2-patch complex (or 4 x 4 real) micro-tile, i.e. 16 FMAs per 8
// doubles of shared-memory operands.  Per tile: gather r in the class's
// canonical order (perm) -> V^-1 transform -> GEMM -> V back-transform ->
// scatter to each patch's own local[] layout.  Tiles cover `order` contiguously
// (tile_start), grouped by class; a CTA reloads G only when the class changes.
constexpr int kClassTile = 32;
constexpr int kClassCtas = 2;   // resident CTAs per SM (smem ~98 KB at cfg2)
constexpr int kClassWarps = 8;

__device__ __forceinline__ void cgemm_item(const double* __restrict__ G, const double* __restrict__ R,
                                           double* __restrict__ Z, int b, int ldc, int i0, int t0) {
  // rows i0, i0+1; patches t0, t0+1; complex, (re, im) interleaved
  double a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll 2
  for (int j = 0; j < b; ++j) {
    const double2 g0 = *reinterpret_cast<const double2*>(G + 2 * (j * ldc + i0));
    const double2 g1 = *reinterpret_cast<const double2*>(G + 2 * (j * ldc + i0) + 2);
    const double2 x0 = *reinterpret_cast<const double2*>(R + 2 * (j * kClassTile + t0));
    const double2 x1 = *reinterpret_cast<const double2*>(R + 2 * (j * kClassTile + t0) + 2);
    a[0] = fma(g0.x, x0.x, fma(-g0.y, x0.y, a[0]));
    a[1] = fma(g0.x, x0.y, fma(g0.y, x0.x, a[1]));
    a[2] = fma(g0.x, x1.x, fma(-g0.y, x1.y, a[2]));
    a[3] = fma(g0.x, x1.y, fma(g0.y, x1.x, a[3]));
    a[4] = fma(g1.x, x0.x, fma(-g1.y, x0.y, a[4]));
    a[5] = fma(g1.x, x0.y, fma(g1.y, x0.x, a[5]));
    a[6] = fma(g1.x, x1.x, fma(-g1.y, x1.y, a[6]));
    a[7] = fma(g1.x, x1.y, fma(g1.y, x1.x, a[7]));
  }
#pragma unroll
  for (int r = 0; r < 2; ++r)
    if (i0 + r < b)
      *reinterpret_cast<double4*>(Z + 2 * ((i0 + r) * kClassTile + t0)) =
          make_double4(a[4 * r], a[4 * r + 1], a[4 * r + 2], a[4 * r + 3]);
}

__device__ __forceinline__ void rgemm_item(const double* __restrict__ G, const double* __restrict__ R,
                                           double* __restrict__ Z, int b, int ldr, int i0, int t0) {
  // rows i0..i0+3; patches t0..t0+3; real
  double a[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) a[u] = 0.0;
#pragma unroll 2
  for (int j = 0; j < b; ++j) {
    const double4 g = *reinterpret_cast<const double4*>(G + j * ldr + i0);
    const double4 x = *reinterpret_cast<const double4*>(R + j * kClassTile + t0);
    const double gv[4] = {g.x, g.y, g.z, g.w};
    const double xv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int t = 0; t < 4; ++t) a[4 * r + t] = fma(gv[r], xv[t], a[4 * r + t]);
  }
#pragma unroll
  for (int r = 0; r < 4; ++r)
    if (i0 + r < b)
      *reinterpret_cast<double4*>(Z + (i0 + r) * kClassTile + t0) =
          make_double4(a[4 * r], a[4 * r + 1], a[4 * r + 2], a[4 * r + 3]);
}

// S stages, NR real eigen-blocks first, then (S - NR) / 2 complex pair blocks:
// the transforms unroll completely, so V / V^-1 / scale are immediate
// constant-bank operands.
template <int S, int NR>
__global__ void __launch_bounds__(kClassWarps * 32, kClassCtas) patch_apply_class_kernel(
    PatchParams pd, DedupParams dd, KronParams kp, const double* __restrict__ r,
    double* __restrict__ local, int g_doubles) {
  constexpr int NB = NR + (S - NR) / 2;
  constexpr int T = kClassTile;
  constexpr int GU = 16;  // gather / scatter loads in flight per thread
  extern __shared__ __align__(32) double csm[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int mt = pd.max_m * T;     // R / Z region size (doubles)
  double* Gs = csm;                // class blocks (+ slack)
  double* Rs = csm + g_doubles;    // transformed residuals, block-major
  double* Zs = Rs + mt;            // raw gather, then block results
  int cur_class = -1;
  for (int tile = blockIdx.x; tile < dd.n_tiles; tile += gridDim.x) {
    const int cnt = dd.tile_start[tile + 1] - dd.tile_start[tile];
    const int cls = dd.tile_class[tile];
    const int toff = dd.tile_off[tile];
    const int m = (dd.tile_off[tile + 1] - toff) / cnt;
    const int b = m / S;
    if (cls != cur_class) {
      // every CTA thread has finished the previous tile (trailing sync)
      const double* src = dd.class_inv + dd.class_inv_off[cls];
      const int nd = (int)(dd.class_inv_off[cls + 1] - dd.class_inv_off[cls]);
      for (int e = tid; e < nd / 2; e += blockDim.x)
        reinterpret_cast<double2*>(Gs)[e] = __ldg(reinterpret_cast<const double2*>(src) + e);
      cur_class = cls;
    }
    // gather (canonical order; the tile's gather list is contiguous), zero
    // padding past cnt; all index loads, then all value loads, in flight
    {
      const int n = cnt * m, nt = T * m;
      const int32_t* ci = dd.cidx + toff;
      for (int e0 = tid; e0 < nt; e0 += GU * blockDim.x) {
        int ix[GU];
        double v[GU];
#pragma unroll
        for (int u = 0; u < GU; ++u) {
          const int e = e0 + u * blockDim.x;
          ix[u] = e < n ? __ldg(ci + e) : -1;
        }
#pragma unroll
        for (int u = 0; u < GU; ++u) v[u] = ix[u] >= 0 ? __ldg(r + ix[u]) : 0.0;
#pragma unroll
        for (int u = 0; u < GU; ++u) {
          const int e = e0 + u * blockDim.x;
          if (e < nt) Zs[e] = v[u];
        }
      }
    }
    __syncthreads();
    // r~_k[a][t] = sum_i Vinv[k][i] r_t[i b + a]; real blocks [b][T], complex [b][T] x 2
    for (int e = tid; e < b * T; e += blockDim.x) {
      const int a = e / T, t = e % T;
      double x[S];
#pragma unroll
      for (int i = 0; i < S; ++i) x[i] = Zs[t * m + i * b + a];
#pragma unroll
      for (int k = 0; k < NB; ++k) {
        double re = 0.0, im = 0.0;
#pragma unroll
        for (int i = 0; i < S; ++i) {
          re = fma(kp.vinv_re[k * S + i], x[i], re);
          if (k >= NR) im = fma(kp.vinv_im[k * S + i], x[i], im);
        }
        if (k < NR)
          Rs[k * b * T + e] = re;
        else
          *reinterpret_cast<double2*>(Rs + (NR + 2 * (k - NR)) * b * T + 2 * e) =
              make_double2(re, im);
      }
    }
    __syncthreads();
    // GEMM items: complex blocks as 8-row x 16-patch warp tiles, real blocks as
    // 512/T-row x T-patch warp tiles (16 FMAs per column either way)
    {
      const int ci = ((b + 7) >> 3) * (T / 16);   // items per complex block
      constexpr int RQ = 128 / T;                 // real: RQ row quads x T/4 patch quads
      const int ri = (b + 4 * RQ - 1) / (4 * RQ); // items per real block
      const int n_items = NR * ri + (NB - NR) * ci;
      for (int it = warp; it < n_items; it += kClassWarps) {
        if (it < NR * ri) {
          const int k = it / ri, li = it - k * ri;
          rgemm_item(Gs + k * b * kron_ldr(b), Rs + k * b * T, Zs + k * b * T, b, kron_ldr(b),
                     4 * RQ * li + 4 * (lane % RQ), 4 * (lane / RQ));
        } else {
          const int kc = (it - NR * ri) / ci, li = it - NR * ri - kc * ci;
          const int goff = NR * b * kron_ldr(b) + kc * 2 * b * kron_ldc_narrow(b);
          const int roff = (NR + 2 * kc) * b * T;
          const int rg = li / (T / 16), pg = li - rg * (T / 16);
          cgemm_item(Gs + goff, Rs + roff, Zs + roff, b, kron_ldc_narrow(b), 8 * rg + 2 * (lane & 3),
                     16 * pg + 2 * (lane >> 2));
        }
      }
    }
    __syncthreads();
    // z_t[i b + a] = sum_k scale_k Re(V[i][k] z~_k[a][t]) into Rs as [t][m]
    for (int e = tid; e < b * T; e += blockDim.x) {
      const int a = e / T, t = e % T;
      double zr[NB], zi[NB];
#pragma unroll
      for (int k = 0; k < NB; ++k) {
        if (k < NR) {
          zr[k] = Zs[k * b * T + e];
          zi[k] = 0.0;
        } else {
          const double2 z =
              *reinterpret_cast<const double2*>(Zs + (NR + 2 * (k - NR)) * b * T + 2 * e);
          zr[k] = z.x;
          zi[k] = z.y;
        }
      }
#pragma unroll
      for (int i = 0; i < S; ++i) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < NB; ++k) {
          if (k < NR)
            acc += kp.scale[k] * kp.v_re[i * S + k] * zr[k];
          else
            acc += kp.scale[k] * (kp.v_re[i * S + k] * zr[k] - kp.v_im[i * S + k] * zi[k]);
        }
        Rs[t * m + i * b + a] = acc;
      }
    }
    __syncthreads();
    // scatter to each patch's own local[] layout (slot-fastest: near-contiguous)
    {
      const int n = cnt * m;
      const int32_t* cd = dd.cdst + toff;
      for (int e0 = tid; e0 < n; e0 += GU * blockDim.x) {
        int ix[GU];
#pragma unroll
        for (int u = 0; u < GU; ++u) {
          const int e = e0 + u * blockDim.x;
          ix[u] = e < n ? __ldg(cd + e) : -1;
        }
#pragma unroll
        for (int u = 0; u < GU; ++u)
          if (ix[u] >= 0) st_keep(local + ix[u], Rs[e0 + u * blockDim.x]);
      }
    }
    __syncthreads();
  }
}

// K3e-sym: complex-symmetric eigen-blocks (Stokes) stored as the lower
// tile-triangle of 4x4 tiles in tile-diagonal order.  Lane L owns rows
// 4L..4L+3.  In step d lane L (>= d) loads tile (L, L-d) -- consecutive lanes
// read consecutive 32-byte chunks, 256-bit evict-first loads -- and uses it
// twice: as stored for its own rows (x chunk L-d) and transposed for rows of
// chunk L-d (x chunk L), whose 4 partial sums it hands to lane L-d with one
// shuffle.  Every tile is read from HBM exactly once.
// One tile of one block in step d: as-stored product into acc, transposed
// product into w (for chunk L - d).
template <bool CPLX>
__device__ __forceinline__ void sym_tile_step(const double* v, const double* xa,
                                              const double* xt, bool diag, double* acc,
                                              double* w) {
#pragma unroll
  for (int r = 0; r < 4; ++r) {
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
      if (CPLX) {
        const double gr = v[8 * r + 2 * cc], gi = v[8 * r + 2 * cc + 1];
        const double ar = xa[2 * cc], ai = xa[2 * cc + 1];
        acc[2 * r] = fma(gr, ar, fma(-gi, ai, acc[2 * r]));
        acc[2 * r + 1] = fma(gr, ai, fma(gi, ar, acc[2 * r + 1]));
        if (!diag) {  // G[4(L-d)+cc][4L+r] = tile[r][cc]
          const double br = xt[2 * r], bi = xt[2 * r + 1];
          w[2 * cc] = fma(gr, br, fma(-gi, bi, w[2 * cc]));
          w[2 * cc + 1] = fma(gr, bi, fma(gi, br, w[2 * cc + 1]));
        }
      } else {
        const double g = v[4 * r + cc];
        acc[r] = fma(g, xa[2 * cc], acc[r]);
        if (!diag) w[cc] = fma(g, xt[2 * r], w[cc]);
      }
    }
  }
}

// One stored block (real or complex) of one patch over the tile diagonals.
// nt: this lane's patch; ntw: warp maximum (uniform loop for the full-mask
// shuffles).
template <bool CPLX>
__device__ __forceinline__ void sym_diag_block(const double* __restrict__ T, int nt, int ntw,
                                               int L, const double* __restrict__ x,
                                               double* __restrict__ z) {
  constexpr int QC = CPLX ? 8 : 4;
  constexpr int NV = CPLX ? 8 : 4;
  double acc[NV];
#pragma unroll
  for (int q = 0; q < NV; ++q) acc[q] = 0.0;
  const double* base = T;
#pragma unroll 1
  for (int d = 0; d < ntw; ++d) {
    const int len = nt - d;
    double w[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) w[q] = 0.0;
    if (d < nt && L >= d && L < nt) {
      double v[4 * QC];
#pragma unroll
      for (int q = 0; q < QC; ++q)
        ld_stream4(base + 4 * (q * len + (L - d)), v[4 * q], v[4 * q + 1], v[4 * q + 2],
                   v[4 * q + 3]);
      sym_tile_step<CPLX>(v, x + 8 * (L - d), x + 8 * L, d == 0, acc, w);
    }
    if (d > 0) {
      const bool take = L + d < nt;
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        const double o = __shfl_down_sync(0xffffffffu, w[q], d);
        if (take) acc[q] += o;
      }
    }
    if (d < nt) base += 4 * QC * len;
  }
  if (L < nt) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      z[2 * (4 * L + r)] = CPLX ? acc[2 * r] : acc[r];
      z[2 * (4 * L + r) + 1] = CPLX ? acc[2 * r + 1] : 0.0;
    }
  }
}

template <int NR, bool HAS_C>
__device__ __forceinline__ void sym_diag_patch(const double* __restrict__ G, int nt, int ntw,
                                               int L, const double* __restrict__ x,
                                               double* __restrict__ z, int MAXP) {
  const int realsz = 16 * (nt * (nt + 1) / 2);
#pragma unroll
  for (int k = 0; k < NR; ++k)
    sym_diag_block<false>(G + k * realsz, nt, ntw, L, x + k * 2 * MAXP, z + k * 2 * MAXP);
  if (HAS_C)
    sym_diag_block<true>(G + NR * realsz, nt, ntw, L, x + NR * 2 * MAXP, z + NR * 2 * MAXP);
}

// Lanes are split into `ng` groups of `gs` lanes (gs >= the largest nt), one
// patch per group, so small blocks (nt = 10 at b = 39) still keep 30 of 32
// lanes busy.  Dynamic shared memory per group:
// rs[S*MAXP] | rt[nblk][2*MAXP] | zt[nblk][2*MAXP].
constexpr int kSymWarps = 4;

template <int NR, bool HAS_C>
__global__ void __launch_bounds__(kSymWarps * 32) patch_apply_kron_sym_kernel(
    PatchParams pd, KronParams kp, const double* __restrict__ r, double* __restrict__ local,
    int MAXP, int gs) {
  extern __shared__ __align__(16) double sym_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ng = 32 / gs;
  const int grp = lane / gs, gl = lane - grp * gs;
  const bool active = grp < ng;
  const int per_group = kp.S * MAXP + 4 * kp.nblk * MAXP;
  double* rs = sym_smem + (warp * ng + (active ? grp : 0)) * per_group;
  double* rt_base = rs + kp.S * MAXP;
  double* zt_base = rt_base + 2 * kp.nblk * MAXP;
  const int S = kp.S;
  const int first = (blockIdx.x * kSymWarps + warp) * ng + grp;
  const int stride = gridDim.x * kSymWarps * ng;
  const int warp_first = (blockIdx.x * kSymWarps + warp) * ng;
  for (int base = warp_first; base < pd.num_patches; base += stride) {
    const int p = first + (base - warp_first);
    const bool valid = active && p < pd.num_patches;
    int off = 0, m = 0, b = 1, nt = 0;
    if (valid) {
      off = pd.idx_off[p];
      m = pd.idx_off[p + 1] - off;
      b = m / S;
      nt = (b + 3) >> 2;
    }
    for (int j = gl; j < m; j += gs) rs[j] = __ldg(r + pd.idx[off + j]);
    __syncwarp();
    for (int e = gl; e < kp.nblk * 4 * nt; e += gs) {
      const int k = e / (4 * nt), a = e - k * 4 * nt;
      double re = 0.0, im = 0.0;
      if (a < b) {
        for (int i = 0; i < S; ++i) {
          const double xv = rs[i * b + a];
          re = fma(kp.vinv_re[k * S + i], xv, re);
          im = fma(kp.vinv_im[k * S + i], xv, im);
        }
      }
      rt_base[k * 2 * MAXP + 2 * a] = re;
      rt_base[k * 2 * MAXP + 2 * a + 1] = im;
    }
    __syncwarp();
    {
      // all lanes take part (the shuffles), inactive groups with nt = 0
      const double* G = valid ? pd.inv + pd.inv_off[p] : pd.inv;
      const int ntv = valid ? nt : 0;
      const int ntw = __reduce_max_sync(0xffffffffu, (unsigned)ntv);
      sym_diag_patch<NR, HAS_C>(G, ntv, ntw, gl, rt_base, zt_base, MAXP);
    }
    __syncwarp();
    for (int e = gl; e < m; e += gs) {
      const int i = e / b, a = e - i * b;
      double acc = 0.0;
      for (int k = 0; k < kp.nblk; ++k) {
        const double zr = zt_base[k * 2 * MAXP + 2 * a], zi = zt_base[k * 2 * MAXP + 2 * a + 1];
        acc += kp.scale[k] * (kp.v_re[i * S + k] * zr - kp.v_im[i * S + k] * zi);
      }
      st_keep(local + (pd.slot_pos ? pd.slot_pos[off + e] : off + e), acc);
    }
    __syncwarp();
  }
}

}  // namespace ivk

using namespace ivk;

extern "C" {

int ivk_patch_apply(const ivk_patch_desc* pd, const double* r, double* local, void* stream) {
  int rc = validate_patches(pd);
  if (rc) return rc;
  IVK_REQUIRE(r && local, "r/local is NULL");
  PatchParams p = make_patch_params(pd);
  const int blocks_needed = (pd->num_patches + kApplyWarps - 1) / kApplyWarps;
  int grid = blocks_needed;
  const int cap = kSMs * 8;  // persistent-ish: 8 CTAs (64 warps) per SM
  if (grid > cap) grid = cap;
  cudaStream_t st = as_stream(stream);
  if (pd->modal) {
    const ivk_modal_desc* md = pd->modal;
    IVK_REQUIRE(pd->node_off != nullptr, "modal store needs the per-patch node counts");
    IVK_REQUIRE(md->stages >= 1 && md->stages <= IVK_MAX_STAGES && (md->ncomp == 2 || md->ncomp == 3),
                "bad modal descriptor");
    ModalParams mp;
    mp.S = md->stages;
    mp.NC = md->ncomp;
    mp.dt = md->dt;
    for (int i = 0; i < IVK_MAX_STAGES * IVK_MAX_STAGES; ++i) mp.a[i] = md->butcher_a[i];
    const int kmax = (pd->max_m / md->stages - 1) / md->ncomp;
    size_t seg = 0;
    void (*fn)(PatchParams, ModalParams, const double*, double*, int) = nullptr;
    size_t seg_tc = 0;
    if (kmax <= 32) {
      IVK_REQUIRE(md->layout == 1, "modal patches with k <= 32 need the fragment layout");
      // FP64 tensor-core variant (K padded to 24 or 32 node slots)
      const int KP = kmax <= 24 ? 24 : 32;
      seg_tc = (size_t)modal_tc_seg(mp.S, mp.NC, kmax, KP) * sizeof(double);
      // K steps: ceil(kmax / 4); below 24 nodes the 24-slot kernel runs 6
      const int ktx = KP == 24 ? ((kmax + 3) / 4 <= 5 ? 5 : 6) : ((kmax + 3) / 4 <= 7 ? 7 : 8);
#define IVK_TC(SS, CC)                                                                         \
  if (mp.S == SS && mp.NC == CC)                                                               \
    fn = KP == 24 ? (ktx == 5 ? patch_apply_modal_tc_kernel<SS, CC, 24, 5>                     \
                              : patch_apply_modal_tc_kernel<SS, CC, 24, 6>)                    \
                  : (ktx == 7 ? patch_apply_modal_tc_kernel<SS, CC, 32, 7>                     \
                              : patch_apply_modal_tc_kernel<SS, CC, 32, 8>);
      IVK_TC(1, 2) IVK_TC(2, 2) IVK_TC(3, 2) IVK_TC(1, 3) IVK_TC(2, 3) IVK_TC(3, 3)
#undef IVK_TC
    }
    if (fn == nullptr && kmax <= 72) {
      IVK_REQUIRE(md->layout == 0, "the modal CTA kernel needs the reference layout");
      // large (3-D: k = 65) patches: CTA per patch, its warps sharing the tiles
      const size_t smem = (size_t)modal_cta_smem(mp.S, mp.NC, kmax, 72) * sizeof(double);
      IVK_REQUIRE(smem <= 200 * 1024, "modal patch (k = %d) exceeds shared memory", kmax);
#define IVK_CTA(SS, CC) \
  if (mp.S == SS && mp.NC == CC) fn = patch_apply_modal_cta_kernel<SS, CC, 72>;
      IVK_CTA(1, 2) IVK_CTA(2, 2) IVK_CTA(3, 2) IVK_CTA(1, 3) IVK_CTA(2, 3) IVK_CTA(3, 3)
#undef IVK_CTA
      if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) {
          set_error("ivk_patch_apply: %s", cudaGetErrorString(e));
          return IVK_ECUDA;
        }
      }
      const int per_sm = (int)((226 * 1024) / (smem + 1024));
      int cgrid = kSMs * (per_sm < 1 ? 1 : per_sm);
      if (cgrid > pd->num_patches) cgrid = pd->num_patches;
      fn<<<cgrid, kModalCtaWarps * 32, smem, st>>>(p, mp, r, local, kmax);
      return check_launch("ivk_patch_apply(modal, cta)");
    }
    if (fn == nullptr) {
      set_error("ivk_patch_apply: modal patches with k = %d > 72 nodes unsupported", kmax);
      return IVK_EUNSUPPORTED;
    }
    seg = seg_tc;
    // CTA shape: cps CTAs per SM (4 x 4 warps at cfg2: 117.9 us vs 119.3 for
    // 3 x 5 and 121.3 for 5 x 3), each as many warps as both the per-warp
    // buffers (cta_kb of shared memory) and the register file allow -- the
    // kernel is bound by its shared-memory pipe, not by latency, so more
    // resident warps past ~15 per SM do not help (measured: 16 warps in two
    // CTAs are 6% slower than 15 in three).  Env overrides for A/B runs.
    static const int cta_kb = getenv("IVK_MODAL_CTA_KB") ? atoi(getenv("IVK_MODAL_CTA_KB")) : 72;
    static const int cps = getenv("IVK_MODAL_CPS") ? atoi(getenv("IVK_MODAL_CPS")) : 4;
    int nw = (int)((cta_kb * 1024) / seg);
    {
      cudaFuncAttributes fa;
      if (cudaFuncGetAttributes(&fa, fn) == cudaSuccess && fa.numRegs > 0) {
        const int regs_warp = ((fa.numRegs * 32 + 255) / 256) * 256;   // 256-register granules
        const int reg_nw = 65536 / regs_warp / cps;
        if (nw > reg_nw) nw = reg_nw;
      }
    }
    if (nw > kApplyWarps) nw = kApplyWarps;
    if (nw > IVK_K3M_MAXT / 32) nw = IVK_K3M_MAXT / 32;
    if (nw < 1) nw = 1;
    IVK_REQUIRE(seg <= 200 * 1024, "modal patch (k = %d) exceeds shared memory", kmax);
    const size_t smem = seg * nw;
    if (smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) {
        set_error("ivk_patch_apply: %s", cudaGetErrorString(e));
        return IVK_ECUDA;
      }
    }
    int mgrid = (pd->num_patches + nw - 1) / nw;
    const int cap = kSMs * cps;
    if (mgrid > cap) mgrid = cap;
    fn<<<mgrid, nw * 32, smem, st>>>(p, mp, r, local, kmax);
    return check_launch("ivk_patch_apply(modal)");
  }
  if (pd->kron) {
    const ivk_kron_desc* k = pd->kron;
    IVK_REQUIRE(k->nblk >= 1 && k->nblk <= IVK_MAX_STAGES, "bad kron block count");
    int S = 0;
    for (int i = 0; i < k->nblk; ++i) S += k->is_complex[i] ? 2 : 1;
    KronParams kp = make_kron(k, S);
    const int bmax = pd->max_m / S;
    if (k->symmetric) {
      IVK_REQUIRE(bmax <= 64, "kron block size %d > 64 unsupported", bmax);
      const int maxp = (bmax + 3) & ~3;
      const int nt_max = maxp >> 2;
      const int gs = nt_max <= 8 ? 8 : nt_max <= 10 ? 10 : nt_max <= 16 ? 16 : 32;
      const int ng = 32 / gs;
      const size_t smem =
          (size_t)kSymWarps * ng * (S * maxp + 4 * k->nblk * maxp) * sizeof(double);
      int nr = 0;
      for (int q = 0; q < k->nblk; ++q) nr += k->is_complex[q] ? 0 : 1;
      const bool hc = nr < k->nblk;
      // stored blocks are real first, then at most one complex (pair) block
      void (*fn)(PatchParams, KronParams, const double*, double*, int, int) = nullptr;
      if (nr == 1 && hc) fn = patch_apply_kron_sym_kernel<1, true>;
      else if (nr == 0 && hc) fn = patch_apply_kron_sym_kernel<0, true>;
      else if (nr == 1) fn = patch_apply_kron_sym_kernel<1, false>;
      else if (nr == 2) fn = patch_apply_kron_sym_kernel<2, false>;
      else if (nr == 3) fn = patch_apply_kron_sym_kernel<3, false>;
      IVK_REQUIRE(fn != nullptr, "unsupported eigen-block signature");
      cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem);
      if (e != cudaSuccess) {
        set_error("ivk_patch_apply: %s", cudaGetErrorString(e));
        return IVK_ECUDA;
      }
      int sgrid = (pd->num_patches + kSymWarps * ng - 1) / (kSymWarps * ng);
      if (sgrid > kSMs * 16) sgrid = kSMs * 16;
      fn<<<sgrid, kSymWarps * 32, smem, st>>>(p, kp, r, local, maxp, gs);
      return check_launch("ivk_patch_apply(kron-sym)");
    }
    if (bmax <= 64 && pd->n_classes > 0) {
      IVK_REQUIRE(pd->class_inv_off && pd->class_inv && pd->tile_start && pd->tile_class &&
                      pd->tile_off && pd->cidx && pd->cdst && pd->n_tiles > 0,
                  "dedup descriptor has a NULL array");
      DedupParams dd;
      dd.n_classes = pd->n_classes;
      dd.n_tiles = pd->n_tiles;
      dd.class_inv_off = pd->class_inv_off;
      dd.class_inv = pd->class_inv;
      dd.tile_start = pd->tile_start;
      dd.tile_class = pd->tile_class;
      dd.tile_off = pd->tile_off;
      dd.cidx = pd->cidx;
      dd.cdst = pd->cdst;
      int g = 0;
      for (int q = 0; q < k->nblk; ++q)
        g += k->is_complex[q] ? 2 * bmax * kron_ldc_narrow(bmax) : bmax * kron_ldr(bmax);
      g = ((g + 3) & ~3) + 32;  // slack: edge micro-tiles read past the last column
      const size_t smem = (size_t)(g + 2 * pd->max_m * kClassTile) * sizeof(double);
      int nr = 0;
      for (int q = 0; q < k->nblk; ++q) nr += k->is_complex[q] ? 0 : 1;
      void (*fn)(PatchParams, DedupParams, KronParams, const double*, double*, int) = nullptr;
      if (S == 1 && nr == 1) fn = patch_apply_class_kernel<1, 1>;
      else if (S == 2 && nr == 2) fn = patch_apply_class_kernel<2, 2>;
      else if (S == 2 && nr == 0) fn = patch_apply_class_kernel<2, 0>;
      else if (S == 3 && nr == 3) fn = patch_apply_class_kernel<3, 3>;
      else if (S == 3 && nr == 1) fn = patch_apply_class_kernel<3, 1>;
      IVK_REQUIRE(fn != nullptr, "unsupported eigen-block signature");
      cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem);
      if (e != cudaSuccess) {
        set_error("ivk_patch_apply: %s", cudaGetErrorString(e));
        return IVK_ECUDA;
      }
      int cgrid = pd->n_tiles < kClassCtas * kSMs ? pd->n_tiles : kClassCtas * kSMs;
      fn<<<cgrid, kClassWarps * 32, smem, st>>>(p, dd, kp, r, local, g);
    } else if (bmax <= 64)
      patch_apply_kron_kernel<64><<<grid, kApplyWarps * 32, 0, st>>>(p, kp, r, local);
    else if (bmax <= 256) {
      const size_t smem =
          (size_t)kApplyWarps * kron_apply_seg(S, k->nblk, bmax) * sizeof(double);
      void (*fn)(PatchParams, KronParams, const double*, double*, int) =
          patch_apply_kron_wide_kernel;
      if (smem > 48 * 1024) {
        cudaError_t e =
            cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) {
          set_error("ivk_patch_apply: %s", cudaGetErrorString(e));
          return IVK_ECUDA;
        }
      }
      fn<<<grid, kApplyWarps * 32, smem, st>>>(p, kp, r, local, bmax);
    } else {
      set_error("ivk_patch_apply: kron block size %d > 256 unsupported", bmax);
      return IVK_EUNSUPPORTED;
    }
    return check_launch("ivk_patch_apply(kron)");
  }
  if (pd->max_m <= 128)
    patch_apply_kernel<128><<<grid, kApplyWarps * 32, 0, st>>>(p, r, local);
  else if (pd->max_m <= 256)
    patch_apply_kernel<256><<<grid, kApplyWarps * 32, 0, st>>>(p, r, local);
  else if (pd->max_m <= 512)
    patch_apply_kernel<512><<<grid, kApplyWarps * 32, 0, st>>>(p, r, local);
  else {
    set_error("ivk_patch_apply: patch size %d > 512 unsupported", pd->max_m);
    return IVK_EUNSUPPORTED;
  }
  return check_launch("ivk_patch_apply");
}

static int patch_combine(const ivk_patch_desc* pd, const int32_t* dofs, int32_t n_dofs,
                         const double* local, const double* x, double alpha, double beta,
                         const double* w, double* out, double* accum, void* stream) {
  int rc = validate_patches(pd);
  if (rc) return rc;
  IVK_REQUIRE(local && out, "local/out is NULL");
  PatchParams p = make_patch_params(pd);
  const int n = dofs ? n_dofs : pd->dim;
  if (n == 0) return IVK_OK;
  int grid = (n + 255) / 256;
  if (grid > kSMs * 16) grid = kSMs * 16;
  patch_combine_kernel<<<grid, 256, 0, as_stream(stream)>>>(p, local, x, alpha, beta, w, out, accum,
                                                            dofs, n_dofs);
  return check_launch("ivk_patch_combine");
}

int ivk_patch_combine(const ivk_patch_desc* pd, const double* local, const double* x, double alpha,
                      double beta, const double* w, double* out, double* accum, void* stream) {
  return patch_combine(pd, nullptr, 0, local, x, alpha, beta, w, out, accum, stream);
}

int ivk_patch_combine_list(const ivk_patch_desc* pd, const int32_t* dofs, int32_t n_dofs,
                           const double* local, const double* x, double alpha, double beta,
                           const double* w, double* out, double* accum, void* stream) {
  IVK_REQUIRE(dofs != nullptr && n_dofs >= 0, "bad DoF list");
  return patch_combine(pd, dofs, n_dofs, local, x, alpha, beta, w, out, accum, stream);
}

int ivk_patch_factor(const ivk_operator_desc* op, const ivk_patch_desc* pd, int32_t* singular_dev,
                     void* stream) {
  int rc = validate_op(op);
  if (rc) return rc;
  rc = validate_patches(pd);
  if (rc) return rc;
  IVK_REQUIRE(pd->vertex && pd->node_off && pd->node && singular_dev,
              "patch factorisation needs vertex/node tables and a singular flag");
  if (pd->kron) {
    const ivk_kron_desc* k = pd->kron;
    int S = 0;
    for (int i = 0; i < k->nblk; ++i) S += k->is_complex[i] ? 2 : 1;
    IVK_REQUIRE(S == op->stages, "kron blocks do not cover %d stages", op->stages);
    IVK_REQUIRE(op->n_conv <= 1, "kron split needs one convection Jacobian shared by all stages");
    const int bmax = pd->max_m / S;
    IVK_REQUIRE(bmax <= 256, "kron block size %d > 256 unsupported", bmax);
    if (bmax > 64 || op->ncomp == 3) {
      IVK_REQUIRE(!k->symmetric, "large kron blocks are stored non-symmetric");
      IVK_REQUIRE(op->n_conv == 0, "large-patch factorisation supports no convection");
      FactorParams f = make_factor_params(op);
      PatchParams p = make_patch_params(pd);
      KronParams kp = make_kron(k, S);
      int grid = pd->num_patches < 2 * kSMs ? pd->num_patches : 2 * kSMs;
      if (f.ncomp == 3)
        patch_factor_kron_global_kernel<3><<<grid, kFactorGlobalThreads, 0, as_stream(stream)>>>(
            f, p, kp, singular_dev);
      else
        patch_factor_kron_global_kernel<2><<<grid, kFactorGlobalThreads, 0, as_stream(stream)>>>(
            f, p, kp, singular_dev);
      return check_launch("ivk_patch_factor(kron, global)");
    }
    const size_t smem = 2 * (size_t)bmax * kron_ldr(bmax) * sizeof(double);
    FactorParams f = make_factor_params(op);
    PatchParams p = make_patch_params(pd);
    KronParams kp = make_kron(k, S);
#define IVK_K7E_REG(RT, CT, MINB)                                                              \
  do {                                                                                         \
    cudaError_t e = cudaFuncSetAttribute(patch_factor_kron_kernel<RT, CT, MINB>,               \
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    if (e != cudaSuccess) {                                                                    \
      set_error("ivk_patch_factor: %s", cudaGetErrorString(e));                                \
      return IVK_ECUDA;                                                                        \
    }                                                                                          \
    patch_factor_kron_kernel<RT, CT, MINB>                                                     \
        <<<pd->num_patches, kKronFactorThreads, smem, as_stream(stream)>>>(f, p, kp,           \
                                                                          singular_dev);      \
  } while (0)
    if (bmax <= 32) IVK_K7E_REG(2, 2, 4);
    else if (bmax <= 48) IVK_K7E_REG(3, 3, 3);
    else IVK_K7E_REG(4, 4, 2);
#undef IVK_K7E_REG
    return check_launch("ivk_patch_factor(kron)");
  }
  const int dmax = pd->max_m;
  if (dmax > 512) {
    set_error("ivk_patch_factor: patch size %d > 512 unsupported", dmax);
    return IVK_EUNSUPPORTED;
  }
  // d x ld doubles for the register kernel (d <= 128: it leaves Inv^T with the
  // store's leading dimension in shared memory), d x d for the shared-memory one
  const size_t smem = dmax <= 128 ? (size_t)dmax * ((dmax + 3) & ~3) * sizeof(double)
                                  : (size_t)dmax * dmax * sizeof(double);
  if (op->ncomp == 3 || smem > 220 * 1024) {
    IVK_REQUIRE(op->n_conv == 0, "large-patch factorisation supports no convection");
    FactorParams f = make_factor_params(op);
    PatchParams p = make_patch_params(pd);
    int grid = pd->num_patches < 128 ? pd->num_patches : 128;  // ~L2-resident working set
    if (f.ncomp == 3)
      patch_factor_global_kernel<3><<<grid, kFactorGlobalThreads, 0, as_stream(stream)>>>(
          f, p, singular_dev);
    else
      patch_factor_global_kernel<2><<<grid, kFactorGlobalThreads, 0, as_stream(stream)>>>(
          f, p, singular_dev);
    return check_launch("ivk_patch_factor(global)");
  }
  FactorParams f = make_factor_params(op);
  PatchParams p = make_patch_params(pd);
  // register-resident elimination for d <= 128 (ivk_gj.cuh); the tile shape
  // follows the level's largest patch, smaller (boundary) patches are padded
  if (dmax <= 128 && !getenv("IVK_K7_SMEM")) {
#define IVK_K7_REG(...) IVK_K7_REG_(__VA_ARGS__)
#define IVK_K7_REG_(TX, RT, CT, MINB)                                                           \
  do {                                                                                          \
    cudaError_t e = cudaFuncSetAttribute(patch_factor_reg_kernel<TX, RT, CT, MINB>,             \
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    if (e != cudaSuccess) {                                                                     \
      set_error("ivk_patch_factor: %s", cudaGetErrorString(e));                                 \
      return IVK_ECUDA;                                                                         \
    }                                                                                           \
    patch_factor_reg_kernel<TX, RT, CT, MINB>                                                   \
        <<<pd->num_patches, 16 * TX, smem, as_stream(stream)>>>(f, p, singular_dev);            \
  } while (0)
    if (dmax <= 48) IVK_K7_REG(16, 3, 3, 4);
    else if (dmax <= 64) IVK_K7_REG(16, 4, 4, 4);
#ifndef IVK_K7_TX  // the d <= 80 tile (2-D Taylor-Hood, s = 2): A/B knobs
#define IVK_K7_TX 16
#define IVK_K7_CT 5
#define IVK_K7_MINB 3
#endif
    else if (dmax <= 80) IVK_K7_REG(IVK_K7_TX, 5, IVK_K7_CT, IVK_K7_MINB);
    else if (dmax <= 96) IVK_K7_REG(16, 6, 6, 2);
    else IVK_K7_REG(32, 8, 4, 1);
#undef IVK_K7_REG
#undef IVK_K7_REG_
    return check_launch("ivk_patch_factor(registers)");
  }
  cudaError_t e = cudaFuncSetAttribute(patch_factor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) {
    set_error("ivk_patch_factor: %s", cudaGetErrorString(e));
    return IVK_ECUDA;
  }
  patch_factor_kernel<<<pd->num_patches, kFactorThreads, smem, as_stream(stream)>>>(f, p,
                                                                                    singular_dev);
  return check_launch("ivk_patch_factor");
}

int ivk_patch_gather_blocks(const ivk_operator_desc* op, const ivk_patch_desc* pd, int32_t kmax,
                            double* Ms, double* Ks, double* C, void* stream) {
  int rc = validate_op(op);
  if (rc) return rc;
  rc = validate_patches(pd);
  if (rc) return rc;
  IVK_REQUIRE(pd->vertex && pd->node_off && pd->node && Ms && Ks && C && kmax >= 1,
              "gather needs vertex/node tables and output buffers");
  IVK_REQUIRE(op->n_conv == 0, "the modal split needs a convection-free (symmetric) operator");
  FactorParams f = make_factor_params(op);
  PatchParams p = make_patch_params(pd);
  if (f.ncomp == 3)
    patch_gather_blocks_kernel<3><<<pd->num_patches, 128, 0, as_stream(stream)>>>(f, p, kmax, Ms, Ks, C);
  else
    patch_gather_blocks_kernel<2><<<pd->num_patches, 128, 0, as_stream(stream)>>>(f, p, kmax, Ms, Ks, C);
  return check_launch("ivk_patch_gather_blocks");
}

int ivk_modal_factor(const ivk_patch_desc* pd, int32_t kmax, const double* Ms, const double* Ks,
                     const double* C, int32_t* singular_dev, void* stream) {
  int rc = validate_patches(pd);
  if (rc) return rc;
  IVK_REQUIRE(pd->modal && pd->vertex && pd->node_off && Ms && Ks && C && singular_dev,
              "modal factorisation needs a modal store, vertex/node tables and the gathered blocks");
  IVK_REQUIRE(kmax >= 1 && kmax <= 32, "modal factorisation: %d nodes per patch > 32 unsupported",
              kmax);
  const ivk_modal_desc* m = pd->modal;
  IVK_REQUIRE(m->stages >= 1 && m->stages <= IVK_MAX_STAGES && (m->ncomp == 2 || m->ncomp == 3),
              "bad modal descriptor");
  ModalParams mp;
  mp.S = m->stages;
  mp.NC = m->ncomp;
  mp.dt = m->dt;
  for (int i = 0; i < IVK_MAX_STAGES * IVK_MAX_STAGES; ++i) mp.a[i] = m->butcher_a[i];
  PatchParams p = make_patch_params(pd);
  const size_t smem = (size_t)kModalSetupWarps * 3 * kmax * (kmax | 1) * sizeof(double);
  const int grid = (pd->num_patches + kModalSetupWarps - 1) / kModalSetupWarps;
#define IVK_K7M(SS, CC)                                                                          \
  do {                                                                                           \
    cudaError_t e = cudaFuncSetAttribute(modal_factor_kernel<SS, CC>,                            \
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    if (e != cudaSuccess) {                                                                      \
      set_error("ivk_modal_factor: %s", cudaGetErrorString(e));                                  \
      return IVK_ECUDA;                                                                          \
    }                                                                                            \
    modal_factor_kernel<SS, CC><<<grid, kModalSetupWarps * 32, smem, as_stream(stream)>>>(       \
        p, mp, kmax, Ms, Ks, C, singular_dev);                                                   \
  } while (0)
  switch (mp.S * 10 + mp.NC) {
    case 12: IVK_K7M(1, 2); break;
    case 22: IVK_K7M(2, 2); break;
    case 32: IVK_K7M(3, 2); break;
    case 13: IVK_K7M(1, 3); break;
    case 23: IVK_K7M(2, 3); break;
    case 33: IVK_K7M(3, 3); break;
  }
#undef IVK_K7M
  return check_launch("ivk_modal_factor");
}

int ivk_peer_combine_update(int32_t n, const int32_t* dofs, const int32_t* holder_ptr,
                            const int32_t* holder_rank, const ivk_peer_view* peers_dev,
                            double omega, const double* w, double* x, void* stream) {
  IVK_REQUIRE(n >= 0 && dofs && holder_ptr && holder_rank && peers_dev && x,
              "bad peer combine arguments");
  if (n == 0) return IVK_OK;
  int grid = (n + 255) / 256;
  if (grid > kSMs * 16) grid = kSMs * 16;
  peer_combine_update_kernel<<<grid, 256, 0, as_stream(stream)>>>(n, dofs, holder_ptr, holder_rank,
                                                                  peers_dev, omega, w, x);
  return check_launch("ivk_peer_combine_update");
}

int ivk_general_patch_factor(const ivk_general_desc* op, const ivk_patch_desc* pd,
                             int32_t* singular_dev, void* stream) {
  int rc = validate_general(op);
  if (rc) return rc;
  rc = validate_patches(pd);
  if (rc) return rc;
  IVK_REQUIRE(pd->vertex && singular_dev, "patch factorisation needs vertex ids and a singular flag");
  const int S = op->stages;
  IVK_REQUIRE(pd->max_m <= kGenMaxD, "patch size %d > %d unsupported", pd->max_m, kGenMaxD);
  GenFactorParams g;
  g.S = S;
  g.dt = op->dt;
  for (int i = 0; i < IVK_MAX_STAGES * IVK_MAX_STAGES; ++i) g.a[i] = op->butcher_a[i];
  g.rowptr = op->rowptr;
  g.col = op->col;
  g.ml = reinterpret_cast<const double2*>(op->ml);
  KronParams kp{};
  size_t smem;
  const int use_kron = pd->kron != nullptr;
  if (use_kron) {
    const ivk_kron_desc* k = pd->kron;
    IVK_REQUIRE(!k->symmetric, "the general path stores non-symmetric eigen-blocks");
    int SS = 0;
    for (int i = 0; i < k->nblk; ++i) SS += k->is_complex[i] ? 2 : 1;
    IVK_REQUIRE(SS == S, "kron blocks do not cover %d stages", S);
    kp = make_kron(k, S);
    const int bmax = pd->max_m / S;
    smem = 2 * (size_t)bmax * kron_ldr(bmax) * sizeof(double);
  } else {
    smem = (size_t)pd->max_m * ((pd->max_m + 3) & ~3) * sizeof(double);
  }
  if (smem > 200 * 1024) {
    set_error("ivk_general_patch_factor: patch (m = %d) exceeds shared memory", pd->max_m);
    return IVK_EUNSUPPORTED;
  }
  PatchParams p = make_patch_params(pd);
  // largest matrix of the launch: an eigen-block (kron) or the whole patch
  const int dmat = use_kron ? pd->max_m / S : pd->max_m;
#define IVK_K7G(RT, CT)                                                                        \
  do {                                                                                         \
    cudaError_t e = cudaFuncSetAttribute(general_factor_kernel<RT, CT>,                        \
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    if (e != cudaSuccess) {                                                                    \
      set_error("ivk_general_patch_factor: %s", cudaGetErrorString(e));                        \
      return IVK_ECUDA;                                                                        \
    }                                                                                          \
    general_factor_kernel<RT, CT>                                                              \
        <<<pd->num_patches, kGenFactorThreads, smem, as_stream(stream)>>>(g, p, kp, use_kron,  \
                                                                         singular_dev);       \
  } while (0)
  if (getenv("IVK_K7_SMEM") || dmat > 96) IVK_K7G(0, 0);
  else if (dmat <= 48) IVK_K7G(3, 3);
  else if (dmat <= 80) IVK_K7G(5, 5);
  else IVK_K7G(6, 6);
#undef IVK_K7G
  return check_launch("ivk_general_patch_factor");
}

int ivk_general_vanka_sweep(const ivk_general_desc* op, const ivk_patch_desc* pd, const double* x,
                            const double* b, double omega, const double* w, double* r,
                            double* local, double* x_out, void* stream) {
  IVK_REQUIRE(x && b && r && local && x_out, "sweep vector is NULL");
  int rc = ivk_general_apply(op, x, b, r, stream);
  if (rc) return rc;
  rc = ivk_patch_apply(pd, r, local, stream);
  if (rc) return rc;
  return ivk_patch_combine(pd, local, x, 1.0, omega, w, x_out, nullptr, stream);
}

int ivk_vanka_sweep(const ivk_operator_desc* op, const ivk_patch_desc* pd, const double* x,
                    const double* b, double omega, const double* w, double* r, double* local,
                    double* x_out, void* stream) {
  IVK_REQUIRE(x && b && r && local && x_out, "sweep vector is NULL");
  int rc = ivk_stage_apply(op, x, b, r, stream);
  if (rc) return rc;
  rc = ivk_patch_apply(pd, r, local, stream);
  if (rc) return rc;
  return ivk_patch_combine(pd, local, x, 1.0, omega, w, x_out, nullptr, stream);
}

}  // extern "C"
