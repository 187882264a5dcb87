// K6: coarsest-level direct solve with FIXED LU factors of A + Z Z^T
// (CoarseSolver, solvers.py:271-292).  The factors are the SuperLU factors the
// host computes once at setup (scipy splu, as the reference does); the
// per-cycle solve -- pressure projection, permuted forward/backward
// substitution, projection -- runs in one CTA on the device.  Re-using the
// same factors (rather than a fresh GPU LU) keeps the ill-conditioned coarse
// solve within the reference's own roundoff floor.
//
// Tile-sparse blocked substitution: the factors are stored as 32 x 32 tiles
// (column-major), only the ~1/3 nonzero ones.  Per block column K one warp
// solves the diagonal tile -- L's (unit, well-conditioned) diagonal tiles are
// stored inverted and applied as a GEMV, U's by a register-shuffle
// substitution with stored reciprocal diagonal -- its tiles streamed two
// steps ahead into a shared-memory ring by TMA bulk copies (cp.async.bulk +
// mbarrier); the other 15 warps hold the (already prefetched) off-diagonal
// tiles of column K in registers and apply the rank-32 update as soon as y_K
// is published, then prefetch their tile of column K+1.  Tile metadata is
// staged in shared memory, so no global load sits on the critical path
// (2 CTA barriers per block column).

#include "ivk_common.cuh"

namespace ivk {

constexpr int kCoarseThreads = 512;
constexpr int kTileWarps = 15;   // warps 0..14 apply off-diagonal tiles
constexpr int kDiagWarp = 15;    // warp 15 solves the diagonal tiles

struct CoarseParams {
  int n, nb, S, n_u, n_p;
  const int32_t* __restrict__ l_colptr;
  const int32_t* __restrict__ l_row;
  const double* __restrict__ l_tiles;
  const double* __restrict__ l_diag;
  const int32_t* __restrict__ u_colptr;
  const int32_t* __restrict__ u_row;
  const double* __restrict__ u_tiles;
  const double* __restrict__ u_diag;
  const int32_t* __restrict__ perm_r;
  const int32_t* __restrict__ perm_c;
};

__device__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    double w = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) w += __shfl_down_sync(0xffffffffu, w, o);
    if (lane == 0) red[0] = w;
  }
  __syncthreads();
  const double s = red[0];
  __syncthreads();
  return s;
}

// In-place removal of the per-stage constant-pressure component of v (smem).
__device__ void project_smem(double* v, int S, int n_u, int n_p, double* red) {
  const int sd = n_u + n_p;
  for (int t = 0; t < S; ++t) {
    double acc = 0.0;
    for (int i = threadIdx.x; i < n_p; i += blockDim.x) acc += v[t * sd + n_u + i];
    const double mean = block_sum(acc, red) / (double)n_p;
    for (int i = threadIdx.x; i < n_p; i += blockDim.x) v[t * sd + n_u + i] -= mean;
    __syncthreads();
  }
}

__device__ __forceinline__ void load_tile(double (&t)[32], const double* __restrict__ tile,
                                          int lane) {
#pragma unroll
  for (int jj = 0; jj < 32; ++jj) t[jj] = __ldg(tile + jj * 32 + lane);
}

constexpr int kDiagRing = 3;  // diagonal tiles in flight (TMA), 2 steps ahead

// One triangular solve.  colptr / rowtile live in shared memory; the diagonal
// tiles stream through a 3-slot TMA ring; each tile warp keeps its next
// off-diagonal tile in registers.
template <bool LOWER>
__device__ void tile_solve(int nb, const int32_t* colptr, const int32_t* rowtile,
                           const double* __restrict__ tiles, const double* __restrict__ diag,
                           double* y, double* ring, uint64_t* bars, uint32_t& phase_bits) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int step = LOWER ? 1 : -1;
  const int K0 = LOWER ? 0 : nb - 1;
  double t[32];
  if (warp == kDiagWarp && lane == 0) {
    for (int s = 0; s < kDiagRing - 1 && s < nb; ++s)
      bulk_load(ring + s * 1024, diag + (long)(K0 + s * step) * 1024, 8192, &bars[s]);
  }
  if (warp < kTileWarps) {
    const int ti = colptr[K0] + warp;
    if (ti < colptr[K0 + 1]) load_tile(t, tiles + (long)ti * 1024, lane);
  }
  int K = K0;
  for (int s = 0; s < nb; ++s, K += step) {
    if (warp == kDiagWarp) {
      const int slot = s % kDiagRing;
      if (lane == 0 && s + kDiagRing - 1 < nb) {
        const int ns = (s + kDiagRing - 1) % kDiagRing;
        bulk_load(ring + ns * 1024, diag + (long)(K + (kDiagRing - 1) * step) * 1024, 8192,
                  &bars[ns]);
      }
      mbar_wait(&bars[slot], (phase_bits >> slot) & 1u);
      const double* D = ring + slot * 1024;
      double yl = y[K * 32 + lane];
      if (LOWER) {
        // the lower diagonal tiles are stored inverted (tile_factor): a
        // 32 x 32 GEMV instead of a 32-step shuffle chain
        const double* yk = y + K * 32;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
        for (int jj = 0; jj < 32; jj += 4) {
          a0 = fma(D[jj * 32 + lane], yk[jj], a0);
          a1 = fma(D[(jj + 1) * 32 + lane], yk[jj + 1], a1);
          a2 = fma(D[(jj + 2) * 32 + lane], yk[jj + 2], a2);
          a3 = fma(D[(jj + 3) * 32 + lane], yk[jj + 3], a3);
        }
        __syncwarp();
        yl = (a0 + a1) + (a2 + a3);
      } else {
        // the diagonal slot of an upper tile holds 1 / U_jj (tile_factor)
#pragma unroll
        for (int jj = 31; jj >= 0; --jj) {
          const double d = D[jj * 32 + lane];
          if (lane == jj) yl = yl * d;
          const double yj = __shfl_sync(0xffffffffu, yl, jj);
          if (lane < jj) yl = fma(-d, yj, yl);
        }
      }
      y[K * 32 + lane] = yl;
    }
    // every thread flips its copy of the slot parity (uniform bookkeeping)
    phase_bits ^= 1u << (s % kDiagRing);
    __syncthreads();
    if (warp < kTileWarps) {
      const int c0 = colptr[K], c1 = colptr[K + 1];
      const double* yk = y + K * 32;
      int ti = c0 + warp;
      if (ti < c1) {
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
        for (int jj = 0; jj < 32; jj += 4) {
          a0 = fma(t[jj], yk[jj], a0);
          a1 = fma(t[jj + 1], yk[jj + 1], a1);
          a2 = fma(t[jj + 2], yk[jj + 2], a2);
          a3 = fma(t[jj + 3], yk[jj + 3], a3);
        }
        y[rowtile[ti] * 32 + lane] -= (a0 + a1) + (a2 + a3);
      }
      for (ti += kTileWarps; ti < c1; ti += kTileWarps) {
        double u[32];
        load_tile(u, tiles + (long)ti * 1024, lane);
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
        for (int jj = 0; jj < 32; jj += 4) {
          a0 = fma(u[jj], yk[jj], a0);
          a1 = fma(u[jj + 1], yk[jj + 1], a1);
          a2 = fma(u[jj + 2], yk[jj + 2], a2);
          a3 = fma(u[jj + 3], yk[jj + 3], a3);
        }
        y[rowtile[ti] * 32 + lane] -= (a0 + a1) + (a2 + a3);
      }
      if (s + 1 < nb) {
        const int Kn = K + step;
        const int tn = colptr[Kn] + warp;
        if (tn < colptr[Kn + 1]) load_tile(t, tiles + (long)tn * 1024, lane);
      }
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kCoarseThreads, 1) coarse_solve_kernel(CoarseParams c,
                                                                         const double* __restrict__ b,
                                                                         double* __restrict__ x) {
  extern __shared__ __align__(128) double sm[];
  const int npad = c.nb * 32;
  const int nl = c.l_colptr[c.nb], nu_t = c.u_colptr[c.nb];
  double* ring = sm;                       // kDiagRing tiles (TMA destination)
  double* v = ring + kDiagRing * 1024;     // npad
  double* y = v + npad;                    // npad
  int32_t* meta = reinterpret_cast<int32_t*>(y + npad);
  int32_t* lcol = meta;                    // nb + 1
  int32_t* lrow = lcol + c.nb + 1;         // nl
  int32_t* ucol = lrow + nl;               // nb + 1
  int32_t* urow = ucol + c.nb + 1;         // nu_t
  __shared__ double red[32];
  __shared__ __align__(8) uint64_t bars[kDiagRing];
  if (threadIdx.x == 0) {
    for (int i = 0; i < kDiagRing; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i <= c.nb; i += blockDim.x) {
    lcol[i] = c.l_colptr[i];
    ucol[i] = c.u_colptr[i];
  }
  for (int i = threadIdx.x; i < nl; i += blockDim.x) lrow[i] = c.l_row[i];
  for (int i = threadIdx.x; i < nu_t; i += blockDim.x) urow[i] = c.u_row[i];
  for (int i = threadIdx.x; i < npad; i += blockDim.x) {
    v[i] = i < c.n ? b[i] : 0.0;
    y[i] = 0.0;
  }
  __syncthreads();
  project_smem(v, c.S, c.n_u, c.n_p, red);
  for (int i = threadIdx.x; i < c.n; i += blockDim.x) y[c.perm_r[i]] = v[i];
  __syncthreads();
  uint32_t phase_bits = 0;
  tile_solve<true>(c.nb, lcol, lrow, c.l_tiles, c.l_diag, y, ring, bars, phase_bits);
  tile_solve<false>(c.nb, ucol, urow, c.u_tiles, c.u_diag, y, ring, bars, phase_bits);
  for (int i = threadIdx.x; i < c.n; i += blockDim.x) v[i] = y[c.perm_c[i]];
  __syncthreads();
  project_smem(v, c.S, c.n_u, c.n_p, red);
  for (int i = threadIdx.x; i < c.n; i += blockDim.x) x[i] = v[i];
}

// Dense coarse operator: warp per row, 256-bit loads along the row, x from
// L1; fixed-order shuffle reduction (deterministic).
constexpr int kGemvWarps = 8;

__global__ void __launch_bounds__(kGemvWarps * 32) dense_gemv_kernel(int n, int ld,
                                                                     const double* __restrict__ A,
                                                                     const double* __restrict__ x,
                                                                     double* __restrict__ y) {
  const int row = blockIdx.x * kGemvWarps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  const double* a = A + (long)row * ld;
  double acc = 0.0;
  // 4 x 32 B of the row in flight per lane (few rows: latency, not bandwidth)
  constexpr int U = 4;
  for (int j0 = 4 * lane; j0 < n; j0 += 128 * U) {
    double4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = j0 + 128 * u;
      v[u] = j < n ? *reinterpret_cast<const double4*>(a + j) : make_double4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = j0 + 128 * u;
      if (j < n) acc = fma(v[u].x, __ldg(x + j), acc);
      if (j + 1 < n) acc = fma(v[u].y, __ldg(x + j + 1), acc);
      if (j + 2 < n) acc = fma(v[u].z, __ldg(x + j + 2), acc);
      if (j + 3 < n) acc = fma(v[u].w, __ldg(x + j + 3), acc);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) y[row] = acc;
}

}  // namespace ivk

using namespace ivk;

extern "C" {

int ivk_coarse_solve(const ivk_coarse_desc* c, const double* b, double* x, void* stream) {
  IVK_REQUIRE(c != nullptr, "bad coarse descriptor");
  if (c->dense) {
    IVK_REQUIRE(b && x && b != x, "bad coarse vectors");
    IVK_REQUIRE(c->n > 0 && c->dense_ld >= c->n && (c->dense_ld & 3) == 0,
                "bad dense coarse operator (n=%d ld=%d)", c->n, c->dense_ld);
    const int grid = (c->n + kGemvWarps - 1) / kGemvWarps;
    dense_gemv_kernel<<<grid, kGemvWarps * 32, 0, as_stream(stream)>>>(c->n, c->dense_ld, c->dense,
                                                                       b, x);
    return check_launch("ivk_coarse_solve(dense)");
  }
  IVK_REQUIRE(c->l_colptr && c->l_row && c->l_tiles && c->l_diag && c->u_colptr &&
                  c->u_row && c->u_tiles && c->u_diag && c->perm_r && c->perm_c,
              "bad coarse descriptor");
  IVK_REQUIRE(b && x && b != x, "bad coarse vectors");
  IVK_REQUIRE(c->n == c->stages * (c->n_u + c->n_p) && c->n > 0, "coarse dimension mismatch");
  IVK_REQUIRE(c->nb * 32 >= c->n && (c->nb - 1) * 32 < c->n, "coarse block count mismatch");
  IVK_REQUIRE(c->l_ntiles >= 0 && c->u_ntiles >= 0, "bad tile counts");
  const size_t smem = (size_t)kDiagRing * 8192 + 2 * (size_t)c->nb * 32 * sizeof(double) +
                      (size_t)(2 * (c->nb + 1) + c->l_ntiles + c->u_ntiles) * sizeof(int32_t);
  if (smem > 200 * 1024) {
    set_error("ivk_coarse_solve: coarse dimension %d too large for one CTA", c->n);
    return IVK_EUNSUPPORTED;
  }
  {  // set on every call: the attribute is per device
    cudaError_t e = cudaFuncSetAttribute(coarse_solve_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) {
      set_error("ivk_coarse_solve: %s", cudaGetErrorString(e));
      return IVK_ECUDA;
    }
  }
  CoarseParams p;
  p.n = c->n;
  p.nb = c->nb;
  p.S = c->stages;
  p.n_u = c->n_u;
  p.n_p = c->n_p;
  p.l_colptr = c->l_colptr;
  p.l_row = c->l_row;
  p.l_tiles = c->l_tiles;
  p.l_diag = c->l_diag;
  p.u_colptr = c->u_colptr;
  p.u_row = c->u_row;
  p.u_tiles = c->u_tiles;
  p.u_diag = c->u_diag;
  p.perm_r = c->perm_r;
  p.perm_c = c->perm_c;
  coarse_solve_kernel<<<1, kCoarseThreads, smem, as_stream(stream)>>>(p, b, x);
  return check_launch("ivk_coarse_solve");
}

}  // extern "C"
