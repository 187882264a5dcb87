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
// solves the diagonal tile with register shuffles while the other 15 warps
// hold the (already prefetched) off-diagonal tiles of column K in registers
// and apply the rank-32 update as soon as y_K is published; each warp then
// prefetches its tile of column K+1, so the L2 latency is off the critical
// path (2 CTA barriers per block column).

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

template <bool LOWER>
__device__ void tile_solve(int nb, const int32_t* __restrict__ colptr,
                           const int32_t* __restrict__ rowtile, const double* __restrict__ tiles,
                           const double* __restrict__ diag, double* y) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int step = LOWER ? 1 : -1;
  int K = LOWER ? 0 : nb - 1;
  double t[32];
  if (warp == kDiagWarp) {
    load_tile(t, diag + (long)K * 1024, lane);
  } else {
    const int ti = colptr[K] + warp;
    if (ti < colptr[K + 1]) load_tile(t, tiles + (long)ti * 1024, lane);
  }
  for (int s = 0; s < nb; ++s, K += step) {
    if (warp == kDiagWarp) {
      double yl = y[K * 32 + lane];
      if (LOWER) {
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) {
          const double yj = __shfl_sync(0xffffffffu, yl, jj);
          if (lane > jj) yl = fma(-t[jj], yj, yl);
        }
      } else {
#pragma unroll
        for (int jj = 31; jj >= 0; --jj) {
          if (lane == jj) yl = yl / t[jj];
          const double yj = __shfl_sync(0xffffffffu, yl, jj);
          if (lane < jj) yl = fma(-t[jj], yj, yl);
        }
      }
      y[K * 32 + lane] = yl;
      if (s + 1 < nb) load_tile(t, diag + (long)(K + step) * 1024, lane);
    }
    __syncthreads();
    if (warp < kTileWarps) {
      const int c0 = colptr[K], c1 = colptr[K + 1];
      const double* yk = y + K * 32;
      int ti = c0 + warp;
      if (ti < c1) {
        double acc = 0.0;
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) acc = fma(t[jj], yk[jj], acc);
        y[rowtile[ti] * 32 + lane] -= acc;
      }
      for (ti += kTileWarps; ti < c1; ti += kTileWarps) {
        const double* tile = tiles + (long)ti * 1024;
        double acc = 0.0;
#pragma unroll 8
        for (int jj = 0; jj < 32; ++jj) acc = fma(__ldg(tile + jj * 32 + lane), yk[jj], acc);
        y[rowtile[ti] * 32 + lane] -= acc;
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
  extern __shared__ double sm[];
  const int npad = c.nb * 32;
  double* v = sm;         // npad
  double* y = sm + npad;  // npad
  __shared__ double red[32];
  for (int i = threadIdx.x; i < npad; i += blockDim.x) {
    v[i] = i < c.n ? b[i] : 0.0;
    y[i] = 0.0;
  }
  __syncthreads();
  project_smem(v, c.S, c.n_u, c.n_p, red);
  for (int i = threadIdx.x; i < c.n; i += blockDim.x) y[c.perm_r[i]] = v[i];
  __syncthreads();
  tile_solve<true>(c.nb, c.l_colptr, c.l_row, c.l_tiles, c.l_diag, y);
  tile_solve<false>(c.nb, c.u_colptr, c.u_row, c.u_tiles, c.u_diag, y);
  for (int i = threadIdx.x; i < c.n; i += blockDim.x) v[i] = y[c.perm_c[i]];
  __syncthreads();
  project_smem(v, c.S, c.n_u, c.n_p, red);
  for (int i = threadIdx.x; i < c.n; i += blockDim.x) x[i] = v[i];
}

}  // namespace ivk

using namespace ivk;

extern "C" {

int ivk_coarse_solve(const ivk_coarse_desc* c, const double* b, double* x, void* stream) {
  IVK_REQUIRE(c && c->l_colptr && c->l_row && c->l_tiles && c->l_diag && c->u_colptr &&
                  c->u_row && c->u_tiles && c->u_diag && c->perm_r && c->perm_c,
              "bad coarse descriptor");
  IVK_REQUIRE(b && x && b != x, "bad coarse vectors");
  IVK_REQUIRE(c->n == c->stages * (c->n_u + c->n_p) && c->n > 0, "coarse dimension mismatch");
  IVK_REQUIRE(c->nb * 32 >= c->n && (c->nb - 1) * 32 < c->n, "coarse block count mismatch");
  const size_t smem = 2 * (size_t)c->nb * 32 * sizeof(double);
  if (smem > 200 * 1024) {
    set_error("ivk_coarse_solve: coarse dimension %d too large for one CTA", c->n);
    return IVK_EUNSUPPORTED;
  }
  static size_t configured = 0;
  if (smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(coarse_solve_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) {
      set_error("ivk_coarse_solve: %s", cudaGetErrorString(e));
      return IVK_ECUDA;
    }
    configured = smem;
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
