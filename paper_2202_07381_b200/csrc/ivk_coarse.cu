// K6: coarsest-level direct solve with FIXED LU factors of A + Z Z^T
// (CoarseSolver, solvers.py:271-292).  The factors are the SuperLU factors the
// host computes once at setup (scipy splu, exactly as the reference does);
// the per-cycle solve -- pressure projection, permuted dense forward/backward
// substitution, projection -- runs in one CTA on the device.  Re-using the
// same factors (rather than a fresh GPU LU) is what keeps the ill-conditioned
// coarse solve within the reference's own roundoff floor.
//
// Blocked substitution: 32-column diagonal blocks are solved by one warp with
// register shuffles; the trailing rows are updated warp-per-row with
// coalesced 256 B reads of the factor row segment.

#include "ivk_common.cuh"

namespace ivk {

constexpr int kCoarseThreads = 1024;
constexpr int kWarps = kCoarseThreads / 32;

__device__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    double w = lane < kWarps ? red[lane] : 0.0;
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

__global__ void __launch_bounds__(kCoarseThreads) coarse_solve_kernel(
    int n, int S, int n_u, int n_p, const double* __restrict__ L, const double* __restrict__ U,
    const int32_t* __restrict__ perm_r, const int32_t* __restrict__ perm_c,
    const double* __restrict__ b, double* __restrict__ x) {
  extern __shared__ double sm[];
  double* v = sm;       // n
  double* y = sm + n;   // n
  __shared__ double red[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

  for (int i = threadIdx.x; i < n; i += blockDim.x) v[i] = b[i];
  __syncthreads();
  project_smem(v, S, n_u, n_p, red);
  for (int i = threadIdx.x; i < n; i += blockDim.x) y[perm_r[i]] = v[i];
  __syncthreads();

  // Forward: L y = P_r c, L unit lower triangular.
  for (int k0 = 0; k0 < n; k0 += 32) {
    const int kb = min(32, n - k0);
    if (warp == 0) {
      double yl = lane < kb ? y[k0 + lane] : 0.0;
      double lrow[32];
#pragma unroll
      for (int jj = 0; jj < 32; ++jj)
        lrow[jj] = (lane < kb && jj < lane) ? L[(long)(k0 + lane) * n + k0 + jj] : 0.0;
#pragma unroll
      for (int jj = 0; jj < 32; ++jj) {
        const double yj = __shfl_sync(0xffffffffu, yl, jj);
        yl = fma(-lrow[jj], yj, yl);
      }
      if (lane < kb) y[k0 + lane] = yl;
    }
    __syncthreads();
    const double yk = lane < kb ? y[k0 + lane] : 0.0;
    for (int i = k0 + kb + warp; i < n; i += kWarps) {
      double t = lane < kb ? L[(long)i * n + k0 + lane] * yk : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
      if (lane == 0) y[i] -= t;
    }
    __syncthreads();
  }
  // Backward: U w = y.
  for (int k1 = n; k1 > 0; k1 -= 32) {
    const int k0 = max(0, k1 - 32), kb = k1 - k0;
    if (warp == 0) {
      double yl = lane < kb ? y[k0 + lane] : 0.0;
      const double dl = lane < kb ? U[(long)(k0 + lane) * n + k0 + lane] : 1.0;
      double urow[32];
#pragma unroll
      for (int jj = 0; jj < 32; ++jj)
        urow[jj] = (lane < kb && jj > lane && jj < kb) ? U[(long)(k0 + lane) * n + k0 + jj] : 0.0;
#pragma unroll
      for (int jj = 31; jj >= 0; --jj) {
        if (jj < kb) {
          if (lane == jj) yl = yl / dl;
          const double yj = __shfl_sync(0xffffffffu, yl, jj);
          if (lane < jj) yl = fma(-urow[jj], yj, yl);
        }
      }
      if (lane < kb) y[k0 + lane] = yl;
    }
    __syncthreads();
    const double yk = lane < kb ? y[k0 + lane] : 0.0;
    for (int i = warp; i < k0; i += kWarps) {
      double t = lane < kb ? U[(long)i * n + k0 + lane] * yk : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
      if (lane == 0) y[i] -= t;
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) v[i] = y[perm_c[i]];
  __syncthreads();
  project_smem(v, S, n_u, n_p, red);
  for (int i = threadIdx.x; i < n; i += blockDim.x) x[i] = v[i];
}

}  // namespace ivk

using namespace ivk;

extern "C" {

int ivk_coarse_solve(const ivk_coarse_desc* c, const double* b, double* x, void* stream) {
  IVK_REQUIRE(c && c->lower && c->upper && c->perm_r && c->perm_c, "bad coarse descriptor");
  IVK_REQUIRE(b && x && b != x, "bad coarse vectors");
  IVK_REQUIRE(c->n == c->stages * (c->n_u + c->n_p) && c->n > 0, "coarse dimension mismatch");
  const size_t smem = 2 * (size_t)c->n * sizeof(double);
  if (smem > 220 * 1024) {
    set_error("ivk_coarse_solve: coarse dimension %d too large for one CTA", c->n);
    return IVK_EUNSUPPORTED;
  }
  cudaError_t e = cudaFuncSetAttribute(coarse_solve_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) {
    set_error("ivk_coarse_solve: %s", cudaGetErrorString(e));
    return IVK_ECUDA;
  }
  coarse_solve_kernel<<<1, kCoarseThreads, smem, as_stream(stream)>>>(
      c->n, c->stages, c->n_u, c->n_p, c->lower, c->upper, c->perm_r, c->perm_c, b, x);
  return check_launch("ivk_coarse_solve");
}

}  // extern "C"
