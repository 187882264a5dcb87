// K9: the Krylov vector work of FGMRES (solvers.py:364-443) on the device --
// modified Gram-Schmidt with deterministic reductions.
//
// MGS keeps the reference's order exactly: h_i = <w, V_i>, w -= h_i V_i for
// i = 0..k-1, then h_k = ||w||, V_k = w / h_k.  The axpy of term i-1 and the
// dot of term i touch the same w, so they are fused into one pass (k + 2
// passes over w instead of 2k + 2).  Every reduction is a fixed grid of block
// partials summed in block order by the last block to finish: bitwise
// reproducible, no host round trip (the coefficients stay in device memory
// and each pass reads its predecessor's from there).

#include "ivk_common.cuh"

namespace ivk {

constexpr int kRedThreads = 512;
constexpr int kRedBlocks = 2 * kSMs;

struct RedScratch {
  double* partial = nullptr;
  unsigned int* counter = nullptr;
};

static RedScratch g_red[64];  // one per device ordinal

static int scratch(RedScratch** out) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
    set_error("ivk krylov: no current device");
    return IVK_ECUDA;
  }
  RedScratch& s = g_red[dev];
  if (!s.partial) {
    if (cudaMalloc(&s.partial, kRedBlocks * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&s.counter, sizeof(unsigned int)) != cudaSuccess ||
        cudaMemset(s.counter, 0, sizeof(unsigned int)) != cudaSuccess) {
      set_error("ivk krylov: scratch allocation failed");
      return IVK_ECUDA;
    }
  }
  *out = &s;
  return IVK_OK;
}

// Block-level sum, then the last block to finish reduces the partials in
// index order and writes (optionally sqrt of) the total to *result.
__device__ void finish_reduction(double v, double* partial, unsigned int* counter, double* result,
                                 bool take_sqrt) {
  __shared__ double red[kRedThreads / 32];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kRedThreads / 32; ++w) s += red[w];
    partial[blockIdx.x] = s;
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    double s = 0.0;
    for (int b = 0; b < (int)gridDim.x; ++b) s += ((volatile double*)partial)[b];
    *result = take_sqrt ? sqrt(s) : s;
    *counter = 0u;
  }
}

// w -= coef[ia] * a (if a != NULL); then result = <w, b> (b == NULL: <w, w>,
// and the sqrt is taken).  One pass over w.
__global__ void __launch_bounds__(kRedThreads) axpy_dot_kernel(long n, const double* __restrict__ a,
                                                               const double* coef, int ia,
                                                               double* __restrict__ w,
                                                               const double* __restrict__ b,
                                                               double* partial,
                                                               unsigned int* counter,
                                                               double* result) {
  const double h = a ? coef[ia] : 0.0;
  double acc = 0.0;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n;
       i += (long)gridDim.x * blockDim.x) {
    double wi = w[i];
    if (a) {
      wi = fma(-h, a[i], wi);
      w[i] = wi;
    }
    acc = fma(wi, b ? b[i] : wi, acc);
  }
  finish_reduction(acc, partial, counter, result, b == nullptr);
}

// out = w / coef[k] when coef[k] > 1e-300 (solvers.py:407-408), else left.
__global__ void scale_kernel(long n, const double* __restrict__ w, const double* coef, int k,
                             double* __restrict__ out) {
  const double h = coef[k];
  if (!(h > 1e-300)) return;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n;
       i += (long)gridDim.x * blockDim.x)
    out[i] = w[i] / h;
}

// x += sum_i y[i] * Z_i (i ascending), y in device memory.
__global__ void lincomb_kernel(long n, const double* __restrict__ Z, long ldz, int k,
                               const double* __restrict__ y, double* __restrict__ x) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n;
       i += (long)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int j = 0; j < k; ++j) acc = fma(y[j], Z[j * ldz + i], acc);
    x[i] += acc;
  }
}

static int grid_for_n(long n) {
  long g = (n + 255) / 256;
  if (g > kSMs * 8) g = kSMs * 8;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace ivk

using namespace ivk;

extern "C" {

int ivk_dot(int64_t n, const double* x, const double* y, double* result, void* stream) {
  IVK_REQUIRE(n >= 0 && x && result, "bad dot arguments");
  RedScratch* s = nullptr;
  int rc = scratch(&s);
  if (rc) return rc;
  // <x, y> via the fused kernel with no axpy part (w = x is only read).
  axpy_dot_kernel<<<kRedBlocks, kRedThreads, 0, as_stream(stream)>>>(
      n, nullptr, nullptr, 0, const_cast<double*>(x), y, s->partial, s->counter, result);
  return check_launch("ivk_dot");
}

int ivk_mgs(int64_t n, const double* V, int64_t ldv, int32_t k, double* w, double* h,
            double* v_next, void* stream) {
  IVK_REQUIRE(n > 0 && V && w && h && k >= 1 && ldv >= n, "bad MGS arguments");
  RedScratch* s = nullptr;
  int rc = scratch(&s);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  // pass 0: h0 = <w, V0>; pass i: w -= h_{i-1} V_{i-1}, h_i = <w, V_i>
  for (int i = 0; i < k; ++i) {
    axpy_dot_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(
        n, i ? V + (long)(i - 1) * ldv : nullptr, h, i - 1, w, V + (long)i * ldv, s->partial,
        s->counter, h + i);
    rc = check_launch("ivk_mgs");
    if (rc) return rc;
  }
  // last axpy fused with the norm: h_k = ||w||
  axpy_dot_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(n, V + (long)(k - 1) * ldv, h, k - 1, w,
                                                     nullptr, s->partial, s->counter, h + k);
  rc = check_launch("ivk_mgs");
  if (rc) return rc;
  if (v_next) {
    scale_kernel<<<grid_for_n(n), 256, 0, st>>>(n, w, h, k, v_next);
    rc = check_launch("ivk_mgs");
  }
  return rc;
}

int ivk_norm(int64_t n, const double* x, double* result, void* stream) {
  IVK_REQUIRE(n >= 0 && x && result, "bad norm arguments");
  RedScratch* s = nullptr;
  int rc = scratch(&s);
  if (rc) return rc;
  axpy_dot_kernel<<<kRedBlocks, kRedThreads, 0, as_stream(stream)>>>(
      n, nullptr, nullptr, 0, const_cast<double*>(x), nullptr, s->partial, s->counter, result);
  return check_launch("ivk_norm");
}

int ivk_scale(int64_t n, const double* x, const double* coef, int32_t k, double* out,
              void* stream) {
  IVK_REQUIRE(n >= 0 && x && coef && out, "bad scale arguments");
  scale_kernel<<<grid_for_n(n), 256, 0, as_stream(stream)>>>(n, x, coef, k, out);
  return check_launch("ivk_scale");
}

int ivk_lincomb(int64_t n, const double* Z, int64_t ldz, int32_t k, const double* y, double* x,
                void* stream) {
  IVK_REQUIRE(n >= 0 && Z && y && x && k >= 0 && ldz >= n, "bad lincomb arguments");
  if (k == 0 || n == 0) return IVK_OK;
  lincomb_kernel<<<grid_for_n(n), 256, 0, as_stream(stream)>>>(n, Z, ldz, k, y, x);
  return check_launch("ivk_lincomb");
}

}  // extern "C"
