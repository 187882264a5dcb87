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

// Caller-owned reduction scratch (ivk_reduction_scratch_bytes()): the block
// partials followed by the last-block counter.  One scratch per stream of
// reductions; the counter returns to 0 after every reduction, so a scratch
// zeroed once serves any number of stream-ordered calls (and CUDA-graph
// capture: nothing is allocated here).
struct RedScratch {
  double* partial;
  unsigned int* counter;
};

static inline RedScratch scratch_of(void* p) {
  RedScratch s;
  s.partial = static_cast<double*>(p);
  s.counter = reinterpret_cast<unsigned int*>(s.partial + kRedBlocks);
  return s;
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

// out = w / coef[k] when coef[k] > 1e-300 (solvers.py:407-408), else 0 (the
// reference's basis rows start as zeros and stay so on breakdown).
__global__ void scale_kernel(long n, const double* __restrict__ w, const double* coef, int k,
                             double* __restrict__ out) {
  const double h = coef[k];
  const bool ok = h > 1e-300;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n;
       i += (long)gridDim.x * blockDim.x)
    out[i] = ok ? w[i] / h : 0.0;
}

// Givens update of Hessenberg column j (solvers.py:409-421) on the device:
// the stored rotations applied to H[:, j] in order, the new rotation formed,
// g rotated; est = |g[j+1]|.  H column-major with leading dimension ldh.
// One thread: j <= restart (<= a few hundred) scalar steps.
__global__ void givens_kernel(int j, int ldh, double* H, double* cs, double* sn, double* g,
                              double* est) {
  double* h = H + (long)j * ldh;
  for (int i = 0; i < j; ++i) {
    const double t = cs[i] * h[i] + sn[i] * h[i + 1];
    h[i + 1] = -sn[i] * h[i] + cs[i] * h[i + 1];
    h[i] = t;
  }
  const double denom = hypot(h[j], h[j + 1]);
  cs[j] = h[j] / denom;
  sn[j] = h[j + 1] / denom;
  h[j] = denom;
  h[j + 1] = 0.0;
  g[j + 1] = -sn[j] * g[j];
  g[j] = cs[j] * g[j];
  *est = fabs(g[j + 1]);
}

// y = triu(H[:k, :k])^-1 g[:k] by back substitution (solvers.py:430), one
// thread.  H column-major (ldh).
__global__ void hessenberg_solve_kernel(int k, int ldh, const double* H, const double* g,
                                        double* y) {
  for (int i = k - 1; i >= 0; --i) {
    double v = g[i];
    for (int c = i + 1; c < k; ++c) v -= H[(long)c * ldh + i] * y[c];
    y[i] = v / H[(long)i * ldh + i];
  }
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

size_t ivk_reduction_scratch_bytes(void) {
  return kRedBlocks * sizeof(double) + 16;
}

int ivk_dot(int64_t n, const double* x, const double* y, double* result, void* scratch,
            void* stream) {
  IVK_REQUIRE(n >= 0 && x && result && scratch, "bad dot arguments");
  const RedScratch s = scratch_of(scratch);
  // <x, y> via the fused kernel with no axpy part (w = x is only read).
  axpy_dot_kernel<<<kRedBlocks, kRedThreads, 0, as_stream(stream)>>>(
      n, nullptr, nullptr, 0, const_cast<double*>(x), y, s.partial, s.counter, result);
  return check_launch("ivk_dot");
}

int ivk_mgs(int64_t n, const double* V, int64_t ldv, int32_t k, double* w, double* h,
            double* v_next, void* scratch, void* stream) {
  IVK_REQUIRE(n > 0 && V && w && h && k >= 1 && ldv >= n && scratch, "bad MGS arguments");
  const RedScratch sc = scratch_of(scratch);
  const RedScratch* s = &sc;
  int rc = IVK_OK;
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

int ivk_norm(int64_t n, const double* x, double* result, void* scratch, void* stream) {
  IVK_REQUIRE(n >= 0 && x && result && scratch, "bad norm arguments");
  const RedScratch s = scratch_of(scratch);
  axpy_dot_kernel<<<kRedBlocks, kRedThreads, 0, as_stream(stream)>>>(
      n, nullptr, nullptr, 0, const_cast<double*>(x), nullptr, s.partial, s.counter, result);
  return check_launch("ivk_norm");
}

int ivk_scale(int64_t n, const double* x, const double* coef, int32_t k, double* out,
              void* stream) {
  IVK_REQUIRE(n >= 0 && x && coef && out, "bad scale arguments");
  scale_kernel<<<grid_for_n(n), 256, 0, as_stream(stream)>>>(n, x, coef, k, out);
  return check_launch("ivk_scale");
}

int ivk_givens(int32_t j, int32_t ldh, double* H, double* cs, double* sn, double* g, double* est,
               void* stream) {
  IVK_REQUIRE(j >= 0 && ldh >= j + 2 && H && cs && sn && g && est, "bad givens arguments");
  givens_kernel<<<1, 1, 0, as_stream(stream)>>>(j, ldh, H, cs, sn, g, est);
  return check_launch("ivk_givens");
}

int ivk_hessenberg_solve(int32_t k, int32_t ldh, const double* H, const double* g, double* y,
                         void* stream) {
  IVK_REQUIRE(k >= 0 && ldh >= k && H && g && y, "bad hessenberg_solve arguments");
  if (k == 0) return IVK_OK;
  hessenberg_solve_kernel<<<1, 1, 0, as_stream(stream)>>>(k, ldh, H, g, y);
  return check_launch("ivk_hessenberg_solve");
}

int ivk_lincomb(int64_t n, const double* Z, int64_t ldz, int32_t k, const double* y, double* x,
                void* stream) {
  IVK_REQUIRE(n >= 0 && Z && y && x && k >= 0 && ldz >= n, "bad lincomb arguments");
  if (k == 0 || n == 0) return IVK_OK;
  lincomb_kernel<<<grid_for_n(n), 256, 0, as_stream(stream)>>>(n, Z, ldz, k, y, x);
  return check_launch("ivk_lincomb");
}

}  // extern "C"
