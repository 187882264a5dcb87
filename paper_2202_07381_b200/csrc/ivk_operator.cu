// K1: Kronecker-structured stage operator apply / residual, and the small
// vector kernels of the smoother and cycle (K8).  sm_100a, fp64.
//
// Reference semantics: StageSystem.matvec (stages.py:110-126)
//   yu_i = M u_i + dt sum_j a_ij (K u_j + B p_j) [+ dt J_i sum_j a_ij u_j]
//   yu[constrained] = u[constrained];   yp_i = dt sum_j a_ij B^T u_j
// M, K (and J) are read ONCE per scalar P2 pattern entry for both velocity
// components and all s stages (M_vec = M_P2 (x) I_2).

#include <stdarg.h>
#include <string.h>

#include "ivk_common.cuh"

namespace ivk {

static thread_local char g_err[512] = "";
std::atomic<long long> g_launches{0};

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int check_launch(const char* what) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return IVK_ECUDA;
  }
  return IVK_OK;
}

// Everything the operator kernel needs, passed by value (kernel parameter
// space), so no device-side descriptor copy is required.
struct OpParams {
  int n_nodes, n_p, n_conv, nnz;
  double dt;
  double a[IVK_MAX_STAGES * IVK_MAX_STAGES];
  const int32_t* __restrict__ p2_rowptr;
  const int32_t* __restrict__ p2_col;
  const double2* __restrict__ p2_mk;
  const double4* __restrict__ conv;
  const int32_t* __restrict__ b_rowptr;
  const int32_t* __restrict__ b_col;
  const double2* __restrict__ b_val;
  const int32_t* __restrict__ bt_rowptr;
  const int32_t* __restrict__ bt_col;
  const double2* __restrict__ bt_val;
  const uint8_t* __restrict__ cmask;
};

// One thread per scalar P2 node (both components, all S stages), then one
// thread per P1 node.  NC = 0 (Stokes), 1 (one J shared by all stages) or
// S (per-stage J_i).
template <int S, int NC>
__global__ void __launch_bounds__(256) stage_apply_kernel(OpParams op, const double* __restrict__ x,
                                                          const double* __restrict__ b,
                                                          double* __restrict__ out) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  const int nu = 2 * op.n_nodes;
  const long sd = nu + op.n_p;
  if (row < op.n_nodes) {
    const int n = row;
    if (op.cmask[n]) {
#pragma unroll
      for (int t = 0; t < S; ++t) {
        const long o = t * sd + 2 * n;
        const double y0 = x[o], y1 = x[o + 1];
        out[o] = b ? b[o] - y0 : y0;
        out[o + 1] = b ? b[o + 1] - y1 : y1;
      }
      return;
    }
    double mu[S][2], ku[S][2], bp[S][2], ju[S][2];
#pragma unroll
    for (int t = 0; t < S; ++t)
#pragma unroll
      for (int c = 0; c < 2; ++c) mu[t][c] = ku[t][c] = bp[t][c] = ju[t][c] = 0.0;

    const int e0 = op.p2_rowptr[n], e1 = op.p2_rowptr[n + 1];
    for (int e = e0; e < e1; ++e) {
      const int col = op.p2_col[e];
      const double2 mk = op.p2_mk[e];
      double ux[S], uy[S];
#pragma unroll
      for (int t = 0; t < S; ++t) {
        ux[t] = x[t * sd + 2 * col];
        uy[t] = x[t * sd + 2 * col + 1];
        mu[t][0] = fma(mk.x, ux[t], mu[t][0]);
        mu[t][1] = fma(mk.x, uy[t], mu[t][1]);
        ku[t][0] = fma(mk.y, ux[t], ku[t][0]);
        ku[t][1] = fma(mk.y, uy[t], ku[t][1]);
      }
      if constexpr (NC == 1) {
        const double4 J = op.conv[e];
#pragma unroll
        for (int t = 0; t < S; ++t) {
          ju[t][0] += J.x * ux[t] + J.y * uy[t];
          ju[t][1] += J.z * ux[t] + J.w * uy[t];
        }
      } else if constexpr (NC == S && NC > 1) {
        // Row stage i uses J_i applied to sum_j a_ij u_j (stages.py:118-123).
#pragma unroll
        for (int i = 0; i < S; ++i) {
          const double4 J = op.conv[(long)i * op.nnz + e];
          double wx = 0.0, wy = 0.0;
#pragma unroll
          for (int j = 0; j < S; ++j) {
            wx += op.a[i * S + j] * ux[j];
            wy += op.a[i * S + j] * uy[j];
          }
          ju[i][0] += J.x * wx + J.y * wy;
          ju[i][1] += J.z * wx + J.w * wy;
        }
      }
    }
    const int f0 = op.b_rowptr[n], f1 = op.b_rowptr[n + 1];
    for (int e = f0; e < f1; ++e) {
      const int q = op.b_col[e];
      const double2 bv = op.b_val[e];
#pragma unroll
      for (int t = 0; t < S; ++t) {
        const double p = x[t * sd + nu + q];
        bp[t][0] = fma(bv.x, p, bp[t][0]);
        bp[t][1] = fma(bv.y, p, bp[t][1]);
      }
    }
#pragma unroll
    for (int i = 0; i < S; ++i) {
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < S; ++j) {
          double kj = ku[j][c] + bp[j][c];
          if constexpr (NC == 1) kj += ju[j][c];
          acc += op.a[i * S + j] * kj;
        }
        double y = mu[i][c] + op.dt * acc;
        if constexpr (NC == S && NC > 1) y += op.dt * ju[i][c];
        const long o = i * sd + 2 * n + c;
        out[o] = b ? b[o] - y : y;
      }
    }
  } else if (row < op.n_nodes + op.n_p) {
    const int q = row - op.n_nodes;
    double btu[S];
#pragma unroll
    for (int t = 0; t < S; ++t) btu[t] = 0.0;
    const int e0 = op.bt_rowptr[q], e1 = op.bt_rowptr[q + 1];
    for (int e = e0; e < e1; ++e) {
      const int n = op.bt_col[e];
      const double2 bv = op.bt_val[e];
#pragma unroll
      for (int t = 0; t < S; ++t) {
        btu[t] = fma(bv.x, x[t * sd + 2 * n], btu[t]);
        btu[t] = fma(bv.y, x[t * sd + 2 * n + 1], btu[t]);
      }
    }
#pragma unroll
    for (int i = 0; i < S; ++i) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < S; ++j) acc += op.a[i * S + j] * btu[j];
      const double y = op.dt * acc;
      const long o = i * sd + nu + q;
      out[o] = b ? b[o] - y : y;
    }
  }
}

OpParams make_op_params(const ivk_operator_desc* d) {
  OpParams p;
  memset(&p, 0, sizeof(p));
  p.n_nodes = d->n_nodes;
  p.n_p = d->n_p;
  p.n_conv = d->n_conv;
  p.nnz = d->nnz;
  p.dt = d->dt;
  for (int i = 0; i < IVK_MAX_STAGES * IVK_MAX_STAGES; ++i) p.a[i] = d->butcher_a[i];
  p.p2_rowptr = d->p2_rowptr;
  p.p2_col = d->p2_col;
  p.p2_mk = reinterpret_cast<const double2*>(d->p2_mk);
  p.conv = reinterpret_cast<const double4*>(d->conv);
  p.b_rowptr = d->b_rowptr;
  p.b_col = d->b_col;
  p.b_val = reinterpret_cast<const double2*>(d->b_val);
  p.bt_rowptr = d->bt_rowptr;
  p.bt_col = d->bt_col;
  p.bt_val = reinterpret_cast<const double2*>(d->bt_val);
  p.cmask = d->node_constrained;
  return p;
}

int validate_op(const ivk_operator_desc* d) {
  IVK_REQUIRE(d != nullptr, "operator descriptor is NULL");
  IVK_REQUIRE(d->stages >= 1 && d->stages <= IVK_MAX_STAGES, "stages=%d outside [1,%d]", d->stages,
              IVK_MAX_STAGES);
  IVK_REQUIRE(d->n_nodes > 0 && d->n_p > 0, "empty operator");
  IVK_REQUIRE(d->n_conv == 0 || d->n_conv == 1 || d->n_conv == d->stages,
              "n_conv must be 0, 1 or stages");
  IVK_REQUIRE(d->n_conv == 0 || d->conv != nullptr, "conv is NULL with n_conv > 0");
  IVK_REQUIRE(d->nnz > 0, "nnz must be positive");
  IVK_REQUIRE(d->p2_rowptr && d->p2_col && d->p2_mk && d->b_rowptr && d->b_col && d->b_val &&
                  d->bt_rowptr && d->bt_col && d->bt_val && d->node_constrained,
              "operator descriptor has a NULL array");
  return IVK_OK;
}

template <int S>
static void launch_stage_apply(const OpParams& q, int nconv, const double* x, const double* b,
                               double* out, cudaStream_t st) {
  const OpParams& p = q;
  const int rows = p.n_nodes + p.n_p;
  const int block = 256;
  const int grid = (rows + block - 1) / block;
  if (nconv == 0)
    stage_apply_kernel<S, 0><<<grid, block, 0, st>>>(q, x, b, out);
  else if (nconv == 1)
    stage_apply_kernel<S, 1><<<grid, block, 0, st>>>(q, x, b, out);
  else
    stage_apply_kernel<S, S><<<grid, block, 0, st>>>(q, x, b, out);
}

// ---------------------------------------------------------------- vectors

__global__ void axpby_kernel(long n, double alpha, const double* __restrict__ x, double beta,
                             const double* __restrict__ y, double* out) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    double v = 0.0;
    if (x) v = alpha * x[i];
    if (y) v += beta * y[i];
    out[i] = v;
  }
}

// One CTA per stage; fixed-order (deterministic) reduction.
__global__ void __launch_bounds__(1024) project_means_kernel(int n_u, int n_p, double* x) {
  __shared__ double red[32];
  const long sd = (long)n_u + n_p;
  double* p = x + blockIdx.x * sd + n_u;
  double acc = 0.0;
  for (int i = threadIdx.x; i < n_p; i += blockDim.x) acc += p[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  const double mean = red[0] / (double)n_p;
  for (int i = threadIdx.x; i < n_p; i += blockDim.x) p[i] -= mean;
}

__global__ void seed_constrained_kernel(int S, int n_nodes, int n_p, const uint8_t* __restrict__ cm,
                                        const double* __restrict__ src, double* __restrict__ out) {
  const long sd = 2L * n_nodes + n_p;
  const long total = S * sd;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total;
       i += (long)gridDim.x * blockDim.x) {
    const long loc = i % sd;
    double v = 0.0;
    if (loc < 2L * n_nodes && cm[loc >> 1]) v = src[i];
    out[i] = v;
  }
}

static int grid_for(long n, int block) {
  long g = (n + block - 1) / block;
  const long cap = (long)kSMs * 16;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

}  // namespace ivk

using namespace ivk;

extern "C" {

const char* ivk_last_error(void) { return g_err; }
int ivk_version(void) { return 1; }
int64_t ivk_launch_count(void) { return g_launches.load(); }

int ivk_stage_apply(const ivk_operator_desc* op, const double* x, const double* b, double* out,
                    void* stream) {
  int rc = validate_op(op);
  if (rc) return rc;
  IVK_REQUIRE(x && out, "x/out is NULL");
  IVK_REQUIRE(out != x, "out must not alias x");
  OpParams p = make_op_params(op);
  cudaStream_t st = as_stream(stream);
  switch (op->stages) {
    case 1: launch_stage_apply<1>(p, op->n_conv, x, b, out, st); break;
    case 2: launch_stage_apply<2>(p, op->n_conv, x, b, out, st); break;
    case 3: launch_stage_apply<3>(p, op->n_conv, x, b, out, st); break;
  }
  return check_launch("ivk_stage_apply");
}

int ivk_axpby(int64_t n, double alpha, const double* x, double beta, const double* y, double* out,
              void* stream) {
  IVK_REQUIRE(out != nullptr && n >= 0, "bad axpby arguments");
  if (n == 0) return IVK_OK;
  axpby_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(n, alpha, x, beta, y, out);
  return check_launch("ivk_axpby");
}

int ivk_project_pressure_means(int32_t stages, int32_t n_u, int32_t n_p, double* x, void* stream) {
  IVK_REQUIRE(x && stages >= 1 && n_p > 0 && n_u >= 0, "bad projection arguments");
  project_means_kernel<<<stages, 1024, 0, as_stream(stream)>>>(n_u, n_p, x);
  return check_launch("ivk_project_pressure_means");
}

int ivk_seed_constrained(int32_t stages, int32_t n_nodes, int32_t n_p, const uint8_t* cm,
                         const double* src, double* out, void* stream) {
  IVK_REQUIRE(cm && src && out && stages >= 1, "bad seed arguments");
  const long total = (long)stages * (2L * n_nodes + n_p);
  seed_constrained_kernel<<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(stages, n_nodes, n_p,
                                                                              cm, src, out);
  return check_launch("ivk_seed_constrained");
}

}  // extern "C"
