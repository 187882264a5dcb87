// The general stage-coupled operator path on sm_100a, fp64 (include/ivk.h,
// ivk_general_*): multi-field systems whose spatial operator L is shared by
// every stage -- BASELINE config 5 (2-D resistive MHD, mhd.py).
//
//  K1g ivk_general_apply      out = b - (I_s (x) M + dt A (x) L) x, identity on
//                             constrained rows (StageSystem.matvec generalised,
//                             stages.py:110-126).  SELL-32, one thread per
//                             single-stage row doing all s stages: each (m, l)
//                             pair and column index is read once per apply and
//                             the s stage values of x are gathered from L2.
//  K5g ivk_general_restrict / ivk_general_prolong_add   I_s (x) P and its
//                             transpose (explicit, so both directions are
//                             deterministic row gathers), solvers.py:340-346.
//  K8g ivk_general_seed_constrained  z[cd] = r[cd] (solvers.py:352-354).
//
// K7g (patch factorisation) lives in ivk_patches.cu next to K7.

#include "ivk_common.cuh"

namespace ivk {

struct GenParams {
  int S, n;
  double dt;
  double a[IVK_MAX_STAGES * IVK_MAX_STAGES];
  const int32_t* __restrict__ sptr;
  const int32_t* __restrict__ scol;
  const double2* __restrict__ sml;
  const uint8_t* __restrict__ cm;
};

int validate_general(const ivk_general_desc* d) {
  IVK_REQUIRE(d != nullptr, "general operator descriptor is NULL");
  IVK_REQUIRE(d->stages >= 1 && d->stages <= IVK_MAX_STAGES, "stages=%d outside [1,%d]",
              d->stages, IVK_MAX_STAGES);
  IVK_REQUIRE(d->n > 0 && d->nnz >= 0, "empty general operator");
  IVK_REQUIRE(d->rowptr && d->col && d->ml && d->sptr && d->scol && d->sml && d->constrained,
              "general operator descriptor has a NULL array");
  return IVK_OK;
}

static GenParams make_gen_params(const ivk_general_desc* d) {
  GenParams g;
  g.S = d->stages;
  g.n = d->n;
  g.dt = d->dt;
  for (int i = 0; i < IVK_MAX_STAGES * IVK_MAX_STAGES; ++i) g.a[i] = d->butcher_a[i];
  g.sptr = d->sptr;
  g.scol = d->scol;
  g.sml = reinterpret_cast<const double2*>(d->sml);
  g.cm = d->constrained;
  return g;
}

constexpr int kGenBlock = 256;

template <int S>
__global__ void __launch_bounds__(kGenBlock) general_apply_kernel(GenParams g,
                                                                  const double* __restrict__ x,
                                                                  const double* b, double* out) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= g.n) return;
  const long n = g.n;
  const int lane = row & 31;
  const int e1 = g.sptr[(row >> 5) + 1];
  int e = g.sptr[row >> 5] + lane;
  double am[S], al[S];
#pragma unroll
  for (int j = 0; j < S; ++j) am[j] = al[j] = 0.0;
  // four entries' index/value loads in flight before their dependent gathers
  for (; e + 3 * 32 < e1; e += 4 * 32) {
    int c[4];
    double2 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      c[u] = __ldg(g.scol + e + 32 * u);
      v[u] = ld_stream2(g.sml + e + 32 * u);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int j = 0; j < S; ++j) {
        const double xv = __ldg(x + j * n + c[u]);
        am[j] = fma(v[u].x, xv, am[j]);
        al[j] = fma(v[u].y, xv, al[j]);
      }
  }
  for (; e < e1; e += 32) {
    const int c = __ldg(g.scol + e);
    const double2 v = ld_stream2(g.sml + e);
#pragma unroll
    for (int j = 0; j < S; ++j) {
      const double xv = __ldg(x + j * n + c);
      am[j] = fma(v.x, xv, am[j]);
      al[j] = fma(v.y, xv, al[j]);
    }
  }
  const bool fixed = g.cm[row] != 0;
#pragma unroll
  for (int i = 0; i < S; ++i) {
    const long k = i * n + row;
    double y;
    if (fixed) {
      y = x[k];
    } else {
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < S; ++j) s = fma(g.a[i * S + j], al[j], s);
      y = fma(g.dt, s, am[i]);
    }
    out[k] = b ? b[k] - y : y;
  }
}

__global__ void general_seed_kernel(int S, int n, const uint8_t* __restrict__ cm,
                                    const double* __restrict__ src, double* __restrict__ out) {
  const long total = (long)S * n;
  for (long k = blockIdx.x * (long)blockDim.x + threadIdx.x; k < total;
       k += (long)gridDim.x * blockDim.x) {
    const int d = (int)(k % n);
    out[k] = cm[d] ? src[k] : 0.0;
  }
}

struct GenTransferParams {
  int S, nf, nc;
  const int32_t* __restrict__ p_rowptr;
  const int32_t* __restrict__ p_col;
  const double* __restrict__ p_val;
  const int32_t* __restrict__ pt_rowptr;
  const int32_t* __restrict__ pt_col;
  const double* __restrict__ pt_val;
  const uint8_t* __restrict__ fcm;
  const uint8_t* __restrict__ ccm;
};

template <int S>
__global__ void general_restrict_kernel(GenTransferParams t, const double* __restrict__ rf,
                                        double* __restrict__ rc) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < t.nc; i += gridDim.x * blockDim.x) {
    double acc[S];
#pragma unroll
    for (int s = 0; s < S; ++s) acc[s] = 0.0;
    if (!t.ccm[i]) {
      for (int e = t.pt_rowptr[i]; e < t.pt_rowptr[i + 1]; ++e) {
        const int c = t.pt_col[e];
        const double v = t.pt_val[e];
#pragma unroll
        for (int s = 0; s < S; ++s) acc[s] = fma(v, rf[(long)s * t.nf + c], acc[s]);
      }
    }
#pragma unroll
    for (int s = 0; s < S; ++s) rc[(long)s * t.nc + i] = acc[s];
  }
}

template <int S>
__global__ void general_prolong_kernel(GenTransferParams t, const double* __restrict__ ec,
                                       double* __restrict__ xf) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < t.nf; i += gridDim.x * blockDim.x) {
    if (t.fcm[i]) continue;
    double acc[S];
#pragma unroll
    for (int s = 0; s < S; ++s) acc[s] = 0.0;
    for (int e = t.p_rowptr[i]; e < t.p_rowptr[i + 1]; ++e) {
      const int c = t.p_col[e];
      const double v = t.p_val[e];
#pragma unroll
      for (int s = 0; s < S; ++s) acc[s] = fma(v, ec[(long)s * t.nc + c], acc[s]);
    }
#pragma unroll
    for (int s = 0; s < S; ++s) xf[(long)s * t.nf + i] += acc[s];
  }
}

static int grid_cap(long n, int block) {
  long g = (n + block - 1) / block;
  const long cap = (long)kSMs * 16;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

static int validate_transfer(const ivk_general_transfer_desc* t) {
  IVK_REQUIRE(t != nullptr, "transfer descriptor is NULL");
  IVK_REQUIRE(t->stages >= 1 && t->stages <= IVK_MAX_STAGES && t->nf > 0 && t->nc > 0,
              "bad transfer dimensions");
  IVK_REQUIRE(t->p_rowptr && t->p_col && t->p_val && t->pt_rowptr && t->pt_col && t->pt_val &&
                  t->fine_constrained && t->coarse_constrained,
              "transfer descriptor has a NULL array");
  return IVK_OK;
}

static GenTransferParams make_transfer(const ivk_general_transfer_desc* d) {
  GenTransferParams t;
  t.S = d->stages;
  t.nf = d->nf;
  t.nc = d->nc;
  t.p_rowptr = d->p_rowptr;
  t.p_col = d->p_col;
  t.p_val = d->p_val;
  t.pt_rowptr = d->pt_rowptr;
  t.pt_col = d->pt_col;
  t.pt_val = d->pt_val;
  t.fcm = d->fine_constrained;
  t.ccm = d->coarse_constrained;
  return t;
}

}  // namespace ivk

using namespace ivk;

extern "C" {

int ivk_general_apply(const ivk_general_desc* op, const double* x, const double* b, double* out,
                      void* stream) {
  int rc = validate_general(op);
  if (rc) return rc;
  IVK_REQUIRE(x && out, "x/out is NULL");
  IVK_REQUIRE(out != x, "out must not alias x");
  GenParams g = make_gen_params(op);
  const int grid = (op->n + kGenBlock - 1) / kGenBlock;
  cudaStream_t st = as_stream(stream);
  switch (op->stages) {
    case 1: general_apply_kernel<1><<<grid, kGenBlock, 0, st>>>(g, x, b, out); break;
    case 2: general_apply_kernel<2><<<grid, kGenBlock, 0, st>>>(g, x, b, out); break;
    case 3: general_apply_kernel<3><<<grid, kGenBlock, 0, st>>>(g, x, b, out); break;
  }
  return check_launch("ivk_general_apply");
}

int ivk_general_seed_constrained(const ivk_general_desc* op, const double* src, double* out,
                                 void* stream) {
  int rc = validate_general(op);
  if (rc) return rc;
  IVK_REQUIRE(src && out, "src/out is NULL");
  const long total = (long)op->stages * op->n;
  general_seed_kernel<<<grid_cap(total, 256), 256, 0, as_stream(stream)>>>(
      op->stages, op->n, op->constrained, src, out);
  return check_launch("ivk_general_seed_constrained");
}

int ivk_general_restrict(const ivk_general_transfer_desc* d, const double* rf, double* rc,
                         void* stream) {
  int e = validate_transfer(d);
  if (e) return e;
  IVK_REQUIRE(rf && rc && rf != rc, "bad restrict vectors");
  GenTransferParams t = make_transfer(d);
  const int grid = grid_cap(d->nc, 256);
  cudaStream_t st = as_stream(stream);
  switch (d->stages) {
    case 1: general_restrict_kernel<1><<<grid, 256, 0, st>>>(t, rf, rc); break;
    case 2: general_restrict_kernel<2><<<grid, 256, 0, st>>>(t, rf, rc); break;
    case 3: general_restrict_kernel<3><<<grid, 256, 0, st>>>(t, rf, rc); break;
  }
  return check_launch("ivk_general_restrict");
}

int ivk_general_prolong_add(const ivk_general_transfer_desc* d, const double* ec, double* xf,
                            void* stream) {
  int e = validate_transfer(d);
  if (e) return e;
  IVK_REQUIRE(ec && xf && ec != xf, "bad prolongation vectors");
  GenTransferParams t = make_transfer(d);
  const int grid = grid_cap(d->nf, 256);
  cudaStream_t st = as_stream(stream);
  switch (d->stages) {
    case 1: general_prolong_kernel<1><<<grid, 256, 0, st>>>(t, ec, xf); break;
    case 2: general_prolong_kernel<2><<<grid, 256, 0, st>>>(t, ec, xf); break;
    case 3: general_prolong_kernel<3><<<grid, 256, 0, st>>>(t, ec, xf); break;
  }
  return check_launch("ivk_general_prolong_add");
}

}  // extern "C"
