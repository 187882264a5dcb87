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
  int n_nodes, n_p, n_conv, nnz_s;
  double dt;
  double a[IVK_MAX_STAGES * IVK_MAX_STAGES];
  const int32_t* __restrict__ p2_sptr;
  const int32_t* __restrict__ p2_scol;
  const double2* __restrict__ p2_smk;
  const double4* __restrict__ conv_s;
  const int32_t* __restrict__ b_sptr;
  const int32_t* __restrict__ b_scol;
  const double2* __restrict__ b_sval;
  const int32_t* __restrict__ bt_sptr;
  const int32_t* __restrict__ bt_scol;
  const double2* __restrict__ bt_sval;
  const uint8_t* __restrict__ cmask;
};

// Velocity rows: SELL-16, one warp per 16-row slice, lane = 2 * row + comp
// (each thread one velocity component of one node, all S stages; the lane
// pair shares the entry's col / (m,k) loads, its x gathers hit one sector).
// Pressure rows: SELL-32, one thread per P1 node.  Entry e of a slice's
// row j sits at ptr[slice] + H e + j (H = 16 / 32).
// NC = 0 (Stokes), 1 (one J shared by all stages) or S (per-stage J_i).
// LIST: only the warps (slices) listed in `slices` run -- the rows a shard's
// patches read (shard.py); the other rows of `out` are left untouched.
// The Stokes variant (S >= 2) is capped at 64 registers (4 CTAs, 32 warps
// per SM): its software-pipelined gathers need 78 otherwise, and the lost
// occupancy costs more than the pipelining gains (57 -> 60 us uncapped, 51.6
// capped, cfg2 fine level).
// Loads of the operator's own streams (SELL columns and values: read once per
// apply).  IVK_K1_STREAM=1 marks them evict-first (ld.global.cs) so the L1
// lines they would take stay with the gathered x.
#ifndef IVK_K1_STREAM
#define IVK_K1_STREAM 0
#endif
template <class T>
__device__ __forceinline__ T k1_ld(const T* p) {
#if IVK_K1_STREAM
  return __ldcs(p);
#else
  return *p;
#endif
}

template <int S, int NC, bool LIST>
__global__ void __launch_bounds__(256, (NC == 0 && S >= 2) ? 4 : 0) stage_apply_kernel(OpParams op, const double* __restrict__ x,
                                                          const double* b,
                                                          double* out,
                                                          const int32_t* __restrict__ slices,
                                                          int n_slices) {
  const int nslice_v = (op.n_nodes + 15) >> 4;
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if constexpr (LIST) {
    if (warp >= n_slices) return;
    warp = __ldg(slices + warp);
  } else {
    // pressure slices (long rows: ~19 B^T entries per thread) first, so they
    // do not form the last wave
    const int npw = (op.n_p + 31) >> 5;
    if (warp >= npw + nslice_v) return;  // grid padding (must not alias a slice: out may be b)
    warp = warp < npw ? nslice_v + warp : warp - npw;
  }
  const int lane = threadIdx.x & 31;
  const int nu = 2 * op.n_nodes;
  const long sd = nu + op.n_p;
  if (warp < nslice_v) {
    const int j = lane >> 1, c = lane & 1;
    const int n = (warp << 4) + j;
    const bool valid = n < op.n_nodes;
    const bool fixed = valid && op.cmask[n];
    double mu[S], ku[S], ju[(NC > 1) ? S : 1];
#pragma unroll
    for (int t = 0; t < S; ++t) mu[t] = ku[t] = 0.0;
#pragma unroll
    for (int t = 0; t < ((NC > 1) ? S : 1); ++t) ju[t] = 0.0;
    if (!fixed) {
      const int e0 = op.p2_sptr[warp], e1 = op.p2_sptr[warp + 1];
      if constexpr (NC == 0) {
        // latency-bound gathers: U entries' (col, m/k) loads, then their 3 U
        // x loads, in flight together (same summation order as one by one)
// batch size of the pipelined gathers: 3 and 4 measure alike (50.8 vs 51.0
// us, cfg2); 5 spills at the 64-register cap
#ifndef IVK_K1_U
#define IVK_K1_U 4
#endif
        constexpr int U = (S >= 2) ? IVK_K1_U : 4;
        if constexpr (S >= 2) {
        // software pipeline: the next batch's (col, m/k) loads are issued
        // before this batch's x gathers are consumed
        int cl[U];
        double2 mk[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int ee = e0 + j + 16 * u;
          const bool ok = ee < e1;
          cl[u] = ok ? k1_ld(op.p2_scol + ee) : -1;
          mk[u] = ok ? k1_ld(op.p2_smk + ee) : make_double2(0.0, 0.0);
        }
        for (int e = e0 + j; e < e1; e += 16 * U) {
          double uu[U][S];
#pragma unroll
          for (int u = 0; u < U; ++u)
#pragma unroll
            for (int t = 0; t < S; ++t) uu[u][t] = cl[u] >= 0 ? x[t * sd + 2 * cl[u] + c] : 0.0;
          int cn[U];
          double2 mn[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int ee = e + 16 * (U + u);
            const bool ok = ee < e1;
            cn[u] = ok ? k1_ld(op.p2_scol + ee) : -1;
            mn[u] = ok ? k1_ld(op.p2_smk + ee) : make_double2(0.0, 0.0);
          }
#pragma unroll
          for (int u = 0; u < U; ++u)
#pragma unroll
            for (int t = 0; t < S; ++t) {
              mu[t] = fma(mk[u].x, uu[u][t], mu[t]);
              ku[t] = fma(mk[u].y, uu[u][t], ku[t]);
            }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            cl[u] = cn[u];
            mk[u] = mn[u];
          }
        }
        } else {
        for (int e = e0 + j; e < e1; e += 16 * U) {
          int cl[U];
          double2 mk[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int ee = e + 16 * u;
            const bool ok = ee < e1;
            cl[u] = ok ? k1_ld(op.p2_scol + ee) : -1;
            mk[u] = ok ? k1_ld(op.p2_smk + ee) : make_double2(0.0, 0.0);
          }
          double uu[U][S];
#pragma unroll
          for (int u = 0; u < U; ++u)
#pragma unroll
            for (int t = 0; t < S; ++t) uu[u][t] = cl[u] >= 0 ? x[t * sd + 2 * cl[u] + c] : 0.0;
#pragma unroll
          for (int u = 0; u < U; ++u)
#pragma unroll
            for (int t = 0; t < S; ++t) {
              mu[t] = fma(mk[u].x, uu[u][t], mu[t]);
              ku[t] = fma(mk[u].y, uu[u][t], ku[t]);
            }
        }
        }
      } else if constexpr (NC == 1) {
        // one shared Jacobian (Oseen): batches of UJ entries -- their (col,
        // m/k, J row) loads, then their 2 S gathers of x, in flight together;
        // each lane reads only its own row (own, other) of the 2x2 block
#ifndef IVK_K1_UJ
#define IVK_K1_UJ 4
#endif
        constexpr int UJ = IVK_K1_UJ;
        for (int e = e0 + j; e < e1; e += 16 * UJ) {
          int cl[UJ];
          double2 mk[UJ], jr[UJ];
#pragma unroll
          for (int u = 0; u < UJ; ++u) {
            const int ee = e + 16 * u;
            const bool ok = ee < e1;
            cl[u] = ok ? op.p2_scol[ee] : -1;
            mk[u] = ok ? op.p2_smk[ee] : make_double2(0.0, 0.0);
            // row c of J: (J.x, J.y) or (J.z, J.w)
            jr[u] = ok ? reinterpret_cast<const double2*>(op.conv_s + ee)[c]
                       : make_double2(0.0, 0.0);
          }
          double uu[UJ][S], vv[UJ][S];
#pragma unroll
          for (int u = 0; u < UJ; ++u)
#pragma unroll
            for (int t = 0; t < S; ++t) {
              const long o = t * sd + 2 * (cl[u] >= 0 ? cl[u] : 0);
              uu[u][t] = cl[u] >= 0 ? x[o + c] : 0.0;
              vv[u][t] = cl[u] >= 0 ? x[o + (c ^ 1)] : 0.0;
            }
#pragma unroll
          for (int u = 0; u < UJ; ++u) {
            const double jd = c ? jr[u].y : jr[u].x, jo = c ? jr[u].x : jr[u].y;
#pragma unroll
            for (int t = 0; t < S; ++t) {
              mu[t] = fma(mk[u].x, uu[u][t], mu[t]);
              ku[t] = fma(mk[u].y, uu[u][t], ku[t]);
              ku[t] += jd * uu[u][t] + jo * vv[u][t];
            }
          }
        }
      } else
#pragma unroll 2
      for (int e = e0 + j; e < e1; e += 16) {
        const int col = op.p2_scol[e];
        const double2 mk = op.p2_smk[e];
        double u[S];
#pragma unroll
        for (int t = 0; t < S; ++t) {
          u[t] = x[t * sd + 2 * col + c];
          mu[t] = fma(mk.x, u[t], mu[t]);
          ku[t] = fma(mk.y, u[t], ku[t]);
        }
        if constexpr (NC >= 1) {
          // the other component of the same node (J couples components)
          double v[S];
#pragma unroll
          for (int t = 0; t < S; ++t) v[t] = x[t * sd + 2 * col + (c ^ 1)];
          if constexpr (NC == 1) {
            const double4 J = op.conv_s[e];
            const double jd = c ? J.w : J.x, jo = c ? J.z : J.y;  // row c: own, other
#pragma unroll
            for (int t = 0; t < S; ++t) ku[t] += jd * u[t] + jo * v[t];
          } else {
            // Row stage i uses J_i applied to sum_j a_ij u_j (stages.py:118-123).
#pragma unroll
            for (int i = 0; i < S; ++i) {
              const double4 J = op.conv_s[(long)i * op.nnz_s + e];
              const double jd = c ? J.w : J.x, jo = c ? J.z : J.y;
              double wu = 0.0, wv = 0.0;
#pragma unroll
              for (int t = 0; t < S; ++t) {
                wu += op.a[i * S + t] * u[t];
                wv += op.a[i * S + t] * v[t];
              }
              ju[i] += jd * wu + jo * wv;
            }
          }
        }
      }
      const int f0 = op.b_sptr[warp], f1 = op.b_sptr[warp + 1];
      {
        constexpr int U = 4;
        for (int e = f0 + j; e < f1; e += 16 * U) {
          int q[U];
          double bc[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int ee = e + 16 * u;
            const bool ok = ee < f1;
            q[u] = ok ? k1_ld(op.b_scol + ee) : -1;
            const double2 bv = ok ? k1_ld(op.b_sval + ee) : make_double2(0.0, 0.0);
            bc[u] = c ? bv.y : bv.x;
          }
          double pp[U][S];
#pragma unroll
          for (int u = 0; u < U; ++u)
#pragma unroll
            for (int t = 0; t < S; ++t) pp[u][t] = q[u] >= 0 ? x[t * sd + nu + q[u]] : 0.0;
#pragma unroll
          for (int u = 0; u < U; ++u)
#pragma unroll
            for (int t = 0; t < S; ++t) ku[t] = fma(bc[u], pp[u][t], ku[t]);
        }
      }
    }
    if (!valid) return;
#pragma unroll
    for (int i = 0; i < S; ++i) {
      const long o = i * sd + 2 * n + c;
      double y;
      if (fixed) {
        y = x[o];
      } else {
        double acc = 0.0;
#pragma unroll
        for (int t = 0; t < S; ++t) acc = fma(op.a[i * S + t], ku[t], acc);
        y = fma(op.dt, acc, mu[i]);
        if constexpr (NC > 1) y += op.dt * ju[i];
      }
      out[o] = b ? b[o] - y : y;
    }
  } else {
    const int ws = warp - nslice_v;
    const int q = (ws << 5) + lane;
    if (ws >= ((op.n_p + 31) >> 5)) return;
    double btu[S];
#pragma unroll
    for (int t = 0; t < S; ++t) btu[t] = 0.0;
    const int e0 = op.bt_sptr[ws], e1 = op.bt_sptr[ws + 1];
    int al = 0;  // stages whose velocity block starts 16-byte aligned
    if ((reinterpret_cast<uintptr_t>(x) & 15) == 0)
#pragma unroll
      for (int t = 0; t < S; ++t) al |= (int)(((t * sd) & 1) == 0) << t;
    constexpr int U = 4;
    for (int e = e0 + lane; e < e1; e += 32 * U) {
      int nn[U];
      double2 bv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int ee = e + 32 * u;
        const bool ok = ee < e1;
        nn[u] = ok ? k1_ld(op.bt_scol + ee) : -1;
        bv[u] = ok ? k1_ld(op.bt_sval + ee) : make_double2(0.0, 0.0);
      }
      double2 xv[U][S];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int t = 0; t < S; ++t)
          // one 16-byte load where the stage offset t * sd is even (half the
          // L1 lookups of two 8-byte loads), else two 8-byte loads
          {
            const double* px = x + t * sd + 2 * (nn[u] >= 0 ? nn[u] : 0);
            double2 v;
            if ((al >> t) & 1) {
              v = *reinterpret_cast<const double2*>(px);
            } else {
              v.x = px[0];
              v.y = px[1];
            }
            xv[u][t] = nn[u] >= 0 ? v : make_double2(0.0, 0.0);
          }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int t = 0; t < S; ++t) {
          btu[t] = fma(bv[u].x, xv[u][t].x, btu[t]);
          btu[t] = fma(bv[u].y, xv[u][t].y, btu[t]);
        }
    }
    if (q >= op.n_p) return;
#pragma unroll
    for (int i = 0; i < S; ++i) {
      double acc = 0.0;
#pragma unroll
      for (int t = 0; t < S; ++t) acc = fma(op.a[i * S + t], btu[t], acc);
      const double y = __dmul_rn(op.dt, acc);  // (no contraction with b - y)
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
  p.nnz_s = d->nnz_s;
  p.dt = d->dt;
  for (int i = 0; i < IVK_MAX_STAGES * IVK_MAX_STAGES; ++i) p.a[i] = d->butcher_a[i];
  p.p2_sptr = d->p2_sptr;
  p.p2_scol = d->p2_scol;
  p.p2_smk = reinterpret_cast<const double2*>(d->p2_smk);
  p.conv_s = reinterpret_cast<const double4*>(d->conv_s);
  p.b_sptr = d->b_sptr;
  p.b_scol = d->b_scol;
  p.b_sval = reinterpret_cast<const double2*>(d->b_sval);
  p.bt_sptr = d->bt_sptr;
  p.bt_scol = d->bt_scol;
  p.bt_sval = reinterpret_cast<const double2*>(d->bt_sval);
  p.cmask = d->node_constrained;
  return p;
}

int validate_op(const ivk_operator_desc* d) {
  IVK_REQUIRE(d != nullptr, "operator descriptor is NULL");
  IVK_REQUIRE(d->stages >= 1 && d->stages <= IVK_MAX_STAGES, "stages=%d outside [1,%d]", d->stages,
              IVK_MAX_STAGES);
  IVK_REQUIRE(d->n_nodes > 0 && d->n_p > 0, "empty operator");
  IVK_REQUIRE(d->ncomp == 0 || d->ncomp == 2 || d->ncomp == 3, "ncomp must be 2 or 3");
  IVK_REQUIRE(d->ncomp != 3 || d->n_conv == 0, "3-D operators carry no convection");
  IVK_REQUIRE(d->n_conv == 0 || d->n_conv == 1 || d->n_conv == d->stages,
              "n_conv must be 0, 1 or stages");
  IVK_REQUIRE(d->n_conv == 0 || d->conv != nullptr, "conv is NULL with n_conv > 0");
  IVK_REQUIRE(d->nnz > 0, "nnz must be positive");
  IVK_REQUIRE(d->p2_rowptr && d->p2_col && d->p2_mk && d->b_rowptr && d->b_col && d->b_val &&
                  d->bt_rowptr && d->bt_col && d->bt_val && d->node_constrained,
              "operator descriptor has a NULL array");
  IVK_REQUIRE(d->p2_sptr && d->p2_scol && d->p2_smk && d->b_sptr && d->b_scol && d->b_sval &&
                  d->bt_sptr && d->bt_scol && d->bt_sval,
              "operator descriptor has a NULL SELL array");
  IVK_REQUIRE(d->n_conv == 0 || d->conv_s != nullptr, "conv_s is NULL with n_conv > 0");
  return IVK_OK;
}

// 3-D (ncomp = 3, Kuhn tetrahedra): velocity rows in SELL-32, one thread per
// scalar node for its 3 components and all S stages; B / B^T values are
// (B_x, B_y, B_z) triples.  Pressure rows as in 2-D.
template <int S, bool LIST>
__global__ void __launch_bounds__(256) stage_apply3_kernel(OpParams op, const double* __restrict__ x,
                                                           const double* b,
                                                           double* out,
                                                           const int32_t* __restrict__ slices,
                                                           int n_slices) {
  const int nslice_v = (op.n_nodes + 31) >> 5;
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if constexpr (LIST) {
    if (warp >= n_slices) return;
    warp = __ldg(slices + warp);
  } else {
    const int npw = (op.n_p + 31) >> 5;
    if (warp >= npw + nslice_v) return;
    warp = warp < npw ? nslice_v + warp : warp - npw;
  }
  const int lane = threadIdx.x & 31;
  const int nu = 3 * op.n_nodes;
  const long sd = nu + op.n_p;
  const double* bsv = reinterpret_cast<const double*>(op.b_sval);
  const double* btv = reinterpret_cast<const double*>(op.bt_sval);
  if (warp < nslice_v) {
    const int n = (warp << 5) + lane;
    const bool valid = n < op.n_nodes;
    const bool fixed = valid && op.cmask[n];
    double mu[S][3], ku[S][3];
#pragma unroll
    for (int t = 0; t < S; ++t)
#pragma unroll
      for (int d = 0; d < 3; ++d) mu[t][d] = ku[t][d] = 0.0;
    if (!fixed) {
      const int e0 = op.p2_sptr[warp], e1 = op.p2_sptr[warp + 1];
      constexpr int U = 2;
      for (int e = e0 + lane; e < e1; e += 32 * U) {
        int cl[U];
        double2 mk[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int ee = e + 32 * u;
          const bool ok = ee < e1;
          cl[u] = ok ? op.p2_scol[ee] : -1;
          mk[u] = ok ? op.p2_smk[ee] : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (cl[u] < 0) continue;
#pragma unroll
          for (int t = 0; t < S; ++t)
#pragma unroll
            for (int d = 0; d < 3; ++d) {
              const double v = x[t * sd + 3 * cl[u] + d];
              mu[t][d] = fma(mk[u].x, v, mu[t][d]);
              ku[t][d] = fma(mk[u].y, v, ku[t][d]);
            }
        }
      }
      const int f0 = op.b_sptr[warp], f1 = op.b_sptr[warp + 1];
      for (int e = f0 + lane; e < f1; e += 32) {
        const int q = op.b_scol[e];
        const double bx = bsv[3L * e], by = bsv[3L * e + 1], bz = bsv[3L * e + 2];
#pragma unroll
        for (int t = 0; t < S; ++t) {
          const double pv = x[t * sd + nu + q];
          ku[t][0] = fma(bx, pv, ku[t][0]);
          ku[t][1] = fma(by, pv, ku[t][1]);
          ku[t][2] = fma(bz, pv, ku[t][2]);
        }
      }
    }
    if (!valid) return;
#pragma unroll
    for (int i = 0; i < S; ++i)
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const long o = i * sd + 3L * n + d;
        double y;
        if (fixed) {
          y = x[o];
        } else {
          double acc = 0.0;
#pragma unroll
          for (int t = 0; t < S; ++t) acc = fma(op.a[i * S + t], ku[t][d], acc);
          y = fma(op.dt, acc, mu[i][d]);
        }
        out[o] = b ? b[o] - y : y;
      }
  } else {
    const int ws = warp - nslice_v;
    const int q = (ws << 5) + lane;
    if (ws >= ((op.n_p + 31) >> 5)) return;
    double btu[S];
#pragma unroll
    for (int t = 0; t < S; ++t) btu[t] = 0.0;
    const int e0 = op.bt_sptr[ws], e1 = op.bt_sptr[ws + 1];
    for (int e = e0 + lane; e < e1; e += 32) {
      const int nn = op.bt_scol[e];
      const double bx = btv[3L * e], by = btv[3L * e + 1], bz = btv[3L * e + 2];
#pragma unroll
      for (int t = 0; t < S; ++t) {
        const double* xv = x + t * sd + 3L * nn;
        btu[t] = fma(bx, xv[0], btu[t]);
        btu[t] = fma(by, xv[1], btu[t]);
        btu[t] = fma(bz, xv[2], btu[t]);
      }
    }
    if (q >= op.n_p) return;
#pragma unroll
    for (int i = 0; i < S; ++i) {
      double acc = 0.0;
#pragma unroll
      for (int t = 0; t < S; ++t) acc = fma(op.a[i * S + t], btu[t], acc);
      const double y = __dmul_rn(op.dt, acc);  // (no contraction with b - y)
      const long o = i * sd + nu + q;
      out[o] = b ? b[o] - y : y;
    }
  }
}

// ---- K1 tiled (2-D Stokes, NC = 0): one CTA per tile of the plan built by
// k1tiles.py (ivk_k1_tiles in ivk.h).  Thread 0 reads the tile's 32-byte
// record and issues three TMA bulk copies: the metadata blob (staged-node
// lists, slice table, row ids) and the tile's whole entry stream (values and
// 16-bit local columns) -- so all of the tile's HBM bytes are in flight at
// once and no thread waits on a dependent index -> value -> gather chain.
// When the blob lands, all threads stage the velocity / pressure values the
// tile reads (all S stages, from the L2-resident x) into shared memory and
// prefetch their rows' b; then every gather is a shared-memory load.  One
// thread per scalar node (both components, all stages) or per P1 node; a
// row's entries keep their CSR order, so each sum equals the SELL kernel's
// bit for bit.
#ifndef IVK_K1T_U
#define IVK_K1T_U 4
#endif
#ifndef IVK_K1T_MAXW
#define IVK_K1T_MAXW 16   // warps per CTA (cap)
#endif

struct TileParams {
  const int4* __restrict__ tile_rec;   // 2 per tile
  const int32_t* __restrict__ blob;
  const uint16_t* __restrict__ ecol;
  const double2* __restrict__ eval;
  int max_u, max_p, max_ent, max_blob;
};

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

template <int S>
__global__ void __launch_bounds__(32 * IVK_K1T_MAXW)
    stage_apply_tile_kernel(OpParams op, TileParams tp, const double* __restrict__ x,
                            const double* b, double* out) {
  extern __shared__ __align__(16) unsigned char k1t_smem[];
  constexpr int U = IVK_K1T_U;
  // shared: [entry values][xs: S x nu_t (u_x, u_y)][ps: S x np_t][entry columns][blob][mbarriers]
  double2* vals_s = reinterpret_cast<double2*>(k1t_smem);
  double2* xs = vals_s + tp.max_ent;
  double* ps = reinterpret_cast<double*>(xs + S * tp.max_u);
  uint16_t* cols_s = reinterpret_cast<uint16_t*>(ps + ((S * tp.max_p + 1) & ~1));
  int32_t* blob = reinterpret_cast<int32_t*>(cols_s + ((tp.max_ent + 7) & ~7));
  uint64_t* bars = reinterpret_cast<uint64_t*>(blob + ((tp.max_blob + 3) & ~3));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  if (threadIdx.x == 0) {
    const int4 r0 = tp.tile_rec[2 * blockIdx.x];  // blob offset, blob words, entry offset, entries
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_expect_tx(&bars[0], (uint32_t)r0.y * 4u);
    bulk_copy(blob, tp.blob + r0.x, (uint32_t)r0.y * 4u, &bars[0]);
    mbar_expect_tx(&bars[1], (uint32_t)r0.w * 18u);
    if (r0.w) {
      bulk_copy(vals_s, tp.eval + r0.z, (uint32_t)r0.w * 16u, &bars[1]);
      bulk_copy(cols_s, tp.ecol + r0.z, (uint32_t)r0.w * 2u, &bars[1]);
    }
  }
  __syncthreads();  // barriers initialised
  mbar_wait(&bars[0], 0);
  const int nu_t = blob[0], np_t = blob[1], ns = blob[2];
  const int32_t* ulist = blob + 8;
  const int32_t* plist = ulist + nu_t;
  const int4* slices = reinterpret_cast<const int4*>(blob + ((8 + nu_t + np_t + 3) & ~3));
  const int32_t* rows = reinterpret_cast<const int32_t*>(slices + ns);
  const int nu = 2 * op.n_nodes;
  const long sd = nu + op.n_p;
#pragma unroll 2
  for (int i = threadIdx.x; i < nu_t; i += blockDim.x) {
    const long node = ulist[i];
    double2 v[S];
#pragma unroll
    for (int t = 0; t < S; ++t)  // (stage offsets may be odd: no 16-byte loads)
      v[t] = make_double2(x[t * sd + 2 * node], x[t * sd + 2 * node + 1]);
#pragma unroll
    for (int t = 0; t < S; ++t) xs[t * nu_t + i] = v[t];
  }
  for (int i = threadIdx.x; i < np_t; i += blockDim.x) {
    const long q = plist[i];
#pragma unroll
    for (int t = 0; t < S; ++t) ps[t * np_t + i] = x[t * sd + nu + q];
  }
  // the first slice's right-hand side, in flight during the barrier waits
  double bb[S][2];
  {
    const int rid = warp < ns ? rows[warp * 32 + lane] : -1;
    const bool vel = warp < ns && slices[warp].w == 0;
#pragma unroll
    for (int i = 0; i < S; ++i) bb[i][0] = bb[i][1] = 0.0;
    if (b && rid != -1) {
      if (vel) {
        const long n = rid < -1 ? -(rid + 2) : rid;
#pragma unroll
        for (int i = 0; i < S; ++i) {
          bb[i][0] = b[i * sd + 2 * n];
          bb[i][1] = b[i * sd + 2 * n + 1];
        }
      } else {
#pragma unroll
        for (int i = 0; i < S; ++i) bb[i][0] = b[i * sd + nu + rid];
      }
    }
  }
  __syncthreads();
  mbar_wait(&bars[1], 0);
  for (int s = warp; s < ns; s += nw) {
    const int4 sl = slices[s];  // entry offset in the tile, wa, wb, kind
    const int rid = rows[s * 32 + lane];
    const uint16_t* ec = cols_s + sl.x + lane;
    const double2* ev = vals_s + sl.x + lane;
    if (s != warp && b && rid != -1) {  // (more slices than warps: load b now)
      if (sl.w == 0) {
        const long n = rid < -1 ? -(rid + 2) : rid;
#pragma unroll
        for (int i = 0; i < S; ++i) {
          bb[i][0] = b[i * sd + 2 * n];
          bb[i][1] = b[i * sd + 2 * n + 1];
        }
      } else {
#pragma unroll
        for (int i = 0; i < S; ++i) bb[i][0] = b[i * sd + nu + rid];
      }
    }
    if (sl.w == 0) {
      double mu[S][2], ku[S][2];
#pragma unroll
      for (int t = 0; t < S; ++t) mu[t][0] = mu[t][1] = ku[t][0] = ku[t][1] = 0.0;
#pragma unroll U
      for (int e = 0; e < sl.y; ++e) {
        const int c = ec[e * 32];
        const double2 v = ev[e * 32];
#pragma unroll
        for (int t = 0; t < S; ++t) {
          const double2 xv = xs[t * nu_t + c];
          mu[t][0] = fma(v.x, xv.x, mu[t][0]);
          mu[t][1] = fma(v.x, xv.y, mu[t][1]);
          ku[t][0] = fma(v.y, xv.x, ku[t][0]);
          ku[t][1] = fma(v.y, xv.y, ku[t][1]);
        }
      }
      ec += sl.y * 32;
      ev += sl.y * 32;
#pragma unroll U
      for (int e = 0; e < sl.z; ++e) {
        const int c = ec[e * 32];
        const double2 v = ev[e * 32];
#pragma unroll
        for (int t = 0; t < S; ++t) {
          const double pv = ps[t * np_t + c];
          ku[t][0] = fma(v.x, pv, ku[t][0]);
          ku[t][1] = fma(v.y, pv, ku[t][1]);
        }
      }
      if (rid == -1) continue;
      const bool fixed = rid < -1;
      const long n = fixed ? -(rid + 2) : rid;
#pragma unroll
      for (int i = 0; i < S; ++i)
#pragma unroll
        for (int d = 0; d < 2; ++d) {
          const long o = i * sd + 2 * n + d;
          double y;
          if (fixed) {
            y = x[o];
          } else {
            double acc = 0.0;
#pragma unroll
            for (int t = 0; t < S; ++t) acc = fma(op.a[i * S + t], ku[t][d], acc);
            y = fma(op.dt, acc, mu[i][d]);
          }
          out[o] = b ? bb[i][d] - y : y;
        }
    } else {
      double btu[S];
#pragma unroll
      for (int t = 0; t < S; ++t) btu[t] = 0.0;
#pragma unroll U
      for (int e = 0; e < sl.y; ++e) {
        const int c = ec[e * 32];
        const double2 v = ev[e * 32];
#pragma unroll
        for (int t = 0; t < S; ++t) {
          const double2 xv = xs[t * nu_t + c];
          btu[t] = fma(v.x, xv.x, btu[t]);
          btu[t] = fma(v.y, xv.y, btu[t]);
        }
      }
      if (rid < 0) continue;
#pragma unroll
      for (int i = 0; i < S; ++i) {
        double acc = 0.0;
#pragma unroll
        for (int t = 0; t < S; ++t) acc = fma(op.a[i * S + t], btu[t], acc);
        const double y = __dmul_rn(op.dt, acc);  // (no contraction with b - y)
        out[i * sd + nu + rid] = b ? bb[i][0] - y : y;
      }
    }
  }
}

static size_t k1t_smem_bytes(int S, const ivk_k1_tiles* tl) {
  const size_t ent = (size_t)tl->max_ent;
  return 16 * ent + (size_t)S * 16 * tl->max_u + 8 * (((size_t)S * tl->max_p + 1) & ~(size_t)1) +
         2 * ((ent + 7) & ~(size_t)7) + 4 * (((size_t)tl->max_blob + 3) & ~(size_t)3) + 16;
}

template <int S>
static int launch_stage_apply_tiles(const OpParams& q, const ivk_k1_tiles* tl, const double* x,
                                    const double* b, double* out, cudaStream_t st) {
  TileParams tp;
  tp.tile_rec = reinterpret_cast<const int4*>(tl->tile_rec);
  tp.blob = tl->blob;
  tp.ecol = tl->ecol;
  tp.eval = reinterpret_cast<const double2*>(tl->eval);
  tp.max_u = tl->max_u;
  tp.max_p = tl->max_p;
  tp.max_ent = tl->max_ent;
  tp.max_blob = tl->max_blob;
  const size_t smem = k1t_smem_bytes(S, tl);
  IVK_REQUIRE(smem <= 220 * 1024, "K1 tile plan needs %zu bytes of shared memory", smem);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(stage_apply_tile_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
  int warps = tl->max_slices < IVK_K1T_MAXW ? tl->max_slices : IVK_K1T_MAXW;
  if (warps < 1) warps = 1;
  stage_apply_tile_kernel<S><<<tl->n_tiles, 32 * warps, smem, st>>>(q, tp, x, b, out);
  return IVK_OK;
}

template <int S>
static void launch_stage_apply(const OpParams& q, int nconv, int ncomp, const double* x,
                               const double* b, double* out, const int32_t* slices, int n_slices,
                               cudaStream_t st) {
  const OpParams& p = q;
  const int node_rows = ncomp == 3 ? 32 : 16;
  const long warps = slices ? n_slices
                            : (p.n_nodes + node_rows - 1) / node_rows + ((p.n_p + 31) >> 5);
  const int block = 256;
  const int grid = (int)((warps * 32 + block - 1) / block);
  if (ncomp == 3) {
    if (slices)
      stage_apply3_kernel<S, true><<<grid, block, 0, st>>>(q, x, b, out, slices, n_slices);
    else
      stage_apply3_kernel<S, false><<<grid, block, 0, st>>>(q, x, b, out, nullptr, 0);
    return;
  }
  if (slices) {
    if (nconv == 0)
      stage_apply_kernel<S, 0, true><<<grid, block, 0, st>>>(q, x, b, out, slices, n_slices);
    else if (nconv == 1)
      stage_apply_kernel<S, 1, true><<<grid, block, 0, st>>>(q, x, b, out, slices, n_slices);
    else
      stage_apply_kernel<S, S, true><<<grid, block, 0, st>>>(q, x, b, out, slices, n_slices);
    return;
  }
  if (nconv == 0)
    stage_apply_kernel<S, 0, false><<<grid, block, 0, st>>>(q, x, b, out, nullptr, 0);
  else if (nconv == 1)
    stage_apply_kernel<S, 1, false><<<grid, block, 0, st>>>(q, x, b, out, nullptr, 0);
  else
    stage_apply_kernel<S, S, false><<<grid, block, 0, st>>>(q, x, b, out, nullptr, 0);
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

// Pressure-mean projection over (IVK_PROJECT_BLOCKS, stages) CTAs: phase 1
// writes one partial sum per CTA (block-strided slice, fixed-order tree),
// phase 2 has every CTA sum its stage's partials in index order -- the same
// bits on every CTA -- and subtract the mean from its slice.
constexpr int kProjThreads = 256;

__device__ __forceinline__ double block_sum(double acc, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  double v = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < kProjThreads / 32; ++w) v += red[w];
  return v;  // valid in thread 0
}

__global__ void __launch_bounds__(kProjThreads) project_partial_kernel(int n_u, int n_p,
                                                                       const double* x,
                                                                       double* partial) {
  __shared__ double red[kProjThreads / 32];
  const long sd = (long)n_u + n_p;
  const double* p = x + blockIdx.y * sd + n_u;
  double acc = 0.0;
  for (int i = blockIdx.x * kProjThreads + threadIdx.x; i < n_p; i += gridDim.x * kProjThreads)
    acc += p[i];
  const double v = block_sum(acc, red);
  if (threadIdx.x == 0) partial[blockIdx.y * gridDim.x + blockIdx.x] = v;
}

__global__ void __launch_bounds__(kProjThreads) project_subtract_kernel(int n_u, int n_p,
                                                                        double* x,
                                                                        const double* partial) {
  __shared__ double mean;
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int b = 0; b < (int)gridDim.x; ++b) s += partial[blockIdx.y * gridDim.x + b];
    mean = s / (double)n_p;
  }
  __syncthreads();
  const long sd = (long)n_u + n_p;
  double* p = x + blockIdx.y * sd + n_u;
  const double m = mean;
  for (int i = blockIdx.x * kProjThreads + threadIdx.x; i < n_p; i += gridDim.x * kProjThreads)
    p[i] -= m;
}

__global__ void seed_constrained_kernel(int S, int n_nodes, int nc, int n_p,
                                        const uint8_t* __restrict__ cm,
                                        const double* __restrict__ src, double* __restrict__ out) {
  const long nu = (long)nc * n_nodes;
  const long sd = nu + n_p;
  const long total = S * sd;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total;
       i += (long)gridDim.x * blockDim.x) {
    const long loc = i % sd;
    double v = 0.0;
    if (loc < nu && cm[loc / nc]) v = src[i];
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

static int stage_apply(const ivk_operator_desc* op, const int32_t* slices, int32_t n_slices,
                       const double* x, const double* b, double* out, void* stream) {
  int rc = validate_op(op);
  if (rc) return rc;
  IVK_REQUIRE(x && out, "x/out is NULL");
  IVK_REQUIRE(out != x, "out must not alias x");
  OpParams p = make_op_params(op);
  cudaStream_t st = as_stream(stream);
  if (op->k1_tiles && !slices && op->n_conv == 0 && op->ncomp != 3) {
    const ivk_k1_tiles* tl = op->k1_tiles;
    IVK_REQUIRE(tl->n_tiles > 0 && tl->tile_rec && tl->blob && tl->ecol && tl->eval,
                "K1 tile plan has a NULL array");
    switch (op->stages) {
      case 1: rc = launch_stage_apply_tiles<1>(p, tl, x, b, out, st); break;
      case 2: rc = launch_stage_apply_tiles<2>(p, tl, x, b, out, st); break;
      case 3: rc = launch_stage_apply_tiles<3>(p, tl, x, b, out, st); break;
    }
    if (rc) return rc;
    return check_launch("ivk_stage_apply (tiles)");
  }
  if (!slices && op->k1_order && op->k1_order_n > 0 && op->ncomp != 3) {
    // a locality order over ALL slices (stages.py): same kernel, same sums
    slices = op->k1_order;
    n_slices = op->k1_order_n;
  }
  switch (op->stages) {
    case 1: launch_stage_apply<1>(p, op->n_conv, op->ncomp, x, b, out, slices, n_slices, st); break;
    case 2: launch_stage_apply<2>(p, op->n_conv, op->ncomp, x, b, out, slices, n_slices, st); break;
    case 3: launch_stage_apply<3>(p, op->n_conv, op->ncomp, x, b, out, slices, n_slices, st); break;
  }
  return check_launch("ivk_stage_apply");
}

int ivk_stage_apply(const ivk_operator_desc* op, const double* x, const double* b, double* out,
                    void* stream) {
  return stage_apply(op, nullptr, 0, x, b, out, stream);
}

int ivk_stage_apply_slices(const ivk_operator_desc* op, const int32_t* slices, int32_t n_slices,
                           const double* x, const double* b, double* out, void* stream) {
  IVK_REQUIRE(slices != nullptr && n_slices >= 0, "bad slice list");
  if (n_slices == 0) return IVK_OK;
  return stage_apply(op, slices, n_slices, x, b, out, stream);
}

__global__ void index_copy_kernel(int64_t n, const int32_t* __restrict__ src_idx,
                                  const double* __restrict__ src, const int32_t* __restrict__ dst_idx,
                                  double* __restrict__ dst, double beta) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double v = src[src_idx ? src_idx[i] : i];
    const int64_t o = dst_idx ? dst_idx[i] : i;
    dst[o] = beta == 0.0 ? v : fma(beta, dst[o], v);
  }
}

__global__ void index_update_kernel(int64_t n, const int32_t* __restrict__ idx, double alpha,
                                    const double* __restrict__ x, double beta,
                                    const double* __restrict__ w, const double* __restrict__ z,
                                    double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int d = idx[i];
    double v = beta * (w ? w[d] : 1.0) * z[d];
    if (x) v = alpha * x[d] + v;
    out[d] = v;
  }
}

int ivk_index_copy(int64_t n, const int32_t* src_idx, const double* src, const int32_t* dst_idx,
                   double* dst, double beta, void* stream) {
  IVK_REQUIRE(n >= 0 && src && dst, "bad index_copy arguments");
  if (n == 0) return IVK_OK;
  index_copy_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(n, src_idx, src, dst_idx, dst,
                                                                     beta);
  return check_launch("ivk_index_copy");
}

int ivk_index_update(int64_t n, const int32_t* idx, double alpha, const double* x, double beta,
                     const double* w, const double* z, double* out, void* stream) {
  IVK_REQUIRE(n >= 0 && idx && z && out, "bad index_update arguments");
  if (n == 0) return IVK_OK;
  index_update_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(n, idx, alpha, x, beta, w,
                                                                       z, out);
  return check_launch("ivk_index_update");
}

int ivk_axpby(int64_t n, double alpha, const double* x, double beta, const double* y, double* out,
              void* stream) {
  IVK_REQUIRE(out != nullptr && n >= 0, "bad axpby arguments");
  if (n == 0) return IVK_OK;
  axpby_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(n, alpha, x, beta, y, out);
  return check_launch("ivk_axpby");
}

int ivk_project_pressure_means(int32_t stages, int32_t n_u, int32_t n_p, double* x,
                               double* scratch, void* stream) {
  IVK_REQUIRE(x && scratch && stages >= 1 && n_p > 0 && n_u >= 0, "bad projection arguments");
  // small n_p (coarse levels, tests): fewer CTAs so none is empty
  int nb = (n_p + kProjThreads - 1) / kProjThreads;
  if (nb > IVK_PROJECT_BLOCKS) nb = IVK_PROJECT_BLOCKS;
  const dim3 grid(nb, stages);
  cudaStream_t st = as_stream(stream);
  project_partial_kernel<<<grid, kProjThreads, 0, st>>>(n_u, n_p, x, scratch);
  int rc = check_launch("ivk_project_pressure_means");
  if (rc) return rc;
  project_subtract_kernel<<<grid, kProjThreads, 0, st>>>(n_u, n_p, x, scratch);
  return check_launch("ivk_project_pressure_means");
}

int ivk_seed_constrained(int32_t stages, int32_t n_nodes, int32_t ncomp, int32_t n_p,
                         const uint8_t* cm, const double* src, double* out, void* stream) {
  IVK_REQUIRE(cm && src && out && stages >= 1 && (ncomp == 2 || ncomp == 3),
              "bad seed arguments");
  const long total = (long)stages * ((long)ncomp * n_nodes + n_p);
  seed_constrained_kernel<<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(
      stages, n_nodes, ncomp, n_p, cm, src, out);
  return check_launch("ivk_seed_constrained");
}

}  // extern "C"
