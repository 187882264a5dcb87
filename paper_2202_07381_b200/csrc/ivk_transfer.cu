// K5: nested P2/P1 grid transfers I_s (x) blockdiag(P_P2 (x) I_2, P_P1) and
// the transpose, as deterministic row-gather kernels (the transpose is stored
// explicitly), one thread per scalar node for both components and all stages.
//
// Reference: MGHierarchyOp.vcycle (solvers.py:340-346)
//   rc = P^T r; rc[constrained_c] = 0; ... corr = P ec; corr[constrained_f] = 0; x += corr
// with P = Discretization.stage_prolong (bench.py:187-194).

#include "ivk_common.cuh"

namespace ivk {

struct TransferParams {
  int S, nf_nodes, nf_p, nc_nodes, nc_p;
  const int32_t* __restrict__ p2_rowptr;
  const int32_t* __restrict__ p2_col;
  const double* __restrict__ p2_val;
  const int32_t* __restrict__ p2t_rowptr;
  const int32_t* __restrict__ p2t_col;
  const double* __restrict__ p2t_val;
  const int32_t* __restrict__ p1_rowptr;
  const int32_t* __restrict__ p1_col;
  const double* __restrict__ p1_val;
  const int32_t* __restrict__ p1t_rowptr;
  const int32_t* __restrict__ p1t_col;
  const double* __restrict__ p1t_val;
  const uint8_t* __restrict__ fcm;
  const uint8_t* __restrict__ ccm;
};

// dst (n_dst_nodes P2 rows + n_dst_p P1 rows) <- CSR * src, per stage and
// velocity component.  add: dst += result on unconstrained rows (prolong);
// else dst = result, constrained rows zeroed (restrict).
template <int S, bool ADD>
__global__ void __launch_bounds__(256) transfer_kernel(
    int n_dst_nodes, int n_dst_p, int n_src_nodes, int n_src_p, const int32_t* __restrict__ v_ptr,
    const int32_t* __restrict__ v_col, const double* __restrict__ v_val,
    const int32_t* __restrict__ p_ptr, const int32_t* __restrict__ p_col,
    const double* __restrict__ p_val, const uint8_t* __restrict__ dst_cm,
    const double* __restrict__ src, double* __restrict__ dst) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  const long sd_dst = 2L * n_dst_nodes + n_dst_p;
  const long sd_src = 2L * n_src_nodes + n_src_p;
  if (row < n_dst_nodes) {
    const bool fixed = dst_cm[row] != 0;
    if (ADD && fixed) return;
    double acc[S][2];
#pragma unroll
    for (int t = 0; t < S; ++t) acc[t][0] = acc[t][1] = 0.0;
    if (!fixed) {
      for (int e = v_ptr[row]; e < v_ptr[row + 1]; ++e) {
        const int c = v_col[e];
        const double w = v_val[e];
#pragma unroll
        for (int t = 0; t < S; ++t) {
          acc[t][0] = fma(w, src[t * sd_src + 2 * c], acc[t][0]);
          acc[t][1] = fma(w, src[t * sd_src + 2 * c + 1], acc[t][1]);
        }
      }
    }
#pragma unroll
    for (int t = 0; t < S; ++t) {
      double* o = dst + t * sd_dst + 2L * row;
      if (ADD) {
        o[0] += acc[t][0];
        o[1] += acc[t][1];
      } else {
        o[0] = acc[t][0];
        o[1] = acc[t][1];
      }
    }
  } else if (row < n_dst_nodes + n_dst_p) {
    const int q = row - n_dst_nodes;
    double acc[S];
#pragma unroll
    for (int t = 0; t < S; ++t) acc[t] = 0.0;
    for (int e = p_ptr[q]; e < p_ptr[q + 1]; ++e) {
      const int c = p_col[e];
      const double w = p_val[e];
#pragma unroll
      for (int t = 0; t < S; ++t) acc[t] = fma(w, src[t * sd_src + 2L * n_src_nodes + c], acc[t]);
    }
#pragma unroll
    for (int t = 0; t < S; ++t) {
      double* o = dst + t * sd_dst + 2L * n_dst_nodes + q;
      if (ADD) *o += acc[t]; else *o = acc[t];
    }
  }
}

static int validate_transfer(const ivk_transfer_desc* t) {
  IVK_REQUIRE(t != nullptr, "transfer descriptor is NULL");
  IVK_REQUIRE(t->stages >= 1 && t->stages <= IVK_MAX_STAGES, "bad stage count");
  IVK_REQUIRE(t->p2_rowptr && t->p2_col && t->p2_val && t->p2t_rowptr && t->p2t_col && t->p2t_val &&
                  t->p1_rowptr && t->p1_col && t->p1_val && t->p1t_rowptr && t->p1t_col &&
                  t->p1t_val && t->fine_constrained && t->coarse_constrained,
              "transfer descriptor has a NULL array");
  return IVK_OK;
}

template <bool ADD>
static void launch_transfer(int S, int nd, int ndp, int ns, int nsp, const int32_t* vp,
                            const int32_t* vc, const double* vv, const int32_t* pp,
                            const int32_t* pc, const double* pv, const uint8_t* cm,
                            const double* src, double* dst, cudaStream_t st) {
  const int rows = nd + ndp;
  const int grid = (rows + 255) / 256;
  switch (S) {
    case 1: transfer_kernel<1, ADD><<<grid, 256, 0, st>>>(nd, ndp, ns, nsp, vp, vc, vv, pp, pc, pv, cm, src, dst); break;
    case 2: transfer_kernel<2, ADD><<<grid, 256, 0, st>>>(nd, ndp, ns, nsp, vp, vc, vv, pp, pc, pv, cm, src, dst); break;
    default: transfer_kernel<3, ADD><<<grid, 256, 0, st>>>(nd, ndp, ns, nsp, vp, vc, vv, pp, pc, pv, cm, src, dst); break;
  }
}

}  // namespace ivk

using namespace ivk;

extern "C" {

int ivk_restrict(const ivk_transfer_desc* t, const double* rf, double* rc, void* stream) {
  int e = validate_transfer(t);
  if (e) return e;
  IVK_REQUIRE(rf && rc && rf != rc, "bad restrict vectors");
  launch_transfer<false>(t->stages, t->nc_nodes, t->nc_p, t->nf_nodes, t->nf_p, t->p2t_rowptr,
                         t->p2t_col, t->p2t_val, t->p1t_rowptr, t->p1t_col, t->p1t_val,
                         t->coarse_constrained, rf, rc, as_stream(stream));
  return check_launch("ivk_restrict");
}

int ivk_prolong_add(const ivk_transfer_desc* t, const double* ec, double* xf, void* stream) {
  int e = validate_transfer(t);
  if (e) return e;
  IVK_REQUIRE(ec && xf && ec != xf, "bad prolong vectors");
  launch_transfer<true>(t->stages, t->nf_nodes, t->nf_p, t->nc_nodes, t->nc_p, t->p2_rowptr,
                        t->p2_col, t->p2_val, t->p1_rowptr, t->p1_col, t->p1_val,
                        t->fine_constrained, ec, xf, as_stream(stream));
  return check_launch("ivk_prolong_add");
}

}  // extern "C"
