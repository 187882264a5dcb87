// K5: nested P2/P1 grid transfers I_s (x) blockdiag(P_P2 (x) I_2, P_P1) and
// the transpose, as deterministic row-gather kernels (the transpose is stored
// explicitly), one thread per scalar node for all NC velocity components (2,
// or 3 for the 3-D Kuhn meshes) and all stages.
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
template <int S, bool ADD, int NC>
__global__ void __launch_bounds__(256) transfer_kernel(
    int n_dst_nodes, int n_dst_p, int n_src_nodes, int n_src_p, const int32_t* __restrict__ v_ptr,
    const int32_t* __restrict__ v_col, const double* __restrict__ v_val,
    const int32_t* __restrict__ p_ptr, const int32_t* __restrict__ p_col,
    const double* __restrict__ p_val, const uint8_t* __restrict__ dst_cm,
    const double* __restrict__ src, double* __restrict__ dst) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  const long sd_dst = (long)NC * n_dst_nodes + n_dst_p;
  const long sd_src = (long)NC * n_src_nodes + n_src_p;
  if (row < n_dst_nodes) {
    const bool fixed = dst_cm[row] != 0;
    if (ADD && fixed) return;
    double acc[S][NC];
#pragma unroll
    for (int t = 0; t < S; ++t)
#pragma unroll
      for (int d = 0; d < NC; ++d) acc[t][d] = 0.0;
    if (!fixed) {
      for (int e = v_ptr[row]; e < v_ptr[row + 1]; ++e) {
        const int c = v_col[e];
        const double w = v_val[e];
#pragma unroll
        for (int t = 0; t < S; ++t)
#pragma unroll
          for (int d = 0; d < NC; ++d)
            acc[t][d] = fma(w, src[t * sd_src + (long)NC * c + d], acc[t][d]);
      }
    }
#pragma unroll
    for (int t = 0; t < S; ++t) {
      double* o = dst + t * sd_dst + (long)NC * row;
#pragma unroll
      for (int d = 0; d < NC; ++d) {
        if (ADD) o[d] += acc[t][d];
        else o[d] = acc[t][d];
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
      for (int t = 0; t < S; ++t)
        acc[t] = fma(w, src[t * sd_src + (long)NC * n_src_nodes + c], acc[t]);
    }
#pragma unroll
    for (int t = 0; t < S; ++t) {
      double* o = dst + t * sd_dst + (long)NC * n_dst_nodes + q;
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
  IVK_REQUIRE(t->ncomp == 0 || t->ncomp == 2 || t->ncomp == 3, "ncomp must be 2 or 3");
  return IVK_OK;
}

template <bool ADD, int NC>
static void launch_transfer_nc(int S, int nd, int ndp, int ns, int nsp, const int32_t* vp,
                               const int32_t* vc, const double* vv, const int32_t* pp,
                               const int32_t* pc, const double* pv, const uint8_t* cm,
                               const double* src, double* dst, cudaStream_t st) {
  const int rows = nd + ndp;
  const int grid = (rows + 255) / 256;
  switch (S) {
    case 1: transfer_kernel<1, ADD, NC><<<grid, 256, 0, st>>>(nd, ndp, ns, nsp, vp, vc, vv, pp, pc, pv, cm, src, dst); break;
    case 2: transfer_kernel<2, ADD, NC><<<grid, 256, 0, st>>>(nd, ndp, ns, nsp, vp, vc, vv, pp, pc, pv, cm, src, dst); break;
    default: transfer_kernel<3, ADD, NC><<<grid, 256, 0, st>>>(nd, ndp, ns, nsp, vp, vc, vv, pp, pc, pv, cm, src, dst); break;
  }
}

template <bool ADD>
static void launch_transfer(int S, int ncomp, int nd, int ndp, int ns, int nsp,
                            const int32_t* vp, const int32_t* vc, const double* vv,
                            const int32_t* pp, const int32_t* pc, const double* pv,
                            const uint8_t* cm, const double* src, double* dst, cudaStream_t st) {
  if (ncomp == 3)
    launch_transfer_nc<ADD, 3>(S, nd, ndp, ns, nsp, vp, vc, vv, pp, pc, pv, cm, src, dst, st);
  else
    launch_transfer_nc<ADD, 2>(S, nd, ndp, ns, nsp, vp, vc, vv, pp, pc, pv, cm, src, dst, st);
}

}  // namespace ivk

using namespace ivk;

extern "C" {

int ivk_restrict(const ivk_transfer_desc* t, const double* rf, double* rc, void* stream) {
  int e = validate_transfer(t);
  if (e) return e;
  IVK_REQUIRE(rf && rc && rf != rc, "bad restrict vectors");
  launch_transfer<false>(t->stages, t->ncomp, t->nc_nodes, t->nc_p, t->nf_nodes, t->nf_p, t->p2t_rowptr,
                         t->p2t_col, t->p2t_val, t->p1t_rowptr, t->p1t_col, t->p1t_val,
                         t->coarse_constrained, rf, rc, as_stream(stream));
  return check_launch("ivk_restrict");
}

int ivk_prolong_add(const ivk_transfer_desc* t, const double* ec, double* xf, void* stream) {
  int e = validate_transfer(t);
  if (e) return e;
  IVK_REQUIRE(ec && xf && ec != xf, "bad prolong vectors");
  launch_transfer<true>(t->stages, t->ncomp, t->nf_nodes, t->nf_p, t->nc_nodes, t->nc_p, t->p2_rowptr,
                        t->p2_col, t->p2_val, t->p1_rowptr, t->p1_col, t->p1_val,
                        t->fine_constrained, ec, xf, as_stream(stream));
  return check_launch("ivk_prolong_add");
}

}  // extern "C"
