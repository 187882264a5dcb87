// K10: convection Jacobian (and residual) assembly on the device, for the
// Navier-Stokes / Oseen linearisation at Newton cadence.
//
// Reference: fem.assemble_convection (fem.py:199-242), both Newton terms
//   J[(a,d),(b,f)] = <phi_a phi_b, d_f u_d> + delta_df <phi_a, u . grad phi_b>
//   N(u)[(a,d)]    = <phi_a, (u . grad) u_d>
// Phase 1: one thread per (cell, row node) evaluates a 1x6 row of 2x2 blocks
// of the element Jacobian at the degree-5 collapsed rule (quadrature tables
// passed by value).
// Phase 2: one thread per scalar-pattern entry sums its cell contributions
// in a fixed (cell-ascending) order -- deterministic, no atomics -- applies
// the Dirichlet elimination and writes both the CSR and the SELL copy the
// operator kernels read.  Patch matrices are then refactorised in place by K7.

#include "ivk_common.cuh"

namespace ivk {

struct QuadTable {
  int nq;
  double w[IVK_MAX_QUAD];
  double phi[IVK_MAX_QUAD][6];
  double dphi[IVK_MAX_QUAD][6][2];
};

// One thread per (cell, local row node a): the six 2x2 blocks J[a][b] and
// N[a] (the per-point field values are recomputed by each of the 6 threads).
__global__ void __launch_bounds__(192) convection_element_kernel(
    int n_cells, const int32_t* __restrict__ cell_nodes, const double* __restrict__ cell_geo,
    const double* __restrict__ u, QuadTable qt, double* __restrict__ jel,
    double* __restrict__ nel) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int c = tid / 6, a = tid - 6 * (tid / 6);
  if (c >= n_cells) return;
  double ul[6][2];
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    const int n = cell_nodes[c * 6 + k];
    ul[k][0] = u[2 * n];
    ul[k][1] = u[2 * n + 1];
  }
  // Jinv (row-major [e][d]) and det J
  const double i00 = cell_geo[c * 5 + 0], i01 = cell_geo[c * 5 + 1];
  const double i10 = cell_geo[c * 5 + 2], i11 = cell_geo[c * 5 + 3];
  const double det = cell_geo[c * 5 + 4];
  double J[6][4];
  double N0 = 0.0, N1 = 0.0;
#pragma unroll
  for (int b = 0; b < 6; ++b) J[b][0] = J[b][1] = J[b][2] = J[b][3] = 0.0;
  for (int q = 0; q < qt.nq; ++q) {
    double G[6][2];
    double uq0 = 0.0, uq1 = 0.0, g00 = 0.0, g01 = 0.0, g10 = 0.0, g11 = 0.0;
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      const double d0 = qt.dphi[q][k][0], d1 = qt.dphi[q][k][1];
      G[k][0] = d0 * i00 + d1 * i10;
      G[k][1] = d0 * i01 + d1 * i11;
      const double ph = qt.phi[q][k];
      uq0 += ul[k][0] * ph;
      uq1 += ul[k][1] * ph;
      g00 += ul[k][0] * G[k][0];  // d_0 u_0
      g01 += ul[k][0] * G[k][1];  // d_1 u_0
      g10 += ul[k][1] * G[k][0];  // d_0 u_1
      g11 += ul[k][1] * G[k][1];  // d_1 u_1
    }
    const double wpa = qt.w[q] * qt.phi[q][a];
    N0 += wpa * (uq0 * g00 + uq1 * g01);  // (u . grad) u_0
    N1 += wpa * (uq0 * g10 + uq1 * g11);
#pragma unroll
    for (int b = 0; b < 6; ++b) {
      const double wpp = wpa * qt.phi[q][b];
      const double adv = wpa * (uq0 * G[b][0] + uq1 * G[b][1]);
      J[b][0] += wpp * g00 + adv;
      J[b][1] += wpp * g01;
      J[b][2] += wpp * g10;
      J[b][3] += wpp * g11 + adv;
    }
  }
  double* out = jel + ((long)c * 36 + a * 6) * 4;
#pragma unroll
  for (int b = 0; b < 6; ++b)
#pragma unroll
    for (int k = 0; k < 4; ++k) out[b * 4 + k] = J[b][k] * det;
  if (nel) {
    nel[(long)c * 12 + 2 * a] = N0 * det;
    nel[(long)c * 12 + 2 * a + 1] = N1 * det;
  }
}

// J on the scalar pattern: entry e sums contributions contrib[ptr[e]..ptr[e+1])
// (index cell*36 + a*6 + b, cell-ascending), eliminated, to CSR and SELL.
__global__ void convection_gather_kernel(int nnz, const int32_t* __restrict__ ptr,
                                         const int32_t* __restrict__ contrib,
                                         const double4* __restrict__ jel,
                                         const int32_t* __restrict__ row_of,
                                         const int32_t* __restrict__ col,
                                         const uint8_t* __restrict__ cmask,
                                         const int32_t* __restrict__ sell_pos, double4* conv,
                                         double4* conv_s) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nnz) return;
  double4 s = make_double4(0.0, 0.0, 0.0, 0.0);
  if (!(cmask[row_of[e]] || cmask[col[e]])) {
    for (int k = ptr[e]; k < ptr[e + 1]; ++k) {
      const double4 v = jel[contrib[k]];
      s.x += v.x;
      s.y += v.y;
      s.z += v.z;
      s.w += v.w;
    }
  }
  if (conv) conv[e] = s;
  if (conv_s) conv_s[sell_pos[e]] = s;
}

// N(u) per scalar node: contributions node_contrib (cell*6 + a, ascending).
__global__ void convection_residual_kernel(int n_nodes, const int32_t* __restrict__ ptr,
                                           const int32_t* __restrict__ contrib,
                                           const double2* __restrict__ nel,
                                           double2* __restrict__ res) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= n_nodes) return;
  double2 s = make_double2(0.0, 0.0);
  for (int k = ptr[n]; k < ptr[n + 1]; ++k) {
    const double2 v = nel[contrib[k]];
    s.x += v.x;
    s.y += v.y;
  }
  res[n] = s;
}

}  // namespace ivk

using namespace ivk;

extern "C" {

int ivk_convection_assemble(const ivk_convection_desc* d, const double* u, double* elem_scratch,
                            double* conv, double* conv_s, double* residual, void* stream) {
  IVK_REQUIRE(d && u && elem_scratch, "bad convection assembly arguments");
  IVK_REQUIRE(d->quad && d->quad->nq > 0 && d->quad->nq <= IVK_MAX_QUAD, "bad quadrature table");
  IVK_REQUIRE(d->cell_nodes && d->cell_geo && d->entry_ptr && d->entry_contrib && d->row_of &&
                  d->col && d->node_constrained,
              "convection descriptor has a NULL array");
  IVK_REQUIRE(!conv_s || d->sell_pos, "SELL output needs sell_pos");
  IVK_REQUIRE(!residual || (d->node_ptr && d->node_contrib), "residual needs the node map");
  QuadTable qt;
  qt.nq = d->quad->nq;
  for (int q = 0; q < qt.nq; ++q) {
    qt.w[q] = d->quad->w[q];
    for (int a = 0; a < 6; ++a) {
      qt.phi[q][a] = d->quad->phi[q * 6 + a];
      qt.dphi[q][a][0] = d->quad->dphi[(q * 6 + a) * 2];
      qt.dphi[q][a][1] = d->quad->dphi[(q * 6 + a) * 2 + 1];
    }
  }
  cudaStream_t st = as_stream(stream);
  double* nel = residual ? elem_scratch + (long)d->n_cells * 144 : nullptr;
  convection_element_kernel<<<(int)(((long)d->n_cells * 6 + 191) / 192), 192, 0, st>>>(
      d->n_cells, d->cell_nodes, d->cell_geo, u, qt, elem_scratch, nel);
  int rc = check_launch("ivk_convection_assemble(element)");
  if (rc) return rc;
  convection_gather_kernel<<<(d->nnz + 255) / 256, 256, 0, st>>>(
      d->nnz, d->entry_ptr, d->entry_contrib, reinterpret_cast<const double4*>(elem_scratch),
      d->row_of, d->col, d->node_constrained, d->sell_pos, reinterpret_cast<double4*>(conv),
      reinterpret_cast<double4*>(conv_s));
  rc = check_launch("ivk_convection_assemble(gather)");
  if (rc || !residual) return rc;
  convection_residual_kernel<<<(d->n_nodes + 255) / 256, 256, 0, st>>>(
      d->n_nodes, d->node_ptr, d->node_contrib, reinterpret_cast<const double2*>(nel),
      reinterpret_cast<double2*>(residual));
  return check_launch("ivk_convection_assemble(residual)");
}

}  // extern "C"
