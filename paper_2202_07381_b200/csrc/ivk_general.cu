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

// ---------------------------------------------------------------- K10g
// Element rows of the linearised MHD operator (mhd.py element_matrices, the
// weak form of PAPER.md "MHD semi-discrete"): thread (cell, local row i).
// Local order: w = 4 a + comp (comp 0, 1: u_x, u_y; 2, 3: B_x, B_y), then
// r at the 3 vertices (24..26), p at the 3 vertices (27..29).
struct MhdTables {
  int nq;
  double Re, Rm, S;
  double w[IVK_MHD_MAX_QUAD];
  double phi[IVK_MHD_MAX_QUAD * 6];
  double dphi[IVK_MHD_MAX_QUAD * 12];
  double psi[IVK_MHD_MAX_QUAD * 3];
  double dpsi[6];
};

__global__ void mhd_element_kernel(MhdTables tb, int n_cells, const double* __restrict__ geo,
                                   const int32_t* __restrict__ cnodes,
                                   const double* __restrict__ u0, const double* __restrict__ B0,
                                   double* __restrict__ Le) {
  const long tid = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (tid >= (long)n_cells * 30) return;
  const int cell = (int)(tid / 30), i = (int)(tid - (long)cell * 30);
  const double* gg = geo + (long)cell * 5;
  const double J00 = gg[0], J01 = gg[1], J10 = gg[2], J11 = gg[3], det = gg[4];
  int nd[6];
  double u0n[6][2], B0n[6][2];
#pragma unroll
  for (int a = 0; a < 6; ++a) {
    nd[a] = cnodes[(long)cell * 6 + a];
    u0n[a][0] = u0[2 * nd[a]];
    u0n[a][1] = u0[2 * nd[a] + 1];
    B0n[a][0] = B0[2 * nd[a]];
    B0n[a][1] = B0[2 * nd[a] + 1];
  }
  double gp[3][2];   // physical P1 gradients (constant)
#pragma unroll
  for (int v = 0; v < 3; ++v) {
    gp[v][0] = tb.dpsi[2 * v] * J00 + tb.dpsi[2 * v + 1] * J10;
    gp[v][1] = tb.dpsi[2 * v] * J01 + tb.dpsi[2 * v + 1] * J11;
  }
  double row[30];
#pragma unroll
  for (int j = 0; j < 30; ++j) row[j] = 0.0;
  const double iRe = 1.0 / tb.Re, iRm = 1.0 / tb.Rm, Sc = tb.S;
  for (int q = 0; q < tb.nq; ++q) {
    const double wq = tb.w[q] * det;
    double ph[6], G[6][2];
#pragma unroll
    for (int a = 0; a < 6; ++a) {
      ph[a] = tb.phi[q * 6 + a];
      const double d0 = tb.dphi[(q * 6 + a) * 2], d1 = tb.dphi[(q * 6 + a) * 2 + 1];
      G[a][0] = d0 * J00 + d1 * J10;
      G[a][1] = d0 * J01 + d1 * J11;
    }
    double U[2] = {0.0, 0.0}, Bq[2] = {0.0, 0.0}, gU[2][2] = {{0.0, 0.0}, {0.0, 0.0}},
           gB[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
    for (int a = 0; a < 6; ++a)
#pragma unroll
      for (int d = 0; d < 2; ++d) {
        U[d] += u0n[a][d] * ph[a];
        Bq[d] += B0n[a][d] * ph[a];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          gU[d][e] += u0n[a][d] * G[a][e];
          gB[d][e] += B0n[a][d] * G[a][e];
        }
      }
    const double j0 = gB[1][0] - gB[0][1];
    const double zB0[2] = {-Bq[1], Bq[0]};     // z^ x B0
    const double cB0[2] = {Bq[1], -Bq[0]};     // e_f x B0
    const double cu0[2] = {-U[1], U[0]};       // u0 x e_g
    if (i < 24) {
      const int a = i >> 2, comp = i & 3;
      const double jca[2] = {-G[a][1], G[a][0]};   // j(phi_a e_h)
      for (int b = 0; b < 6; ++b) {
        const double jcb[2] = {-G[b][1], G[b][0]};
        const double lap = G[a][0] * G[b][0] + G[a][1] * G[b][1];
        const double adv = ph[a] * (U[0] * G[b][0] + U[1] * G[b][1]);
        if (comp < 2) {
          const int d = comp;
#pragma unroll
          for (int f = 0; f < 2; ++f) {
            // (1/Re)[delta_df grad.grad + d_f phi_a d_d phi_b] + convection
            double v = iRe * ((d == f ? lap : 0.0) + G[a][f] * G[b][d]);
            v += (d == f ? adv : 0.0) + ph[a] * ph[b] * gU[d][f];
            row[4 * b + f] += wq * v;
          }
#pragma unroll
          for (int g2 = 0; g2 < 2; ++g2) {
            // -S [phi_a (z^xB0)_d j(phi_b e_g) + phi_a phi_b j0 (z^ x e_g)_d]
            const double Zgd = (g2 == 0) ? (d == 1 ? 1.0 : 0.0) : (d == 0 ? -1.0 : 0.0);
            row[4 * b + 2 + g2] += wq * (-Sc) * (ph[a] * zB0[d] * jcb[g2] + ph[a] * ph[b] * j0 * Zgd);
          }
        } else {
          const int h = comp - 2;
#pragma unroll
          for (int f = 0; f < 2; ++f) row[4 * b + f] += wq * (-ph[b] * cB0[f] * jca[h]);
#pragma unroll
          for (int g2 = 0; g2 < 2; ++g2)
            row[4 * b + 2 + g2] += wq * (-ph[b] * cu0[g2] * jca[h] + iRm * jcb[g2] * jca[h]);
        }
      }
      if (comp < 2) {
#pragma unroll
        for (int v = 0; v < 3; ++v) row[27 + v] += wq * (-tb.psi[q * 3 + v] * G[a][comp]);
      } else {
#pragma unroll
        for (int v = 0; v < 3; ++v) row[24 + v] += wq * (-gp[v][comp - 2] * ph[a]);
      }
    } else if (i < 27) {
      const int v = i - 24;   // -(B, grad s_v)
      for (int b = 0; b < 6; ++b)
#pragma unroll
        for (int g2 = 0; g2 < 2; ++g2) row[4 * b + 2 + g2] += wq * (-ph[b] * gp[v][g2]);
    } else {
      const int v = i - 27;   // -(div u, q_v)
      for (int b = 0; b < 6; ++b)
#pragma unroll
        for (int f = 0; f < 2; ++f) row[4 * b + f] += wq * (-tb.psi[q * 3 + v] * G[b][f]);
    }
  }
  double* out = Le + (long)cell * 900 + i * 30;
#pragma unroll
  for (int j = 0; j < 30; ++j) out[j] = row[j];
}

__global__ void mhd_gather_kernel(int nnz, const int32_t* __restrict__ ptr,
                                  const int32_t* __restrict__ contrib,
                                  const double* __restrict__ Le, double* __restrict__ ml,
                                  const int32_t* __restrict__ sell_pos, double* __restrict__ sml) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += gridDim.x * blockDim.x) {
    double v = 0.0;
    for (int k = ptr[e]; k < ptr[e + 1]; ++k) v += Le[contrib[k]];
    ml[2L * e + 1] = v;
    if (sml) sml[2L * sell_pos[e] + 1] = v;
  }
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

int ivk_mhd_assemble(const ivk_mhd_desc* d, const double* u0, const double* B0,
                     double* elem_scratch, double* ml, double* sml, void* stream) {
  IVK_REQUIRE(d && u0 && B0 && elem_scratch && ml, "bad MHD assembly arguments");
  IVK_REQUIRE(d->nq >= 1 && d->nq <= IVK_MHD_MAX_QUAD, "quadrature rule size");
  IVK_REQUIRE(d->cell_geo && d->cell_nodes && d->entry_ptr && d->entry_contrib,
              "MHD descriptor has a NULL array");
  IVK_REQUIRE(!sml || d->sell_pos, "SELL output needs sell_pos");
  MhdTables tb;
  tb.nq = d->nq;
  tb.Re = d->Re;
  tb.Rm = d->Rm;
  tb.S = d->S;
  for (int i = 0; i < IVK_MHD_MAX_QUAD; ++i) tb.w[i] = d->w[i];
  for (int i = 0; i < IVK_MHD_MAX_QUAD * 6; ++i) tb.phi[i] = d->phi[i];
  for (int i = 0; i < IVK_MHD_MAX_QUAD * 12; ++i) tb.dphi[i] = d->dphi[i];
  for (int i = 0; i < IVK_MHD_MAX_QUAD * 3; ++i) tb.psi[i] = d->psi[i];
  for (int i = 0; i < 6; ++i) tb.dpsi[i] = d->dpsi[i];
  cudaStream_t st = as_stream(stream);
  const long nthr = (long)d->n_cells * 30;
  mhd_element_kernel<<<(int)((nthr + 127) / 128), 128, 0, st>>>(tb, d->n_cells, d->cell_geo,
                                                                 d->cell_nodes, u0, B0, elem_scratch);
  int rc = check_launch("ivk_mhd_assemble(elements)");
  if (rc) return rc;
  mhd_gather_kernel<<<grid_cap(d->nnz, 256), 256, 0, st>>>(d->nnz, d->entry_ptr, d->entry_contrib,
                                                           elem_scratch, ml, d->sell_pos, sml);
  return check_launch("ivk_mhd_assemble(gather)");
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
