// K7 core: register-resident Gauss-Jordan inverse of one d x d patch matrix
// per CTA (replaces np.linalg.inv per patch, reference solvers.py:177).
//
// The CTA's threads form a 16 x TX grid over the matrix in a cyclic layout:
// thread (ty, tx) = (tid & 15, tid >> 4) holds rows ty + 16 ri (ri < RT) and
// column slots tx + TX cj (cj < CT) in registers for the whole elimination, so
// the rank-1 update of a pivot step is RT x CT (complex: 4x) FMAs per thread
// against RT + CT shared-memory loads -- the FP64 pipe, not shared memory,
// sets the pace (the previous kernel kept the matrix in shared memory: three
// loads and a store per FMA, an integer division per element, five barriers
// per pivot).
//
// Pivoting is partial (largest |re| + |im| of the pivot column among the rows
// not yet used, first on ties -- LAPACK's idamax rule) but IMPLICIT: rows are
// never swapped.  Step k publishes column k (its owners sit in one half-warp,
// which also finds the pivot row with four shuffles and publishes 1/pivot),
// CTA barrier, the pivot row's owners publish the scaled row -- each to its own
// half-warp, which holds exactly the column slots it needs, so a warp-level
// barrier suffices -- and every thread updates its tile.  The published column
// / row are double-buffered (the step loop is unrolled by two so the buffer is
// static): a step costs ONE CTA barrier.  Writing the update as  a_ij <- a'_ij - c_i r_j  with a' = a
// except zero in the pivot row and pivot column, c_prow = -1 (stored into the
// published column) and r_k = 1/pivot makes it uniform: no per-element
// predicates.  With r_k the pivot row of step k, slot (i, k) ends up holding
// Inv[step(i)][r_k]; the routine writes the unscrambled, transposed inverse
// (the layout the apply kernels stream) back over the input in shared memory.

#pragma once

namespace ivk {

// Published column / row of the current pivot step (double-buffered), the
// pivot bookkeeping.  NR >= 16 RT rows, NC >= TX CT column slots.
template <bool CPLX, int NR, int NC>
struct GjScratch {
  double col_re[2][NR], col_im[2][CPLX ? NR : 1];
  double row_re[2][NC], row_im[2][CPLX ? NC : 1];
  double pinv_re[2], pinv_im[2];
  int order[NC];  // order[k] = pivot row of step k
  int step[NR];   // step[row] = k
  int prow[2];    // pivot row of the step, -1: singular / non-finite
};

// One pivot step (BUF = k & 1 selects the published column / row buffers).
template <bool CPLX, int TX, int RT, int CT, int BUF, class Scratch>
__device__ __forceinline__ bool gj_step(int k, int d, int ty, int tx, unsigned half,
                                        double (&ar)[RT][CT], double (&ai)[CPLX ? RT : 1][CPLX ? CT : 1],
                                        unsigned& used, Scratch& s) {
  double* colp_re = &s.col_re[BUF][ty];
  double* colp_im = &s.col_im[BUF][CPLX ? ty : 0];
  double* rowp_re = &s.row_re[BUF][tx];
  double* rowp_im = &s.row_im[BUF][CPLX ? tx : 0];
  const int kc = k / TX, kt = k & (TX - 1);
  if (tx == kt) {
    // Column k's owners (one half-warp): publish it, clear it, find the pivot
    // row, publish 1/pivot and put -1 in the pivot row's slot of the column.
    double cr[RT] = {}, ci[RT] = {};
#pragma unroll
    for (int cj = 0; cj < CT; ++cj)
      if (cj == kc) {
#pragma unroll
        for (int ri = 0; ri < RT; ++ri) {
          cr[ri] = ar[ri][cj];
          ar[ri][cj] = 0.0;
          if constexpr (CPLX) { ci[ri] = ai[ri][cj]; ai[ri][cj] = 0.0; }
        }
      }
    // pivot search on a 32-bit key: the top 25 bits of |re| + |im| (exponent +
    // 14 mantissa bits) above 127 - row, so one hardware max-reduction
    // (redux.sync) over the half-warp yields the largest entry (to 6e-5
    // relative -- near-ties go to the first row, still a partial pivot with
    // the usual growth bound) and its row; used rows carry key 0.
    unsigned key = 0;
#pragma unroll
    for (int ri = 0; ri < RT; ++ri) {
      colp_re[16 * ri] = cr[ri];
      if constexpr (CPLX) colp_im[16 * ri] = ci[ri];
      double a = fabs(cr[ri]);
      if constexpr (CPLX) a += fabs(ci[ri]);
      const unsigned kk = ((unsigned)__double2hiint(a) >> 6 << 7) | (unsigned)(127 - (ty + 16 * ri));
      if (!((used >> ri) & 1u)) key = max(key, kk);
    }
    key = __reduce_max_sync(half, key);
    __syncwarp(half);
    if (ty == 0) {
      const int bi = 127 - (int)(key & 127u);
      const double pr = s.col_re[BUF][bi];
      double pi = 0.0;
      if constexpr (CPLX) pi = s.col_im[BUF][bi];
      const double mag = fabs(pr) + fabs(pi);
      if (key == 0 || !(mag > 0.0) || !(mag < 1.79e308)) {
        s.prow[BUF] = -1;
      } else {
        if constexpr (CPLX) {
          const double den = pr * pr + pi * pi;
          s.pinv_re[BUF] = pr / den;
          s.pinv_im[BUF] = -pi / den;
          s.col_im[BUF][bi] = 0.0;
        } else {
          s.pinv_re[BUF] = 1.0 / pr;
        }
        s.col_re[BUF][bi] = -1.0;
        s.prow[BUF] = bi;
        s.order[k] = bi;
        s.step[bi] = k;
      }
    }
  }
  __syncthreads();
  const int prow = s.prow[BUF];
  if (prow < 0) return false;
  if (ty == (prow & 15)) {
    // the pivot row's owners: publish it scaled by 1/pivot (slot k: 1/pivot
    // itself -- the slot's register was cleared above), clear it
    const double inv_re = s.pinv_re[BUF];
    double inv_im = 0.0;
    if constexpr (CPLX) inv_im = s.pinv_im[BUF];
    const int pri = prow >> 4;
#pragma unroll
    for (int ri = 0; ri < RT; ++ri)
      if (ri == pri) {
#pragma unroll
        for (int cj = 0; cj < CT; ++cj) {
          if constexpr (CPLX) {
            rowp_re[TX * cj] = ar[ri][cj] * inv_re - ai[ri][cj] * inv_im;
            rowp_im[TX * cj] = ar[ri][cj] * inv_im + ai[ri][cj] * inv_re;
            ai[ri][cj] = 0.0;
          } else {
            rowp_re[TX * cj] = ar[ri][cj] * inv_re;
          }
          ar[ri][cj] = 0.0;
        }
      }
    if (tx == kt) {
      s.row_re[BUF][k] = inv_re;
      if constexpr (CPLX) s.row_im[BUF][k] = inv_im;
    }
    used |= 1u << pri;
  }
  // the row slots tx + TX cj a half-warp reads are the ones its own lane
  // (prow & 15) just wrote: a warp-level barrier is enough
  __syncwarp();
  double cr[RT], ci[RT], rr[CT], rim[CT];
#pragma unroll
  for (int ri = 0; ri < RT; ++ri) {
    cr[ri] = colp_re[16 * ri];
    if constexpr (CPLX) ci[ri] = colp_im[16 * ri];
  }
#pragma unroll
  for (int cj = 0; cj < CT; ++cj) {
    rr[cj] = rowp_re[TX * cj];
    if constexpr (CPLX) rim[cj] = rowp_im[TX * cj];
  }
#pragma unroll
  for (int ri = 0; ri < RT; ++ri)
#pragma unroll
    for (int cj = 0; cj < CT; ++cj) {
      if constexpr (CPLX) {
        ar[ri][cj] = fma(-cr[ri], rr[cj], fma(ci[ri], rim[cj], ar[ri][cj]));
        ai[ri][cj] = fma(-cr[ri], rim[cj], fma(-ci[ri], rr[cj], ai[ri][cj]));
      } else {
        ar[ri][cj] = fma(-cr[ri], rr[cj], ar[ri][cj]);
      }
    }
  (void)ci; (void)rim;
  return true;
}

// Are / Aim: the matrix, row-major with leading dimension d (Aim unused for
// real).  On success the same arrays hold the TRANSPOSED inverse with leading
// dimension ldo >= d:  T[j * ldo + i] = Inv[i][j] (i, j < d; rows d..ldo-1 of
// a column are zero-filled) -- the Inv^T layout the apply kernels stream, so
// the caller's store to HBM is a straight copy.  The arrays must hold d * ldo
// doubles.  All threads of the CTA (16 * TX of them) must call.  Returns
// false for a singular or non-finite matrix (uniformly over the CTA).
template <bool CPLX, int TX, int RT, int CT, class Scratch>
__device__ __forceinline__ bool gj_invert_registers(double* Are, double* Aim, int d, int ldo,
                                                    Scratch& s) {
  static_assert(sizeof(s.col_re[0]) >= 16 * RT * sizeof(double) &&
                sizeof(s.row_re[0]) >= TX * CT * sizeof(double), "tile exceeds the scratch");
  static_assert(!CPLX || sizeof(s.col_im[0]) >= 16 * RT * sizeof(double), "real-only scratch");
  static_assert(16 * RT <= 128, "the pivot key holds 7 row bits");
  static_assert((TX & (TX - 1)) == 0, "TX must be a power of two");
  const int tid = threadIdx.x, ty = tid & 15, tx = tid >> 4;
  const unsigned half = 0xffffu << (tid & 16);
  double ar[RT][CT], ai[CPLX ? RT : 1][CPLX ? CT : 1];
  unsigned used = 0;
#pragma unroll
  for (int ri = 0; ri < RT; ++ri) {
    const int i = ty + 16 * ri;
    if (i >= d) used |= 1u << ri;
#pragma unroll
    for (int cj = 0; cj < CT; ++cj) {
      const int j = tx + TX * cj;
      const bool in = i < d && j < d;
      ar[ri][cj] = in ? Are[i * d + j] : 0.0;
      if constexpr (CPLX) ai[ri][cj] = in ? Aim[i * d + j] : 0.0;
    }
  }
  for (int k = 0; k < d; k += 2) {
    if (!gj_step<CPLX, TX, RT, CT, 0>(k, d, ty, tx, half, ar, ai, used, s)) return false;
    if (k + 1 < d && !gj_step<CPLX, TX, RT, CT, 1>(k + 1, d, ty, tx, half, ar, ai, used, s))
      return false;
  }
  __syncthreads();  // order / step complete, every thread past its reads of Are
  // unscramble: slot (i, j) holds Inv[step(i)][order(j)]
#pragma unroll
  for (int cj = 0; cj < CT; ++cj) {
    const int j = tx + TX * cj;
    if (j >= d) continue;
    const int oj = s.order[j] * ldo;
#pragma unroll
    for (int ri = 0; ri < RT; ++ri) {
      const int i = ty + 16 * ri;
      if (i >= d) continue;
      const int o = oj + s.step[i];
      Are[o] = ar[ri][cj];
      if constexpr (CPLX) Aim[o] = ai[ri][cj];
    }
  }
  for (int e = tid; e < d * (ldo - d); e += blockDim.x) {
    const int j = e / (ldo - d), o = j * ldo + d + (e - j * (ldo - d));
    Are[o] = 0.0;
    if constexpr (CPLX) Aim[o] = 0.0;
  }
  __syncthreads();
  return true;
}

}  // namespace ivk
