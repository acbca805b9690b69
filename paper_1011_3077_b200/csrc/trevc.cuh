// trevc.cuh -- eigenvectors of an upper triangular T (TREVC).
//
// TX = XD, D = diag(T), X upper triangular with X_jj = 1.  Blocked as
// Alg. 8 with the two outer loops exchanged: block rows i are
// processed bottom-up and, for each, ALL block columns j > i at once --
//   S[i, j]  = sum_{k > i} T[i, k] X[k, j]        one DMMA GEMM per block row (the B
//              operand X is upper triangular, so each column tile stops its K loop at
//              its last column: n^3/3 flops in total)
//   X[i, j]  : (T[i,i] - d_c I) x_c = -s_c        per column c, shift d_c = T_cc  (this
//              kernel; the shifted block solves are what Alg. 8 leaves to "solve")
// The diagonal block X[i, i] is the same recurrence with s_c = T[i-rows, c]; one launch per
// block row covers its diagonal-block columns and all columns to the right.
//
// Near-equal eigenvalues (reading Q19, LAPACK dtrevc/dlaln2): a denominator
// |T_qq - d_c| < smin = max(ulp |d_c|, smlnum) is replaced by smin.
#pragma once
#include "common.cuh"

namespace sdc {

constexpr int TREVC_B = 64;            // block size b (rows of a block row)
constexpr int TREVC_LDS = TREVC_B + 1; // padded SMEM column stride of the diagonal block

// One warp per column c in [c_lo, c_hi) of block row [i0, i0 + nbk):
//   rows r = lane, lane + 32 hold num_r = s_rc (+ T_rq x_q added as x_q become known)
//   x_q = num_q * (-1 / (T_qq - d_c)), q = qtop .. 0  (reciprocals precomputed per lane)
// Diagonal-block columns (c < i0 + nbk): num_r = T_rc X_cc = T_rc, qtop = c - i0 - 1, and
// X_cc = 1 is written.  Off-diagonal columns: num = sum_z P[z] (split-K partials of S,
// fixed order; column c of S is column c - pc0 of every partial), qtop = nbk - 1.
__global__ void __launch_bounds__(256) k_trevc_block(const double* __restrict__ T, long long ldt,
                                                     int i0, int nbk, int c_lo, int c_hi,
                                                     const double* __restrict__ P, int splits,
                                                     long long zs, long long ldp, int pc0,
                                                     double* X, long long ldx, int n) {
  __shared__ double Tb[TREVC_B * TREVC_LDS];   // Tb[q * LDS + r] = T(i0 + r, i0 + q)
  for (int e = threadIdx.x; e < nbk * nbk; e += blockDim.x) {
    const int r = e % nbk, q = e / nbk;
    Tb[q * TREVC_LDS + r] = r <= q ? T[(i0 + r) + (long long)(i0 + q) * ldt] : 0.0;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  const double ulp = 2.220446049250313e-16, smlnum = 2.2250738585072014e-308 * (double)n / ulp;
  for (int c = c_lo + blockIdx.x * wpb + warp; c < c_hi; c += gridDim.x * wpb) {
    const double dc = T[c + (long long)c * ldt];
    const double smin = fmax(ulp * fabs(dc), smlnum);
    const bool diag = c < i0 + nbk;
    int qtop;
    double r0 = 0.0, r1 = 0.0;
    if (diag) {
      const int cc = c - i0;
      qtop = cc - 1;
      if (lane < cc) r0 = T[(i0 + lane) + (long long)c * ldt];
      if (lane + 32 < cc) r1 = T[(i0 + lane + 32) + (long long)c * ldt];
    } else {
      qtop = nbk - 1;
      const long long off = (long long)(c - pc0) * ldp;   // P column of c
      for (int z = 0; z < splits; ++z) {
        if (lane < nbk) r0 += P[(long long)z * zs + off + lane];
        if (lane + 32 < nbk) r1 += P[(long long)z * zs + off + lane + 32];
      }
    }
    // reciprocal denominators of this lane's two rows, off the dependency chain: each step
    // of the back substitution is then one multiply by the owner lane + one shuffle
    double inv0, inv1;
    {
      double d0 = Tb[lane * TREVC_LDS + lane] - dc, d1 = Tb[(lane + 32) * TREVC_LDS + lane + 32] - dc;
      if (fabs(d0) < smin) d0 = smin;
      if (fabs(d1) < smin) d1 = smin;
      inv0 = -1.0 / d0;
      inv1 = -1.0 / d1;
    }
    double x0 = 0.0, x1 = 0.0;
    for (int q = qtop; q >= 0; --q) {
      if (lane == (q & 31)) {
        if (q < 32) x0 = r0 * inv0;
        else x1 = r1 * inv1;
      }
      const double xq = __shfl_sync(0xffffffffu, q < 32 ? x0 : x1, q & 31);
      if (lane < q) r0 = fma(Tb[q * TREVC_LDS + lane], xq, r0);
      if (lane + 32 < q) r1 = fma(Tb[q * TREVC_LDS + lane + 32], xq, r1);
    }
    const int rows = diag ? c - i0 : nbk;       // rows of this block row above the diagonal
    if (lane < rows) X[(i0 + lane) + (long long)c * ldx] = x0;
    if (lane + 32 < rows) X[(i0 + lane + 32) + (long long)c * ldx] = x1;
    if (diag && lane == 0) X[c + (long long)c * ldx] = 1.0;
  }
}

}  // namespace sdc
