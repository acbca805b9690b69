// cqr.cuh -- CholeskyQR2 panel factorisation with Householder reconstruction (round 2).
//
// The Householder panel (panel.cuh) needs one grid-wide exchange per COLUMN: a chain of 64
// latency-bound rounds (2.3-2.9 us each).  For a well-conditioned panel P (m x 64) the same
// compact-WY factor can be built with THREE exchanges:
//   CholeskyQR2:  G1 = P^T P,  R1 = chol(G1),  Q1 = P R1^{-1};
//                 G2 = Q1^T Q1, R2 = chol(G2),  Q  = Q1 R2^{-1},  P = Q R,  R = R2 R1
//     (Yamamoto-Nakatsukasa-Yanagisawa-Fukaya 2015: orthogonality and residual O(eps) while
//     kappa(P) ~< eps^{-1/2});
//   Householder reconstruction (Ballard-Demmel-Grigori-Jacquelin-Knight-Nguyen 2015, the
//     dorhr_col construction): LU without pivoting of (Q(0:64,:) - D), D = diag(+-1) chosen
//     pivot by pivot so that |U_kk| >= 1:  Q_top - D = L U;  then
//       Y = [L; Q(64:m,:) U^{-1}],  T = -U D L^{-T},  I - Y T Y^T = H,  H(:, 0:64) = Q D,
//     so H^T P = [D R; 0]: a valid Householder representation of the panel's QR, with R's
//     diagonal signs D (the callers only ever use |diag R| or normalise by its signs).
// The exchanges: G1 and G2 are reduced across the panel's CTAs through L2 (packed upper
// triangles, flag-carrying words as in the multi-cluster Householder exchange; each entry is
// summed by ONE owner CTA in a fixed order, so every CTA receives bit-identical Grams and
// takes the same decisions), and CTA 0 publishes M = R2^{-1} U^{-1} (Y(64:m,:) = Q1 M).
// Breakdown: a Cholesky pivot below 1e-6 of its column's squared norm (a panel column within
// ~1e-3 of the span of the previous ones) makes every CTA fall back -- uniformly -- to the
// Householder column loop, which is rank-revealing where CholeskyQR is not.
#pragma once
#include "common.cuh"

namespace sdc {

constexpr int CQ_LD = 68;                 // ld of the 64 x 64 shared scratch matrices
constexpr int CQ_E = 64 * 65 / 2;         // packed upper triangle of a 64 x 64 matrix
constexpr int CQ_GMAX = 160;              // most CTAs of one panel
constexpr int CQ_REGION = (CQ_GMAX + 1) * CQ_E * 2;          // doubles: partials + reduced (LL)
constexpr size_t CQ_DOUBLES = 2 * (size_t)CQ_REGION + 2 * CQ_E + 64;   // exchange buffer per context
constexpr int CQ_SCRATCH = 2 * 64 * CQ_LD + 6 * 64;          // shared doubles used by the path
constexpr double CQ_PIVOT_TOL = 1e-6;

SDC_DEV int cq_col(int p) {               // column j of packed upper index p = j(j+1)/2 + i
  int j = (int)((sqrt(8.0 * p + 1.0) - 1.0) * 0.5);
  while (j * (j + 1) / 2 > p) --j;
  while ((j + 1) * (j + 2) / 2 <= p) ++j;
  return j;
}

SDC_DEV void cq_ll_store(double* slot, double v, unsigned flag) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  const unsigned long long w0 = ((unsigned long long)flag << 32) | (b & 0xffffffffull);
  const unsigned long long w1 = ((unsigned long long)flag << 32) | (b >> 32);
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};\n" ::"l"(slot), "l"(w0), "l"(w1) : "memory");
}
SDC_DEV bool cq_ll_load(const double* slot, unsigned flag, double& v) {
  unsigned long long w0, w1;
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];\n" : "=l"(w0), "=l"(w1) : "l"(slot) : "memory");
  v = __longlong_as_double((long long)((w1 << 32) | (w0 & 0xffffffffull)));
  return (unsigned)(w0 >> 32) == flag && (unsigned)(w1 >> 32) == flag;
}
// poll one slot until its flag matches (bounded: a co-residency violation sets *err)
SDC_DEV double cq_ll_wait(const double* slot, unsigned flag, unsigned* err) {
  double v;
  unsigned polls = 0;
  while (!cq_ll_load(slot, flag, v)) {
    if (++polls > (1u << 24)) { atomicExch(err, 1u); return 0.0; }
  }
  return v;
}

// ---- warp tile: acc (16 x 16 as 2 x 2 DMMA fragments) += A(16 x K) B(K x 16) ------------
// fa(i, k) / fb(k, j) read the operands (i, j in [0, 16)); fragments per the PTX layout
// (lane t: A[t/4][t%4], B[t%4][t/4], D[t/4][2(t%4) + {0,1}]).
template <class FA, class FB>
SDC_DEV void cq_tile16(double (&acc)[2][2][2], int k0, int k1, FA fa, FB fb) {
  const int lane = threadIdx.x & 31, lr = lane >> 2, lc = lane & 3;
  for (int k = k0; k < k1; k += 4) {
    double a0 = fa(lr, k + lc), a1 = fa(8 + lr, k + lc);
    double b0 = fb(k + lc, lr), b1 = fb(k + lc, 8 + lr);
    dmma_8x8x4(acc[0][0], a0, b0);
    dmma_8x8x4(acc[0][1], a0, b1);
    dmma_8x8x4(acc[1][0], a1, b0);
    dmma_8x8x4(acc[1][1], a1, b1);
  }
}

// ---- packed Gram partial of the CTA's rows -> exchange slot (upper 16x16 tiles, warps 0-9)
SDC_DEV void cq_gram_partial(const double* X, int ldx, int R, double* slot, unsigned flag) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (w >= 10) return;
  // upper tile w of the 4 x 4 block grid: (bi, bj), bi <= bj
  int bi = 0, bj = 0, t = w;
  for (int j = 0; j < 4; ++j) { if (t <= j) { bi = t; bj = j; break; } t -= j + 1; }
  double acc[2][2][2] = {};
  const int K = (R + 3) & ~3;
  cq_tile16(acc, 0, K,
            [&](int i, int k) { return k < R ? X[k * ldx + 16 * bi + i] : 0.0; },
            [&](int k, int j) { return k < R ? X[k * ldx + 16 * bj + j] : 0.0; });
  const int lr = lane >> 2, lc = lane & 3;
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int i = 16 * bi + 8 * mi + lr, j = 16 * bj + 8 * ni + 2 * lc + c;
        if (i <= j) cq_ll_store(slot + 2 * (size_t)(j * (j + 1) / 2 + i), acc[mi][ni][c], flag);
      }
}

// ---- N slots polled together: every load in flight at once, then only the missing ones
// again (one L2 round trip once all are written)
template <int N>
SDC_DEV void cq_ll_wait_n(const double* const (&slot)[N], int cnt, unsigned flag, double (&v)[N],
                          unsigned* err) {
  bool ok[N];
#pragma unroll
  for (int u = 0; u < N; ++u) ok[u] = u >= cnt;
  unsigned polls = 0;
  for (;;) {
    bool all = true;
#pragma unroll
    for (int u = 0; u < N; ++u)
      if (!ok[u]) { ok[u] = cq_ll_load(slot[u], flag, v[u]); all &= ok[u]; }
    if (all) break;
    if (++polls > (1u << 24)) { atomicExch(err, 1u); break; }
  }
}

// ---- owner reduction of packed entries [e0, e1): sum over the G partial slots in a fixed
// order (groups of 16 threads per entry, each thread the CTAs q, q+16, ... in order, then a
// fixed xor tree), published to the reduced slot with the same flag
SDC_DEV void cq_owner_reduce(double* region, int G, int e0, int e1, unsigned flag, unsigned* err) {
  constexpr int NS = CQ_GMAX / 16;
  const int grp = threadIdx.x >> 4, q = threadIdx.x & 15;
  const int rounds = (e1 - e0 + 31) / 32;                 // uniform across the warp
  for (int t = 0; t < rounds; ++t) {
    const int e = e0 + grp + 32 * t;
    const bool act = e < e1;
    const double* sl[NS];
    double v[NS];
    int cnt = 0;
#pragma unroll
    for (int u = 0; u < NS; ++u) {
      const int c = q + 16 * u;
      sl[u] = region + 2 * ((size_t)(c < G ? c : 0) * CQ_E + (act ? e : e0));
      if (act && c < G) cnt = u + 1;
    }
    cq_ll_wait_n(sl, cnt, flag, v, err);
    double s = 0.0;
#pragma unroll
    for (int u = 0; u < NS; ++u)
      if (u < cnt) s += v[u];
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 4);
    s += __shfl_xor_sync(0xffffffffu, s, 8);
    if (act && q == 0) cq_ll_store(region + 2 * ((size_t)G * CQ_E + e), s, flag);
  }
}

// ---- gather a packed upper triangle into a 64 x 64 (ld CQ_LD): symmetric, or upper with
// a zero strictly lower part
template <bool SYM>
SDC_DEV void cq_gather(const double* red, unsigned flag, double* M, unsigned* err) {
  constexpr int NP = (CQ_E + 511) / 512;   // 5 entries per thread (512 threads)
  const double* sl[NP];
  double v[NP];
  int cnt = 0;
#pragma unroll
  for (int u = 0; u < NP; ++u) {
    const int p = threadIdx.x + 512 * u;
    sl[u] = red + 2 * (size_t)(p < CQ_E ? p : 0);
    if (p < CQ_E) cnt = u + 1;
  }
  cq_ll_wait_n(sl, cnt, flag, v, err);
#pragma unroll
  for (int u = 0; u < NP; ++u) {
    const int p = threadIdx.x + 512 * u;
    if (p >= CQ_E) continue;
    const int j = cq_col(p), i = p - j * (j + 1) / 2;
    M[j + i * CQ_LD] = SYM || i == j ? v[u] : 0.0;
    M[i + j * CQ_LD] = v[u];
  }
}

// ---- Cholesky (upper, G = R^T R) in place, right-looking with the unscaled pivot row:
// one CTA barrier per step.  Returns false (every thread, same decision) if a pivot falls
// below CQ_PIVOT_TOL of its column's squared norm gd[k] (kept in gd[]).
SDC_DEV bool cq_chol(double* M, double* gd, double* dv) {
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int k = tid; k < 64; k += nt) gd[k] = M[k + k * CQ_LD];
  __syncthreads();
  for (int k = 0; k < 64; ++k) {
    const double akk = M[k + k * CQ_LD];
    if (!(akk > CQ_PIVOT_TOL * gd[k])) { __syncthreads(); return false; }
    const double rinv = 1.0 / akk;
    // trailing upper triangle (k < i <= j < 64): thread tid owns column j = tid & 63 and
    // rows i = k + 1 + (tid >> 6) + 8 s
    const int j = tid & 63;
    if (j > k) {
      const double akj = M[k + j * CQ_LD] * rinv;
      for (int i = k + 1 + (tid >> 6); i <= j; i += 8) M[i + j * CQ_LD] -= M[k + i * CQ_LD] * akj;
    }
    __syncthreads();
  }
  // scale rows: R(k, j) = A(k, j) / sqrt(A_kk), j >= k; zero the strictly lower part
  for (int k = tid; k < 64; k += nt) dv[k] = 1.0 / sqrt(M[k + k * CQ_LD]);
  __syncthreads();
  for (int e = tid; e < 64 * 64; e += nt) {
    const int i = e & 63, j = e >> 6;
    M[i + j * CQ_LD] = i <= j ? M[i + j * CQ_LD] * dv[i] : 0.0;
  }
  __syncthreads();
  return true;
}

// ---- inverse of an upper triangular U (ld CQ_LD) into X (upper, ld CQ_LD), X != U:
// columns are independent back substitutions; 8 threads per column (fixed-order shuffle sums)
SDC_DEV void cq_trinv_upper(const double* U, double* X) {
  const int j = threadIdx.x >> 3, q = threadIdx.x & 7;   // 64 columns x 8 threads
  double x[8];                                            // x[s] = X(q + 8 s, j)
#pragma unroll
  for (int s = 0; s < 8; ++s) x[s] = 0.0;
  for (int i = 63; i >= 0; --i) {                         // every lane runs every step (shuffles)
    double part = 0.0;
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const int l = q + 8 * s;
      if (l > i && l <= j) part = fma(U[i + l * CQ_LD], x[s], part);
    }
    part += __shfl_xor_sync(0xffffffffu, part, 1);
    part += __shfl_xor_sync(0xffffffffu, part, 2);
    part += __shfl_xor_sync(0xffffffffu, part, 4);
    const double v = ((i == j ? 1.0 : 0.0) - part) / U[i + i * CQ_LD];
#pragma unroll
    for (int s = 0; s < 8; ++s)
      if (q + 8 * s == i && i <= j) x[s] = v;
  }
#pragma unroll
  for (int s = 0; s < 8; ++s) X[q + 8 * s + j * CQ_LD] = q + 8 * s <= j ? x[s] : 0.0;
}

// ---- rows of X (R rows, ld ldx, 64 columns) <- X * B, B upper triangular (ld CQ_LD), in
// place: each warp owns 8-row stripes and reads its whole stripe before writing it
SDC_DEV void cq_rows_times_upper(double* X, int ldx, int R, int rbeg, const double* B) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, lr = lane >> 2, lc = lane & 3;
  const int nw = blockDim.x >> 5;
  for (int s0 = rbeg + 8 * w; s0 < R; s0 += 8 * nw) {
    double acc[8][2];
#pragma unroll
    for (int nj = 0; nj < 8; ++nj) { acc[nj][0] = 0.0; acc[nj][1] = 0.0; }
    const int row = s0 + lr;
#pragma unroll
    for (int k = 0; k < 64; k += 4) {
      const double a = row < R ? X[row * ldx + k + lc] : 0.0;
#pragma unroll
      for (int nj = 0; nj < 8; ++nj) {
        if (k >= 8 * (nj + 1)) continue;                  // B upper: rows k > column block
        dmma_8x8x4(acc[nj], a, B[(k + lc) + (8 * nj + lr) * CQ_LD]);
      }
    }
    __syncwarp();
    const int orow = s0 + lr;
    if (orow < R) {
#pragma unroll
      for (int nj = 0; nj < 8; ++nj) {
        X[orow * ldx + 8 * nj + 2 * lc] = acc[nj][0];
        X[orow * ldx + 8 * nj + 2 * lc + 1] = acc[nj][1];
      }
    }
  }
}

// ---- rows 0..63 of X (ld ldx) <- X(0:64, :) U^{-1}, U upper (ld CQ_LD): independent forward
// substitutions per row, 8 threads per row (x_j = (x_j - sum_{l<j} x_l U_lj) / U_jj)
SDC_DEV void cq_trsm_rows64(double* X, int ldx, const double* U) {
  const int row = threadIdx.x >> 3, q = threadIdx.x & 7;
  double x[8];
#pragma unroll
  for (int s = 0; s < 8; ++s) x[s] = 0.0;
  for (int j = 0; j < 64; ++j) {
    double part = 0.0;
#pragma unroll
    for (int s = 0; s < 8; ++s)
      if (q + 8 * s < j) part = fma(x[s], U[(q + 8 * s) + j * CQ_LD], part);
    part += __shfl_xor_sync(0xffffffffu, part, 1);
    part += __shfl_xor_sync(0xffffffffu, part, 2);
    part += __shfl_xor_sync(0xffffffffu, part, 4);
    const double v = (X[row * ldx + j] - part) / U[j + j * CQ_LD];
#pragma unroll
    for (int s = 0; s < 8; ++s)
      if (q + 8 * s == j) x[s] = v;
  }
  __syncwarp();
#pragma unroll
  for (int s = 0; s < 8; ++s) X[row * ldx + q + 8 * s] = x[s];
}

// ---- modified LU without pivoting (dorhr_col): X(0:64, 0:64) (ld ldx) - D = L U in place,
// D_k = -sign(pivot) so that |U_kk| = |pivot| + 1 >= 1; one CTA barrier per step.  On return
// X holds L (strictly lower, unit diagonal implied) and U (upper); D in dsg, U_kk in ukk.
SDC_DEV void cq_lu_signed(double* X, int ldx, double* dsg, double* ukk) {
  const int tid = threadIdx.x;
  const int j = tid & 63, i0 = tid >> 6;
  for (int k = 0; k < 64; ++k) {
    const double piv = X[k * ldx + k];
    const double sk = piv >= 0.0 ? -1.0 : 1.0;
    const double pk = piv - sk;
    if (tid == 0) { dsg[k] = sk; ukk[k] = pk; }
    if (j > k) {
      const double akj = X[k * ldx + j] / pk;
      for (int i = k + 1 + i0; i < 64; i += 8) X[i * ldx + j] -= X[i * ldx + k] * akj;
    }
    __syncthreads();
  }
  for (int e = tid; e < 64 * 64; e += blockDim.x) {   // L = column k / U_kk, U_kk on the diagonal
    const int r = e >> 6, c = e & 63;
    if (r > c) X[r * ldx + c] /= ukk[c];
    else if (r == c) X[r * ldx + c] = ukk[c];
  }
  __syncthreads();
}

// ---- inverse of the unit lower triangular L (strictly lower part of X rows 0..63, ld ldx)
// into Li (lower, unit diagonal, zero upper; ld CQ_LD): 8 threads per column
SDC_DEV void cq_trinv_unit_lower(const double* X, int ldx, double* Li) {
  const int j = threadIdx.x >> 3, q = threadIdx.x & 7;
  double x[8];
#pragma unroll
  for (int s = 0; s < 8; ++s) x[s] = 0.0;
  for (int i = 0; i < 64; ++i) {
    double part = 0.0;
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const int l = q + 8 * s;
      if (l >= j && l < i) part = fma(X[i * ldx + l], x[s], part);
    }
    part += __shfl_xor_sync(0xffffffffu, part, 1);
    part += __shfl_xor_sync(0xffffffffu, part, 2);
    part += __shfl_xor_sync(0xffffffffu, part, 4);
    const double v = i == j ? 1.0 : -part;
#pragma unroll
    for (int s = 0; s < 8; ++s)
      if (q + 8 * s == i && i >= j) x[s] = v;
  }
#pragma unroll
  for (int s = 0; s < 8; ++s) Li[q + 8 * s + j * CQ_LD] = q + 8 * s >= j ? x[s] : 0.0;
}

}  // namespace sdc
