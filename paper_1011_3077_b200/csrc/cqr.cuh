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
constexpr int CQ_SCRATCH = 2 * 64 * CQ_LD + 2 * 64 + 512 + 8;  // shared doubles used by the path
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
            [=](int i, int k) { return k < R ? X[k * ldx + 16 * bi + i] : 0.0; },
            [=](int k, int j) { return k < R ? X[k * ldx + 16 * bj + j] : 0.0; });
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
    if (row < R) {
#pragma unroll
      for (int nj = 0; nj < 8; ++nj) {
        X[row * ldx + 8 * nj + 2 * lc] = acc[nj][0];
        X[row * ldx + 8 * nj + 2 * lc + 1] = acc[nj][1];
      }
    }
  }
}

// =======================================================================================
// 64 x 64 building blocks (CTA of 512 threads = 16 warps; matrices col-major in shared
// memory, X(i, j) = X[i + j * ld]).  The serial parts (a 64-step pivot chain) are factored
// in 16 x 16 diagonal blocks by ONE warp in registers (lane j holds column j; shuffles, no
// barriers), everything off the diagonal blocks is 16 x 16 DMMA tiles -- a few CTA barriers
// per 64 x 64 factorisation instead of one per pivot.
// =======================================================================================
#define CQX(X, ld, i, j) (X)[(i) + (j) * (ld)]
constexpr unsigned CQ_FULL = 0xffffffffu;

// lane-column registers of the 16 x 16 block at (r0, c0): a[i] = X(r0 + i, c0 + (lane & 15))
SDC_DEV void cq_blk_load(const double* X, int ld, int r0, int c0, double (&a)[16]) {
  const int j = threadIdx.x & 15;
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = CQX(X, ld, r0 + i, c0 + j);
}
// store rows selected by `part` (0 all, 1 upper incl. diagonal, 2 strictly lower) of the
// block; other rows of the block are written as zero when zero_rest
SDC_DEV void cq_blk_store(double* X, int ld, int r0, int c0, const double (&a)[16], int part, bool zero_rest) {
  const int lane = threadIdx.x & 31, j = lane & 15;
  if (lane >= 16) return;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const bool keep = part == 0 || (part == 1 ? i <= j : i > j);
    if (keep) CQX(X, ld, r0 + i, c0 + j) = a[i];
    else if (zero_rest) CQX(X, ld, r0 + i, c0 + j) = 0.0;
  }
}

// one warp: upper Cholesky of the 16 x 16 block in registers (a: lane j = column j); pivot k
// must exceed CQ_PIVOT_TOL * gk[k] (its column's squared norm in the original Gram)
SDC_DEV bool cq_chol16(double (&a)[16], const double* gk) {
  bool ok = true;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const double piv = __shfl_sync(CQ_FULL, a[k], k);
    ok = ok && piv > CQ_PIVOT_TOL * gk[k];
    const double rd = piv > 0.0 ? rsqrt(piv) : 0.0;
    a[k] *= rd;                                   // row k of R (columns >= k)
#pragma unroll
    for (int i = k + 1; i < 16; ++i) a[i] = fma(-__shfl_sync(CQ_FULL, a[k], i), a[k], a[i]);
  }
  return ok;
}

// one warp: x = U^{-1} for a 16 x 16 upper triangular block of the accessor u(i, j) (block
// coordinates); unit != 0 assumes a unit diagonal.  Lane j returns column j of the inverse.
template <class FU>
SDC_DEV void cq_trinv16(FU u, bool unit, double (&x)[16]) {
  const int j = threadIdx.x & 15;
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = i == j ? 1.0 : 0.0;   // right-hand side e_j, solved in place
#pragma unroll
  for (int l = 15; l >= 0; --l) {
    x[l] = unit ? x[l] : x[l] * __drcp_rn(u(l, l));
#pragma unroll
    for (int i = 0; i < l; ++i) x[i] = fma(-u(i, l), x[l], x[i]);
  }
}

// one warp: modified LU (dorhr_col) of the 16 x 16 block in registers: pivot p -> p - s_k,
// s_k = -sign(p); returns L (strictly lower, rows > k of column k), U (upper) in a; signs to
// dsg[0..16) (lane 0)
SDC_DEV void cq_lu16(double (&a)[16], double* dsg) {
  const int lane = threadIdx.x & 31, j = lane & 15;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const double piv = __shfl_sync(CQ_FULL, a[k], k);
    const double sk = piv >= 0.0 ? -1.0 : 1.0;
    const double pk = piv - sk;
    const double rp = 1.0 / pk;                   // every lane (uniform, no divergent slow path)
    if (lane == 0) dsg[k] = sk;
#pragma unroll
    for (int i = k + 1; i < 16; ++i) {           // l_ik from lane k's unscaled column
      const double lik = __shfl_sync(CQ_FULL, a[i], k) * rp;
      a[i] = j > k ? fma(-lik, a[k], a[i]) : (j == k ? a[i] * rp : a[i]);
    }
    a[k] = j == k ? pk : a[k];
  }
}

// one warp: 16 x 16 tile product acc = op(A) op(B) over k in [0, K) (accessors in tile-local
// row / column coordinates); D fragments per the PTX m8n8k4 layout
template <class FA, class FB>
SDC_DEV void cq_mm16(double (&acc)[2][2][2], int K, FA fa, FB fb) {
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) { acc[mi][ni][0] = 0.0; acc[mi][ni][1] = 0.0; }
  cq_tile16(acc, 0, K, fa, fb);
}
template <class FS>
SDC_DEV void cq_acc_store(const double (&acc)[2][2][2], FS st) {
  const int lane = threadIdx.x & 31, lr = lane >> 2, lc = lane & 3;
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni)
#pragma unroll
      for (int c = 0; c < 2; ++c) st(8 * mi + lr, 8 * ni + 2 * lc + c, acc[mi][ni][c]);
}

// ---- C(64 x 64) = alpha A B with accessors; every warp one 16 x 16 tile, the K loop of tile
// (ti, tj) restricted to [16 kl(ti, tj), 16 kh(ti, tj)) (triangular operands); the products
// are formed in registers and stored after a CTA barrier, so C may alias A or B
template <class FA, class FB, class FKL, class FKH, class FS>
SDC_DEV void cq_gemm64(FA fa, FB fb, FKL kl, FKH kh, double alpha, FS st) {
  const int w = threadIdx.x >> 5, ti = w >> 2, tj = w & 3;
  double acc[2][2][2];
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) { acc[mi][ni][0] = 0.0; acc[mi][ni][1] = 0.0; }
  cq_tile16(acc, 16 * kl(ti, tj), 16 * kh(ti, tj), [=](int i, int k) { return fa(16 * ti + i, k); },
            [=](int k, int j) { return fb(k, 16 * tj + j); });
  __syncthreads();
  cq_acc_store(acc, [=](int i, int j, double v) { st(16 * ti + i, 16 * tj + j, alpha * v); });
  __syncthreads();
}

// ---- one warp, lanes 0..15 own the columns of the 16 x 16 tile B (block coordinates via
// the accessor): B <- U^{-T} B for U upper (forward substitution, rinv = 1/diag), or
// B <- L^{-1} B for L unit lower (accessor l(i, k), i > k).  16-step chains of FMAs with
// broadcast shared-memory operands, no shuffles.
template <class FU, class FB>
SDC_DEV void cq_solve_cols_ut(FU u, const double* rinv, FB b) {
  const int j = threadIdx.x & 31;
  if (j >= 16) return;
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = b(i, j);
#pragma unroll
  for (int i = 0; i < 16; ++i) {                 // (U^T x)_i = sum_{k <= i} U(k, i) x_k
#pragma unroll
    for (int k = 0; k < i; ++k) x[i] = fma(-u(k, i), x[k], x[i]);
    x[i] *= rinv[i];
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) b(i, j) = x[i];
}
template <class FL, class FB>
SDC_DEV void cq_solve_cols_unit_lower(FL l, FB b) {
  const int j = threadIdx.x & 31;
  if (j >= 16) return;
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = b(i, j);
#pragma unroll
  for (int i = 1; i < 16; ++i)
#pragma unroll
    for (int k = 0; k < i; ++k) x[i] = fma(-l(i, k), x[k], x[i]);
#pragma unroll
  for (int i = 0; i < 16; ++i) b(i, j) = x[i];
}
// rows of B (16 x 16, lanes own rows) <- B U^{-1}, U upper: x_j = (b_j - sum_{k<j} x_k U(k,j)) / U(j,j)
template <class FU, class FB>
SDC_DEV void cq_solve_rows_upper(FU u, const double* rinv, FB b) {
  const int i = threadIdx.x & 31;
  if (i >= 16) return;
  double x[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) x[j] = b(i, j);
#pragma unroll
  for (int j = 0; j < 16; ++j) {
#pragma unroll
    for (int k = 0; k < j; ++k) x[j] = fma(-x[k], u(k, j), x[j]);
    x[j] *= rinv[j];
  }
#pragma unroll
  for (int j = 0; j < 16; ++j) b(i, j) = x[j];
}

// ---- upper Cholesky G = R^T R of the 64 x 64 A (ld CQ_LD) in place (strictly lower part
// zeroed); false (every thread) on a pivot below CQ_PIVOT_TOL of its column's squared norm.
// Per 16-block step K: warp 0 factors the diagonal block in registers, warps solve the row
// panel R(K, J) = R_KK^{-T} A(K, J) tile by tile, DMMA tiles update the trailing blocks.
// sc: >= 16 doubles of scratch; gd: 64 doubles (the original diagonal).
__device__ __noinline__ bool cq_chol64(double* A, double* gd, double* sc, int* flag) {
  const int tid = threadIdx.x, w = tid >> 5;
  if (tid < 64) gd[tid] = CQX(A, CQ_LD, tid, tid);
  if (tid == 0) *flag = 1;
  __syncthreads();
  for (int K = 0; K < 4; ++K) {
    const int o = 16 * K;
    if (w == 0) {
      double a[16];
      cq_blk_load(A, CQ_LD, o, o, a);
      if (!cq_chol16(a, gd + o) && tid == 0) *flag = 0;
      cq_blk_store(A, CQ_LD, o, o, a, 1, true);
      if (tid < 16) sc[tid] = 1.0 / a[tid];       // lane j's a[j] = R_jj
    }
    __syncthreads();
    if (!*flag) return false;
    if (K == 3) break;
    if (w < 3 - K) {   // row panel tile J = K + 1 + w
      const int c = o + 16 * (w + 1);
      cq_solve_cols_ut([=](int i, int k) { return CQX(A, CQ_LD, o + i, o + k); }, sc,
                       [=](int i, int j) -> double& { return CQX(A, CQ_LD, o + i, c + j); });
    }
    __syncthreads();
    {   // trailing A(I, J) -= R(K, I)^T R(K, J), K < I <= J
      int t = w, I = -1, J = -1;
      for (int ii = K + 1; ii < 4 && I < 0; ++ii)
        for (int jj = ii; jj < 4; ++jj) {
          if (t == 0) { I = ii; J = jj; break; }
          --t;
        }
      if (I >= 0) {
        double acc[2][2][2];
        cq_mm16(acc, 16, [=](int i, int k) { return CQX(A, CQ_LD, o + k, 16 * I + i); },
                [=](int k, int j) { return CQX(A, CQ_LD, o + k, 16 * J + j); });
        __syncwarp();
        cq_acc_store(acc, [=](int i, int j, double v) { CQX(A, CQ_LD, 16 * I + i, 16 * J + j) -= v; });
      }
    }
    __syncthreads();
  }
  for (int e = tid; e < 64 * 64; e += blockDim.x) {   // zero the strictly lower part
    const int i = e & 63, j = e >> 6;
    if (i > j) CQX(A, CQ_LD, i, j) = 0.0;
  }
  __syncthreads();
  return true;
}

// ---- modified LU (dorhr_col) of the 64 x 64 A (ld lda) in place: A - D = L U, L unit lower
// (strictly lower part), U upper; D to dsg.  sc: >= 16 doubles of scratch.
__device__ __noinline__ void cq_lu64(double* A, int lda, double* dsg, double* sc) {
  const int tid = threadIdx.x, w = tid >> 5;
  for (int K = 0; K < 4; ++K) {
    const int o = 16 * K;
    if (w == 0) {
      double a[16];
      cq_blk_load(A, lda, o, o, a);
      cq_lu16(a, dsg + o);
      cq_blk_store(A, lda, o, o, a, 0, false);
      if (tid < 16) sc[tid] = 1.0 / a[tid];       // lane j's a[j] = U_jj
    }
    __syncthreads();
    if (K == 3) break;
    if (w < 6 - 2 * K) {   // L(I, K) = A(I, K) U_KK^{-1} (rows), U(K, J) = L_KK^{-1} A(K, J) (columns)
      const bool lpan = w < 3 - K;
      const int b = 16 * (K + 1 + (lpan ? w : w - (3 - K)));
      if (lpan)
        cq_solve_rows_upper([=](int k, int j) { return CQX(A, lda, o + k, o + j); }, sc,
                            [=](int i, int j) -> double& { return CQX(A, lda, b + i, o + j); });
      else
        cq_solve_cols_unit_lower([=](int i, int k) { return CQX(A, lda, o + i, o + k); },
                                 [=](int i, int j) -> double& { return CQX(A, lda, o + i, b + j); });
    }
    __syncthreads();
    {   // trailing A(I, J) -= L(I, K) U(K, J), I, J > K
      const int nt = 3 - K;
      if (w < nt * nt) {
        const int I = 16 * (K + 1 + w / nt), J = 16 * (K + 1 + w % nt);
        double acc[2][2][2];
        cq_mm16(acc, 16, [=](int i, int k) { return CQX(A, lda, I + i, o + k); },
                [=](int k, int j) { return CQX(A, lda, o + k, J + j); });
        __syncwarp();
        cq_acc_store(acc, [=](int i, int j, double v) { CQX(A, lda, I + i, J + j) -= v; });
      }
    }
    __syncthreads();
  }
}

// ---- X = U^{-1} for the 64 x 64 upper triangular accessor u (unit: unit diagonal), X col-major
// (ld ldx, X must not alias u's storage): diagonal blocks by 4 warps, then two levels of
// block merges X12 = -X11 U12 X22 with DMMA tiles
template <class FU>
__device__ __noinline__ void cq_trinv64(FU u, bool unit, double* X, int ldx) {
  const int tid = threadIdx.x, w = tid >> 5;
  if (w < 4) {
    double x[16];
    const int o = 16 * w;
    cq_trinv16([=](int i, int j) { return u(o + i, o + j); }, unit, x);
    cq_blk_store(X, ldx, o, o, x, 1, true);
  }
  for (int e = tid; e < 64 * 64; e += blockDim.x) {   // zero every block below the diagonal blocks
    const int i = e & 63, j = e >> 6;
    if ((i >> 4) > (j >> 4)) CQX(X, ldx, i, j) = 0.0;
  }
  __syncthreads();
  // level 1: blocks (2b, 2b+1), b = 0, 1 (warps 0, 1)
  if (w < 2) {
    const int r = 32 * w, c = r + 16;
    double acc[2][2][2];
    cq_mm16(acc, 16, [=](int i, int k) { return u(r + i, c + k); },
            [=](int k, int j) { return CQX(X, ldx, c + k, c + j); });        // U12 X22
    __syncwarp();
    cq_acc_store(acc, [=](int i, int j, double v) { CQX(X, ldx, r + i, c + j) = v; });
    __syncwarp();
    cq_mm16(acc, 16, [=](int i, int k) { return CQX(X, ldx, r + i, r + k); },
            [=](int k, int j) { return CQX(X, ldx, r + k, c + j); });        // X11 (U12 X22)
    __syncwarp();
    cq_acc_store(acc, [=](int i, int j, double v) { CQX(X, ldx, r + i, c + j) = -v; });
  }
  __syncthreads();
  // level 2: X(0:32, 32:64) = -X(0:32, 0:32) U(0:32, 32:64) X(32:64, 32:64)
  double acc[2][2][2];
  const int I = 16 * (w >> 1), J = 32 + 16 * (w & 1);
  if (w < 4) {   // T = U(0:32, 32:64) X(32:64, 32:64) (X upper: K range 32 .. J + 16)
    cq_mm16(acc, J + 16 - 32, [=](int i, int k) { return u(I + i, 32 + k); },
            [=](int k, int j) { return CQX(X, ldx, 32 + k, J + j); });
    __syncwarp();
    cq_acc_store(acc, [=](int i, int j, double v) { CQX(X, ldx, I + i, J + j) = v; });
  }
  __syncthreads();
  if (w < 4)     // X(I, J) = -X(I, 0:32) T(0:32, J) (X upper: K range I .. 32)
    cq_mm16(acc, 32 - I, [=](int i, int k) { return CQX(X, ldx, I + i, I + k); },
            [=](int k, int j) { return CQX(X, ldx, I + k, J + j); });
  __syncthreads();
  if (w < 4) cq_acc_store(acc, [=](int i, int j, double v) { CQX(X, ldx, I + i, J + j) = -v; });
  __syncthreads();
}

}  // namespace sdc
