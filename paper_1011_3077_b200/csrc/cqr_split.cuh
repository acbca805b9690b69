// cqr_split.cuh -- the CholeskyQR2 panel (cqr.cuh) as a chain of small kernels, for tall
// panels that run NEXT TO the bulk trailing update (look-ahead QR of the 2n x n stack).
//
// The cluster panel kernel keeps its row block in registers, so a 32768-row panel holds 120
// SMs for ~230 us while almost all of that time is a serial 64 x 64 chain on one CTA
// (two Choleskys, the dorhr_col LU, triangular inverses).  Measured at n = 16384: the bulk
// update GEMMs run ~12% slower during a QR than alone, and the lost SM time equals the panels'
// 120 SMs x 230 us (profiles/r02_qr_timeline.txt).  Here the same arithmetic is split by width:
//   k_cqs_gram     (m/256 CTAs)  partial Grams G1 of 256-row chunks               ~5 us
//   k_cqs_mid1     (32 CTAs)     fixed-order sum; the last CTA: R1 = chol(G1), R1^{-1}
//   k_cqs_q1       (m/256 CTAs)  Q1 = P R1^{-1} -> Y, partial Grams G2
//   k_cqs_mid2     (32 CTAs)     sum; last CTA: R2 = chol(G2), R = D R2 R1, Q_top = Q1(0:64,:) R2^{-1},
//                                Q_top - D = L U, M = R2^{-1} U^{-1}, T = -U D L^{-T}
//   k_cqs_y        (m/256 CTAs)  Y = [L; Q1(64:m,:) M], Y^T, v below the diagonal of P
//   k_cqs_fallback (1 CTA)       exits at once unless a Cholesky pivot broke down; then an
//                                unblocked Householder panel on global memory (slow, rare)
// The wide kernels are bandwidth-trivial and the serial chains occupy ONE SM, so the bulk
// GEMM keeps the other 147.  No CTA waits on another (no flags, no co-residency requirement).
// Same formulas, pivot rule and fixed summation orders as panel_cqr(): deterministic, and
// the compact-WY factor is a valid Householder factor of the panel (reading Q22).
#pragma once
#include "batched.cuh"
#include "cqr.cuh"
#include "panel.cuh"

namespace sdc {

constexpr int CQS_ROWS = 256;               // rows per wide CTA (two 128-row sub-blocks)
constexpr int CQS_SUB = 128;
constexpr int CQS_GMAX = 192;               // most wide CTAs (m <= 49152)
constexpr int CQS_MIDS = 32;                // CTAs of the reduction stage
constexpr int CQS_EPER = (CQ_E + CQS_MIDS - 1) / CQS_MIDS;   // 65 packed entries per CTA
// workspace (doubles): 2 x partial Grams, the reduced Gram, R1 / R1^{-1} / M (64 x 64, ld 64)
constexpr size_t CQS_DOUBLES = 2 * (size_t)CQS_GMAX * CQ_E + CQ_E + 3 * 64 * 64;
constexpr size_t CQS_WIDE_SMEM = sizeof(double) * ((size_t)CQS_SUB * PANEL_LD + 64 * CQ_LD);
constexpr size_t CQS_MID_SMEM = sizeof(double) * (2 * 64 * CQ_LD + 2 * 64 + 512 + 8 + 64 * PANEL_LD);

struct CqsArgs {
  double* P; long long ldp; int m;       // panel (m x 64, m >= 64), factored in place
  double* Y; long long ldy;              // out: explicit Y (also holds Q1 between the stages)
  double* Yt; long long ldyt;            // out: Y^T
  double* T; double* tau;                // out: 64 x 64 T (ld 64), tau
  int zero_above;
  double* ws;                            // CQS_DOUBLES
  unsigned* sync;                        // [0] breakdown of THIS panel, [1] arrival counter (self-
                                         // resetting), [2] breakdowns since reset (host reads it)
};
SDC_DEV double* cqs_part(const CqsArgs& a, int which) { return a.ws + (size_t)which * CQS_GMAX * CQ_E; }
SDC_DEV double* cqs_red(const CqsArgs& a) { return a.ws + 2 * (size_t)CQS_GMAX * CQ_E; }
SDC_DEV double* cqs_mat(const CqsArgs& a, int which) { return cqs_red(a) + CQ_E + (size_t)which * 64 * 64; }

// rows [r0, r0 + R) of the 64-column matrix X (col-major, ld ldx) -> Ps (row-major, ld PANEL_LD)
SDC_DEV void cqs_load_rows(double* Ps, const double* X, long long ldx, int r0, int R) {
  for (int e = threadIdx.x; e < R * 64; e += blockDim.x) {
    const int j = e / R, r = e % R;
    cp_async_zfill<8>(Ps + r * PANEL_LD + j, X + (long long)(r0 + r) + (long long)j * ldx, 8);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
}

// acc += (rows of Ps)^T (rows of Ps) for this warp's 16 x 16 tile (ti, tj) of the Gram
SDC_DEV void cqs_gram_acc(double (&acc)[2][2][2], const double* Ps, int R) {
  const int w = threadIdx.x >> 5, ti = w >> 2, tj = w & 3;
  const int K = (R + 3) & ~3;
  cq_tile16(acc, 0, K,
            [=](int i, int k) { return k < R ? Ps[k * PANEL_LD + 16 * ti + i] : 0.0; },
            [=](int k, int j) { return k < R ? Ps[k * PANEL_LD + 16 * tj + j] : 0.0; });
}
SDC_DEV void cqs_gram_store(const double (&acc)[2][2][2], double* part) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, ti = w >> 2, tj = w & 3;
  const int lr = lane >> 2, lc = lane & 3;
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int i = 16 * ti + 8 * mi + lr, j = 16 * tj + 8 * ni + 2 * lc + c;
        if (i <= j) part[j * (j + 1) / 2 + i] = acc[mi][ni][c];
      }
}

// (1) partial Gram of the CTA's rows of P
__global__ void __launch_bounds__(512) k_cqs_gram(const CqsArgs a) {
  extern __shared__ __align__(16) double sm_cqs[];
  double* Ps = sm_cqs;
  const int cta = blockIdx.x, r0 = cta * CQS_ROWS, r1 = min(a.m, r0 + CQS_ROWS);
  if (cta == 0 && threadIdx.x == 0) a.sync[0] = 0u;        // this panel: no breakdown yet
  double acc[2][2][2] = {};
  for (int s0 = r0; s0 < r1; s0 += CQS_SUB) {
    const int R = min(CQS_SUB, r1 - s0);
    __syncthreads();
    cqs_load_rows(Ps, a.P, a.ldp, s0, R);
    cqs_gram_acc(acc, Ps, R);
  }
  cqs_gram_store(acc, cqs_part(a, 0) + (size_t)cta * CQ_E);
}

// fixed-order sum of the G partials of this CTA's packed entries -> red; true in the LAST CTA
// to arrive (which then sees every entry of red)
SDC_DEV bool cqs_reduce_arrive(const CqsArgs& a, const double* part, int G) {
  __shared__ unsigned last;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int e0 = blockIdx.x * CQS_EPER, e1 = min(CQ_E, e0 + CQS_EPER);
  double* red = cqs_red(a);
  for (int e = e0 + w; e < e1; e += 16) {
    double s = 0.0;
    for (int g = lane; g < G; g += 32) s += part[(size_t)g * CQ_E + e];
    s += __shfl_xor_sync(0xffffffffu, s, 16);
    s += __shfl_xor_sync(0xffffffffu, s, 8);
    s += __shfl_xor_sync(0xffffffffu, s, 4);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    if (lane == 0) red[e] = s;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned old = atomicAdd(a.sync + 1, 1u);
    last = old == gridDim.x - 1 ? 1u : 0u;
    if (last) a.sync[1] = 0u;                               // ready for the next stage
  }
  __syncthreads();
  if (last) __threadfence();
  return last != 0u;
}

// packed upper triangle (global) -> symmetric 64 x 64 (ld CQ_LD) in shared memory
SDC_DEV void cqs_unpack_sym(const double* red, double* M) {
  for (int p = threadIdx.x; p < CQ_E; p += blockDim.x) {
    const int j = cq_col(p), i = p - j * (j + 1) / 2;
    const double v = __ldcg(red + p);
    M[j + i * CQ_LD] = v;
    M[i + j * CQ_LD] = v;
  }
  __syncthreads();
}
SDC_DEV void cqs_breakdown(const CqsArgs& a) {
  if (threadIdx.x == 0) { a.sync[0] = 1u; atomicAdd(a.sync + 2, 1u); }
}

// (2) G1 summed; last CTA: R1 = chol(G1) -> mat 0, R1^{-1} -> mat 1
__global__ void __launch_bounds__(512) k_cqs_mid1(const CqsArgs a, int G) {
  extern __shared__ __align__(16) double sm_cqs[];
  if (!cqs_reduce_arrive(a, cqs_part(a, 0), G)) return;
  double* Am = sm_cqs;
  double* Bm = Am + 64 * CQ_LD;
  double* gd = Bm + 64 * CQ_LD;
  double* sc = gd + 128;
  int* flag = reinterpret_cast<int*>(sc + 512);
  cqs_unpack_sym(cqs_red(a), Am);
  if (!cq_chol64(Am, gd, sc, flag)) { cqs_breakdown(a); return; }
  cq_trinv64([=](int i, int j) { return CQX(Am, CQ_LD, i, j); }, false, Bm, CQ_LD);
  double *R1 = cqs_mat(a, 0), *R1i = cqs_mat(a, 1);
  for (int e = threadIdx.x; e < 64 * 64; e += blockDim.x) {
    R1[e] = CQX(Am, CQ_LD, e & 63, e >> 6);
    R1i[e] = CQX(Bm, CQ_LD, e & 63, e >> 6);
  }
}

// 64 x 64 matrix (global, ld 64) -> shared (ld CQ_LD)
SDC_DEV void cqs_load_mat(double* Bm, const double* src) {
  for (int e = threadIdx.x; e < 64 * 64; e += blockDim.x) CQX(Bm, CQ_LD, e & 63, e >> 6) = __ldcg(src + e);
  __syncthreads();
}

// (3) Q1 = P R1^{-1} -> Y (rows of this CTA), partial Gram of Q1
__global__ void __launch_bounds__(512) k_cqs_q1(const CqsArgs a) {
  extern __shared__ __align__(16) double sm_cqs[];
  if (*(volatile unsigned*)a.sync) return;
  double* Ps = sm_cqs;
  double* Bm = Ps + CQS_SUB * PANEL_LD;
  const int cta = blockIdx.x, r0 = cta * CQS_ROWS, r1 = min(a.m, r0 + CQS_ROWS);
  cqs_load_mat(Bm, cqs_mat(a, 1));
  double acc[2][2][2] = {};
  for (int s0 = r0; s0 < r1; s0 += CQS_SUB) {
    const int R = min(CQS_SUB, r1 - s0);
    __syncthreads();
    cqs_load_rows(Ps, a.P, a.ldp, s0, R);
    cq_rows_times_upper(Ps, PANEL_LD, R, 0, Bm);
    __syncthreads();
    for (int e = threadIdx.x; e < R * 64; e += blockDim.x) {
      const int j = e / R, r = e % R;
      a.Y[(long long)(s0 + r) + (long long)j * a.ldy] = Ps[r * PANEL_LD + j];
    }
    cqs_gram_acc(acc, Ps, R);
  }
  cqs_gram_store(acc, cqs_part(a, 1) + (size_t)cta * CQ_E);
}

// (4) G2 summed; last CTA: the serial 64 x 64 chain of panel_cqr() steps (3)-(6)
__global__ void __launch_bounds__(512) k_cqs_mid2(const CqsArgs a, int G) {
  extern __shared__ __align__(16) double sm_cqs[];
  if (*(volatile unsigned*)a.sync) return;
  if (!cqs_reduce_arrive(a, cqs_part(a, 1), G)) return;
  const int tid = threadIdx.x;
  double* Am = sm_cqs;
  double* Bm = Am + 64 * CQ_LD;
  double* gd = Bm + 64 * CQ_LD;
  double* dsg = gd + 64;
  double* sc = dsg + 64;
  int* flag = reinterpret_cast<int*>(sc + 512);
  double* Ps = sc + 512 + 8;                 // Q1(0:64, :) row-major (ld PANEL_LD); later U^{-1}, L^{-T}
  double* Cm = Ps;
  double* GS = cqs_mat(a, 0);                // R1, then R2 R1 (global)
  auto up = [](int ti, int tj) { return ti; };
  auto upk = [](int ti, int tj) { return tj + 1; };
  auto k0 = [](int ti, int tj) { return 0; };
  cqs_unpack_sym(cqs_red(a), Am);
  if (!cq_chol64(Am, gd, sc, flag)) { cqs_breakdown(a); return; }
  for (int e = tid; e < 64 * 64; e += blockDim.x) {          // Q1(0:64, :) (written by k_cqs_q1)
    const int i = e & 63, j = e >> 6;
    Ps[i * PANEL_LD + j] = __ldcg(a.Y + (long long)i + (long long)j * a.ldy);
  }
  // R2^{-1}; R = R2 R1 (GS); Q_top = Q1(0:64,:) R2^{-1}; Q_top - D = L U
  cq_trinv64([=](int i, int j) { return CQX(Am, CQ_LD, i, j); }, false, Bm, CQ_LD);
  cq_gemm64([=](int i, int k) { return CQX(Am, CQ_LD, i, k); }, [=](int k, int j) { return GS[k + 64 * j]; },
            up, upk, 1.0, [=](int i, int j, double v) { GS[i + 64 * j] = v; });
  cq_gemm64([=](int i, int k) { return Ps[i * PANEL_LD + k]; }, [=](int k, int j) { return CQX(Bm, CQ_LD, k, j); },
            k0, upk, 1.0, [=](int i, int j, double v) { CQX(Am, CQ_LD, i, j) = v; });
  cq_lu64(Am, CQ_LD, dsg, sc);
  // M = R2^{-1} U^{-1} -> mat 2
  cq_trinv64([=](int i, int j) { return CQX(Am, CQ_LD, i, j); }, false, Cm, PANEL_LD);
  cq_gemm64([=](int i, int k) { return CQX(Bm, CQ_LD, i, k); }, [=](int k, int j) { return CQX(Cm, PANEL_LD, k, j); },
            up, upk, 1.0, [=](int i, int j, double v) { CQX(Bm, CQ_LD, i, j) = v; });
  double* Mg = cqs_mat(a, 2);
  for (int e = tid; e < 64 * 64; e += blockDim.x) {
    const int i = e & 63, j = e >> 6;
    Mg[e] = i <= j ? CQX(Bm, CQ_LD, i, j) : 0.0;
  }
  __threadfence();
  __syncthreads();
  // R with D -> P(0:64, 0:64) upper; T = -U D L^{-T} -> a.T, tau; L -> Y(0:64, :) strictly lower
  for (int e = tid; e < 64 * 64; e += blockDim.x) {
    const int i = e & 63, j = e >> 6;
    if (i <= j) a.P[(long long)i + (long long)j * a.ldp] = dsg[i] * GS[e];
  }
  cq_trinv64([=](int i, int j) { return i < j ? CQX(Am, CQ_LD, j, i) : (i == j ? 1.0 : 0.0); }, true, Cm, PANEL_LD);
  cq_gemm64([=](int i, int k) { return k >= i ? CQX(Am, CQ_LD, i, k) * dsg[k] : 0.0; },
            [=](int k, int j) { return CQX(Cm, PANEL_LD, k, j); }, up, upk, -1.0,
            [=](int i, int j, double v) {
              a.T[i + 64 * j] = v;
              if (i == j) a.tau[i] = v;
            });
  for (int e = tid; e < 64 * 64; e += blockDim.x) {
    const int i = e & 63, j = e >> 6;
    if (i > j) a.Y[(long long)i + (long long)j * a.ldy] = CQX(Am, CQ_LD, i, j);
  }
}

// (5) Y(64:m, :) = Q1(64:m, :) M; explicit Y, Y^T, v below the diagonal of P
__global__ void __launch_bounds__(512) k_cqs_y(const CqsArgs a) {
  extern __shared__ __align__(16) double sm_cqs[];
  if (*(volatile unsigned*)a.sync) return;
  double* Ps = sm_cqs;
  double* Bm = Ps + CQS_SUB * PANEL_LD;
  const int cta = blockIdx.x, r0 = cta * CQS_ROWS, r1 = min(a.m, r0 + CQS_ROWS), tid = threadIdx.x;
  cqs_load_mat(Bm, cqs_mat(a, 2));
  for (int s0 = r0; s0 < r1; s0 += CQS_SUB) {
    const int R = min(CQS_SUB, r1 - s0);
    __syncthreads();
    cqs_load_rows(Ps, a.Y, a.ldy, s0, R);
    cq_rows_times_upper(Ps, PANEL_LD, R, s0 < 64 ? min(R, 64 - s0) : 0, Bm);   // rows < 64 hold L
    __syncthreads();
    for (int e = tid; e < R * 64; e += blockDim.x) {
      const int j = e / R, r = e % R, gr = s0 + r;
      const double x = Ps[r * PANEL_LD + j];
      if (gr > j) a.P[(long long)gr + (long long)j * a.ldp] = x;
      a.Y[(long long)gr + (long long)j * a.ldy] = gr > j ? x : (gr == j ? 1.0 : 0.0);
    }
    for (int e = tid; e < R * 64; e += blockDim.x) {          // Y^T: contiguous along j
      const int r = e / 64, j = e % 64, gr = s0 + r;
      a.Yt[(long long)j + (long long)gr * a.ldyt] = gr > j ? Ps[r * PANEL_LD + j] : (gr == j ? 1.0 : 0.0);
    }
  }
  if (cta == 0) {   // rows [-zero_above, 0) of this panel's Y columns belong to the outer block: zeros
    for (int e = tid; e < a.zero_above * 64; e += blockDim.x) {
      const int j = e / a.zero_above, r = e % a.zero_above - a.zero_above;
      a.Y[(long long)r + (long long)j * a.ldy] = 0.0;
    }
    for (int e = tid; e < a.zero_above * 64; e += blockDim.x) {
      const int r = e / 64 - a.zero_above, j = e % 64;
      a.Yt[(long long)j + (long long)r * a.ldyt] = 0.0;
    }
  }
}

// (6) breakdown only: unblocked Householder QR of the panel in global memory by ONE CTA (the
// batched kernel's bq_qr: unscaled reflector columns, compact-WY T).  Rank-revealing where
// CholeskyQR is not; ~100x slower than the cluster panel, which is why the host stops using the
// split chain on a handle once a step has reported a breakdown.
__global__ void __launch_bounds__(BQ_THREADS, 1) k_cqs_fallback(const CqsArgs a) {
  extern __shared__ __align__(16) double sm_cqs[];
  if (*(volatile unsigned*)a.sync == 0u) return;
  const int tid = threadIdx.x, tld = CQ_LD;
  double* T = sm_cqs;                      // 64 x tld
  double* sc = T + 64 * tld;
  double* beta = sc + 64;
  double* g = beta + 64;
  double* drow = g + 64;
  bq_qr(a.m, 64, 64, a.P, (int)a.ldp, T, tld, sc, beta, g, drow);
  __syncthreads();
  for (long long e = tid; e < (long long)a.m * 64; e += BQ_THREADS) {
    const int j = (int)(e / a.m), r = (int)(e % a.m);
    const double x = a.P[(long long)r + (long long)j * a.ldp];
    const double v = r > j ? sc[j] * x : (r == j ? beta[j] : x);
    a.P[(long long)r + (long long)j * a.ldp] = v;
    const double y = r > j ? v : (r == j ? 1.0 : 0.0);
    a.Y[(long long)r + (long long)j * a.ldy] = y;
    a.Yt[(long long)j + (long long)r * a.ldyt] = y;
  }
  for (int e = tid; e < 64 * 64; e += BQ_THREADS) {
    const int i = e & 63, j = e >> 6;
    a.T[e] = i <= j ? T[i + j * tld] : 0.0;
    if (i == j) a.tau[i] = T[i + j * tld];
  }
  for (int e = tid; e < a.zero_above * 64; e += BQ_THREADS) {
    const int j = e / a.zero_above, r = e % a.zero_above - a.zero_above;
    a.Y[(long long)r + (long long)j * a.ldy] = 0.0;
    a.Yt[(long long)j + (long long)r * a.ldyt] = 0.0;
  }
}
constexpr size_t CQS_FB_SMEM = sizeof(double) * (64 * CQ_LD + 4 * 64);

}  // namespace sdc
