// gemm.cuh -- FP64 tensor-core GEMM for sm_100a (DMMA.8x8x4 via mma.sync.m8n8k4.f64).
//
//   C[z] (M x N) = alpha * op(A) op(B) [K-slice z] + beta * C[z]     (column-major)
//   optional second output  D2 = alpha2 * op(A) op(B)               (dual epilogue)
//
// Used for every dense contraction of the split step (PAPER.md:
// 916 "matrix multiply", 930 "two n x n matrix multiplications"):
//   * WY trailing updates / complement / Q^T C:  W0 = Y^T C (TN, split-K), C -= Y W (NN)
//   * A_{j+1} = Q12^T A_j, B_{j+1} = Q22^T B_j (TN; dual epilogue writes the next stack)
//   * X = A_p V^T (NT), similarity Q^T (A Q) (NN, TN)
//
// Design: CTA tile BM x BN x BK, warps tiled WM x WN, multistage cp.async (LDGSTS) ring
// in shared memory (zero-fill at ragged edges), fragments read with conflict-free padded
// ld.shared.b64 (ldmatrix has no b64 form), accumulators in registers.  The FP64 tensor
// pipe (128 flop/clk/SM) is slow relative to smem/L2, so operand staging is easy to hide.
#pragma once
#include "common.cuh"

namespace sdc {

struct GemmArgs {
  int M, N, K;
  const double* A; long long lda;
  const double* B; long long ldb;
  double* C; long long ldc;
  double alpha, beta;
  double* D2; long long ldd2; double alpha2;   // optional second output (nullptr: none)
  int kchunk;                 // K per z-slice (multiple of BK); == K when no split
  long long c_zstride;        // element stride between the z-slices of C (split-K partials)
};

template <int BM_, int BN_, int BK_, int WM_, int WN_, int STAGES_>
struct GemmTile {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, WM = WM_, WN = WN_, STAGES = STAGES_;
  static constexpr int WARPS_M = BM / WM, WARPS_N = BN / WN;
  static constexpr int THREADS = WARPS_M * WARPS_N * 32;
  static constexpr int MI = WM / 8, NI = WN / 8;
};

// Shared-memory layout of one stage.  The fragment reads of a half-warp touch a 4 x 4 block
// (4 k-values x 4 m/n-values); an ld of 4 (mod 16) doubles makes those 16 addresses hit
// distinct bank pairs.
template <class T, bool TA, bool TB>
struct GemmSmem {
  // op(A) tile BM x BK:  !TA -> [k][m] (ld BM+4);  TA -> [m][k] (ld BK+4)
  static constexpr int A_LD = TA ? (T::BK + 4) : (T::BM + 4);
  static constexpr int A_ELEMS = TA ? T::BM * A_LD : T::BK * A_LD;
  // op(B) tile BK x BN:  !TB -> [n][k] (ld BK+4);  TB -> [k][n] (ld BN+4)
  static constexpr int B_LD = TB ? (T::BN + 4) : (T::BK + 4);
  static constexpr int B_ELEMS = TB ? T::BK * B_LD : T::BN * B_LD;
  static constexpr int STAGE = A_ELEMS + B_ELEMS;
  static constexpr size_t BYTES = sizeof(double) * (size_t)STAGE * T::STAGES;
};

// Load one K-tile (k0) of op(A) and op(B) into stage buffer sA/sB with cp.async.
// VEC = doubles per cp.async (2 when the operand's rows are 16-byte aligned, else 1).
template <class T, bool TA, bool TB, int VEC>
SDC_DEV void gemm_load_tile(const GemmArgs& g, double* sA, double* sB, int m0, int n0, int k0,
                            int kend) {
  using S = GemmSmem<T, TA, TB>;
  const int tid = threadIdx.x;
  // ---- A ----
  if constexpr (!TA) {
    // global A: M x K col-major; contiguous along m.  chunks of VEC along m.
    constexpr int CPR = T::BM / VEC;               // chunks per k-row
    constexpr int TOTAL = CPR * T::BK;
#pragma unroll
    for (int c = tid; c < TOTAL; c += T::THREADS) {
      int kk = c / CPR, mm = (c % CPR) * VEC;
      int gm = m0 + mm, gk = k0 + kk;
      int valid = (gk < kend) ? min(VEC, max(0, g.M - gm)) : 0;
      const double* src = valid ? g.A + gm + (long long)gk * g.lda : g.A;
      cp_async_zfill<VEC * 8>(sA + kk * S::A_LD + mm, src, valid * 8);
    }
  } else {
    // global A: K x M col-major (op(A) = A^T); contiguous along k.
    constexpr int CPR = T::BK / VEC;
    constexpr int TOTAL = CPR * T::BM;
#pragma unroll
    for (int c = tid; c < TOTAL; c += T::THREADS) {
      int mm = c / CPR, kk = (c % CPR) * VEC;
      int gm = m0 + mm, gk = k0 + kk;
      int valid = (gm < g.M) ? min(VEC, max(0, kend - gk)) : 0;
      const double* src = valid ? g.A + gk + (long long)gm * g.lda : g.A;
      cp_async_zfill<VEC * 8>(sA + mm * S::A_LD + kk, src, valid * 8);
    }
  }
  // ---- B ----
  if constexpr (!TB) {
    // global B: K x N col-major; contiguous along k.
    constexpr int CPR = T::BK / VEC;
    constexpr int TOTAL = CPR * T::BN;
#pragma unroll
    for (int c = tid; c < TOTAL; c += T::THREADS) {
      int nn = c / CPR, kk = (c % CPR) * VEC;
      int gn = n0 + nn, gk = k0 + kk;
      int valid = (gn < g.N) ? min(VEC, max(0, kend - gk)) : 0;
      const double* src = valid ? g.B + gk + (long long)gn * g.ldb : g.B;
      cp_async_zfill<VEC * 8>(sB + nn * S::B_LD + kk, src, valid * 8);
    }
  } else {
    // global B: N x K col-major (op(B) = B^T); contiguous along n.
    constexpr int CPR = T::BN / VEC;
    constexpr int TOTAL = CPR * T::BK;
#pragma unroll
    for (int c = tid; c < TOTAL; c += T::THREADS) {
      int kk = c / CPR, nn = (c % CPR) * VEC;
      int gn = n0 + nn, gk = k0 + kk;
      int valid = (gk < kend) ? min(VEC, max(0, g.N - gn)) : 0;
      const double* src = valid ? g.B + gn + (long long)gk * g.ldb : g.B;
      cp_async_zfill<VEC * 8>(sB + kk * S::B_LD + nn, src, valid * 8);
    }
  }
}

template <class T, bool TA, bool TB, int VEC>
__global__ void __launch_bounds__(T::THREADS)
gemm_dmma_kernel(const GemmArgs g) {
  using S = GemmSmem<T, TA, TB>;
  extern __shared__ __align__(16) double smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp % T::WARPS_M, wn = warp / T::WARPS_M;
  const int m0 = blockIdx.x * T::BM, n0 = blockIdx.y * T::BN;
  const int kbeg = blockIdx.z * g.kchunk;
  const int kend = min(g.K, kbeg + g.kchunk);
  double* C = g.C + (long long)blockIdx.z * g.c_zstride;

  double acc[T::MI][T::NI][2];
#pragma unroll
  for (int i = 0; i < T::MI; ++i)
#pragma unroll
    for (int j = 0; j < T::NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int ktiles = kend > kbeg ? (kend - kbeg + T::BK - 1) / T::BK : 0;
#pragma unroll
  for (int s = 0; s < T::STAGES - 1; ++s) {
    if (s < ktiles)
      gemm_load_tile<T, TA, TB, VEC>(g, smem + s * S::STAGE, smem + s * S::STAGE + S::A_ELEMS,
                                     m0, n0, kbeg + s * T::BK, kend);
    cp_async_commit();
  }

  const int fr = lane >> 2, fc = lane & 3;   // fragment row (m or n), fragment col (k)
  for (int kt = 0; kt < ktiles; ++kt) {
    cp_async_wait<T::STAGES - 2>();
    __syncthreads();
    {
      int nt = kt + T::STAGES - 1;
      if (nt < ktiles) {
        int st = nt % T::STAGES;
        gemm_load_tile<T, TA, TB, VEC>(g, smem + st * S::STAGE, smem + st * S::STAGE + S::A_ELEMS,
                                       m0, n0, kbeg + nt * T::BK, kend);
      }
      cp_async_commit();
    }
    const double* sA = smem + (kt % T::STAGES) * S::STAGE;
    const double* sB = sA + S::A_ELEMS;
#pragma unroll
    for (int kk = 0; kk < T::BK; kk += 4) {
      double af[T::MI], bf[T::NI];
#pragma unroll
      for (int i = 0; i < T::MI; ++i) {
        int m = wm * T::WM + i * 8 + fr, k = kk + fc;
        af[i] = TA ? sA[m * S::A_LD + k] : sA[k * S::A_LD + m];
      }
#pragma unroll
      for (int j = 0; j < T::NI; ++j) {
        int n = wn * T::WN + j * 8 + fr, k = kk + fc;
        bf[j] = TB ? sB[k * S::B_LD + n] : sB[n * S::B_LD + k];
      }
#pragma unroll
      for (int i = 0; i < T::MI; ++i)
#pragma unroll
        for (int j = 0; j < T::NI; ++j) dmma_8x8x4(acc[i][j], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

  // ---- epilogue ----
#pragma unroll
  for (int i = 0; i < T::MI; ++i) {
    int m = m0 + wm * T::WM + i * 8 + fr;
    if (m >= g.M) continue;
#pragma unroll
    for (int j = 0; j < T::NI; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        int n = n0 + wn * T::WN + j * 8 + fc * 2 + h;
        if (n >= g.N) continue;
        double v = acc[i][j][h];
        double* cp = C + m + (long long)n * g.ldc;
        double out = g.alpha * v;
        if (g.beta != 0.0) out = fma(g.beta, *cp, out);
        *cp = out;
        if (g.D2) g.D2[m + (long long)n * g.ldd2] = g.alpha2 * v;
      }
    }
  }
}

}  // namespace sdc
