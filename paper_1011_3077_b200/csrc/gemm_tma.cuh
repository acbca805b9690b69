// gemm_tma.cuh -- warp-specialised FP64 tensor-core GEMM for sm_100a, TMA-fed.
//
//   C[z] (M x N) = alpha * A^T B [K-slice z] + beta * C[z]    ("TN": both operands K-major)
//   optional second output  D2 = alpha2 * A^T B               (dual epilogue)
//
// A is stored K x M column-major (ld lda), B is stored K x N column-major (ld ldb), so
// both tiles are K-contiguous; every contraction of the split step is written in this
// form: W0 = Y^T C, C -= (Y^T)^T W, Q12^T A_j, (A_p^T)^T (V^T), A^T Q, G^T Q.
//
// Pipeline: lane 0 of warp 0 streams 16-deep K slices of the A and B tiles into a
// STAGES-deep shared-memory ring with TMA (cp.async.bulk.tensor.2d, 128-byte swizzle, zero
// fill outside the tensor -> ragged edges need no code), completion tracked by mbarrier
// transaction counts; every warp waits on the slot's "full" barrier, runs
// mma.sync.m8n8k4.f64 (DMMA) on register accumulators and releases the slot through its
// "empty" barrier, which the issuing lane waits on before refilling it.  No
// __syncthreads in the main loop, no per-thread address math.  (A dedicated producer warp
// would put 3 warps on one SM sub-partition and cap the accumulator registers at 168.)
//
// Bank conflicts: with the 128B swizzle, element (row, k) of a 16-wide K slice lives at
// double index row*16 + ((k/2 XOR row%8)*2 + k%2).  A DMMA fragment's half-warp reads 4
// rows x 4 k; mapping fragment row r (0..7) to tile row 2*(r%4) + r/4 makes the 4 rows of a
// half-warp {0,2,4,6} (or {1,3,5,7}) and the 16 addresses distinct mod 16 doubles.
#pragma once
#include <cuda.h>

#include "common.cuh"

namespace sdc {

struct TmaGemmArgs {
  int M, N, K;
  double* C; long long ldc;
  double alpha, beta;
  double* D2; long long ldd2; double alpha2;
  int kchunk;             // K per z-slice (multiple of 16)
  long long c_zstride;    // element stride between z-slices of C
  int red_ok;             // RED tiles: C += alpha A^T B may use bulk reduce-add (host-checked)
  int kupper;             // B_s upper triangular (B_s(k, n) = 0 for k > n): a tile's K loop
                          // stops at its last column (skips products with zeros only)
};

// CPRE: the C tile (beta != 0) is brought into shared memory by TMA at kernel start, in
// 16-row boxes with the same 128B swizzle, so the epilogue of short-K updates (K <= 256,
// C -= Y W) reads C on-chip instead of exposing HBM/L2 latency after the main loop.
// RED (persistent kernel): when beta == 1 the epilogue never reads C: each warp stages
// alpha*acc column segments in shared memory and the bulk-copy engine adds them into C in
// L2 (cp.reduce.async.bulk .add.f64, round-to-nearest: the same RN(C + alpha*acc) as the
// load/FMA/store epilogue, bit for bit), so no C load latency is exposed after the K loop.
template <int BM_, int BN_, int WM_, int WN_, int STAGES_, int MINB_ = 1, bool CPRE_ = false,
          bool RED_ = false>
struct TmaTile {
  static constexpr int BM = BM_, BN = BN_, WM = WM_, WN = WN_, STAGES = STAGES_, MINB = MINB_;
  static constexpr bool CPRE = CPRE_, RED = RED_;
  static constexpr int RED_LD = WM + 2;               // staged column stride (conflict-free)
  static constexpr int RED_WARP = RED ? 2 * 8 * RED_LD : 0;   // 2 buffers x 8 columns
  static constexpr int BK = 16;                       // one 128-byte swizzle row of doubles
  static constexpr int WARPS_M = BM / WM, WARPS_N = BN / WN;
  static constexpr int CWARPS = WARPS_M * WARPS_N;    // all warps consume
  static constexpr int THREADS = CWARPS * 32;
  static constexpr int MI = WM / 8, NI = WN / 8;
  static constexpr int A_BYTES = BM * BK * 8, B_BYTES = BN * BK * 8;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int C_BYTES = CPRE ? BM * BN * 8 : 0;
  static constexpr size_t SMEM =
      (size_t)STAGES * STAGE_BYTES + C_BYTES + (size_t)CWARPS * RED_WARP * 8 + 2 * STAGES * 8 + 16 + 1024;
};

SDC_DEV void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
SDC_DEV void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes) : "memory");
}
SDC_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
SDC_DEV void mbar_wait(uint64_t* bar, unsigned parity) {
  uint32_t ok;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  } while (!ok);
}
SDC_DEV void tma_load_2d(void* dst, const CUtensorMap* tm, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// Tensor-map acquire: the TMA unit caches descriptors by address, and the parameter buffer
// of a launch may reuse an address a descriptor of an earlier (possibly concurrent) launch
// occupied; acquiring through the tensormap proxy makes this launch's descriptor the one used.
SDC_DEV void tmap_acquire(const CUtensorMap* tm) {
#ifdef SDC_TMAP_FENCE
  asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;\n" ::"l"(reinterpret_cast<uint64_t>(tm))
               : "memory");
#else
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(tm)) : "memory");
#endif
}

SDC_DEV void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

SDC_DEV int frag_row(int r) { return 2 * (r & 3) + (r >> 2); }   // conflict-free row map
SDC_DEV int swz(int row, int k) { return row * 16 + ((((k >> 1) ^ (row & 7)) << 1) | (k & 1)); }

template <class T>
__global__ void __launch_bounds__(T::THREADS, T::MINB)
gemm_tn_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmC, const TmaGemmArgs g) {
  extern __shared__ unsigned char smem_raw[];
  // 1024-byte aligned (128B-swizzle atoms); offset arithmetic on the __shared__ pointer keeps
  // the address space visible to the compiler, so fragment loads are LDS, not generic LD
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  double* sC = reinterpret_cast<double*>(base + (size_t)T::STAGES * T::STAGE_BYTES);
  double* sred = reinterpret_cast<double*>(base + (size_t)T::STAGES * T::STAGE_BYTES + T::C_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + (size_t)T::STAGES * T::STAGE_BYTES + T::C_BYTES +
                                               (size_t)T::CWARPS * T::RED_WARP * 8);
  uint64_t* empty = full + T::STAGES;
  uint64_t* cbar = empty + T::STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { tmap_acquire(&tmA); tmap_acquire(&tmB); if (T::CPRE) tmap_acquire(&tmC); }
  // grouped rasterisation (no split-K): consecutive CTAs sweep GROUP M-tiles x all N-tiles
  // column by column, so the ~148 co-resident CTAs share A and B tiles in L2
  int bx = blockIdx.x, by = blockIdx.y;
  if (gridDim.z == 1 && gridDim.x > 16) {
    constexpr int GROUP = 16;
    const int nm = gridDim.x, nn = gridDim.y;
    const int pid = blockIdx.x + blockIdx.y * nm;
    const int width = GROUP * nn, first = (pid / width) * GROUP, gs = min(nm - first, GROUP);
    bx = first + (pid % width) % gs;
    by = (pid % width) / gs;
  }
  const int m0 = bx * T::BM, n0 = by * T::BN;
  const int kbeg = blockIdx.z * g.kchunk;
  const int kend = min(g.kupper ? min(g.K, n0 + T::BN) : g.K, kbeg + g.kchunk);
  const int ktiles = kend > kbeg ? (kend - kbeg + T::BK - 1) / T::BK : 0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < T::STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, T::CWARPS);
    }
    if (T::CPRE) mbar_init(cbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  // stage issue (one lane): tile kt -> slot kt % STAGES, after the slot's previous use
  auto issue = [&](int kt) {
    const int s = kt % T::STAGES;
    if (kt >= T::STAGES) mbar_wait(empty + s, ((kt / T::STAGES) - 1) & 1);
    unsigned char* st = base + (size_t)s * T::STAGE_BYTES;
    mbar_expect_tx(full + s, T::STAGE_BYTES);
    const int k = kbeg + kt * T::BK;
    tma_load_2d(st, &tmA, k, m0, full + s);
    tma_load_2d(st + T::A_BYTES, &tmB, k, n0, full + s);
  };
  const bool cpre = T::CPRE && g.beta != 0.0;
  if (cpre && threadIdx.x == 0) {   // C tile -> smem: BM/16 boxes of 16 rows x BN columns
    mbar_expect_tx(cbar, T::C_BYTES);
#pragma unroll 1
    for (int b = 0; b < T::BM / 16; ++b)
      tma_load_2d(sC + b * 16 * T::BN, &tmC, m0 + 16 * b, n0, cbar);
  }
  if (!cpre && g.beta != 0.0) {   // warm L2 with this CTA's C tile: one prefetch per 128-byte line
    const double* Cz = g.C + (long long)blockIdx.z * g.c_zstride;
    constexpr int LPC = (T::BM * 8 + 127) / 128;            // lines per column
    for (int e = threadIdx.x; e < LPC * T::BN; e += T::THREADS) {
      const int n = n0 + e / LPC, m = m0 + (e % LPC) * 16;
      if (n < g.N && m < g.M)
        asm volatile("prefetch.global.L2 [%0];\n" ::"l"(Cz + m + (long long)n * g.ldc));
    }
  }
  const bool producer = (threadIdx.x == 0);
  if (producer)
    for (int kt = 0; kt < min(ktiles, T::STAGES - 1); ++kt) issue(kt);
  __syncwarp();

  // ---- consumers ----
  const int wm = warp % T::WARPS_M, wn = warp / T::WARPS_M;
  double acc[T::MI][T::NI][2];
#pragma unroll
  for (int i = 0; i < T::MI; ++i)
#pragma unroll
    for (int j = 0; j < T::NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int fr = frag_row(lane >> 2), fc = lane & 3;
  int aoff[T::MI], boff[T::NI];       // fragment row offsets within the stage tile
#pragma unroll
  for (int i = 0; i < T::MI; ++i) aoff[i] = wm * T::WM + i * 8 + fr;
#pragma unroll
  for (int j = 0; j < T::NI; ++j) boff[j] = wn * T::WN + j * 8 + fr;
  // swz(row, 4kq + fc) = row*16 + ktab[kq] for every fragment row (row % 8 == fr)
  int ktab[T::BK / 4];
#pragma unroll
  for (int kq = 0; kq < T::BK / 4; ++kq) ktab[kq] = swz(fr, 4 * kq + fc) - fr * 16;
  const int abase = (wm * T::WM + fr) * 16, bbase = (wn * T::WN + fr) * 16;

  for (int kt = 0; kt < ktiles; ++kt) {
    const int s = kt % T::STAGES;
    if (producer && kt + T::STAGES - 1 < ktiles) issue(kt + T::STAGES - 1);
    __syncwarp();   // the issuing lane may have waited on an "empty" barrier: reconverge warp 0
                    // before the warp-wide mma.sync.aligned below
    mbar_wait(full + s, (kt / T::STAGES) & 1);
    const double* sA = reinterpret_cast<const double*>(base + (size_t)s * T::STAGE_BYTES);
    const double* sB = reinterpret_cast<const double*>(base + (size_t)s * T::STAGE_BYTES + T::A_BYTES);
#pragma unroll
    for (int kq = 0; kq < T::BK / 4; ++kq) {
      // every fragment row r has r % 8 == fr, so the swizzled in-row offset depends only on
      // (kq, lane): rows differ by compile-time multiples of 128 doubles (LDS immediates)
      double af[T::MI], bf[T::NI];
      const double* pa = sA + abase + ktab[kq];
      const double* pb = sB + bbase + ktab[kq];
#pragma unroll
      for (int i = 0; i < T::MI; ++i) af[i] = pa[i * 128];
#pragma unroll
      for (int j = 0; j < T::NI; ++j) bf[j] = pb[j * 128];
#pragma unroll
      for (int i = 0; i < T::MI; ++i)
#pragma unroll
        for (int j = 0; j < T::NI; ++j) dmma_8x8x4(acc[i][j], af[i], bf[j]);
    }
    // WAR across proxies: this warp's LDS reads of the slot (generic proxy) must be ordered
    // before the TMA refill (async proxy) that the arrive below allows.  Without the fence the
    // refill can land under a still-pending read when other kernels load the SMs (observed as
    // a corrupted K slice with two streams running).
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + s);
  }

  // ---- epilogue: C = alpha acc + beta C (C prefetched into L2 at kernel start) ----------
  double* __restrict__ C = g.C + (long long)blockIdx.z * g.c_zstride;
  double* __restrict__ D2 = g.D2;
  const int c0 = frag_row(2 * fc), c1 = frag_row(2 * fc + 1);
  if constexpr (T::RED) {   // beta = 1: bulk reduce-add of alpha*acc into C (see the persistent kernel)
    if (g.red_ok && g.beta == 1.0 && g.D2 == nullptr) {
      const int mw = m0 + wm * T::WM;
      const int rows = min(T::WM, g.M - mw);
#pragma unroll
      for (int j = 0; j < T::NI; ++j) {
        double* buf = sred + (size_t)warp * T::RED_WARP + (j & 1) * 8 * T::RED_LD;
        if (lane < 8) asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
        __syncwarp();
#pragma unroll
        for (int i = 0; i < T::MI; ++i)
#pragma unroll
          for (int h = 0; h < 2; ++h) buf[(h ? c1 : c0) * T::RED_LD + i * 8 + fr] = g.alpha * acc[i][j][h];
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncwarp();
        const int n = n0 + wn * T::WN + j * 8 + lane;
        if (lane < 8 && rows > 0 && n < g.N) {
          asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;\n" ::"l"(
                           C + mw + (long long)n * g.ldc),
                       "r"(smem_u32(buf + lane * T::RED_LD)), "r"(rows * 8)
                       : "memory");
        }
        if (lane < 8) asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      }
      if (lane < 8) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
      return;
    }
  }
  const bool use_beta = g.beta != 0.0;
  if (cpre) mbar_wait(cbar, 0);
#pragma unroll
  for (int i = 0; i < T::MI; ++i) {
    const int m = m0 + aoff[i];
    const bool mok = m < g.M;
    double old[T::NI][2];
    if (use_beta) {          // issue this row-fragment's loads together (MLP), then update
#pragma unroll
      for (int j = 0; j < T::NI; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int nl = wn * T::WN + j * 8 + (h ? c1 : c0);   // tile-local column
          const int n = n0 + nl;
          if (cpre) {   // smem box b = aoff/16 holds rows 16b..16b+15 as [n][16 m] swizzled
            const int ml = aoff[i];
            old[j][h] = sC[(ml >> 4) * 16 * T::BN + nl * 16 +
                           (((((ml & 15) >> 1) ^ (nl & 7)) << 1) | (ml & 1))];
          } else {
            old[j][h] = (mok && n < g.N) ? C[m + (long long)n * g.ldc] : 0.0;
          }
        }
    }
#pragma unroll
    for (int j = 0; j < T::NI; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int n = n0 + wn * T::WN + j * 8 + (h ? c1 : c0);
        if (!mok || n >= g.N) continue;
        const double v = acc[i][j][h];
        double out = g.alpha * v;
        if (use_beta) out = fma(g.beta, old[j][h], out);
        C[m + (long long)n * g.ldc] = out;
        if (D2) D2[m + (long long)n * g.ldd2] = g.alpha2 * v;
      }
  }
}

// ---------------------------------------------------------------------------------------
// Persistent variant: gridDim.x CTAs (<= resident capacity) walk the tile sequence
// t = blockIdx.x, blockIdx.x + gridDim.x, ... (grouped rasterisation inside each K-slice);
// the TMA ring runs continuously across tiles, so the next tile's first K slices are in
// flight while the current tile's epilogue runs (hides the prologue of short-K updates).
// ---------------------------------------------------------------------------------------
template <class T>
__global__ void __launch_bounds__(T::THREADS, T::MINB)
gemm_tn_tma_persist_kernel(const __grid_constant__ CUtensorMap tmA,
                           const __grid_constant__ CUtensorMap tmB, const TmaGemmArgs g) {
  extern __shared__ unsigned char smem_raw[];
  // 1024-byte aligned (128B-swizzle atoms); offset arithmetic on the __shared__ pointer keeps
  // the address space visible to the compiler, so fragment loads are LDS, not generic LD
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  double* sred = reinterpret_cast<double*>(base + (size_t)T::STAGES * T::STAGE_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + (size_t)T::STAGES * T::STAGE_BYTES +
                                               (size_t)T::CWARPS * T::RED_WARP * 8);
  uint64_t* empty = full + T::STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { tmap_acquire(&tmA); tmap_acquire(&tmB); }
  const int tx = (g.M + T::BM - 1) / T::BM, ty = (g.N + T::BN - 1) / T::BN;
  const bool red = T::RED && g.red_ok && g.beta == 1.0 && g.D2 == nullptr;
  unsigned red_chunk = 0;                      // this warp's staged chunks so far (buffer parity)
  const int tz = (g.K + g.kchunk - 1) / g.kchunk;
  const int ntiles = tx * ty * tz;

  auto decode = [&](int t, int& m0, int& n0, int& z) {
    z = t / (tx * ty);
    const int pid = t - z * tx * ty;
    constexpr int GROUP = 16;
    const int width = GROUP * ty, first = (pid / width) * GROUP, gs = min(tx - first, GROUP);
    m0 = (first + (pid % width) % gs) * T::BM;
    n0 = ((pid % width) / gs) * T::BN;
  };
  auto ktiles_of = [&](int z, int n0) {
    const int kb = z * g.kchunk, ke = min(g.kupper ? min(g.K, n0 + T::BN) : g.K, kb + g.kchunk);
    return ke > kb ? (ke - kb + T::BK - 1) / T::BK : 0;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < T::STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, T::CWARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  // producer cursor (thread 0): the (tile, k-slice) stream of this CTA
  const bool producer = (threadIdx.x == 0);
  int p_tile = blockIdx.x, p_kt = 0, p_nk = 0, p_m0 = 0, p_n0 = 0, p_kb = 0;
  unsigned g_issue = 0;
  if (producer && p_tile < ntiles) {
    int z;
    decode(p_tile, p_m0, p_n0, z);
    p_nk = ktiles_of(z, p_n0);
    p_kb = z * g.kchunk;
  }
  auto issue_next = [&]() {
    while (p_tile < ntiles && p_kt >= p_nk) {
      p_tile += gridDim.x;
      p_kt = 0;
      if (p_tile < ntiles) {
        int z;
        decode(p_tile, p_m0, p_n0, z);
        p_nk = ktiles_of(z, p_n0);
        p_kb = z * g.kchunk;
      }
    }
    if (p_tile >= ntiles) return;
    const int s = g_issue % T::STAGES;
    if (g_issue >= (unsigned)T::STAGES) mbar_wait(empty + s, ((g_issue / T::STAGES) - 1) & 1);
    unsigned char* st = base + (size_t)s * T::STAGE_BYTES;
    mbar_expect_tx(full + s, T::STAGE_BYTES);
    const int k = p_kb + p_kt * T::BK;
    tma_load_2d(st, &tmA, k, p_m0, full + s);
    tma_load_2d(st + T::A_BYTES, &tmB, k, p_n0, full + s);
    ++g_issue;
    ++p_kt;
  };
  if (producer)
    for (int i = 0; i < T::STAGES - 1; ++i) issue_next();
  __syncwarp();

  const int wm = warp % T::WARPS_M, wn = warp / T::WARPS_M;
  const int fr = frag_row(lane >> 2), fc = lane & 3;
  int ktab[T::BK / 4];
#pragma unroll
  for (int kq = 0; kq < T::BK / 4; ++kq) ktab[kq] = swz(fr, 4 * kq + fc) - fr * 16;
  const int abase = (wm * T::WM + fr) * 16, bbase = (wn * T::WN + fr) * 16;
  const int c0 = frag_row(2 * fc), c1 = frag_row(2 * fc + 1);
  unsigned gstep = 0;

  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    int m0, n0, z;
    decode(t, m0, n0, z);
    const int nk = ktiles_of(z, n0);
    double* __restrict__ C = g.C + (long long)z * g.c_zstride;
    if (g.beta != 0.0 && !red) {   // warm L2 with this tile's C while its K loop runs
      constexpr int LPC = (T::BM * 8 + 127) / 128;
      for (int e = threadIdx.x; e < LPC * T::BN; e += T::THREADS) {
        const int n = n0 + e / LPC, m = m0 + (e % LPC) * 16;
        if (n < g.N && m < g.M)
          asm volatile("prefetch.global.L2 [%0];\n" ::"l"(C + m + (long long)n * g.ldc));
      }
    }
    double acc[T::MI][T::NI][2];
#pragma unroll
    for (int i = 0; i < T::MI; ++i)
#pragma unroll
      for (int j = 0; j < T::NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int kt = 0; kt < nk; ++kt, ++gstep) {
      const int s = gstep % T::STAGES;
      if (producer) issue_next();
      __syncwarp();   // reconverge warp 0 (see gemm_tn_tma_kernel) before mma.sync.aligned
      mbar_wait(full + s, (gstep / T::STAGES) & 1);
      const double* sA = reinterpret_cast<const double*>(base + (size_t)s * T::STAGE_BYTES);
      const double* sB = reinterpret_cast<const double*>(base + (size_t)s * T::STAGE_BYTES + T::A_BYTES);
#pragma unroll
      for (int kq = 0; kq < T::BK / 4; ++kq) {
        double af[T::MI], bf[T::NI];
        const double* pa = sA + abase + ktab[kq];
        const double* pb = sB + bbase + ktab[kq];
#pragma unroll
        for (int i = 0; i < T::MI; ++i) af[i] = pa[i * 128];
#pragma unroll
        for (int j = 0; j < T::NI; ++j) bf[j] = pb[j * 128];
#pragma unroll
        for (int i = 0; i < T::MI; ++i)
#pragma unroll
          for (int j = 0; j < T::NI; ++j) dmma_8x8x4(acc[i][j], af[i], bf[j]);
      }
      fence_proxy_async_smem();   // WAR across proxies (see gemm_tn_tma_kernel)
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + s);
    }
    // epilogue
    if constexpr (T::RED) {
      if (red) {
        const int mw = m0 + wm * T::WM;                        // this warp's first row
        const int rows = min(T::WM, g.M - mw);                 // even (host: M even)
#pragma unroll
        for (int j = 0; j < T::NI; ++j, ++red_chunk) {
          double* buf = sred + (size_t)warp * T::RED_WARP + (red_chunk & 1) * 8 * T::RED_LD;
          // the bulk reads of the chunk staged two steps ago (same buffer) must be done
          if (lane < 8) asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
          __syncwarp();
#pragma unroll
          for (int i = 0; i < T::MI; ++i)
#pragma unroll
            for (int h = 0; h < 2; ++h)
              buf[(h ? c1 : c0) * T::RED_LD + i * 8 + fr] = g.alpha * acc[i][j][h];
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          __syncwarp();
          const int n = n0 + wn * T::WN + j * 8 + lane;
          if (lane < 8 && rows > 0 && n < g.N) {
            asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;\n" ::"l"(
                             C + mw + (long long)n * g.ldc),
                         "r"(smem_u32(buf + lane * T::RED_LD)), "r"(rows * 8)
                         : "memory");
          }
          if (lane < 8) asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        }
        continue;
      }
    }
    const bool use_beta = g.beta != 0.0;
#pragma unroll
    for (int i = 0; i < T::MI; ++i) {
      const int m = m0 + wm * T::WM + i * 8 + fr;
      const bool mok = m < g.M;
      double old[T::NI][2];
      if (use_beta) {
#pragma unroll
        for (int j = 0; j < T::NI; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int n = n0 + wn * T::WN + j * 8 + (h ? c1 : c0);
            old[j][h] = (mok && n < g.N) ? C[m + (long long)n * g.ldc] : 0.0;
          }
      }
#pragma unroll
      for (int j = 0; j < T::NI; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int n = n0 + wn * T::WN + j * 8 + (h ? c1 : c0);
          if (!mok || n >= g.N) continue;
          const double v = acc[i][j][h];
          double out = g.alpha * v;
          if (use_beta) out = fma(g.beta, old[j][h], out);
          C[m + (long long)n * g.ldc] = out;
          if (g.D2) g.D2[m + (long long)n * g.ldd2] = g.alpha2 * v;
        }
    }
  }
  if (T::RED && red && lane < 8) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

}  // namespace sdc
