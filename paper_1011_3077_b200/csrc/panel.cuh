// panel.cuh -- Householder panel factorisation of a tall m x nb panel (nb <= 64), one
// cooperative kernel, panel resident in shared memory across the whole grid.
//
// Paper: the QR of the 2n x n stack [B_j; -A_j] (Alg. 3 line 3) and of the
// GRURV operands (Alg. 1 line 4, Alg. 2 lines 9/13) is done by
// blocked Householder QR; this kernel is the panel step of it ("communication-avoiding"
// QR: each CTA reads its row block of the panel from HBM once and
// writes it once, the panel never round-trips memory between columns).
//
// Reflector convention: LAPACK dlarfg (reading Q7): beta = -sign(alpha)||x||,
// tau = (beta - alpha)/beta, v = [1; x/(alpha - beta)]; ||x_below|| = 0 -> tau = 0.
//
// Per column k ONE grid-wide reduction of nb numbers suffices:
//   part[j] = sum_{rows r > k} x_r P[r][j],  x = P[:,k]
// gives sigma = ||x_below||^2 (j = k), the update inner products z_j (j > k) and the
// Gram entries x_i^T x (i < k) that build the compact-WY T column:
//   w_j   = tau (P[k][j] + scale z_j),           P[r][j] -= w_j * scale * x_r
//   g_i   = s_i (x_i[k] + scale * part[i]),      T(0:k,k) = -tau T(0:k,0:k) g, T(k,k)=tau
// Reflector columns stay unscaled in shared memory (v_i = s_i x_i, applied at write-back),
// so no thread ever reads a column another thread is rewriting in the same step: 3 CTA
// barriers + 1 grid barrier per column.  Each CTA sums the per-CTA partials in the same
// fixed order, so all CTAs agree bit-for-bit and the result is run-to-run deterministic.
#pragma once
#include <cooperative_groups.h>

#include <algorithm>

#include "common.cuh"
#include "cqr.cuh"

namespace sdc {

constexpr int PANEL_NB = 64;        // max panel width
constexpr int PANEL_THREADS = 512;
constexpr int PANEL_RG = PANEL_THREADS / PANEL_NB;   // row groups (8)

// fixed-order pairwise sum of 16 values
SDC_DEV double tree16(const double* v) {
  return (((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]))) +
         (((v[8] + v[9]) + (v[10] + v[11])) + ((v[12] + v[13]) + (v[14] + v[15])));
}
// fixed-order sum of the first n (<= 16) exchange slots x[c * PANEL_NB]
SDC_DEV double sum_slots(const double* x, int n) {
  double v[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) v[c] = c < n ? x[c * 64] : 0.0;
  return tree16(v);
}

// fixed-order sum of the PANEL_RG row-group partials of column j
SDC_DEV double sum_groups(const double* red, int j) {
  static_assert(PANEL_RG == 8, "tree below");
  const double* r = red + j;
  return ((r[0] + r[64]) + (r[128] + r[192])) + ((r[256] + r[320]) + (r[384] + r[448]));
}
constexpr int PANEL_LD = PANEL_NB + 1;

// (q == i) computed opaquely, so that per-element selects on a register array are not
// folded into a dynamically indexed (local-memory) access
SDC_DEV bool sel_bit(int q, int i) {
  unsigned r;
  asm("{\n .reg .pred p;\n setp.eq.s32 p, %1, %2;\n selp.u32 %0, 1, 0, p;\n}\n" : "=r"(r) : "r"(q), "r"(i));
  return r != 0;
}  // smem row stride (doubles) of the local panel

struct PanelArgs {
  double* P; long long ldp;   // panel (m x nb), factored in place (R upper, v below)
  int m, nb;                  // rows, columns (nb <= PANEL_NB, m >= nb)
  double* Y; long long ldy;   // out: explicit Y (m x nb): 0 above diag, 1 on diag, v below
  double* Yt; long long ldyt; // out: Y^T (nb x m), the K-major operand of C -= Y W
  double* T;                  // out: nb x nb upper-triangular T (ld nb), I - Y T Y^T = H_0..H_{nb-1}
  double* tau;                // out: nb
  double* gbuf;               // workspace: 2 * (gridDim.x + 1) * PANEL_NB doubles
  unsigned int* bar;          // grid barrier counter
  unsigned int bar_base;      // value of *bar before this launch (sum of G*nb of earlier launches)
  int rows_per;               // rows owned per CTA (CTA 0 owns rows [0, rows_per) >= nb)
  unsigned long long* dbg;    // optional phase timers (CTA 0 / last CTA, thread 0), or null
  int zero_above;             // rows above the panel (inside its outer WY block) to zero in Y/Y^T
  int csize;                  // cluster mode: CTAs per cluster (G / csize clusters)
  double* ll;                 // multi-cluster: flag-carrying slots, 2 x (16 + 1) x PANEL_NB x 16 B
  unsigned epoch;             // multi-cluster: flag of column k is epoch + k + 1 (unique per call)
  double* cq;                 // CholeskyQR2 exchange slots (CQ_DOUBLES), flags epoch + 1..3
  int use_cqr;                // try the CholeskyQR2 panel first (cqr.cuh); Householder on breakdown
  unsigned long long* cqstat; // [0] panels factored by CholeskyQR2, [1] Householder fallbacks
};
constexpr size_t PANEL_LL_DOUBLES = 2 * 17 * 64 * 2;

// "LL" exchange through L2: a double travels as two 8-byte words {flag:32 | half:32}; each
// word is single-copy atomic, so a reader that sees both flags sees the value -- no fence,
// no separate counter (one L2 round trip instead of release + counter + acquire + load).
SDC_DEV void ll_store(double* slot, double v, unsigned flag) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  const unsigned long long w0 = ((unsigned long long)flag << 32) | (b & 0xffffffffull);
  const unsigned long long w1 = ((unsigned long long)flag << 32) | (b >> 32);
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};\n" ::"l"(slot), "l"(w0), "l"(w1) : "memory");
}
SDC_DEV bool ll_load(const double* slot, unsigned flag, double& v) {
  unsigned long long w0, w1;
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];\n" : "=l"(w0), "=l"(w1) : "l"(slot) : "memory");
  v = __longlong_as_double((long long)((w1 << 32) | (w0 & 0xffffffffull)));
  return (unsigned)(w0 >> 32) == flag && (unsigned)(w1 >> 32) == flag;
}

// ---- cluster exchange by asynchronous remote stores (st.async + mbarrier tx counts) ----
SDC_DEV uint32_t cluster_map(uint32_t local_smem_addr, int cta) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(local_smem_addr), "r"(cta));
  return r;
}
SDC_DEV void st_async_f64(uint32_t remote_addr, double v, uint32_t remote_mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];\n" ::"r"(remote_addr),
               "l"(__double_as_longlong(v)), "r"(remote_mbar)
               : "memory");
}
SDC_DEV void xmbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
SDC_DEV void xmbar_expect(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
SDC_DEV void xmbar_wait(uint64_t* bar, unsigned parity) {
  uint32_t ok;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  } while (!ok);
}

// T column c of the compact-WY factor (CTA 0), from the step-c reduction results:
//   g_i = s_i (x_i[c] + scale_c * sum_{r>c} x_i[r] x_c[r])  = Y(:,i)^T v_c   (i < c)
//   T(0:c, c) = -tau_c T(0:c, 0:c) g,  T(c, c) = tau_c
// (columns are kept unscaled in shared memory; s_i is the scale that turns x_i into v_i)
SDC_DEV void panel_t_column(double* Ts, int c, const double* tot, const double* drow,
                            const double* sc, const double* tauv) {
  const int i = threadIdx.x >> 2, q = threadIdx.x & 3;
  const double tau = tauv[c], scale = sc[c];
  double acc = 0.0;
  if (i < c)
    for (int l = i + q; l < c; l += 4)
      acc = fma(Ts[l * PANEL_NB + i], sc[l] * fma(scale, tot[l], drow[l]), acc);
  acc += __shfl_xor_sync(0xffffffffu, acc, 1);
  acc += __shfl_xor_sync(0xffffffffu, acc, 2);
  if (i < c && q == 0) Ts[c * PANEL_NB + i] = -tau * acc;
  if (threadIdx.x == 0) Ts[c * PANEL_NB + c] = tau;
}

// CholeskyQR2 + Householder reconstruction of the panel (cqr.cuh).  Ps holds the CTA's R
// rows (row-major, ld PANEL_LD); scr >= CQ_SCRATCH doubles of shared memory.  Returns
// 0: factored -- Ps rows with global index >= 64 hold Y, CTA 0's rows 0..63 hold L (strictly
//    lower) and U; R (with D) is already in P(0:64, 0:64) upper, T and tau in a.T / a.tau;
// 1: breakdown at the first Cholesky (Ps untouched); 2: breakdown at the second (Ps holds
//    Q1: the caller reloads the panel).  Every CTA returns the same code.
__device__ __noinline__ int panel_cqr(const PanelArgs& a, double* Ps, int R, double* scr) {
  const int G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x;
  double* Am = scr;                        // 64 x CQ_LD
  double* Bm = Am + 64 * CQ_LD;            // 64 x CQ_LD
  double* gd = Bm + 64 * CQ_LD;            // Cholesky column norms^2
  double* dsg = gd + 64;                   // D
  double* sc = dsg + 64;                   // 512: diagonal-block inverses
  int* flag = reinterpret_cast<int*>(sc + 512);
  double* Cm = Ps;                         // CTA 0, after Q_top: rows 0..63 as a 64 x 64 (ld 65)
  double* GS = a.T;                        // CTA 0: R1, then R2 R1 (global scratch; T at the end)
  unsigned* err = a.bar + 1;
  double* reg0 = a.cq;
  double* reg1 = a.cq + CQ_REGION;
  double* mreg = a.cq + 2 * (size_t)CQ_REGION;
  const unsigned f1 = a.epoch + 1u, f2 = a.epoch + 2u, f3 = a.epoch + 3u;
  const int eper = (CQ_E + G - 1) / G, e0 = min(CQ_E, cta * eper), e1 = min(CQ_E, e0 + eper);
  // phase timers (SDC_DEBUG_COUNTERS): CTA 0 -> dbg[32..47], last CTA -> dbg[48..63]
  const bool tmd = a.dbg && tid == 0 && (cta == 0 || cta == G - 1);
  unsigned long long tq = tmd ? clock64() : 0ull;
  int ph = 0;
  auto stamp = [&]() {
    if (tmd) {
      const unsigned long long t = clock64();
      atomicAdd(a.dbg + (cta == 0 ? 32 : 48) + ph, t - tq);
      tq = t;
    }
    ++ph;
  };
  auto up = [](int ti, int tj) { return ti; };            // K range of upper x upper tiles:
  auto upk = [](int ti, int tj) { return tj + 1; };       //   blocks ti .. tj
  auto k0 = [](int ti, int tj) { return 0; };
  // (1) G1 = P^T P (owner-reduced through L2), R1 = chol(G1)
  cq_gram_partial(Ps, PANEL_LD, R, reg0 + 2 * (size_t)cta * CQ_E, f1);
  stamp();                                             // 0: Gram 1 partial (thread 0's warp)
  cq_owner_reduce(reg0, G, e0, e1, f1, err);
  stamp();                                             // 1: owner reduce
  cq_gather<true>(reg0 + 2 * (size_t)G * CQ_E, f1, Am, err);
  __syncthreads();
  stamp();                                             // 2: gather
  if (!cq_chol64(Am, gd, sc, flag)) return 1;
  stamp();                                             // 3: chol 1
  // (2) Q1 = P R1^{-1} in place; CTA 0 keeps R1 in GS
  cq_trinv64([=](int i, int j) { return CQX(Am, CQ_LD, i, j); }, false, Bm, CQ_LD);
  stamp();                                             // 4: R1^{-1}
  cq_rows_times_upper(Ps, PANEL_LD, R, 0, Bm);
  if (cta == 0)
    for (int e = tid; e < 64 * 64; e += PANEL_THREADS) GS[e] = CQX(Am, CQ_LD, e & 63, e >> 6);
  __syncthreads();
  stamp();                                             // 5: Q1 = P R1^{-1}
  stamp();                                             // 6: (unused)
  // (3) G2 = Q1^T Q1, R2 = chol(G2)
  cq_gram_partial(Ps, PANEL_LD, R, reg1 + 2 * (size_t)cta * CQ_E, f2);
  cq_owner_reduce(reg1, G, e0, e1, f2, err);
  cq_gather<true>(reg1 + 2 * (size_t)G * CQ_E, f2, Am, err);
  __syncthreads();
  stamp();                                             // 7: Gram 2 (partial + exchange)
  if (!cq_chol64(Am, gd, sc, flag)) return 2;
  stamp();                                             // 8: chol 2
  if (cta == 0) {
    // (4) R2^{-1}; R = R2 R1 (GS); Q_top = Q1(0:64,:) R2^{-1}; Q_top - D = L U
    cq_trinv64([=](int i, int j) { return CQX(Am, CQ_LD, i, j); }, false, Bm, CQ_LD);
    cq_gemm64([=](int i, int k) { return CQX(Am, CQ_LD, i, k); }, [=](int k, int j) { return GS[k + 64 * j]; },
              up, upk, 1.0, [=](int i, int j, double v) { GS[i + 64 * j] = v; });
    cq_gemm64([=](int i, int k) { return Ps[i * PANEL_LD + k]; }, [=](int k, int j) { return CQX(Bm, CQ_LD, k, j); },
              k0, upk, 1.0, [=](int i, int j, double v) { CQX(Am, CQ_LD, i, j) = v; });
    stamp();                                           // 9: R2^{-1}, R, Q_top
    cq_lu64(Am, CQ_LD, dsg, sc);
    stamp();                                           // 10: LU
    // (5) M = R2^{-1} U^{-1} (Bm), published for every CTA
    cq_trinv64([=](int i, int j) { return CQX(Am, CQ_LD, i, j); }, false, Cm, PANEL_LD);
    cq_gemm64([=](int i, int k) { return CQX(Bm, CQ_LD, i, k); }, [=](int k, int j) { return CQX(Cm, PANEL_LD, k, j); },
              up, upk, 1.0, [=](int i, int j, double v) { CQX(Bm, CQ_LD, i, j) = v; });
    for (int p = tid; p < CQ_E; p += PANEL_THREADS) {
      const int j = cq_col(p), i = p - j * (j + 1) / 2;
      cq_ll_store(mreg + 2 * (size_t)p, CQX(Bm, CQ_LD, i, j), f3);
    }
    stamp();                                           // 11: U^{-1}, M published
    // (6) R with D -> P(0:64, 0:64) upper; T = -U D L^{-T} -> a.T, tau; L -> Ps rows 0..63
    for (int e = tid; e < 64 * 64; e += PANEL_THREADS) {
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
    for (int e = tid; e < 64 * 64; e += PANEL_THREADS) {
      const int i = e & 63, j = e >> 6;
      if (i > j) Ps[i * PANEL_LD + j] = CQX(Am, CQ_LD, i, j);
    }
  } else {
    ph = 12;
    cq_gather<false>(mreg, f3, Am, err);
  }
  __syncthreads();
  stamp();                                             // 12: T (CTA 0) / wait for M (others)
  // (7) Y(64:m, :) = Q1 M for the rows below the panel's top 64
  cq_rows_times_upper(Ps, PANEL_LD, R, cta == 0 ? 64 : 0, cta == 0 ? Bm : Am);
  __syncthreads();
  stamp();                                             // 13: Y = Q1 M
  return 0;
}

// CLUSTER = false: G CTAs of a cooperative grid exchange per-CTA partials through L2 and a
//                  grid barrier (any m; used for the tall stacks of large n).
// CLUSTER = true : the G <= 16 CTAs form ONE thread-block cluster and exchange partials
//                  through distributed shared memory with a cluster barrier (~0.2 us instead
//                  of ~1-2 us per column; used when the panel fits in 16 SMs' shared memory).
//
// RPT > 0: the column loop runs out of REGISTERS: thread (jj, rg) holds rows rg + 8i
// (i < RPT) of column jj, so the partial products and the rank-1 update are register FMAs;
// only the reflector column x_k (zeroed at rows <= k, staged by its owner thread during the
// previous update) and row k (CTA 0) pass through shared memory.  RPT = 0: the panel
// stays in shared memory (any rows_per).  Shared memory still stages the coalesced
// load / write-back of the row block.
template <bool CLUSTER, int RPT>
__global__ void __launch_bounds__(PANEL_THREADS)
panel_qr_kernel_t(const PanelArgs a) {
  extern __shared__ __align__(16) double sm[];
  const unsigned long long tstart = clock64();
  constexpr bool REG = RPT > 0;
  constexpr int XS = REG ? PANEL_RG * RPT : 0;      // one staged column (by owner layout)
  const int G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x;
  const int nb = a.nb;
  const int r0 = cta * a.rows_per;
  const int r1 = min(a.m, r0 + a.rows_per);
  const int R = max(0, r1 - r0);
  double* xs = sm;                                  // REG: 2 x XS staged column x_k (parity)
  double* rowst = sm + 2 * XS;                      // REG: row k of the panel (CTA 0)
  double* Ps = rowst + (REG ? PANEL_NB : 0);        // R x PANEL_LD, row-major local block
  double* red = Ps + (size_t)a.rows_per * PANEL_LD; // PANEL_RG x PANEL_NB
  double* totb = red + (PANEL_RG + 1) * PANEL_NB;                // 2 x PANEL_NB (by column parity)
  double* drowb = totb + 2 * PANEL_NB;              // 2 x PANEL_NB
  double* sc = drowb + 2 * PANEL_NB;                // PANEL_NB: v_i = sc[i] * x_i
  double* tauv = sc + PANEL_NB;                     // PANEL_NB
  double* Ts = tauv + PANEL_NB;                     // PANEL_NB x PANEL_NB (T CTA), col-major
  double* xch = Ts + PANEL_NB * PANEL_NB;           // cluster mode: 2 x {-, row k, 16 partials}

  // load the CTA's row block
  // all loads in flight at once (cp.async), one HBM round trip instead of R*nb/threads
  for (int e = tid; e < R * nb; e += PANEL_THREADS) {
    int j = e / R, r = e % R;                       // coalesced along rows
    cp_async_zfill<8>(Ps + r * PANEL_LD + j, a.P + (long long)(r0 + r) + (long long)j * a.ldp, 8);
  }
  cp_async_commit();
  cp_async_wait<0>();
  const int tcta = G - 1;                          // builds T (fewest rows: off the critical path)
  bool cqr_done = false;
  const bool timed = a.dbg && tid == 0 && (cta == 0 || cta == G - 1);
  unsigned long long ph[4] = {0, 0, 0, 0}, tloop = 0, tlend = 0;
  if constexpr (CLUSTER) {
    // CholeskyQR2 + Householder reconstruction: 3 exchanges instead of one per column
    if (a.use_cqr && nb == PANEL_NB) {
      __syncthreads();
      const int rc = panel_cqr(a, Ps, R, red);
      cqr_done = rc == 0;
      if (cta == 0 && tid == 0 && a.cqstat) atomicAdd(a.cqstat + (cqr_done ? 0 : 1), 1ull);
      if (rc == 2) {                               // Ps holds Q1: reload the panel
        for (int e = tid; e < R * nb; e += PANEL_THREADS) {
          int j = e / R, r = e % R;
          cp_async_zfill<8>(Ps + r * PANEL_LD + j, a.P + (long long)(r0 + r) + (long long)j * a.ldp, 8);
        }
        cp_async_commit();
        cp_async_wait<0>();
      }
    }
  }
  if (!cqr_done) {                                 // Householder column loop (fallback)
  if (cta == tcta)
    for (int e = tid; e < PANEL_NB * PANEL_NB; e += PANEL_THREADS) Ts[e] = 0.0;
  __syncthreads();

  uint64_t* xbar = reinterpret_cast<uint64_t*>(xch + 2 * 18 * PANEL_NB);   // 2 exchange mbarriers
  if constexpr (CLUSTER) {
    if (tid == 0) {
      xmbar_init(xbar, 1);
      xmbar_init(xbar + 1, 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    cooperative_groups::this_cluster().sync();   // every peer's barriers exist before any push
  }
  const int jj = tid & (PANEL_NB - 1), rg = tid / PANEL_NB;  // column lane, row group
  double p[REG ? RPT : 1];                          // REG: rows rg + 8i of column jj
  if constexpr (REG) {
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int r = rg + PANEL_RG * i;
      p[i] = (r < R && jj < nb) ? Ps[r * PANEL_LD + jj] : 0.0;
    }
    if (jj == 0) {                                  // stage x_0 (rows > 0)
#pragma unroll
      for (int i = 0; i < RPT; ++i) xs[rg * RPT + i] = r0 + rg + PANEL_RG * i > 0 ? p[i] : 0.0;
    }
    if (cta == 0 && rg == 0) rowst[jj] = p[0];     // row 0
    __syncthreads();
  }
  const int CS = CLUSTER ? a.csize : 1;               // CTAs per cluster
  const int NCL = CLUSTER ? G / CS : 1;               // clusters (> 1: two-level exchange)
  const int crank = cta % CS, cid = cta / CS;
  unsigned long long t0 = 0, t1;
#ifdef SDC_PANEL_SUBPHASES   // fine-grained phase timers (tools/panel_bench.py; costs registers)
  unsigned long long sp[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0}, tsp = 0;
#define PSTAMP(q) if (timed) { const unsigned long long _t = clock64(); sp[q] += _t - tsp; tsp = _t; }
#define PSTAMP0() if (timed) tsp = t0
#else
#define PSTAMP(q)
#define PSTAMP0()
#endif
  tloop = clock64();
  for (int k = 0; k < nb; ++k) {
    if (timed) t0 = clock64();
    PSTAMP0();
    const int lbeg = max(0, k + 1 - r0);               // local rows with global index > k
    // (a) partial inner products part[j] = sum_{r > k} x_r P[r][j], x = P[:,k]
    double s = 0.0;
    const double* xk = xs + (k & 1) * XS + rg * RPT;   // REG: x_k at this thread's rows
    if constexpr (REG) {
      double s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
      for (int i = 0; i < RPT; i += 4) {
        const double2 u = *reinterpret_cast<const double2*>(xk + i);
        const double2 v = *reinterpret_cast<const double2*>(xk + i + 2);
        s = fma(u.x, p[i], s);
        s1 = fma(u.y, p[i + 1], s1);
        s2 = fma(v.x, p[i + 2], s2);
        s3 = fma(v.y, p[i + 3], s3);
      }
      s = (s + s1) + (s2 + s3);
    } else if (jj < nb) {
      // 4 rows per iteration, all 8 loads issued before the FMAs (latency-bound smem loop)
      double s1 = 0.0, s2 = 0.0, s3 = 0.0;
      int r = lbeg + rg;
      for (; r + 3 * PANEL_RG < R; r += 4 * PANEL_RG) {
        const double* q = Ps + r * PANEL_LD;
        const double x0 = q[k], x1 = q[PANEL_RG * PANEL_LD + k], x2 = q[2 * PANEL_RG * PANEL_LD + k],
                     x3 = q[3 * PANEL_RG * PANEL_LD + k];
        const double p0 = q[jj], p1 = q[PANEL_RG * PANEL_LD + jj], p2 = q[2 * PANEL_RG * PANEL_LD + jj],
                     p3 = q[3 * PANEL_RG * PANEL_LD + jj];
        s = fma(x0, p0, s);
        s1 = fma(x1, p1, s1);
        s2 = fma(x2, p2, s2);
        s3 = fma(x3, p3, s3);
      }
      for (; r < R; r += PANEL_RG) s = fma(Ps[r * PANEL_LD + k], Ps[r * PANEL_LD + jj], s);
      s = (s + s1) + (s2 + s3);
    }
    red[rg * PANEL_NB + jj] = s;
    PSTAMP(0);
    __syncthreads();
    double* gb = a.gbuf + (size_t)(k & 1) * (G + 1) * PANEL_NB;
    double* xp = xch + (k & 1) * 18 * PANEL_NB;       // cluster mode exchange slot
    if (tid < nb) {
      const double pv = sum_groups(red, tid);
      if constexpr (CLUSTER) {
        red[PANEL_RG * PANEL_NB + tid] = pv;      // staged for the push below
      } else {
        __stcg(gb + (size_t)cta * PANEL_NB + tid, pv);
        if (cta == 0) __stcg(gb + (size_t)G * PANEL_NB + tid, REG ? rowst[tid] : Ps[k * PANEL_LD + tid]);
      }
    }
    PSTAMP(1);
    if constexpr (CLUSTER) {
      // push: every CTA stores its partial vector (and, single-cluster, CTA 0 row k) into
      // every peer's exchange slot with st.async; each receiver's mbarrier counts the
      // bytes, so no cluster-wide barrier is needed and all reads below are local
      if (tid == 0)
        xmbar_expect(xbar + (k & 1), (unsigned)(CS * nb + (NCL == 1 ? nb : 0)) * 8u);
      __syncthreads();
      if (jj < nb) {
        const double pv = red[PANEL_RG * PANEL_NB + jj];
        const double rv = cta == 0 ? (REG ? rowst[jj] : Ps[k * PANEL_LD + jj]) : 0.0;
        const uint32_t lpart = smem_u32(xp + 2 * PANEL_NB + crank * PANEL_NB + jj);
        const uint32_t lrow = smem_u32(xp + PANEL_NB + jj);
        const uint32_t lbar = smem_u32(xbar + (k & 1));
        for (int d = rg; d < CS; d += PANEL_RG) {
          const uint32_t rbar = cluster_map(lbar, d);
          st_async_f64(cluster_map(lpart, d), pv, rbar);
          if (cta == 0 && NCL == 1) st_async_f64(cluster_map(lrow, d), rv, rbar);
        }
      }
    }
    PSTAMP(2);
    // T column of the previous step (inputs double-buffered), overlapping the exchange
    if (cta == tcta && k > 0)
      panel_t_column(Ts, k - 1, totb + ((k - 1) & 1) * PANEL_NB, drowb + ((k - 1) & 1) * PANEL_NB,
                     sc, tauv);
    PSTAMP(3);
    if (timed) { t1 = clock64(); ph[0] += t1 - t0; t0 = t1; }
    if constexpr (CLUSTER) {
      xmbar_wait(xbar + (k & 1), (k >> 1) & 1);
      PSTAMP(4);
      if (NCL > 1 && tid < nb && crank == 0) {
        // two-level: the cluster leaders publish their cluster's sum (and CTA 0 row k)
        // through L2 as flag-carrying words (read below by every CTA)
        double* ll = a.ll + (size_t)(k & 1) * 17 * PANEL_NB * 2;
        const unsigned flag = a.epoch + (unsigned)k + 1u;
        ll_store(ll + ((size_t)cid * PANEL_NB + tid) * 2, sum_slots(xp + 2 * PANEL_NB + tid, CS), flag);
        if (cta == 0)
          ll_store(ll + ((size_t)16 * PANEL_NB + tid) * 2, REG ? rowst[tid] : Ps[k * PANEL_LD + tid], flag);
      }
    } else {
      grid_barrier(a.bar, a.bar_base + (unsigned)(k + 1) * (unsigned)G);
    }
    PSTAMP(5);
    if (timed) { t1 = clock64(); ph[1] += t1 - t0; t0 = t1; }
    // (b) the column totals tot[j] = sum over all CTAs of part[j] (same fixed order in every
    // CTA) and row k of the panel (owned by CTA 0) -> totb / drowb (double-buffered by
    // column parity: the T column of this step reads them during the next exchange)
    double* totk = totb + (k & 1) * PANEL_NB;
    double* drowk = drowb + (k & 1) * PANEL_NB;
    if (CLUSTER && NCL == 1) {
      if (tid < nb) {
        totk[tid] = sum_slots(xp + 2 * PANEL_NB + tid, CS);
        drowk[tid] = xp[PANEL_NB + tid];
      }
    } else if (CLUSTER) {
      // thread (jj, rg) polls the slots of clusters rg and rg + 8 (and rg = 7 row k)
      double v0 = 0.0, v1 = 0.0;
      if (jj < nb) {
        const double* ll = a.ll + (size_t)(k & 1) * 17 * PANEL_NB * 2;
        const unsigned flag = a.epoch + (unsigned)k + 1u;
        const bool has0 = rg < NCL, has1 = rg + PANEL_RG < NCL, hasr = rg == PANEL_RG - 1;
        double rk = 0.0;
        unsigned polls = 0;
        bool ok;
        do {   // all slots in flight per poll: one L2 round trip once they are written
          ok = true;
          if (has0) ok &= ll_load(ll + ((size_t)rg * PANEL_NB + jj) * 2, flag, v0);
          if (has1) ok &= ll_load(ll + ((size_t)(rg + PANEL_RG) * PANEL_NB + jj) * 2, flag, v1);
          if (hasr) ok &= ll_load(ll + ((size_t)16 * PANEL_NB + jj) * 2, flag, rk);
          if (!ok && ++polls > (1u << 24)) {   // co-residency violated: flag it, do not hang
            atomicExch(a.bar + 1, 1u);
            break;
          }
        } while (!ok);
        if (!has0) v0 = 0.0;
        if (!has1) v1 = 0.0;
        if (hasr) drowk[jj] = rk;
      }
      red[rg * PANEL_NB + jj] = v0 + v1;
      __syncthreads();
      if (tid < nb) totk[tid] = sum_groups(red, tid);
    } else {
      double t = 0.0;
      if (jj < nb) {
        int c = rg;
        for (; c + 7 * PANEL_RG < G; c += 8 * PANEL_RG) {   // 8 independent L2 loads in flight
          double v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = __ldcg(gb + (size_t)(c + PANEL_RG * u) * PANEL_NB + jj);
#pragma unroll
          for (int u = 0; u < 8; ++u) t += v[u];
        }
        for (; c < G; c += PANEL_RG) t += __ldcg(gb + (size_t)c * PANEL_NB + jj);
        if (rg == PANEL_RG - 1) drowk[jj] = __ldcg(gb + (size_t)G * PANEL_NB + jj);
      }
      red[rg * PANEL_NB + jj] = t;
      __syncthreads();
      if (tid < nb) totk[tid] = sum_groups(red, tid);
    }
    __syncthreads();
    PSTAMP(6);
    if (timed) { t1 = clock64(); ph[2] += t1 - t0; t0 = t1; }
    // (c) reflector of column k, computed redundantly by every thread (identical values)
    const double alpha = drowk[k];
    const double sigma = totk[k];
    double tau = 0.0, scale = 0.0, beta = alpha;
    if (sigma != 0.0) {
      // beta = -sign(alpha) nrm, tau = (beta - alpha)/beta = 1 + |alpha|/nrm,
      // scale = 1/(alpha - beta) = sign(alpha)/(|alpha| + nrm): one rsqrt + one reciprocal
      const double q = fma(alpha, alpha, sigma);
      const double rn = rsqrt(q);
      const double nrm = q * rn;
      const double aa = fabs(alpha);
      beta = alpha < 0.0 ? nrm : -nrm;
      tau = fma(aa, rn, 1.0);
      const double sa = __drcp_rn(aa + nrm);
      scale = alpha < 0.0 ? -sa : sa;
    }
    PSTAMP(7);
    if (jj < nb) {
      const double totj = totk[jj];
      const double drowj = drowk[jj];
      if (REG && jj > k) {
        const double w = tau * fma(scale, totj, drowj);
        const double ws = w * scale;
#pragma unroll
        for (int i = 0; i < RPT; i += 2) {             // x_k is 0 at rows <= k
          const double2 u = *reinterpret_cast<const double2*>(xk + i);
          p[i] = fma(-ws, u.x, p[i]);
          p[i + 1] = fma(-ws, u.y, p[i + 1]);
        }
        if (cta == 0 && rg == (k & 7)) {               // diagonal row k
#pragma unroll
          for (int i = 0; i < 8 && i < RPT; ++i) p[i] -= sel_bit(k >> 3, i) ? w : 0.0;
        }
        if (jj == k + 1) {                             // stage x_{k+1} for the next step
          double* xn = xs + ((k + 1) & 1) * XS + rg * RPT;
#pragma unroll
          for (int i = 0; i < RPT; i += 2) *reinterpret_cast<double2*>(xn + i) = make_double2(p[i], p[i + 1]);
          if (cta == 0) {                              // rows <= k+1 (all inside CTA 0's first 64)
#pragma unroll
            for (int i = 0; i < 8 && i < RPT; ++i)
              if (rg + PANEL_RG * i <= k + 1) xn[i] = 0.0;
          }
        }
      } else if (!REG && jj > k) {
        // H_k applied to column jj: w = tau (P[k][jj] + scale z_jj); rows r > k: P -= w scale x_r
        const double w = tau * fma(scale, totj, drowj);
        const double ws = w * scale;
        int r = lbeg + rg;
        for (; r + 3 * PANEL_RG < R; r += 4 * PANEL_RG) {   // loads first, then the stores
          double* q = Ps + r * PANEL_LD;
          const double x0 = q[k], x1 = q[PANEL_RG * PANEL_LD + k], x2 = q[2 * PANEL_RG * PANEL_LD + k],
                       x3 = q[3 * PANEL_RG * PANEL_LD + k];
          const double p0 = q[jj], p1 = q[PANEL_RG * PANEL_LD + jj], p2 = q[2 * PANEL_RG * PANEL_LD + jj],
                       p3 = q[3 * PANEL_RG * PANEL_LD + jj];
          q[jj] = fma(-ws, x0, p0);
          q[PANEL_RG * PANEL_LD + jj] = fma(-ws, x1, p1);
          q[2 * PANEL_RG * PANEL_LD + jj] = fma(-ws, x2, p2);
          q[3 * PANEL_RG * PANEL_LD + jj] = fma(-ws, x3, p3);
        }
        for (; r < R; r += PANEL_RG)
          Ps[r * PANEL_LD + jj] = fma(-ws, Ps[r * PANEL_LD + k], Ps[r * PANEL_LD + jj]);
        if (cta == 0 && rg == 0) Ps[k * PANEL_LD + jj] -= w;      // diagonal row k
      }
    }
    PSTAMP(8);
    if constexpr (REG) {
      if (cta == 0 && rg == (k & 7) && jj == k) {   // beta on the diagonal
#pragma unroll
        for (int i = 0; i < 8 && i < RPT; ++i) p[i] = sel_bit(k >> 3, i) ? beta : p[i];
      }
      if (cta == 0 && rg == ((k + 1) & 7) && jj < nb && k + 1 < nb) {   // stage row k+1
        double v = 0.0;
#pragma unroll
        for (int i = 0; i < 8 && i < RPT; ++i) v += sel_bit((k + 1) >> 3, i) ? p[i] : 0.0;
        rowst[jj] = v;
      }
    }
    if (tid == 0) {
      sc[k] = scale;
      tauv[k] = tau;
      if (cta == 0) { if (!REG) Ps[k * PANEL_LD + k] = beta; a.tau[k] = tau; }
    }
    __syncthreads();
    PSTAMP(9);
    if (timed) { t1 = clock64(); ph[3] += t1 - t0; }
  }
  tlend = clock64();
  if (cta == tcta) {
    panel_t_column(Ts, nb - 1, totb + ((nb - 1) & 1) * PANEL_NB, drowb + ((nb - 1) & 1) * PANEL_NB,
                   sc, tauv);
  }
  if constexpr (REG) {
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int r = rg + PANEL_RG * i;
      if (r < R && jj < nb) Ps[r * PANEL_LD + jj] = p[i];
    }
  }
  if constexpr (CLUSTER) cooperative_groups::this_cluster().sync();  // peers done reading our smem
  else __syncthreads();
  }  // Householder column loop
  if (cqr_done)                                   // CQR path: sc = 1 (Y stored unscaled in Ps)
    for (int j = tid; j < PANEL_NB; j += PANEL_THREADS) sc[j] = 1.0;
  __syncthreads();
  const unsigned long long tend = clock64();

  // write back: R above the diagonal, v = s_j x below it (LAPACK layout), explicit Y, Y^T
  for (int e = tid; e < R * nb; e += PANEL_THREADS) {
    int j = e / R, r = e % R;
    int gr = r0 + r;
    double x = Ps[r * PANEL_LD + j];
    double v = gr > j ? sc[j] * x : x;
    if (!(cqr_done && gr <= j)) a.P[(long long)gr + (long long)j * a.ldp] = v;   // CQR: R written
    a.Y[(long long)gr + (long long)j * a.ldy] = gr > j ? v : (gr == j ? 1.0 : 0.0);
  }
  for (int e = tid; e < R * nb; e += PANEL_THREADS) {     // Y^T: contiguous along j
    int r = e / nb, j = e % nb;
    int gr = r0 + r;
    double v = gr > j ? sc[j] * Ps[r * PANEL_LD + j] : (gr == j ? 1.0 : 0.0);
    a.Yt[(long long)j + (long long)gr * a.ldyt] = v;
  }
  if (cta == tcta && !cqr_done)
    for (int e = tid; e < nb * nb; e += PANEL_THREADS) {
      int j = e / nb, i = e % nb;
      a.T[e] = Ts[j * PANEL_NB + i];
    }
  if (cta == 0) {
    // rows [-zero_above, 0) of this panel's Y columns belong to the outer block: zeros
    for (int e = tid; e < a.zero_above * nb; e += PANEL_THREADS) {
      int j = e / a.zero_above, r = e % a.zero_above - a.zero_above;
      a.Y[(long long)r + (long long)j * a.ldy] = 0.0;
    }
    for (int e = tid; e < a.zero_above * nb; e += PANEL_THREADS) {
      int r = e / nb - a.zero_above, j = e % nb;
      a.Yt[(long long)j + (long long)r * a.ldyt] = 0.0;
    }
  }
  if (timed && !cqr_done) {
    const int o = cta == 0 ? 0 : 4;
    for (int q = 0; q < 4; ++q) atomicAdd(a.dbg + o + q, ph[q]);
#ifdef SDC_PANEL_SUBPHASES
    if (cta == 0)
      for (int q = 0; q < 10; ++q) atomicAdd(a.dbg + 20 + q, sp[q]);
#endif
    atomicAdd(a.dbg + 8, 1ull);
    atomicAdd(a.dbg + 9 + (cta == 0 ? 0 : 3), tloop - tstart);       // prologue
    atomicAdd(a.dbg + 10 + (cta == 0 ? 0 : 3), tlend - tloop - (ph[0] + ph[1] + ph[2] + ph[3]));
    atomicAdd(a.dbg + 16 + (cta == 0 ? 0 : 1), tend - tlend);        // T tail + cluster sync
    atomicAdd(a.dbg + 11 + (cta == 0 ? 0 : 3), clock64() - tend);    // write-back
  }
}

// rows per thread of the register-resident variant for a given rows_per (0: smem variant)
inline int panel_rpt(int rows_per) {
  return rows_per <= 64 ? 8 : rows_per <= 128 ? 16 : rows_per <= 256 ? 32 : 0;
}

inline size_t panel_smem_bytes(int rows_per, bool cqr = false) {
  const int rpt = panel_rpt(rows_per);
  // after the row block: the Householder loop's scratch, or (aliased, only when the CQR path
  // may run) the CQR path's -- the larger footprint would otherwise cost co-resident clusters
  const size_t hh = (PANEL_RG + 1) * PANEL_NB + 4 * PANEL_NB + 2 * PANEL_NB + PANEL_NB * PANEL_NB +
                    36 * PANEL_NB + 2;
  const size_t scratch = cqr ? std::max(hh, (size_t)CQ_SCRATCH) : hh;
  return sizeof(double) * ((size_t)rows_per * PANEL_LD + scratch + (rpt ? 2 * PANEL_RG * rpt + PANEL_NB : 0));
}

#undef PSTAMP
#undef PSTAMP0
}  // namespace sdc
