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

#include "common.cuh"

namespace sdc {

constexpr int PANEL_NB = 64;        // max panel width
constexpr int PANEL_THREADS = 512;
constexpr int PANEL_RG = PANEL_THREADS / PANEL_NB;   // row groups (8)

// fixed-order sum of the PANEL_RG row-group partials of column j
SDC_DEV double sum_groups(const double* red, int j) {
  double t = 0.0;
#pragma unroll
  for (int g = 0; g < PANEL_RG; ++g) t += red[g * 64 + j];
  return t;
}
constexpr int PANEL_LD = PANEL_NB + 1;  // smem row stride (doubles) of the local panel

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
};

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
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
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

// CLUSTER = false: G CTAs of a cooperative grid exchange per-CTA partials through L2 and a
//                  grid barrier (any m; used for the tall stacks of large n).
// CLUSTER = true : the G <= 16 CTAs form ONE thread-block cluster and exchange partials
//                  through distributed shared memory with a cluster barrier (~0.2 us instead
//                  of ~1-2 us per column; used when the panel fits in 16 SMs' shared memory).
template <bool CLUSTER>
__global__ void __launch_bounds__(PANEL_THREADS)
panel_qr_kernel_t(const PanelArgs a) {
  extern __shared__ __align__(16) double sm[];
  const int G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x;
  const int nb = a.nb;
  const int r0 = cta * a.rows_per;
  const int r1 = min(a.m, r0 + a.rows_per);
  const int R = max(0, r1 - r0);
  double* Ps = sm;                                  // R x PANEL_LD, row-major local block
  double* red = Ps + (size_t)a.rows_per * PANEL_LD; // PANEL_RG x PANEL_NB
  double* totb = red + (PANEL_RG + 1) * PANEL_NB;                // 2 x PANEL_NB (by column parity)
  double* drowb = totb + 2 * PANEL_NB;              // 2 x PANEL_NB
  double* sc = drowb + 2 * PANEL_NB;                // PANEL_NB: v_i = sc[i] * x_i
  double* tauv = sc + PANEL_NB;                     // PANEL_NB
  double* Ts = tauv + PANEL_NB;                     // PANEL_NB x PANEL_NB (T CTA), col-major
  double* xch = Ts + PANEL_NB * PANEL_NB;           // cluster mode: 2 x {-, row k, 16 partials}

  // load the CTA's row block
  for (int e = tid; e < R * nb; e += PANEL_THREADS) {
    int j = e / R, r = e % R;                       // coalesced along rows
    Ps[r * PANEL_LD + j] = a.P[(long long)(r0 + r) + (long long)j * a.ldp];
  }
  const int tcta = G - 1;                          // builds T (fewest rows: off the critical path)
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
  const bool timed = a.dbg && tid == 0 && (cta == 0 || cta == G - 1);
  unsigned long long ph[4] = {0, 0, 0, 0}, t0 = 0, t1;
  for (int k = 0; k < nb; ++k) {
    if (timed) t0 = clock64();
    const int lbeg = max(0, k + 1 - r0);               // local rows with global index > k
    // (a) partial inner products part[j] = sum_{r > k} x_r P[r][j], x = P[:,k]
    double s = 0.0;
    if (jj < nb) {
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
    __syncthreads();
    double* gb = a.gbuf + (size_t)(k & 1) * (G + 1) * PANEL_NB;
    double* xp = xch + (k & 1) * 18 * PANEL_NB;       // cluster mode exchange slot
    if (tid < nb) {
      double p = sum_groups(red, tid);
      if constexpr (CLUSTER) {
        red[PANEL_RG * PANEL_NB + tid] = p;       // staged for the push below
      } else {
        __stcg(gb + (size_t)cta * PANEL_NB + tid, p);
        if (cta == 0) __stcg(gb + (size_t)G * PANEL_NB + tid, Ps[k * PANEL_LD + tid]);  // row k
      }
    }
    const int CS = CLUSTER ? a.csize : 1;               // CTAs per cluster
    const int NCL = CLUSTER ? G / CS : 1;               // clusters (> 1: two-level exchange)
    const int crank = cta % CS, cid = cta / CS;
    if constexpr (CLUSTER) {
      // push: every CTA stores its partial vector (and, single-cluster, CTA 0 row k) into
      // every peer's exchange slot with st.async; each receiver's mbarrier counts the
      // bytes, so no cluster-wide barrier is needed and all reads below are local
      if (tid == 0)
        xmbar_expect(xbar + (k & 1), (unsigned)(CS * nb + (NCL == 1 ? nb : 0)) * 8u);
      __syncthreads();
      if (jj < nb) {
        const double pv = red[PANEL_RG * PANEL_NB + jj];
        const double rv = cta == 0 ? Ps[k * PANEL_LD + jj] : 0.0;
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
    // T column of the previous step (inputs double-buffered), overlapping the exchange
    if (cta == tcta && k > 0)
      panel_t_column(Ts, k - 1, totb + ((k - 1) & 1) * PANEL_NB, drowb + ((k - 1) & 1) * PANEL_NB,
                     sc, tauv);
    if (timed) { t1 = clock64(); ph[0] += t1 - t0; t0 = t1; }
    if constexpr (CLUSTER) {
      xmbar_wait(xbar + (k & 1), (k >> 1) & 1);
      if (NCL > 1) {
        // two-level: every CTA forms its cluster's sum (same fixed order); the leaders
        // publish them (and CTA 0 row k) through L2; one counter arrival per cluster
        double t = 0.0;
        if (jj < nb) {
#pragma unroll
          for (int u = 0; u < 16 / PANEL_RG; ++u) {
            const int c = rg + PANEL_RG * u;
            t += c < CS ? xp[2 * PANEL_NB + c * PANEL_NB + jj] : 0.0;
          }
        }
        red[rg * PANEL_NB + jj] = t;
        __syncthreads();
        if (tid < nb && crank == 0) {
          __stcg(gb + (size_t)cid * PANEL_NB + tid, sum_groups(red, tid));
          if (cta == 0) __stcg(gb + (size_t)NCL * PANEL_NB + tid, Ps[k * PANEL_LD + tid]);
        }
        leaders_barrier(a.bar, a.bar_base + (unsigned)(k + 1) * (unsigned)NCL, crank == 0);
      }
    } else {
      grid_barrier(a.bar, a.bar_base + (unsigned)(k + 1) * (unsigned)G);
    }
    if (timed) { t1 = clock64(); ph[1] += t1 - t0; t0 = t1; }
    // row k of the panel (owned by CTA 0): local in cluster mode; in grid mode staged into
    // shared memory by the rg == last group during the partial-sum loads (same L2 round trip)
    double* rows = red + PANEL_RG * PANEL_NB;          // staging row (free after the push)
    const double* row0;
    if (CLUSTER && NCL == 1) row0 = xp + PANEL_NB;
    else row0 = rows;
    if ((!CLUSTER || NCL > 1) && rg == PANEL_RG - 1 && jj < nb)
      rows[jj] = __ldcg(gb + (size_t)(CLUSTER ? NCL : G) * PANEL_NB + jj);
    // (b) every CTA sums the per-CTA (per-cluster) partials in the same fixed order
    if (CLUSTER && NCL > 1) {
      double t = 0.0;
      if (jj < nb) {
#pragma unroll
        for (int u = 0; u < 16 / PANEL_RG; ++u) {
          const int c = rg + PANEL_RG * u;
          t += c < NCL ? __ldcg(gb + (size_t)c * PANEL_NB + jj) : 0.0;
        }
      }
      red[rg * PANEL_NB + jj] = t;
    } else if constexpr (CLUSTER) {
      double t = 0.0;
      if (jj < nb) {
#pragma unroll
        for (int u = 0; u < 16 / PANEL_RG; ++u) {
          const int c = rg + PANEL_RG * u;
          t += c < G ? xp[2 * PANEL_NB + c * PANEL_NB + jj] : 0.0;
        }
      }
      red[rg * PANEL_NB + jj] = t;
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
      }
      red[rg * PANEL_NB + jj] = t;
    }
    __syncthreads();
    if (timed) { t1 = clock64(); ph[2] += t1 - t0; t0 = t1; }
    // (c) reflector of column k, computed redundantly by every thread (identical values)
    const double alpha = row0[k];
    const double sigma = sum_groups(red, k);
    double tau = 0.0, scale = 0.0, beta = alpha;
    if (sigma != 0.0) {
      const double nrm = sqrt(alpha * alpha + sigma);
      beta = alpha < 0.0 ? nrm : -nrm;
      tau = (beta - alpha) / beta;
      scale = 1.0 / (alpha - beta);
    }
    if (jj < nb) {
      const double totj = sum_groups(red, jj);
      const double drowj = row0[jj];
      if (rg == 0) { totb[(k & 1) * PANEL_NB + jj] = totj; drowb[(k & 1) * PANEL_NB + jj] = drowj; }
      if (jj > k) {
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
    if (tid == 0) {
      sc[k] = scale;
      tauv[k] = tau;
      if (cta == 0) { Ps[k * PANEL_LD + k] = beta; a.tau[k] = tau; }
    }
    __syncthreads();
    if (timed) { t1 = clock64(); ph[3] += t1 - t0; }
  }
  if (cta == tcta) {
    panel_t_column(Ts, nb - 1, totb + ((nb - 1) & 1) * PANEL_NB, drowb + ((nb - 1) & 1) * PANEL_NB,
                   sc, tauv);
  }
  if constexpr (CLUSTER) cooperative_groups::this_cluster().sync();  // peers done reading our smem
  else __syncthreads();
  if (timed) {
    const int o = cta == 0 ? 0 : 4;
    for (int q = 0; q < 4; ++q) atomicAdd(a.dbg + o + q, ph[q]);
    atomicAdd(a.dbg + 8, 1ull);
  }

  // write back: R above the diagonal, v = s_j x below it (LAPACK layout), explicit Y, Y^T
  for (int e = tid; e < R * nb; e += PANEL_THREADS) {
    int j = e / R, r = e % R;
    int gr = r0 + r;
    double x = Ps[r * PANEL_LD + j];
    double v = gr > j ? sc[j] * x : x;
    a.P[(long long)gr + (long long)j * a.ldp] = v;
    a.Y[(long long)gr + (long long)j * a.ldy] = gr > j ? v : (gr == j ? 1.0 : 0.0);
  }
  for (int e = tid; e < R * nb; e += PANEL_THREADS) {     // Y^T: contiguous along j
    int r = e / nb, j = e % nb;
    int gr = r0 + r;
    double v = gr > j ? sc[j] * Ps[r * PANEL_LD + j] : (gr == j ? 1.0 : 0.0);
    a.Yt[(long long)j + (long long)gr * a.ldyt] = v;
  }
  if (cta == tcta)
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
}

inline size_t panel_smem_bytes(int rows_per) {
  return sizeof(double) * ((size_t)rows_per * PANEL_LD + (PANEL_RG + 1) * PANEL_NB + 4 * PANEL_NB +
                           2 * PANEL_NB + PANEL_NB * PANEL_NB + 36 * PANEL_NB + 2);
}

}  // namespace sdc
