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
// Gram entries Y(:,i)^T x (i < k) that build the compact-WY T column:
//   w_j   = tau (P[k][j] + scale z_j),           P[r][j] -= w_j * scale * x_r
//   g_i   = Y[k][i] + scale * part[i],           T(0:k,k) = -tau T(0:k,0:k) g, T(k,k)=tau
// Each CTA sums the per-CTA partials in the same fixed order, so all CTAs agree
// bit-for-bit and the result is run-to-run deterministic.
#pragma once
#include "common.cuh"

namespace sdc {

constexpr int PANEL_NB = 64;        // max panel width
constexpr int PANEL_THREADS = 256;
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
};

__global__ void __launch_bounds__(PANEL_THREADS)
panel_qr_kernel(const PanelArgs a) {
  extern __shared__ __align__(16) double sm[];
  const int G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x;
  const int nb = a.nb;
  const int r0 = cta * a.rows_per;
  const int r1 = min(a.m, r0 + a.rows_per);
  const int R = max(0, r1 - r0);
  double* Ps = sm;                                  // R x PANEL_LD
  double* xs = Ps + (size_t)a.rows_per * PANEL_LD;  // rows_per
  double* red = xs + a.rows_per;                    // 4 x PANEL_NB
  double* tot = red + 4 * PANEL_NB;                 // PANEL_NB
  double* drow = tot + PANEL_NB;                    // PANEL_NB
  double* Ts = drow + PANEL_NB;                     // PANEL_NB x PANEL_NB (CTA 0), col-major
  double* wv = Ts + PANEL_NB * PANEL_NB;            // PANEL_NB
  __shared__ double s_tau, s_scale, s_beta;

  // load the CTA's row block
  for (int e = tid; e < R * nb; e += PANEL_THREADS) {
    int j = e / R, r = e % R;                       // coalesced along rows
    Ps[r * PANEL_LD + j] = a.P[(long long)(r0 + r) + (long long)j * a.ldp];
  }
  if (cta == 0)
    for (int e = tid; e < PANEL_NB * PANEL_NB; e += PANEL_THREADS) Ts[e] = 0.0;
  __syncthreads();

  const int jj = tid & (PANEL_NB - 1), rg = tid >> 6;  // column lane, row group (0..3)
  for (int k = 0; k < nb; ++k) {
    // rows r (local) with global index > k
    const int lbeg = max(0, k + 1 - r0);
    for (int r = lbeg + tid; r < R; r += PANEL_THREADS) xs[r] = Ps[r * PANEL_LD + k];
    __syncthreads();
    // partial dot products part[j] = sum_r x_r P[r][j]
    double s = 0.0;
    if (jj < nb) {
      double s1 = 0.0;
      int r = lbeg + rg;
      for (; r + 4 < R; r += 8) {
        s = fma(xs[r], Ps[r * PANEL_LD + jj], s);
        s1 = fma(xs[r + 4], Ps[(r + 4) * PANEL_LD + jj], s1);
      }
      if (r < R) s = fma(xs[r], Ps[r * PANEL_LD + jj], s);
      s += s1;
    }
    red[rg * PANEL_NB + jj] = s;
    __syncthreads();
    double* gb = a.gbuf + (size_t)(k & 1) * (G + 1) * PANEL_NB;
    if (tid < nb) {
      double p = ((red[tid] + red[PANEL_NB + tid]) + red[2 * PANEL_NB + tid]) + red[3 * PANEL_NB + tid];
      __stcg(gb + (size_t)cta * PANEL_NB + tid, p);
      if (cta == 0) __stcg(gb + (size_t)G * PANEL_NB + tid, Ps[k * PANEL_LD + tid]);  // row k
    }
    grid_barrier(a.bar, a.bar_base + (unsigned)(k + 1) * (unsigned)G);
    // all CTAs: fixed-order sum over CTAs
    {
      double t = 0.0;
      if (jj < nb) {
        int c = rg;
        for (; c + 28 < G; c += 32) {   // batch 8 independent L2 loads, add in order
          double v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = __ldcg(gb + (size_t)(c + 4 * u) * PANEL_NB + jj);
#pragma unroll
          for (int u = 0; u < 8; ++u) t += v[u];
        }
        for (; c < G; c += 4) t += __ldcg(gb + (size_t)c * PANEL_NB + jj);
      }
      red[rg * PANEL_NB + jj] = t;
    }
    __syncthreads();
    if (tid < nb) {
      tot[tid] = ((red[tid] + red[PANEL_NB + tid]) + red[2 * PANEL_NB + tid]) + red[3 * PANEL_NB + tid];
      drow[tid] = __ldcg(gb + (size_t)G * PANEL_NB + tid);
    }
    __syncthreads();
    if (tid == 0) {
      double alpha = drow[k], sigma = tot[k];
      double tau = 0.0, scale = 0.0, beta = alpha;
      if (sigma != 0.0) {
        double nrm = sqrt(alpha * alpha + sigma);
        beta = alpha < 0.0 ? nrm : -nrm;
        tau = (beta - alpha) / beta;
        scale = 1.0 / (alpha - beta);
      }
      s_tau = tau; s_scale = scale; s_beta = beta;
    }
    __syncthreads();
    const double tau = s_tau, scale = s_scale;
    if (tid < nb) wv[tid] = (tid > k) ? tau * fma(scale, tot[tid], drow[tid]) : 0.0;
    __syncthreads();
    // update local rows below the diagonal, turn column k into v
    for (int e = tid; e < (R - lbeg) * nb; e += PANEL_THREADS) {
      int r = lbeg + e / nb, j = e % nb;
      double xv = xs[r] * scale;
      if (j > k) Ps[r * PANEL_LD + j] = fma(-wv[j], xv, Ps[r * PANEL_LD + j]);
      else if (j == k) Ps[r * PANEL_LD + j] = xv;
    }
    if (cta == 0) {
      if (tid < nb && tid > k) Ps[k * PANEL_LD + tid] -= wv[tid];
      if (tid == 0) { Ps[k * PANEL_LD + k] = s_beta; a.tau[k] = tau; }
      // T column k:  g_i = Y[k][i] + scale * part[i] (i < k);  T(0:k,k) = -tau T g
      if (tid < k) {
        double acc = 0.0;
        for (int l = tid; l < k; ++l)
          acc = fma(Ts[l * PANEL_NB + tid], fma(scale, tot[l], drow[l]), acc);
        Ts[k * PANEL_NB + tid] = -tau * acc;
      }
      if (tid == k) Ts[k * PANEL_NB + k] = tau;
    }
    __syncthreads();
  }

  // write back: factored panel (R above / v below) and explicit Y
  for (int e = tid; e < R * nb; e += PANEL_THREADS) {
    int j = e / R, r = e % R;
    int gr = r0 + r;
    double v = Ps[r * PANEL_LD + j];
    a.P[(long long)gr + (long long)j * a.ldp] = v;
    a.Y[(long long)gr + (long long)j * a.ldy] = gr > j ? v : (gr == j ? 1.0 : 0.0);
  }
  for (int e = tid; e < R * nb; e += PANEL_THREADS) {     // Y^T: contiguous along j
    int r = e / nb, j = e % nb;
    int gr = r0 + r;
    double v = Ps[r * PANEL_LD + j];
    a.Yt[(long long)j + (long long)gr * a.ldyt] = gr > j ? v : (gr == j ? 1.0 : 0.0);
  }
  if (cta == 0)
    for (int e = tid; e < nb * nb; e += PANEL_THREADS) {
      int j = e / nb, i = e % nb;
      a.T[e] = Ts[j * PANEL_NB + i];
    }
}

inline size_t panel_smem_bytes(int rows_per) {
  return sizeof(double) * ((size_t)rows_per * PANEL_LD + rows_per + 4 * PANEL_NB + 2 * PANEL_NB +
                           PANEL_NB * PANEL_NB + PANEL_NB);
}

}  // namespace sdc
