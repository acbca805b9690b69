// batched.cuh -- the split step for MANY small problems in one launch (SURVEY §8(f) row f3,
// "a batched small-n mode"): one CTA per problem, the whole RNEP step (Alg. 5, PAPER.md:
// 412-423) -- IRS passes, GRURV, similarity, split selection -- resident in shared memory.
//
// For n <= 64 the large-n machinery (64-wide panels, DMMA GEMM tiles, per-column grid
// exchanges) is all latency: a single problem keeps one SM busy for ~3 ms at n = 64.  Here
// each CTA runs the whole step with every matrix in SMEM, so a launch of B problems runs
// B/148 waves of independent CTAs: data-parallel over problems, which is
// also how the batch shards across GPUs (no collective, `bench.py --config 10`).
#pragma once
#include "common.cuh"

namespace sdc {

constexpr int BAT_NMAX = 64;
constexpr int BAT_THREADS = 512;
constexpr int BAT_WARPS = BAT_THREADS / 32;

struct BatArgs {
  const double* A; long long lda, sa;    // problem b: A + b*sa, n x n, ld lda
  const double* V; long long ldv, sv;    // Haar V of problem b
  double* Q; long long ldq, sq;          // out: Q of problem b
  double* out;                           // out: 4 doubles per problem {r, metric, metric_fro, nonfinite}
  int n, passes;
};

// fixed-order block sum (warp shuffles, then warps in order by thread 0); result to all
SDC_DEV double bat_sum(double v, double* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < BAT_WARPS; ++i) t += red[i];
    red[BAT_WARPS] = t;
  }
  __syncthreads();
  const double t = red[BAT_WARPS];
  __syncthreads();
  return t;
}

// =======================================================================================
// Compact-WY kernel: the step with every O(n^3) contraction on the FP64 tensor cores
// (mma.sync m8n8k4 DMMA on shared-memory operands) and 2 CTA barriers per Householder
// column (the first, unblocked version with the oracle's dgeqr2 / complement / dgerq2 order
// needed ~5 and ran 3.7x slower; removed in round 2):
//   QR (bq_qr): reflector columns stay UNSCALED during the factorisation (v_k = sc_k x_k),
//     one pass of column dot products g_j = x_k^T P(:, j) per column gives the norm, the
//     update coefficients and the Gram entries of the compact-WY T column (PAPER.md:331's
//     "QR", LAPACK dgeqr2 + dlarft arithmetic in a blocked order);
//   IRS pass (Alg. 3): with Q = I - Y T Y^T and the complement C = Q [0; I] = [0; I] - Y Z,
//     Z = T Y2^T (Y2 = rows n..2n-1 of Y), the products need no explicit C:
//     A_{j+1} = C1^T A_j = -Z^T (Y1^T A_j),  B_{j+1} = C2^T B_j = B_j - Z^T (Y2^T B_j);
//   GRURV: QR(A_p V^T) -> U^T (A_p + B_p) = S - Y T^T (Y^T S), row signs, RQ as the QR of
//     C^T J with explicit Q_qr = I - Y (T Y^T), Q = Q_qr D J (reading Q10);
//   similarity Q^T A Q with the original A, selection as above.
// All matrices live in shared memory with leading dimension NP = n rounded up to 16 (2 NP for
// the stack) and zero padding; accessors return 0 outside the logical ranges.
// =======================================================================================
constexpr int BQ_THREADS = 512;

struct BqShape { int n, m, np; };

// out(i, j) (16x16 warp tiles over P_ x Q_) = sum_k fa(i, k) fb(k, j), then fo(i, j, v)
template <class FA, class FB, class FO>
SDC_DEV void bq_mma(int P_, int Q_, int K_, FA fa, FB fb, FO fo) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int tm = P_ / 16, tn = Q_ / 16;
  for (int tile = warp; tile < tm * tn; tile += BQ_THREADS / 32) {
    const int i0 = (tile % tm) * 16, j0 = (tile / tm) * 16;
    double acc[2][2][2] = {{{0.0, 0.0}, {0.0, 0.0}}, {{0.0, 0.0}, {0.0, 0.0}}};
    for (int k0 = 0; k0 < K_; k0 += 4) {
      double a[2], b[2];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) a[mi] = fa(i0 + mi * 8 + g, k0 + t);
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) b[ni] = fb(k0 + t, j0 + ni * 8 + g);
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) dmma_8x8x4(acc[mi][ni], a[mi], b[ni]);
    }
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int ni = 0; ni < 2; ++ni)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) fo(i0 + mi * 8 + g, j0 + ni * 8 + 2 * t + hh, acc[mi][ni][hh]);
  }
  __syncthreads();
}

// unscaled Householder QR of the m x n P (ld ldp) with compact-WY T (NP x NP, ld np, upper):
// on exit P holds x_k below the diagonal (v_k = sc[k] x_k, unit diagonal implied), R above,
// beta[k] = R(k, k); I - Y T Y^T = H_0 ... H_{n-1}.  Two CTA barriers per column.
SDC_DEV void bq_qr(int m, int n, int np, double* P, int ldp, double* T, int tld, double* sc,
                   double* beta, double* g, double* drow) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < np * tld; e += BQ_THREADS) T[e] = 0.0;
  __syncthreads();
  for (int k = 0; k < n; ++k) {
    // (A) g_j = sum_{r > k} x_k(r) P(r, j), every column j (j < k: Gram entries for T).
    // A warp owns 4 consecutive columns; the 4 lane sums are reduced by recursive halving
    // (xor 16 and 8 exchange half of the columns, xor 4, 2, 1 finish): 6 shuffles instead
    // of 4 full butterflies (20), fixed order per column.
    for (int jb = warp * 4; jb < n; jb += BQ_THREADS / 8) {
      double s[4] = {0.0, 0.0, 0.0, 0.0};
      for (int r = k + 1 + lane; r < m; r += 32) {
        const double x = P[r + k * ldp];
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (jb + c < n) s[c] = fma(x, P[r + (jb + c) * ldp], s[c]);
      }
      const bool h16 = (lane & 16) != 0, h8 = (lane & 8) != 0;
      double k0 = h16 ? s[2] : s[0], k1 = h16 ? s[3] : s[1];
      k0 += __shfl_xor_sync(0xffffffffu, h16 ? s[0] : s[2], 16);
      k1 += __shfl_xor_sync(0xffffffffu, h16 ? s[1] : s[3], 16);
      double v = h8 ? k1 : k0;
      v += __shfl_xor_sync(0xffffffffu, h8 ? k0 : k1, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      v += __shfl_xor_sync(0xffffffffu, v, 2);
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      const int c = (h16 ? 2 : 0) + (h8 ? 1 : 0);
      if ((lane & 7) == 0 && jb + c < n) {
        g[jb + c] = v;
        drow[jb + c] = P[k + (jb + c) * ldp];   // x_j(k): row k, read by the T column below
      }
    }
    __syncthreads();
    // (B) reflector (dlarfg, Q7), identical in every thread
    const double alpha = P[k + k * ldp], sigma = g[k];
    double tk = 0.0, scale = 0.0, bk = alpha;
    if (sigma != 0.0) {   // one rsqrt + one reciprocal (the panel kernel's formulas)
      const double qq = fma(alpha, alpha, sigma);
      const double rn = rsqrt(qq);
      const double nrm = qq * rn, aa = fabs(alpha);
      bk = alpha < 0.0 ? nrm : -nrm;
      tk = fma(aa, rn, 1.0);                       // (beta - alpha) / beta
      const double sa = __drcp_rn(aa + nrm);       // 1 / (alpha - beta) = sign(alpha) / (|alpha| + nrm)
      scale = alpha < 0.0 ? -sa : sa;
    }
    for (int j = k + 1 + warp; j < n; j += BQ_THREADS / 32) {   // columns j > k
      const double w = tk * fma(scale, g[j], P[k + j * ldp]);
      const double ws = w * scale;
      for (int r = k + 1 + lane; r < m; r += 32) P[r + j * ldp] = fma(-ws, P[r + k * ldp], P[r + j * ldp]);
      __syncwarp();
      if (lane == 0) P[k + j * ldp] -= w;
    }
    // T(0:k, k) = -tau_k T(0:k, 0:k) g',  g'_l = sc_l (x_l(k) + scale g_l);  T(k, k) = tau_k
    {
      const int i = tid >> 2, q = tid & 3;
      double acc = 0.0;
      if (i < k)
        for (int l = i + q; l < k; l += 4) acc = fma(T[i + l * tld], sc[l] * fma(scale, g[l], drow[l]), acc);
      acc += __shfl_xor_sync(0xffffffffu, acc, 1);
      acc += __shfl_xor_sync(0xffffffffu, acc, 2);
      if (i < k && q == 0) T[i + k * tld] = -tk * acc;
      if (tid == 0) {
        T[k + k * tld] = tk;
        sc[k] = scale;
        beta[k] = bk;
      }
    }
    __syncthreads();
  }
}

// Shared-memory layout of one problem of order n (np = n rounded up to 16).  Leading
// dimensions = 4 (mod 16) doubles: the DMMA fragment loads (8 rows x 4 k of one operand per
// instruction) and the T column loop hit 16 distinct bank pairs per half-warp.
struct BqSm {
  int n, np, ld, NL, ldp;
  double *Aj, *Bj;        // np x np (ld): A_j, B_j; after bq_split_tail: Ahat, Q
  double* P;              // 2np x np (ldp): stack / factored matrices
  double *T, *W, *Z;      // np x np (ld); W aliases T (T is dead whenever W is live)
  double *sc, *beta, *g, *msel, *red;
  // implicit unit-lower Y of the last factorisation of P (rows m_, columns n)
  SDC_DEV double Yv(int r, int k, int m_) const {
    if (k >= n || r >= m_ || r < k) return 0.0;
    return r == k ? 1.0 : sc[k] * P[r + k * ldp];
  }
};

SDC_DEV BqSm bq_carve(double* smq, int n) {
  BqSm s;
  s.n = n;
  s.np = (n + 15) & ~15;
  s.ld = s.np + 4;
  s.NL = s.ld * s.np;
  s.ldp = 2 * s.np + 4;
  s.Aj = smq;
  s.Bj = s.Aj + s.NL;
  s.P = s.Bj + s.NL;
  s.T = s.P + (size_t)s.ldp * s.np;
  s.W = s.T;
  s.Z = s.T + s.NL;
  s.sc = s.Z + s.NL;
  s.beta = s.sc + s.np;
  s.g = s.beta + s.np;
  s.msel = s.g + s.np;
  s.red = s.msel + s.np;   // 2 * BAT_WARPS + 16
  return s;
}

// one IRS pass (Alg. 3 l.3): (A_j, B_j) -> (A_{j+1}, B_{j+1}) in place
SDC_DEV void bq_irs_pass(const BqSm& s) {
  const int n = s.n, m = 2 * n, np = s.np, ld = s.ld, ldp = s.ldp, tid = threadIdx.x;
  double *Aj = s.Aj, *Bj = s.Bj, *P = s.P, *T = s.T, *W = s.W, *Z = s.Z;
  for (int e = tid; e < ldp * np; e += BQ_THREADS) {   // P = [B_j; -A_j] (rows >= 2n zero)
    const int i = e % ldp, j = e / ldp;
    double v = 0.0;
    if (j < n) v = i < n ? Bj[i + j * ld] : (i < m ? -Aj[(i - n) + j * ld] : 0.0);
    P[e] = v;
  }
  __syncthreads();
  bq_qr(m, n, np, P, ldp, T, ld, s.sc, s.beta, s.g, s.msel);
  // Z = T Y2^T  (T dead afterwards: W may overwrite it)
  bq_mma(np, np, np, [&](int i, int k) { return T[i + k * ld]; },
         [&](int k, int j) { return s.Yv(n + j, k, m); },
         [&](int i, int j, double v) { Z[i + j * ld] = v; });
  // W = Y1^T A_j ;  A_{j+1} = -Z^T W
  bq_mma(np, np, np, [&](int i, int k) { return s.Yv(k, i, n); },
         [&](int k, int j) { return Aj[k + j * ld]; },
         [&](int i, int j, double v) { W[i + j * ld] = v; });
  bq_mma(np, np, np, [&](int i, int k) { return Z[k + i * ld]; },
         [&](int k, int j) { return W[k + j * ld]; },
         [&](int i, int j, double v) { Aj[i + j * ld] = -v; });
  // W = Y2^T B_j ;  B_{j+1} = B_j - Z^T W
  bq_mma(np, np, np, [&](int i, int k) { return s.Yv(n + k, i, m); },
         [&](int k, int j) { return Bj[k + j * ld]; },
         [&](int i, int j, double v) { W[i + j * ld] = v; });
  bq_mma(np, np, np, [&](int i, int k) { return Z[k + i * ld]; },
         [&](int k, int j) { return W[k + j * ld]; },
         [&](int i, int j, double v) { Bj[i + j * ld] -= v; });
}

// Explicit Q of the last bq_qr of an n x n P with the columns scaled by sign(R_jj):
// out(i, j) = sign(beta[j]) (I - (Y T) Y^T)(i, j)   (the Haar factor of a Gaussian P)
template <class FO>
SDC_DEV void bq_form_q_signed(const BqSm& s, FO out) {
  const int n = s.n, np = s.np, ld = s.ld;
  double *T = s.T, *W = s.W, *Z = s.Z;
  bq_mma(np, np, np, [&](int i, int k) { return s.Yv(i, k, n); },
         [&](int k, int j) { return T[k + j * ld]; },
         [&](int i, int j, double v) { Z[i + j * ld] = v; });
  bq_mma(np, np, np, [&](int i, int k) { return Z[i + k * ld]; },
         [&](int k, int j) { return s.Yv(j, k, n); },
         [&](int i, int j, double v) { W[i + j * ld] = (i == j && i < n ? 1.0 : 0.0) - v; });
  for (int e = threadIdx.x; e < n * n; e += BQ_THREADS) {
    const int i = e % n, j = e / n;
    out(i, j, (s.beta[j] < 0.0 ? -1.0 : 1.0) * W[i + j * ld]);
  }
  __syncthreads();
}

// GRURV(2, A_p + B_p, A_p; -1, +1) with the Haar V0, similarity with the original A0 and the
// split selection.  In: Aj = A_p, Bj = B_p (destroyed).  Out: Bj = Q, Aj = Ahat = Q^T A0 Q,
// red[2 BAT_WARPS] = r, red[2 BAT_WARPS + 1] = min_r ||Ahat(r:, :r)||_1 / nA (ties: smallest r).
SDC_DEV void bq_split_tail(const BqSm& s, const double* A0, long long lda, const double* V0,
                           long long ldv, double nA) {
  const int n = s.n, np = s.np, ld = s.ld, ldp = s.ldp, tid = threadIdx.x;
  double *Aj = s.Aj, *Bj = s.Bj, *P = s.P, *T = s.T, *W = s.W, *Z = s.Z;
  double *beta = s.beta, *msel = s.msel, *red = s.red;
  // X = A_p V^T into P (ld 2np)
  bq_mma(np, np, np, [&](int i, int k) { return Aj[i + k * ld]; },
         [&](int k, int j) { return (k < n && j < n) ? V0[j + (long long)k * ldv] : 0.0; },
         [&](int i, int j, double v) { P[i + j * ldp] = v; });
  bq_qr(n, n, np, P, ldp, T, ld, s.sc, beta, s.g, msel);               // X = U R_2
  for (int e = tid; e < np * np; e += BQ_THREADS) {                   // S = A_p + B_p
    const int i = e % np, j = e / np;
    Aj[i + j * ld] += Bj[i + j * ld];
  }
  __syncthreads();
  // U^T S = S - (Y T^T)(Y^T S):  Z = Y T^T (last use of T), W = Y^T S, S -= Z W, row signs
  bq_mma(np, np, np, [&](int i, int k) { return s.Yv(i, k, n); },
         [&](int k, int j) { return T[j + k * ld]; },
         [&](int i, int j, double v) { Z[i + j * ld] = v; });
  bq_mma(np, np, np, [&](int i, int k) { return s.Yv(k, i, n); },
         [&](int k, int j) { return Aj[k + j * ld]; },
         [&](int i, int j, double v) { W[i + j * ld] = v; });
  bq_mma(np, np, np, [&](int i, int k) { return Z[i + k * ld]; },
         [&](int k, int j) { return W[k + j * ld]; },
         [&](int i, int j, double v) {
           const double t = Aj[i + j * ld] - v;
           Aj[i + j * ld] = (i < n && beta[i] < 0.0) ? -t : t;     // U <- U D_U
         });
  // M = C^T J into P: M(i, j) = C(n-1-j, i)
  for (int e = tid; e < ldp * np; e += BQ_THREADS) {
    const int i = e % ldp, j = e / ldp;
    P[e] = (i < n && j < n) ? Aj[(n - 1 - j) + i * ld] : 0.0;
  }
  __syncthreads();
  bq_qr(n, n, np, P, ldp, T, ld, s.sc, beta, s.g, msel);
  // Q_qr = I - (Y T) Y^T:  Z = Y T (last use of T), W = I - Z Y^T
  bq_mma(np, np, np, [&](int i, int k) { return s.Yv(i, k, n); },
         [&](int k, int j) { return T[k + j * ld]; },
         [&](int i, int j, double v) { Z[i + j * ld] = v; });
  bq_mma(np, np, np, [&](int i, int k) { return Z[i + k * ld]; },
         [&](int k, int j) { return s.Yv(j, k, n); },
         [&](int i, int j, double v) { W[i + j * ld] = (i == j && i < n ? 1.0 : 0.0) - v; });
  // Q(:, j) = sign(R(jj, jj)) Q_qr(:, jj), jj = n-1-j  -> Bj
  for (int e = tid; e < np * np; e += BQ_THREADS) {
    const int i = e % np, j = e / np;
    double v = 0.0;
    if (i < n && j < n) {
      const int jj = n - 1 - j;
      v = (beta[jj] < 0.0 ? -1.0 : 1.0) * W[i + jj * ld];
    }
    Bj[i + j * ld] = v;
  }
  __syncthreads();

  // ---- similarity Ahat = Q^T A Q (original A), split selection ------------------------------
  bq_mma(np, np, np, [&](int i, int k) { return (i < n && k < n) ? A0[i + (long long)k * lda] : 0.0; },
         [&](int k, int j) { return Bj[k + j * ld]; },
         [&](int i, int j, double v) { W[i + j * ld] = v; });
  bq_mma(np, np, np, [&](int i, int k) { return Bj[k + i * ld]; },
         [&](int k, int j) { return W[k + j * ld]; },
         [&](int i, int j, double v) { Aj[i + j * ld] = v; });
  // suffix column sums: Z[c + r ld] = sum_{i >= r} |Ahat(i, c)| for c < r
  if (tid < n) {
    double t = 0.0;
    for (int r = n - 1; r >= 1; --r) {
      t += fabs(Aj[r + tid * ld]);
      Z[tid + r * ld] = t;
    }
  }
  __syncthreads();
  if (tid >= 1 && tid < n) {
    const int r = tid;
    double ma = 0.0;
    for (int c = 0; c < r; ++c) {
      const double v = Z[c + r * ld];
      if (v > ma || v != v) ma = v;
    }
    msel[r] = ma / nA;
  }
  __syncthreads();
  if (tid == 0) {
    int best = 1;
    for (int r = 2; r <= n - 1; ++r)
      if (msel[r] < msel[best]) best = r;
    red[2 * BAT_WARPS] = best;
    red[2 * BAT_WARPS + 1] = msel[best];
  }
  __syncthreads();
}

// ||A||_1 (max column sum) and ||A||_F of the n x n matrix in Aj (uses msel, red)
SDC_DEV void bq_norms(const BqSm& s, const double* X, double& n1, double& nf) {
  const int n = s.n, np = s.np, ld = s.ld, tid = threadIdx.x;
  double f = 0.0;
  for (int e = tid; e < np * np; e += BQ_THREADS) { const double v = X[e % np + (e / np) * ld]; f += v * v; }
  nf = sqrt(bat_sum(f, s.red));
  if (tid < n) {
    double c = 0.0;
    for (int i = 0; i < n; ++i) c += fabs(X[i + tid * ld]);
    s.msel[tid] = c;
  }
  __syncthreads();
  n1 = 0.0;
  for (int j = 0; j < n; ++j) n1 = fmax(n1, s.msel[j]);
  __syncthreads();
}

__global__ void __launch_bounds__(BQ_THREADS, 1) k_split_batched_wy(const BatArgs a) {
  extern __shared__ __align__(16) double smq[];
  const int n = a.n, b = blockIdx.x, tid = threadIdx.x;
  const BqSm s = bq_carve(smq, n);
  const int np = s.np, ld = s.ld;
  double *Aj = s.Aj, *Bj = s.Bj, *red = s.red;
  const double* A0 = a.A + (long long)b * a.sa;
  const double* V0 = a.V + (long long)b * a.sv;

  for (int e = tid; e < np * np; e += BQ_THREADS) {
    const int i = e % np, j = e / np;
    const bool in = i < n && j < n;
    Aj[i + j * ld] = in ? A0[i + (long long)j * a.lda] : 0.0;
    Bj[i + j * ld] = (in && i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  double nA, fA;
  bq_norms(s, Aj, nA, fA);

  for (int pass = 0; pass < a.passes; ++pass) bq_irs_pass(s);          // IRS (Alg. 3)
  bq_split_tail(s, A0, a.lda, V0, a.ldv, nA);                          // GRURV, similarity, selection

  const int rbest = (int)red[2 * BAT_WARPS];
  double f = 0.0, nf = 0.0;
  for (int e = tid; e < np * np; e += BQ_THREADS) {
    const int i = e % np, j = e / np;
    if (i >= n || j >= n) continue;
    const double v = Aj[i + j * ld];
    if (i >= rbest && j < rbest) f += v * v;
    if (!(fabs(v) <= 1.79e308)) nf = 1.0;
  }
  const double e21f = sqrt(bat_sum(f, red));
  const double nonfinite = bat_sum(nf, red);
  double* Qo = a.Q + (long long)b * a.sq;
  for (int e = tid; e < n * n; e += BQ_THREADS) {
    const int i = e % n, j = e / n;
    Qo[i + (long long)j * a.ldq] = Bj[i + j * ld];
  }
  if (tid == 0) {
    a.out[4 * b + 0] = rbest;
    a.out[4 * b + 1] = red[2 * BAT_WARPS + 1];
    a.out[4 * b + 2] = e21f / fA;
    a.out[4 * b + 3] = nonfinite;
  }
}

inline size_t bq_smem_bytes(int n) {
  const size_t np = (size_t)((n + 15) & ~15), ld = np + 4, ldp = 2 * np + 4;
  return sizeof(double) * (4 * ld * np + ldp * np + 4 * np + 2 * BAT_WARPS + 16);
}

}  // namespace sdc
