// schur_batched.cuh -- the recursion's small blocks, many at a time (SURVEY §8(f) row f2:
// "batching the small subproblems"; "zero out E21 ... recurse").
//
// sdc_schur sends every diagonal block of order <= BAT_NMAX (64) through ONE launch per
// recursion level instead of the large-n kernel sequence per attempt and pass: one CTA per
// block runs the whole node of DESIGN.md §10 -- the search interval from (trace, ||T - cI||_F),
// up to 16 attempts, each a keyed line a and Haar V (same counter-based streams as the
// large-n path and the oracle), the half-plane step on the Moebius pencil
// (A - (a-1) I, A - (a+1) I) in monitor mode (a full GRURV + similarity +
// selection after every IRS pass) with the E21 / PLATEAU / ONESIDED stop rules,
// the acceptance rule (status 0 and 1e-3 <= side <= 1 - 1e-3), the interval update of a
// rejected one-sided step -- with every matrix in shared memory (batched.cuh's DMMA pieces).
// Same decisions as schur_node() in sdc.cu and orc_schur_node(); only the arithmetic order
// of the contractions differs (rounding level).
//
// A_p, B_p are parked in a per-block global scratch (L2-resident) while the monitor split
// reuses their shared-memory space; V, Q and Ahat live there too.
#pragma once
#include "batched.cuh"

namespace sdc {

constexpr int SB_SLOT = 5 * BAT_NMAX * BAT_NMAX;   // doubles of scratch per block: V, A_p, B_p, Q, Ahat

struct SchurLeafArgs {
  double* T; long long ldt;          // the n x n working matrix (diagonal blocks updated in place)
  const int* off; const int* ord;    // per block: local offset in T, order (2 <= order <= 64)
  int key_off;                       // global offset of T(0, 0) (keys of the draws)
  int leaf;
  unsigned long long seed;
  int max_iters;
  double tol;
  double* scratch;                   // nblocks * SB_SLOT doubles
  int* r_out;                        // per block: accepted split r in [1, m-1], or 0
  int* stats;                        // per block: 4 ints {splits, failed attempts, unsplit, passes}
  double* metric;                    // per block: metric of the accepted split (or 0)
  int trace;                         // SDC_SCHUR_TRACE: one line per attempt (orc_schur_node's format)
};

SDC_DEV unsigned long long sb_attempt_ctr(int o, int m, int t) {
  const unsigned long long id = (unsigned long long)o * 65537ull + (unsigned long long)m;
  return ((mix64(0x5DC0FFEEull, id) & 0x7FFFFull) << 4) | (unsigned long long)t;
}

__global__ void __launch_bounds__(BQ_THREADS, 1) k_schur_leaves(const SchurLeafArgs a) {
  extern __shared__ __align__(16) double smq[];
  const int b = blockIdx.x, tid = threadIdx.x;
  const int m = a.ord[b], o = a.off[b];
  double* Tb = a.T + o + (long long)o * a.ldt;
  const long long ldt = a.ldt;
  int* st = a.stats + 4 * b;
  auto finish = [&](int r, double met) {
    if (tid == 0) { a.r_out[b] = r; a.metric[b] = met; }
  };
  if (tid == 0) { st[0] = st[1] = st[2] = st[3] = 0; }
  if (m <= a.leaf || m < 2) { finish(0, 0.0); return; }
  if (m == 2) {   // 2x2 with complex eigenvalues: a standardised leaf
    const double p = Tb[0], c = Tb[1], q = Tb[ldt], d = Tb[1 + ldt];
    if ((p - d) * (p - d) + 4.0 * q * c < 0.0) { finish(0, 0.0); return; }
  }
  const BqSm s = bq_carve(smq, m);
  const int n = m, np = s.np, ld = s.ld, ldp = s.ldp;
  double *Aj = s.Aj, *Bj = s.Bj, *P = s.P, *red = s.red;
  double* Vg = a.scratch + (size_t)b * SB_SLOT;       // m x m, ld m
  double* Apg = Vg + BAT_NMAX * BAT_NMAX;
  double* Bpg = Apg + BAT_NMAX * BAT_NMAX;
  double* Qg = Bpg + BAT_NMAX * BAT_NMAX;
  double* Ahg = Qg + BAT_NMAX * BAT_NMAX;

  // original block -> Aj (padded); ||T_b||_1; trace and ||T_b - c I||_F
  for (int e = tid; e < np * np; e += BQ_THREADS) {
    const int i = e % np, j = e / np;
    Aj[i + j * ld] = (i < n && j < n) ? Tb[i + j * ldt] : 0.0;
  }
  __syncthreads();
  double nA, fA;
  bq_norms(s, Aj, nA, fA);
  double tr = 0.0;
  for (int i = tid; i < n; i += BQ_THREADS) tr += Aj[i + i * ld];
  const double c = bat_sum(tr, red) / n;
  double f = 0.0;
  for (int e = tid; e < n * n; e += BQ_THREADS) {
    const int i = e % n, j = e / n;
    const double v = Aj[i + j * ld] - (i == j ? c : 0.0);
    f += v * v;
  }
  const double sdev = sqrt(bat_sum(f, red) / n);
  if (!(sdev > 0.0)) {
    if (tid == 0) st[2] = 1;
    finish(0, 0.0);
    return;
  }
  double lo = c - 2.0 * sdev, hi = c + 2.0 * sdev;
  const double tolb = fmax(a.tol, 8e-15 * m);   // rounding floor grows ~ m eps
  int failed = 0, passes = 0;

  for (int att = 0; att < 16; ++att) {
    const unsigned long long ctr = sb_attempt_ctr(a.key_off + o, m, att);
    const double u = (double)(mix64(a.seed, 2ull * ctr) >> 11) * 1.1102230246251565e-16;
    const double ash = lo + (0.25 + 0.5 * u) * (hi - lo);
    // Haar V: QR of the Gaussian of stream 2 ctr + 1, columns scaled by sign(R_jj)
    const unsigned long long key = 2ull * ctr + 1ull;
    for (int e = tid; e < ldp * np; e += BQ_THREADS) {
      const int i = e % ldp, j = e / ldp;
      double v = 0.0;
      if (i < n && j < n) {
        const unsigned long long base = (key << 40) + 2ull * ((unsigned long long)i + (unsigned long long)j * m);
        const double u1 = (double)((mix64(a.seed, base) >> 11) + 1ull) * 1.1102230246251565e-16;
        const double u2 = (double)(mix64(a.seed, base + 1ull) >> 11) * 1.1102230246251565e-16;
        v = sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
      }
      P[e] = v;
    }
    __syncthreads();
    bq_qr(n, n, np, P, ldp, s.T, ld, s.sc, s.beta, s.g, s.msel);
    bq_form_q_signed(s, [&](int i, int j, double v) { Vg[i + j * m] = v; });
    __threadfence_block();
    __syncthreads();

    // (A_0, B_0) = (T_b - (a-1) I, T_b - (a+1) I)
    for (int e = tid; e < np * np; e += BQ_THREADS) {
      const int i = e % np, j = e / np;
      const double v = (i < n && j < n) ? Tb[i + j * ldt] : 0.0;
      const bool dg = i == j && i < n;
      Aj[i + j * ld] = dg ? v - (ash - 1.0) : v;
      Bj[i + j * ld] = dg ? v - (ash + 1.0) : v;
    }
    __syncthreads();

    // monitor-mode passes
    double prev = INFINITY, metric = NAN, fa = 0.0, fb = 0.0;
    int r = 0, p = a.max_iters;
    bool have_split = false;
    for (int j = 0; j < a.max_iters; ++j) {
      bq_irs_pass(s);
      {
        double d1;
        bq_norms(s, Aj, d1, fa);
        bq_norms(s, Bj, d1, fb);
      }
      if (j >= 2) {   // every eigenvalue on one side: one of A_p, B_p vanishes relative to the other
        const double sd = fa + fb > 0.0 ? fb / (fa + fb) : 0.5;
        if (sd < 1e-6 || sd > 1.0 - 1e-6) { p = j + 1; break; }
      }
      for (int e = tid; e < n * n; e += BQ_THREADS) {   // park A_p, B_p
        const int i = e % n, jj = e / n;
        Apg[e] = Aj[i + jj * ld];
        Bpg[e] = Bj[i + jj * ld];
      }
      bq_split_tail(s, Tb, ldt, Vg, m, nA);
      have_split = true;
      r = (int)red[2 * BAT_WARPS];
      metric = red[2 * BAT_WARPS + 1];
      for (int e = tid; e < n * n; e += BQ_THREADS) {   // Q, Ahat of this pass
        const int i = e % n, jj = e / n;
        Qg[e] = Bj[i + jj * ld];
        Ahg[e] = Aj[i + jj * ld];
      }
      __syncthreads();
      bool stop = false;
      if (metric <= tolb) stop = true;
      else if (metric <= 10.0 * tolb && metric > 0.5 * prev) stop = true;   // plateau: the rounding floor
      if (stop) { p = j + 1; break; }
      prev = metric;
      if (j + 1 < a.max_iters) {
        for (int e = tid; e < np * np; e += BQ_THREADS) {   // restore A_p, B_p (zero padding)
          const int i = e % np, jj = e / np;
          const bool in = i < n && jj < n;
          Aj[i + jj * ld] = in ? Apg[i + jj * n] : 0.0;
          Bj[i + jj * ld] = in ? Bpg[i + jj * n] : 0.0;
        }
        __syncthreads();
      }
    }
    passes += p;
    // status: 0 iff the metric is finite and <= the acceptance threshold (reading Q4)
    bool bad = !have_split;
    if (have_split) {
      double nf = 0.0;
      for (int e = tid; e < n * n; e += BQ_THREADS)
        if (!(fabs(Ahg[e]) <= 1.79e308)) nf = 1.0;
      bad = bat_sum(nf, red) != 0.0 || !(fabs(metric) <= 1.79e308);
    }
    const double side = fa + fb > 0.0 ? fb / (fa + fb) : 0.5;
    const bool ok = !bad && metric <= 1e-8;
    const bool onesided = side < 1e-3 || side > 1.0 - 1e-3;
    if (a.trace && tid == 0)
      printf("node o=%d m=%d att=%d a=%.6f iters=%d status=%d r=%d metric=%.3e side=%.3e\n", a.key_off + o, m,
             att, ash, p, bad ? 2 : (ok ? 0 : 1), r, metric, side);
    if (!ok || onesided) {   // a one-sided pair's split is incidental
      ++failed;
      if (side > 0.95) hi = ash;          // every eigenvalue left of the line
      else if (side < 0.05) lo = ash;     // every eigenvalue right of the line
      __syncthreads();
      continue;
    }
    // accepted: T_b <- Ahat with E21 := 0; Q_b stays in the block's scratch slot
    for (int e = tid; e < n * n; e += BQ_THREADS) {
      const int i = e % n, jj = e / n;
      Tb[i + jj * ldt] = (i >= r && jj < r) ? 0.0 : Ahg[e];
    }
    if (tid == 0) { st[0] = 1; st[1] = failed; st[3] = passes; }
    finish(r, metric);
    return;
  }
  if (tid == 0) { st[1] = failed; st[2] = 1; st[3] = passes; }   // 16 failed attempts: an unsplit leaf
  finish(0, 0.0);
}

// ---------------------------------------------------------------------------------------
// Off-diagonal updates of one recursion level: for every accepted block (o, m, Q_b)
//   left : T(o:o+m, o+m:n) <- Q_b^T T(o:o+m, o+m:n)
//   right: T(0:o, o:o+m) <- T(0:o, o:o+m) Q_b   and   Q(:, o:o+m) <- Q(:, o:o+m) Q_b
// The left updates of all blocks run in one launch, then the right ones in another: blocks are
// disjoint, so each launch's tiles are independent, and a tile that receives both (rows of
// block i, columns of block j > i) gets Q_i^T X Q_j either way.
// grid = (tiles of 64 columns / rows, accepted blocks); 256 threads.
// ---------------------------------------------------------------------------------------
constexpr size_t SB_APPLY_SMEM = 2 * sizeof(double) * BAT_NMAX * (BAT_NMAX + 1);
struct SchurApplyArgs {
  double* T; long long ldt;
  double* Q; long long ldq;
  int n;                           // order of T; rows of Q
  const int* off; const int* ord;  // per block
  const int* r;                    // per block: 0 = not split (skipped)
  const double* scratch;           // Q_b at scratch + b * SB_SLOT + 3 * 64 * 64, ld = order
};

__global__ void __launch_bounds__(256) k_schur_apply_left(const SchurApplyArgs a) {
  extern __shared__ __align__(16) double sm_apply[];
  double* Qs = sm_apply;
  double* Xs = sm_apply + BAT_NMAX * (BAT_NMAX + 1);
  const int b = blockIdx.y;
  if (a.r[b] == 0) return;
  const int m = a.ord[b], o = a.off[b], c0 = o + m + 64 * blockIdx.x;
  if (c0 >= a.n) return;
  const int nc = min(64, a.n - c0);
  const double* Qb = a.scratch + (size_t)b * SB_SLOT + 3 * BAT_NMAX * BAT_NMAX;
  for (int e = threadIdx.x; e < m * m; e += 256) Qs[(e % m) + (e / m) * (BAT_NMAX + 1)] = Qb[e];
  for (int e = threadIdx.x; e < m * nc; e += 256) {
    const int i = e % m, j = e / m;
    Xs[i + j * (BAT_NMAX + 1)] = a.T[(o + i) + (long long)(c0 + j) * a.ldt];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < m * nc; e += 256) {
    const int i = e % m, j = e / m;
    double v = 0.0;
    for (int k = 0; k < m; ++k) v = fma(Qs[k + i * (BAT_NMAX + 1)], Xs[k + j * (BAT_NMAX + 1)], v);
    a.T[(o + i) + (long long)(c0 + j) * a.ldt] = v;
  }
}

__global__ void __launch_bounds__(256) k_schur_apply_right(const SchurApplyArgs a) {
  extern __shared__ __align__(16) double sm_apply[];
  double* Qs = sm_apply;
  double* Xs = sm_apply + BAT_NMAX * (BAT_NMAX + 1);
  const int b = blockIdx.y;
  if (a.r[b] == 0) return;
  const int m = a.ord[b], o = a.off[b];
  // row tiles: first those of T(0:o, :), then those of Q(0:n, :)
  const int tT = (o + 63) / 64;
  const bool onQ = (int)blockIdx.x >= tT;
  const int r0 = 64 * (onQ ? blockIdx.x - tT : blockIdx.x);
  const int rows = onQ ? a.n : o;
  if (r0 >= rows) return;
  const int nr = min(64, rows - r0);
  double* X = onQ ? a.Q : a.T;
  const long long ldx = onQ ? a.ldq : a.ldt;
  const double* Qb = a.scratch + (size_t)b * SB_SLOT + 3 * BAT_NMAX * BAT_NMAX;
  for (int e = threadIdx.x; e < m * m; e += 256) Qs[(e % m) + (e / m) * (BAT_NMAX + 1)] = Qb[e];
  for (int e = threadIdx.x; e < nr * m; e += 256) {
    const int i = e % nr, k = e / nr;
    Xs[k + i * (BAT_NMAX + 1)] = X[(r0 + i) + (long long)(o + k) * ldx];   // row i of the tile, K-major
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nr * m; e += 256) {
    const int i = e % nr, j = e / nr;
    double v = 0.0;
    for (int k = 0; k < m; ++k) v = fma(Xs[k + i * (BAT_NMAX + 1)], Qs[k + j * (BAT_NMAX + 1)], v);
    X[(r0 + i) + (long long)(o + j) * ldx] = v;
  }
}

}  // namespace sdc
