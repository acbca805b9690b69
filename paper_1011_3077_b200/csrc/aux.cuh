// aux.cuh -- HBM-bound O(n^2) kernels of the split step: stack/identity set-up, sums,
// index-remapped copies (transpose / reversal for RQ and QL via QR), norms, the R-test
// (Alg. 3 line 4) and the split selection (Alg. 4 line 5 / Alg. 5 line 3).
// All column-major; one thread per element with coalesced row-fastest indexing unless
// noted.  Reductions use fixed orders (no atomics) so results are run-to-run identical.
#pragma once
#include "common.cuh"

namespace sdc {

// grid-stride 2-D loop over an m x n column-major index space
#define SDC_FOR_MN(m, n)                                                                   \
  for (long long _e = (long long)blockIdx.x * blockDim.x + threadIdx.x,                      \
                 _tot = (long long)(m) * (n);                                              \
       _e < _tot; _e += (long long)gridDim.x * blockDim.x)

// out = alpha * identity (m x n)
__global__ void k_set_identity(double* out, long long ld, int m, int n, double alpha) {
  SDC_FOR_MN(m, n) {
    int i = (int)(_e % m), j = (int)(_e / m);
    out[i + (long long)j * ld] = (i == j) ? alpha : 0.0;
  }
}

// out (2n x n) = [0; I]   -- initial value for the IRS complement
__global__ void k_set_zero_identity(double* out, long long ld, int n) {
  SDC_FOR_MN(2 * n, n) {
    int i = (int)(_e % (2 * n)), j = (int)(_e / (2 * n));
    out[i + (long long)j * ld] = (i == n + j) ? 1.0 : 0.0;
  }
}

// out = op(src): trans=0 copy, trans=1 transpose (m x n result)
__global__ void k_copy(double* out, long long ldo, const double* src, long long lds, int m, int n,
                       double alpha) {
  SDC_FOR_MN(m, n) {
    int i = (int)(_e % m), j = (int)(_e / m);
    out[i + (long long)j * ldo] = alpha * src[i + (long long)j * lds];
  }
}

// hermitian embedding for the singular-value split:
//   H = [[0, A], [A^T, 0]]  (N = m + n, ld N), A m x n
__global__ void k_embed(double* H, const double* A, long long lda, int m, int n) {
  const int N = m + n;
  SDC_FOR_MN(N, N) {
    const int i = (int)(_e % N), j = (int)(_e / N);
    double v = 0.0;
    if (i < m && j >= m) v = A[i + (long long)(j - m) * lda];
    else if (i >= m && j < m) v = A[j + (long long)(i - m) * lda];
    H[i + (long long)j * N] = v;
  }
}

// ---- recursive divide-and-conquer helpers (sdc_schur, DESIGN.md §10 "recursion") ----------
// counter-based generator shared (re-implemented) by the oracle: splitmix64 of (seed, ctr)
SDC_DEV unsigned long long mix64(unsigned long long seed, unsigned long long ctr) {
  unsigned long long z = seed + 0x9E3779B97F4A7C15ull * (ctr + 1ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
// Gaussian (Box-Muller) matrix of order m from stream `key`: entry (i, j) uses counters
// (key << 40) + 2 (i + j m) and +1
__global__ void k_gauss(double* G, long long ldg, int m, unsigned long long seed, unsigned long long key) {
  SDC_FOR_MN(m, m) {
    const int i = (int)(_e % m), j = (int)(_e / m);
    const unsigned long long base = (key << 40) + 2ull * ((unsigned long long)i + (unsigned long long)j * m);
    const double u1 = (double)((mix64(seed, base) >> 11) + 1ull) * 1.1102230246251565e-16;
    const double u2 = (double)(mix64(seed, base + 1ull) >> 11) * 1.1102230246251565e-16;
    G[i + (long long)j * ldg] = sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
  }
}
// line search interval of the m x m block (invariant under orthogonal similarity):
// out[0] = c = trace/m, out[1] = ||T - c I||_F / sqrt(m)  (one CTA, fixed-order reductions)
__global__ void k_block_scale(const double* T, long long ldt, int m, double* out) {
  __shared__ double red[256];
  __shared__ double cs;
  double t = 0.0;
  for (int i = threadIdx.x; i < m; i += blockDim.x) t += T[i + (long long)i * ldt];
  red[threadIdx.x] = t;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) cs = red[0] / m;
  __syncthreads();
  const double c = cs;
  double f = 0.0;
  for (long long e = threadIdx.x; e < (long long)m * m; e += blockDim.x) {
    const int i = (int)(e % m), j = (int)(e / m);
    const double v = T[i + (long long)j * ldt] - (i == j ? c : 0.0);
    f += v * v;
  }
  __syncthreads();
  red[threadIdx.x] = f;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) { out[0] = c; out[1] = sqrt(red[0] / m); }
}
// T block (m x m) <- Ahat with E21 = Ahat(r:m, 0:r) set to zero
__global__ void k_place_ahat(double* T, long long ldt, const double* Ah, long long ldah, int m, int r) {
  SDC_FOR_MN(m, m) {
    const int i = (int)(_e % m), j = (int)(_e / m);
    T[i + (long long)j * ldt] = (i >= r && j < r) ? 0.0 : Ah[i + (long long)j * ldah];
  }
}

// tiled transpose-with-remap:  out(i, j) = s(j) * src(ri(i, j), rj(i, j)) where the mode
// selects the remap (used for RQ = reversed QR of C^T J and QL = reversed QR of J X J):
//   mode 0: out(i,j) = src(j, i)                      (transpose)
//   mode 1: out(i,j) = src(n-1-j, i)                  (C^T J)
//   mode 2: out(i,j) = src(n-1-i, n-1-j)              (J X J, no transpose)
//   mode 3: out(i,j) = src(n-1-i, j)                  (J X, row reversal)
// out1 = out2 = rho * src^T (n x n).  The first IRS pass of an RNEP step has B_0 = rho I, so
// B_1 = Q22^T B_0 = rho Q22^T: the product with the identity is a scaled transpose (the same
// values the GEMM would produce: every other term of its dot products is an exact zero).
__global__ void k_transpose_scale2(double* out1, long long ld1, double* out2, long long ld2,
                                   const double* src, long long lds, int n, double rho) {
  __shared__ double tile[32][33];
  const int bi = blockIdx.x * 32, bj = blockIdx.y * 32, tx = threadIdx.x, ty = threadIdx.y;
  for (int r = ty; r < 32; r += 8) {
    const int sr = bj + tx, sc = bi + r;
    if (sr < n && sc < n) tile[r][tx] = src[sr + (long long)sc * lds];
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int i = bi + tx, j = bj + r;
    if (i < n && j < n) {
      const double v = rho * tile[tx][r];
      out1[i + (long long)j * ld1] = v;
      out2[i + (long long)j * ld2] = v;
    }
  }
}

__global__ void k_transpose_rev(double* out, long long ldo, const double* src, long long lds, int n,
                                int mode) {
  __shared__ double tile[32][33];
  int bi = blockIdx.x * 32, bj = blockIdx.y * 32;
  int tx = threadIdx.x, ty = threadIdx.y;   // 32 x 8
  if (mode >= 2) {
    for (int r = ty; r < 32; r += 8) {
      int i = bi + tx, j = bj + r;
      int sj = mode == 2 ? n - 1 - j : j;
      if (i < n && j < n) out[i + (long long)j * ldo] = src[(n - 1 - i) + (long long)sj * lds];
    }
    return;
  }
  // read src block (rows bj.., cols bi..) coalesced, write transposed
  for (int r = ty; r < 32; r += 8) {
    int sr = bj + tx, sc = bi + r;           // src row (maps to out col), src col (out row)
    if (sr < n && sc < n) {
      int srow = (mode == 1) ? (n - 1 - sr) : sr;
      tile[r][tx] = src[srow + (long long)sc * lds];
    }
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    int i = bi + tx, j = bj + r;             // out(i,j) = src(map(j), i)
    if (i < n && j < n) out[i + (long long)j * ldo] = tile[tx][r];
  }
}

// X(i,i) += c  (n x n)
__global__ void k_add_diag(double* X, long long ldx, int n, double c) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    X[i + (long long)i * ldx] += c;
}

// RSEP (Alg. 6): X <- (X + X^T)/2 in place; one thread per pair i < j
__global__ void k_symmetrize(double* X, long long ldx, int n) {
  SDC_FOR_MN(n, n) {
    int i = (int)(_e % n), j = (int)(_e / n);
    if (i < j) {
      double v = 0.5 * (X[i + (long long)j * ldx] + X[j + (long long)i * ldx]);
      X[i + (long long)j * ldx] = v;
      X[j + (long long)i * ldx] = v;
    }
  }
}

// out = a + b (m x n)
__global__ void k_add(double* out, long long ldo, const double* a, long long lda, const double* b,
                      long long ldb, int m, int n) {
  SDC_FOR_MN(m, n) {
    int i = (int)(_e % m), j = (int)(_e / m);
    out[i + (long long)j * ldo] = a[i + (long long)j * lda] + b[i + (long long)j * ldb];
  }
}

// stack S (2n x n, ld lds) = [B; -A]
__global__ void k_build_stack(double* S, long long lds, const double* A, long long lda,
                              const double* B, long long ldb, int n) {
  SDC_FOR_MN(2 * n, n) {
    int i = (int)(_e % (2 * n)), j = (int)(_e / (2 * n));
    S[i + (long long)j * lds] = (i < n) ? B[i + (long long)j * ldb] : -A[(i - n) + (long long)j * lda];
  }
}

// rows i of X scaled by sign(diag(Rf)(i)) (sign(0)=+1): U <- U D_U applied as U^T C rows
__global__ void k_row_sign(double* X, long long ldx, const double* Rf, long long ldr, int n, int ncols) {
  SDC_FOR_MN(n, ncols) {
    int i = (int)(_e % n), j = (int)(_e / n);
    if (Rf[i + (long long)i * ldr] < 0.0) X[i + (long long)j * ldx] = -X[i + (long long)j * ldx];
  }
}

// Q(:, j) = sign(R(jj,jj)) * Qs(:, jj) with jj = rev ? n-1-j : j   (sign fix + reversal)
__global__ void k_col_sign_rev(double* Q, long long ldq, const double* Qs, long long lds,
                               const double* Rf, long long ldr, int n, int rev) {
  SDC_FOR_MN(n, n) {
    int i = (int)(_e % n), j = (int)(_e / n);
    int jj = rev ? n - 1 - j : j;
    double d = Rf[jj + (long long)jj * ldr] < 0.0 ? -1.0 : 1.0;
    Q[i + (long long)j * ldq] = d * Qs[i + (long long)jj * lds];
  }
}

// X(:, j) *= sign(Rf(j,j))  (m x n)
__global__ void k_col_sign(double* X, long long ldx, int m, int n, const double* Rf, long long ldr) {
  SDC_FOR_MN(m, n) {
    int i = (int)(_e % m), j = (int)(_e / m);
    if (Rf[j + (long long)j * ldr] < 0.0) X[i + (long long)j * ldx] = -X[i + (long long)j * ldx];
  }
}

// R(i, i:n) *= sign(R(i,i)) for the upper triangle of A (one warp per row: the diagonal is
// read before any lane of that warp writes the row, and no other warp touches it)
__global__ void k_r_rows_nonneg(double* A, long long lda, int n) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= n) return;
  const int i = warp;
  const bool neg = A[i + (long long)i * lda] < 0.0;
  __syncwarp();
  if (neg)
    for (int j = i + lane; j < n; j += 32) A[i + (long long)j * lda] = -A[i + (long long)j * lda];
}

// ---- norms: one warp per column -> per-column abs-sum and sum of squares ------------
__global__ void k_colnorms(const double* X, long long ldx, int m, int n, double* colabs,
                           double* colsq) {
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  int nw = (gridDim.x * blockDim.x) >> 5;
  for (int j = warp; j < n; j += nw) {
    double sa = 0.0, sq = 0.0;
    for (int i = lane; i < m; i += 32) {
      double v = X[i + (long long)j * ldx];
      sa += fabs(v);
      sq = fma(v, v, sq);
    }
    sa = warp_sum(sa);
    sq = warp_sum(sq);
    if (lane == 0) { colabs[j] = sa; colsq[j] = sq; }
  }
}

// single-CTA fixed-order reduction: out[0] = max_j colabs[j], out[1] = sqrt(sum_j colsq[j])
__global__ void k_norm_finish(const double* colabs, const double* colsq, int n, double* out) {
  __shared__ double smx[32], ssq[32];
  double mx = 0.0, sq = 0.0;
  bool nan = false;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    double a = colabs[j];
    nan |= (a != a);
    mx = fmax(mx, a);
    sq += colsq[j];
  }
  mx = warp_max(mx);
  sq = warp_sum(sq);
  nan = __any_sync(0xffffffffu, nan);
  int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __shared__ int snan;
  if (threadIdx.x == 0) snan = 0;
  __syncthreads();
  if (nan && l == 0) snan = 1;
  if (l == 0) { smx[w] = mx; ssq[w] = sq; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double M = 0.0, Q = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) { M = fmax(M, smx[i]); Q += ssq[i]; }
    out[0] = snan ? __longlong_as_double(0x7ff8000000000000ll) : M;
    out[1] = sqrt(Q);
  }
}

// ---- R-test (Alg. 3 line 4) -------------------------------------------
// R_j = D S(0:n,0:n) upper (D = sign(diag)), per column c:
//   dabs[c] = sum_{i<=c} |R_j(i,c) - Rprev(i,c)|,  pabs[c] = sum_{i<=c} |Rprev(i,c)|
// then Rprev <- R_j.  One warp per column.
__global__ void k_rtest_cols(const double* S, long long lds, double* Rprev, int n, double* dabs,
                             double* pabs) {
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  int nw = (gridDim.x * blockDim.x) >> 5;
  for (int c = warp; c < n; c += nw) {
    double sd = 0.0, sp = 0.0;
    for (int i = lane; i <= c; i += 32) {
      double d = S[i + (long long)i * lds] < 0.0 ? -1.0 : 1.0;
      double r = d * S[i + (long long)c * lds];
      double p = Rprev[i + (long long)c * n];
      sd += fabs(r - p);
      sp += fabs(p);
      Rprev[i + (long long)c * n] = r;
    }
    sd = warp_sum(sd);
    sp = warp_sum(sp);
    if (lane == 0) { dabs[c] = sd; pabs[c] = sp; }
  }
}

// ratio = max(dabs)/max(pabs) -> hist[slot] (single CTA)
__global__ void k_rtest_finish(const double* dabs, const double* pabs, int n, double* out) {
  __shared__ double sd[32], sp[32];
  double md = 0.0, mp = 0.0;
  for (int j = threadIdx.x; j < n; j += blockDim.x) { md = fmax(md, dabs[j]); mp = fmax(mp, pabs[j]); }
  md = warp_max(md);
  mp = warp_max(mp);
  if ((threadIdx.x & 31) == 0) { sd[threadIdx.x >> 5] = md; sp[threadIdx.x >> 5] = mp; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double D = 0.0, P = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) { D = fmax(D, sd[i]); P = fmax(P, sp[i]); }
    *out = D / P;
  }
}

// ---- split selection (blocked column prefix-sum, then row max) ----------
// Stage 1: CTA b owns columns [32b, 32b+32).  Walking rows bottom-up in 32-row chunks it
// keeps the column suffix sums s_c(r) = sum_{i >= r} |Ah(i,c)| (0-based; E21 for a leading
// block of order r is rows r..n-1, columns 0..r-1) and writes, for every row r, the block's
// max over its columns c < r:   pm[b][r] = max_{c in block, c < r} s_c(r).
constexpr int SEL_T = 32;
__global__ void __launch_bounds__(256) k_select_cols(const double* Ah, long long lda, int n,
                                                     double* pm) {
  __shared__ double tile[SEL_T][SEL_T + 1];   // [row][col]
  const int b = blockIdx.x, c0 = b * SEL_T;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 x 8
  double run = 0.0;                            // running suffix sum of column c0+tx (warp 0)
  const int nchunks = (n + SEL_T - 1) / SEL_T;
  for (int ch = nchunks - 1; ch >= 0; --ch) {
    const int rb = ch * SEL_T;
    if (rb + SEL_T <= c0) {                    // rows all above the block's columns: only r <= c
      // rows r < c0+1 can still need pm for r > c for some c in block: r > c >= c0 impossible
      for (int r = threadIdx.x; r < SEL_T; r += blockDim.x)
        if (rb + r < n) pm[(long long)b * n + rb + r] = 0.0;
      continue;
    }
    for (int r = ty; r < SEL_T; r += 8) {      // coalesced: lanes along rows of one column
      int gr = rb + tx, gc = c0 + r;
      tile[tx][r] = (gr < n && gc < n) ? fabs(Ah[gr + (long long)gc * lda]) : 0.0;
    }
    __syncthreads();
    if (ty == 0) {
      // lane tx = column c0+tx: suffix sums bottom-up within the chunk (row order n-1 -> 0)
      for (int r = SEL_T - 1; r >= 0; --r) {
        run += tile[r][tx];
        tile[r][tx] = run;                     // s_c(rb + r)
      }
    }
    __syncthreads();
    if (ty == 0) {
      // lane tx = row rb+tx: max over block columns c < row
      int gr = rb + tx;
      double mx = 0.0;
      for (int c = 0; c < SEL_T; ++c)
        if (c0 + c < gr && c0 + c < n) mx = fmax(mx, tile[tx][c]);
      if (gr < n) pm[(long long)b * n + gr] = mx;
    }
    __syncthreads();
  }
}

// Stage 2: m(r) = max_{b} pm[b][r] / normA (+ same for B), r = 1..n-1 -> mvals[r]
__global__ void k_select_rows(const double* pmA, const double* pmB, int n, int nblk,
                              const double* normA, const double* normB, double* mvals) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < 1 || r >= n) return;
  int bmax = min(nblk, (r + SEL_T - 1) / SEL_T);   // blocks with c0 < r
  double ma = 0.0, mb = 0.0;
  for (int b = 0; b < bmax; ++b) {
    ma = fmax(ma, pmA[(long long)b * n + r]);
    if (pmB) mb = fmax(mb, pmB[(long long)b * n + r]);
  }
  mvals[r] = ma / normA[0] + (pmB ? mb / normB[0] : 0.0);
}

// Stage 3 (single CTA, 1024 threads): argmin over r = 1..n-1, ties -> smallest r
// (SPEC.md:255); out = {r, metric}.  NaN never wins a comparison; all-NaN -> r = 1.
__global__ void __launch_bounds__(1024) k_select_argmin(const double* mvals, int n, double* out) {
  __shared__ double sv[1024];
  __shared__ int si[1024];
  const int NONE = 0x7fffffff;
  double best = __longlong_as_double(0x7ff0000000000000ll);  // +inf
  int bi = NONE;
  for (int r = 1 + threadIdx.x; r < n; r += blockDim.x) {
    double v = mvals[r];
    if (v < best) { best = v; bi = r; }
  }
  sv[threadIdx.x] = best;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int s = blockDim.x >> 1; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      double v2 = sv[threadIdx.x + s];
      int i2 = si[threadIdx.x + s];
      if (v2 < sv[threadIdx.x] || (v2 == sv[threadIdx.x] && i2 < si[threadIdx.x])) {
        sv[threadIdx.x] = v2;
        si[threadIdx.x] = i2;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    int r = si[0] == NONE ? 1 : si[0];
    out[0] = (double)r;
    out[1] = mvals[r];
  }
}

// ||Ah(r:n, 0:r)||_F^2 per column (warp per column), r read from sel[0]
__global__ void k_e21_fro_cols(const double* Ah, long long lda, int n, const double* sel,
                               double* colsq) {
  int r = (int)sel[0];
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  int nw = (gridDim.x * blockDim.x) >> 5;
  for (int c = warp; c < n; c += nw) {
    double s = 0.0;
    if (c < r)
      for (int i = r + lane; i < n; i += 32) { double v = Ah[i + (long long)c * lda]; s = fma(v, v, s); }
    s = warp_sum(s);
    if (lane == 0) colsq[c] = s;
  }
}

// out = sqrt(sum colsqA)/froA (+ sqrt(sum colsqB)/froB), single CTA, fixed order
__global__ void k_e21_fro_finish(const double* colsqA, const double* colsqB, int n,
                                 const double* nrmA, const double* nrmB, double* out) {
  __shared__ double sa[32], sb[32];
  double a = 0.0, b = 0.0;
  for (int j = threadIdx.x; j < n; j += blockDim.x) { a += colsqA[j]; if (colsqB) b += colsqB[j]; }
  a = warp_sum(a);
  b = warp_sum(b);
  if ((threadIdx.x & 31) == 0) { sa[threadIdx.x >> 5] = a; sb[threadIdx.x >> 5] = b; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double A = 0.0, B = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) { A += sa[i]; B += sb[i]; }
    *out = sqrt(A) / nrmA[1] + (colsqB ? sqrt(B) / nrmB[1] : 0.0);
  }
}

// non-finite scan: flag[0] |= any(!isfinite(X))
__global__ void k_nonfinite(const double* X, long long ldx, int n, int* flag) {
  bool bad = false;
  SDC_FOR_MN(n, n) {
    int i = (int)(_e % n), j = (int)(_e / n);
    double v = X[i + (long long)j * ldx];
    bad |= !isfinite(v);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

// WY reduction for split-K partials:  W(:, c) = op(T) * sum_s Wp[s](:, c)
//   trans = 1: W = T^T W0 (apply H^T = I - Y T^T Y^T, i.e. Q^T C);  trans = 0: W = T W0.
// One CTA (256 threads) per block of cpb <= WYR_COLS columns (cpb chosen by the host so the
// grid covers the SMs even for the 64..192-column inner updates); when a block has fewer
// than 256 entries, g = 256 / (cpb nb) thread groups sum interleaved split slices and the
// group sums are added in a fixed order (deterministic).  T staged in smem.
constexpr int WYR_COLS = 16;
__global__ void __launch_bounds__(256) k_wy_reduce(const double* Wp, int splits, long long zstride,
                                                   int nb, int ncols, const double* T, int trans,
                                                   double* W, int cpb) {
  __shared__ double Ts[64 * 64];
  __shared__ double part[WYR_COLS * 64];
  __shared__ double w0[WYR_COLS * 64];
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) Ts[e] = T[e];
  const int c0 = blockIdx.x * cpb;
  const int elems = cpb * nb;
  const int g = elems >= (int)blockDim.x ? 1 : (int)blockDim.x / elems;
  // partial sums over the split slices z = q0, q0 + dz, ...: 4 independent accumulators
  // (loads in flight together; the split count reaches ~150 for tall panels), combined in
  // a fixed order
  auto slice_sum = [&](const double* p, int q0, int dz) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int z = q0;
    for (; z + 3 * dz < splits; z += 4 * dz) {
      s0 += p[(long long)z * zstride];
      s1 += p[(long long)(z + dz) * zstride];
      s2 += p[(long long)(z + 2 * dz) * zstride];
      s3 += p[(long long)(z + 3 * dz) * zstride];
    }
    for (; z < splits; z += dz) s0 += p[(long long)z * zstride];
    return (s0 + s1) + (s2 + s3);
  };
  if (g == 1) {
    for (int e = threadIdx.x; e < elems; e += blockDim.x) {
      const int c = c0 + e / nb;
      double s = 0.0;
      if (c < ncols) s = slice_sum(Wp + (e % nb) + (long long)c * nb, 0, 1);
      w0[e] = s;
    }
  } else {
    const int e = threadIdx.x % elems, q = threadIdx.x / elems;
    if (q < g) {
      const int c = c0 + e / nb;
      double s = 0.0;
      if (c < ncols) s = slice_sum(Wp + (e % nb) + (long long)c * nb, q, g);
      part[q * elems + e] = s;
    }
    __syncthreads();
    if (threadIdx.x < elems) {
      double s = part[threadIdx.x];
      for (int r = 1; r < g; ++r) s += part[r * elems + threadIdx.x];
      w0[threadIdx.x] = s;
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < elems; e += blockDim.x) {
    const int cc = e / nb, i = e % nb, c = c0 + cc;
    if (c >= ncols) continue;
    const double* w = w0 + cc * nb;
    double s = 0.0;
    if (trans) {   // (T^T w)(i) = sum_{l <= i} T(l, i) w(l)
      for (int l = 0; l <= i; ++l) s = fma(Ts[i * nb + l], w[l], s);
    } else {       // (T w)(i) = sum_{l >= i} T(i, l) w(l)
      for (int l = i; l < nb; ++l) s = fma(Ts[l * nb + i], w[l], s);
    }
    W[i + (long long)c * nb] = s;
  }
}

// Z = sum_z P[z] (m x n blocks, z-stride zs, ld m), fixed order
__global__ void k_sum_partials(const double* P, int splits, long long zs, long long total, double* Z) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;   // 4 loads in flight, fixed combine order
    int z = 0;
    for (; z + 3 < splits; z += 4) {
      s0 += P[(long long)z * zs + e];
      s1 += P[(long long)(z + 1) * zs + e];
      s2 += P[(long long)(z + 2) * zs + e];
      s3 += P[(long long)(z + 3) * zs + e];
    }
    for (; z < splits; ++z) s0 += P[(long long)z * zs + e];
    Z[e] = (s0 + s1) + (s2 + s3);
  }
}

// Outer compact-WY block assembly.  T_O (nbo x nbo, ld nbo) and its transpose T_Ot:
// k_tout_place zeroes both and copies the inner 64x64 T blocks onto the diagonal.
__global__ void k_tout_place(double* TO, double* TOt, int nbo, const double* Tinner) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nbo * nbo; e += gridDim.x * blockDim.x) {
    int i = e % nbo, j = e / nbo;
    double v = 0.0;
    if ((i >> 6) == (j >> 6) && i <= j) {
      int b = i >> 6, nbb = min(64, nbo - b * 64);
      v = Tinner[(size_t)b * 64 * 64 + (size_t)(j & 63) * nbb + (i & 63)];
    }
    TO[i + (long long)j * nbo] = v;
    TOt[j + (long long)i * nbo] = v;
  }
}

// Merge of two adjacent compact-WY blocks (the recursive T of Elmroth-Gustavson):
//   (I - Ya Ta Ya^T)(I - Yb Tb Yb^T) = I - [Ya Yb] [[Ta, X], [0, Tb]] [Ya Yb]^T,
//   X = -Ta (Ya^T Yb) Tb.
// Ta = TO[a0:a0+p, a0:a0+p], Tb = TO[b0:b0+q, b0:b0+q] (upper triangular, zeros below),
// G = Y_O^T Y_O (ld nbo).  CTA (bx, by) computes the 32x32 block of X at rows 32bx, cols
// 32by; writes X into TO and X^T into TOt.
__global__ void __launch_bounds__(256) k_tmerge(double* TO, double* TOt, int nbo, const double* G,
                                                int a0, int p, int b0, int q) {
  __shared__ double Ta[32][33];    // Ta[rb:rb+32, l0:l0+32]
  __shared__ double Gc[32][33];    // G[a0+l0 : +32, b0+c0 : +32]
  __shared__ double U[32][33];
  __shared__ double Tb[32][33];
  const int rb = blockIdx.x * 32, cb = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 x 8
  double acc[4] = {0, 0, 0, 0};
  for (int c0 = 0; c0 < q; c0 += 32) {
    double u[4] = {0, 0, 0, 0};
    for (int l0 = 0; l0 < p; l0 += 32) {
      __syncthreads();
      for (int e = threadIdx.x; e < 32 * 32; e += 256) {
        int r = e % 32, c = e / 32;
        Ta[r][c] = (rb + r < p && l0 + c < p) ? TO[(a0 + rb + r) + (long long)(a0 + l0 + c) * nbo] : 0.0;
        Gc[r][c] = (l0 + r < p && c0 + c < q) ? G[(a0 + l0 + r) + (long long)(b0 + c0 + c) * nbo] : 0.0;
      }
      __syncthreads();
      for (int t = 0; t < 4; ++t) {      // U += Ta(32 x 32) Gc(32 x 32)
        const int c = ty + 8 * t;
        double sum = u[t];
        for (int l = 0; l < 32; ++l) sum = fma(Ta[tx][l], Gc[l][c], sum);
        u[t] = sum;
      }
    }
    __syncthreads();
    for (int t = 0; t < 4; ++t) U[tx][ty + 8 * t] = u[t];
    for (int e = threadIdx.x; e < 32 * 32; e += 256) {
      int r = e % 32, c = e / 32;
      Tb[r][c] = (c0 + r < q && cb + c < q) ? TO[(b0 + c0 + r) + (long long)(b0 + cb + c) * nbo] : 0.0;
    }
    __syncthreads();
    for (int t = 0; t < 4; ++t) {        // acc += U(32 x 32) Tb(32 x 32)
      const int c = ty + 8 * t;
      double sum = acc[t];
      for (int l = 0; l < 32; ++l) sum = fma(U[tx][l], Tb[l][c], sum);
      acc[t] = sum;
    }
  }
  for (int t = 0; t < 4; ++t) {
    int r = rb + tx, c = cb + ty + 8 * t;
    if (r < p && c < q) {
      TO[(a0 + r) + (long long)(b0 + c) * nbo] = -acc[t];
      TOt[(b0 + c) + (long long)(a0 + r) * nbo] = -acc[t];
    }
  }
}

}  // namespace sdc
