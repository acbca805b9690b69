/*
 * sdc_oracle.c -- plain, slow, CPU fp64 ORACLE for one inverse-free split step
 * of randomized spectral divide-and-conquer (arXiv 1011.3077, Ballard-Demmel-Dumitriu).
 *
 * THIS IS TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  It shares no code,
 * header, table or helper with the CUDA path (paper_1011_3077_b200/csrc), and neither
 * side includes or links the other.
 *
 * Every routine is the textbook unblocked algorithm, written out in the paper's order:
 *   - Householder reflector (LAPACK dlarfg convention)      DESIGN.md reading Q7
 *   - Householder QR / RQ / QL (dgeqr2 / dgerq2 / dgeql2)   PAPER.md:331 ("QR, RQ, QL")
 *   - IRS pass  [B_j;-A_j] = Q [R_j;0], A_{j+1}=Q12^T A_j,
 *               B_{j+1}=Q22^T B_j                           PAPER.md:362-375 (Alg. 3)
 *   - GRURV(2, A_p+B_p, A_p; -1,+1)                         PAPER.md:164-174, 262-283 (Alg. 1, 2)
 *   - GRURV(2, A'_p^T, (A'_p+B'_p)^T; +1,-1)  (pencil Q_L)  PAPER.md:388 (Alg. 4 line 4)
 *   - similarity  Ahat = Q_L^T A Q_R                        PAPER.md:389-390, 418 (Alg. 4/5)
 *   - split selection  min_r ||E21||_1/||A||_1 (+F21)
 * There is no blocking, fusion or reordering beyond what those definitions state.  Every
 * output element is produced by one thread with a fixed summation order (OpenMP only
 * splits independent columns, static schedule), so results are bit-identical for any
 * thread count.  Build: gcc -O2 -ffp-contract=off -fopenmp (no -ffast-math).
 *
 * Storage: column-major, element (i,j) of a matrix with leading dimension ld is
 * a[i + j*ld], indices 0-based in the code (the paper's are 1-based).
 *
 * Parity pins: see tests/test_oracle_*.py; every function here is pinned.
 */
#include "sdc_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define EL(a, i, j, ld) ((a)[(size_t)(j) * (size_t)(ld) + (size_t)(i)])
/* OpenMP only for large problems (thread start-up dominates tiny ones).  Scheduling only:
 * every output element is still computed by one thread in the same loop order, so the
 * results do not depend on this threshold or on the thread count. */
#define ORC_PAR_MIN 65536L

static double sgn_nonneg(double x) { return x < 0.0 ? -1.0 : 1.0; } /* sign(0)=+1 (Q7) */

/* ------------------------------------------------------------------------------------
 * Householder reflector, LAPACK dlarfg convention (reading Q7):
 *   given alpha and x (length nx), find beta, tau, v = [1; x/(alpha-beta)] with
 *   (I - tau v v^T) [alpha; x] = [beta; 0],  beta = -sign(alpha) * ||[alpha; x]||.
 *   If ||x|| = 0 then tau = 0 (H = I) and beta = alpha.
 * ---------------------------------------------------------------------------------- */
static void larfg(int nx, double *alpha, double *x, size_t incx, double *tau) {
  double xn2 = 0.0;
  for (int i = 0; i < nx; ++i) xn2 += x[i * incx] * x[i * incx];
  if (xn2 == 0.0) { *tau = 0.0; return; }
  double a = *alpha;
  double nrm = sqrt(a * a + xn2);
  double beta = -sgn_nonneg(a) * nrm;
  *tau = (beta - a) / beta;
  double scal = 1.0 / (a - beta);
  for (int i = 0; i < nx; ++i) x[i * incx] *= scal;
  *alpha = beta;
}

/* ------------------------------------------------------------------------------------
 * Householder QR (dgeqr2): A (m x n, m >= n) = H_0 H_1 ... H_{n-1} [R; 0].
 * On exit R is in the upper triangle, v_k (below its implicit unit diagonal) in column k
 * below the diagonal, tau[k] the scalar of H_k = I - tau_k v_k v_k^T.
 * ---------------------------------------------------------------------------------- */
void orc_geqr2(int m, int n, double *A, int lda, double *tau) {
  int kmax = m < n ? m : n;
  for (int k = 0; k < kmax; ++k) {
    larfg(m - k - 1, &EL(A, k, k, lda), &EL(A, k + 1, k, lda), 1, &tau[k]);
    double t = tau[k];
    if (t == 0.0) continue;
#pragma omp parallel for schedule(static) if ((long)m * n >= ORC_PAR_MIN)
    for (int j = k + 1; j < n; ++j) {           /* apply H_k to column j */
      double w = EL(A, k, j, lda);
      for (int i = k + 1; i < m; ++i) w += EL(A, i, k, lda) * EL(A, i, j, lda);
      w *= t;
      EL(A, k, j, lda) -= w;
      for (int i = k + 1; i < m; ++i) EL(A, i, j, lda) -= w * EL(A, i, k, lda);
    }
  }
}

/* Apply H_k (reflector k of a geqr2 factorisation stored in Y) to columns [c0,c1) of
 * C (rows k..m-1 are touched):  C <- (I - tau v v^T) C. */
static void apply_qr_reflector(int m, int k, const double *Y, int ldy, double tau,
                               double *C, int ldc, int c0, int c1) {
  if (tau == 0.0) return;
#pragma omp parallel for schedule(static) if ((long)m * (c1 - c0) >= ORC_PAR_MIN)
  for (int j = c0; j < c1; ++j) {
    double w = EL(C, k, j, ldc);
    for (int i = k + 1; i < m; ++i) w += EL(Y, i, k, ldy) * EL(C, i, j, ldc);
    w *= tau;
    EL(C, k, j, ldc) -= w;
    for (int i = k + 1; i < m; ++i) EL(C, i, j, ldc) -= w * EL(Y, i, k, ldy);
  }
}

/* C (m x nc) <- Q^T C = H_{n-1} ... H_1 H_0 C for the QR factorisation in (Y, tau). */
void orc_apply_qt(int m, int n, const double *Y, int ldy, const double *tau,
                  int nc, double *C, int ldc) {
  for (int k = 0; k < n; ++k) apply_qr_reflector(m, k, Y, ldy, tau[k], C, ldc, 0, nc);
}

/* Explicit square Q (n x n) = H_0 ... H_{n-1} of a geqr2 factorisation of an n x n
 * matrix, column-scaled by D = sign(diag R) so that Q*(D R) is the QR with diag >= 0
 * (dorg2r; H_{n-1} is applied first).  Q may not alias Y. */
void orc_org2r_signed(int n, const double *Y, int ldy, const double *tau,
                      double *Q, int ldq) {
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) EL(Q, i, j, ldq) = (i == j) ? 1.0 : 0.0;
  for (int k = n - 1; k >= 0; --k) apply_qr_reflector(n, k, Y, ldy, tau[k], Q, ldq, k, n);
  for (int j = 0; j < n; ++j) {
    double d = sgn_nonneg(EL(Y, j, j, ldy));
    if (d < 0) for (int i = 0; i < n; ++i) EL(Q, i, j, ldq) = -EL(Q, i, j, ldq);
  }
}

/* Complement of an IRS stack QR: the last n columns of the 2n x 2n
 * Q = H_0 ... H_{n-1}, i.e. [Q12; Q22] = H_0 ... H_{n-1} [0; I_n] (H_{n-1} applied first).
 * The diag(R) >= 0 normalisation only flips the FIRST n columns of Q, so it does not
 * touch the complement (reading Q6). */
void orc_complement(int n, const double *Y, int ldy, const double *tau, double *C, int ldc) {
  int m = 2 * n;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < m; ++i) EL(C, i, j, ldc) = (i == n + j) ? 1.0 : 0.0;
  for (int k = n - 1; k >= 0; --k) apply_qr_reflector(m, k, Y, ldy, tau[k], C, ldc, 0, n);
}

/* ------------------------------------------------------------------------------------
 * RQ (dgerq2) of a square n x n matrix:  A = R * Q_rq with Q_rq = H(0) H(1) ... H(n-1).
 * Row i (processed from n-1 down to 0) is annihilated left of the diagonal by a
 * reflector acting on columns 0..i from the right; v_i = [x*scale, 1] is stored in
 * row i, columns 0..i-1 (unit element at column i implicit).
 * ---------------------------------------------------------------------------------- */
void orc_gerq2(int n, double *A, int lda, double *tau) {
  for (int i = n - 1; i >= 0; --i) {
    larfg(i, &EL(A, i, i, lda), &EL(A, i, 0, lda), (size_t)lda, &tau[i]);
    double t = tau[i];
    if (t == 0.0) continue;
    /* A(0:i-1, 0:i) <- A(0:i-1, 0:i) (I - t v v^T), v = [A(i,0:i-1), 1] */
#pragma omp parallel for schedule(static) if ((long)n * n >= ORC_PAR_MIN)
    for (int r = 0; r < i; ++r) {
      double w = EL(A, r, i, lda);
      for (int c = 0; c < i; ++c) w += EL(A, r, c, lda) * EL(A, i, c, lda);
      w *= t;
      EL(A, r, i, lda) -= w;
      for (int c = 0; c < i; ++c) EL(A, r, c, lda) -= w * EL(A, i, c, lda);
    }
  }
}

/* Explicit Q_rq = H(0) ... H(n-1) of a gerq2 factorisation, row-scaled by D = sign(diag R)
 * so that A = (R D)(D Q_rq) has diag(R D) >= 0 (reading Q10). */
void orc_orgr2_signed(int n, const double *Y, int ldy, const double *tau, double *Q, int ldq) {
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) EL(Q, i, j, ldq) = (i == j) ? 1.0 : 0.0;
  /* H(n-1) first, H(0) last; H(i) acts on rows 0..i, v = [Y(i,0:i-1), 1] */
  for (int i = n - 1; i >= 0; --i) {
    double t = tau[i];
    if (t == 0.0) continue;
#pragma omp parallel for schedule(static) if ((long)n * n >= ORC_PAR_MIN)
    for (int j = 0; j < n; ++j) {
      double w = EL(Q, i, j, ldq);
      for (int c = 0; c < i; ++c) w += EL(Y, i, c, ldy) * EL(Q, c, j, ldq);
      w *= t;
      EL(Q, i, j, ldq) -= w;
      for (int c = 0; c < i; ++c) EL(Q, c, j, ldq) -= w * EL(Y, i, c, ldy);
    }
  }
  for (int i = 0; i < n; ++i) {
    double d = sgn_nonneg(EL(Y, i, i, ldy));
    if (d < 0) for (int j = 0; j < n; ++j) EL(Q, i, j, ldq) = -EL(Q, i, j, ldq);
  }
}

/* ------------------------------------------------------------------------------------
 * QL (dgeql2) of a square n x n matrix: A = Q_ql * L, Q_ql = H(n-1) ... H(1) H(0).
 * Column i (from n-1 down to 0) is annihilated above the diagonal by a reflector on
 * rows 0..i; v_i = [x*scale; 1] stored in column i, rows 0..i-1.
 * ---------------------------------------------------------------------------------- */
void orc_geql2(int n, double *A, int lda, double *tau) {
  for (int i = n - 1; i >= 0; --i) {
    larfg(i, &EL(A, i, i, lda), &EL(A, 0, i, lda), 1, &tau[i]);
    double t = tau[i];
    if (t == 0.0) continue;
    /* A(0:i, 0:i-1) <- (I - t v v^T) A(0:i, 0:i-1), v = [A(0:i-1,i); 1] */
#pragma omp parallel for schedule(static) if ((long)n * n >= ORC_PAR_MIN)
    for (int j = 0; j < i; ++j) {
      double w = EL(A, i, j, lda);
      for (int r = 0; r < i; ++r) w += EL(A, r, i, lda) * EL(A, r, j, lda);
      w *= t;
      EL(A, i, j, lda) -= w;
      for (int r = 0; r < i; ++r) EL(A, r, j, lda) -= w * EL(A, r, i, lda);
    }
  }
}

/* Explicit Q_ql = H(n-1) ... H(0) of a geql2 factorisation, column-scaled by
 * D = sign(diag L) so that A = (Q_ql D)(D L) has diag(D L) >= 0 (dorg2l). */
void orc_org2l_signed(int n, const double *Y, int ldy, const double *tau, double *Q, int ldq) {
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) EL(Q, i, j, ldq) = (i == j) ? 1.0 : 0.0;
  /* Q = H(n-1) ( ... (H(0) I)): H(0) applied first */
  for (int i = 0; i < n; ++i) {
    double t = tau[i];
    if (t == 0.0) continue;
#pragma omp parallel for schedule(static) if ((long)n * n >= ORC_PAR_MIN)
    for (int j = 0; j < n; ++j) {
      double w = EL(Q, i, j, ldq);
      for (int r = 0; r < i; ++r) w += EL(Y, r, i, ldy) * EL(Q, r, j, ldq);
      w *= t;
      EL(Q, i, j, ldq) -= w;
      for (int r = 0; r < i; ++r) EL(Q, r, j, ldq) -= w * EL(Y, r, i, ldy);
    }
  }
  for (int j = 0; j < n; ++j) {
    double d = sgn_nonneg(EL(Y, j, j, ldy));
    if (d < 0) for (int i = 0; i < n; ++i) EL(Q, i, j, ldq) = -EL(Q, i, j, ldq);
  }
}

/* ------------------------------------------------------------------------------------
 * Plain GEMM  C (m x n) = op(A) op(B), K inner; op = transpose when ta/tb != 0.
 * Each C(i,j) is one sum over k ascending.
 * ---------------------------------------------------------------------------------- */
void orc_gemm(int ta, int tb, int m, int n, int K, const double *A, int lda,
              const double *B, int ldb, double *C, int ldc) {
#pragma omp parallel for schedule(static) if ((long)m * n * K / 64 >= ORC_PAR_MIN)
  for (int j = 0; j < n; ++j) {
    for (int i = 0; i < m; ++i) {
      double s = 0.0;
      for (int k = 0; k < K; ++k) {
        double a = ta ? EL(A, k, i, lda) : EL(A, i, k, lda);
        double b = tb ? EL(B, j, k, ldb) : EL(B, k, j, ldb);
        s += a * b;
      }
      EL(C, i, j, ldc) = s;
    }
  }
}

/* ||X||_1 = max column absolute sum (m x n). */
double orc_norm1(int m, int n, const double *X, int ldx) {
  double best = 0.0;
  for (int j = 0; j < n; ++j) {
    double s = 0.0;
    for (int i = 0; i < m; ++i) s += fabs(EL(X, i, j, ldx));
    if (s > best || s != s) best = s;
  }
  return best;
}

static double norm_fro(int m, int n, const double *X, int ldx) {
  double s = 0.0;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < m; ++i) s += EL(X, i, j, ldx) * EL(X, i, j, ldx);
  return sqrt(s);
}

/* ------------------------------------------------------------------------------------
 * One IRS pass (Alg. 3 line 3):
 *   [B_j; -A_j] = Q [R_j; 0],  A_{j+1} = Q12^T A_j,  B_{j+1} = Q22^T B_j,
 * with Q12 = rows 0..n-1 (aligned with B_j) and Q22 = rows n..2n-1 of the complement
 * (reading Q9).  Rout (n x n, ld n), if not NULL, receives R_j with its
 * diagonal made non-negative (rows scaled by sign(diag)), zeros below the diagonal.
 * Aj/Bj are read, Aout/Bout written (may alias Aj/Bj).
 * ---------------------------------------------------------------------------------- */
void orc_irs_pass(int n, const double *Aj, int lda, const double *Bj, int ldb,
                  double *Aout, int ldao, double *Bout, int ldbo, double *Rout) {
  int m = 2 * n;
  double *S = (double *)malloc(sizeof(double) * (size_t)m * n);
  double *C = (double *)malloc(sizeof(double) * (size_t)m * n);
  double *tau = (double *)malloc(sizeof(double) * n);
  double *Anew = (double *)malloc(sizeof(double) * (size_t)n * n);
  double *Bnew = (double *)malloc(sizeof(double) * (size_t)n * n);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      EL(S, i, j, m) = EL(Bj, i, j, ldb);
      EL(S, n + i, j, m) = -EL(Aj, i, j, lda);
    }
  orc_geqr2(m, n, S, m, tau);
  if (Rout) {
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i)
        EL(Rout, i, j, n) = (i <= j) ? sgn_nonneg(EL(S, i, i, m)) * EL(S, i, j, m) : 0.0;
  }
  orc_complement(n, S, m, tau, C, m);
  orc_gemm(1, 0, n, n, n, C, m, Aj, lda, Anew, n);       /* Q12^T A_j */
  orc_gemm(1, 0, n, n, n, C + n, m, Bj, ldb, Bnew, n);   /* Q22^T B_j */
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      EL(Aout, i, j, ldao) = EL(Anew, i, j, n);
      EL(Bout, i, j, ldbo) = EL(Bnew, i, j, n);
    }
  free(S); free(C); free(tau); free(Anew); free(Bnew);
}

/* ------------------------------------------------------------------------------------
 * GRURV(2, A_p+B_p, A_p; -1, +1)  (Alg. 2 with k=2, m_1=-1, m_2=+1; Alg. 5 line 2):
 *   line 2 (RURV on A_2=A_p, Alg. 1): X = A_p V^T, [U, R_2] = QR(X)  (Q8)
 *   line 9 (m_1=-1):  [U', R_1] = RQ(U^T (A_p+B_p)),  U_current = U'^T
 * so (A_p+B_p)^{-1} A_p = Q R_1^{-1} R_2 V with Q = U'^T (lemma).
 * Both triangular factors get non-negative diagonals (U <- U D_U, U' <- D_R U').
 * Outputs: Q (n x n); optionally R1 and R2 (n x n, ld n, zero below diagonal).
 * ---------------------------------------------------------------------------------- */
void orc_grurv_right(int n, const double *Ap, int ldap, const double *Bp, int ldbp,
                     const double *V, int ldv, double *Q, int ldq, double *R1, double *R2) {
  size_t nn = (size_t)n * n;
  double *X = (double *)malloc(sizeof(double) * nn);
  double *Cm = (double *)malloc(sizeof(double) * nn);
  double *tx = (double *)malloc(sizeof(double) * n);
  double *tr = (double *)malloc(sizeof(double) * n);
  double *Qrq = (double *)malloc(sizeof(double) * nn);
  orc_gemm(0, 1, n, n, n, Ap, ldap, V, ldv, X, n);          /* X = A_p V^T */
  orc_geqr2(n, n, X, n, tx);                                 /* X = U R_2 */
  for (int j = 0; j < n; ++j)                                /* S = A_p + B_p */
    for (int i = 0; i < n; ++i) EL(Cm, i, j, n) = EL(Ap, i, j, ldap) + EL(Bp, i, j, ldbp);
  orc_apply_qt(n, n, X, n, tx, n, Cm, n);                    /* H_{n-1}..H_0 S */
  for (int i = 0; i < n; ++i) {                              /* U^T S with U <- U D_U */
    double d = sgn_nonneg(EL(X, i, i, n));
    if (d < 0) for (int j = 0; j < n; ++j) EL(Cm, i, j, n) = -EL(Cm, i, j, n);
  }
  if (R2)
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i)
        R2[(size_t)j * n + i] = (i <= j) ? sgn_nonneg(EL(X, i, i, n)) * EL(X, i, j, n) : 0.0;
  orc_gerq2(n, Cm, n, tr);                                   /* U^T S = R_1 U'  */
  if (R1)
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i)
        R1[(size_t)j * n + i] = (i <= j) ? EL(Cm, i, j, n) * sgn_nonneg(EL(Cm, j, j, n)) : 0.0;
  orc_orgr2_signed(n, Cm, n, tr, Qrq, n);                    /* U' (rows sign-fixed) */
  for (int j = 0; j < n; ++j)                                /* Q = U'^T */
    for (int i = 0; i < n; ++i) EL(Q, i, j, ldq) = EL(Qrq, j, i, n);
  free(X); free(Cm); free(tx); free(tr); free(Qrq);
}

/* ------------------------------------------------------------------------------------
 * GRURV(2, A'_p^T, (A'_p+B'_p)^T; +1, -1)  (Alg. 4 line 4), (A'_p, B'_p) = IRS(A^T, B^T):
 *   lines 4-5 (m_2=-1): RULV of ((A'_p+B'_p)^T)^T = A'_p+B'_p:
 *       X' = (A'_p+B'_p) V_L^T,  [U, L] = QL(X')
 *   line 6 (m_1=+1):  [U_current, R_1] = QR(A'_p^T U)   -> Q_L = U_current (explicit).
 * ---------------------------------------------------------------------------------- */
void orc_grurv_left(int n, const double *Ap, int ldap, const double *Bp, int ldbp,
                    const double *VL, int ldv, double *QL, int ldq) {
  size_t nn = (size_t)n * n;
  double *S = (double *)malloc(sizeof(double) * nn);
  double *X = (double *)malloc(sizeof(double) * nn);
  double *U = (double *)malloc(sizeof(double) * nn);
  double *Z = (double *)malloc(sizeof(double) * nn);
  double *tl = (double *)malloc(sizeof(double) * n);
  double *tq = (double *)malloc(sizeof(double) * n);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) EL(S, i, j, n) = EL(Ap, i, j, ldap) + EL(Bp, i, j, ldbp);
  orc_gemm(0, 1, n, n, n, S, n, VL, ldv, X, n);               /* X' = (A'+B') V_L^T */
  orc_geql2(n, X, n, tl);                                      /* X' = U L */
  orc_org2l_signed(n, X, n, tl, U, n);                         /* U explicit, diag(L) >= 0 */
  orc_gemm(1, 0, n, n, n, Ap, ldap, U, n, Z, n);               /* Z = A'_p^T U */
  orc_geqr2(n, n, Z, n, tq);
  orc_org2r_signed(n, Z, n, tq, QL, ldq);                      /* Q_L explicit */
  free(S); free(X); free(U); free(Z); free(tl); free(tq);
}

/* ------------------------------------------------------------------------------------
 * Split selection (readings Q3, Q4):
 *   for r = 1..n-1 (leading block order r, 1-based):
 *     m(r) = ||Ahat(r+1:n, 1:r)||_1 / normA  [+ ||Bhat(r+1:n,1:r)||_1 / normB]
 *   ||E21||_1 = max over columns c <= r of sum_{i > r} |Ahat(i,c)|.
 *   The column sums are accumulated bottom-up (row n first), r from n-1 down to 1.
 *   Returns r* = argmin (ties -> smallest r) and m(r*).  mvals (length n-1, optional)
 *   receives m(1..n-1).
 * ---------------------------------------------------------------------------------- */
double orc_split_select(int n, const double *Ah, int ldah, double normA,
                        const double *Bh, int ldbh, double normB, int *r_out, double *mvals) {
  double *sa = (double *)calloc((size_t)n, sizeof(double));
  double *sb = (double *)calloc((size_t)n, sizeof(double));
  double *m = (double *)malloc(sizeof(double) * (size_t)n);
  for (int r = n - 1; r >= 1; --r) {       /* 1-based r; add row r+1 (0-based row r) */
    double ma = 0.0, mb = 0.0;
    for (int c = 0; c < r; ++c) {           /* 0-based columns 0..r-1 (1-based 1..r) */
      sa[c] += fabs(EL(Ah, r, c, ldah));
      if (sa[c] > ma || sa[c] != sa[c]) ma = sa[c];
      if (Bh) {
        sb[c] += fabs(EL(Bh, r, c, ldbh));
        if (sb[c] > mb || sb[c] != sb[c]) mb = sb[c];
      }
    }
    m[r] = ma / normA + (Bh ? mb / normB : 0.0);
  }
  int best = 1;
  for (int r = 2; r <= n - 1; ++r)
    if (m[r] < m[best]) best = r;
  if (mvals)
    for (int r = 1; r <= n - 1; ++r) mvals[r - 1] = m[r];
  double out = m[best];
  *r_out = best;
  free(sa); free(sb); free(m);
  return out;
}

/* ||Ahat(r+1:n,1:r)||_F / ||A||_F  (+ B part) at a given split r (diagnostic only). */
static double e21_fro(int n, int r, const double *Ah, int ldah, double fA,
                      const double *Bh, int ldbh, double fB) {
  double sa = 0.0, sb = 0.0;
  for (int c = 0; c < r; ++c)
    for (int i = r; i < n; ++i) {
      sa += EL(Ah, i, c, ldah) * EL(Ah, i, c, ldah);
      if (Bh) sb += EL(Bh, i, c, ldbh) * EL(Bh, i, c, ldbh);
    }
  return sqrt(sa) / fA + (Bh ? sqrt(sb) / fB : 0.0);
}

static int all_finite(size_t cnt, const double *x) {
  for (size_t i = 0; i < cnt; ++i) if (!isfinite(x[i])) return 0;
  return 1;
}

/* Â = Q_L^T A Q_R (+ B̂) and the split; returns metric. */
static double similarity_and_select(int n, const double *A, int lda, const double *B, int ldb,
                                    const double *QR, int ldqr, const double *QLm, int ldql,
                                    double nA, double nB, double fA, double fB,
                                    double *Ah, double *Bh, int *r, double *mfro, int sym) {
  size_t nn = (size_t)n * n;
  double *T = (double *)malloc(sizeof(double) * nn);
  orc_gemm(0, 0, n, n, n, A, lda, QR, ldqr, T, n);        /* A Q_R */
  orc_gemm(1, 0, n, n, n, QLm, ldql, T, n, Ah, n);        /* Q_L^T (A Q_R) */
  if (sym)                                                 /* RSEP: (Ahat + Ahat^T)/2, Alg. 6 */
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < j; ++i) {
        double v = 0.5 * (EL(Ah, i, j, n) + EL(Ah, j, i, n));
        EL(Ah, i, j, n) = v;
        EL(Ah, j, i, n) = v;
      }
  if (B) {
    orc_gemm(0, 0, n, n, n, B, ldb, QR, ldqr, T, n);
    orc_gemm(1, 0, n, n, n, QLm, ldql, T, n, Bh, n);
  }
  double met = orc_split_select(n, Ah, n, nA, B ? Bh : NULL, n, nB, r, NULL);
  *mfro = e21_fro(n, *r, Ah, n, fA, B ? Bh : NULL, n, fB);
  free(T);
  return met;
}

/* ------------------------------------------------------------------------------------
 * The whole split step (RNEP Alg. 5 when B == NULL, RGNEP Alg. 4 otherwise).
 * Mirrors the product ABI sdc_split (include/sdc.h) with HOST pointers.
 * hist (optional, hist_cap passes x 3 doubles): per pass {r*, metric, R-test ratio};
 * r* and metric are NaN unless stop_mode == ORC_STOP_E21; the R-test ratio is
 * ||R_j - R_{j-1}||_1/||R_{j-1}||_1 (NaN at j = 0) of the right IRS.
 * ---------------------------------------------------------------------------------- */
/* Regions (the step is written for the unit disk; the others map to it):
 *   ORC_REGION_DISK, param rho > 0: |z| < rho  <=>  unit disk of the pencil (A, rho B)
 *     (radius-rho circles of the pencil strategy);
 *   ORC_REGION_HALFPLANE, param a: Re z < a for B = I, via the Moebius map
 *     f(z) = (z-a+1)/(z-a-1) that sends the line Re z = a to the unit circle:
 *     IRS on the pencil (A-(a-1)I, A-(a+1)I); right subspace only and the
 *     similarity Q^T A Q of the ORIGINAL A (single-matrix split, Alg. 5).
 * Flag ORC_FLAG_SYMMETRIC (B = I only): RSEP, Ahat <- (Ahat + Ahat^T)/2 before the
 * selection (Alg. 6). */
int orc_split(int n, const double *A, int lda, const double *B, int ldb,
              const double *V, int ldv, const double *VL, int ldvl,
              int max_iters, double tol, int stop_mode,
              double *Q, int ldq, double *QLout, int ldql, double *Ahat_out, int ldah,
              double *hist, int hist_cap, orc_result *res) {
  return orc_split_region(n, A, lda, B, ldb, V, ldv, VL, ldvl, ORC_REGION_UNIT_DISK, 1.0, 0,
                          max_iters, tol, stop_mode, Q, ldq, QLout, ldql, Ahat_out, ldah, hist,
                          hist_cap, res);
}

/* Cheaper left basis for pencils: the left deflating
 * subspace of the |lambda| > 1 part is A X for X = span Q_R(:, 1:r) (A is nonsingular on it:
 * A x = lambda B x with lambda != 0, infinite eigenvalues included), and QR preserves nested
 * column spans, so Q_L := Q of QR(A Q_R) (diag R >= 0) spans it for every r at once. */
static void ql_from_aq(int n, const double *A, int lda, const double *Q, int ldq, double *QL, int ldql) {
  double *W = (double *)malloc(sizeof(double) * (size_t)n * n), *tau = (double *)malloc(sizeof(double) * n);
  orc_gemm(0, 0, n, n, n, A, lda, Q, ldq, W, n);
  orc_geqr2(n, n, W, n, tau);
  orc_org2r_signed(n, W, n, tau, QL, ldql);
  free(W);
  free(tau);
}

int orc_split_region(int n, const double *A, int lda, const double *B, int ldb,
                     const double *V, int ldv, const double *VL, int ldvl,
                     int region, double param, int flags,
                     int max_iters, double tol, int stop_mode,
                     double *Q, int ldq, double *QLout, int ldql, double *Ahat_out, int ldah,
                     double *hist, int hist_cap, orc_result *res) {
  if (region < 0 || region > 2) return -30;
  if (region == ORC_REGION_DISK && !(param > 0.0)) return -31;
  if ((region == ORC_REGION_HALFPLANE || (flags & ORC_FLAG_SYMMETRIC)) && B) return -32;
  if (flags & ~(ORC_FLAG_SYMMETRIC | ORC_FLAG_PLATEAU | ORC_FLAG_ONESIDED | ORC_FLAG_QL_ORTH)) return -33;
  if ((flags & ORC_FLAG_QL_ORTH) && !B) return -34;
  const int ql_orth = (flags & ORC_FLAG_QL_ORTH) != 0;   /* no left IRS: Q_L from QR(A Q_R) */
  const int sym = (flags & ORC_FLAG_SYMMETRIC) != 0;
  const double rho = region == ORC_REGION_DISK ? param : 1.0;
  if (n < 2) return -1;
  if (lda < n) return -3;
  if (B && ldb < n) return -5;
  if (!V || ldv < n) return -6;
  if (B && !(flags & ORC_FLAG_QL_ORTH) && (!VL || ldvl < n)) return -8;
  if (max_iters < 1) return -10;
  if (!(tol >= 0.0)) return -11;
  if (stop_mode < 0 || stop_mode > 2) return -12;
  if (!Q || ldq < n) return -13;
  if (!res) return -20;
  const int pencil = (B != NULL);
  size_t nn = (size_t)n * n;
  double *Aj = (double *)malloc(sizeof(double) * nn), *Bj = (double *)malloc(sizeof(double) * nn);
  double *Lj = NULL, *Mj = NULL;     /* left IRS on (A^T, B^T) */
  double *Rp = (double *)malloc(sizeof(double) * nn), *Rc = (double *)malloc(sizeof(double) * nn);
  double *Ah = (double *)malloc(sizeof(double) * nn), *Bh = pencil ? (double *)malloc(sizeof(double) * nn) : NULL;
  double *QLw = pencil ? (double *)malloc(sizeof(double) * nn) : NULL;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      if (region == ORC_REGION_HALFPLANE) {           /* (A - (a-1) I, A - (a+1) I) */
        EL(Aj, i, j, n) = EL(A, i, j, lda) - (i == j ? param - 1.0 : 0.0);
        EL(Bj, i, j, n) = EL(A, i, j, lda) - (i == j ? param + 1.0 : 0.0);
      } else {                                         /* (A, rho B) */
        EL(Aj, i, j, n) = EL(A, i, j, lda);
        EL(Bj, i, j, n) = rho * (pencil ? EL(B, i, j, ldb) : (i == j ? 1.0 : 0.0));
      }
    }
  if (pencil) {
    Lj = (double *)malloc(sizeof(double) * nn); Mj = (double *)malloc(sizeof(double) * nn);
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) { EL(Lj, i, j, n) = EL(A, j, i, lda); EL(Mj, i, j, n) = rho * EL(B, j, i, ldb); }
  }
  double nA = orc_norm1(n, n, A, lda), fA = norm_fro(n, n, A, lda);
  double nB = pencil ? orc_norm1(n, n, B, ldb) : 1.0, fB = pencil ? norm_fro(n, n, B, ldb) : 1.0;
  for (int i = 0; i < hist_cap * 3 && hist; ++i) hist[i] = NAN;

  int p = max_iters, conv = 0, r = 1;
  double met = INFINITY, mfro = INFINITY, prev = INFINITY;
  int have_split = 0;
  for (int j = 0; j < max_iters; ++j) {
    orc_irs_pass(n, Aj, n, Bj, n, Aj, n, Bj, n, Rc);
    if (pencil && !ql_orth) orc_irs_pass(n, Lj, n, Mj, n, Lj, n, Mj, n, NULL);
    if ((flags & ORC_FLAG_ONESIDED) && stop_mode == ORC_STOP_E21 && j >= 2) {
      /* every eigenvalue on one side: (A^{-1}B)^{2^p} -> 0 or infinity, one of A_p, B_p
       * vanishes relative to the other -- no split exists, stop */
      const double fa = norm_fro(n, n, Aj, n), fb = norm_fro(n, n, Bj, n);
      const double sd = fa + fb > 0.0 ? fb / (fa + fb) : 0.5;
      if (sd < 1e-6 || sd > 1.0 - 1e-6) { p = j + 1; break; }
    }
    double ratio = NAN;
    if (j >= 1) {
      double *D = (double *)malloc(sizeof(double) * nn);
      for (size_t t = 0; t < nn; ++t) D[t] = Rc[t] - Rp[t];
      ratio = orc_norm1(n, n, D, n) / orc_norm1(n, n, Rp, n);
      free(D);
    }
    memcpy(Rp, Rc, sizeof(double) * nn);
    if (hist && j < hist_cap) hist[3 * j + 2] = ratio;
    if (stop_mode == ORC_STOP_RTEST && j >= 1 && ratio <= tol) { p = j + 1; conv = 1; break; }
    if (stop_mode == ORC_STOP_E21) {
      orc_grurv_right(n, Aj, n, Bj, n, V, ldv, Q, ldq, NULL, NULL);
      const double *QLm = Q; int ldqlm = ldq;
      if (pencil) {
        if (ql_orth) ql_from_aq(n, A, lda, Q, ldq, QLw, n);
        else orc_grurv_left(n, Lj, n, Mj, n, VL, ldvl, QLw, n);
        QLm = QLw; ldqlm = n;
      }
      met = similarity_and_select(n, A, lda, B, ldb, Q, ldq, QLm, ldqlm, nA, nB, fA, fB,
                                  Ah, Bh, &r, &mfro, sym);
      have_split = 1;
      if (hist && j < hist_cap) { hist[3 * j] = r; hist[3 * j + 1] = met; }
      if (met <= tol) { p = j + 1; conv = 1; break; }
      /* plateau: a metric within 10 tol that no longer halves -- the rounding floor */
      if ((flags & ORC_FLAG_PLATEAU) && met <= 10.0 * tol && met > 0.5 * prev) {
        p = j + 1; conv = 1; break;
      }
      prev = met;
    }
  }
  if (!have_split) {
    orc_grurv_right(n, Aj, n, Bj, n, V, ldv, Q, ldq, NULL, NULL);
    const double *QLm = Q; int ldqlm = ldq;
    if (pencil) {
      if (ql_orth) ql_from_aq(n, A, lda, Q, ldq, QLw, n);
      else orc_grurv_left(n, Lj, n, Mj, n, VL, ldvl, QLw, n);
      QLm = QLw; ldqlm = n;
    }
    met = similarity_and_select(n, A, lda, B, ldb, Q, ldq, QLm, ldqlm, nA, nB, fA, fB,
                                Ah, Bh, &r, &mfro, sym);
  }
  if (pencil && QLout)
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) EL(QLout, i, j, ldql) = EL(QLw, i, j, n);
  if (Ahat_out)
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) EL(Ahat_out, i, j, ldah) = EL(Ah, i, j, n);
  res->r = r;
  res->k = n - r;
  res->metric = met;
  res->metric_fro = mfro;
  res->iters = p;
  res->converged = conv;
  {   /* side indicator of the final right IRS pair: ||B_p||_F / (||A_p||_F + ||B_p||_F) */
    const double fa = norm_fro(n, n, Aj, n), fb = norm_fro(n, n, Bj, n);
    res->side = fa + fb > 0.0 ? fb / (fa + fb) : 0.5;
  }
  res->status = !all_finite(nn, Ah) || !isfinite(met) ? ORC_STATUS_NONFINITE
              : (met <= ORC_SPLIT_ACCEPT ? ORC_STATUS_SPLIT : ORC_STATUS_NO_SPLIT);
  free(Aj); free(Bj); free(Rp); free(Rc); free(Ah);
  if (pencil) { free(Lj); free(Mj); free(Bh); free(QLw); }
  return 0;
}

/* Singular-value split: "construct the hermitian matrix
 * B = [[0, A], [A^H, 0]] and compute its eigenvalues (which are the singular values of A
 * and their negatives)".  The m x n matrix A is embedded into the (m+n) x (m+n) symmetric
 * H = [[0, A], [A^T, 0]] and one RSEP step (Alg. 6: IRS(H, I), GRURV,
 * Ahat = Q^T H Q, Ahat := (Ahat + Ahat^T)/2, split selection) splits it along |z| = rho.
 * k = #{|eig(H)| < rho} = 2 #{sigma_i < rho} + |m - n|. */
int orc_svd_split(int m, int n, const double *A, int lda, double rho,
                  const double *V, int ldv, int max_iters, double tol, int stop_mode,
                  double *Q, int ldq, double *Ahat_out, int ldah,
                  double *hist, int hist_cap, orc_result *res) {
  if (m < 1 || n < 1) return -1;
  if (lda < m) return -4;
  const int N = m + n;
  double *H = (double *)calloc((size_t)N * N, sizeof(double));
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < m; ++i) {
      EL(H, i, m + j, N) = EL(A, i, j, lda);      /* H(0:m, m:m+n) = A   */
      EL(H, m + j, i, N) = EL(A, i, j, lda);      /* H(m:m+n, 0:m) = A^T */
    }
  int rc = orc_split_region(N, H, N, NULL, 0, V, ldv, NULL, 0, ORC_REGION_DISK, rho,
                            ORC_FLAG_SYMMETRIC, max_iters, tol, stop_mode, Q, ldq, NULL, 0,
                            Ahat_out, ldah, hist, hist_cap, res);
  free(H);
  return rc;
}

/* TREVC (eq. (trevc)): eigenvectors of an upper triangular T,
 * TX = XD with D = diag(T), X upper triangular with X_jj = 1 ("X_jj can be
 * arbitrarily chosen"), for i < j:
 *   X_ij = (T_ij X_jj + sum_{k=i+1}^{j-1} T_ik X_kj) / (T_jj - T_ii)
 * evaluated exactly in that order.  Near-equal eigenvalues (reading Q19, the
 * LAPACK dtrevc/dlaln2 rule): if |T_ii - T_jj| < smin = max(ulp |T_jj|, smlnum) the
 * denominator T_ii - T_jj is replaced by smin, i.e. X_ij = -(numerator) / smin, with
 * ulp = 2^-52 and smlnum = DBL_MIN n / ulp.  If Q != NULL the eigenvectors of
 * A = Q T Q^T are returned instead: X := Q X. */
/* columns j0 <= j < j1 of X (column j depends on T(0:j, 0:j) only); X is n x n, the other
 * columns are not touched */
void orc_trevc_cols(int n, const double *T, int ldt, int j0, int j1, double *Xt, int ldx) {
  const double ulp = 2.220446049250313e-16, smlnum = 2.2250738585072014e-308 * (double)n / ulp;
#pragma omp parallel for schedule(static) if ((long)n * (j1 - j0) >= ORC_PAR_MIN)
  for (int j = j0; j < j1; ++j) {
    for (int i = j + 1; i < n; ++i) EL(Xt, i, j, ldx) = 0.0;
    const double d = EL(T, j, j, ldt);
    const double smin = fmax(ulp * fabs(d), smlnum);
    EL(Xt, j, j, ldx) = 1.0;
    for (int i = j - 1; i >= 0; --i) {
      double num = EL(T, i, j, ldt) * EL(Xt, j, j, ldx);
      for (int k = i + 1; k <= j - 1; ++k) num += EL(T, i, k, ldt) * EL(Xt, k, j, ldx);
      double den = EL(T, i, i, ldt) - d;               /* (T_ii - T_jj) x = -num */
      if (fabs(den) < smin) den = smin;
      EL(Xt, i, j, ldx) = -num / den;
    }
  }
}

void orc_trevc(int n, const double *T, int ldt, const double *Q, int ldq, double *X, int ldx) {
  double *Xt = (double *)calloc((size_t)n * n, sizeof(double));
  orc_trevc_cols(n, T, ldt, 0, n, Xt, n);
  if (Q) {
    orc_gemm(0, 0, n, n, n, Q, ldq, Xt, n, X, ldx);
  } else {
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) EL(X, i, j, ldx) = EL(Xt, i, j, n);
  }
  free(Xt);
}

/* ---------------------------------------------------------------------------------------
 * Recursive divide-and-conquer ("zero out E21 and
 * recurse on A11, A22", random splitting lines PAPER.md:472-475, 545).  Real arithmetic:
 * the lines are vertical, Re z = a (theta in {0, pi}), mapped to the unit circle through
 * the Moebius pencil (A - (a-1)I, A - (a+1)I) (orc_split_region HALFPLANE).  The
 * decisions follow DESIGN.md §10 "recursion" exactly, shared with sdc_schur:
 *   - block (o, m) with m <= leaf, or m == 2 with complex eigenvalues: a leaf;
 *   - search interval for the line: c = trace/m, s = ||T_blk - c I||_F / sqrt(m) (both
 *     invariant under orthogonal similarity, so rounding-level basis differences do not
 *     change decisions), [lo, hi] = [c - 2s, c + 2s] (PAPER.md:472-475 uses a disk of radius
 *     R/2 around the centre; Gershgorin radii of dense blocks are ~sqrt(m) too wide); s = 0:
 *     unsplittable leaf;
 *   - attempt t (t < 16): a = lo + (0.25 + 0.5 u)(hi - lo), u = U01(seed, 2 c), V = Haar of
 *     order m from the Gaussian stream 2 c + 1, c = orc_attempt_ctr(global offset, m, t)
 *     (keyed by the block, so any processing order draws the same numbers); RNEP step in
 *     monitor mode (stop at the first pass with ||E21||_1/||A||_1 <= tol_b = max(tol, 8e-15 m),
 *     PAPER.md:597, or at a plateau <= 10 tol_b that no longer halves, or once the IRS pair
 *     is one-sided) with at most max_iters passes; accepted iff status 0 (<= 1e-8, Q4) and
 *     the pair is not one-sided (res.side within 1e-6 of 0 or 1); a
 *     rejected step whose IRS pair shows every eigenvalue on one side of the line
 *     (res.side > 0.95: all Re < a; < 0.05: all Re > a) moves hi (lo) to a -- the paper's
 *     "progress without a split" -- otherwise the line hit
 *     the pseudospectrum and the next attempt draws a new a in the same interval;
 *   - accepted: T(o:o+m, o:o+m) = Ahat with E21 := 0, T(o:o+m, o+m:n) = Qb^T T(...),
 *     T(0:o, o:o+m) = T(...) Qb, Q(:, o:o+m) = Q(...) Qb; children (o, r) then (o+r, m-r)
 *     (processed depth first, leading block first);
 *   - 16 failed attempts: an unsplit leaf.
 * Counter-based generator (splitmix64) so both sides draw the same numbers. */
static uint64_t orc_mix64(uint64_t seed, uint64_t ctr) {
  uint64_t z = seed + 0x9E3779B97F4A7C15ull * (ctr + 1ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static double orc_u01(uint64_t seed, uint64_t ctr) {
  return (double)(orc_mix64(seed, ctr) >> 11) * 1.1102230246251565e-16;   /* [0, 1) */
}
/* Gaussian (Box-Muller) entry (i, j) of the order-m matrix of stream `key` */
static double orc_gauss(uint64_t seed, uint64_t key, int m, int i, int j) {
  const uint64_t base = (key << 40) + 2ull * ((uint64_t)i + (uint64_t)j * (uint64_t)m);
  const double u1 = (double)((orc_mix64(seed, base) >> 11) + 1ull) * 1.1102230246251565e-16;  /* (0,1] */
  const double u2 = orc_u01(seed, base + 1ull);
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

void orc_haar(int m, unsigned long long seed, unsigned long long key, double *V, int ldv) {
  double *G = (double *)malloc(sizeof(double) * (size_t)m * m), *tau = (double *)malloc(sizeof(double) * m);
  for (int j = 0; j < m; ++j)
    for (int i = 0; i < m; ++i) EL(G, i, j, m) = orc_gauss(seed, key, m, i, j);
  orc_geqr2(m, m, G, m, tau);
  orc_org2r_signed(m, G, m, tau, V, ldv);
  free(G);
  free(tau);
}

/* Counter of attempt t (< 16) on the diagonal block at GLOBAL offset o of order m: keyed by
 * the block's identity (not by a running counter), so the draws -- and hence every decision
 * -- do not depend on the order in which blocks are processed: depth first on one rank, or
 * subproblems handed to other ranks.  23 bits, so the Gaussian stream key
 * 2 ctr + 1 shifted left by 40 stays inside 64 bits. */
static uint64_t orc_attempt_ctr(int o, int m, int t) {
  const uint64_t id = (uint64_t)o * 65537ull + (uint64_t)m;
  return ((orc_mix64(0x5DC0FFEEull, id) & 0x7FFFFull) << 4) | (uint64_t)t;
}

/* One node of the recursion: the attempt loop on the diagonal block Tb (m x m, ld ldtb) at
 * global offset o.  Accepted: Tb <- Ahat with E21 := 0, Qb <- the block's orthogonal factor
 * (m x m, ld ldqb), returns r in [1, m-1].  Returns 0 for a leaf (m <= leaf or a 2x2 with
 * complex eigenvalues) or an unsplit block (s = 0, or 16 failed attempts: stats[2]++); Tb is
 * then unchanged.  stats (splits, failed attempts, unsplit, passes) and max_metric accumulate. */
int orc_schur_node(int m, double *Tb, int ldtb, int o, int leaf, unsigned long long seed, int max_iters,
                   double tol, double *Qb, int ldqb, int *stats, double *max_metric) {
  if (m < 1 || ldtb < m || ldqb < m || leaf < 1) return -1;
  if (m <= leaf) return 0;
  if (m == 2) {   /* 2x2 with complex eigenvalues: a standardised leaf */
    const double a = EL(Tb, 0, 0, ldtb), b = EL(Tb, 0, 1, ldtb), c = EL(Tb, 1, 0, ldtb), d = EL(Tb, 1, 1, ldtb);
    if ((a - d) * (a - d) + 4.0 * b * c < 0.0) return 0;
  }
  double tr = 0.0;
  for (int i = 0; i < m; ++i) tr += EL(Tb, i, i, ldtb);
  const double c = tr / m;
  double f2 = 0.0;
  for (int j = 0; j < m; ++j)
    for (int i = 0; i < m; ++i) {
      const double t = EL(Tb, i, j, ldtb) - (i == j ? c : 0.0);
      f2 += t * t;
    }
  const double sd = sqrt(f2 / m);
  double lo = c - 2.0 * sd, hi = c + 2.0 * sd;
  if (!(sd > 0.0)) { stats[2]++; return 0; }
  const size_t mm = (size_t)m * m;
  double *Tw = (double *)malloc(sizeof(double) * mm), *V = (double *)malloc(sizeof(double) * mm);
  double *Ab = (double *)malloc(sizeof(double) * mm), *Qw = (double *)malloc(sizeof(double) * mm);
  int r = 0;
  for (int att = 0; att < 16; ++att) {
    const uint64_t ctr = orc_attempt_ctr(o, m, att);
    const double u = orc_u01(seed, 2ull * ctr);
    const double a = lo + (0.25 + 0.5 * u) * (hi - lo);
    orc_haar(m, seed, 2ull * ctr + 1ull, V, m);
    for (int j = 0; j < m; ++j)
      for (int i = 0; i < m; ++i) EL(Tw, i, j, m) = EL(Tb, i, j, ldtb);
    orc_result res;
    const double tolb = fmax(tol, 8e-15 * m);   /* rounding floor grows ~ m eps */
    int rc = orc_split_region(m, Tw, m, NULL, 0, V, m, NULL, 0, ORC_REGION_HALFPLANE, a,
                              ORC_FLAG_PLATEAU | ORC_FLAG_ONESIDED, max_iters, tolb, ORC_STOP_E21,
                              Qw, m, NULL, 0, Ab, m, NULL, 0, &res);
    if (rc) { r = rc; break; }
    stats[3] += res.iters;
    /* accept only clearly two-sided pairs: side within 1e-3 of 0 or 1 means (nearly) every
     * eigenvalue lies on one side, and whether the iteration stopped on the E21 rule just
     * before or on the one-sided rule just after is a rounding race (reading Q20) */
    const int onesided = res.side < 1e-3 || res.side > 1.0 - 1e-3;
    if (getenv("ORC_SCHUR_TRACE"))   /* decision trace (debugging the recursion's margins) */
      fprintf(stderr, "node o=%d m=%d att=%d a=%.6f iters=%d conv=%d status=%d r=%d metric=%.3e side=%.3e\n", o, m,
              att, a, res.iters, res.converged, res.status, res.r, res.metric, res.side);
    if (res.status != ORC_STATUS_SPLIT || onesided) {   /* a one-sided pair's split is incidental */
      stats[1]++;
      if (res.side > 0.95) hi = a;          /* every eigenvalue left of the line  */
      else if (res.side < 0.05) lo = a;     /* every eigenvalue right of the line */
      continue;
    }
    r = res.r;
    stats[0]++;
    *max_metric = fmax(*max_metric, res.metric);
    for (int j = 0; j < m; ++j)   /* Tb = Ahat with E21 = 0 */
      for (int i = 0; i < m; ++i) {
        EL(Tb, i, j, ldtb) = (i >= r && j < r) ? 0.0 : EL(Ab, i, j, m);
        EL(Qb, i, j, ldqb) = EL(Qw, i, j, m);
      }
    break;
  }
  if (r == 0) stats[2]++;   /* 16 failed attempts: an unsplit leaf */
  free(Tw); free(V); free(Ab); free(Qw);
  return r;
}

int orc_schur_keyed(int n, const double *A, int lda, int key_off, int leaf, unsigned long long seed,
                    int max_iters, double tol, double *Q, int ldq, double *T, int ldt, int *blk_off,
                    int *blk_size, int *nblk, int *stats, double *max_metric) {
  if (n < 1 || lda < n || ldq < n || ldt < n || leaf < 1 || key_off < 0) return -1;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      EL(T, i, j, ldt) = EL(A, i, j, lda);
      EL(Q, i, j, ldq) = i == j ? 1.0 : 0.0;
    }
  for (int q = 0; q < 4; ++q) stats[q] = 0;   /* splits, failed attempts, unsplit leaves, passes */
  *max_metric = 0.0;                           /* largest accepted ||E21||_1/||A_blk||_1 */
  int *st_o = (int *)malloc(sizeof(int) * 2 * n), *st_m = (int *)malloc(sizeof(int) * 2 * n);
  int sp = 0, nb = 0, rc = 0;
  st_o[sp] = 0; st_m[sp] = n; ++sp;
  double *Qb = (double *)malloc(sizeof(double) * (size_t)n * n);
  double *W = (double *)malloc(sizeof(double) * (size_t)n * n);
  while (sp > 0) {
    --sp;
    const int o = st_o[sp], m = st_m[sp];
    const int r = orc_schur_node(m, &EL(T, o, o, ldt), ldt, key_off + o, leaf, seed, max_iters, tol, Qb, m,
                                 stats, max_metric);
    if (r < 0) { rc = r; break; }
    if (r == 0) { blk_off[nb] = o; blk_size[nb] = m; ++nb; continue; }
    /* T(o:o+m, o+m:n) = Qb^T T(o:o+m, o+m:n) */
    const int nr = n - o - m;
    if (nr > 0) {
      orc_gemm(1, 0, m, nr, m, Qb, m, &EL(T, o, o + m, ldt), ldt, W, m);
      for (int j = 0; j < nr; ++j)
        for (int i = 0; i < m; ++i) EL(T, o + i, o + m + j, ldt) = EL(W, i, j, m);
    }
    /* T(0:o, o:o+m) = T(0:o, o:o+m) Qb */
    if (o > 0) {
      orc_gemm(0, 0, o, m, m, &EL(T, 0, o, ldt), ldt, Qb, m, W, o);
      for (int j = 0; j < m; ++j)
        for (int i = 0; i < o; ++i) EL(T, i, o + j, ldt) = EL(W, i, j, o);
    }
    /* Q(:, o:o+m) = Q(:, o:o+m) Qb */
    orc_gemm(0, 0, n, m, m, &EL(Q, 0, o, ldq), ldq, Qb, m, W, n);
    for (int j = 0; j < m; ++j)
      for (int i = 0; i < n; ++i) EL(Q, i, o + j, ldq) = EL(W, i, j, n);
    st_o[sp] = o + r; st_m[sp] = m - r; ++sp;   /* trailing (Re < a), processed second */
    st_o[sp] = o; st_m[sp] = r; ++sp;           /* leading (Re > a), processed first   */
  }
  *nblk = nb;
  free(st_o); free(st_m); free(Qb); free(W);
  return rc;
}

int orc_schur(int n, const double *A, int lda, int leaf, unsigned long long seed, int max_iters, double tol,
              double *Q, int ldq, double *T, int ldt, int *blk_off, int *blk_size, int *nblk,
              int *stats, double *max_metric) {
  return orc_schur_keyed(n, A, lda, 0, leaf, seed, max_iters, tol, Q, ldq, T, ldt, blk_off, blk_size, nblk,
                         stats, max_metric);
}
