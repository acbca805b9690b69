/*
 * sdc_oracle.h -- declarations of the CPU fp64 ORACLE (test infrastructure only).
 * Independent of include/sdc.h: the oracle keeps its own constants and result struct.
 * All matrices are host memory, column-major, fp64.  See sdc_oracle.c for citations.
 */
#ifndef SDC_ORACLE_H
#define SDC_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_STOP_FIXED = 0, ORC_STOP_RTEST = 1, ORC_STOP_E21 = 2 };
enum { ORC_REGION_UNIT_DISK = 0, ORC_REGION_DISK = 1, ORC_REGION_HALFPLANE = 2 };
enum { ORC_FLAG_SYMMETRIC = 1,
       ORC_FLAG_PLATEAU = 2,   /* E21 mode: also stop at a metric <= 10 tol that stopped halving */
       ORC_FLAG_ONESIDED = 4,  /* E21 mode: stop after pass >= 3 once ||B_p||/(||A_p||+||B_p||) is
                                  within 1e-6 of 0 or 1 (every eigenvalue on one side)       */
       ORC_FLAG_QL_ORTH = 8    /* pencils: no left IRS; Q_L = Q of QR(A Q_R), diag R >= 0    */ };
enum { ORC_STATUS_SPLIT = 0, ORC_STATUS_NO_SPLIT = 1, ORC_STATUS_NONFINITE = 2 };
#define ORC_SPLIT_ACCEPT 1e-8 /* split_accept_tol (SPEC.md design decision; Q4) */

typedef struct {
  int k;             /* n - r: eigenvalues strictly inside the unit circle   */
  int r;             /* order of the leading (|lambda| > 1) block            */
  double metric;     /* ||E21||_1/||A||_1 (+ ||F21||_1/||B||_1)              */
  double metric_fro; /* ||E21||_F/||A||_F (+ F21) at the same r              */
  int iters;         /* IRS passes executed                                   */
  int converged;     /* 1 if the stop rule fired before max_iters             */
  int status;        /* ORC_STATUS_*                                          */
  double side;       /* ||B_p||_F/(||A_p||_F+||B_p||_F) of the final right IRS pair: -> 0
                        when every eigenvalue of the (mapped) pencil is outside the unit
                        circle, -> 1 when every one is inside (A_p^{-1}B_p = (A^{-1}B)^{2^p},
                        PAPER.md:460); the recursion's one-sided test */
} orc_result;

void orc_geqr2(int m, int n, double *A, int lda, double *tau);
void orc_apply_qt(int m, int n, const double *Y, int ldy, const double *tau,
                  int nc, double *C, int ldc);
void orc_org2r_signed(int n, const double *Y, int ldy, const double *tau, double *Q, int ldq);
void orc_complement(int n, const double *Y, int ldy, const double *tau, double *C, int ldc);
void orc_gerq2(int n, double *A, int lda, double *tau);
void orc_orgr2_signed(int n, const double *Y, int ldy, const double *tau, double *Q, int ldq);
void orc_geql2(int n, double *A, int lda, double *tau);
void orc_org2l_signed(int n, const double *Y, int ldy, const double *tau, double *Q, int ldq);
void orc_gemm(int ta, int tb, int m, int n, int K, const double *A, int lda,
              const double *B, int ldb, double *C, int ldc);
double orc_norm1(int m, int n, const double *X, int ldx);
void orc_irs_pass(int n, const double *Aj, int lda, const double *Bj, int ldb,
                  double *Aout, int ldao, double *Bout, int ldbo, double *Rout);
void orc_grurv_right(int n, const double *Ap, int ldap, const double *Bp, int ldbp,
                     const double *V, int ldv, double *Q, int ldq, double *R1, double *R2);
void orc_grurv_left(int n, const double *Ap, int ldap, const double *Bp, int ldbp,
                    const double *VL, int ldv, double *QL, int ldq);
double orc_split_select(int n, const double *Ah, int ldah, double normA,
                        const double *Bh, int ldbh, double normB, int *r_out, double *mvals);
int orc_split(int n, const double *A, int lda, const double *B, int ldb,
              const double *V, int ldv, const double *VL, int ldvl,
              int max_iters, double tol, int stop_mode,
              double *Q, int ldq, double *QLout, int ldql, double *Ahat_out, int ldah,
              double *hist, int hist_cap, orc_result *res);

int orc_split_region(int n, const double *A, int lda, const double *B, int ldb,
                     const double *V, int ldv, const double *VL, int ldvl,
                     int region, double param, int flags,
                     int max_iters, double tol, int stop_mode,
                     double *Q, int ldq, double *QLout, int ldql, double *Ahat_out, int ldah,
                     double *hist, int hist_cap, orc_result *res);

/* singular values below rho: RSEP step on [[0, A], [A^T, 0]] */
int orc_svd_split(int m, int n, const double *A, int lda, double rho,
                  const double *V, int ldv, int max_iters, double tol, int stop_mode,
                  double *Q, int ldq, double *Ahat_out, int ldah,
                  double *hist, int hist_cap, orc_result *res);

/* eigenvectors of an upper triangular T (TREVC); X := Q X if Q != NULL */
void orc_trevc(int n, const double *T, int ldt, const double *Q, int ldq, double *X, int ldx);
/* columns j0..j1-1 only (column j depends on T(0:j, 0:j)); the sampled full-size check */
void orc_trevc_cols(int n, const double *T, int ldt, int j0, int j1, double *X, int ldx);

/* Haar orthogonal V of order m from the counter-based Gaussian stream `key` (QR, diag R >= 0) */
void orc_haar(int m, unsigned long long seed, unsigned long long key, double *V, int ldv);
/* recursive divide-and-conquer to block upper triangular form A = Q T Q^T */
int orc_schur(int n, const double *A, int lda, int leaf, unsigned long long seed, int max_iters,
              double tol, double *Q, int ldq, double *T, int ldt, int *blk_off, int *blk_size,
              int *nblk, int *stats, double *max_metric);
/* the same with the random draws keyed by GLOBAL block offsets key_off + o (a subproblem of
 * a larger recursion, e.g. handed to another rank: PAPER.md:989-991) */
int orc_schur_keyed(int n, const double *A, int lda, int key_off, int leaf, unsigned long long seed,
                    int max_iters, double tol, double *Q, int ldq, double *T, int ldt, int *blk_off,
                    int *blk_size, int *nblk, int *stats, double *max_metric);
/* one node: the attempt loop on the diagonal block Tb at global offset o; returns r > 0
 * (Tb <- Ahat with E21 = 0, Qb <- the block's orthogonal factor), 0 (leaf / unsplit), < 0 error */
int orc_schur_node(int m, double *Tb, int ldtb, int o, int leaf, unsigned long long seed, int max_iters,
                   double tol, double *Qb, int ldqb, int *stats, double *max_metric);

#ifdef __cplusplus
}
#endif
#endif
