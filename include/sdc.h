/*
 * sdc.h -- C ABI of libsdc.so: one inverse-free split step of randomized spectral
 * divide-and-conquer (arXiv 1011.3077, Ballard-Demmel-Dumitriu) on one B200 (sm_100a).
 *
 * The step (PAPER.md:335-354 problem statement; Alg. 3/4/5 at PAPER.md:358-423):
 *   1. IRS (Alg. 3): for j = 0..p-1:  [B_j; -A_j] = Q [R_j; 0],
 *                    A_{j+1} = Q12^T A_j,  B_{j+1} = Q22^T B_j
 *   2. Q = GRURV(2, A_p+B_p, A_p; -1, +1)  with the caller's Haar V
 *      (and, for a pencil, Q_L = GRURV(2, A'_p^T, (A'_p+B'_p)^T; +1,-1) on IRS(A^T,B^T),
 *       PAPER.md:387-388)
 *   3. Ahat = Q_L^T A Q  (Q_L = Q when B = I)
 *   4. r = argmin_{1<=r<=n-1} ||Ahat(r+1:n,1:r)||_1/||A||_1 (+ ||Bhat21||_1/||B||_1),
 *      ties -> smallest r
 *
 * Polarity (reading Q1): (A_p+B_p)^{-1}A_p -> projector onto the |lambda| > 1
 * right deflating subspace, so Q(:,1:r) spans the OUTSIDE subspace,
 * Ahat(1:r,1:r) holds the eigenvalues with |lambda| > 1, and k = n - r is the number of
 * eigenvalues strictly inside the unit circle (the north_star's split index).
 *
 * Conventions for every function below:
 *   - matrices: IEEE fp64, column-major, element (i,j) at ptr[i + j*ld], ld >= rows;
 *   - device pointers live on the handle's device and are caller-owned; inputs are
 *     never modified; outputs must not alias inputs or each other;
 *   - all GPU work is enqueued on `stream` (a cudaStream_t, NULL = legacy default);
 *     functions returning host results synchronise that stream before returning;
 *   - return value 0 = success; -i = argument i invalid (LAPACK style, 1-based position);
 *     SDC_ERR_CUDA (-100) = CUDA error, SDC_ERR_NOMEM (-101) = out of memory,
 *     SDC_ERR_NOT_SUPPORTED (-102); text of the last error via sdc_last_error();
 *   - numerical outcomes (no split, non-finite) are NOT errors: see sdc_result.status;
 *   - no CPU fallback: without a usable sm_100 device every call fails with -100/-102.
 *   - a handle is not re-entrant: use one handle per concurrent stream.  Handles on
 *     different streams may run concurrently; their results are bit-identical to serial
 *     runs (tests/test_gpu_concurrency.py);
 *   - inside a call the handle may fork work from `stream` onto its own streams: a
 *     high-priority stream for the look-ahead QR chain, and a second factorization
 *     context for the pencil's left chain or monitor-mode GRURV.  Every fork is joined back
 *     into `stream` by events before the call's last operation on `stream`, so stream
 *     ordering for the caller is unchanged.  A fixed-mode step with n <= 4096 is
 *     additionally replayed as one CUDA graph whose edges carry these forks and joins.
 */
#ifndef SDC_H
#define SDC_H

#ifdef __cplusplus
extern "C" {
#endif

#define SDC_ERR_CUDA (-100)
#define SDC_ERR_NOMEM (-101)
#define SDC_ERR_NOT_SUPPORTED (-102)

/* stop rules of the IRS loop */
enum {
  SDC_STOP_FIXED = 0, /* exactly max_iters passes                                          */
  SDC_STOP_RTEST = 1, /* Alg. 3 line 4: stop after pass j >= 1 when
                         ||R_j - R_{j-1}||_1 <= tol ||R_{j-1}||_1; p = j+1    */
  SDC_STOP_E21 = 2    /* PAPER.md:597 protocol: full split after every pass, stop at the
                         first pass whose metric <= tol (one host sync per pass)            */
};
/* split regions: the step itself splits along the unit circle; the others
 * are mapped to it before the IRS (see sdc_split_region) */
enum {
  SDC_REGION_UNIT_DISK = 0, /* |z| < 1                                                       */
  SDC_REGION_DISK = 1,      /* |z| < rho (param rho > 0): unit disk of the pencil (A, rho B),
                               the radius-rho circles of the pencil strategy */
  SDC_REGION_HALFPLANE = 2  /* Re z < a (param a), B = I only: the line Re z = a mapped to the
                               unit circle by f(z) = (z-a+1)/(z-a-1), i.e. the IRS runs on the
                               pencil (A-(a-1)I, A-(a+1)I); Q^T A Q of the
                               original A, single right subspace                             */
};
enum { SDC_FLAG_SYMMETRIC = 1, /* RSEP, Alg. 6: Ahat <- (Ahat + Ahat^T)/2
                                  before the split selection; B = I only                     */
       SDC_FLAG_PLATEAU = 2,   /* SDC_STOP_E21 only: also stop once the metric is <= 10 tol and
                                  no longer halves (the rounding floor)       */
       SDC_FLAG_ONESIDED = 4,  /* SDC_STOP_E21 only: stop after pass >= 3 once res.side is within
                                  1e-6 of 0 or 1 (no eigenvalue on one side of the boundary) */
       SDC_FLAG_QL_ORTH = 8    /* pencils: no left IRS / left GRURV; Q_L = Q of
                                  QR(A Q_R), diag R >= 0 (same left deflating subspace as Alg. 4,
                                  Q_L^T A Q_R upper triangular, the split chosen by F21); VL may
                                  be NULL.  Halves the pencil step            */ };
enum { SDC_STATUS_SPLIT = 0, SDC_STATUS_NO_SPLIT = 1, SDC_STATUS_NONFINITE = 2 };
#define SDC_SPLIT_ACCEPT 1e-8 /* status 0 iff metric <= this (reading Q4)       */

typedef struct {
  int k;             /* n - r: eigenvalues strictly inside the unit circle                  */
  int r;             /* order of the leading block (|lambda| > 1), 1 <= r <= n-1            */
  double metric;     /* ||E21||_1/||A||_1 (+ ||F21||_1/||B||_1) at r                        */
  double metric_fro; /* ||E21||_F/||A||_F (+ F21 term) at r (diagnostic)                    */
  int iters;         /* IRS passes executed (p)                                            */
  int converged;     /* 1 if the RTEST/E21 stop rule fired before max_iters                 */
  int status;        /* SDC_STATUS_*                                                       */
  double side;       /* ||B_p||_F / (||A_p||_F + ||B_p||_F) of the final right IRS pair:
                        -> 0 when every eigenvalue is outside the region, -> 1 when every one
                        is inside (A_p^{-1} B_p = (A^{-1} B)^{2^p}); used by
                        sdc_schur to move its line after a one-sided step */
} sdc_result;

typedef struct sdc_handle sdc_handle;

/* Create a handle on CUDA device `device` with workspace for matrices up to n_max
 * (pencil != 0 also reserves the RGNEP buffers).  Workspace: 19 n_max^2 doubles (stack,
 * Y, Y^T, complement: 2 n^2 each; V^T, A_j x2, B_j x2, G1-G3, T1, Ahat, R_{j-1}: n^2 each)
 * + ~ n_max^2/32 (selection partials) + ~ 20 M doubles (split-K partials of both streams)
 * for RNEP; pencil handles add 9 n_max^2 (left stack, A'_j/B'_j x2, Bhat, Q_L, V_L^T).
 * The second factorization context (allocated on the first monitor-mode or pencil call)
 * adds 9 n_max^2 (Y, Y^T, complement, G1-G3) + ~ 10 M doubles; handles with 2 n_max > 4096
 * add 0.8 M doubles for the split CholeskyQR2 panel chain.  At n_max = 16384: 41 GB
 * (RNEP), 60 GB with the second context.  The caller's current device is restored on
 * return (as by every entry point below).  Supported: 2 <= n_max <= 24576.  Returns 0 or <0. */
int sdc_create(sdc_handle** h, int device, int n_max, int pencil);
void sdc_destroy(sdc_handle* h);

/* The split step (RNEP, Alg. 5, when B == NULL; RGNEP, Alg. 4, otherwise).
 *  1 h          handle
 *  2 stream     cudaStream_t to enqueue on
 *  3 n          order, 2 <= n <= n_max   (n < 2 is an error)
 *  4 A, 5 lda   input A (device)
 *  6 B, 7 ldb   input B (device) or NULL for B = I
 *  8 V, 9 ldv   Haar V for Q_R (Alg. 1 lines 1-2 are done by the caller; X = A_p V^T)
 * 10 VL,11 ldvl Haar V for Q_L; required iff B != NULL (ignored otherwise)
 * 12 region     SDC_REGION_UNIT_DISK
 * 13 max_iters  >= 1: number of IRS passes (cap for RTEST/E21)
 * 14 tol        >= 0: R-test tau (RTEST) or metric threshold (E21); unused for FIXED
 * 15 stop_mode  SDC_STOP_*
 * 16 Q, 17 ldq  out (device): Q (= Q_R), n x n orthogonal
 * 18 QL,19 ldql out (device): Q_L for pencils, or NULL
 * 20 Ahat,21 ldah optional out (device): Q_L^T A Q, or NULL
 * 22 hist, 23 hist_cap optional HOST buffer, hist_cap rows of 3 doubles per pass j:
 *              {r*, metric} (E21 mode only, else NaN) and the R-test ratio
 *              ||R_j - R_{j-1}||_1/||R_{j-1}||_1 of the right IRS (NaN at j = 0)
 * 24 res       HOST out
 * Synchronises `stream` before returning. */
int sdc_split(sdc_handle* h, void* stream, int n, const double* A, int lda, const double* B,
              int ldb, const double* V, int ldv, const double* VL, int ldvl, int region,
              int max_iters, double tol, int stop_mode, double* Q, int ldq, double* QL, int ldql,
              double* Ahat, int ldah, double* hist, int hist_cap, sdc_result* res);

/* The step for another split region and/or the RSEP variant (region, region_param, flags as
 * in the enums above; all other arguments as sdc_split).  k counts the eigenvalues inside
 * the region (|z| < rho, or Re z < a); Q(:,1:r) spans the complementary invariant subspace.
 * Errors: -12 unknown region, -13 bad region_param, -14 unknown flag, -6 B != NULL with the
 * half plane or the symmetric flag. */
int sdc_split_region(sdc_handle* h, void* stream, int n, const double* A, int lda, const double* B,
                     int ldb, const double* V, int ldv, const double* VL, int ldvl, int region,
                     double region_param, int flags, int max_iters, double tol, int stop_mode,
                     double* Q, int ldq, double* QL, int ldql, double* Ahat, int ldah, double* hist,
                     int hist_cap, sdc_result* res);

/* Singular-value split ("construct the hermitian matrix [[0, A], [A^H, 0]]
 * and compute its eigenvalues (which are the singular values of A and their negatives)";
 * SURVEY §8(f) row f3): the m x n matrix A is embedded on the device into the order
 * N = m + n symmetric H = [[0, A], [A^T, 0]] and one RSEP step (Alg. 6, PAPER.md:436-447:
 * the unit-disk step with Ahat := (Ahat + Ahat^T)/2) splits H along |z| = rho.
 *  1 h          handle with n_max >= m + n
 *  2 stream
 *  3 m, 4 n     rows / columns of A (>= 1)
 *  5 A, 6 lda   input (device), lda >= m
 *  7 rho        > 0, finite: the threshold on the singular values
 *  8 V, 9 ldv   Haar V of order N for GRURV (ldv >= N)
 * 10 max_iters, 11 tol, 12 stop_mode   as sdc_split
 * 13 Q, 14 ldq  out (device): N x N orthogonal; Q(:, r:N-1) spans {[u_i; +-v_i] : sigma_i < rho}
 *               plus the null vectors of H: its rows 0..m-1 span the left and its rows m..N-1
 *               the right singular vectors of the singular values below rho
 * 15 Ahat,16 ldah optional out (device): the symmetrised Q^T H Q (N x N)
 * 17 hist, 18 hist_cap, 19 res   as sdc_split; res->k = 2 #{sigma_i < rho} + |m - n|
 * Workspace: an N x N embedding buffer (n_max^2 doubles) is allocated on first use. */
int sdc_svd_split(sdc_handle* h, void* stream, int m, int n, const double* A, int lda, double rho,
                  const double* V, int ldv, int max_iters, double tol, int stop_mode, double* Q,
                  int ldq, double* Ahat, int ldah, double* hist, int hist_cap, sdc_result* res);

/* Batched small-n split step: `batch` independent RNEP steps on the
 * unit disk (Alg. 5, FIXED passes), one CTA per problem with the whole step in shared
 * memory (compact-WY Householder QR, complement-free IRS products, GRURV with the RQ as a
 * reversed QR, similarity with the original A, split selection; every O(n^3) product on
 * DMMA from shared memory).  2 <= n <= 64.
 *  1 h, 2 stream
 *  3 batch      >= 0 problems
 *  4 n          order of every problem
 *  5 A, 6 lda, 7 strideA   problem b at A + b strideA (device), ld lda >= n, stride >= lda n
 *  8 V, 9 ldv, 10 strideV  Haar V of problem b (device)
 * 11 max_iters  IRS passes (>= 1)
 * 12 Q, 13 ldq, 14 strideQ out (device): Q of problem b
 * 15 res        HOST out: batch sdc_result (iters = max_iters, converged = 0, side = NaN)
 * Synchronises `stream`. */
int sdc_split_batched(sdc_handle* h, void* stream, int batch, int n, const double* A, int lda,
                      long long strideA, const double* V, int ldv, long long strideV, int max_iters,
                      double* Q, int ldq, long long strideQ, sdc_result* res);

/* Recursive divide-and-conquer to block upper triangular form A = Q T Q^T (
 * PAPER.md:406-410 "zero E21 and recurse on (A11, A22)", random splitting lines
 * PAPER.md:472-475 restricted to real arithmetic: vertical lines Re z = a).
 * Decisions (DESIGN.md §10 "recursion", identical in orc_schur): a block of order m is a leaf
 * if m <= leaf, or m == 2 with complex eigenvalues; else up to 16 attempts, each a random
 * line in the middle half of [c - 2s, c + 2s] (c = trace/m, s = ||T_blk - cI||_F/sqrt(m)),
 * a counter-based Haar V (seed; draws keyed by the block's offset and order, see
 * sdc_schur_keyed), and one RNEP half-plane step in monitor mode
 * (SDC_STOP_E21 with `tol`, at most max_iters passes), accepted iff its status is 0; a
 * rejected step whose res.side shows every eigenvalue on one side moves that end of the
 * interval to the line.  On acceptance E21 := 0,
 * T and Q are updated by the block's Q_b and the two diagonal blocks are processed depth
 * first (eigenvalues right of the line first).  16 failed attempts: an unsplit leaf.
 * Blocks of order <= 64 are deferred and run BATCHED: one launch per recursion level, one CTA
 * per block running the whole node in shared memory (same decisions and draws; csrc/
 * schur_batched.cuh, SDC_SCHUR_BATCH=0 disables it), then two launches applying the accepted
 * Q_b to T's strips and to Q.  The draws are keyed by the block, so the order of processing
 * does not change them; the block list is returned sorted by offset (= depth-first order).
 *  1 h, 2 stream, 3 n (<= n_max), 4 A, 5 lda (device input)
 *  6 leaf        >= 1: largest diagonal block left unsplit (1: real Schur-like form)
 *  7 seed        generator seed (lines and Haar matrices)
 *  8 max_iters, 9 tol   per split (monitor mode)
 * 10 Q, 11 ldq  out (device): orthogonal n x n
 * 12 T, 13 ldt  out (device): block upper triangular, exactly 0 below the diagonal blocks
 * 14 blk_off, 15 blk_size   HOST out (n ints each): the diagonal blocks by increasing offset
 * 16 nblk       HOST out: number of blocks
 * 17 stats      HOST out (4 ints): accepted splits, failed attempts, unsplit leaves, passes
 * 18 max_metric HOST out: largest accepted ||E21||_1/||A_block||_1 (the backward error per split)
 * Allocates 5 n x n scratch matrices for the duration of the call; synchronises `stream`. */
int sdc_schur(sdc_handle* h, void* stream, int n, const double* A, int lda, int leaf,
              unsigned long long seed, int max_iters, double tol, double* Q, int ldq, double* T,
              int ldt, int* blk_off, int* blk_size, int* nblk, int* stats, double* max_metric);

/* sdc_schur with the random draws keyed by GLOBAL block offsets: the attempt-t line and
 * Haar V of the diagonal block at offset o (of A) use the counter c = key(key_off + o, m, t)
 * (DESIGN.md §10), so a subproblem A = T(o0:o0+n, o0:o0+n) of a larger recursion, solved
 * on its own with key_off = o0 -- e.g. on the rank it was handed to --
 * takes exactly the decisions the whole recursion takes there.  Arguments as sdc_schur with
 * 6 key_off >= 0 inserted (later positions shift by one).  sdc_schur = key_off 0. */
int sdc_schur_keyed(sdc_handle* h, void* stream, int n, const double* A, int lda, int key_off, int leaf,
                    unsigned long long seed, int max_iters, double tol, double* Q, int ldq, double* T,
                    int ldt, int* blk_off, int* blk_size, int* nblk, int* stats, double* max_metric);

/* One node of the recursion: the attempt loop of sdc_schur on the diagonal block Tb
 * (m x m, device, ld ldtb >= m) at global offset key_off, IN PLACE.
 *  13 r  HOST out: r in [1, m-1] when a split was accepted -- then Tb holds Ahat = Q_b^T Tb Q_b
 *        with E21 := 0 and Qb (device, m x m, ld ldqb) the orthogonal Q_b; r = 0 for a leaf
 *        (m <= leaf, or a 2x2 with complex eigenvalues) or an unsplit block (Tb unchanged)
 *  14 stats, 15 max_metric  HOST, ACCUMULATED (not reset) as in sdc_schur
 * Errors: -3 m, -4 Tb, -5 ldtb, -6 key_off, -7 leaf, -9 max_iters, -10 tol, -11 Qb, -12 ldqb,
 * -13 NULL host output.  Allocates 3 m x m scratch matrices; synchronises `stream`.  Blocks of
 * order <= 64 run in the batched kernel of sdc_schur (one block), so a node solved on its own
 * takes the decisions the whole recursion takes there. */
int sdc_schur_node(sdc_handle* h, void* stream, int m, double* Tb, int ldtb, int key_off, int leaf,
                   unsigned long long seed, int max_iters, double tol, double* Qb, int ldqb, int* r,
                   int* stats, double* max_metric);

/* Eigenvectors of an upper triangular matrix (TREVC):
 * X upper triangular with X_jj = 1 and TX = XD, D = diag(T), or, when
 * Q != NULL, the eigenvectors Q X of A = Q T Q^T.  Real T with real
 * eigenvalues (the triangular case of the paper; 2x2 blocks of a real quasi-triangular
 * Schur form are not supported).  No overflow scaling: X_ij grows with the departure from
 * normality over eigenvalue gaps; a gap below smin = max(2^-52 |T_jj|, DBL_MIN n 2^52) is
 * replaced by smin (LAPACK dtrevc rule, reading Q19).
 *  1 h          handle, n <= n_max
 *  2 stream
 *  3 n          order >= 1
 *  4 T, 5 ldt   upper triangular input (device; the strictly lower part is not read)
 *  6 Q, 7 ldq   optional orthogonal n x n (device) or NULL
 *  8 X, 9 ldx   out (device) n x n; must not alias T or Q
 * Blocked (b = 64) as Alg. 8 with block rows swept bottom-up: one DMMA GEMM
 * S = T[i, i+1:] X[i+1:, i+1:] per block row (n^3/3 flops; + 2 n^3 / 2 for Q X) and one
 * shifted-block-solve launch.  Enqueued on `stream`; does not synchronise. */
int sdc_trevc(sdc_handle* h, void* stream, int n, const double* T, int ldt, const double* Q,
              int ldq, double* X, int ldx);

/* Same step with HOST matrices (column-major, tightly packed ld = n): copies A, B, V, VL to
 * the device, runs sdc_split, and copies Q (and QL, Ahat when non-NULL) back -- the
 * end-to-end path of the public API.  Host buffers may be pageable or pinned. */
int sdc_split_host(sdc_handle* h, void* stream, int n, const double* A, const double* B,
                   const double* V, const double* VL, int max_iters, double tol, int stop_mode,
                   double* Q, double* QL, double* Ahat, double* hist, int hist_cap,
                   sdc_result* res);

/* ---- building blocks of the step, exported for kernel-level parity tests ---------- */

/* C = alpha op(A) op(B) + beta C on the FP64 tensor cores (DMMA); op = transpose when
 * transa/transb != 0.  M x N result, K inner.  PAPER.md:916 (matrix multiply). */
int sdc_dgemm(sdc_handle* h, void* stream, int transa, int transb, int M, int N, int K,
              double alpha, const double* A, int lda, const double* B, int ldb, double beta,
              double* C, int ldc);

/* Blocked Householder QR of the m x n matrix A (m >= n, m <= 2 n_max, n <= n_max) in
 * place: on return the upper triangle of A holds R with a NON-NEGATIVE diagonal (rows
 * scaled by sign(R_ii); the strictly lower part is workspace).  If Qthin != NULL it
 * receives the explicit m x n Q of the same factorization (A = Qthin R).  PAPER.md:331;
 * north_star "R diagonal forced non-negative".  Synchronises `stream`. */
int sdc_qr(sdc_handle* h, void* stream, int m, int n, double* A, int lda, double* Qthin,
           int ldq);

/* One IRS pass (Alg. 3 line 3): Aout = Q12^T A, Bout = Q22^T B for [B; -A] = Q [R; 0],
 * and Rout (n x n, optional) = R with non-negative diagonal. */
int sdc_irs_pass(sdc_handle* h, void* stream, int n, const double* A, int lda, const double* B,
                 int ldb, double* Aout, int ldao, double* Bout, int ldbo, double* Rout, int ldr);

/* Split selection on Ahat (and Bhat, or NULL) with the given norms:
 * returns r (1..n-1, ties -> smallest) and the metric on the host; mvals (optional,
 * DEVICE, length n) receives m(r) at index r (index 0 unused). */
int sdc_split_select(sdc_handle* h, void* stream, int n, const double* Ahat, int ldah,
                     double normA, const double* Bhat, int ldbh, double normB, int* r,
                     double* metric, double* mvals);

/* Per-kernel-class timing with CUDA events recorded on the launching stream around every
 * launch of the class (measurement support for bench.py's roofline numbers).
 * sdc_profile(h, 1) resets the counters and starts recording, (h, 0) stops.
 * sdc_profile_read returns, for class cls, the class time (ms), the number of launches
 * and the summed ALGORITHMIC work: flops 2MNK for SDC_PROF_GEMM, bytes (read + write of
 * the operands the definition touches) for the other classes.  The class time is the
 * UNION of the launch intervals, i.e. the wall time during which at least one launch of the
 * class ran.  Launches of a class can overlap on the look-ahead and second-context streams;
 * on a serial schedule the union equals the summed durations. */
enum { SDC_PROF_GEMM = 0,        /* every DMMA GEMM launch                                */
       SDC_PROF_PANEL = 1, SDC_PROF_WYRED = 2, SDC_PROF_SELECT = 3,
       SDC_PROF_GEMM_W0 = 4,     /* subset of GEMM: split-K W0 = Y^T C of WY applications    */
       SDC_PROF_GEMM_UPD = 5,    /* subset of GEMM: rank-nb updates C -= Y W                 */
       SDC_PROF_GEMM_OTHER = 6,  /* subset of GEMM: the n x n products (a5, a7, a8)         */
       SDC_PROF_TREVC = 7,       /* sdc_trevc shifted block solves (bytes: T block + column) */
       SDC_PROF_CLASSES = 8 };
int sdc_profile(sdc_handle* h, int enable);
int sdc_profile_read(sdc_handle* h, int cls, double* ms, long long* launches, double* work);

/* Debug counters (enabled by env SDC_DEBUG_COUNTERS at sdc_create): copies `count` (<= 64)
 * device counters to the HOST array `out`; reset != 0 zeroes them.  Slots 0-3 / 4-7: panel
 * kernel clock64 cycles (partials, grid barrier, partial sums, update) of CTA 0 / the last
 * CTA summed over columns; slot 8: number of timed panel CTAs. */
int sdc_debug_counters(sdc_handle* h, unsigned long long* out, int count, int reset);

/* Number of kernels launched by this handle since creation (evidence counter). */
long long sdc_kernel_launches(const sdc_handle* h);

/* Schedule evidence: how often each code path of the step was ENQUEUED by this handle
 * (launches inside a captured CUDA graph count once, at capture).  Tests use them to prove
 * that a parity case ran the path it names (look-ahead fork, multi-cluster panel, ...). */
enum { SDC_SCHED_LOOKAHEAD_FORKS = 0,  /* look-ahead QR schedules forked to the hi-prio stream */
       SDC_SCHED_XPASS_FORKS = 1,      /* look-ahead QRs forked by the previous pass (SDC_XPASS) */
       SDC_SCHED_CTX_FORKS = 2,        /* forks to the second factorization context            */
       SDC_SCHED_PANEL_CLUSTER = 3,    /* panels as one cluster (DSMEM exchange)               */
       SDC_SCHED_PANEL_MCLUSTER = 4,   /* panels as several 16-CTA clusters (DSMEM + L2 flags)  */
       SDC_SCHED_PANEL_GRID = 5,       /* panels as a cooperative grid (L2 + grid barrier)      */
       SDC_SCHED_GRAPH_CAPTURES = 6,   /* fixed-mode steps captured into a CUDA graph           */
       SDC_SCHED_GRAPH_REPLAYS = 7,    /* fixed-mode steps replayed from the graph              */
       SDC_SCHED_PANEL_MCLUSTER_CAPPED = 8, /* multi-cluster panels limited to half the
                                          resident clusters (two contexts share the SMs)   */
       SDC_SCHED_PANEL_CQR_TRIED = 9,  /* panels launched with the CholeskyQR2 path first     */
       SDC_SCHED_PANEL_CQR_DONE = 10,  /* ... factored by it (device count; reading it syncs)  */
       SDC_SCHED_PANEL_CQR_FALLBACK = 11, /* ... that fell back to the Householder loop      */
       SDC_SCHED_GEMM_CPASYNC = 12,    /* step GEMMs staged by cp.async (an operand not 16-byte
                                          aligned) instead of TMA                            */
       SDC_SCHED_MAX_CLUSTERS16 = 13,  /* (constant) 16-CTA panel clusters resident at once    */
       SDC_SCHED_PANEL_MCLUSTER8 = 14, /* multi-cluster panels built from 8-CTA clusters (tall
                                          stacks: keeps <= 256 rows per CTA in registers)    */
       SDC_SCHED_GEMM_TMA = 15,        /* step GEMMs staged by TMA                              */
       SDC_SCHED_SCHUR_BATCH_LAUNCHES = 16, /* sdc_schur: launches of the batched small-block
                                          kernel (one per recursion level and size class)   */
       SDC_SCHED_SCHUR_BATCH_BLOCKS = 17,   /* ... diagonal blocks (order <= 64) they processed */
       SDC_SCHED_PANEL_CQ_SPLIT = 18,  /* panels factored by the split CholeskyQR2 kernel chain
                                          (tall stack panels next to the bulk update)         */
       SDC_SCHED_CQ_SPLIT_BREAKDOWNS = 19, /* ... whose Cholesky broke down (fallback kernel ran;
                                          known after the call's final synchronisation)       */
       SDC_SCHED_COUNTERS = 20 };
/* Copies `count` (<= SDC_SCHED_COUNTERS) counters to the HOST array out; reset != 0 zeroes
 * them.  count > SDC_SCHED_PANEL_CQR_DONE synchronises the device (device-side counters).
 * Returns 0, -1 (null handle), -3 (bad count) or -100. */
int sdc_schedule_counters(sdc_handle* h, long long* out, int count, int reset);

/* Text of the last error on this thread ("" if none). */
const char* sdc_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* SDC_H */
