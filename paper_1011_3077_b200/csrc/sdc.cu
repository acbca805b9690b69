// sdc.cu -- libsdc.so: host orchestration + C ABI (include/sdc.h) of one inverse-free
// split step on one B200 (sm_100a).  Every arithmetic step runs in the kernels of
// gemm.cuh (FP64 tensor-core DMMA), panel.cuh (Householder panels) and aux.cuh (O(n^2)
// passes); this file only sequences them on the caller's stream and owns the workspace.
//
// Step structure:
//   IRS pass j (Alg. 3):  blocked Householder QR of S = [B_j; -A_j] (panels + WY
//     trailing updates), complement [Q12;Q22] = H_0..H_{n-1}[0;I] (backward WY), then
//     A_{j+1} = Q12^T A_j, B_{j+1} = Q22^T B_j whose epilogue also writes the next stack.
//   GRURV (Alg. 1/2):  X = A_p V^T, QR(X) -> U, C = U^T (A_p+B_p), RQ(C) computed as the
//     QR of C^T J with explicit Q, Q = Q_qr D J (reading Q10).
//   Similarity Q_L^T A Q and split selection.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: per-stage ranges

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/sdc.h"
#include "aux.cuh"
#include "common.cuh"
#include "gemm.cuh"
#include "gemm_tma.cuh"
#include "panel.cuh"
#include "trevc.cuh"
#include "batched.cuh"
#include "schur_batched.cuh"
#include "cqr_split.cuh"

using namespace sdc;

namespace {

thread_local char g_err[1024] = "";

void set_err(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

#define SDC_CK(x)                                                              \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      set_err("%s:%d %s: %s", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      return e_ == cudaErrorMemoryAllocation ? SDC_ERR_NOMEM : SDC_ERR_CUDA;  \
    }                                                                          \
  } while (0)
#define SDC_TRY(x)            \
  do {                        \
    int rc_ = (x);            \
    if (rc_ != 0) return rc_; \
  } while (0)

// NVTX range per stage of the step (IRS pass, QR, GRURV, similarity + selection, ...), so
// an nsys/ncu timeline groups the kernels by the paper's steps; no-ops without a tool
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
};

// Per-device "already set" flags for cudaFuncSetAttribute (the attribute is per device;
// a process may hold handles on several devices)
constexpr int MAX_DEV = 64;
struct DevOnce {
  std::atomic<unsigned long long> mask{0};
  static unsigned long long bit(int dev) { return 1ull << (dev & (MAX_DEV - 1)); }
  bool has(int dev) const { return (mask.load(std::memory_order_relaxed) & bit(dev)) != 0; }
  void set(int dev) { mask.fetch_or(bit(dev), std::memory_order_relaxed); }
};

constexpr int NB = PANEL_NB;       // panel / WY block width
constexpr int SCAL_HIST = 12;      // scal[12 + j]: R-test ratio of pass j; scal[8..11]: norms of
                                   // the final right IRS pair (1, F) of A_p and of B_p
constexpr int MAX_HIST = 65536;

}  // namespace

struct sdc_handle {
  int device = 0, n_max = 0, pencil = 0, num_sms = 0;
  cudaStream_t st = nullptr;
  // workspace (see sdc_create for sizes)
  double *S = nullptr, *SL = nullptr, *Y = nullptr, *Yt = nullptr, *C = nullptr;
  double *Vt = nullptr, *VLt = nullptr;
  double *A[2] = {nullptr, nullptr}, *B[2] = {nullptr, nullptr};
  double *AL[2] = {nullptr, nullptr}, *BL[2] = {nullptr, nullptr};
  double *G1 = nullptr, *G2 = nullptr, *G3 = nullptr, *T1 = nullptr, *Ah = nullptr, *Bh = nullptr;
  double *QLb = nullptr, *Rprev = nullptr;
  double* Emb = nullptr;               // hermitian embedding of sdc_svd_split (lazy, n_max^2)
  double* bat_out = nullptr;           // sdc_split_batched per-problem results (lazy)
  size_t bat_out_n = 0;
  double *Tb = nullptr, *tau = nullptr, *Wp = nullptr, *W = nullptr, *gbuf = nullptr;
  double* llbuf = nullptr;             // flag-carrying exchange slots of the multi-cluster panel
  double* cqbuf = nullptr;             // CholeskyQR2 panel exchange slots (CQ_DOUBLES)
  bool cqr = true;                     // CholeskyQR2 panels allowed (workspace, smem)
  int cqr_mode = 1;                    // SDC_CQR: 0 never, 1 tall multi-cluster panels, 2 always
  unsigned long long* cqstat = nullptr;   // device: [0] CQR panels done, [1] fallbacks
  unsigned ll_epoch = 0;               // advanced by nb per multi-cluster panel launch
  double *pmA = nullptr, *pmB = nullptr, *vec = nullptr, *scal = nullptr;
  size_t wp_elems = 0;
  unsigned int* bar = nullptr;
  unsigned long long bar_count = 0;
  int* flag = nullptr;
  long long launches = 0;
  long long sched[SDC_SCHED_COUNTERS] = {0};   // schedule evidence (sdc_schedule_counters)
  bool share_sms = false;              // two factorization contexts may run panels at once
  unsigned long long* dbg = nullptr;   // debug counters (sdc_debug_counters)
  bool dbg_on = false;
  int panel_rows = 128;                // target rows per panel CTA
  bool cluster_ok = false;             // 16-CTA clusters usable for the panel kernel
  bool mcluster_ok = false;            // several co-resident 16-CTA clusters (tall panels)
  bool panel_reg = true;               // register-resident panel column loop (rows_per <= 256)
  bool ql_orth = false;                // current call: SDC_FLAG_QL_ORTH
  int max_clusters16 = 0;
  int max_clusters8 = 0;               // 8-CTA clusters resident at once (256-row blocks)
  int cluster_max_rows = 4096;         // panels with at most this many rows use one cluster
  int nbo = 256;                       // outer compact-WY block width of the current call
  int nbo_max = 256;                   // width the workspace is sized for
  bool nbo_fixed = false;              // SDC_NBO given: no per-size choice
  double *Tob = nullptr, *Tobt = nullptr, *Zb = nullptr, *Gb = nullptr;
  // look-ahead QR (blocked_qr): panels and the next block's update on a high-priority
  // handle stream, the bulk trailing update of each outer block on the caller's stream with
  // its own split-K workspace (Wp2, W2, Zb2)
  bool lookahead = true;
  bool on_side = false;                // issuing on the look-ahead side stream
  bool in_alt = false;                 // issuing on the second factorization context
  bool two_chains = false;             // both factorization contexts busy (pencil, Alg. 4)
  bool xpass_pending = false;          // la_fork / la_B recorded by the previous IRS pass
  bool xpass_on = false;               // cross-pass look-ahead in the fixed-mode pass loop
                                       // (SDC_XPASS=1; measured no gain: the first panels'
                                       // cluster waits for the products' CTAs to drain)
  // GEMM schedule knobs (env at sdc_create; DESIGN.md §6 table): persistent grids for short-K
  // updates (0 off, 1 short-K, 2 every TMA GEMM), bulk reduce-add epilogue for beta = 1,
  // persistent grids on the side stream / second chain too
  int split_kmin = 128;                // SDC_SPLIT_KMIN: shortest K slice of a split-K GEMM (256 -> 128:
                                       // config 2 82.8 -> 76.5 ms; the small W0 = Y^T C products of the
                                       // panel chain were 64 CTAs of 16 K-tiles)
  int persist_mode = 1, red_mode = 1;
  bool side_persist = false;
  // CholeskyQR2 panel as a chain of small kernels (cqr_split.cuh): SDC_CQ_SPLIT 0 never, 1 tall
  // panels (> cq_split_rows rows) of the look-ahead stack QR of an IRS pass, 2 every full-width
  // panel of >= 128 rows (tests).  cq_split_ctx: inside such a QR.  A reported breakdown turns
  // mode 1 off for the handle (the fallback is correct but slow).
  int cq_split = 1, cq_split_rows = 8192;
  // two chains sharing the SMs (monitor mode, pencils): every multi-cluster stack panel takes the
  // chain -- a cluster launch has to gather 16 SMs of one GPC between the other chain's CTAs,
  // ordinary CTAs do not (config 3: 2286 -> 2111 ms; alone the cluster kernel is faster there)
  int cq_split_rows_shared = 4096;
  bool cq_split_ctx = false;
  double* cqs = nullptr;
  unsigned* cqs_sync = nullptr;
  bool schur_batch = true;             // SDC_SCHUR_BATCH: blocks of order <= 64 of the recursion in
                                       // one launch per level (schur_batched.cuh)
  cudaStream_t st_hi = nullptr;
  cudaEvent_t la_fork = nullptr, la_fac = nullptr, la_B = nullptr, la_join = nullptr;
  double *Wp2 = nullptr, *W2 = nullptr, *Zb2 = nullptr;
  // Second factorization context (lazy): its own stream and every buffer a QR / GRURV chain
  // writes, so two independent chains run concurrently -- the left and right IRS of a
  // pencil (Alg. 4), and in monitor mode GRURV(j) + similarity next to IRS pass j+1.
  // swap_ctx() exchanges these fields with the active ones (host code is single-threaded).
  struct Ctx {
    cudaStream_t st = nullptr, st_hi = nullptr;
    cudaEvent_t la_fork = nullptr, la_fac = nullptr, la_B = nullptr, la_join = nullptr;
    double *Y = nullptr, *Yt = nullptr, *Tb = nullptr, *Tob = nullptr, *Tobt = nullptr, *Zb = nullptr,
           *Gb = nullptr, *tau = nullptr, *Wp = nullptr, *W = nullptr, *gbuf = nullptr, *llbuf = nullptr,
           *vec = nullptr, *Wp2 = nullptr, *W2 = nullptr, *Zb2 = nullptr, *C = nullptr, *G1 = nullptr,
           *G2 = nullptr, *G3 = nullptr, *cqbuf = nullptr, *cqs = nullptr;
    unsigned int* bar = nullptr;
    unsigned int* cqs_sync = nullptr;
    unsigned long long bar_count = 0;
    unsigned ll_epoch = 0;
    int gemm_force = -1;
    bool xpass_pending = false;
  } alt;
  int gemm_force = -1;   // debug: force a GEMM variant in this context
  bool alt_ready = false, pipeline = true, alt_fail_hook = false;
  cudaEvent_t ev_a = nullptr, ev_b = nullptr, ev_c = nullptr;   // cross-context dependencies
  // CUDA graph of the FIXED-mode step (replayed while the call signature is unchanged)
  struct GraphKey {
    int n = 0, max_iters = 0, nbo = 0, region = 0, rflags = 0;
    double rparam = 0.0;
    const void *A = nullptr, *B = nullptr, *V = nullptr, *VL = nullptr, *Q = nullptr, *QL = nullptr,
               *Ahat = nullptr;
    long long lda = 0, ldb = 0, ldv = 0, ldvl = 0, ldq = 0, ldql = 0, ldah = 0;
    bool operator==(const GraphKey& o) const {
      return n == o.n && max_iters == o.max_iters && nbo == o.nbo && region == o.region &&
             rflags == o.rflags && rparam == o.rparam && A == o.A && B == o.B && V == o.V &&
             VL == o.VL && Q == o.Q && QL == o.QL && Ahat == o.Ahat && lda == o.lda && ldb == o.ldb &&
             ldv == o.ldv && ldvl == o.ldvl && ldq == o.ldq && ldql == o.ldql && ldah == o.ldah;
    }
  } gkey;
  cudaGraphExec_t gexec = nullptr;
  cudaStream_t cap_st = nullptr;
  long long glaunches = 0;
  int graph_max_n = 4096;
  double* hscal = nullptr;             // pinned host copies of the result scalars
  const double *cur_V = nullptr, *cur_VL = nullptr;
  int region = SDC_REGION_UNIT_DISK, rflags = 0;   // region / flags of the current call
  double rparam = 1.0;
  const double* b_ident = nullptr;     // B buffer known to hold b_ident_rho * I (first pass)
  double b_ident_rho = 1.0;
  long long cur_ldv = 0, cur_ldvl = 0;
  unsigned int* hflags = nullptr;      // pinned: [0] non-finite flag, [1] barrier error
  // optional per-kernel-class timing with CUDA events on the launching stream
  bool prof_on = false;
  int gemm_sub = SDC_PROF_GEMM_OTHER;   // sub-class of the GEMMs being launched
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  struct ProfRec { int cls; int e0, e1; double work; int tag; };
  std::vector<ProfRec> recs;
  double prof_ms[SDC_PROF_CLASSES] = {0}, prof_work[SDC_PROF_CLASSES] = {0};
  long long prof_n[SDC_PROF_CLASSES] = {0};
  // staging for sdc_split_host
  double *hA = nullptr, *hB = nullptr, *hV = nullptr, *hVL = nullptr, *hQ = nullptr,
         *hQL = nullptr, *hAh = nullptr;
  std::vector<void*> allocs;
};

namespace {

int dalloc(sdc_handle* h, double** p, size_t elems) {
  void* q = nullptr;
  cudaError_t e = cudaMalloc(&q, std::max<size_t>(elems, 1) * sizeof(double));
  if (e != cudaSuccess) {
    set_err("cudaMalloc(%zu doubles): %s", elems, cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? SDC_ERR_NOMEM : SDC_ERR_CUDA;
  }
  h->allocs.push_back(q);
  *p = static_cast<double*>(q);
  return 0;
}

// exchange the active factorization context with h->alt
void swap_ctx(sdc_handle* h) {
  auto& a = h->alt;
  std::swap(h->st, a.st); std::swap(h->st_hi, a.st_hi);
  std::swap(h->la_fork, a.la_fork); std::swap(h->la_fac, a.la_fac);
  std::swap(h->la_B, a.la_B); std::swap(h->la_join, a.la_join);
  std::swap(h->Y, a.Y); std::swap(h->Yt, a.Yt); std::swap(h->Tb, a.Tb); std::swap(h->Tob, a.Tob);
  std::swap(h->Tobt, a.Tobt); std::swap(h->Zb, a.Zb); std::swap(h->Gb, a.Gb); std::swap(h->tau, a.tau);
  std::swap(h->Wp, a.Wp); std::swap(h->W, a.W); std::swap(h->gbuf, a.gbuf); std::swap(h->llbuf, a.llbuf);
  std::swap(h->vec, a.vec); std::swap(h->Wp2, a.Wp2); std::swap(h->W2, a.W2); std::swap(h->Zb2, a.Zb2);
  std::swap(h->bar, a.bar); std::swap(h->bar_count, a.bar_count); std::swap(h->ll_epoch, a.ll_epoch);
  std::swap(h->C, a.C); std::swap(h->G1, a.G1); std::swap(h->G2, a.G2); std::swap(h->G3, a.G3);
  std::swap(h->gemm_force, a.gemm_force);
  std::swap(h->cqbuf, a.cqbuf);
  std::swap(h->cqs, a.cqs); std::swap(h->cqs_sync, a.cqs_sync);
  std::swap(h->xpass_pending, a.xpass_pending);
}
struct AltScope {   // issue on the second context for the scope's lifetime
  sdc_handle* h;
  explicit AltScope(sdc_handle* h_) : h(h_) { swap_ctx(h); h->in_alt = true; }
  ~AltScope() { swap_ctx(h); h->in_alt = false; }
};

inline int cdiv(long long a, long long b) { return (int)((a + b - 1) / b); }
// leading dimension of the n x n workspace matrices: n rounded up to even, so that every
// column starts 16-byte aligned and odd n keeps the TMA GEMM path
inline long long wld(long long n) { return n + (n & 1); }
inline bool al16(const void* p, long long ld) {
  return ((reinterpret_cast<uintptr_t>(p) & 15) == 0) && (ld % 2 == 0);
}
inline int ew_grid(long long elems) { return (int)std::min<long long>(cdiv(elems, 256), 148LL * 16); }

#define SDC_LAUNCHED(h)                                                            \
  do {                                                                             \
    (h)->launches++;                                                               \
    cudaError_t e_ = cudaGetLastError();                                           \
    if (e_ != cudaSuccess) {                                                       \
      set_err("%s:%d launch: %s", __FILE__, __LINE__, cudaGetErrorString(e_));     \
      return SDC_ERR_CUDA;                                                         \
    }                                                                              \
  } while (0)

// ---- per-class CUDA-event timing (sdc_profile) --------------------------------------
int prof_event(sdc_handle* h) {
  if (h->ev_used == h->ev_pool.size()) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return -1;
    h->ev_pool.push_back(e);
  }
  int id = (int)h->ev_used++;
  cudaEventRecord(h->ev_pool[id], h->st);
  return id;
}
struct ProfScope {
  sdc_handle* h; int cls, sub; double work; int e0;
  ProfScope(sdc_handle* h_, int cls_, double work_, int sub_ = -1)
      : h(h_), cls(cls_), sub(sub_), work(work_), e0(-1) {
    if (h->prof_on) e0 = prof_event(h);
  }
  ~ProfScope() {
    if (h->prof_on && e0 >= 0) {
      int e1 = prof_event(h);
      if (e1 >= 0) {
        const int tag = (h->st == h->st_hi ? 1 : 0) | (h->on_side ? 2 : 0) | (h->in_alt ? 4 : 0);   // stream
        h->recs.push_back({cls, e0, e1, work, tag});
        if (sub >= 0) h->recs.push_back({sub, e0, e1, work, tag});
      }
    }
  }
};
// Launches of one class can overlap (look-ahead QR, second context), so the class time is
// the UNION of its launch intervals -- the wall time during which at least one launch of the
// class ran -- not the sum of durations; for a serial schedule the two are equal.
void prof_collect(sdc_handle* h) {
  if (h->recs.empty()) return;
  for (auto& r : h->recs) cudaEventSynchronize(h->ev_pool[r.e1]);   // events on several streams
  const cudaEvent_t ref = h->ev_pool[h->recs.front().e0];
  std::vector<std::pair<float, float>> iv[SDC_PROF_CLASSES];
  FILE* dump = nullptr;   // SDC_PROF_DUMP=path: one line per launch record (class, start, end in ms, work)
  if (const char* dp = getenv("SDC_PROF_DUMP")) dump = fopen(dp, "a");
  for (auto& r : h->recs) {
    float a = 0.f, b = 0.f;
    cudaEventElapsedTime(&a, ref, h->ev_pool[r.e0]);
    cudaEventElapsedTime(&b, ref, h->ev_pool[r.e1]);
    if (dump) fprintf(dump, "%d %d %.4f %.4f %.6g\n", r.cls, r.tag, a, b, r.work);
    iv[r.cls].push_back({a, b});
    h->prof_work[r.cls] += r.work;
    h->prof_n[r.cls] += 1;
  }
  for (int c = 0; c < SDC_PROF_CLASSES; ++c) {
    auto& v = iv[c];
    if (v.empty()) continue;
    std::sort(v.begin(), v.end());
    double tot = 0.0, lo = v[0].first, hi = v[0].second;
    for (size_t i = 1; i < v.size(); ++i) {
      if (v[i].first > hi) { tot += hi - lo; lo = v[i].first; hi = v[i].second; }
      else hi = std::max(hi, (double)v[i].second);
    }
    tot += hi - lo;
    h->prof_ms[c] += tot;
  }
  if (dump) fclose(dump);
  h->recs.clear();
  h->ev_used = 0;
}

// ---------------------------------------------------------------------------------------
// GEMM dispatch.  Every contraction of the step is TN (both operands K-major):
//   C = alpha A_s^T B_s + beta C, A_s K x M, B_s K x N (column-major).
// TMA path (gemm_tma.cuh) when both operands are 16-byte aligned with even ld; otherwise
// the cp.async kernel (gemm.cuh) -- same arithmetic, only the operand staging differs.
// ---------------------------------------------------------------------------------------
using TileL = GemmTile<128, 128, 16, 64, 32, 4>;  // cp.async fallback tiles
using TileM = GemmTile<64, 128, 16, 32, 32, 4>;
using TileS = GemmTile<64, 64, 16, 32, 32, 4>;

using TmaL = TmaTile<128, 128, 64, 32, 6>;      // 8 consumer warps, 192 KB ring
using TmaM = TmaTile<64, 128, 32, 32, 6>;       // M <= 64 (W0 = Y^T C), 8 consumer warps
using TmaS = TmaTile<64, 64, 32, 32, 6>;        // small grids, 4 consumer warps
using TmaU = TmaTile<128, 64, 64, 32, 4, 2>;    // rank-nb updates: 2 CTAs/SM, epilogue overlap
using TmaC = TmaTile<128, 128, 64, 32, 3, 1, true>;  // K <= 256 updates, C tile prefetched by TMA
using TmaR = TmaTile<128, 64, 64, 32, 3, 2, false, true>;  // updates with beta = 1: bulk reduce-add
template <class T, bool TA, bool TB, int VEC>
int launch_gemm_t(sdc_handle* h, const GemmArgs& g, int splits) {
  using Sm = GemmSmem<T, TA, TB>;
  static DevOnce attr;   // per instantiation and device
  if (!attr.has(h->device)) {
    SDC_CK(cudaFuncSetAttribute(gemm_dmma_kernel<T, TA, TB, VEC>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Sm::BYTES));
    attr.set(h->device);
  }
  dim3 grid(cdiv(g.M, T::BM), cdiv(g.N, T::BN), splits);
  ProfScope ps(h, SDC_PROF_GEMM, 2.0 * g.M * g.N * (double)g.K, h->gemm_sub);
  gemm_dmma_kernel<T, TA, TB, VEC><<<grid, T::THREADS, Sm::BYTES, h->st>>>(g);
  SDC_LAUNCHED(h);
  return 0;
}

template <class T, bool TA, bool TB>
int launch_gemm_v(sdc_handle* h, const GemmArgs& g, int splits) {
  if (al16(g.A, g.lda) && al16(g.B, g.ldb)) return launch_gemm_t<T, TA, TB, 2>(h, g, splits);
  return launch_gemm_t<T, TA, TB, 1>(h, g, splits);
}

template <bool TA, bool TB>
int launch_gemm_tile(sdc_handle* h, const GemmArgs& g, int splits) {
  if (g.M <= 64) return launch_gemm_v<TileM, TA, TB>(h, g, splits);
  long long tilesL = (long long)cdiv(g.M, 128) * cdiv(g.N, 128) * splits;
  if (tilesL >= h->num_sms) return launch_gemm_v<TileL, TA, TB>(h, g, splits);
  return launch_gemm_v<TileS, TA, TB>(h, g, splits);
}

// ---- TMA descriptors (driver entry point fetched once through the runtime) ----------
PFN_cuTensorMapEncodeTiled_v12000 tma_encode_fn() {
  // initialised once, thread-safely (handles may live on several host threads)
  static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
  }();
  return fn;
}

// 2-D fp64 K-major operand: rows = K (contiguous), cols = M or N, ld in elements.
// Box = 16 (one 128-byte swizzle row) x box_cols; zero fill outside the tensor.
bool make_tmap(CUtensorMap* tm, const double* ptr, int rows, int cols, long long ld, int box_cols) {
  auto fn = tma_encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)rows, (cuuint64_t)cols};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
  cuuint32_t box[2] = {16, (cuuint32_t)box_cols};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(ptr), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// algorithmic flops of a TMA GEMM launch: 2 M N K, or with kupper (B_s upper triangular,
// zero products skipped) 2 M sum_{c < N} min(K, c + 1)
double tma_gemm_work(const TmaGemmArgs& g) {
  const double M = g.M, N = g.N, K = g.K;
  if (!g.kupper) return 2.0 * M * N * K;
  const double cols = K >= N ? N * (N + 1) / 2 : K * (K + 1) / 2 + (N - K) * K;
  return 2.0 * M * cols;
}


template <class T>
int launch_tma_t(sdc_handle* h, const double* A, long long lda, const double* B, long long ldb,
                 const TmaGemmArgs& g, int splits) {
  static DevOnce attr;
  const int smem = (int)T::SMEM;
  if (!attr.has(h->device)) {
    SDC_CK(cudaFuncSetAttribute(gemm_tn_tma_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr.set(h->device);
  }
  CUtensorMap tA, tB, tC;
  if (!make_tmap(&tA, A, g.K, g.M, lda, T::BM) || !make_tmap(&tB, B, g.K, g.N, ldb, T::BN)) {
    set_err("cuTensorMapEncodeTiled failed");
    return SDC_ERR_CUDA;
  }
  if (T::CPRE) {   // C as a 2-D tensor: rows = M (contiguous), cols = N; 16-row boxes
    if (!make_tmap(&tC, g.C, g.M, g.N, g.ldc, T::BN)) {
      set_err("cuTensorMapEncodeTiled (C) failed");
      return SDC_ERR_CUDA;
    }
  } else {
    tC = tA;
  }
  dim3 grid(cdiv(g.M, T::BM), cdiv(g.N, T::BN), splits);
  ProfScope ps(h, SDC_PROF_GEMM, tma_gemm_work(g), h->gemm_sub);
  gemm_tn_tma_kernel<T><<<grid, T::THREADS, smem, h->st>>>(tA, tB, tC, g);
  SDC_LAUNCHED(h);
  return 0;
}

template <class T>
int launch_tma_persist(sdc_handle* h, const double* A, long long lda, const double* B, long long ldb,
                       const TmaGemmArgs& g, int splits) {
  static DevOnce attr;
  const int smem = (int)T::SMEM;
  if (!attr.has(h->device)) {
    SDC_CK(cudaFuncSetAttribute(gemm_tn_tma_persist_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr.set(h->device);
  }
  CUtensorMap tA, tB;
  if (!make_tmap(&tA, A, g.K, g.M, lda, T::BM) || !make_tmap(&tB, B, g.K, g.N, ldb, T::BN)) {
    set_err("cuTensorMapEncodeTiled failed");
    return SDC_ERR_CUDA;
  }
  const long long tiles = (long long)cdiv(g.M, T::BM) * cdiv(g.N, T::BN) * splits;
  const int grid = (int)std::min<long long>(tiles, (long long)h->num_sms * T::MINB);
  ProfScope ps(h, SDC_PROF_GEMM, tma_gemm_work(g), h->gemm_sub);
  gemm_tn_tma_persist_kernel<T><<<grid, T::THREADS, smem, h->st>>>(tA, tB, g);
  SDC_LAUNCHED(h);
  return 0;
}


// C = alpha A_s^T B_s + beta C  [+ D2 = alpha2 A_s^T B_s];  K-split into `splits` slices of
// kchunk (multiple of 16) written to C + z * c_zstride when splits > 1.
int gemm_tn(sdc_handle* h, int M, int N, int K, double alpha, const double* A, long long lda,
            const double* B, long long ldb, double beta, double* C, long long ldc,
            double* D2 = nullptr, long long ldd2 = 0, double alpha2 = 0.0, int splits = 1,
            int kchunk = 0, long long c_zstride = 0, int kupper = 0) {
  if (M <= 0 || N <= 0) return 0;
  if (splits <= 1) { splits = 1; kchunk = std::max(K, 1); }
  const bool tma = K > 0 && al16(A, lda) && al16(B, ldb) && tma_encode_fn() != nullptr;
  if (tma) {
    h->sched[SDC_SCHED_GEMM_TMA]++;
    TmaGemmArgs g{M, N, K, C, ldc, alpha, beta, D2, ldd2, alpha2, kchunk, c_zstride,
                  (int)(al16(C, ldc) && M % 2 == 0), kupper};
    int v = h->gemm_force;
    const bool cok = beta != 0.0 && splits == 1 && al16(C, ldc) && D2 == nullptr;
    if (v < 0) {
      if (M <= 64) v = 1;
      else if (K <= 128) v = 3;
      else if (K <= 256) v = 3;   // short-K update: 2 CTAs/SM overlap epilogue and prologue
      else if ((long long)cdiv(M, 128) * cdiv(N, 128) * splits >= h->num_sms) v = 0;
      else v = 2;
    }
    if (v == 4 && !cok) v = 0;
    const int pm = h->persist_mode;
    // On the look-ahead side stream the short-K updates use one-tile CTAs: a persistent grid
    // would hold every SM until the whole update finished, and the critical chain's kernels
    // (panels, next-block updates, reductions) on the high-priority stream would queue
    // behind it; one-tile CTAs retire continuously, so the scheduler can hand SMs to them.
    if (v == 3 && (h->on_side || h->two_chains) && !h->side_persist) {
      if (h->red_mode && beta == 1.0 && D2 == nullptr && g.red_ok)
        return launch_tma_t<TmaR>(h, A, lda, B, ldb, g, splits);
      return launch_tma_t<TmaU>(h, A, lda, B, ldb, g, splits);
    }
    if (pm == 2 || (pm == 1 && v == 3)) {
      switch (v) {
        case 0: return launch_tma_persist<TmaL>(h, A, lda, B, ldb, g, splits);
        case 1: return launch_tma_persist<TmaM>(h, A, lda, B, ldb, g, splits);
        case 2: return launch_tma_persist<TmaS>(h, A, lda, B, ldb, g, splits);
        case 3:
          if (h->red_mode && beta == 1.0 && D2 == nullptr && g.red_ok)
            return launch_tma_persist<TmaR>(h, A, lda, B, ldb, g, splits);
          return launch_tma_persist<TmaU>(h, A, lda, B, ldb, g, splits);
        default: break;
      }
    }
    switch (v) {
      case 0: return launch_tma_t<TmaL>(h, A, lda, B, ldb, g, splits);
      case 1: return launch_tma_t<TmaM>(h, A, lda, B, ldb, g, splits);
      case 2: return launch_tma_t<TmaS>(h, A, lda, B, ldb, g, splits);
      case 4: return launch_tma_t<TmaC>(h, A, lda, B, ldb, g, splits);
      default: return launch_tma_t<TmaU>(h, A, lda, B, ldb, g, splits);
    }
  }
  GemmArgs g{M, N, K, A, lda, B, ldb, C, ldc, alpha, beta, D2, ldd2, alpha2, kchunk, c_zstride};
  h->sched[SDC_SCHED_GEMM_CPASYNC]++;   // operands not 16-byte aligned: cp.async staging
  return launch_gemm_tile<true, false>(h, g, splits);
}

// general op(A) op(B) (test entry point sdc_dgemm only; the step itself is all-TN)
int gemm_general(sdc_handle* h, bool ta, bool tb, int M, int N, int K, double alpha,
                 const double* A, long long lda, const double* B, long long ldb, double beta,
                 double* C, long long ldc) {
  if (M <= 0 || N <= 0) return 0;
  if (ta && !tb) return gemm_tn(h, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
  GemmArgs g{M, N, K, A, lda, B, ldb, C, ldc, alpha, beta, nullptr, 0, 0.0, std::max(K, 1), 0};
  if (!ta && !tb) return launch_gemm_tile<false, false>(h, g, 1);
  if (!ta && tb) return launch_gemm_tile<false, true>(h, g, 1);
  return launch_gemm_tile<true, true>(h, g, 1);
}

// split-K factor for a tall-K GEMM with `tiles` output tiles: at least ~2 waves of CTAs,
// K slices >= 256, and the fewest splits whose last wave is >= 90% full (wave quantisation)
int pick_splits(sdc_handle* h, int tiles, int K, long long cap) {
  const int smax = (int)std::max(1LL, std::min<long long>(std::min(K / h->split_kmin, 64), cap));
  const int P = h->num_sms;
  int best = 1;
  double best_eff = 0.0;
  for (int s = 1; s <= smax; ++s) {
    const long long ctas = (long long)tiles * s;
    const long long waves = (ctas + P - 1) / P;
    const double eff = (double)ctas / (double)(waves * P);
    if (ctas >= 2LL * P && eff >= 0.9) return s;
    if (eff > best_eff + 1e-9 || (ctas < 2LL * P && s == smax)) { best_eff = eff; best = s; }
  }
  return best;
}

// ---------------------------------------------------------------------------------------
// Householder factors of a blocked QR of an m x n matrix: explicit Y (m x n, ld ldy) and
// its transpose Yt (n x m, ld ldyt), T blocks in h->Tb.  Y(i0:, i0:i0+nb) is panel i0.
// ---------------------------------------------------------------------------------------
struct Fac {
  double* Y; long long ldy;
  double* Yt; long long ldyt;
  const double* Yp(int i0) const { return Y + i0 + (long long)i0 * ldy; }
  const double* Ytp(int i0) const { return Yt + i0 + (long long)i0 * ldyt; }
};

// ---------------------------------------------------------------------------------------
// compact-WY application:  C (m x ncols) <- (I - Y op(T) Y^T) C,
//   trans = 1: op(T) = T^T  (H_{nb-1}..H_0 C, i.e. Q^T C)
//   trans = 0: op(T) = T    (H_0..H_{nb-1} C, i.e. Q C)
// W0 = Y^T C (split-K TN GEMM) -> W = op(T) W0 (k_wy_reduce) -> C -= (Y^T)^T W (TN GEMM)
// ---------------------------------------------------------------------------------------
int wy_apply(sdc_handle* h, int trans, int m, int ncols, const double* Y, long long ldy,
             const double* Yt, long long ldyt, const double* T, int nb, double* C, long long ldc) {
  if (m <= 0 || ncols <= 0) return 0;
  const int tilesN = cdiv(ncols, 128);
  int splits = std::max(1, std::min(cdiv(2 * h->num_sms, tilesN), std::max(1, m / h->split_kmin)));
  int kchunk = cdiv(cdiv(m, splits), 16) * 16;
  splits = cdiv(m, kchunk);
  if ((size_t)splits * nb * ncols > h->wp_elems) {
    set_err("wy_apply: split-K workspace too small");
    return SDC_ERR_CUDA;
  }
  h->gemm_sub = SDC_PROF_GEMM_W0;
  int rc0 = gemm_tn(h, nb, ncols, m, 1.0, Y, ldy, C, ldc, 0.0, h->Wp, nb, nullptr, 0, 0.0, splits,
                    kchunk, (long long)nb * ncols);
  h->gemm_sub = SDC_PROF_GEMM_OTHER;
  SDC_TRY(rc0);
  {
    ProfScope ps(h, SDC_PROF_WYRED, 8.0 * ((double)splits * nb * ncols + (double)nb * ncols));
    const int cpb = std::max(1, std::min(WYR_COLS, ncols / (2 * h->num_sms)));
    k_wy_reduce<<<cdiv(ncols, cpb), 256, 0, h->st>>>(h->Wp, splits, (long long)nb * ncols, nb, ncols,
                                                     T, trans, h->W, cpb);
    SDC_LAUNCHED(h);
  }
  h->gemm_sub = SDC_PROF_GEMM_UPD;
  int rc1 = gemm_tn(h, m, ncols, nb, -1.0, Yt, ldyt, h->W, nb, 1.0, C, ldc);
  h->gemm_sub = SDC_PROF_GEMM_OTHER;
  return rc1;
}

// ---------------------------------------------------------------------------------------
// panel (cooperative) and blocked QR
// ---------------------------------------------------------------------------------------
// panel kernel instance: cluster or grid exchange x register (RPT rows/thread) or smem column loop
const void* panel_fn(bool cluster, int rpt) {
  if (cluster) {
    switch (rpt) {
      case 8: return (const void*)panel_qr_kernel_t<true, 8>;
      case 16: return (const void*)panel_qr_kernel_t<true, 16>;
      case 32: return (const void*)panel_qr_kernel_t<true, 32>;
      default: return (const void*)panel_qr_kernel_t<true, 0>;
    }
  }
  switch (rpt) {
    case 8: return (const void*)panel_qr_kernel_t<false, 8>;
    case 16: return (const void*)panel_qr_kernel_t<false, 16>;
    case 32: return (const void*)panel_qr_kernel_t<false, 32>;
    default: return (const void*)panel_qr_kernel_t<false, 0>;
  }
}
inline int rpt_slot(int rpt) { return rpt == 8 ? 1 : rpt == 16 ? 2 : rpt == 32 ? 3 : 0; }
// dynamic shared memory currently allowed per (device, exchange mode, RPT variant) of the panel
// kernel (the attribute is per device; sdc_create re-sets the cluster RPT=0 entry it probes)
size_t g_panel_attr[MAX_DEV][2][4] = {};
std::mutex g_panel_mu;   // the limits only grow, under this lock (handles on several host threads)

// The CholeskyQR2 panel as six small kernels (cqr_split.cuh): wide, bandwidth-trivial stages
// on m/256 CTAs and the serial 64 x 64 chains on one CTA, so a tall panel that runs next to the
// bulk trailing update holds one SM instead of 120 for most of its ~200 us.
int panel_split(sdc_handle* h, double* P, long long ldp, int m, double* Y, long long ldy, double* Yt,
                long long ldyt, double* T, double* tau, int zero_above) {
  static DevOnce attr;
  if (!attr.has(h->device)) {
    SDC_CK(cudaFuncSetAttribute(k_cqs_gram, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CQS_WIDE_SMEM));
    SDC_CK(cudaFuncSetAttribute(k_cqs_q1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CQS_WIDE_SMEM));
    SDC_CK(cudaFuncSetAttribute(k_cqs_y, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CQS_WIDE_SMEM));
    SDC_CK(cudaFuncSetAttribute(k_cqs_mid1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CQS_MID_SMEM));
    SDC_CK(cudaFuncSetAttribute(k_cqs_mid2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CQS_MID_SMEM));
    attr.set(h->device);
  }
  const int G = cdiv(m, CQS_ROWS);
  CqsArgs a{P, ldp, m, Y, ldy, Yt, ldyt, T, tau, zero_above, h->cqs, h->cqs_sync};
  ProfScope ps(h, SDC_PROF_PANEL, 8.0 * 4.0 * m * NB);
  k_cqs_gram<<<G, 512, CQS_WIDE_SMEM, h->st>>>(a);
  k_cqs_mid1<<<CQS_MIDS, 512, CQS_MID_SMEM, h->st>>>(a, G);
  k_cqs_q1<<<G, 512, CQS_WIDE_SMEM, h->st>>>(a);
  k_cqs_mid2<<<CQS_MIDS, 512, CQS_MID_SMEM, h->st>>>(a, G);
  k_cqs_y<<<G, 512, CQS_WIDE_SMEM, h->st>>>(a);
  k_cqs_fallback<<<1, BQ_THREADS, CQS_FB_SMEM, h->st>>>(a);
  SDC_CK(cudaGetLastError());
  h->launches += 6;
  h->sched[SDC_SCHED_PANEL_CQ_SPLIT]++;
  return 0;
}

int panel(sdc_handle* h, double* P, long long ldp, int m, int nb, double* Y, long long ldy,
          double* Yt, long long ldyt, double* T, double* tau, int zero_above) {
  if (nb == NB && h->cqs && m <= CQS_GMAX * CQS_ROWS &&
      (h->cq_split == 2 ? m >= 128
                        : (h->cq_split == 1 && h->cq_split_ctx &&
                           m > (h->share_sms ? std::min(h->cq_split_rows, h->cq_split_rows_shared) : h->cq_split_rows))))
    return panel_split(h, P, ldp, m, Y, ldy, Yt, ldyt, T, tau, zero_above);
  // one cluster of <= 16 CTAs when the panel fits (DSMEM exchange); taller panels: several
  // 16-CTA clusters with a two-level exchange (DSMEM inside, L2 between cluster leaders);
  // otherwise a cooperative grid exchanging through L2
  bool cluster = h->cluster_ok && m <= h->cluster_max_rows;
  int csize = 1, G;
  if (cluster) {
    G = std::min(16, std::max(1, cdiv(m, h->panel_rows)));
  } else if (h->mcluster_ok) {
    // The clusters of a multi-cluster panel spin on each other's L2 flags, so all of them
    // must become resident.  When both factorization contexts can issue such panels at the
    // same time (pencil chains, pipelined monitor mode), each panel takes at most half the
    // clusters that fit the GPU: two partly resident panels can then never wait on each
    // other (VERDICT r01 weak 8 / ADVICE r01).
    const int cap = h->share_sms ? std::max(2, h->max_clusters16 / 2) : h->max_clusters16;
    const int want = cdiv(m, 16 * h->panel_rows);
    int ncl = std::max(2, std::min(cap, want));
    int cs = 16;
    if (h->share_sms && want > cap) h->sched[SDC_SCHED_PANEL_MCLUSTER_CAPPED]++;
    // 16-CTA clusters tile the GPCs unevenly (7 fit on 148 SMs): when that leaves more than
    // 256 rows per CTA -- the shared-memory column loop instead of registers -- use 8-CTA
    // clusters (more of them fit; the L2 exchange takes up to 16 cluster leaders)
    if (cdiv(m, 16 * ncl) > 256 && h->max_clusters8 >= 4) {
      const int cap8 = std::min(16, h->share_sms ? h->max_clusters8 / 2 : h->max_clusters8);
      const int n8 = std::max(2, std::min(cap8, cdiv(m, 8 * h->panel_rows)));
      if (8 * n8 > 16 * ncl) { ncl = n8; cs = 8; }
    }
    if (panel_smem_bytes(cdiv(m, cs * ncl), h->cqr) <= 227 * 1024) {
      cluster = true;
      csize = cs;
      G = cs * ncl;
    } else {
      G = std::min(h->num_sms, std::max(1, m / h->panel_rows));
    }
  } else {
    G = std::min(h->num_sms, std::max(1, m / h->panel_rows));
  }
  int rows_per = cdiv(m, G);
  if (rows_per < nb) {
    rows_per = nb;
    G = cdiv(m, rows_per);
    if (csize > 1) { cluster = false; csize = 1; G = std::min(G, h->num_sms); rows_per = cdiv(m, G); }
  }
  if (cluster && csize == 1) csize = G;
  size_t smem = panel_smem_bytes(rows_per, h->cqr);
  const int rpt = h->panel_reg ? panel_rpt(rows_per) : 0;
  const void* fn = panel_fn(cluster, rpt);
  {
    // several handles may run on several host threads (thread-ranks of the recursion): the
    // limit only ever grows, under a lock, so no thread lowers it below another's launch
    std::lock_guard<std::mutex> lk(g_panel_mu);
    size_t& cur = g_panel_attr[h->device & (MAX_DEV - 1)][cluster][rpt_slot(rpt)];
    if (smem > cur) {
      cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) {
        set_err("panel: %d rows per CTA need %zu B of shared memory (n too large): %s", rows_per,
                smem, cudaGetErrorString(e));
        return SDC_ERR_NOT_SUPPORTED;
      }
      cur = smem;
    }
  }
  // CholeskyQR2 first (register variants in cluster mode, full-width panels), Householder on
  // breakdown (cqr.cuh)
  // CholeskyQR2 pays off on TALL panels, where the Householder loop's per-column exchange
  // crosses several clusters (measured: 228 vs 309 us per panel at 32768 rows, 175 vs 212 us at
  // 16384, even at 8192, slower below): default for multi-cluster panels above 8192 rows
  const bool cqr_here = h->cqr_mode == 2 || (h->cqr_mode == 1 && G > csize && m > 8192);
  const int use_cqr = cqr_here && cluster && nb == NB && G <= CQ_GMAX ? 1 : 0;
  if (getenv("SDC_DEBUG_PANEL"))
    fprintf(stderr, "panel m=%d nb=%d G=%d csize=%d rows_per=%d rpt=%d cluster=%d use_cqr=%d cqr=%d\n", m, nb, G,
            csize, rows_per, rpt, (int)cluster, use_cqr, (int)h->cqr);
  PanelArgs a{P, ldp, m, nb, Y, ldy, Yt, ldyt, T, tau, h->gbuf, h->bar, (unsigned)h->bar_count,
              rows_per, h->dbg_on ? h->dbg : nullptr, zero_above, csize, h->llbuf, h->ll_epoch,
              h->cqbuf, use_cqr, h->cqstat};
  ProfScope ps(h, SDC_PROF_PANEL, 8.0 * 4.0 * m * nb);   // read panel, write panel + Y + Y^T
  if (cluster) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(PANEL_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = h->st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = csize;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    void* args[] = {&a};
    SDC_CK(cudaLaunchKernelExC(&cfg, fn, args));
    if (G > csize || use_cqr) h->ll_epoch += nb;
    if (use_cqr) h->sched[SDC_SCHED_PANEL_CQR_TRIED]++;
    h->sched[G > csize ? SDC_SCHED_PANEL_MCLUSTER : SDC_SCHED_PANEL_CLUSTER]++;
    if (G > csize && csize == 8) h->sched[SDC_SCHED_PANEL_MCLUSTER8]++;
  } else {
    void* args[] = {&a};
    SDC_CK(cudaLaunchCooperativeKernel(fn, dim3(G),
                                       dim3(PANEL_THREADS), args, smem, h->st));
    h->bar_count += (unsigned long long)G * nb;
    h->sched[SDC_SCHED_PANEL_GRID]++;
  }
  h->launches++;
  return 0;
}

inline double* Tblk(sdc_handle* h, int i0) { return h->Tb + (size_t)(i0 / NB) * NB * NB; }
inline double* TOblk(sdc_handle* h, int I0) { return h->Tob + (size_t)(I0 / h->nbo) * h->nbo * h->nbo; }
inline double* TOtblk(sdc_handle* h, int I0) { return h->Tobt + (size_t)(I0 / h->nbo) * h->nbo * h->nbo; }

// Outer compact-WY factor of the nbo columns starting at I0 (rows I0..m-1):
// T_O from the inner 64-wide T blocks and G = Y_O^T Y_O by a merge tree.
int build_tout(sdc_handle* h, int m, int I0, int nbo, const Fac& f) {
  double* TO = TOblk(h, I0);
  double* TOt = TOtblk(h, I0);
  k_tout_place<<<cdiv((long long)nbo * nbo, 256), 256, 0, h->st>>>(TO, TOt, nbo, Tblk(h, I0));
  SDC_LAUNCHED(h);
  if (nbo <= NB) return 0;
  const int rows = m - I0;
  // G = Y_O^T Y_O (split-K TN GEMM + fixed-order sum)
  int splits = std::max(1, std::min(cdiv(2 * h->num_sms, cdiv(nbo, 128) * cdiv(nbo, 128)),
                                    std::max(1, rows / h->split_kmin)));
  int kchunk = cdiv(cdiv(rows, splits), 16) * 16;
  splits = cdiv(rows, kchunk);
  if ((size_t)splits * nbo * nbo > h->wp_elems) { set_err("build_tout: workspace"); return SDC_ERR_CUDA; }
  SDC_TRY(gemm_tn(h, nbo, nbo, rows, 1.0, f.Yp(I0), f.ldy, f.Yp(I0), f.ldy, 0.0, h->Wp, nbo, nullptr,
                  0, 0.0, splits, kchunk, (long long)nbo * nbo));
  k_sum_partials<<<cdiv((long long)nbo * nbo, 256), 256, 0, h->st>>>(h->Wp, splits, (long long)nbo * nbo,
                                                                    (long long)nbo * nbo, h->Gb);
  SDC_LAUNCHED(h);
  for (int s = NB; s < nbo; s *= 2)
    for (int a0 = 0; a0 + s < nbo; a0 += 2 * s) {
      const int p = s, q = std::min(s, nbo - a0 - s);
      k_tmerge<<<dim3(cdiv(p, 32), cdiv(q, 32)), 256, 0, h->st>>>(TO, TOt, nbo, h->Gb, a0, p, a0 + s, q);
      SDC_LAUNCHED(h);
    }
  return 0;
}

// C (m x ncols) <- (I - Y_O op(T_O) Y_O^T) C for the outer block at I0 (rows I0.. of the
// factored matrix = rows 0.. of C):  Z = Y_O^T C (split-K), W = op(T_O) Z, C -= Y_O W.
int wy_apply_outer(sdc_handle* h, int trans, int I0, int nbo, int m, int ncols, const Fac& f,
                   double* C, long long ldc) {
  if (nbo <= NB) return wy_apply(h, trans, m, ncols, f.Yp(I0), f.ldy, f.Ytp(I0), f.ldyt, Tblk(h, I0),
                                 nbo, C, ldc);
  if (m <= 0 || ncols <= 0) return 0;
  const int tilesMN = cdiv(nbo, 128) * cdiv(ncols, 128);
  int splits = pick_splits(h, tilesMN, m, (long long)(h->wp_elems / ((size_t)nbo * ncols)));
  int kchunk = cdiv(cdiv(m, splits), 16) * 16;
  splits = cdiv(m, kchunk);
  if ((size_t)splits * nbo * ncols > h->wp_elems) { set_err("wy_apply_outer: workspace"); return SDC_ERR_CUDA; }
  h->gemm_sub = SDC_PROF_GEMM_W0;
  int rc0 = gemm_tn(h, nbo, ncols, m, 1.0, f.Yp(I0), f.ldy, C, ldc, 0.0, h->Wp, nbo, nullptr, 0, 0.0,
                    splits, kchunk, (long long)nbo * ncols);
  h->gemm_sub = SDC_PROF_GEMM_OTHER;
  SDC_TRY(rc0);
  const double* Z = h->Wp;
  if (splits > 1) {
    ProfScope ps(h, SDC_PROF_WYRED, 8.0 * ((double)splits + 1) * nbo * ncols);
    k_sum_partials<<<std::min(cdiv((long long)nbo * ncols, 256), 148 * 8), 256, 0, h->st>>>(
        h->Wp, splits, (long long)nbo * ncols, (long long)nbo * ncols, h->Zb);
    SDC_LAUNCHED(h);
    Z = h->Zb;
  }
  // W = T_O^T Z (trans) or T_O Z: TN with A_s = T_O or T_O^T (both stored)
  SDC_TRY(gemm_tn(h, nbo, ncols, nbo, 1.0, trans ? TOblk(h, I0) : TOtblk(h, I0), nbo, Z, nbo, 0.0,
                  h->W, nbo));
  h->gemm_sub = SDC_PROF_GEMM_UPD;
  int rc1 = gemm_tn(h, m, ncols, nbo, -1.0, f.Ytp(I0), f.ldyt, h->W, nbo, 1.0, C, ldc);
  h->gemm_sub = SDC_PROF_GEMM_OTHER;
  return rc1;
}

// outer block width for an order-n step (measured): 64 up to n = 1024 (single-level
// blocking: no T merges or nested updates between panels; 6% faster than 256 at n = 1024),
// 128 up to n = 4096 / 8192 (1-2% faster than 256, 15% faster than 64 at n = 4096), the
// full 256 above (rank-256 updates run closer to the DMMA peak at n = 16384).
// Two concurrent chains (Alg. 4 pencils) keep 256 above n = 4096 (1.4% faster at n = 8192
// than 128); a single chain uses 128 up to n = 8192 (2% faster than 256 there).
inline void choose_nbo(sdc_handle* h, int n, bool two_chains = false) {
  const int lim128 = two_chains ? 4096 : 8192;
  if (h->nbo_fixed || n > lim128) h->nbo = h->nbo_max;
  else h->nbo = std::min(h->nbo_max, n <= 1024 ? 64 : 128);
}

inline bool lookahead_qr(const sdc_handle* h, int n) {
  return h->lookahead && h->st_hi && h->nbo > NB && n > 2 * h->nbo;
}

// panels + inner WY updates + T_O of the outer block at I0 (columns I0..I0+nbo-1 only)
int factor_block(sdc_handle* h, double* A, long long lda, int m, int n, int I0, int nbo, const Fac& f) {
  for (int i0 = I0; i0 < I0 + nbo; i0 += NB) {
    const int nbp = std::min(NB, I0 + nbo - i0);
    SDC_TRY(panel(h, A + i0 + (long long)i0 * lda, lda, m - i0, nbp, f.Y + i0 + (long long)i0 * f.ldy,
                  f.ldy, f.Yt + i0 + (long long)i0 * f.ldyt, f.ldyt, Tblk(h, i0), h->tau + i0, i0 - I0));
    const int rest = I0 + nbo - (i0 + nbp);
    if (rest > 0)
      SDC_TRY(wy_apply(h, 1, m - i0, rest, f.Yp(i0), f.ldy, f.Ytp(i0), f.ldyt, Tblk(h, i0), nbp,
                       A + i0 + (long long)(i0 + nbp) * lda, lda));
  }
  return build_tout(h, m, I0, nbo, f);
}

// Look-ahead (depth 1) schedule of the two-level QR.  The critical chain -- panels, inner
// updates, T_O, and the trailing update of the NEXT outer block's nbo columns -- runs on
// the high-priority handle stream st_hi; the bulk trailing update of the remaining columns
// runs on the caller's stream (own workspace) and overlaps the next block's panels, which
// occupy only the panel kernel's clusters.  Same arithmetic as the serial order, per column
// block; the split-K slicing of the bulk update differs (rounding-level only).
struct LaScope {   // restores the caller's stream and the primary workspace on every exit
  sdc_handle* h; cudaStream_t side;
  explicit LaScope(sdc_handle* h_) : h(h_), side(h_->st) {}
  void use_side(bool on) {
    h->st = on ? side : h->st_hi;
    h->on_side = on;
    if ((h->Wp2 != nullptr) && on != swapped) {
      std::swap(h->Wp, h->Wp2); std::swap(h->W, h->W2); std::swap(h->Zb, h->Zb2);
      swapped = on;
    }
  }
  bool swapped = false;
  ~LaScope() {
    if (swapped) { std::swap(h->Wp, h->Wp2); std::swap(h->W, h->W2); std::swap(h->Zb, h->Zb2); }
    h->st = side;
    h->on_side = false;
  }
};

int blocked_qr_lookahead(sdc_handle* h, double* A, long long lda, int m, int n, const Fac& f) {
  LaScope la(h);
  bool pendingB = false;
  if (h->xpass_pending) {   // fork point and pending bulk columns left by the previous IRS pass
    h->xpass_pending = false;
    pendingB = true;
  } else {
    SDC_CK(cudaEventRecord(h->la_fork, la.side));
  }
  h->sched[pendingB ? SDC_SCHED_XPASS_FORKS : SDC_SCHED_LOOKAHEAD_FORKS]++;
  SDC_CK(cudaStreamWaitEvent(h->st_hi, h->la_fork, 0));
  la.use_side(false);
  for (int I0 = 0; I0 < n; I0 += h->nbo) {
    const int nbo = std::min(h->nbo, n - I0);
    SDC_TRY(factor_block(h, A, lda, m, n, I0, nbo, f));
    const int c1 = I0 + nbo, rem = n - c1;
    if (rem <= 0) break;
    const int na = std::min(h->nbo, rem);
    if (rem > na) SDC_CK(cudaEventRecord(h->la_fac, h->st_hi));
    if (pendingB) SDC_CK(cudaStreamWaitEvent(h->st_hi, h->la_B, 0));
    SDC_TRY(wy_apply_outer(h, 1, I0, nbo, m - I0, na, f, A + I0 + (long long)c1 * lda, lda));
    if (rem > na) {
      la.use_side(true);
      SDC_CK(cudaStreamWaitEvent(la.side, h->la_fac, 0));
      SDC_TRY(wy_apply_outer(h, 1, I0, nbo, m - I0, rem - na, f, A + I0 + (long long)(c1 + na) * lda, lda));
      SDC_CK(cudaEventRecord(h->la_B, la.side));
      la.use_side(false);
      pendingB = true;
    }
  }
  SDC_CK(cudaEventRecord(h->la_join, h->st_hi));
  SDC_CK(cudaStreamWaitEvent(la.side, h->la_join, 0));
  return 0;
}

// A (m x n, m >= n) <- Householder QR in place, two-level: 64-wide cooperative panels inside
// nbo-wide outer blocks (inner WY updates restricted to the block), then one rank-nbo
// trailing update per outer block.  Factors into f, T blocks into h->Tb / h->Tob.
int blocked_qr(sdc_handle* h, double* A, long long lda, int m, int n, const Fac& f) {
  Nvtx nv("blocked_qr");
  if (lookahead_qr(h, n)) return blocked_qr_lookahead(h, A, lda, m, n, f);
  h->xpass_pending = false;
  for (int I0 = 0; I0 < n; I0 += h->nbo) {
    const int nbo = std::min(h->nbo, n - I0);
    for (int i0 = I0; i0 < I0 + nbo; i0 += NB) {
      const int nbp = std::min(NB, I0 + nbo - i0);
      SDC_TRY(panel(h, A + i0 + (long long)i0 * lda, lda, m - i0, nbp, f.Y + i0 + (long long)i0 * f.ldy,
                    f.ldy, f.Yt + i0 + (long long)i0 * f.ldyt, f.ldyt, Tblk(h, i0), h->tau + i0,
                    i0 - I0));
      const int rest = (nbo > NB ? I0 + nbo : n) - (i0 + nbp);   // columns the inner WY updates
      if (rest > 0)
        SDC_TRY(wy_apply(h, 1, m - i0, rest, f.Yp(i0), f.ldy, f.Ytp(i0), f.ldyt, Tblk(h, i0), nbp,
                         A + i0 + (long long)(i0 + nbp) * lda, lda));
    }
    if (nbo > NB) {
      SDC_TRY(build_tout(h, m, I0, nbo, f));
      if (I0 + nbo < n)
        SDC_TRY(wy_apply_outer(h, 1, I0, nbo, m - I0, n - I0 - nbo, f, A + I0 + (long long)(I0 + nbo) * lda,
                               lda));
    }
  }
  return 0;
}

// C (m x ncols) <- Q^T C  (forward over outer blocks) for the last blocked_qr of an m x n matrix
int apply_qt(sdc_handle* h, int m, int n, const Fac& f, double* C, long long ldc, int ncols) {
  for (int I0 = 0; I0 < n; I0 += h->nbo) {
    const int nbo = std::min(h->nbo, n - I0);
    SDC_TRY(wy_apply_outer(h, 1, I0, nbo, m - I0, ncols, f, C + I0, ldc));
  }
  return 0;
}

// C (m x ncols) <- Q C  (backward over outer blocks)
int apply_q(sdc_handle* h, int m, int n, const Fac& f, double* C, long long ldc, int ncols) {
  const int last = ((n - 1) / h->nbo) * h->nbo;
  for (int I0 = last; I0 >= 0; I0 -= h->nbo) {
    const int nbo = std::min(h->nbo, n - I0);
    SDC_TRY(wy_apply_outer(h, 0, I0, nbo, m - I0, ncols, f, C + I0, ldc));
  }
  return 0;
}

// explicit square Q (n x n) = H_0..H_{n-1} (dorgqr order: only the trailing block changes)
int form_q(sdc_handle* h, int n, const Fac& f, double* Q, long long ldq) {
  k_set_identity<<<ew_grid((long long)n * n), 256, 0, h->st>>>(Q, ldq, n, n, 1.0);
  SDC_LAUNCHED(h);
  const int last = ((n - 1) / h->nbo) * h->nbo;
  for (int I0 = last; I0 >= 0; I0 -= h->nbo) {
    const int nbo = std::min(h->nbo, n - I0);
    SDC_TRY(wy_apply_outer(h, 0, I0, nbo, n - I0, n - I0, f, Q + I0 + (long long)I0 * ldq, ldq));
  }
  return 0;
}

int transpose_rev(sdc_handle* h, double* out, long long ldo, const double* src, long long lds,
                  int n, int mode) {
  dim3 grid(cdiv(n, 32), cdiv(n, 32));
  k_transpose_rev<<<grid, dim3(32, 8), 0, h->st>>>(out, ldo, src, lds, n, mode);
  SDC_LAUNCHED(h);
  return 0;
}

int norms(sdc_handle* h, const double* X, long long ldx, int n, double* out2) {
  k_colnorms<<<cdiv((long long)n * 32, 256), 256, 0, h->st>>>(X, ldx, n, n, h->vec, h->vec + h->n_max);
  SDC_LAUNCHED(h);
  k_norm_finish<<<1, 1024, 0, h->st>>>(h->vec, h->vec + h->n_max, n, out2);
  SDC_LAUNCHED(h);
  return 0;
}

Fac fac_stack(sdc_handle* h, int n) { return Fac{h->Y, 2LL * n, h->Yt, wld(n)}; }
Fac fac_square(sdc_handle* h, int n) { return Fac{h->Y, wld(n), h->Yt, wld(n)}; }

// ---------------------------------------------------------------------------------------
// one IRS pass: S holds [B_j; -A_j]; writes A_{j+1}, B_{j+1} and the next stack into S
// ---------------------------------------------------------------------------------------
int irs_pass(sdc_handle* h, int n, const double* Aj, long long lda, const double* Bj,
             long long ldb, double* An, long long ldan, double* Bn, long long ldbn, double* S,
             int rtest_slot, double* Rout, long long ldr, bool xpass = false) {
  Nvtx nv("irs_pass (Alg. 3 l.3)");
  const long long m = 2LL * n;
  const Fac f = fac_stack(h, n);
  {
    // the stack [B_j; -A_j] has full column rank (R_j = chol(A_j^T A_j + B_j^T B_j)): its tall
    // panels may run as the split CholeskyQR2 chain (GRURV's operands are rank-deficient by
    // construction and keep the cluster kernel with its in-kernel Householder fallback)
    struct SplitCtx {
      sdc_handle* h; bool prev;
      explicit SplitCtx(sdc_handle* h_) : h(h_), prev(h_->cq_split_ctx) { h->cq_split_ctx = true; }
      ~SplitCtx() { h->cq_split_ctx = prev; }
    } sctx(h);
    SDC_TRY(blocked_qr(h, S, m, (int)m, n, f));
  }
  if (rtest_slot >= 0) {
    k_rtest_cols<<<cdiv((long long)n * 32, 256), 256, 0, h->st>>>(S, m, h->Rprev, n, h->vec,
                                                                  h->vec + h->n_max);
    SDC_LAUNCHED(h);
    k_rtest_finish<<<1, 1024, 0, h->st>>>(h->vec, h->vec + h->n_max, n,
                                          h->scal + SCAL_HIST + rtest_slot);
    SDC_LAUNCHED(h);
  }
  if (Rout) {   // R with non-negative diagonal (test entry point)
    SDC_CK(cudaMemsetAsync(h->Rprev, 0, sizeof(double) * (size_t)n * n, h->st));
    k_rtest_cols<<<cdiv((long long)n * 32, 256), 256, 0, h->st>>>(S, m, h->Rprev, n, h->vec,
                                                                  h->vec + h->n_max);
    SDC_LAUNCHED(h);
    k_copy<<<ew_grid((long long)n * n), 256, 0, h->st>>>(Rout, ldr, h->Rprev, n, n, n, 1.0);
    SDC_LAUNCHED(h);
  }
  // complement [Q12; Q22] = H_0..H_{n-1} [0; I]
  k_set_zero_identity<<<ew_grid(m * n), 256, 0, h->st>>>(h->C, m, n);
  SDC_LAUNCHED(h);
  SDC_TRY(apply_q(h, (int)m, n, f, h->C, m, n));
  // A_{j+1} = Q12^T A_j (-> next stack lower half, negated); B_{j+1} = Q22^T B_j (upper).
  // Cross-pass look-ahead (xpass: the next operation of this context is pass j+1's QR):
  // the first nbo columns of the next stack are formed first, the fork point of pass j+1's
  // look-ahead QR is recorded there, and the remaining columns follow as that QR's pending
  // "bulk update" -- so pass j+1's first block of panels overlaps this pass's products.
  const bool xp = xpass && lookahead_qr(h, n);
  const int w = xp ? h->nbo : n;
  const bool bid = Bj != nullptr && Bj == h->b_ident;   // B_j = rho I (first RNEP pass)
  if (bid) {                                            // B_{j+1} = rho Q22^T (all columns)
    h->b_ident = nullptr;
    dim3 grid(cdiv(n, 32), cdiv(n, 32));
    k_transpose_scale2<<<grid, dim3(32, 8), 0, h->st>>>(Bn, ldbn, S, m, h->C + n, m, n, h->b_ident_rho);
    SDC_LAUNCHED(h);
  }
  for (int part = 0; part < (xp ? 2 : 1); ++part) {
    const int c0 = part == 0 ? 0 : w, nc = part == 0 ? w : n - w;
    SDC_TRY(gemm_tn(h, n, nc, n, 1.0, h->C, m, Aj + (long long)c0 * lda, lda, 0.0, An + (long long)c0 * ldan,
                    ldan, S + n + (long long)c0 * m, m, -1.0));
    if (!bid)
      SDC_TRY(gemm_tn(h, n, nc, n, 1.0, h->C + n, m, Bj + (long long)c0 * ldb, ldb, 0.0,
                      Bn + (long long)c0 * ldbn, ldbn, S + (long long)c0 * m, m, 1.0));
    if (xp && part == 0) SDC_CK(cudaEventRecord(h->la_fork, h->st));
  }
  if (xp) {
    SDC_CK(cudaEventRecord(h->la_B, h->st));
    h->xpass_pending = true;
  }
  return 0;
}

// Q = GRURV(2, A_p+B_p, A_p; -1, +1)   (Alg. 2 with Alg. 1)
// Vt = V^T (prepared once per split).
int grurv_right(sdc_handle* h, int n, const double* Ap, const double* Bp, const double* Vt,
                double* Q, long long ldq) {
  Nvtx nv("grurv_right (Alg. 1/2)");
  const long long ld = wld(n);
  const Fac f = fac_square(h, n);
  k_add<<<ew_grid((long long)n * n), 256, 0, h->st>>>(h->G1, ld, Ap, ld, Bp, ld, n, n);
  SDC_LAUNCHED(h);                                                     // S = A_p + B_p
  SDC_TRY(transpose_rev(h, h->G3, ld, Ap, ld, n, 0));                  // A_p^T
  SDC_TRY(gemm_tn(h, n, n, n, 1.0, h->G3, ld, Vt, ld, 0.0, h->G2, ld)); // X = A_p V^T
  SDC_TRY(blocked_qr(h, h->G2, ld, n, n, f));                          // X = U R_2
  SDC_TRY(apply_qt(h, n, n, f, h->G1, ld, n));                         // U^T S
  k_row_sign<<<ew_grid((long long)n * n), 256, 0, h->st>>>(h->G1, ld, h->G2, ld, n, n);
  SDC_LAUNCHED(h);                                                     // U <- U D_U
  SDC_TRY(transpose_rev(h, h->G3, ld, h->G1, ld, n, 1));               // M = C^T J
  SDC_TRY(blocked_qr(h, h->G3, ld, n, n, f));                          // M = Q_qr R_qr
  SDC_TRY(form_q(h, n, f, h->G1, ld));                                 // Q_qr explicit
  k_col_sign_rev<<<ew_grid((long long)n * n), 256, 0, h->st>>>(Q, ldq, h->G1, ld, h->G3, ld, n, 1);
  SDC_LAUNCHED(h);                                                     // Q = Q_qr D J
  return 0;
}

// Q_L = GRURV(2, A'_p^T, (A'_p+B'_p)^T; +1, -1)  (Alg. 4 line 4); VLt = V_L^T
int grurv_left(sdc_handle* h, int n, const double* Ap, const double* Bp, const double* VLt,
               double* QL, long long ldq) {
  Nvtx nv("grurv_left (Alg. 4 l.4)");
  const long long ld = wld(n);
  const Fac f = fac_square(h, n);
  k_add<<<ew_grid((long long)n * n), 256, 0, h->st>>>(h->G1, ld, Ap, ld, Bp, ld, n, n);
  SDC_LAUNCHED(h);
  SDC_TRY(transpose_rev(h, h->G3, ld, h->G1, ld, n, 0));               // (A'+B')^T
  SDC_TRY(gemm_tn(h, n, n, n, 1.0, h->G3, ld, VLt, ld, 0.0, h->G2, ld)); // X' = (A'+B') V_L^T
  SDC_TRY(transpose_rev(h, h->G3, ld, h->G2, ld, n, 2));               // J X' J
  SDC_TRY(blocked_qr(h, h->G3, ld, n, n, f));                          // = Qt Rt  (QL of X')
  SDC_TRY(transpose_rev(h, h->G1, ld, Ap, ld, n, 3));                  // J A'_p
  SDC_TRY(apply_qt(h, n, n, f, h->G1, ld, n));                         // Qt^T J A'_p
  k_row_sign<<<ew_grid((long long)n * n), 256, 0, h->st>>>(h->G1, ld, h->G3, ld, n, n);
  SDC_LAUNCHED(h);                                                     // D Qt^T J A'_p
  SDC_TRY(transpose_rev(h, h->G2, ld, h->G1, ld, n, 1));               // Z = A'^T U
  SDC_TRY(blocked_qr(h, h->G2, ld, n, n, f));
  SDC_TRY(form_q(h, n, f, h->G1, ld));
  k_col_sign_rev<<<ew_grid((long long)n * n), 256, 0, h->st>>>(QL, ldq, h->G1, ld, h->G2, ld, n, 0);
  SDC_LAUNCHED(h);
  return 0;
}

// Cheaper pencil left basis (SDC_FLAG_QL_ORTH): Q_L = Q of QR(A Q_R) with
// diag R >= 0 -- A X spans the left deflating subspace of the outside eigenvalues for every
// leading column block X of Q_R, and QR preserves nested column spans.
int ql_from_aq(sdc_handle* h, int n, const double* A, long long lda, const double* Q, long long ldq,
               double* QL, long long ldql) {
  const long long ld = wld(n);
  const Fac f = fac_square(h, n);
  SDC_TRY(transpose_rev(h, h->G3, ld, A, lda, n, 0));                   // A^T (K-major)
  SDC_TRY(gemm_tn(h, n, n, n, 1.0, h->G3, ld, Q, ldq, 0.0, h->G2, ld));  // W = A Q_R
  SDC_TRY(blocked_qr(h, h->G2, ld, n, n, f));
  SDC_TRY(form_q(h, n, f, QL, ldql));
  k_col_sign<<<ew_grid((long long)n * n), 256, 0, h->st>>>(QL, ldql, n, n, h->G2, ld);
  SDC_LAUNCHED(h);
  return 0;
}

int select_dev(sdc_handle* h, int n, const double* Ah, long long ldah, const double* Bh,
               long long ldbh, const double* nrmA, const double* nrmB, double* sel) {
  const int nblk = cdiv(n, SEL_T);
  ProfScope ps(h, SDC_PROF_SELECT, 8.0 * (double)n * n * (Bh ? 2 : 1));
  k_select_cols<<<nblk, 256, 0, h->st>>>(Ah, ldah, n, h->pmA);
  SDC_LAUNCHED(h);
  if (Bh) {
    k_select_cols<<<nblk, 256, 0, h->st>>>(Bh, ldbh, n, h->pmB);
    SDC_LAUNCHED(h);
  }
  double* mvals = h->vec + 2 * h->n_max;
  k_select_rows<<<cdiv(n, 256), 256, 0, h->st>>>(h->pmA, Bh ? h->pmB : nullptr, n, nblk, nrmA,
                                                 nrmB, mvals);
  SDC_LAUNCHED(h);
  k_select_argmin<<<1, 1024, 0, h->st>>>(mvals, n, sel);
  SDC_LAUNCHED(h);
  return 0;
}

// Ahat = QL^T A Q = (A^T QL)^T Q (+ Bhat), split selection -> scal[4..6]
int similarity_select(sdc_handle* h, int n, const double* A, long long lda, const double* B,
                      long long ldb, const double* Q, long long ldq, const double* QL,
                      long long ldql) {
  Nvtx nv("similarity + split selection");
  const long long ld = wld(n);
  SDC_TRY(gemm_tn(h, n, n, n, 1.0, A, lda, QL, ldql, 0.0, h->T1, ld));     // G = A^T QL
  SDC_TRY(gemm_tn(h, n, n, n, 1.0, h->T1, ld, Q, ldq, 0.0, h->Ah, ld));    // G^T Q
  if (B) {
    SDC_TRY(gemm_tn(h, n, n, n, 1.0, B, ldb, QL, ldql, 0.0, h->T1, ld));
    SDC_TRY(gemm_tn(h, n, n, n, 1.0, h->T1, ld, Q, ldq, 0.0, h->Bh, ld));
  }
  if (h->rflags & SDC_FLAG_SYMMETRIC) {   // RSEP (Alg. 6)
    k_symmetrize<<<ew_grid((long long)n * n), 256, 0, h->st>>>(h->Ah, ld, n);
    SDC_LAUNCHED(h);
  }
  SDC_TRY(select_dev(h, n, h->Ah, ld, B ? h->Bh : nullptr, ld, h->scal, h->scal + 2, h->scal + 4));
  k_e21_fro_cols<<<cdiv((long long)n * 32, 256), 256, 0, h->st>>>(h->Ah, ld, n, h->scal + 4, h->vec);
  SDC_LAUNCHED(h);
  if (B) {
    k_e21_fro_cols<<<cdiv((long long)n * 32, 256), 256, 0, h->st>>>(h->Bh, ld, n, h->scal + 4,
                                                                    h->vec + h->n_max);
    SDC_LAUNCHED(h);
  }
  k_e21_fro_finish<<<1, 1024, 0, h->st>>>(h->vec, B ? h->vec + h->n_max : nullptr, n, h->scal,
                                          h->scal + 2, h->scal + 6);
  SDC_LAUNCHED(h);
  return 0;
}

// synchronise and report a grid-barrier timeout recorded by a panel kernel (bar[1])
// start of a call: grid-barrier counter and LL exchange flags back to a known state (also
// inside a captured graph, so every replay starts from the same epochs)
int reset_sync(sdc_handle* h) {
  SDC_CK(cudaMemsetAsync(h->bar, 0, 64, h->st));
  SDC_CK(cudaMemsetAsync(h->llbuf, 0, PANEL_LL_DOUBLES * sizeof(double), h->st));
  SDC_CK(cudaMemsetAsync(h->cqbuf, 0, CQ_DOUBLES * sizeof(double), h->st));
  h->bar_count = 0;
  h->ll_epoch = 0;
  h->xpass_pending = h->alt.xpass_pending = false;
  if (h->alt_ready) {   // (on the caller's stream: ordered before any fork to the context)
    SDC_CK(cudaMemsetAsync(h->alt.bar, 0, 64, h->st));
    SDC_CK(cudaMemsetAsync(h->alt.llbuf, 0, PANEL_LL_DOUBLES * sizeof(double), h->st));
    SDC_CK(cudaMemsetAsync(h->alt.cqbuf, 0, CQ_DOUBLES * sizeof(double), h->st));
    h->alt.bar_count = 0;
    h->alt.ll_epoch = 0;
  }
  return 0;
}

// allocate the second factorization context on first use (outside any graph capture)
int ensure_alt(sdc_handle* h) {
  if (h->alt_ready || !h->pipeline) return 0;
  auto& a = h->alt;
  const size_t n = (size_t)h->n_max, nn = (size_t)wld((long long)n) * n;   // n x n buffers with ld wld(n)
  int rc = 0;
  const size_t first_alloc = h->allocs.size();
#define ALLOC(p, e) \
  if (!rc) rc = dalloc(h, &(p), (e))
  ALLOC(a.Y, 2 * nn);
  ALLOC(a.Yt, 2 * nn);
  ALLOC(a.Tb, (n / NB + 1) * NB * NB);
  ALLOC(a.Tob, (n / h->nbo_max + 1) * (size_t)h->nbo_max * h->nbo_max);
  ALLOC(a.Tobt, (n / h->nbo_max + 1) * (size_t)h->nbo_max * h->nbo_max);
  ALLOC(a.Zb, (size_t)h->nbo_max * (n + 64));
  ALLOC(a.Gb, (size_t)h->nbo_max * h->nbo_max);
  ALLOC(a.tau, n + NB);
  ALLOC(a.Wp, h->wp_elems);
  ALLOC(a.W, (size_t)std::max(256, h->nbo_max) * (n + 64));
  ALLOC(a.gbuf, 2 * ((size_t)h->num_sms + 1) * PANEL_NB);
  ALLOC(a.llbuf, PANEL_LL_DOUBLES);
  ALLOC(a.cqbuf, CQ_DOUBLES);
  if (h->cqs) ALLOC(a.cqs, CQS_DOUBLES);
  ALLOC(a.vec, 4 * n + 64);
  ALLOC(a.C, 2 * nn);
  ALLOC(a.G1, nn); ALLOC(a.G2, nn); ALLOC(a.G3, nn);
  if (h->lookahead) {
    ALLOC(a.Wp2, h->wp_elems);
    ALLOC(a.W2, (size_t)std::max(256, h->nbo_max) * (n + 64));
    ALLOC(a.Zb2, (size_t)h->nbo_max * (n + 64));
  }
#undef ALLOC
  if (!rc && h->alt_fail_hook) rc = SDC_ERR_NOMEM;   // test hook (SDC_ALT_FAIL_ALLOC): the fallback
  if (rc == SDC_ERR_NOMEM) {
    // not enough HBM for a second context next to the handle's workspace: release what was
    // taken and run every chain on the single context (same results, no overlap)
    for (size_t i = first_alloc; i < h->allocs.size(); ++i) cudaFree(h->allocs[i]);
    h->allocs.resize(first_alloc);
    cudaGetLastError();
    a = sdc_handle::Ctx{};
    h->pipeline = false;
    g_err[0] = 0;
    return 0;
  }
  if (rc) return rc;
  void* q = nullptr;
  SDC_CK(cudaMalloc(&q, 64));
  h->allocs.push_back(q);
  a.bar = (unsigned*)q;
  SDC_CK(cudaMemset(a.bar, 0, 64));
  if (a.cqs) {
    SDC_CK(cudaMalloc(&q, 64));
    h->allocs.push_back(q);
    a.cqs_sync = (unsigned*)q;
    SDC_CK(cudaMemset(q, 0, 64));
  }
  SDC_CK(cudaMemset(a.llbuf, 0, PANEL_LL_DOUBLES * sizeof(double)));
  SDC_CK(cudaMemset(a.cqbuf, 0, CQ_DOUBLES * sizeof(double)));
  SDC_CK(cudaStreamCreateWithFlags(&a.st, cudaStreamNonBlocking));
  if (h->lookahead) {
    int least = 0, greatest = 0;
    cudaDeviceGetStreamPriorityRange(&least, &greatest);
    SDC_CK(cudaStreamCreateWithPriority(&a.st_hi, cudaStreamNonBlocking, greatest));
    for (cudaEvent_t* e : {&a.la_fork, &a.la_fac, &a.la_B, &a.la_join})
      SDC_CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  }
  for (cudaEvent_t* e : {&h->ev_a, &h->ev_b, &h->ev_c})
    SDC_CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  h->alt_ready = true;
  return 0;
}

// make `to` wait for the work issued so far on `from` (fork / join between the contexts)
int stream_dep(sdc_handle* h, cudaStream_t from, cudaStream_t to, cudaEvent_t ev) {
  if (to == h->alt.st) h->sched[SDC_SCHED_CTX_FORKS]++;
  SDC_CK(cudaEventRecord(ev, from));
  SDC_CK(cudaStreamWaitEvent(to, ev, 0));
  return 0;
}

// split CholeskyQR2 panels that broke down since the last call (the fallback kernel factored
// them, correctly but slowly): counted, and mode 1 is switched off for this handle
void note_split_breakdowns(sdc_handle* h, unsigned nbrk) {
  if (!nbrk) return;
  h->sched[SDC_SCHED_CQ_SPLIT_BREAKDOWNS] += nbrk;
  if (h->cq_split == 1) h->cq_split = 0;
}

int check_barrier(sdc_handle* h) {
  unsigned int err = 0, nbrk = 0;
  SDC_CK(cudaMemcpyAsync(&err, h->bar + 1, sizeof(err), cudaMemcpyDeviceToHost, h->st));
  if (h->cqs_sync) {
    SDC_CK(cudaMemcpyAsync(&nbrk, h->cqs_sync + 2, sizeof(nbrk), cudaMemcpyDeviceToHost, h->st));
    SDC_CK(cudaMemsetAsync(h->cqs_sync + 2, 0, sizeof(unsigned), h->st));
  }
  SDC_CK(cudaStreamSynchronize(h->st));
  note_split_breakdowns(h, nbrk);
  if (err) {
    set_err("panel grid barrier timed out (co-residency violated?)");
    return SDC_ERR_CUDA;
  }
  return 0;
}

// Every entry point runs on the handle's device and restores the caller's current device
// on return (the caller's -- and torch's -- current device must not change).
struct DevGuard {
  int prev = -1;
  ~DevGuard() { if (prev >= 0) cudaSetDevice(prev); }
};
int check_handle(sdc_handle* h, DevGuard* g) {
  if (!h) {
    set_err("null handle");
    return -1;
  }
  int dev = -1;
  SDC_CK(cudaGetDevice(&dev));
  if (dev != h->device) {
    SDC_CK(cudaSetDevice(h->device));
    g->prev = dev;
  }
  return 0;
}
#define SDC_ENTER(h)  \
  DevGuard dg_;       \
  SDC_TRY(check_handle((h), &dg_))

}  // namespace

// ---------------------------------------------------------------------------------------
// step phases (enqueue only; no host synchronisation)
// ---------------------------------------------------------------------------------------
int enqueue_init(sdc_handle* h, int n, const double* A, long long lda, const double* B, long long ldb,
                 const double* V, long long ldv, const double* VL, long long ldvl) {
  const long long ld = wld(n), m = 2LL * n;
  const bool pencil = B != nullptr;
  SDC_TRY(reset_sync(h));
  h->b_ident = nullptr;
  SDC_CK(cudaMemsetAsync(h->Rprev, 0, sizeof(double) * (size_t)n * n, h->st));
  SDC_TRY(norms(h, A, lda, n, h->scal));
  if (pencil) SDC_TRY(norms(h, B, ldb, n, h->scal + 2));
  // A_0 = A, B_0 = rho B (or rho I) -- unit disk (rho = 1) or disk of radius rho;
  // half plane Re z < a: (A_0, B_0) = (A - (a-1) I, A - (a+1) I) (Moebius map)
  const double rho = h->region == SDC_REGION_DISK ? h->rparam : 1.0;
  k_copy<<<ew_grid((long long)n * n), 256, 0, h->st>>>(h->A[0], ld, A, lda, n, n, 1.0);
  SDC_LAUNCHED(h);
  if (h->region == SDC_REGION_HALFPLANE) {
    k_copy<<<ew_grid((long long)n * n), 256, 0, h->st>>>(h->B[0], ld, A, lda, n, n, 1.0);
    SDC_LAUNCHED(h);
    k_add_diag<<<cdiv(n, 256), 256, 0, h->st>>>(h->A[0], ld, n, -(h->rparam - 1.0));
    SDC_LAUNCHED(h);
    k_add_diag<<<cdiv(n, 256), 256, 0, h->st>>>(h->B[0], ld, n, -(h->rparam + 1.0));
  } else if (pencil) {
    k_copy<<<ew_grid((long long)n * n), 256, 0, h->st>>>(h->B[0], ld, B, ldb, n, n, rho);
  } else {
    k_set_identity<<<ew_grid((long long)n * n), 256, 0, h->st>>>(h->B[0], ld, n, n, rho);
    h->b_ident = h->B[0];
    h->b_ident_rho = rho;
  }
  SDC_LAUNCHED(h);
  k_build_stack<<<ew_grid(m * n), 256, 0, h->st>>>(h->S, m, h->A[0], ld, h->B[0], ld, n);
  SDC_LAUNCHED(h);
  if (pencil && !h->ql_orth) {   // left IRS on (A^T, B^T)
    SDC_TRY(transpose_rev(h, h->AL[0], ld, A, lda, n, 0));
    SDC_TRY(transpose_rev(h, h->BL[0], ld, B, ldb, n, 0));
    if (rho != 1.0) {
      k_copy<<<ew_grid((long long)n * n), 256, 0, h->st>>>(h->BL[0], ld, h->BL[0], ld, n, n, rho);
      SDC_LAUNCHED(h);
    }
    k_build_stack<<<ew_grid(m * n), 256, 0, h->st>>>(h->SL, m, h->AL[0], ld, h->BL[0], ld, n);
    SDC_LAUNCHED(h);
  }
  SDC_TRY(transpose_rev(h, h->Vt, ld, V, ldv, n, 0));                   // V^T (K-major operand)
  if (pencil && !h->ql_orth) SDC_TRY(transpose_rev(h, h->VLt, ld, VL, ldvl, n, 0));
  return 0;
}

int enqueue_finish(sdc_handle* h, int n, const double* A, long long lda, const double* B, long long ldb,
                   double* Q, long long ldq, double* QLd, double* QL, long long ldql, double* Ahat,
                   long long ldah, bool have_split, int cur, int max_iters) {
  const long long ld = wld(n);
  const bool pencil = B != nullptr;
  if (!have_split) {
    const bool two = pencil && !h->ql_orth && h->alt_ready;   // left GRURV on the second context
    if (two) {
      SDC_TRY(stream_dep(h, h->st, h->alt.st, h->ev_a));
      AltScope as(h);
      SDC_TRY(grurv_left(h, n, h->AL[cur], h->BL[cur], h->VLt, QLd, ld));
    }
    SDC_TRY(grurv_right(h, n, h->A[cur], h->B[cur], h->Vt, Q, ldq));
    if (pencil && h->ql_orth) SDC_TRY(ql_from_aq(h, n, A, lda, Q, ldq, QLd, ld));
    else if (pencil && !two) SDC_TRY(grurv_left(h, n, h->AL[cur], h->BL[cur], h->VLt, QLd, ld));
    if (two) SDC_TRY(stream_dep(h, h->alt.st, h->st, h->ev_b));
    SDC_TRY(similarity_select(h, n, A, lda, B, ldb, Q, ldq, pencil ? QLd : Q, pencil ? ld : ldq));
  }
  SDC_TRY(norms(h, h->A[cur], ld, n, h->scal + 8));    // side indicator (res->side)
  SDC_TRY(norms(h, h->B[cur], ld, n, h->scal + 10));
  SDC_CK(cudaMemsetAsync(h->flag, 0, sizeof(int), h->st));
  k_nonfinite<<<ew_grid((long long)n * n), 256, 0, h->st>>>(h->Ah, ld, n, h->flag);
  SDC_LAUNCHED(h);
  if (pencil) SDC_CK(cudaMemcpy2DAsync(QL, sizeof(double) * ldql, QLd, sizeof(double) * ld,
                                       sizeof(double) * n, n, cudaMemcpyDeviceToDevice, h->st));
  if (Ahat) SDC_CK(cudaMemcpy2DAsync(Ahat, sizeof(double) * ldah, h->Ah, sizeof(double) * ld,
                                     sizeof(double) * n, n, cudaMemcpyDeviceToDevice, h->st));
  SDC_CK(cudaMemcpyAsync(h->hscal, h->scal, sizeof(double) * (SCAL_HIST + (size_t)max_iters),
                         cudaMemcpyDeviceToHost, h->st));
  SDC_CK(cudaMemcpyAsync(h->hflags, h->flag, sizeof(int), cudaMemcpyDeviceToHost, h->st));
  SDC_CK(cudaMemcpyAsync(h->hflags + 1, h->bar + 1, sizeof(unsigned), cudaMemcpyDeviceToHost, h->st));
  if (h->alt_ready)
    SDC_CK(cudaMemcpyAsync(h->hflags + 2, h->alt.bar + 1, sizeof(unsigned), cudaMemcpyDeviceToHost, h->st));
  else
    h->hflags[2] = 0;
  h->hflags[3] = h->hflags[4] = 0;
  if (h->cqs_sync) {
    SDC_CK(cudaMemcpyAsync(h->hflags + 3, h->cqs_sync + 2, sizeof(unsigned), cudaMemcpyDeviceToHost, h->st));
    SDC_CK(cudaMemsetAsync(h->cqs_sync + 2, 0, sizeof(unsigned), h->st));
  }
  if (h->alt.cqs_sync) {   // (the second context's chains were joined into this stream before)
    SDC_CK(cudaMemcpyAsync(h->hflags + 4, h->alt.cqs_sync + 2, sizeof(unsigned), cudaMemcpyDeviceToHost, h->st));
    SDC_CK(cudaMemsetAsync(h->alt.cqs_sync + 2, 0, sizeof(unsigned), h->st));
  }
  return 0;
}

int enqueue_fixed(sdc_handle* h, int n, const double* A, long long lda, const double* B, long long ldb,
                  double* Q, long long ldq, double* QLd, double* QL, long long ldql, double* Ahat,
                  long long ldah, int max_iters) {
  // V/VL are read through the graph key's pointers; pass them via the handle's last key
  const long long ld = wld(n);
  const bool pencil = B != nullptr;
  SDC_TRY(enqueue_init(h, n, A, lda, B, ldb, h->cur_V, h->cur_ldv, h->cur_VL, h->cur_ldvl));
  int cur = 0;
  // Alg. 4: the right IRS on (A, B) and the left IRS on (A^T, B^T) are independent chains;
  // with the second context they run concurrently (joined before the similarity)
  const bool two = pencil && !h->ql_orth && h->alt_ready;
  if (two) SDC_TRY(stream_dep(h, h->st, h->alt.st, h->ev_a));
  // two chains share the SMs: one-tile CTAs for the short-K updates (measured 2.8% faster
  // at config 4 than persistent grids, which hold SMs the other chain's panels wait for)
  struct TwoChains {
    sdc_handle* h;
    TwoChains(sdc_handle* h_, bool on) : h(h_) { h->two_chains = on; h->share_sms = on; }
    ~TwoChains() { h->two_chains = false; h->share_sms = false; }
  } tc(h, two);
  const bool xpass = h->xpass_on;
  for (int j = 0; j < max_iters; ++j) {
    const bool more = xpass && j + 1 < max_iters;
    SDC_TRY(irs_pass(h, n, h->A[cur], ld, h->B[cur], ld, h->A[cur ^ 1], ld, h->B[cur ^ 1], ld, h->S, j,
                     nullptr, 0, more));
    if (two) {
      AltScope as(h);
      SDC_TRY(irs_pass(h, n, h->AL[cur], ld, h->BL[cur], ld, h->AL[cur ^ 1], ld, h->BL[cur ^ 1], ld,
                       h->SL, -1, nullptr, 0, more));
    } else if (pencil && !h->ql_orth) {
      SDC_TRY(irs_pass(h, n, h->AL[cur], ld, h->BL[cur], ld, h->AL[cur ^ 1], ld, h->BL[cur ^ 1], ld,
                       h->SL, -1, nullptr, 0));
    }
    cur ^= 1;
  }
  return enqueue_finish(h, n, A, lda, B, ldb, Q, ldq, QLd, QL, ldql, Ahat, ldah, false, cur, max_iters);
}

// =======================================================================================
// C ABI
// =======================================================================================
extern "C" {

const char* sdc_last_error(void) { return g_err; }

long long sdc_kernel_launches(const sdc_handle* h) { return h ? h->launches : 0; }

int sdc_debug_counters(sdc_handle* h, unsigned long long* out, int count, int reset) {
  if (!h || count < 0 || count > 64) return -1;
  if (count && cudaMemcpy(out, h->dbg, sizeof(unsigned long long) * count, cudaMemcpyDeviceToHost) != cudaSuccess)
    return SDC_ERR_CUDA;
  if (reset) cudaMemset(h->dbg, 0, 64 * sizeof(unsigned long long));
  return 0;
}

int sdc_schedule_counters(sdc_handle* h, long long* out, int count, int reset) {
  if (!h) { set_err("null handle"); return -1; }
  if (count < 0 || count > SDC_SCHED_COUNTERS || (count > 0 && !out)) { set_err("bad count"); return -3; }
  if (count > SDC_SCHED_PANEL_CQR_DONE) {   // device-side outcomes of the CholeskyQR2 panels
    DevGuard dg_;
    SDC_TRY(check_handle(h, &dg_));
    unsigned long long st[2] = {0, 0};
    SDC_CK(cudaDeviceSynchronize());
    SDC_CK(cudaMemcpy(st, h->cqstat, sizeof(st), cudaMemcpyDeviceToHost));
    h->sched[SDC_SCHED_PANEL_CQR_DONE] = (long long)st[0];
    h->sched[SDC_SCHED_PANEL_CQR_FALLBACK] = (long long)st[1];
  }
  h->sched[SDC_SCHED_MAX_CLUSTERS16] = h->max_clusters16;
  for (int i = 0; i < count; ++i) out[i] = h->sched[i];
  if (reset) {
    for (int i = 0; i < SDC_SCHED_COUNTERS; ++i) h->sched[i] = 0;
    cudaMemset(h->cqstat, 0, 16);
  }
  return 0;
}

int sdc_profile(sdc_handle* h, int enable) {
  if (!h) return -1;
  prof_collect(h);
  h->prof_on = enable != 0;
  for (int c = 0; c < SDC_PROF_CLASSES; ++c) { h->prof_ms[c] = 0; h->prof_work[c] = 0; h->prof_n[c] = 0; }
  return 0;
}

int sdc_profile_read(sdc_handle* h, int cls, double* ms, long long* launches, double* work) {
  if (!h) return -1;
  if (cls < 0 || cls >= SDC_PROF_CLASSES) return -2;
  prof_collect(h);
  if (ms) *ms = h->prof_ms[cls];
  if (launches) *launches = h->prof_n[cls];
  if (work) *work = h->prof_work[cls];
  return 0;
}

void sdc_destroy(sdc_handle* h) {
  if (!h) return;
  DevGuard dg_;
  if (check_handle(h, &dg_) != 0) return;
  for (cudaEvent_t e : h->ev_pool) cudaEventDestroy(e);
  if (h->gexec) cudaGraphExecDestroy(h->gexec);
  if (h->cap_st) cudaStreamDestroy(h->cap_st);
  if (h->st_hi) cudaStreamDestroy(h->st_hi);
  for (cudaEvent_t e : {h->la_fork, h->la_fac, h->la_B, h->la_join, h->alt.la_fork, h->alt.la_fac,
                        h->alt.la_B, h->alt.la_join, h->ev_a, h->ev_b, h->ev_c})
    if (e) cudaEventDestroy(e);
  if (h->alt.st) cudaStreamDestroy(h->alt.st);
  if (h->alt.st_hi) cudaStreamDestroy(h->alt.st_hi);
  if (h->hscal) cudaFreeHost(h->hscal);
  if (h->hflags) cudaFreeHost(h->hflags);
  for (void* p : h->allocs) cudaFree(p);
  if (h->bat_out) cudaFree(h->bat_out);
  delete h;
}

int sdc_create(sdc_handle** out, int device, int n_max, int pencil) {
  if (!out) { set_err("sdc_create: null output"); return -1; }
  *out = nullptr;
  if (n_max < 2 || n_max > 24576) { set_err("sdc_create: n_max %d out of [2, 24576]", n_max); return -3; }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    set_err("sdc_create: no CUDA device (no CPU fallback)");
    return SDC_ERR_CUDA;
  }
  if (device < 0 || device >= ndev) { set_err("sdc_create: bad device %d", device); return -2; }
  DevGuard dg_;                  // the caller's current device is restored on return
  {
    int cur = -1;
    SDC_CK(cudaGetDevice(&cur));
    if (cur != device) { SDC_CK(cudaSetDevice(device)); dg_.prev = cur; }
  }
  cudaDeviceProp prop;
  SDC_CK(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) {
    set_err("sdc_create: device is sm_%d%d; libsdc is built for sm_100a only", prop.major, prop.minor);
    return SDC_ERR_NOT_SUPPORTED;
  }
  int coop = 0;
  SDC_CK(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device));
  if (!coop) { set_err("sdc_create: cooperative launch unsupported"); return SDC_ERR_NOT_SUPPORTED; }
  sdc_handle* h = new sdc_handle();
  h->device = device;
  h->n_max = n_max;
  h->pencil = pencil ? 1 : 0;
  h->num_sms = prop.multiProcessorCount;
  const size_t n = (size_t)n_max, nn = (size_t)wld((long long)n) * n;   // n x n buffers with ld wld(n)
  int rc = 0;
#define ALLOC(p, e) \
  if (!rc) rc = dalloc(h, &(p), (e))
  ALLOC(h->S, 2 * nn);
  ALLOC(h->Y, 2 * nn);
  ALLOC(h->Yt, 2 * nn);
  ALLOC(h->Vt, nn);
  ALLOC(h->C, 2 * nn);
  ALLOC(h->A[0], nn); ALLOC(h->A[1], nn); ALLOC(h->B[0], nn); ALLOC(h->B[1], nn);
  ALLOC(h->G1, nn); ALLOC(h->G2, nn); ALLOC(h->G3, nn); ALLOC(h->T1, nn); ALLOC(h->Ah, nn);
  ALLOC(h->Rprev, nn);
  if (h->pencil) {
    ALLOC(h->SL, 2 * nn);
    ALLOC(h->AL[0], nn); ALLOC(h->AL[1], nn); ALLOC(h->BL[0], nn); ALLOC(h->BL[1], nn);
    ALLOC(h->Bh, nn); ALLOC(h->QLb, nn); ALLOC(h->VLt, nn);
  }
  if (const char* e = getenv("SDC_NBO")) {
    h->nbo = std::max(64, std::min(512, atoi(e) / 64 * 64));
    h->nbo_fixed = true;
  }
  h->nbo_max = h->nbo;   // workspace is sized for this width; calls may use a narrower one
  ALLOC(h->Tb, (n / NB + 1) * NB * NB);
  ALLOC(h->Tob, (n / h->nbo + 1) * (size_t)h->nbo * h->nbo);
  ALLOC(h->Tobt, (n / h->nbo + 1) * (size_t)h->nbo * h->nbo);
  ALLOC(h->Zb, (size_t)h->nbo * (n + 64));
  ALLOC(h->Gb, (size_t)h->nbo * h->nbo);
  ALLOC(h->tau, n + NB);
  h->wp_elems = (size_t)std::max(256, h->nbo) * (2 * (size_t)h->num_sms * 128 + 2 * n + 256);
  ALLOC(h->Wp, h->wp_elems);
  ALLOC(h->W, (size_t)std::max(256, h->nbo) * (n + 64));
  ALLOC(h->gbuf, 2 * ((size_t)h->num_sms + 1) * PANEL_NB);
  ALLOC(h->llbuf, PANEL_LL_DOUBLES);
  if (!rc && cudaMemset(h->llbuf, 0, PANEL_LL_DOUBLES * sizeof(double)) != cudaSuccess) rc = SDC_ERR_CUDA;
  ALLOC(h->cqbuf, CQ_DOUBLES);
  if (!rc && cudaMemset(h->cqbuf, 0, CQ_DOUBLES * sizeof(double)) != cudaSuccess) rc = SDC_ERR_CUDA;
  if (!rc && 2LL * n_max > 4096) {   // split CholeskyQR2 panels (tall stacks only)
    ALLOC(h->cqs, CQS_DOUBLES);
    void* q = nullptr;
    if (!rc && cudaMalloc(&q, 64) != cudaSuccess) rc = SDC_ERR_NOMEM;
    else if (!rc) { h->allocs.push_back(q); h->cqs_sync = (unsigned*)q; cudaMemset(q, 0, 64); }
  }
  ALLOC(h->pmA, (n / SEL_T + 1) * n);
  if (h->pencil) ALLOC(h->pmB, (n / SEL_T + 1) * n);
  ALLOC(h->vec, 4 * n + 64);
  ALLOC(h->scal, SCAL_HIST + MAX_HIST);
#undef ALLOC
  if (!rc) {
    void* q = nullptr;
    cudaError_t e = cudaMalloc(&q, 64);
    if (e != cudaSuccess) { set_err("cudaMalloc: %s", cudaGetErrorString(e)); rc = SDC_ERR_NOMEM; }
    else { h->allocs.push_back(q); h->bar = (unsigned*)q; h->flag = (int*)((char*)q + 32); }
  }
  if (!rc) {
    void* q = nullptr;
    if (cudaMalloc(&q, 64 * sizeof(unsigned long long)) != cudaSuccess) rc = SDC_ERR_NOMEM;
    else { h->allocs.push_back(q); h->dbg = (unsigned long long*)q; cudaMemset(q, 0, 64 * 8); }
  }
  if (!rc) {
    void* q = nullptr;
    if (cudaMalloc(&q, 2 * sizeof(unsigned long long)) != cudaSuccess) rc = SDC_ERR_NOMEM;
    else { h->allocs.push_back(q); h->cqstat = (unsigned long long*)q; cudaMemset(q, 0, 16); }
  }
  if (const char* e = getenv("SDC_PANEL_ROWS")) h->panel_rows = std::max(16, atoi(e));
  if (getenv("SDC_DEBUG_COUNTERS")) h->dbg_on = true;
  if (getenv("SDC_PANEL_SMEM")) h->panel_reg = false;
  if (const char* e = getenv("SDC_CQR")) h->cqr_mode = std::max(0, std::min(2, atoi(e)));
  h->cqr = h->cqr_mode != 0;
  if (const char* e = getenv("SDC_GRAPH_MAX_N")) h->graph_max_n = atoi(e);
  if (const char* e = getenv("SDC_CLUSTER_MAX_ROWS")) h->cluster_max_rows = atoi(e);
  if (!rc) {   // non-portable cluster size 16 for the small-panel kernel (if the part allows it)
    int cl = 0;
    cudaDeviceGetAttribute(&cl, cudaDevAttrClusterLaunch, device);
    bool np = cl != 0;
    for (int rpt : {0, 8, 16, 32})
      np = np && cudaFuncSetAttribute(panel_fn(true, rpt), cudaFuncAttributeNonPortableClusterSizeAllowed,
                                      1) == cudaSuccess;
    const void* fn16 = panel_fn(true, 0);
    if (np) {
      // the occupancy probes need the limit >= their footprints; it is never lowered (another
      // handle, possibly on another host thread, may be launching this variant)
      std::lock_guard<std::mutex> lk(g_panel_mu);
      size_t& cur0 = g_panel_attr[device & (MAX_DEV - 1)][1][rpt_slot(0)];
      cur0 = std::max({cur0, panel_smem_bytes(cdiv(h->cluster_max_rows, 16), h->cqr), panel_smem_bytes(256, h->cqr)});
      cudaFuncSetAttribute(fn16, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cur0);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(16);
      cfg.blockDim = dim3(PANEL_THREADS);
      cfg.dynamicSmemBytes = panel_smem_bytes(cdiv(h->cluster_max_rows, 16), h->cqr);
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = 16;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      int ncl = 0;
      if (cudaOccupancyMaxActiveClusters(&ncl, fn16, &cfg) == cudaSuccess && ncl >= 1)
        h->cluster_ok = true;
      // tall panels: how many 16-CTA clusters with ~256-row blocks can be resident at once
      cfg.dynamicSmemBytes = panel_smem_bytes(256, h->cqr);
      int ncl2 = 0;
      if (cudaOccupancyMaxActiveClusters(&ncl2, fn16, &cfg) == cudaSuccess && ncl2 >= 2) {
        h->max_clusters16 = ncl2;
        h->mcluster_ok = true;
      }
      int ncl8 = 0;
      attr[0].val.clusterDim.x = 8;
      cfg.gridDim = dim3(8);
      if (cudaOccupancyMaxActiveClusters(&ncl8, fn16, &cfg) == cudaSuccess) h->max_clusters8 = ncl8;
      cudaGetLastError();
    }
    if (getenv("SDC_NO_CLUSTER")) h->cluster_ok = h->mcluster_ok = false;
    if (getenv("SDC_NO_MCLUSTER")) h->mcluster_ok = false;
  }
  if (!rc && cudaMallocHost(&h->hscal, sizeof(double) * (SCAL_HIST + MAX_HIST)) != cudaSuccess) rc = SDC_ERR_NOMEM;
  if (!rc && cudaMallocHost(&h->hflags, 64) != cudaSuccess) rc = SDC_ERR_NOMEM;
  if (!rc && cudaStreamCreateWithFlags(&h->cap_st, cudaStreamNonBlocking) != cudaSuccess) rc = SDC_ERR_CUDA;
  if (const char* e = getenv("SDC_LOOKAHEAD")) h->lookahead = atoi(e) != 0;
  if (const char* e = getenv("SDC_PERSIST")) h->persist_mode = atoi(e);
  if (const char* e = getenv("SDC_RED")) h->red_mode = atoi(e);
  if (const char* e = getenv("SDC_SIDE_PERSIST")) h->side_persist = atoi(e) != 0;
  if (const char* e = getenv("SDC_SPLIT_KMIN")) h->split_kmin = std::max(16, atoi(e));
  if (const char* e = getenv("SDC_SCHUR_BATCH")) h->schur_batch = atoi(e) != 0;
  if (const char* e = getenv("SDC_CQ_SPLIT")) h->cq_split = std::max(0, std::min(2, atoi(e)));
  if (const char* e = getenv("SDC_CQ_SPLIT_ROWS")) h->cq_split_rows = std::max(128, atoi(e));
  if (const char* e = getenv("SDC_CQ_SPLIT_ROWS_SHARED")) h->cq_split_rows_shared = std::max(128, atoi(e));
  if (const char* e = getenv("SDC_GEMM_VARIANT")) h->gemm_force = h->alt.gemm_force = atoi(e);
  if (const char* e = getenv("SDC_XPASS")) h->xpass_on = atoi(e) != 0;
  if (const char* e = getenv("SDC_PIPELINE")) h->pipeline = atoi(e) != 0;
  if (getenv("SDC_ALT_FAIL_ALLOC")) h->alt_fail_hook = true;
  if (const char* e = getenv("SDC_MAIN_GEMM")) h->gemm_force = atoi(e);
  if (const char* e = getenv("SDC_ALT_GEMM")) h->alt.gemm_force = atoi(e);
  if (!rc && h->lookahead) {
    int least = 0, greatest = 0;
    cudaDeviceGetStreamPriorityRange(&least, &greatest);
    if (cudaStreamCreateWithPriority(&h->st_hi, cudaStreamNonBlocking, greatest) != cudaSuccess) rc = SDC_ERR_CUDA;
    for (cudaEvent_t* e : {&h->la_fork, &h->la_fac, &h->la_B, &h->la_join})
      if (!rc && cudaEventCreateWithFlags(e, cudaEventDisableTiming) != cudaSuccess) rc = SDC_ERR_CUDA;
    if (!rc) rc = dalloc(h, &h->Wp2, h->wp_elems);
    if (!rc) rc = dalloc(h, &h->W2, (size_t)std::max(256, h->nbo) * (n + 64));
    if (!rc) rc = dalloc(h, &h->Zb2, (size_t)h->nbo * (n + 64));
  }
  if (rc) { sdc_destroy(h); return rc; }
  *out = h;
  return 0;
}

int sdc_split(sdc_handle* h, void* stream, int n, const double* A, int lda, const double* B,
              int ldb, const double* V, int ldv, const double* VL, int ldvl, int region,
              int max_iters, double tol, int stop_mode, double* Q, int ldq, double* QL, int ldql,
              double* Ahat, int ldah, double* hist, int hist_cap, sdc_result* res) {
  if (region != SDC_REGION_UNIT_DISK) { set_err("sdc_split: use sdc_split_region for region %d", region); return -12; }
  return sdc_split_region(h, stream, n, A, lda, B, ldb, V, ldv, VL, ldvl, region, 1.0, 0, max_iters,
                          tol, stop_mode, Q, ldq, QL, ldql, Ahat, ldah, hist, hist_cap, res);
}

// host side of the shared counter-based generator (same constants as mix64 in aux.cuh)
static unsigned long long host_mix64(unsigned long long seed, unsigned long long ctr) {
  unsigned long long z = seed + 0x9E3779B97F4A7C15ull * (ctr + 1ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

}  // extern "C"

namespace {
// Counter of attempt t (< 16) on the diagonal block at GLOBAL offset o of order m (the same
// 23-bit key as orc_attempt_ctr): keyed by the block, so any processing order -- depth first
// here, or subproblems handed to other ranks -- draws the same numbers.
unsigned long long attempt_ctr(int o, int m, int t) {
  const unsigned long long id = (unsigned long long)o * 65537ull + (unsigned long long)m;
  return ((host_mix64(0x5DC0FFEEull, id) & 0x7FFFFull) << 4) | (unsigned long long)t;
}

struct SchurScratch { double *Vb, *Gb, *Ab, *sc; };

// One node of the recursion: the attempt loop on the diagonal block Tb
// (m x m, ld ldtb, global offset o).  Accepted: Tb <- Ahat with E21 := 0, Qb <- Q_b, *r in
// [1, m-1]; *r = 0 for a leaf / unsplit block (Tb unchanged).  Same decisions as
// orc_schur_node.
int schur_node(sdc_handle* h, cudaStream_t st, int m, double* Tb, long long ldtb, int o, int leaf,
               unsigned long long seed, int max_iters, double tol, double* Qb, long long ldqb,
               const SchurScratch& w, int* r_out, int* stats, double* max_metric) {
  Nvtx nv("schur_node");
  *r_out = 0;
  if (m <= leaf) return 0;
  double hs[4];
  if (m == 2) {   // 2x2 with complex eigenvalues: a standardised leaf
    SDC_CK(cudaMemcpy2DAsync(hs, 2 * sizeof(double), Tb, ldtb * sizeof(double), 2 * sizeof(double), 2,
                             cudaMemcpyDeviceToHost, st));
    SDC_CK(cudaStreamSynchronize(st));
    const double a = hs[0], c = hs[1], b = hs[2], d = hs[3];
    if ((a - d) * (a - d) + 4.0 * b * c < 0.0) return 0;
  }
  // [c - 2s, c + 2s], c = trace/m, s = ||T_blk - cI||_F / sqrt(m)
  k_block_scale<<<1, 256, 0, st>>>(Tb, ldtb, m, w.sc);
  SDC_LAUNCHED(h);
  SDC_CK(cudaMemcpyAsync(hs, w.sc, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
  SDC_CK(cudaStreamSynchronize(st));
  double lo = hs[0] - 2.0 * hs[1], hi = hs[0] + 2.0 * hs[1];
  if (!(hs[1] > 0.0)) { stats[2]++; return 0; }
  for (int att = 0; att < 16; ++att) {
    const unsigned long long ctr = attempt_ctr(o, m, att);
    const double u = (double)(host_mix64(seed, 2ull * ctr) >> 11) * 1.1102230246251565e-16;
    const double a = lo + (0.25 + 0.5 * u) * (hi - lo);
    k_gauss<<<ew_grid((long long)m * m), 256, 0, st>>>(w.Gb, m, m, seed, 2ull * ctr + 1ull);
    SDC_LAUNCHED(h);
    SDC_TRY(sdc_qr(h, st, m, m, w.Gb, m, w.Vb, m));                 // Haar V (diag R >= 0)
    sdc_result res;
    const double tolb = std::max(tol, 8e-15 * m);   // rounding floor grows ~ m eps
    SDC_TRY(sdc_split_region(h, st, m, Tb, (int)ldtb, nullptr, 0, w.Vb, m, nullptr, 0, SDC_REGION_HALFPLANE,
                             a, SDC_FLAG_PLATEAU | SDC_FLAG_ONESIDED, max_iters, tolb, SDC_STOP_E21, Qb,
                             (int)ldqb, nullptr, 0, w.Ab, m, nullptr, 0, &res));
    h->st = st;
    stats[3] += res.iters;
    // accept only clearly two-sided pairs (same rule as orc_schur_node; reading Q20)
    const bool onesided = res.side < 1e-3 || res.side > 1.0 - 1e-3;
    if (getenv("SDC_SCHUR_TRACE"))   // decision trace (orc_schur_node's ORC_SCHUR_TRACE format)
      fprintf(stderr, "node o=%d m=%d att=%d a=%.6f iters=%d status=%d r=%d metric=%.3e side=%.3e\n", o, m, att, a,
              res.iters, res.status, res.r, res.metric, res.side);
    if (res.status != 0 || onesided) {   // a one-sided pair's split is incidental
      stats[1]++;
      if (res.side > 0.95) hi = a;          // every eigenvalue left of the line
      else if (res.side < 0.05) lo = a;     // every eigenvalue right of the line
      continue;
    }
    stats[0]++;
    *max_metric = std::max(*max_metric, res.metric);
    k_place_ahat<<<ew_grid((long long)m * m), 256, 0, st>>>(Tb, ldtb, w.Ab, m, m, res.r);
    SDC_LAUNCHED(h);
    *r_out = res.r;
    return 0;
  }
  stats[2]++;   // 16 failed attempts: an unsplit leaf
  return 0;
}

// ---- batched small blocks of the recursion (schur_batched.cuh) ---------------------------
// Device workspace of one wave: block lists, per-block results and scratch slots.
struct SchurWave {
  int cap = 0;
  int *off = nullptr, *ord = nullptr, *r = nullptr, *stats = nullptr;
  double *metric = nullptr, *scratch = nullptr;
  void release() {
    for (void* p : {(void*)off, (void*)ord, (void*)r, (void*)stats, (void*)metric, (void*)scratch})
      if (p) cudaFree(p);
    *this = SchurWave();
  }
  int reserve(int nb) {
    if (nb <= cap) return 0;
    release();
    if (cudaMalloc(&off, sizeof(int) * nb) || cudaMalloc(&ord, sizeof(int) * nb) ||
        cudaMalloc(&r, sizeof(int) * nb) || cudaMalloc(&stats, sizeof(int) * 4 * nb) ||
        cudaMalloc(&metric, sizeof(double) * nb) ||
        cudaMalloc(&scratch, sizeof(double) * (size_t)SB_SLOT * nb)) {
      release();
      set_err("sdc_schur: out of device memory (batched blocks)");
      return SDC_ERR_NOMEM;
    }
    cap = nb;
    return 0;
  }
};
constexpr int SCHUR_WAVE_MAX = 148 * 8;   // blocks per launch (scratch: 160 KB per block)

// One launch of k_schur_leaves over the blocks (off[i], ord[i]) of T, all of order <= BAT_NMAX,
// sorted by the caller so that max_ord bounds them; results to the host vectors.  Q_b of
// accepted blocks stay in w.scratch (slot 3) for the apply kernels.
int schur_leaves_launch(sdc_handle* h, cudaStream_t st, SchurWave& w, double* T, long long ldt, int key_off,
                        int leaf, unsigned long long seed, int max_iters, double tol, const int* off,
                        const int* ord, int nb, int max_ord, int* r_out, int* stats_out, double* metric_out) {
  static DevOnce attr;
  if (!attr.has(h->device)) {
    SDC_CK(cudaFuncSetAttribute(k_schur_leaves, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)bq_smem_bytes(BAT_NMAX)));
    SDC_CK(cudaFuncSetAttribute(k_schur_apply_left, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)SB_APPLY_SMEM));
    SDC_CK(cudaFuncSetAttribute(k_schur_apply_right, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)SB_APPLY_SMEM));
    attr.set(h->device);
  }
  SDC_TRY(w.reserve(nb));
  SDC_CK(cudaMemcpyAsync(w.off, off, sizeof(int) * nb, cudaMemcpyHostToDevice, st));
  SDC_CK(cudaMemcpyAsync(w.ord, ord, sizeof(int) * nb, cudaMemcpyHostToDevice, st));
  SchurLeafArgs a{T, ldt, w.off, w.ord, key_off, leaf, seed, max_iters, tol, w.scratch, w.r, w.stats, w.metric,
                  getenv("SDC_SCHUR_TRACE") ? 1 : 0};
  k_schur_leaves<<<nb, BQ_THREADS, bq_smem_bytes(max_ord), st>>>(a);
  SDC_LAUNCHED(h);
  h->sched[SDC_SCHED_SCHUR_BATCH_LAUNCHES]++;
  h->sched[SDC_SCHED_SCHUR_BATCH_BLOCKS] += nb;
  SDC_CK(cudaMemcpyAsync(r_out, w.r, sizeof(int) * nb, cudaMemcpyDeviceToHost, st));
  SDC_CK(cudaMemcpyAsync(stats_out, w.stats, sizeof(int) * 4 * nb, cudaMemcpyDeviceToHost, st));
  SDC_CK(cudaMemcpyAsync(metric_out, w.metric, sizeof(double) * nb, cudaMemcpyDeviceToHost, st));
  return 0;
}

// All blocks of `small` (order <= BAT_NMAX) and their descendants, one level per wave; leaves
// are appended to blocks.  T (n x n) and Q (n rows) receive the off-diagonal updates.
int schur_small_waves(sdc_handle* h, cudaStream_t st, int n, double* T, long long ldt, double* Q, long long ldq,
                      int key_off, int leaf, unsigned long long seed, int max_iters, double tol,
                      std::vector<std::pair<int, int>> small, std::vector<std::pair<int, int>>& blocks,
                      int* stats, double* max_metric) {
  SchurWave w;
  struct Guard { SchurWave& w; ~Guard() { w.release(); } } guard{w};
  std::vector<int> off, ord, r, sst;
  std::vector<double> met;
  while (!small.empty()) {
    std::vector<std::pair<int, int>> work, next;
    for (auto& b : small) {
      if (b.second <= leaf || b.second < 2) blocks.push_back(b);   // a leaf by size
      else work.push_back(b);
    }
    // by order (descending): each launch's shared memory is sized by its first block
    std::stable_sort(work.begin(), work.end(), [](const std::pair<int, int>& x, const std::pair<int, int>& y) {
      return ((x.second + 15) & ~15) > ((y.second + 15) & ~15);
    });
    for (size_t b0 = 0; b0 < work.size();) {
      const int cls = (work[b0].second + 15) & ~15;
      size_t b1 = b0;
      while (b1 < work.size() && b1 - b0 < (size_t)SCHUR_WAVE_MAX && ((work[b1].second + 15) & ~15) == cls) ++b1;
      const int nb = (int)(b1 - b0);
      off.resize(nb); ord.resize(nb); r.resize(nb); sst.resize(4 * (size_t)nb); met.resize(nb);
      int omin = n;
      for (int i = 0; i < nb; ++i) {
        off[i] = work[b0 + i].first;
        ord[i] = work[b0 + i].second;
        omin = std::min(omin, off[i] + ord[i]);
      }
      SDC_TRY(schur_leaves_launch(h, st, w, T, ldt, key_off, leaf, seed, max_iters, tol, off.data(), ord.data(),
                                  nb, cls, r.data(), sst.data(), met.data()));
      SchurApplyArgs ap{T, ldt, Q, ldq, n, w.off, w.ord, w.r, w.scratch};
      if (n - omin > 0) {
        k_schur_apply_left<<<dim3(cdiv(n - omin, 64), nb), 256, SB_APPLY_SMEM, st>>>(ap);
        SDC_LAUNCHED(h);
      }
      k_schur_apply_right<<<dim3(2 * cdiv(n, 64), nb), 256, SB_APPLY_SMEM, st>>>(ap);
      SDC_LAUNCHED(h);
      SDC_CK(cudaStreamSynchronize(st));
      for (int i = 0; i < nb; ++i) {
        for (int q = 0; q < 4; ++q) stats[q] += sst[4 * (size_t)i + q];
        if (r[i] == 0) { blocks.push_back({off[i], ord[i]}); continue; }
        *max_metric = std::max(*max_metric, met[i]);
        next.push_back({off[i], r[i]});
        next.push_back({off[i] + r[i], ord[i] - r[i]});
      }
      b0 = b1;
    }
    small.swap(next);
  }
  return 0;
}
}  // namespace

extern "C" {

int sdc_schur_keyed(sdc_handle* h, void* stream, int n, const double* A, int lda, int key_off, int leaf,
                    unsigned long long seed, int max_iters, double tol, double* Q, int ldq, double* T,
                    int ldt, int* blk_off, int* blk_size, int* nblk, int* stats, double* max_metric) {
  SDC_ENTER(h);
  if (n < 1 || n > h->n_max) { set_err("n=%d outside [1, n_max=%d]", n, h->n_max); return -3; }
  if (!A) { set_err("A is NULL"); return -4; }
  if (lda < n) { set_err("lda < n"); return -5; }
  if (key_off < 0) { set_err("key_off < 0"); return -6; }
  if (leaf < 1) { set_err("leaf < 1"); return -7; }
  if (max_iters < 1 || max_iters > MAX_HIST) { set_err("max_iters out of range"); return -9; }
  if (!(tol >= 0.0)) { set_err("tol < 0"); return -10; }
  if (!Q) { set_err("Q is NULL"); return -11; }
  if (ldq < n) { set_err("ldq < n"); return -12; }
  if (!T) { set_err("T is NULL"); return -13; }
  if (ldt < n) { set_err("ldt < n"); return -14; }
  if (!blk_off || !blk_size || !nblk || !stats || !max_metric) { set_err("NULL host output"); return -15; }
  Nvtx nv("sdc_schur");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  h->st = st;
  // workspace of this call: V / Gaussian, Q_b, Ahat_b, product scratch, scalars
  double *Vb = nullptr, *Gb = nullptr, *Qb = nullptr, *Ab = nullptr, *W = nullptr, *sc = nullptr;
  const size_t nn = (size_t)n * n;
  auto cleanup = [&]() {
    for (double* p : {Vb, Gb, Qb, Ab, W, sc}) if (p) cudaFree(p);
  };
  if (cudaMalloc(&Vb, nn * 8) || cudaMalloc(&Gb, nn * 8) || cudaMalloc(&Qb, nn * 8) ||
      cudaMalloc(&Ab, nn * 8) || cudaMalloc(&W, nn * 8) || cudaMalloc(&sc, 64)) {
    cleanup();
    set_err("sdc_schur: out of device memory");
    return SDC_ERR_NOMEM;
  }
  const SchurScratch wk{Vb, Gb, Ab, sc};
  auto run = [&]() -> int {
    k_copy<<<ew_grid((long long)nn), 256, 0, st>>>(T, ldt, A, lda, n, n, 1.0);
    SDC_LAUNCHED(h);
    k_set_identity<<<ew_grid((long long)nn), 256, 0, st>>>(Q, ldq, n, n, 1.0);
    SDC_LAUNCHED(h);
    for (int q = 0; q < 4; ++q) stats[q] = 0;
    *max_metric = 0.0;
    std::vector<std::pair<int, int>> stack{{0, n}}, small, blocks;
    while (!stack.empty()) {
      const int o = stack.back().first, m = stack.back().second;
      stack.pop_back();
      // blocks of order <= 64 wait for the batched waves below (one launch per recursion level)
      if (h->schur_batch && m <= BAT_NMAX) { small.push_back({o, m}); continue; }
      int r = 0;
      SDC_TRY(schur_node(h, st, m, T + o + (long long)o * ldt, ldt, key_off + o, leaf, seed, max_iters, tol,
                         Qb, m, wk, &r, stats, max_metric));
      if (r == 0) { blocks.push_back({o, m}); continue; }
      const int nr = n - o - m;
      if (nr > 0) {   // T(o:o+m, o+m:n) = Qb^T T(o:o+m, o+m:n)
        double* Tr = T + o + (long long)(o + m) * ldt;
        SDC_TRY(gemm_tn(h, m, nr, m, 1.0, Qb, m, Tr, ldt, 0.0, W, m));
        k_copy<<<ew_grid((long long)m * nr), 256, 0, st>>>(Tr, ldt, W, m, m, nr, 1.0);
        SDC_LAUNCHED(h);
      }
      if (o > 0) {    // T(0:o, o:o+m) = T(0:o, o:o+m) Qb
        double* Tu = T + (long long)o * ldt;
        SDC_TRY(gemm_general(h, false, false, o, m, m, 1.0, Tu, ldt, Qb, m, 0.0, W, o));
        k_copy<<<ew_grid((long long)o * m), 256, 0, st>>>(Tu, ldt, W, o, o, m, 1.0);
        SDC_LAUNCHED(h);
      }
      {               // Q(:, o:o+m) = Q(:, o:o+m) Qb
        double* Qc = Q + (long long)o * ldq;
        SDC_TRY(gemm_general(h, false, false, n, m, m, 1.0, Qc, ldq, Qb, m, 0.0, W, n));
        k_copy<<<ew_grid((long long)n * m), 256, 0, st>>>(Qc, ldq, W, n, n, m, 1.0);
        SDC_LAUNCHED(h);
      }
      stack.push_back({o + r, m - r});   // trailing (Re < a), processed second
      stack.push_back({o, r});           // leading (Re > a), processed first
    }
    SDC_TRY(schur_small_waves(h, st, n, T, ldt, Q, ldq, key_off, leaf, seed, max_iters, tol, small, blocks,
                              stats, max_metric));
    std::sort(blocks.begin(), blocks.end());   // by offset: the order of the depth-first recursion
    for (size_t i = 0; i < blocks.size(); ++i) { blk_off[i] = blocks[i].first; blk_size[i] = blocks[i].second; }
    *nblk = (int)blocks.size();
    SDC_CK(cudaStreamSynchronize(st));
    return 0;
  };
  const int rc = run();
  cleanup();
  return rc;
}

int sdc_schur(sdc_handle* h, void* stream, int n, const double* A, int lda, int leaf,
              unsigned long long seed, int max_iters, double tol, double* Q, int ldq, double* T,
              int ldt, int* blk_off, int* blk_size, int* nblk, int* stats, double* max_metric) {
  const int rc = sdc_schur_keyed(h, stream, n, A, lda, 0, leaf, seed, max_iters, tol, Q, ldq, T, ldt, blk_off,
                                 blk_size, nblk, stats, max_metric);
  return rc <= -6 && rc >= -15 ? rc + 1 : rc;   // argument positions of this signature
}

int sdc_schur_node(sdc_handle* h, void* stream, int m, double* Tb, int ldtb, int key_off, int leaf,
                   unsigned long long seed, int max_iters, double tol, double* Qb, int ldqb, int* r,
                   int* stats, double* max_metric) {
  SDC_ENTER(h);
  if (m < 1 || m > h->n_max) { set_err("m=%d outside [1, n_max=%d]", m, h->n_max); return -3; }
  if (!Tb) { set_err("Tb is NULL"); return -4; }
  if (ldtb < m) { set_err("ldtb < m"); return -5; }
  if (key_off < 0) { set_err("key_off < 0"); return -6; }
  if (leaf < 1) { set_err("leaf < 1"); return -7; }
  if (max_iters < 1 || max_iters > MAX_HIST) { set_err("max_iters out of range"); return -9; }
  if (!(tol >= 0.0)) { set_err("tol < 0"); return -10; }
  if (!Qb) { set_err("Qb is NULL"); return -11; }
  if (ldqb < m) { set_err("ldqb < m"); return -12; }
  if (!r || !stats || !max_metric) { set_err("NULL host output"); return -13; }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  h->st = st;
  if (h->schur_batch && m <= BAT_NMAX) {
    // the same kernel (and so the same decisions) as the batched waves of sdc_schur_keyed
    *r = 0;
    if (m <= leaf || m < 2) return 0;
    SchurWave w;
    struct Guard { SchurWave& w; ~Guard() { w.release(); } } guard{w};
    const int off0 = 0;
    int rr = 0, sst[4] = {0, 0, 0, 0};
    double met = 0.0;
    // key_off is the block's own global offset (its local offset in Tb is 0)
    SDC_TRY(schur_leaves_launch(h, st, w, Tb, ldtb, key_off, leaf, seed, max_iters, tol, &off0, &m, 1,
                                (m + 15) & ~15, &rr, sst, &met));
    SDC_CK(cudaStreamSynchronize(st));
    for (int q = 0; q < 4; ++q) stats[q] += sst[q];
    if (rr > 0) {
      *max_metric = std::max(*max_metric, met);
      SDC_CK(cudaMemcpy2DAsync(Qb, sizeof(double) * ldqb, w.scratch + 3 * BAT_NMAX * BAT_NMAX, sizeof(double) * m,
                               sizeof(double) * m, m, cudaMemcpyDeviceToDevice, st));
      SDC_CK(cudaStreamSynchronize(st));
    }
    *r = rr;
    return 0;
  }
  double *Vb = nullptr, *Gb = nullptr, *Ab = nullptr, *sc = nullptr;
  const size_t mm = (size_t)m * m;
  int rc = 0;
  if (cudaMalloc(&Vb, mm * 8) || cudaMalloc(&Gb, mm * 8) || cudaMalloc(&Ab, mm * 8) || cudaMalloc(&sc, 64)) {
    set_err("sdc_schur_node: out of device memory");
    rc = SDC_ERR_NOMEM;
  } else {
    rc = schur_node(h, st, m, Tb, ldtb, key_off, leaf, seed, max_iters, tol, Qb, ldqb, SchurScratch{Vb, Gb, Ab, sc},
                    r, stats, max_metric);
    if (!rc) { cudaError_t e = cudaStreamSynchronize(st); if (e != cudaSuccess) { set_err("%s", cudaGetErrorString(e)); rc = SDC_ERR_CUDA; } }
  }
  for (double* p : {Vb, Gb, Ab, sc}) if (p) cudaFree(p);
  return rc;
}

int sdc_split_batched(sdc_handle* h, void* stream, int batch, int n, const double* A, int lda,
                      long long strideA, const double* V, int ldv, long long strideV, int max_iters,
                      double* Q, int ldq, long long strideQ, sdc_result* res) {
  SDC_ENTER(h);
  if (batch < 0) { set_err("batch < 0"); return -3; }
  if (n < 2 || n > BAT_NMAX) { set_err("batched n=%d outside [2, %d]", n, BAT_NMAX); return -4; }
  if (!A && batch) { set_err("A is NULL"); return -5; }
  if (lda < n) { set_err("lda < n"); return -6; }
  if (strideA < (long long)lda * n) { set_err("strideA < lda n"); return -7; }
  if (!V && batch) { set_err("V is NULL"); return -8; }
  if (ldv < n) { set_err("ldv < n"); return -9; }
  if (strideV < (long long)ldv * n) { set_err("strideV < ldv n"); return -10; }
  if (max_iters < 1) { set_err("max_iters < 1"); return -11; }
  if (!Q && batch) { set_err("Q is NULL"); return -12; }
  if (ldq < n) { set_err("ldq < n"); return -13; }
  if (strideQ < (long long)ldq * n) { set_err("strideQ < ldq n"); return -14; }
  if (!res && batch) { set_err("res is NULL"); return -15; }
  if (batch == 0) return 0;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  h->st = st;
  static DevOnce attr;
  if (!attr.has(h->device)) {
    SDC_CK(cudaFuncSetAttribute(k_split_batched_wy, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)bq_smem_bytes(BAT_NMAX)));
    attr.set(h->device);
  }
  if ((size_t)batch * 4 > h->bat_out_n) {
    if (h->bat_out) cudaFree(h->bat_out);
    h->bat_out = nullptr;
    h->bat_out_n = 0;
    if (cudaMalloc(&h->bat_out, (size_t)batch * 4 * sizeof(double)) != cudaSuccess) {
      set_err("sdc_split_batched: out of memory");
      return SDC_ERR_NOMEM;
    }
    h->bat_out_n = (size_t)batch * 4;
  }
  BatArgs a{A, lda, strideA, V, ldv, strideV, Q, ldq, strideQ, h->bat_out, n, max_iters};
  k_split_batched_wy<<<batch, BQ_THREADS, bq_smem_bytes(n), st>>>(a);
  SDC_LAUNCHED(h);
  std::vector<double> out((size_t)batch * 4);
  SDC_CK(cudaMemcpyAsync(out.data(), h->bat_out, out.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
  SDC_CK(cudaStreamSynchronize(st));
  for (int b = 0; b < batch; ++b) {
    sdc_result& r = res[b];
    r.r = (int)out[4 * b];
    r.k = n - r.r;
    r.metric = out[4 * b + 1];
    r.metric_fro = out[4 * b + 2];
    r.iters = max_iters;
    r.converged = 0;
    r.side = NAN;
    r.status = (out[4 * b + 3] != 0.0 || !std::isfinite(r.metric)) ? SDC_STATUS_NONFINITE
               : (r.metric <= SDC_SPLIT_ACCEPT ? SDC_STATUS_SPLIT : SDC_STATUS_NO_SPLIT);
  }
  return 0;
}

int sdc_trevc(sdc_handle* h, void* stream, int n, const double* T, int ldt, const double* Q,
              int ldq, double* X, int ldx) {
  SDC_ENTER(h);
  if (n < 1 || n > h->n_max) { set_err("n=%d outside [1, n_max=%d]", n, h->n_max); return -3; }
  if (!T) { set_err("T is NULL"); return -4; }
  if (ldt < n) { set_err("ldt < n"); return -5; }
  if (Q && ldq < n) { set_err("ldq < n"); return -7; }
  if (!X) { set_err("X is NULL"); return -8; }
  if (ldx < n) { set_err("ldx < n"); return -9; }
  h->st = static_cast<cudaStream_t>(stream);
  double* Xw = Q ? h->G2 : X;                  // X_T (the eigenvectors of T)
  const long long ldw = Q ? n : ldx;
  SDC_CK(cudaMemset2DAsync(Xw, ldw * sizeof(double), 0, (size_t)n * sizeof(double), n, h->st));
  double* Tt = h->G1;                          // T^T: K-major A operand of S = T[i,:] X
  SDC_TRY(transpose_rev(h, Tt, n, T, ldt, n, 0));
  const int nblk = cdiv(n, TREVC_B);
  for (int ib = nblk - 1; ib >= 0; --ib) {
    const int i0 = ib * TREVC_B, nbk = std::min(TREVC_B, n - i0), c0 = i0 + nbk;
    const int N = n - c0;
    int splits = 1;
    if (N > 0) {   // S = T[i0:c0, c0:n] X[c0:n, c0:n]  (X upper triangular: kupper)
      const int tiles = cdiv(N, 128);
      splits = pick_splits(h, tiles, N, (long long)(h->wp_elems / ((size_t)TREVC_B * N)));
      int kchunk = cdiv(cdiv(N, splits), 16) * 16;
      splits = cdiv(N, kchunk);
      SDC_TRY(gemm_tn(h, nbk, N, N, 1.0, Tt + c0 + (long long)i0 * n, n, Xw + c0 + (long long)c0 * ldw,
                      ldw, 0.0, h->Wp, TREVC_B, nullptr, 0, 0.0, splits, kchunk,
                      (long long)TREVC_B * N, 1));
    }
    const int cols = n - i0;
    ProfScope ps(h, SDC_PROF_TREVC, 8.0 * ((double)nbk * nbk + (double)cols * (nbk * (splits + 1))));
    k_trevc_block<<<std::min(cdiv(cols, 8), h->num_sms * 8), 256, 0, h->st>>>(
        T, ldt, i0, nbk, i0, n, h->Wp, splits, (long long)TREVC_B * N, TREVC_B, c0, Xw, ldw, n);
    SDC_LAUNCHED(h);
  }
  if (Q) {   // eigenvectors of A = Q T Q^T: X = Q X_T (TN: A_s = Q^T; X_T upper triangular)
    double* Qt = h->G3;
    SDC_TRY(transpose_rev(h, Qt, n, Q, ldq, n, 0));
    SDC_TRY(gemm_tn(h, n, n, n, 1.0, Qt, n, Xw, ldw, 0.0, X, ldx, nullptr, 0, 0.0, 1, 0, 0, 1));
  }
  return 0;
}

int sdc_svd_split(sdc_handle* h, void* stream, int m, int n, const double* A, int lda, double rho,
                  const double* V, int ldv, int max_iters, double tol, int stop_mode, double* Q,
                  int ldq, double* Ahat, int ldah, double* hist, int hist_cap, sdc_result* res) {
  SDC_ENTER(h);
  if (m < 1) { set_err("m < 1"); return -3; }
  if (n < 1) { set_err("n < 1"); return -4; }
  if (m + n > h->n_max) { set_err("m + n = %d exceeds n_max = %d", m + n, h->n_max); return -4; }
  if (!A) { set_err("A is NULL"); return -5; }
  if (lda < m) { set_err("lda < m"); return -6; }
  if (!(rho > 0.0) || !std::isfinite(rho)) { set_err("rho must be finite and > 0"); return -7; }
  const int N = m + n;
  if (!h->Emb) SDC_TRY(dalloc(h, &h->Emb, (size_t)h->n_max * h->n_max));
  h->st = static_cast<cudaStream_t>(stream);
  k_embed<<<ew_grid((long long)N * N), 256, 0, h->st>>>(h->Emb, A, lda, m, n);
  SDC_LAUNCHED(h);
  const int rc = sdc_split_region(h, stream, N, h->Emb, N, nullptr, 0, V, ldv, nullptr, 0,
                                  SDC_REGION_DISK, rho, SDC_FLAG_SYMMETRIC, max_iters, tol, stop_mode,
                                  Q, ldq, nullptr, 0, Ahat, ldah, hist, hist_cap, res);
  // argument positions of the inner call map back onto this signature
  if (rc == -8) return -8;
  if (rc == -9) return -9;
  if (rc == -13) return -10;
  if (rc == -14) return -11;
  if (rc == -15) return -12;
  if (rc == -16) return -13;
  if (rc == -17) return -14;
  if (rc == -21) return -16;
  if (rc == -23) return -18;
  if (rc == -24) return -19;
  return rc;
}

int sdc_split_region(sdc_handle* h, void* stream, int n, const double* A, int lda, const double* B,
                     int ldb, const double* V, int ldv, const double* VL, int ldvl, int region,
                     double region_param, int flags, int max_iters, double tol, int stop_mode,
                     double* Q, int ldq, double* QL, int ldql, double* Ahat, int ldah, double* hist,
                     int hist_cap, sdc_result* res) {
  SDC_ENTER(h);
  if (region < 0 || region > 2) { set_err("unknown region %d", region); return -12; }
  if (region == SDC_REGION_DISK && !(region_param > 0.0)) { set_err("disk radius must be > 0"); return -13; }
  if (region == SDC_REGION_HALFPLANE && !std::isfinite(region_param)) { set_err("bad half-plane abscissa"); return -13; }
  if ((region == SDC_REGION_HALFPLANE || (flags & SDC_FLAG_SYMMETRIC)) && B) {
    set_err("half-plane regions and the symmetric flag take B = NULL (B = I)");
    return -6;
  }
  if (flags & ~(SDC_FLAG_SYMMETRIC | SDC_FLAG_PLATEAU | SDC_FLAG_ONESIDED | SDC_FLAG_QL_ORTH)) {
    set_err("unknown flags");
    return -14;
  }
  if ((flags & SDC_FLAG_QL_ORTH) && !B) { set_err("SDC_FLAG_QL_ORTH needs a pencil (B != NULL)"); return -6; }
  h->ql_orth = (flags & SDC_FLAG_QL_ORTH) != 0;
  h->region = region;
  h->rparam = region == SDC_REGION_UNIT_DISK ? 1.0 : region_param;
  h->rflags = flags;
  if (n < 2 || n > h->n_max) { set_err("n=%d outside [2, n_max=%d]", n, h->n_max); return -3; }
  if (!A) { set_err("A is NULL"); return -4; }
  if (lda < n) { set_err("lda < n"); return -5; }
  const bool pencil = B != nullptr;
  if (pencil && ldb < n) { set_err("ldb < n"); return -7; }
  if (pencil && !h->pencil) { set_err("handle created without pencil workspace"); return -6; }
  if (!V) { set_err("V is NULL"); return -8; }
  if (ldv < n) { set_err("ldv < n"); return -9; }
  if (pencil && !h->ql_orth && !VL) { set_err("VL is NULL for a pencil"); return -10; }
  if (pencil && !h->ql_orth && ldvl < n) { set_err("ldvl < n"); return -11; }
  if (max_iters < 1 || max_iters > MAX_HIST) { set_err("max_iters out of range"); return -13; }
  if (!(tol >= 0.0)) { set_err("tol < 0"); return -14; }
  if (stop_mode < 0 || stop_mode > 2) { set_err("unknown stop mode"); return -15; }
  if (!Q) { set_err("Q is NULL"); return -16; }
  if (ldq < n) { set_err("ldq < n"); return -17; }
  if (pencil && !QL) { set_err("QL is NULL for a pencil"); return -18; }
  if (QL && ldql < n) { set_err("ldql < n"); return -19; }
  if (Ahat && ldah < n) { set_err("ldah < n"); return -21; }
  if (hist_cap < 0 || (hist_cap > 0 && !hist)) { set_err("bad hist"); return -23; }
  if (!res) { set_err("res is NULL"); return -24; }
  if (stop_mode == SDC_STOP_E21 || (pencil && !h->ql_orth)) SDC_TRY(ensure_alt(h));
  choose_nbo(h, n, pencil && !h->ql_orth && h->alt_ready);
  h->st = static_cast<cudaStream_t>(stream);
  h->cur_V = V; h->cur_ldv = ldv; h->cur_VL = VL; h->cur_ldvl = ldvl;
  const bool pencil_ = pencil;
  double* QLd = pencil_ ? h->QLb : nullptr;
  std::vector<double> hbuf;
  if (hist_cap > 0) hbuf.assign((size_t)hist_cap * 3, NAN);
  int p = max_iters, conv = 0;

  if (stop_mode == SDC_STOP_FIXED) {
    // whole step enqueued without host syncs; captured once into a CUDA graph (n <= graph_max_n)
    // and replayed while the call signature is unchanged
    sdc_handle::GraphKey key;
    key.n = n; key.max_iters = max_iters; key.nbo = h->nbo;
    key.region = h->region; key.rflags = h->rflags; key.rparam = h->rparam;
    key.A = A; key.B = B; key.V = V; key.VL = VL; key.Q = Q; key.QL = QL; key.Ahat = Ahat;
    key.lda = lda; key.ldb = ldb; key.ldv = ldv; key.ldvl = ldvl; key.ldq = ldq; key.ldql = ldql;
    key.ldah = ldah;
    const bool graph = n <= h->graph_max_n && !h->prof_on;
    if (graph && h->gexec && key == h->gkey) {
      SDC_CK(cudaGraphLaunch(h->gexec, h->st));
      h->launches += h->glaunches;
      h->sched[SDC_SCHED_GRAPH_REPLAYS]++;
    } else if (graph) {
      if (h->gexec) { cudaGraphExecDestroy(h->gexec); h->gexec = nullptr; }
      const long long l0 = h->launches;
      cudaStream_t user = h->st;           // capture on the handle's own stream (the legacy
      h->st = h->cap_st;                   // default stream cannot be captured), launch on user's
      SDC_CK(cudaStreamBeginCapture(h->st, cudaStreamCaptureModeRelaxed));
      int rc = enqueue_fixed(h, n, A, lda, B, ldb, Q, ldq, QLd, QL, ldql, Ahat, ldah, max_iters);
      cudaGraph_t g = nullptr;
      cudaError_t ec = cudaStreamEndCapture(h->st, &g);
      h->st = user;
      if (rc) { if (g) cudaGraphDestroy(g); return rc; }
      if (ec != cudaSuccess) { set_err("graph capture: %s", cudaGetErrorString(ec)); return SDC_ERR_CUDA; }
      cudaError_t ei = cudaGraphInstantiate(&h->gexec, g, 0);
      cudaGraphDestroy(g);
      if (ei != cudaSuccess) { h->gexec = nullptr; set_err("graph instantiate: %s", cudaGetErrorString(ei)); return SDC_ERR_CUDA; }
      h->gkey = key;
      h->glaunches = h->launches - l0;
      h->sched[SDC_SCHED_GRAPH_CAPTURES]++;
      SDC_CK(cudaGraphLaunch(h->gexec, h->st));
    } else {
      SDC_TRY(enqueue_fixed(h, n, A, lda, B, ldb, Q, ldq, QLd, QL, ldql, Ahat, ldah, max_iters));
    }
  } else if (stop_mode == SDC_STOP_E21 && h->alt_ready && !(pencil && !h->ql_orth)) {
    // monitor mode, pipelined: GRURV(j) + similarity + selection of pass j run on the second
    // context while IRS pass j+1 runs on the caller's stream (issued before the host reads
    // pass j's metric; if pass j stops, that pass is discarded).  Same kernels on the same
    // inputs as the sequential order, so the results are bit-identical to it.
    const long long ld = wld(n);
    struct Share {   // GRURV(j) panels on the second context run next to pass j+1's panels
      sdc_handle* h;
      explicit Share(sdc_handle* h_) : h(h_) {
        h->share_sms = true;
        h->two_chains = true;   // one-tile update CTAs in both chains, as for the pencil's (config 3: -1%)
      }
      ~Share() { h->share_sms = false; h->two_chains = false; }
    } share(h);
    SDC_TRY(enqueue_init(h, n, A, lda, B, ldb, V, ldv, VL, ldvl));
    int cur = 0;
    bool have_split = false;
    double prev = INFINITY;
    SDC_TRY(irs_pass(h, n, h->A[0], ld, h->B[0], ld, h->A[1], ld, h->B[1], ld, h->S, 0, nullptr, 0));
    for (int j = 0; j < max_iters; ++j) {
      const int cj = cur ^ 1;   // buffers holding the output of pass j
      if ((flags & SDC_FLAG_ONESIDED) && j >= 2) {
        SDC_TRY(norms(h, h->A[cj], ld, n, h->scal + 8));
        SDC_TRY(norms(h, h->B[cj], ld, n, h->scal + 10));
        SDC_CK(cudaMemcpyAsync(h->hscal, h->scal + 8, 4 * sizeof(double), cudaMemcpyDeviceToHost, h->st));
        SDC_CK(cudaStreamSynchronize(h->st));
        const double fa = h->hscal[1], fb = h->hscal[3];
        const double sd = fa + fb > 0.0 ? fb / (fa + fb) : 0.5;
        if (sd < 1e-6 || sd > 1.0 - 1e-6) { cur = cj; p = j + 1; break; }
      }
      SDC_TRY(stream_dep(h, h->st, h->alt.st, h->ev_a));
      {
        AltScope as(h);
        SDC_TRY(grurv_right(h, n, h->A[cj], h->B[cj], h->Vt, Q, ldq));
        if (pencil) SDC_TRY(ql_from_aq(h, n, A, lda, Q, ldq, QLd, ld));
        SDC_TRY(similarity_select(h, n, A, lda, B, ldb, Q, ldq, pencil ? QLd : Q, pencil ? ld : ldq));
        SDC_CK(cudaMemcpyAsync(h->hscal + 16, h->scal + 4, 2 * sizeof(double), cudaMemcpyDeviceToHost, h->st));
        SDC_CK(cudaEventRecord(h->ev_b, h->st));
      }
      have_split = true;
      // next pass (reads pass j's output, overwrites pass j-1's, whose GRURV has completed)
      if (j + 1 < max_iters)
        SDC_TRY(irs_pass(h, n, h->A[cj], ld, h->B[cj], ld, h->A[cur], ld, h->B[cur], ld, h->S, j + 1,
                         nullptr, 0));
      cur = cj;
      SDC_CK(cudaEventSynchronize(h->ev_b));
      const double r_j = h->hscal[16], m_j = h->hscal[17];
      if (j < hist_cap) { hbuf[3 * j] = r_j; hbuf[3 * j + 1] = m_j; }
      if (m_j <= tol) { p = j + 1; conv = 1; break; }
      if ((flags & SDC_FLAG_PLATEAU) && m_j <= 10.0 * tol && m_j > 0.5 * prev) { p = j + 1; conv = 1; break; }
      prev = m_j;
    }
    SDC_TRY(stream_dep(h, h->alt.st, h->st, h->ev_c));
    SDC_TRY(enqueue_finish(h, n, A, lda, B, ldb, Q, ldq, QLd, QL, ldql, Ahat, ldah, have_split, cur, max_iters));
  } else {
    // RTEST / E21: host decisions between passes (one scalar D2H per pass)
    const long long ld = wld(n);
    SDC_TRY(enqueue_init(h, n, A, lda, B, ldb, V, ldv, VL, ldvl));
    int cur = 0;
    bool have_split = false;
    double prev = INFINITY;
    for (int j = 0; j < max_iters; ++j) {
      SDC_TRY(irs_pass(h, n, h->A[cur], ld, h->B[cur], ld, h->A[cur ^ 1], ld, h->B[cur ^ 1], ld, h->S,
                       j, nullptr, 0));
      if (pencil && !h->ql_orth)
        SDC_TRY(irs_pass(h, n, h->AL[cur], ld, h->BL[cur], ld, h->AL[cur ^ 1], ld, h->BL[cur ^ 1], ld,
                         h->SL, -1, nullptr, 0));
      cur ^= 1;
      if ((flags & SDC_FLAG_ONESIDED) && stop_mode == SDC_STOP_E21 && j >= 2) {
        // every eigenvalue on one side: one of A_p, B_p vanishes relative to the other
        SDC_TRY(norms(h, h->A[cur], ld, n, h->scal + 8));
        SDC_TRY(norms(h, h->B[cur], ld, n, h->scal + 10));
        SDC_CK(cudaMemcpyAsync(h->hscal, h->scal + 8, 4 * sizeof(double), cudaMemcpyDeviceToHost, h->st));
        SDC_CK(cudaStreamSynchronize(h->st));
        const double fa = h->hscal[1], fb = h->hscal[3];
        const double sd = fa + fb > 0.0 ? fb / (fa + fb) : 0.5;
        if (sd < 1e-6 || sd > 1.0 - 1e-6) { p = j + 1; break; }
      }
      if (stop_mode == SDC_STOP_RTEST && j >= 1) {
        SDC_CK(cudaMemcpyAsync(h->hscal, h->scal + SCAL_HIST + j, sizeof(double), cudaMemcpyDeviceToHost, h->st));
        SDC_CK(cudaStreamSynchronize(h->st));
        if (h->hscal[0] <= tol) { p = j + 1; conv = 1; break; }
      }
      if (stop_mode == SDC_STOP_E21) {
        SDC_TRY(grurv_right(h, n, h->A[cur], h->B[cur], h->Vt, Q, ldq));
        if (pencil && h->ql_orth) SDC_TRY(ql_from_aq(h, n, A, lda, Q, ldq, QLd, ld));
        else if (pencil) SDC_TRY(grurv_left(h, n, h->AL[cur], h->BL[cur], h->VLt, QLd, ld));
        SDC_TRY(similarity_select(h, n, A, lda, B, ldb, Q, ldq, pencil ? QLd : Q, pencil ? ld : ldq));
        have_split = true;
        SDC_CK(cudaMemcpyAsync(h->hscal, h->scal + 4, 2 * sizeof(double), cudaMemcpyDeviceToHost, h->st));
        SDC_CK(cudaStreamSynchronize(h->st));
        if (j < hist_cap) { hbuf[3 * j] = h->hscal[0]; hbuf[3 * j + 1] = h->hscal[1]; }
        if (h->hscal[1] <= tol) { p = j + 1; conv = 1; break; }
        // plateau: a metric within 10 tol that no longer halves -- the rounding floor
        if ((flags & SDC_FLAG_PLATEAU) && h->hscal[1] <= 10.0 * tol && h->hscal[1] > 0.5 * prev) {
          p = j + 1; conv = 1; break;
        }
        prev = h->hscal[1];
      }
    }
    SDC_TRY(enqueue_finish(h, n, A, lda, B, ldb, Q, ldq, QLd, QL, ldql, Ahat, ldah, have_split, cur, max_iters));
  }
  SDC_CK(cudaStreamSynchronize(h->st));
  if (h->hflags[1] || h->hflags[2]) { set_err("panel grid barrier timed out (co-residency violated?)"); return SDC_ERR_CUDA; }
  note_split_breakdowns(h, h->hflags[3] + h->hflags[4]);
  const double* sc = h->hscal;
  for (int j = 1; j < std::min(hist_cap, p); ++j) hbuf[3 * j + 2] = sc[SCAL_HIST + j];
  if (hist_cap > 0) memcpy(hist, hbuf.data(), sizeof(double) * hbuf.size());
  res->r = (int)sc[4];
  res->k = n - res->r;
  res->metric = sc[5];
  res->metric_fro = sc[6];
  res->iters = p;
  res->converged = conv;
  res->side = sc[9] + sc[11] > 0.0 ? sc[11] / (sc[9] + sc[11]) : 0.5;
  res->status = (h->hflags[0] || !std::isfinite(res->metric)) ? SDC_STATUS_NONFINITE
               : (res->metric <= SDC_SPLIT_ACCEPT ? SDC_STATUS_SPLIT : SDC_STATUS_NO_SPLIT);
  return 0;
}

int sdc_split_host(sdc_handle* h, void* stream, int n, const double* A, const double* B,
                   const double* V, const double* VL, int max_iters, double tol, int stop_mode,
                   double* Q, double* QL, double* Ahat, double* hist, int hist_cap,
                   sdc_result* res) {
  SDC_ENTER(h);
  if (n < 2 || n > h->n_max) { set_err("n=%d outside [2, n_max=%d]", n, h->n_max); return -3; }
  if (!A || !V || !Q || (B && !VL) || (B && !QL)) { set_err("null host pointer"); return -4; }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t nn = (size_t)h->n_max * h->n_max, bytes = sizeof(double) * (size_t)n * n;
  int rc = 0;
  if (!h->hA) { rc = dalloc(h, &h->hA, nn); if (!rc) rc = dalloc(h, &h->hV, nn); if (!rc) rc = dalloc(h, &h->hQ, nn); }
  if (!rc && B && !h->hB) { rc = dalloc(h, &h->hB, nn); if (!rc) rc = dalloc(h, &h->hVL, nn); if (!rc) rc = dalloc(h, &h->hQL, nn); }
  if (!rc && Ahat && !h->hAh) rc = dalloc(h, &h->hAh, nn);
  if (rc) return rc;
  SDC_CK(cudaMemcpyAsync(h->hA, A, bytes, cudaMemcpyHostToDevice, st));
  SDC_CK(cudaMemcpyAsync(h->hV, V, bytes, cudaMemcpyHostToDevice, st));
  if (B) {
    SDC_CK(cudaMemcpyAsync(h->hB, B, bytes, cudaMemcpyHostToDevice, st));
    SDC_CK(cudaMemcpyAsync(h->hVL, VL, bytes, cudaMemcpyHostToDevice, st));
  }
  SDC_TRY(sdc_split(h, stream, n, h->hA, n, B ? h->hB : nullptr, n, h->hV, n, B ? h->hVL : nullptr, n,
                    SDC_REGION_UNIT_DISK, max_iters, tol, stop_mode, h->hQ, n, B ? h->hQL : nullptr, n,
                    Ahat ? h->hAh : nullptr, n, hist, hist_cap, res));
  SDC_CK(cudaMemcpyAsync(Q, h->hQ, bytes, cudaMemcpyDeviceToHost, st));
  if (B) SDC_CK(cudaMemcpyAsync(QL, h->hQL, bytes, cudaMemcpyDeviceToHost, st));
  if (Ahat) SDC_CK(cudaMemcpyAsync(Ahat, h->hAh, bytes, cudaMemcpyDeviceToHost, st));
  SDC_CK(cudaStreamSynchronize(st));
  return 0;
}

int sdc_dgemm(sdc_handle* h, void* stream, int transa, int transb, int M, int N, int K,
              double alpha, const double* A, int lda, const double* B, int ldb, double beta,
              double* C, int ldc) {
  SDC_ENTER(h);
  if (M < 0) { set_err("invalid argument (M < 0)"); return -5; }
  if (N < 0) { set_err("invalid argument (N < 0)"); return -6; }
  if (K < 0) { set_err("invalid argument (K < 0)"); return -7; }
  if (lda < std::max(1, transa ? K : M)) { set_err("invalid argument (lda < std::max(1, transa ? K : M))"); return -10; }
  if (ldb < std::max(1, transb ? N : K)) { set_err("invalid argument (ldb < std::max(1, transb ? N : K))"); return -12; }
  if (ldc < std::max(1, M)) { set_err("invalid argument (ldc < std::max(1, M))"); return -15; }
  h->st = static_cast<cudaStream_t>(stream);
  return gemm_general(h, transa != 0, transb != 0, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
}

int sdc_qr(sdc_handle* h, void* stream, int m, int n, double* A, int lda, double* Qthin, int ldq) {
  SDC_ENTER(h);
  if (m < n || m > 2 * h->n_max) { set_err("invalid argument (m < n || m > 2 * h->n_max)"); return -3; }
  if (n < 1 || n > h->n_max) { set_err("invalid argument (n < 1 || n > h->n_max)"); return -4; }
  if (lda < m) { set_err("invalid argument (lda < m)"); return -6; }
  if (Qthin && ldq < m) { set_err("invalid argument (Qthin && ldq < m)"); return -8; }
  choose_nbo(h, n);
  h->st = static_cast<cudaStream_t>(stream);
  SDC_TRY(reset_sync(h));
  const Fac f{h->Y, wld(m), h->Yt, wld(n)};
  SDC_TRY(blocked_qr(h, A, lda, m, n, f));
  if (Qthin) {
    k_set_identity<<<ew_grid((long long)m * n), 256, 0, h->st>>>(Qthin, ldq, m, n, 1.0);
    SDC_LAUNCHED(h);
    SDC_TRY(apply_q(h, m, n, f, Qthin, ldq, n));
    k_col_sign<<<ew_grid((long long)m * n), 256, 0, h->st>>>(Qthin, ldq, m, n, A, lda);
    SDC_LAUNCHED(h);
  }
  // rows of R scaled by sign(R_ii): R with a non-negative diagonal (after Q's column signs,
  // which read the original diagonal)
  k_r_rows_nonneg<<<cdiv((long long)n * 32, 256), 256, 0, h->st>>>(A, lda, n);
  SDC_LAUNCHED(h);
  SDC_TRY(check_barrier(h));
  return 0;
}

int sdc_irs_pass(sdc_handle* h, void* stream, int n, const double* A, int lda, const double* B,
                 int ldb, double* Aout, int ldao, double* Bout, int ldbo, double* Rout, int ldr) {
  SDC_ENTER(h);
  if (n < 1 || n > h->n_max) { set_err("invalid argument (n < 1 || n > h->n_max)"); return -3; }
  if (!A || lda < n) { set_err("invalid argument (!A || lda < n)"); return -4; }
  if (!B || ldb < n) { set_err("invalid argument (!B || ldb < n)"); return -6; }
  if (!Aout || ldao < n) { set_err("invalid argument (!Aout || ldao < n)"); return -8; }
  if (!Bout || ldbo < n) { set_err("invalid argument (!Bout || ldbo < n)"); return -10; }
  if (Rout && ldr < n) { set_err("invalid argument (Rout && ldr < n)"); return -13; }
  choose_nbo(h, n);
  h->st = static_cast<cudaStream_t>(stream);
  const long long m = 2LL * n;
  SDC_TRY(reset_sync(h));
  k_build_stack<<<ew_grid(m * n), 256, 0, h->st>>>(h->S, m, A, lda, B, ldb, n);
  SDC_LAUNCHED(h);
  h->b_ident = nullptr;
  SDC_TRY(irs_pass(h, n, A, lda, B, ldb, Aout, ldao, Bout, ldbo, h->S, -1, Rout, ldr));
  SDC_TRY(check_barrier(h));
  return 0;
}

int sdc_split_select(sdc_handle* h, void* stream, int n, const double* Ahat, int ldah,
                     double normA, const double* Bhat, int ldbh, double normB, int* r,
                     double* metric, double* mvals) {
  SDC_ENTER(h);
  if (n < 2 || n > h->n_max) { set_err("invalid argument (n < 2 || n > h->n_max)"); return -3; }
  if (!Ahat || ldah < n) { set_err("invalid argument (!Ahat || ldah < n)"); return -4; }
  if (Bhat && (ldbh < n || !h->pencil)) { set_err("invalid argument (Bhat && (ldbh < n || !h->pencil))"); return -7; }
  if (!r || !metric) { set_err("invalid argument (!r || !metric)"); return -10; }
  h->st = static_cast<cudaStream_t>(stream);
  double nr[4] = {normA, 0.0, normB, 0.0};
  SDC_CK(cudaMemcpyAsync(h->scal, nr, sizeof(nr), cudaMemcpyHostToDevice, h->st));
  SDC_TRY(select_dev(h, n, Ahat, ldah, Bhat, ldbh, h->scal, h->scal + 2, h->scal + 4));
  double sel[2];
  SDC_CK(cudaMemcpyAsync(sel, h->scal + 4, sizeof(sel), cudaMemcpyDeviceToHost, h->st));
  if (mvals)
    SDC_CK(cudaMemcpyAsync(mvals, h->vec + 2 * h->n_max, sizeof(double) * n, cudaMemcpyDeviceToDevice, h->st));
  SDC_CK(cudaStreamSynchronize(h->st));
  *r = (int)sel[0];
  *metric = sel[1];
  return 0;
}

}  // extern "C"
