// libcpd.so: C ABI (include/cpd.h), device state, the MSDT / DT / PP schedulers and
// the 1-D-grid collectives.  Citations: P:n = PAPER.md line n.
//
// Host-side scheduling:
//  * MSDT (§III, Fig. 2): a continuous stream of factor updates t = 0,1,...
//    (mode t mod N); root k = T x_j A^(j) with j = ((k+1)(N-1)) mod N (0-based, i.e.
//    T x_N, T x_{N-1}, ..., T x_1 cyclically) serves updates t in
//    [k(N-1), (k+1)(N-1)), i.e. modes (j+1, ..., j+N-1) mod N.  Inside a subtree the
//    served list L is split binary: left = first ceil(|L|/2) modes built by contracting
//    the right ones (not yet updated), right = the rest built after the left updates
//    (reading Q5; reproduces Fig. 2 for N=4).  Nodes are built lazily, just before first
//    use, and freed when no longer an ancestor of the next leaf.
//  * DT (Fig. 1a): per sweep root T x_N (then modes ceil(N/2)+1..N-1) serves
//    1..ceil(N/2), root T x_1 (then 2..ceil(N/2), already updated) serves the rest.
//  * PP (Alg. 2, Eqs. 4-8; Alg. 4): pp_init builds every pair operator from three
//    first-level roots (one reused from the live MSDT root when still valid, P:384
//    footnote); pp_approx_sweep streams the N-1 operators of each mode (Eq. 6) and adds
//    the second-order term V (Eq. 7).
//  * Multi-GPU (Alg. 3 / Alg. 4 on the grid 1x..x1xP): local contractions, NCCL
//    reduce-scatter of the partial M^(n) (n < N-1), solve on own rows, all-gather of
//    A^(n); the last mode's rows are local, S^(N), dS^(N) and the scalars all-reduced.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <unordered_map>
#include <string>
#include <utility>
#include <vector>

#include "../../include/cpd.h"
#include "comm.h"
#include "kernels.h"

namespace {

thread_local std::string g_init_error;

constexpr int64_t kMttvWs = 1 << 22;  // doubles (32 MB) of mTTV K-split partials
constexpr int kCholMaxR = 232;        // packed Cholesky factor in one CTA's shared memory

enum Phase { PH_TTM = 0, PH_MTTV = 1, PH_SOLVE = 2, PH_HAD = 3, PH_OTHER = 4 };

struct Node {
  double* buf = nullptr;
  std::vector<int> kept;  // ascending modes; dims = ext(k)..., R
};

struct Subtree {
  int j = -1;                              // contracted mode of the root (-1: a block of modes)
  std::vector<int> served;                 // service order
  std::map<std::pair<int, int>, Node> cache;
  bool active = false;
};

struct PhaseRec {
  cudaEvent_t a, b;
  int phase;
};

}  // namespace

struct cpd_ctx {
  int N = 0, R = 0;
  int64_t shape[CPD_MAX_ORDER] = {0};
  int rank = 0, world = 1;
  // processor grid I_1 x ... x I_N (Alg. 3): this rank's coordinates x_n (row-major rank
  // order, last mode fastest) and block extents loc[n] = s_n / I_n; the 1-D default is 1 x..x 1 x P
  int grid[CPD_MAX_ORDER] = {0}, coord[CPD_MAX_ORDER] = {0};
  int64_t loc[CPD_MAX_ORDER] = {0};
  int dev = 0;
  cudaStream_t st = nullptr;
  bool own_stream = false;
  // every device allocation of the ctx comes from this private stream-ordered pool (release
  // threshold unbounded, so the node cache's repeat allocations never map memory again); the
  // process's default pool (PyTorch, other contexts) is left untouched, and cpd_destroy trims
  // and destroys the pool so all of it returns to the device
  cudaMemPool_t pool = nullptr;
  // the library's work runs on its own stream `st` (priority above the default so the PP filler
  // stream st3 never delays the critical path); `ust` is the caller's stream (opts.stream),
  // ordered before each call's work and after it by events
  cudaStream_t ust = nullptr;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  ncclComm_t comm = nullptr;
  cpd::Comm cm;              // collective backend (NCCL or in-process local group), all ranks
  // per mode: Proc-Slice(x_n) (ranks with the same x_n: reduce-scatter of M^(n), all-gather of the
  // A^(n) block) and the fiber (ranks that differ only in x_n: gathers of the global A^(n), Grams)
  cpd::Comm slice[CPD_MAX_ORDER], fiber[CPD_MAX_ORDER];
  // fused reduce-scatter epilogue (opts.fused_rs): per mode with a multi-rank slice, this
  // rank's receive buffer [slice world][own rows x R] (NCCL: ncclMemAlloc'd symmetric window) and the
  // map of its own slot in every slice peer's buffer
  double* rs_recv[CPD_MAX_ORDER] = {};
  void* rs_win[CPD_MAX_ORDER] = {};
  cpd::OutMap rs_map[CPD_MAX_ORDER] = {};
  double* bar_scratch = nullptr;
  const double* T = nullptr;
  int64_t T_elems = 0;
  cpd_opts opts{};
  // factors: mode N-1 holds only the local slab rows
  std::vector<double*> A, Aold, dA, Mlast, Ap, Mp, Mt, Mt2;
  // PP sweeps alternate between the M~ buffer sets Mt / Mt2 (mt_par): at the end of a sweep the
  // filler stream already starts the next sweep's mode-1 independent streams into the other set
  // (pp_spec); any call other than pp_approx_sweep first waits for that work and drops it
  int mt_par = 0;
  bool pp_spec = false;
  bool pp_spec0 = false;  // the next sweep's mode-0 M~ (M_p + all U^(0,i)) is also speculated
  bool pp_fresh = false;  // no approximated sweep since pp_init: dA = 0 exactly (Alg. 2 line 7)
  std::vector<double*> Mlast_src;  // non-null: the last M of mode n lives there (PP: Mt[n])
  double* S_all = nullptr;   // N x R x R
  double* dS_all = nullptr;  // N x R x R
  double* Lp[2] = {nullptr, nullptr};  // packed Cholesky factors (double-buffered)
  double* Gi[2] = {nullptr, nullptr};  // Γ^{-1} (dense, for the fused update) (double-buffered)
  double* Wb[2] = {nullptr, nullptr};  // PP second-order W (double-buffered)
  int* pf_status = nullptr;            // Cholesky status per buffer
  cudaStream_t st2 = nullptr;          // side stream: Γ factorisation / W ahead of their mode
  cudaEvent_t ev_s = nullptr, ev_pf = nullptr;
  // PP sweeps: the operator streams of mode n whose dA is already final (all i != n, n-1) run
  // on st3 while the main stream still finishes update n-1; ev_pp_a orders st3 after the main
  // stream's work so far, ev_pp_side[n] hands M_p^(n) + Σ_indep U^(n,i) back to the main stream
  cudaStream_t st3 = nullptr;
  cudaEvent_t ev_pp_a = nullptr, ev_pp_side[CPD_MAX_ORDER] = {};
  double* ws_mttv3 = nullptr;          // st3's mTTV K-split partials
  double* ws_gj = nullptr;             // grid-wide Gauss-Jordan workspace (R > kCholMaxR)
  int pf_mode = -1, pf_buf = 0;        // mode whose Γ factor (and W if pf_pp) is being prepared
  bool pf_pp = false;
  bool pf_fused = false;               // the prefetch formed Γ^{-1} (fused update) rather than L
  double* ws_gram = nullptr; // 2 x 16 x R x R Gram partials
  double* ws_mttv = nullptr; // mTTV K-split partials
  double* st_part = nullptr; // update-stats block partials
  double* upd_part = nullptr;  // fused-update block partials (3 x kUpdMaxBlocks)
  double* upd_gpart = nullptr; // fused-update per-CTA Gram partials (kUpdMaxBlocks x 2 R^2)
  unsigned int* st_counter = nullptr;
  double* scal = nullptr;    // device scalars (see SC_*)
  double* partial = nullptr;
  int* status = nullptr;     // N ints, Cholesky status per mode
  double* hscal = nullptr;   // pinned mirror of scal
  int* hstatus = nullptr;
  double* gather_tmp = nullptr;  // s_N x R for get_factor of the last mode
  // scheduler state
  int64_t t = 0;             // MSDT update stream position
  Subtree sub;               // live subtree (MSDT or DT)
  bool sub_is_msdt = false;
  std::map<std::pair<int, int>, double*> ops;  // PP operators
  bool pp_valid = false;
  bool pp_regime = false;    // dA = A - A_p (PP) vs one-sweep update (regular)
  bool have_fit = false;
  double last_f = 0.0, last_r = 0.0;
  int last_flags = 0;          // cpd_last_sweep_status: bit 0 = Eq. 3 radicand < -1e-8 ||T||^2
  double last_rad_rel = 0.0;   // the last sweep's Eq. 3 radicand / ||T||^2
  bool have_dA = false;
  double dA2[CPD_MAX_ORDER] = {0}, A2[CPD_MAX_ORDER] = {0};
  // diagnostics
  bool poisoned = false;
  std::string err;
  double phase_ms[5] = {0};
  double counters[5] = {0};
  // PP operator streams on the low-priority filler stream (overlapped with the main stream, so not
  // timed as launches of their own): bytes, launches (cpd_get_filler_counters)
  double filler[2] = {0};
  std::vector<PhaseRec> pending;
  std::multimap<size_t, void*> node_cache;         // free device blocks by exact size
  std::unordered_map<void*, size_t> node_bytes;    // size of every block from dalloc
  std::vector<cudaEvent_t> free_events;
  // INT8 tensor-core TTM (opts.ttm_impl == CPD_TTM_INT8)
  int* texp = nullptr;       // device: 2^texp > max|T| over all ranks' slabs
  void* ws_i8 = nullptr;     // sliced factor digits + exponents
  uint8_t* Td = nullptr;     // T's 7 int8 digit planes (computed once; null -> convert T per TTM)
  size_t ws_i8_bytes = 0;
  int engine = CPD_ENGINE_DMMA;  // first-level TTM engine chosen at init
  // upper-level fusion (opts.msdt_levels): each MSDT root contracts lv modes at once
  int lv = 1;
  // auxiliary memory ledger (cpd_get_memory): bytes of live dalloc blocks (tree nodes, PP operators,
  // block-contraction Khatri-Rao products) and their high-water mark since init / reset
  double node_live = 0.0, node_peak = 0.0;
  // algorithmic HBM bytes of the first-level TTMs / block contractions since init or reset (cpd_get_ttm_bytes)
  double ttm_bytes = 0.0;
};

// scalar slots
enum { SC_NT2 = 0, SC_MA = 1, SC_GS = 2, SC_DA2 = 3 /* N */, SC_A2 = 3 + CPD_MAX_ORDER /* N */,
       SC_LASTN2 = 3 + 2 * CPD_MAX_ORDER, SC_TMAX = 4 + 2 * CPD_MAX_ORDER, SC_COUNT = 8 + 2 * CPD_MAX_ORDER };

namespace {

cpd_status fail(cpd_ctx* c, cpd_status s, const std::string& msg) {
  if (c) {
    c->err = msg;
    if (s == CPD_ERR_CUDA || s == CPD_ERR_NCCL) c->poisoned = true;
  } else {
    g_init_error = msg;
  }
  return s;
}

#define CU(x)                                                                                 \
  do {                                                                                        \
    cudaError_t e_ = (x);                                                                     \
    if (e_ != cudaSuccess)                                                                    \
      return fail(ctx, e_ == cudaErrorMemoryAllocation ? CPD_ERR_OOM : CPD_ERR_CUDA,          \
                  std::string(#x) + ": " + cudaGetErrorString(e_));                          \
  } while (0)
#define NC(x)                                                                                 \
  do {                                                                                        \
    ncclResult_t r_ = (x);                                                                    \
    if (r_ != ncclSuccess)                                                                    \
      return fail(ctx, CPD_ERR_NCCL, std::string(#x) + ": " + ncclGetErrorString(r_));       \
  } while (0)
#define CM(call)                                                                              \
  do {                                                                                        \
    std::string m_;                                                                           \
    int r_ = (call);                                                                          \
    if (r_) return fail(ctx, r_ == 5 ? CPD_ERR_NCCL : CPD_ERR_CUDA, m_);                      \
  } while (0)
#define TRY(x)                        \
  do {                                \
    cpd_status s_ = (x);              \
    if (s_ != CPD_OK) return s_;      \
  } while (0)

inline int64_t ext(const cpd_ctx* c, int m) { return c->loc[m]; }
// own rows of mode n (the Q distribution of Alg. 3): the block's loc[n] rows split over Proc-Slice(x_n)
inline int64_t rows_own(const cpd_ctx* c, int n) { return c->loc[n] / c->slice[n].world; }
inline int64_t own_off(const cpd_ctx* c, int n) {  // row offset of own rows in the local block
  return c->slice[n].rank * rows_own(c, n);
}
inline int64_t node_elems(const cpd_ctx* c, const std::vector<int>& kept) {
  int64_t e = c->R;
  for (int k : kept) e *= ext(c, k);
  return e;
}

// ---------------- phase timers ----------------
cudaEvent_t get_event(cpd_ctx* c) {
  if (!c->free_events.empty()) {
    cudaEvent_t e = c->free_events.back();
    c->free_events.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
struct PhaseScope {
  cpd_ctx* c;
  PhaseRec rec;
  bool on;
  cudaStream_t s;
  // profile level 1: only the two roofline kernels (TTM, mTTV) are bracketed, so the timers
  // add ~4 event records per mode update; level 2: every phase (P:748 breakdown).  `stream`: the
  // stream the bracketed launch goes to (default the main stream; the PP filler stream's operator
  // streams are timed on their own stream, so the stream ledger's bytes and times match)
  PhaseScope(cpd_ctx* ctx, int phase, cudaStream_t stream = nullptr)
      : c(ctx), on(ctx->opts.profile_phases >= 2 || (ctx->opts.profile_phases == 1 && phase <= PH_MTTV)),
        s(stream ? stream : ctx->st) {
    if (on) {
      rec.a = get_event(c);
      rec.b = get_event(c);
      rec.phase = phase;
      cudaEventRecord(rec.a, s);
    }
  }
  ~PhaseScope() {
    if (on) {
      cudaEventRecord(rec.b, s);
      c->pending.push_back(rec);
    }
  }
};
// accumulate the completed timers; ones still in flight (filler-stream work) stay pending
void drain_timers(cpd_ctx* c, bool all = false) {
  std::vector<PhaseRec> keep;
  for (auto& r : c->pending) {
    if (!all && cudaEventQuery(r.b) == cudaErrorNotReady) {
      cudaGetLastError();
      keep.push_back(r);
      continue;
    }
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, r.a, r.b) == cudaSuccess) c->phase_ms[r.phase] += ms;
    cudaGetLastError();
    c->free_events.push_back(r.a);
    c->free_events.push_back(r.b);
  }
  c->pending.swap(keep);
}

// ---------------- memory ----------------
// Exact-size caching allocator for tree nodes / PP operators.  Node sizes repeat every
// cycle (a handful of distinct shapes), so after the first cycle every allocation is a
// cache hit; splitting a pool block for a small node could otherwise force the next
// root-sized allocation to map new memory (measured: tens of ms for 6.4 GB).  All users
// of these buffers run on ctx->st, so stream order makes immediate reuse safe.
void release_cache(cpd_ctx* c) {
  for (auto& kv : c->node_cache) cudaFreeAsync(kv.second, c->st);
  c->node_cache.clear();
}

cpd_status dalloc(cpd_ctx* ctx, double** p, int64_t elems) {
  *p = nullptr;
  if (elems <= 0) elems = 1;
  const size_t bytes = sizeof(double) * (size_t)elems;
  auto it = ctx->node_cache.find(bytes);
  if (it != ctx->node_cache.end()) {
    *p = (double*)it->second;
    ctx->node_cache.erase(it);
    ctx->node_live += (double)bytes;
    ctx->node_peak = std::max(ctx->node_peak, ctx->node_live);
    return CPD_OK;  // node_bytes[*p] already recorded
  }
  static const bool dbg = getenv("CPD_DEBUG_ALLOC") != nullptr;
  auto t0 = std::chrono::steady_clock::now();
  cudaError_t e = cudaMallocFromPoolAsync((void**)p, bytes, ctx->pool, ctx->st);
  if (e == cudaErrorMemoryAllocation) {  // give the cached blocks back and retry once
    cudaGetLastError();
    release_cache(ctx);
    cudaStreamSynchronize(ctx->st);
    cudaMemPoolTrimTo(ctx->pool, 0);
    e = cudaMallocFromPoolAsync((void**)p, bytes, ctx->pool, ctx->st);
  }
  CU(e);
  ctx->node_bytes[(void*)*p] = bytes;
  ctx->node_live += (double)bytes;
  ctx->node_peak = std::max(ctx->node_peak, ctx->node_live);
  if (dbg) {
    double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (ms > 0.5) fprintf(stderr, "[cpd] cudaMallocAsync %.3f GB took %.2f ms\n", 1e-9 * bytes, ms);
  }
  return CPD_OK;
}
// raw (non-node) device buffer from the ctx's pool
cudaError_t palloc(cpd_ctx* c, void** p, size_t bytes) { return cudaMallocFromPoolAsync(p, bytes, c->pool, c->st); }

void dfree(cpd_ctx* c, double*& p) {
  if (p) {
    const size_t b = c->node_bytes[(void*)p];
    c->node_cache.emplace(b, (void*)p);
    c->node_live -= (double)b;
  }
  p = nullptr;
}

// ---------------- kernels with accounting ----------------
cpd_status ttm(cpd_ctx* ctx, int j, double* out) {
  // T x_j A^(j): T viewed as [pre, ext(j), post]
  int64_t pre = 1, post = 1;
  for (int m = 0; m < j; m++) pre *= ext(ctx, m);
  for (int m = j + 1; m < ctx->N; m++) post *= ext(ctx, m);
  PhaseScope ps(ctx, PH_TTM);
  if (ctx->engine != CPD_ENGINE_DMMA && ext(ctx, j) <= cpd::kMaxKI8) {
    cpd::DigitView dv;
    if (ctx->Td) {
      dv.planes = ctx->Td;
      dv.w = ext(ctx, ctx->N - 1);
      dv.ipad = cpd::digit_inner_pad(dv.w);
      dv.plane_stride = cpd::digit_plane_bytes(ctx->T_elems, dv.w);
    }
    CU(cpd::launch_ttm_i8(ctx->T, pre, ext(ctx, j), post, ctx->A[j], ctx->R, out, 0, ctx->texp, ctx->ws_i8,
                          ctx->ws_i8_bytes, ctx->st, ctx->Td ? &dv : nullptr));
  } else {
    CU(cpd::launch_ttm(ctx->T, pre, ext(ctx, j), post, ctx->A[j], ctx->R, out, 0, ctx->st));
  }
  ctx->counters[0] += 2.0 * (double)pre * post * ext(ctx, j) * ctx->R;
  ctx->counters[1] += 1;
  ctx->counters[4] += 1;
  // T read once (7 B per element as digit planes, 8 B as FP64), the FP64 output written, the factor
  // (its digit image or FP64) read
  const bool dig = ctx->engine == CPD_ENGINE_INT8_DIGITS && ext(ctx, j) <= cpd::kMaxKI8;
  ctx->ttm_bytes += (dig ? 7.0 : 8.0) * (double)pre * post * ext(ctx, j) + 8.0 * (double)pre * post * ctx->R +
                    (dig ? 7.0 : 8.0) * (double)ext(ctx, j) * ctx->R;
  return CPD_OK;
}

// out = beta*out + contraction of node X (kept) over mode m with v (ext(m) x R)
cpd_status mttv(cpd_ctx* ctx, const double* X, const std::vector<int>& kept, int m,
                const double* v, double* out, int beta, const cpd::OutMap* map = nullptr) {
  int a = (int)(std::find(kept.begin(), kept.end(), m) - kept.begin());
  if (a >= (int)kept.size()) return fail(ctx, CPD_ERR_INTERNAL, "mttv: mode not kept");
  int64_t pre = 1, post = 1;
  for (int q = 0; q < a; q++) pre *= ext(ctx, kept[q]);
  for (int q = a + 1; q < (int)kept.size(); q++) post *= ext(ctx, kept[q]);
  int64_t K = ext(ctx, m);
  PhaseScope ps(ctx, PH_MTTV);
  {
    cpd::MttvSpec sp{X, v, pre, K, post};
    CU(cpd::launch_mttv_multi(&sp, 1, ctx->R, nullptr, out, beta, ctx->ws_mttv, kMttvWs, ctx->st, map));
  }
  double C = (double)post * ctx->R;
  ctx->counters[2] += 8.0 * ((double)pre * K * C + (double)pre * C * (beta ? 2 : 1) + (double)K * ctx->R);
  ctx->counters[3] += 1;
  return CPD_OK;
}

// Upper-level fusion ("combining several upper level contractions"): T contracted with the
// Khatri-Rao product of the factors of a cyclic block C of lv modes in ONE pass over T, giving the node
// that keeps the other modes (s^(N-lv) R elements instead of the s^(N-1) R of a first-level TTM).
// C is [c0, c0+lv) or, wrapping, [0, b) + [N-a, N) (a + b = lv).  int8 digit engine: one GEMM whose K
// index is (prefix p, padded suffix q) over the digit planes (launch_ttm_i8_block; a middle block is a
// plain TTM with the KRP as factor); DMMA engine: the FP64 TTM with the KRP as factor, a wrapping
// block as a TTM over the suffix then an mTTV over the prefix.
cpd_status ttm_block(cpd_ctx* ctx, const std::vector<int>& Cin, double* out) {
  const int N = ctx->N, R = ctx->R, l = (int)Cin.size();
  if (l == 1) return ttm(ctx, Cin[0], out);
  std::vector<int> C(Cin);
  std::sort(C.begin(), C.end());
  const bool contiguous = C.back() - C.front() == l - 1;
  if (!contiguous && (C.front() != 0 || C.back() != N - 1)) return fail(ctx, CPD_ERR_INTERNAL, "ttm_block: not a cyclic block");
  // wrapping: prefix [0, b), suffix [s0, N); contiguous: block [c0, c0 + l)
  int b = 0, s0 = C.front();
  if (!contiguous) {
    while (b < l && C[b] == b) b++;
    s0 = C[b];
  }
  auto prodx = [&](int lo, int hi) {
    int64_t p = 1;
    for (int m = lo; m < hi; m++) p *= ext(ctx, m);
    return p;
  };
  PhaseScope ps(ctx, PH_TTM);
  const double flops = 2.0 * (double)prodx(0, N) * R;
  // algorithmic bytes: T read once (digit planes 7 B / FP64 8 B per element), the output (the kept modes
  // x R) written once, the block's Khatri-Rao factor read (digit image 7 B / FP64 8 B per entry)
  const double kelem = (double)prodx(0, N), oelem = kelem / [&] {
    double k = 1;
    for (int c : C) k *= (double)ext(ctx, c);
    return k;
  }();
  auto account = [&](bool digits) {
    ctx->counters[0] += flops;
    ctx->counters[1] += 1;
    ctx->counters[4] += 1;
    ctx->ttm_bytes += (digits ? 7.0 : 8.0) * kelem + 8.0 * oelem * R + (digits ? 7.0 : 8.0) * (kelem / oelem) * R;
    return CPD_OK;
  };
  auto krp = [&](const std::vector<int>& modes, const std::vector<int64_t>& stride, double* dst, int64_t rows,
                 bool pad) -> cudaError_t {
    cpd::KrpSpec sp{};
    sp.n = (int)modes.size();
    for (int c = 0; c < sp.n; c++) {
      sp.A[c] = ctx->A[modes[c]];
      sp.ext[c] = ext(ctx, modes[c]);
      sp.stride[c] = stride[c];
    }
    return cpd::launch_krp_block(sp, R, dst, rows, pad, ctx->st);
  };
  // row-major strides of a plain KRP over consecutive modes
  auto plain = [&](const std::vector<int>& modes) {
    std::vector<int64_t> st(modes.size());
    int64_t acc = 1;
    for (int c = (int)modes.size() - 1; c >= 0; c--) {
      st[c] = acc;
      acc *= ext(ctx, modes[c]);
    }
    return st;
  };
  const bool tail = !contiguous || C.back() == N - 1;  // the block holds the innermost mode
  if (ctx->engine == CPD_ENGINE_INT8_DIGITS) {
    cpd::DigitView dv;
    dv.planes = ctx->Td;
    dv.w = ext(ctx, N - 1);
    dv.ipad = cpd::digit_inner_pad(dv.w);
    dv.plane_stride = cpd::digit_plane_bytes(ctx->T_elems, dv.w);
    if (tail) {
      // K = (p, q): the prefix modes [0, b) slowest, then the suffix [s0, N) with the innermost padded
      const int64_t P = prodx(0, b), Mrows = prodx(b, s0), Qp = prodx(s0, N - 1) * dv.ipad;
      const int64_t Ks = (Qp + 31) / 32 * 32;
      std::vector<int> modes;
      std::vector<int64_t> stride;
      for (int m = 0; m < b; m++) modes.push_back(m);
      for (int m = s0; m < N; m++) modes.push_back(m);
      stride.assign(modes.size(), 0);
      int64_t acc = 1;
      for (int c = (int)modes.size() - 1; c >= 0; c--) {
        const int m = modes[c];
        if (m == b - 1) acc = Ks;  // the last prefix mode steps over one padded suffix slab
        stride[c] = acc;
        acc *= (m == N - 1) ? dv.ipad : ext(ctx, m);
      }
      double* kb = nullptr;
      TRY(dalloc(ctx, &kb, P * Ks * R));
      CU(krp(modes, stride, kb, P * Ks, true));
      cudaError_t e = cpd::launch_ttm_i8_block(P, Mrows, Qp, kb, R, out, 0, ctx->texp, ctx->ws_i8,
                                               ctx->ws_i8_bytes, ctx->st, dv);
      dfree(ctx, kb);
      if (e == cudaSuccess) return account(true);
      if (e != cudaErrorNotSupported) CU(e);
      cudaGetLastError();
    } else {
      const int64_t pre = prodx(0, C.front()), K = prodx(C.front(), C.back() + 1), post = prodx(C.back() + 1, N);
      double* kb = nullptr;
      TRY(dalloc(ctx, &kb, K * R));
      CU(krp(C, plain(C), kb, K, false));
      cudaError_t e = cpd::launch_ttm_i8(ctx->T, pre, K, post, kb, R, out, 0, ctx->texp, ctx->ws_i8,
                                         ctx->ws_i8_bytes, ctx->st, &dv);
      dfree(ctx, kb);
      if (e == cudaSuccess) return account(true);
      cudaGetLastError();  // no digit layout for this view and K too long for the converting kernel
    }
  }
  if (contiguous) {
    const int64_t pre = prodx(0, C.front()), K = prodx(C.front(), C.back() + 1), post = prodx(C.back() + 1, N);
    double* kb = nullptr;
    TRY(dalloc(ctx, &kb, K * R));
    CU(krp(C, plain(C), kb, K, false));
    if (ctx->engine != CPD_ENGINE_DMMA && K <= cpd::kMaxKI8)
      CU(cpd::launch_ttm_i8(ctx->T, pre, K, post, kb, R, out, 0, ctx->texp, ctx->ws_i8, ctx->ws_i8_bytes, ctx->st,
                            nullptr));
    else
      CU(cpd::launch_ttm(ctx->T, pre, K, post, kb, R, out, 0, ctx->st));
    dfree(ctx, kb);
    return account(false);
  }
  // wrapping block on the FP64 engine: X[p, m, r] = T x_suffix KRP(suffix), then out = X x_p KRP(prefix)
  std::vector<int> pm, sm;
  for (int m = 0; m < b; m++) pm.push_back(m);
  for (int m = s0; m < N; m++) sm.push_back(m);
  const int64_t P = prodx(0, b), Mrows = prodx(b, s0), Q = prodx(s0, N);
  double *ks = nullptr, *kp = nullptr, *X = nullptr;
  TRY(dalloc(ctx, &ks, Q * R));
  TRY(dalloc(ctx, &kp, P * R));
  TRY(dalloc(ctx, &X, P * Mrows * R));
  CU(krp(sm, plain(sm), ks, Q, false));
  CU(krp(pm, plain(pm), kp, P, false));
  CU(cpd::launch_ttm(ctx->T, P * Mrows, Q, 1, ks, R, X, 0, ctx->st));
  cpd::MttvSpec sp{X, kp, 1, P, Mrows};
  CU(cpd::launch_mttv_multi(&sp, 1, R, nullptr, out, 0, ctx->ws_mttv, kMttvWs, ctx->st));
  dfree(ctx, X);
  dfree(ctx, kp);
  dfree(ctx, ks);
  return account(false);
}

// contract the modes `drop` of a node in `order`, returning a new node (input not freed)
// `map` (fused reduce-scatter): the contraction that produces the final node stores it into the
// owners' receive slots instead (the node buffer is then left unwritten)
cpd_status contract_modes(cpd_ctx* ctx, const Node& in, const std::vector<int>& drop,
                          const std::vector<int>& order, Node* out, const cpd::OutMap* map = nullptr) {
  int remaining = 0;
  for (int m : order)
    if (std::find(drop.begin(), drop.end(), m) != drop.end()) remaining++;
  Node cur;
  cur.buf = in.buf;
  cur.kept = in.kept;
  bool owned = false;
  for (int m : order) {
    if (std::find(drop.begin(), drop.end(), m) == drop.end()) continue;
    Node nx;
    for (int k : cur.kept)
      if (k != m) nx.kept.push_back(k);
    TRY(dalloc(ctx, &nx.buf, node_elems(ctx, nx.kept)));
    TRY(mttv(ctx, cur.buf, cur.kept, m, ctx->A[m], nx.buf, 0, --remaining == 0 ? map : nullptr));
    if (owned) dfree(ctx, cur.buf);
    cur = nx;
    owned = true;
  }
  if (!owned) return fail(ctx, CPD_ERR_INTERNAL, "contract_modes: nothing to contract");
  *out = cur;
  return CPD_OK;
}

void clear_subtree(cpd_ctx* c) {
  for (auto& kv : c->sub.cache) dfree(c, kv.second.buf);
  c->sub.cache.clear();
  c->sub.active = false;
  c->sub.j = -1;
}

// start a subtree: root T x_C (one mode, or a block of modes with upper-level fusion), then contract
// `pre` (in order), served list
cpd_status start_subtree(cpd_ctx* ctx, const std::vector<int>& C, const std::vector<int>& pre,
                         const std::vector<int>& served) {
  clear_subtree(ctx);
  Node root;
  for (int m = 0; m < ctx->N; m++)
    if (std::find(C.begin(), C.end(), m) == C.end()) root.kept.push_back(m);
  TRY(dalloc(ctx, &root.buf, node_elems(ctx, root.kept)));
  TRY(ttm_block(ctx, C, root.buf));
  const int j = C.size() == 1 ? C[0] : -1;
  if (!pre.empty()) {
    Node nx;
    TRY(contract_modes(ctx, root, pre, pre, &nx));
    dfree(ctx, root.buf);
    root = nx;
  }
  ctx->sub.j = j;
  ctx->sub.served = served;
  ctx->sub.cache[{0, (int)served.size()}] = root;
  ctx->sub.active = true;
  return CPD_OK;
}

// leaf q of the live subtree (lazy binary descent, O3)
// fused reduce-scatter map of mode n, or null
const cpd::OutMap* rs_map_of(const cpd_ctx* c, int n) { return c->rs_map[n].nq > 0 ? &c->rs_map[n] : nullptr; }

// *scattered: the leaf was computed now straight into the owners' receive slots (fused RS)
cpd_status subtree_leaf(cpd_ctx* ctx, int q, const double** leaf, bool* scattered) {
  *scattered = false;
  auto& sub = ctx->sub;
  const auto& L = sub.served;
  int lo = 0, hi = (int)L.size();
  auto it = sub.cache.find({lo, hi});
  if (it == sub.cache.end()) return fail(ctx, CPD_ERR_INTERNAL, "subtree root missing");
  while (hi - lo > 1) {
    int mid = lo + (hi - lo + 1) / 2;
    std::pair<int, int> child;
    std::vector<int> drop;
    if (q < mid) {
      child = {lo, mid};
      drop.assign(L.begin() + mid, L.begin() + hi);
    } else {
      child = {mid, hi};
      drop.assign(L.begin() + lo, L.begin() + mid);
    }
    if (!sub.cache.count(child)) {
      // free finished nodes: everything that is not an ancestor of `child`
      for (auto c2 = sub.cache.begin(); c2 != sub.cache.end();) {
        bool anc = c2->first.first <= child.first && child.second <= c2->first.second;
        if (!anc) {
          dfree(ctx, c2->second.buf);
          c2 = sub.cache.erase(c2);
        } else {
          ++c2;
        }
      }
      const Node& parent = sub.cache[{lo, hi}];
      std::vector<int> order(L.begin() + lo, L.begin() + hi);
      Node nx;
      const bool is_leaf = child.second - child.first == 1;
      const cpd::OutMap* mp = is_leaf ? rs_map_of(ctx, L[q]) : nullptr;
      TRY(contract_modes(ctx, parent, drop, order, &nx, mp));
      if (mp) *scattered = true;
      sub.cache[child] = nx;
    }
    lo = child.first;
    hi = child.second;
  }
  const Node& leafn = sub.cache[{lo, hi}];
  if (leafn.kept.size() != 1 || leafn.kept[0] != L[q])
    return fail(ctx, CPD_ERR_INTERNAL, "stale or wrong leaf");
  *leaf = leafn.buf;
  return CPD_OK;
}

// after the update of mode n's own rows (Alg. 3 lines 15-18, Alg. 4 lines 13-15): S^(n) (and dS^(n))
// and the ||dA||^2, ||A||^2 (and <M^(N), A^(N)>) partial sums of the own rows all-reduced over all
// ranks (line 17), then the A^(n) (and dA^(n)) block all-gathered in Proc-Slice(x_n) (line 18)
cpd_status exchange_mode(cpd_ctx* ctx, int n, bool pp) {
  if (ctx->world == 1) return CPD_OK;
  const int R = ctx->R;
  const int64_t RR = (int64_t)R * R;
  const bool last = n == ctx->N - 1;
  PhaseScope ps(ctx, PH_OTHER);
  CM(cpd::comm_group_start(ctx->cm, &m_));
  CM(cpd::comm_all_reduce(ctx->cm, ctx->S_all + n * RR, RR, &m_));
  if (pp) CM(cpd::comm_all_reduce(ctx->cm, ctx->dS_all + n * RR, RR, &m_));
  if (last) CM(cpd::comm_all_reduce(ctx->cm, ctx->scal + SC_MA, 1, &m_));
  CM(cpd::comm_all_reduce(ctx->cm, ctx->scal + SC_DA2 + n, 1, &m_));
  CM(cpd::comm_all_reduce(ctx->cm, ctx->scal + SC_A2 + n, 1, &m_));
  CM(cpd::comm_group_end(ctx->cm, &m_));
  cpd::Comm& sl = ctx->slice[n];
  if (sl.world > 1) {
    const int64_t ro = rows_own(ctx, n), off = own_off(ctx, n);
    CM(cpd::comm_group_start(sl, &m_));
    CM(cpd::comm_all_gather(sl, ctx->A[n] + off * R, ctx->A[n], ro * R, &m_));
    CM(cpd::comm_all_gather(sl, ctx->dA[n] + off * R, ctx->dA[n], ro * R, &m_));
    CM(cpd::comm_group_end(sl, &m_));
  }
  return CPD_OK;
}

// <Γ^(N), S^(N)> = Σ_e (∗_{k<N-1} S_k)[e] S_{N-1}[e]  (after S_{N-1} is final)
__global__ void gamma_dot_kernel(const double* __restrict__ S_all, int N, int R, double* dst) {
  __shared__ double red[32];
  const int64_t RR = (int64_t)R * R;
  double s = 0.0;
  for (int64_t e = threadIdx.x; e < RR; e += blockDim.x) {
    double gv = S_all[e];
    for (int k = 1; k < N - 1; k++) gv *= S_all[k * RR + e];
    s = fma(gv, S_all[(N - 1) * RR + e], s);
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = (threadIdx.x < blockDim.x / 32) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) dst[0] = s;
  }
}

// whether mode n's update runs as the single fused cooperative kernel (update.cu)
bool use_fused(const cpd_ctx* ctx, int n, bool pp) {
  static const bool off = getenv("CPD_NO_FUSED_UPDATE") != nullptr;  // experiment switch: Cholesky path
  if (off) return false;
  const int64_t ro = rows_own(ctx, n);
  const int blocks = cpd::update_fused_blocks(ro);
  return ctx->R <= cpd::kUpdMaxR && ctx->Gi[0] &&
         cpd::update_fused_smem(ctx->R, pp, (int)((ro + blocks - 1) / blocks)) <= 225 * 1024;
}

// experiment switch CPD_LOCAL_INV (R <= 32 on the fused path): Γ^{-1} (and W) formed inside the update
// launch by one warp of every CTA (update.cu gj32_warp) instead of on the side stream.  Measured slower
// (C4 PP sweep 0.25 -> 0.46 ms, C1 0.125 -> 0.21 ms: ~1000 dependent shuffles per CTA before any row
// work), so off by default
bool local_inv(const cpd_ctx* ctx) {
  static const bool on = getenv("CPD_LOCAL_INV") != nullptr;
  return on && ctx->R <= 32;
}

// Γ^(m) = ∗_{k≠m} S^(k) depends only on the Grams, so its Cholesky factorisation (and the
// PP Hadamard sum W^(m) of Eq. 7) can run on a side stream as soon as the previous update
// has produced its S, overlapping the latency-bound single-CTA factorisation with the
// HBM-bound MTTKRP stream of mode m.  Buffers alternate so the side stream never
// overwrites a factor the main stream still reads.
cpd_status prefetch_solve(cpd_ctx* ctx, int m, bool pp) {
  const int b = ctx->pf_buf ^ 1;
  CU(cudaEventRecord(ctx->ev_s, ctx->st));
  CU(cudaStreamWaitEvent(ctx->st2, ctx->ev_s, 0));
  // the SPD verdict goes to pf_status[b] (side stream); the update that consumes buffer b hands
  // it to status[m] on the main stream (acquire_solve), so every status finish_sweep reads is
  // ordered on the main stream and a prefetch for the next sweep never touches this sweep's
  const bool fz = use_fused(ctx, m, pp);
  int* pst = ctx->pf_status + b;
  if (fz && local_inv(ctx)) {
    // nothing to prepare: the update launch forms Γ^{-1} (and W) itself
  } else if (fz) {
    // the fused update multiplies by Γ^{-1}: form it directly (Gauss-Jordan, SPD check)
    // with W of Eq. 7 in the same launch for PP sweeps
    CU(cpd::launch_gamma_inverse(ctx->S_all, ctx->N, m, ctx->R, ctx->Gi[b], pst, ctx->st2, pp ? ctx->dS_all : nullptr,
                                 pp ? ctx->Wb[b] : nullptr));
  } else if (ctx->R > kCholMaxR) {
    // beyond the single-CTA packed Cholesky: Γ^{-1} by the grid-wide blocked Gauss-Jordan
    CU(cpd::launch_gamma_inverse_big(ctx->S_all, ctx->N, m, ctx->R, ctx->ws_gj, ctx->Gi[b], pst, ctx->st2));
  } else {
    CU(cpd::launch_gamma_chol(ctx->S_all, ctx->N, m, ctx->R, ctx->Lp[b], pst, ctx->st2));
  }
  if (pp && !fz) CU(cpd::launch_pp_w(ctx->S_all, ctx->dS_all, ctx->N, m, ctx->R, ctx->Wb[b], ctx->st2));
  CU(cudaEventRecord(ctx->ev_pf, ctx->st2));
  ctx->pf_buf = b;
  ctx->pf_mode = m;
  ctx->pf_pp = pp;
  ctx->pf_fused = fz;
  return CPD_OK;
}

void invalidate_prefetch(cpd_ctx* ctx) { ctx->pf_mode = -1; }

// wait for the prepared Γ factor of mode n; `fused`: the fused update kernel copies the SPD
// verdict pf_status[b] -> status[n] itself, otherwise it is copied here on the main stream
cpd_status acquire_solve(cpd_ctx* ctx, int n, bool pp, int* buf, bool fused) {
  if (!(ctx->pf_mode == n && (ctx->pf_pp || !pp) && ctx->pf_fused == use_fused(ctx, n, pp)))
    TRY(prefetch_solve(ctx, n, pp));
  CU(cudaStreamWaitEvent(ctx->st, ctx->ev_pf, 0));
  *buf = ctx->pf_buf;
  ctx->pf_mode = -1;
  if (!fused)
    CU(cudaMemcpyAsync(ctx->status + n, ctx->pf_status + *buf, sizeof(int), cudaMemcpyDeviceToDevice, ctx->st));
  return CPD_OK;
}

// Solve-and-update for mode n given the local (block-partial) MTTKRP Mloc (ext(n) x R, may be
// overwritten): reduce-scatter in Proc-Slice(x_n) to the own rows (Alg. 3 line 14), solve them
// (line 15; pp: V = A^(n) W added first, Eq. 7), dA, statistics, S (and dS) of the own rows, then
// exchange_mode (all-reduce, all-gather of the block).
// pend: the K-split reduction of the mTTV that produced Mloc, left to the fused update (PP critical chain)
cpd_status update_mode(cpd_ctx* ctx, int n, double* Mloc, bool pp, bool scattered = false,
                       const cpd::MPending* pend = nullptr) {
  const int R = ctx->R;
  const int64_t RR = (int64_t)R * R;
  const int64_t ro = rows_own(ctx, n), off = own_off(ctx, n);
  double* Mown = Mloc + off * R;
  const bool last = n == ctx->N - 1;
  const bool fused = use_fused(ctx, n, pp);
  if (pend && pend->slots > 0 && (scattered || ctx->slice[n].world > 1 || !fused || !pp))
    return fail(ctx, CPD_ERR_INTERNAL, "deferred mTTV reduction without a fused single-slice PP update");
  if (scattered) {
    // fused reduce-scatter: every slice rank stored its partial rows into its slot of the owner's
    // receive buffer; after the stream-ordered barrier the owner sums the slots in rank order
    PhaseScope ps(ctx, PH_OTHER);
    CM(cpd::comm_barrier(ctx->slice[n], ctx->bar_scratch, &m_));
    CU(cpd::launch_slot_sum(ctx->rs_recv[n], ctx->slice[n].world, ro * R, Mown, ctx->st));
  } else if (ctx->slice[n].world > 1) {
    PhaseScope ps(ctx, PH_OTHER);
    CM(cpd::comm_reduce_scatter(ctx->slice[n], Mloc, Mown, ro * R, &m_));
  }
  // Γ^(n) factor (and W^(n) for PP): prepared on the side stream while the MTTKRP of mode n
  // streamed, or computed here if no matching prefetch is pending
  int b;
  TRY(acquire_solve(ctx, n, pp, &b, fused));
  {
    PhaseScope ps(ctx, PH_OTHER);
    if (pp) {
      ctx->Mlast_src[n] = Mloc;  // persistent M~ buffer: no copy, read on demand
    } else {
      ctx->Mlast_src[n] = nullptr;
      CU(cudaMemcpyAsync(ctx->Mlast[n] + off * R, Mown, sizeof(double) * ro * R, cudaMemcpyDeviceToDevice, ctx->st));
    }
  }
  if (fused) {
    // fused: V term, row solve, dA, statistics, S (and dS) of the own rows in one cooperative launch
    PhaseScope ps(ctx, PH_SOLVE);
    const bool loc = local_inv(ctx);
    CU(cpd::launch_update_fused(R, ro, ctx->Gi[b], pp ? ctx->Wb[b] : nullptr, Mown, ctx->A[n] + off * R,
                                pp ? ctx->Ap[n] + off * R : nullptr, ctx->dA[n] + off * R, ctx->S_all + n * RR,
                                pp ? ctx->dS_all + n * RR : nullptr, ctx->upd_part, ctx->upd_gpart,
                                ctx->scal + SC_DA2 + n, ctx->scal + SC_A2 + n, last ? ctx->scal + SC_MA : nullptr,
                                loc ? nullptr : ctx->pf_status + b, loc ? nullptr : ctx->status + n, ctx->st,
                                loc ? ctx->S_all : nullptr, loc ? ctx->dS_all : nullptr, ctx->N, n,
                                loc ? ctx->status + n : nullptr, pend));
  } else {
    if (pp) {
      // V^(n) = A^(n) W^(n) with the current (pre-update) A^(n): Eq. 7; M~ += V (Eq. 5)
      PhaseScope ps(ctx, PH_HAD);
      CU(cpd::launch_ttm(ctx->A[n] + off * R, ro, R, 1, ctx->Wb[b], R, Mown, 1, ctx->st));
    }
    if (!pp) {
      PhaseScope ps(ctx, PH_OTHER);
      CU(cudaMemcpyAsync(ctx->Aold[n] + off * R, ctx->A[n] + off * R, sizeof(double) * ro * R,
                         cudaMemcpyDeviceToDevice, ctx->st));
    }
    {
      PhaseScope ps(ctx, PH_SOLVE);
      if (R > kCholMaxR)  // x = M Γ^{-1} as a GEMM on the DMMA kernel
        CU(cpd::launch_ttm(Mown, ro, R, 1, ctx->Gi[b], R, ctx->A[n] + off * R, 0, ctx->st));
      else
        CU(cpd::launch_trisolve(ctx->Lp[b], Mown, ro, R, ctx->A[n] + off * R, ctx->st));
    }
    {
      PhaseScope ps(ctx, PH_HAD);
      const double* base = (pp ? ctx->Ap[n] : ctx->Aold[n]) + off * R;
      // dA, ||dA||^2, ||A||^2 (and <M^(N), A^(N)> of Eq. 3 for the last mode) of the own rows in one pass
      CU(cpd::launch_update_stats(ctx->A[n] + off * R, base, ctx->dA[n] + off * R, last ? Mown : nullptr, ro * R,
                                  ctx->st_part, ctx->st_counter, ctx->scal + SC_DA2 + n, ctx->scal + SC_A2 + n,
                                  ctx->scal + SC_MA, ctx->st));
      CU(cpd::launch_gram(ctx->A[n] + off * R, ctx->A[n] + off * R, pp ? ctx->dA[n] + off * R : nullptr, ro, R,
                          ctx->S_all + n * RR, pp ? ctx->dS_all + n * RR : nullptr, ctx->ws_gram, 32 * RR, ctx->st));
    }
  }
  TRY(exchange_mode(ctx, n, pp));
  if (last) {
    PhaseScope ps(ctx, PH_OTHER);
    cpd::g_launches++;
    gamma_dot_kernel<<<1, 1024, 0, ctx->st>>>(ctx->S_all, ctx->N, R, ctx->scal + SC_GS);
    CU(cudaGetLastError());
  }
  // S^(n) is final: start Γ^(n+1) (the next update in every schedule) on the side stream
  TRY(prefetch_solve(ctx, (n + 1) % ctx->N, pp));
  return CPD_OK;
}

// after a sweep: one D2H of the scalars, fitness (Eq. 3), PP condition
cpd_status finish_sweep(cpd_ctx* ctx, double* f_out) {
  CU(cudaMemcpyAsync(ctx->hscal, ctx->scal, sizeof(double) * SC_COUNT, cudaMemcpyDeviceToHost, ctx->st));
  CU(cudaMemcpyAsync(ctx->hstatus, ctx->status, sizeof(int) * ctx->N, cudaMemcpyDeviceToHost, ctx->st));
  CU(cudaStreamSynchronize(ctx->st));
  drain_timers(ctx);
  for (int n = 0; n < ctx->N; n++)
    if (ctx->hstatus[n] != 0) return fail(ctx, CPD_ERR_NUMERIC, "Gamma not SPD (Cholesky failed)");
  const double nt2 = ctx->hscal[SC_NT2];
  const double rad = nt2 + ctx->hscal[SC_GS] - 2.0 * ctx->hscal[SC_MA];
  if (!std::isfinite(rad)) return fail(ctx, CPD_ERR_NUMERIC, "non-finite residual");
  // Eq. 3 cannot be negative beyond rounding: a (forced) approximated sweep outside the ε regime
  // left M~ and A inconsistent; the fitness is then clamped (f = 1) and flagged
  ctx->last_flags = rad < -1e-8 * nt2 ? 1 : 0;
  ctx->last_rad_rel = rad / nt2;
  ctx->last_r = std::sqrt(std::max(rad, 0.0)) / std::sqrt(nt2);
  ctx->last_f = 1.0 - ctx->last_r;
  ctx->have_fit = true;
  for (int n = 0; n < ctx->N; n++) {
    ctx->dA2[n] = ctx->hscal[SC_DA2 + n];
    ctx->A2[n] = ctx->hscal[SC_A2 + n];
  }
  ctx->have_dA = true;
  if (f_out) *f_out = ctx->last_f;
  return CPD_OK;
}

bool pp_cond(const cpd_ctx* c) {
  for (int n = 0; n < c->N; n++)
    if (!(std::sqrt(c->dA2[n]) < c->opts.pp_eps * std::sqrt(c->A2[n]))) return false;
  return true;
}

void free_pp(cpd_ctx* c) {
  for (auto& kv : c->ops) dfree(c, kv.second);
  c->ops.clear();
  for (auto& p : c->Mp) dfree(c, p);
  for (int n = 0; n < (int)c->Mlast_src.size(); n++)
    if (c->Mlast_src[n]) {  // keep the last M~ readable after the PP buffers go away
      const int64_t ro = rows_own(c, n), off = own_off(c, n);
      cudaMemcpyAsync(c->Mlast[n] + off * c->R, c->Mlast_src[n] + off * c->R, sizeof(double) * ro * c->R,
                      cudaMemcpyDeviceToDevice, c->st);
      c->Mlast_src[n] = nullptr;
    }
  for (auto& p : c->Mt) dfree(c, p);
  for (auto& p : c->Mt2) dfree(c, p);
  c->pp_valid = false;
}

// the speculative next-sweep PP streams (filler stream st3) read the operators, M_p and dA and
// write the spare M~ set: the main stream waits for them before it writes any of those
void drop_spec(cpd_ctx* c) {
  if (c->pp_spec || c->pp_spec0) {
    cudaStreamWaitEvent(c->st, c->ev_pp_side[1], 0);  // recorded after every speculative launch on st3
    c->pp_spec = false;
    c->pp_spec0 = false;
  }
}

// orders a public call's work after the caller's stream and the caller's stream after it
struct UserSync {
  cpd_ctx* c;
  explicit UserSync(cpd_ctx* ctx, bool keep_spec = false) : c(ctx) {
    if (c && c->ev_in) {
      cudaEventRecord(c->ev_in, c->ust);
      cudaStreamWaitEvent(c->st, c->ev_in, 0);
    }
    if (c && !keep_spec) drop_spec(c);  // speculative PP work must finish before anything else
  }
  ~UserSync() {
    if (c && c->ev_out) {
      cudaEventRecord(c->ev_out, c->st);
      cudaStreamWaitEvent(c->ust, c->ev_out, 0);
    }
  }
};

cpd_status check_ctx(cpd_ctx* ctx) {
  if (!ctx) return CPD_ERR_INVALID_ARG;
  if (ctx->poisoned) return CPD_ERR_STATE;
  cudaError_t e = cudaSetDevice(ctx->dev);
  if (e != cudaSuccess) return fail(ctx, CPD_ERR_CUDA, cudaGetErrorString(e));
  return CPD_OK;
}

cpd_status regular_sweep(cpd_ctx* ctx, bool msdt, double* f_out) {
  const int N = ctx->N;
  if (ctx->pp_regime || !ctx->sub_is_msdt || !msdt) {
    // any factor change not made by msdt_sweep restarts the MSDT cycle
    if (msdt && (ctx->pp_regime || !ctx->sub_is_msdt)) {
      clear_subtree(ctx);
      ctx->t = 0;
    }
  }
  ctx->pp_regime = false;
  if (msdt) {
    ctx->sub_is_msdt = true;
    // root k serves the S = N - lv updates [kS, (k+1)S) (modes f, .., f+S-1 mod N, f = kS mod N) and
    // contracts the lv modes that follow them cyclically (not updated while it is in use); lv = 1:
    // j = ((k+1)(N-1)) mod N, T x_N, T x_{N-1}, ... (R4)
    const int S = N - ctx->lv;
    for (int n = 0; n < N; n++) {
      int64_t k = ctx->t / S;
      int q = (int)(ctx->t % S);
      if (q == 0 || !ctx->sub.active) {
        const int f = (int)((k * S) % N);
        std::vector<int> served, C;
        for (int d = 0; d < S; d++) served.push_back((f + d) % N);
        for (int d = S; d < N; d++) C.push_back((f + d) % N);
        TRY(start_subtree(ctx, C, {}, served));
      }
      if (ctx->sub.served[q] != n) return fail(ctx, CPD_ERR_INTERNAL, "MSDT schedule out of phase");
      const double* leaf;
      bool sc = false;
      TRY(subtree_leaf(ctx, q, &leaf, &sc));
      drop_spec(ctx);  // first write of factor state (dA) in this sweep
      TRY(update_mode(ctx, n, const_cast<double*>(leaf), false, sc));
      ctx->t++;
    }
  } else {
    ctx->sub_is_msdt = false;
    clear_subtree(ctx);
    ctx->t = 0;
    const int h = (N + 1) / 2;
    for (int n = 0; n < N; n++) {
      if (n == 0) {
        std::vector<int> pre, served;
        for (int m = h; m < N - 1; m++) pre.push_back(m);
        for (int m = 0; m < h; m++) served.push_back(m);
        TRY(start_subtree(ctx, {N - 1}, pre, served));
      } else if (n == h) {
        std::vector<int> pre, served;
        for (int m = 1; m < h; m++) pre.push_back(m);
        for (int m = h; m < N; m++) served.push_back(m);
        TRY(start_subtree(ctx, {0}, pre, served));
      }
      int q = n < h ? n : n - h;
      const double* leaf;
      bool sc = false;
      TRY(subtree_leaf(ctx, q, &leaf, &sc));
      drop_spec(ctx);
      TRY(update_mode(ctx, n, const_cast<double*>(leaf), false, sc));
    }
    clear_subtree(ctx);
  }
  TRY(finish_sweep(ctx, f_out));
  return CPD_OK;
}

// produce all pair operators in `targets` (subsets of node.kept) from `node` (greedy
// shared descent); node buffer is not freed here
// filler-stream operator streams at 3 CTAs/SM (CPD_FILLER_OCC4: 4, the main-stream build)
bool filler_occ3() {
  static const bool occ4 = getenv("CPD_FILLER_OCC4") != nullptr;
  return !occ4;
}
// K-split target of the filler-stream launches (experiment switch CPD_FILLER_WAVES; 0 = the default)
int filler_waves() {
  static const int w = getenv("CPD_FILLER_WAVES") ? atoi(getenv("CPD_FILLER_WAVES")) : 0;
  return w;
}

// the mode of `node` whose contraction keeps the most of `targets`
int pp_best_mode(const Node& node, const std::vector<std::pair<int, int>>& targets) {
  int best = -1, bestc = -1;
  for (int m : node.kept) {
    int cnt = 0;
    for (auto& pr : targets)
      if (pr.first != m && pr.second != m) cnt++;
    if (cnt > bestc) {
      bestc = cnt;
      best = m;
    }
  }
  return best;
}

// two children of `node` (contract mode ma, resp. mb) from ONE read of the node (mTTV dual kernel)
cpd_status contract_dual(cpd_ctx* ctx, const Node& node, int ma, int mb, Node* ca, Node* cb) {
  const auto& kp = node.kept;
  int qa = (int)(std::find(kp.begin(), kp.end(), ma) - kp.begin());
  int qb = (int)(std::find(kp.begin(), kp.end(), mb) - kp.begin());
  const bool swap = qa > qb;
  if (swap) std::swap(qa, qb);
  int64_t P = 1, Q = 1, C = ctx->R;
  for (int i = 0; i < qa; i++) P *= ext(ctx, kp[i]);
  for (int i = qa + 1; i < qb; i++) Q *= ext(ctx, kp[i]);
  for (int i = qb + 1; i < (int)kp.size(); i++) C *= ext(ctx, kp[i]);
  const int m1 = kp[qa], m2 = kp[qb];  // out1 contracts m1, out2 contracts m2
  Node c1, c2;
  for (int k : kp) {
    if (k != m1) c1.kept.push_back(k);
    if (k != m2) c2.kept.push_back(k);
  }
  TRY(dalloc(ctx, &c1.buf, node_elems(ctx, c1.kept)));
  TRY(dalloc(ctx, &c2.buf, node_elems(ctx, c2.kept)));
  const int64_t K1 = ext(ctx, m1), K2 = ext(ctx, m2);
  const int64_t nkb = (K1 + 31) / 32;
  const int64_t E1 = node_elems(ctx, c1.kept);
  double* ws = nullptr;
  if (nkb > 1) TRY(dalloc(ctx, &ws, nkb * E1));
  {
    PhaseScope ps(ctx, PH_MTTV);
    CU(cpd::launch_mttv_dual(node.buf, P, K1, Q, K2, C, ctx->R, ctx->A[m1], ctx->A[m2], c1.buf, c2.buf, ws,
                             nkb * E1, ctx->st));
  }
  if (ws) dfree(ctx, ws);
  ctx->counters[2] += 8.0 * ((double)node_elems(ctx, kp) + E1 + node_elems(ctx, c2.kept) + (K1 + K2) * ctx->R);
  ctx->counters[3] += 1;
  *ca = swap ? c2 : c1;
  *cb = swap ? c1 : c2;
  return CPD_OK;
}

// produce all pair operators in `targets` (subsets of node.kept) from `node` (greedy shared
// descent: the child keeping the most targets first; the next child, for the targets the first
// one cannot give, is built in the same read of the node by the dual mTTV); the node buffer is
// not freed here
cpd_status pp_descend(cpd_ctx* ctx, const Node& node, std::vector<std::pair<int, int>> targets) {
  if (node.kept.size() == 2) return fail(ctx, CPD_ERR_INTERNAL, "pp_descend on a pair");
  static const bool no_dual = getenv("CPD_PP_NO_DUAL") != nullptr;
  auto take = [&](Node& child, std::vector<std::pair<int, int>>& sub) -> cpd_status {
    if (child.kept.size() == 2) {
      ctx->ops[{child.kept[0], child.kept[1]}] = child.buf;
    } else {
      TRY(pp_descend(ctx, child, sub));
      dfree(ctx, child.buf);
    }
    return CPD_OK;
  };
  auto split = [](const std::vector<std::pair<int, int>>& t, int m, std::vector<std::pair<int, int>>& sub,
                  std::vector<std::pair<int, int>>& rest) {
    for (auto& pr : t) (pr.first != m && pr.second != m ? sub : rest).push_back(pr);
  };
  while (!targets.empty()) {
    const int best = pp_best_mode(node, targets);
    std::vector<std::pair<int, int>> sub, rest;
    split(targets, best, sub, rest);
    if (!rest.empty() && !no_dual) {
      const int best2 = pp_best_mode(node, rest);
      std::vector<std::pair<int, int>> sub2, rest2;
      split(rest, best2, sub2, rest2);
      Node c1, c2;
      TRY(contract_dual(ctx, node, best, best2, &c1, &c2));
      TRY(take(c1, sub));
      TRY(take(c2, sub2));
      targets = rest2;
      continue;
    }
    Node child;
    TRY(contract_modes(ctx, node, {best}, {best}, &child));
    TRY(take(child, sub));
    targets = rest;
  }
  return CPD_OK;
}

// ||T||^2 (all-reduced) and the TTM engine's view of T: exponent and digit planes
// (cp_als_init, cpd_set_tensor).  Buffers from a previous call (exponent, factor-digit
// workspace, digit planes: all sized by the shape, not the contents) are reused.
cpd_status prepare_tensor(cpd_ctx* ctx) {
  CU(cpd::launch_norm2(ctx->T, ctx->T_elems, ctx->partial, ctx->scal + SC_NT2, ctx->st));
  {
    std::string m_;
    int r_ = cpd::comm_all_reduce(ctx->cm, ctx->scal + SC_NT2, 1, &m_);
    if (r_) {
      return fail(ctx, r_ == 5 ? CPD_ERR_NCCL : CPD_ERR_CUDA, m_);
    }
  }
  const cpd_opts& o = ctx->opts;
  const int N = ctx->N, R = ctx->R;
  ctx->engine = CPD_ENGINE_DMMA;
  if (o.ttm_impl == CPD_TTM_INT8 || o.ttm_impl == CPD_TTM_AUTO) {
    // one exponent for this rank's slab (T is read-only, so once per ctx); ranks may differ,
    // which changes results only at the rounding level
    if (!ctx->texp) CU(palloc(ctx, (void**)&ctx->texp, sizeof(int)));
    CU(cpd::launch_absmax_exp(ctx->T, ctx->T_elems, ctx->partial, ctx->texp, ctx->st, ctx->scal + SC_TMAX));
    bool use_i8 = true;
    if (o.ttm_impl == CPD_TTM_AUTO) {
      // the digit TTM's norm-wise error is ~2^-55 max|T|/rms(T) (DESIGN.md §6 K2i): use it when
      // that is FP64-class (max|T| <= 256 rms(T), i.e. <= 2^-47), else the FP64 DMMA engine
      double h[SC_COUNT];
      CU(cudaMemcpyAsync(h, ctx->scal, sizeof(double) * SC_COUNT, cudaMemcpyDeviceToHost, ctx->st));
      CU(cudaStreamSynchronize(ctx->st));
      const double numel = (double)ctx->T_elems * ctx->world;
      const double rms = std::sqrt(h[SC_NT2] / numel);
      use_i8 = h[SC_TMAX] <= 256.0 * rms;
    }
    if (!use_i8) {  // AUTO chose DMMA for these contents: the int8 engine's buffers go back
      if (ctx->Td) cudaFreeAsync(ctx->Td, ctx->st);
      if (ctx->ws_i8) cudaFreeAsync(ctx->ws_i8, ctx->st);
      ctx->Td = nullptr;
      ctx->ws_i8 = nullptr;
      ctx->ws_i8_bytes = 0;
    }
    if (use_i8) {
      int64_t kmax = 1;
      for (int n = 0; n < N; n++) kmax = std::max(kmax, ext(ctx, n));
      // the workspace depends only on the shape and R, so a later cpd_set_tensor reuses it
      if (!ctx->ws_i8) {
        // block contractions (upper-level fusion) run K chunks of up to kMaxKI8 rows
        if (ctx->lv > 1) kmax = cpd::kMaxKI8;
        ctx->ws_i8_bytes = cpd::ttm_i8_workspace_bytes(std::min(kmax, cpd::kMaxKI8), R);
        CU(palloc(ctx, &ctx->ws_i8, ctx->ws_i8_bytes));
      }
      ctx->engine = CPD_ENGINE_INT8_CONVERT;
      // T's digit planes once (7 bytes per element): every first-level TTM then streams them
      // instead of converting T; without the memory the TTM converts T on the fly
      const int64_t w = ext(ctx, N - 1);
      if (ctx->Td || palloc(ctx, (void**)&ctx->Td, (size_t)7 * cpd::digit_plane_bytes(ctx->T_elems, w)) ==
                         cudaSuccess) {
        CU(cpd::launch_slice_digits(ctx->T, ctx->T_elems, w, ctx->texp, ctx->Td, ctx->st));
        ctx->engine = CPD_ENGINE_INT8_DIGITS;
      } else {
        cudaGetLastError();
        ctx->Td = nullptr;
      }
    }
  }
  return CPD_OK;
}

}  // namespace

// ============================== C ABI ==============================================

extern "C" {

cpd_status cpd_opts_default(cpd_opts* o) {
  if (!o) return CPD_ERR_INVALID_ARG;
  std::memset(o, 0, sizeof(*o));
  o->struct_size = sizeof(cpd_opts);
  o->device = 0;
  o->rank = 0;
  o->world = 1;
  o->nccl_unique_id = nullptr;
  o->stream = nullptr;
  o->pp_eps = 0.1;
  o->reuse_root_in_pp_init = 1;
  o->profile_phases = 0;
  o->local_group = nullptr;
  o->ttm_impl = CPD_TTM_AUTO;
  return CPD_OK;
}

cpd_status cpd_nccl_unique_id(void* out) {
  if (!out) return CPD_ERR_INVALID_ARG;
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) {
    g_init_error = ncclGetErrorString(r);
    return CPD_ERR_NCCL;
  }
  static_assert(sizeof(ncclUniqueId) == CPD_NCCL_ID_BYTES, "nccl id size");
  std::memcpy(out, &id, sizeof(id));
  return CPD_OK;
}

cpd_status cpd_local_group_create(int world, cpd_local_group** out) {
  if (!out || world < 1 || world > 8) return CPD_ERR_INVALID_ARG;
  *out = (cpd_local_group*)cpd::local_group_create(world);
  return *out ? CPD_OK : CPD_ERR_OOM;
}

cpd_status cpd_local_group_destroy(cpd_local_group* g) {
  cpd::local_group_destroy((cpd::LocalGroup*)g);
  return CPD_OK;
}

const char* cpd_last_error(const cpd_ctx* c) { return c ? c->err.c_str() : g_init_error.c_str(); }

cpd_status cpd_destroy(cpd_ctx* c) {
  if (!c) return CPD_OK;
  cudaSetDevice(c->dev);
  if (c->st2) cudaStreamSynchronize(c->st2);  // side and filler (speculative PP) work first
  if (c->st3) cudaStreamSynchronize(c->st3);
  clear_subtree(c);
  free_pp(c);
  for (auto* v : {&c->A, &c->Aold, &c->dA, &c->Mlast, &c->Ap, &c->Mp, &c->Mt, &c->Mt2})
    for (auto& p : *v) dfree(c, p);
  dfree(c, c->S_all);
  dfree(c, c->dS_all);
  if (c->st2) cudaStreamSynchronize(c->st2);
  if (c->st3) cudaStreamSynchronize(c->st3);
  for (int b = 0; b < 2; b++) {
    dfree(c, c->Lp[b]);
    dfree(c, c->Wb[b]);
    dfree(c, c->Gi[b]);
  }
  if (c->pf_status) cudaFreeAsync(c->pf_status, c->st);
  dfree(c, c->ws_gram);
  dfree(c, c->ws_mttv);
  dfree(c, c->ws_mttv3);
  dfree(c, c->ws_gj);
  dfree(c, c->st_part);
  dfree(c, c->upd_part);
  dfree(c, c->upd_gpart);
  if (c->st_counter) cudaFreeAsync(c->st_counter, c->st);
  dfree(c, c->scal);
  dfree(c, c->partial);
  dfree(c, c->gather_tmp);
  dfree(c, c->bar_scratch);
  for (int n = 0; n < CPD_MAX_ORDER; n++)
    if (!c->rs_win[n]) dfree(c, c->rs_recv[n]);
  release_cache(c);
  if (c->status) cudaFreeAsync(c->status, c->st);
  if (c->texp) cudaFreeAsync(c->texp, c->st);
  if (c->ws_i8) cudaFreeAsync(c->ws_i8, c->st);
  if (c->Td) cudaFreeAsync(c->Td, c->st);
  cudaStreamSynchronize(c->st);
  if (c->pool) {  // everything was freed above (stream-ordered): hand the memory back to the device
    cudaMemPoolTrimTo(c->pool, 0);
    cudaMemPoolDestroy(c->pool);
    c->pool = nullptr;
  }
  for (auto& r : c->pending) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (auto e : c->free_events) cudaEventDestroy(e);
  if (c->hscal) cudaFreeHost(c->hscal);
  if (c->hstatus) cudaFreeHost(c->hstatus);
  for (int n = 0; n < CPD_MAX_ORDER; n++) {
    if (c->rs_win[n]) {
      cpd::nccl_window_free(c->slice[n].nccl, c->rs_recv[n], c->rs_win[n]);
      c->rs_recv[n] = nullptr;
    }
    cpd::comm_free(c->slice[n]);
    cpd::comm_free(c->fiber[n]);
  }
  if (c->comm) ncclCommDestroy(c->comm);
  if (c->ev_s) cudaEventDestroy(c->ev_s);
  if (c->ev_pf) cudaEventDestroy(c->ev_pf);
  if (c->st2) cudaStreamDestroy(c->st2);
  if (c->ev_in) cudaEventDestroy(c->ev_in);
  if (c->ev_out) cudaEventDestroy(c->ev_out);
  if (c->ev_pp_a) cudaEventDestroy(c->ev_pp_a);
  for (auto e : c->ev_pp_side)
    if (e) cudaEventDestroy(e);
  if (c->st3) cudaStreamDestroy(c->st3);
  if (c->own_stream && c->st) cudaStreamDestroy(c->st);
  delete c;
  return CPD_OK;
}

cpd_status cp_als_init(cpd_ctx** out, int N, const int64_t* shape, int R, const double* T_local_dev,
                       const double* const* A0_host, const cpd_opts* opts) {
  cpd_ctx* ctx = nullptr;
  if (!out || !shape || !T_local_dev || !A0_host) return fail(ctx, CPD_ERR_INVALID_ARG, "null argument");
  *out = nullptr;
  if (N < 3 || N > CPD_MAX_ORDER) return fail(ctx, CPD_ERR_INVALID_ARG, "N must be in [3, 8]");
  if (R < 1 || R > CPD_MAX_RANK) return fail(ctx, CPD_ERR_INVALID_ARG, "R must be in [1, 1024]");
  cpd_opts o;
  cpd_opts_default(&o);
  if (opts) {
    if (opts->struct_size != sizeof(cpd_opts)) return fail(ctx, CPD_ERR_INVALID_ARG, "cpd_opts size mismatch");
    o = *opts;
  }
  if (!(o.pp_eps > 0.0 && o.pp_eps < 1.0)) return fail(ctx, CPD_ERR_INVALID_ARG, "pp_eps must be in (0,1)");
  if (o.world < 1 || o.rank < 0 || o.rank >= o.world) return fail(ctx, CPD_ERR_INVALID_ARG, "bad rank/world");
  if (o.ttm_impl != CPD_TTM_DMMA && o.ttm_impl != CPD_TTM_INT8 && o.ttm_impl != CPD_TTM_AUTO)
    return fail(ctx, CPD_ERR_INVALID_ARG, "bad ttm_impl");
  if (o.msdt_levels == 0) o.msdt_levels = 1;
  if (o.msdt_levels < 1 || o.msdt_levels > N - 2)
    return fail(ctx, CPD_ERR_INVALID_ARG, "msdt_levels must be in [1, N-2] (P:700-702: l <= N-2)");
  if (o.world > 1 && !o.nccl_unique_id && !o.local_group)
    return fail(ctx, CPD_ERR_INVALID_ARG, "world > 1 needs nccl_unique_id or local_group");
  if (o.local_group && cpd::local_group_world((cpd::LocalGroup*)o.local_group) != o.world)
    return fail(ctx, CPD_ERR_INVALID_ARG, "local_group size != world");
  for (int n = 0; n < N; n++)
    if (shape[n] < 1 || !A0_host[n]) return fail(ctx, CPD_ERR_INVALID_ARG, "bad shape or factor");
  // processor grid (Alg. 3 line 1): opts.grid, or the 1-D default 1 x .. x 1 x world
  int grid[CPD_MAX_ORDER];
  {
    bool given = false;
    for (int n = 0; n < CPD_MAX_ORDER; n++) given |= o.grid[n] != 0;
    int64_t prod = 1;
    for (int n = 0; n < N; n++) {
      grid[n] = given ? o.grid[n] : (n == N - 1 ? o.world : 1);
      if (grid[n] < 1) return fail(ctx, CPD_ERR_INVALID_ARG, "grid entries must be >= 1");
      prod *= grid[n];
    }
    for (int n = N; n < CPD_MAX_ORDER; n++)
      if (given && o.grid[n] != 0) return fail(ctx, CPD_ERR_INVALID_ARG, "grid entries beyond N must be 0");
    if (prod != o.world) return fail(ctx, CPD_ERR_INVALID_ARG, "prod(grid) must equal world");
    for (int n = 0; n < N; n++) {
      // blocks of s_n / I_n rows (reading Q20: no padding), own rows of loc / (P / I_n)
      if (shape[n] % grid[n] != 0) return fail(ctx, CPD_ERR_INVALID_ARG, "s_n must be divisible by grid[n]");
      if ((shape[n] / grid[n]) % (o.world / grid[n]) != 0)
        return fail(ctx, CPD_ERR_INVALID_ARG, "s_n / grid[n] must be divisible by world / grid[n] (reduce-scatter)");
    }
  }

  ctx = new cpd_ctx();
  ctx->N = N;
  ctx->lv = o.msdt_levels;
  ctx->R = R;
  for (int n = 0; n < N; n++) ctx->shape[n] = shape[n];
  ctx->rank = o.rank;
  ctx->world = o.world;
  {
    int rem = o.rank;
    for (int n = N - 1; n >= 0; n--) {  // row-major rank order, last mode fastest
      ctx->grid[n] = grid[n];
      ctx->coord[n] = rem % grid[n];
      rem /= grid[n];
      ctx->loc[n] = shape[n] / grid[n];
    }
  }
  ctx->dev = o.device;
  ctx->opts = o;
  ctx->T = T_local_dev;
  ctx->T_elems = 1;
  for (int n = 0; n < N; n++) ctx->T_elems *= ctx->loc[n];

  auto bail = [&](cpd_status s) {
    g_init_error = ctx->err;
    cpd_destroy(ctx);
    return s;
  };
#define ICU(x)                                                                   \
  do {                                                                           \
    cudaError_t e_ = (x);                                                        \
    if (e_ != cudaSuccess) {                                                     \
      fail(ctx, CPD_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
      return bail(CPD_ERR_CUDA);                                                 \
    }                                                                            \
  } while (0)
#define ITRY(x)                   \
  do {                            \
    cpd_status s_ = (x);          \
    if (s_ != CPD_OK) return bail(s_); \
  } while (0)

  ICU(cudaSetDevice(ctx->dev));
  {
    int major = 0;
    ICU(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, ctx->dev));
    if (major != 10) {
      fail(ctx, CPD_ERR_CUDA, "libcpd.so is built for sm_100a (B200) only");
      return bail(CPD_ERR_CUDA);
    }
  }
  {
    int lo = 0, hi = 0;
    ICU(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    ICU(cudaStreamCreateWithPriority(&ctx->st, cudaStreamNonBlocking, hi < lo ? hi + 1 : hi));
    ctx->own_stream = true;
    ctx->ust = (cudaStream_t)o.stream;
    ICU(cudaEventCreateWithFlags(&ctx->ev_in, cudaEventDisableTiming));
    ICU(cudaEventCreateWithFlags(&ctx->ev_out, cudaEventDisableTiming));
    // the borrowed T (and anything else the caller enqueued) precedes the library's work
    ICU(cudaEventRecord(ctx->ev_in, ctx->ust));
    ICU(cudaStreamWaitEvent(ctx->st, ctx->ev_in, 0));
  }
  {
    cudaMemPoolProps pp{};
    pp.allocType = cudaMemAllocationTypePinned;
    pp.handleTypes = cudaMemHandleTypeNone;
    pp.location.type = cudaMemLocationTypeDevice;
    pp.location.id = ctx->dev;
    ICU(cudaMemPoolCreate(&ctx->pool, &pp));
    uint64_t thr = UINT64_MAX;
    ICU(cudaMemPoolSetAttribute(ctx->pool, cudaMemPoolAttrReleaseThreshold, &thr));
  }
  if (o.world > 1 && !o.local_group) {
    ncclUniqueId id;
    std::memcpy(&id, o.nccl_unique_id, sizeof(id));
    ncclResult_t r = ncclCommInitRank(&ctx->comm, o.world, id, o.rank);
    if (r != ncclSuccess) {
      fail(ctx, CPD_ERR_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
      return bail(CPD_ERR_NCCL);
    }
  }
  ctx->cm.nccl = ctx->comm;
  ctx->cm.lg = (cpd::LocalGroup*)o.local_group;
  ctx->cm.rank = o.rank;
  ctx->cm.world = o.world;
  ctx->cm.st = ctx->st;
  {
    // Proc-Slice(x_n) and the fibre of mode n; the whole world or a single rank need no new
    // communicator (the 1-D grid: slices of modes < N are the world, of mode N single ranks)
    cpd::Comm self;
    self.st = ctx->st;
    for (int n = 0; n < N; n++) {
      std::string m;
      int rest = 0;  // rank with x_n removed
      for (int k = 0; k < N; k++)
        if (k != n) rest = rest * grid[k] + ctx->coord[k];
      if (grid[n] == 1) ctx->slice[n] = ctx->cm;
      else if (grid[n] == o.world) ctx->slice[n] = self;
      else if (cpd::comm_split(ctx->cm, ctx->coord[n], o.rank, &ctx->slice[n], &m)) {
        fail(ctx, CPD_ERR_NCCL, m);
        return bail(CPD_ERR_NCCL);
      }
      if (grid[n] == 1) ctx->fiber[n] = self;
      else if (grid[n] == o.world) ctx->fiber[n] = ctx->cm;
      else if (cpd::comm_split(ctx->cm, rest, ctx->coord[n], &ctx->fiber[n], &m)) {
        fail(ctx, CPD_ERR_NCCL, m);
        return bail(CPD_ERR_NCCL);
      }
    }
  }
  const int64_t RR = (int64_t)R * R;
  ctx->A.assign(N, nullptr);
  ctx->Aold.assign(N, nullptr);
  ctx->dA.assign(N, nullptr);
  ctx->Mlast.assign(N, nullptr);
  ctx->Ap.assign(N, nullptr);
  ctx->Mp.assign(N, nullptr);
  ctx->Mt.assign(N, nullptr);
  ctx->Mt2.assign(N, nullptr);
  ctx->Mlast_src.assign(N, nullptr);
  for (int n = 0; n < N; n++) {
    int64_t e = ext(ctx, n) * R;
    ITRY(dalloc(ctx, &ctx->A[n], e));
    ITRY(dalloc(ctx, &ctx->Aold[n], e));
    ITRY(dalloc(ctx, &ctx->dA[n], e));
    ITRY(dalloc(ctx, &ctx->Mlast[n], e));
    ITRY(dalloc(ctx, &ctx->Ap[n], e));
  }
  ITRY(dalloc(ctx, &ctx->S_all, N * RR));
  ITRY(dalloc(ctx, &ctx->dS_all, N * RR));
  for (int b2 = 0; b2 < 2; b2++) {
    ITRY(dalloc(ctx, &ctx->Lp[b2], RR + R));
    ITRY(dalloc(ctx, &ctx->Wb[b2], RR));
    if (R <= cpd::kUpdMaxR || R > kCholMaxR) ITRY(dalloc(ctx, &ctx->Gi[b2], RR));
  }
  ICU(palloc(ctx, (void**)&ctx->pf_status, sizeof(int) * 2));
  ICU(cudaMemsetAsync(ctx->pf_status, 0, sizeof(int) * 2, ctx->st));
  {
    // the side stream (Γ factor / inverse, W) must not queue behind the MTTKRP stream's CTAs
    int lo = 0, hi = 0;
    ICU(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    ICU(cudaStreamCreateWithPriority(&ctx->st2, cudaStreamNonBlocking, hi));
  }
  ICU(cudaEventCreateWithFlags(&ctx->ev_s, cudaEventDisableTiming));
  ICU(cudaEventCreateWithFlags(&ctx->ev_pf, cudaEventDisableTiming));
  {
    // filler stream for PP operator streams off the critical path: lowest priority
    int lo = 0, hi = 0;
    ICU(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    ICU(cudaStreamCreateWithPriority(&ctx->st3, cudaStreamNonBlocking, lo));
  }
  ICU(cudaEventCreateWithFlags(&ctx->ev_pp_a, cudaEventDisableTiming));
  for (int n = 0; n < N; n++) ICU(cudaEventCreateWithFlags(&ctx->ev_pp_side[n], cudaEventDisableTiming));
  ITRY(dalloc(ctx, &ctx->ws_gram, 32 * RR));
  ITRY(dalloc(ctx, &ctx->ws_mttv, kMttvWs));
  ITRY(dalloc(ctx, &ctx->ws_mttv3, kMttvWs));
  if (R > kCholMaxR) ITRY(dalloc(ctx, &ctx->ws_gj, (int64_t)cpd::gamma_inverse_big_ws(R)));
  ITRY(dalloc(ctx, &ctx->st_part, 3 * 64));
  ITRY(dalloc(ctx, &ctx->upd_part, 3 * cpd::kUpdMaxBlocks));
  if (R <= cpd::kUpdMaxR) ITRY(dalloc(ctx, &ctx->upd_gpart, (int64_t)cpd::kUpdMaxBlocks * 2 * RR));
  ICU(palloc(ctx, (void**)&ctx->st_counter, sizeof(unsigned int)));
  ICU(cudaMemsetAsync(ctx->st_counter, 0, sizeof(unsigned int), ctx->st));
  ITRY(dalloc(ctx, &ctx->scal, SC_COUNT));
  ITRY(dalloc(ctx, &ctx->partial, cpd::kNormBlocks));
  ICU(palloc(ctx, (void**)&ctx->status, sizeof(int) * CPD_MAX_ORDER));
  ICU(cudaMemsetAsync(ctx->status, 0, sizeof(int) * CPD_MAX_ORDER, ctx->st));
  ICU(cudaMemsetAsync(ctx->scal, 0, sizeof(double) * SC_COUNT, ctx->st));
  ICU(cudaMemsetAsync(ctx->dS_all, 0, sizeof(double) * N * RR, ctx->st));
  ICU(cudaMallocHost((void**)&ctx->hscal, sizeof(double) * SC_COUNT));
  ICU(cudaMallocHost((void**)&ctx->hstatus, sizeof(int) * CPD_MAX_ORDER));
  if (o.fused_rs && o.world > 1) {
    // fused reduce-scatter epilogue: receive buffers and every rank's slot map
    ITRY(dalloc(ctx, &ctx->bar_scratch, 1));
    ICU(cudaMemsetAsync(ctx->bar_scratch, 0, sizeof(double), ctx->st));
    for (int n = 0; n < N; n++) {
      cpd::Comm& sl = ctx->slice[n];
      if (sl.world == 1) continue;
      if (sl.world > 8) {
        fail(ctx, CPD_ERR_INVALID_ARG, "fused_rs: at most 8 ranks per slice");
        return bail(CPD_ERR_INVALID_ARG);
      }
      const int64_t chunk = (ctx->loc[n] / sl.world) * R;
      void* peers[8] = {};
      std::string m;
      if (sl.lg) {
        ITRY(dalloc(ctx, &ctx->rs_recv[n], sl.world * chunk));
        ICU(cudaStreamSynchronize(ctx->st));
        if (cpd::comm_exchange_ptr(sl, ctx->rs_recv[n], peers, &m)) {
          fail(ctx, CPD_ERR_CUDA, m);
          return bail(CPD_ERR_CUDA);
        }
      } else {
        void* buf = nullptr;
        if (cpd::nccl_window_peers(sl.nccl, sizeof(double) * sl.world * chunk, sl.world, &buf, peers, &ctx->rs_win[n],
                                   ctx->st, &m)) {
          fail(ctx, CPD_ERR_NCCL, m);
          return bail(CPD_ERR_NCCL);
        }
        ctx->rs_recv[n] = static_cast<double*>(buf);
      }
      ctx->rs_map[n].nq = sl.world;
      ctx->rs_map[n].chunk = chunk;
      for (int q = 0; q < sl.world; q++) ctx->rs_map[n].dst[q] = static_cast<double*>(peers[q]) + sl.rank * chunk;
    }
  }
  *out = ctx;  // provisional for cpd_set_factors
  // ||T||^2 once, all-reduced
  {
    cpd_status ps = prepare_tensor(ctx);
    if (ps != CPD_OK) {
      *out = nullptr;
      return bail(ps);
    }
  }
  cpd_status s = cpd_set_factors(ctx, A0_host);
  if (s != CPD_OK) {
    *out = nullptr;
    return bail(s);
  }
  ICU(cudaStreamSynchronize(ctx->st));
  ICU(cudaMemcpy(ctx->hscal, ctx->scal, sizeof(double) * SC_COUNT, cudaMemcpyDeviceToHost));
  if (!(ctx->hscal[SC_NT2] > 0.0) || !std::isfinite(ctx->hscal[SC_NT2])) {
    *out = nullptr;
    fail(ctx, CPD_ERR_NUMERIC, "||T||^2 is zero or not finite");
    return bail(CPD_ERR_NUMERIC);
  }
  // dA <- A (Alg. 2 line 2): the first regular sweep always precedes PP
  for (int n = 0; n < N; n++) {
    ctx->dA2[n] = 1.0;
    ctx->A2[n] = 1.0;
  }
  ctx->have_dA = false;
  return CPD_OK;
#undef ICU
#undef ITRY
}

cpd_status cpd_set_factors(cpd_ctx* ctx, const double* const* A_host) {
  TRY(check_ctx(ctx));
  UserSync us_(ctx);
  if (!A_host) return fail(ctx, CPD_ERR_INVALID_ARG, "null factors");
  const int R = ctx->R;
  const int64_t RR = (int64_t)R * R;
  for (int n = 0; n < ctx->N; n++) {
    if (!A_host[n]) return fail(ctx, CPD_ERR_INVALID_ARG, "null factor");
    // the block rows of mode n (Alg. 3 lines 4-8); S^(n) = the sum of the blocks' Grams over the fibre
    const double* src = A_host[n] + ctx->coord[n] * ext(ctx, n) * R;
    CU(cudaMemcpyAsync(ctx->A[n], src, sizeof(double) * ext(ctx, n) * R, cudaMemcpyHostToDevice, ctx->st));
    CU(cpd::launch_gram(ctx->A[n], ctx->A[n], nullptr, ext(ctx, n), R, ctx->S_all + n * RR, nullptr,
                        ctx->ws_gram, 32 * RR, ctx->st));
    CM(cpd::comm_all_reduce(ctx->fiber[n], ctx->S_all + n * RR, RR, &m_));
  }
  clear_subtree(ctx);
  ctx->t = 0;
  ctx->sub_is_msdt = false;
  free_pp(ctx);
  ctx->pp_regime = false;
  ctx->have_dA = false;
  invalidate_prefetch(ctx);
  CU(cudaStreamSynchronize(ctx->st));
  return CPD_OK;
}

cpd_status cpd_set_tensor(cpd_ctx* ctx) {
  TRY(check_ctx(ctx));
  UserSync us_(ctx);
  TRY(prepare_tensor(ctx));
  CU(cudaStreamSynchronize(ctx->st));
  CU(cudaMemcpy(ctx->hscal, ctx->scal, sizeof(double) * SC_COUNT, cudaMemcpyDeviceToHost));
  if (!(ctx->hscal[SC_NT2] > 0.0) || !std::isfinite(ctx->hscal[SC_NT2]))
    return fail(ctx, CPD_ERR_NUMERIC, "||T||^2 is zero or not finite");
  // every cached tree node and PP operator was built from the old contents
  clear_subtree(ctx);
  ctx->t = 0;
  ctx->sub_is_msdt = false;
  free_pp(ctx);
  ctx->pp_regime = false;
  ctx->have_dA = false;
  ctx->have_fit = false;
  return CPD_OK;
}

// a regular sweep after a PP sweep drops the speculative next-sweep PP streams without waiting
// for them up front: its first-level TTM (reads T and A only) overlaps them, and the main stream
// waits for them just before its first factor update (drop_spec in regular_sweep)
cpd_status msdt_sweep(cpd_ctx* ctx, double* fitness_out) {
  TRY(check_ctx(ctx));
  UserSync us_(ctx, true);
  return regular_sweep(ctx, true, fitness_out);
}

cpd_status dt_sweep(cpd_ctx* ctx, double* fitness_out) {
  TRY(check_ctx(ctx));
  UserSync us_(ctx, true);
  return regular_sweep(ctx, false, fitness_out);
}

cpd_status pp_init(cpd_ctx* ctx) {
  TRY(check_ctx(ctx));
  UserSync us_(ctx);
  const int N = ctx->N;
  free_pp(ctx);
  // A_p <- A, dA <- 0 (Alg. 2 line 7)
  for (int n = 0; n < N; n++) {
    CU(cudaMemcpyAsync(ctx->Ap[n], ctx->A[n], sizeof(double) * ext(ctx, n) * ctx->R,
                       cudaMemcpyDeviceToDevice, ctx->st));
    CU(cudaMemsetAsync(ctx->dA[n], 0, sizeof(double) * ext(ctx, n) * ctx->R, ctx->st));
  }
  CU(cudaMemsetAsync(ctx->dS_all, 0, sizeof(double) * N * ctx->R * ctx->R, ctx->st));
  invalidate_prefetch(ctx);  // W depends on dS
  // three first-level roots; reuse the live MSDT root when valid (P:384 footnote)
  std::vector<int> js;
  int live = (ctx->opts.reuse_root_in_pp_init && ctx->sub_is_msdt && ctx->sub.active && !ctx->pp_regime)
                 ? ctx->sub.j
                 : -1;
  Node live_root;
  if (live >= 0) {
    auto it = ctx->sub.cache.find({0, (int)ctx->sub.served.size()});
    if (it != ctx->sub.cache.end() && (int)it->second.kept.size() == N - 1) {
      live_root = it->second;
      ctx->sub.cache.erase(it);
      js.push_back(live);
    } else {
      live = -1;
    }
  }
  clear_subtree(ctx);
  ctx->t = 0;
  ctx->sub_is_msdt = false;
  for (int j : {N - 1, 1, 0, 2, 3})
    if ((int)js.size() < 3 && std::find(js.begin(), js.end(), j) == js.end()) js.push_back(j);
  std::map<int, std::vector<std::pair<int, int>>> assign;
  for (int a = 0; a < N; a++)
    for (int b = a + 1; b < N; b++)
      for (int j : js)
        if (j != a && j != b) {
          assign[j].push_back({a, b});
          break;
        }
  // factors used for the operators are A_p (== A now)
  for (int j : js) {
    Node root;
    if (j == live) {
      root = live_root;
    } else {
      for (int m = 0; m < N; m++)
        if (m != j) root.kept.push_back(m);
      TRY(dalloc(ctx, &root.buf, node_elems(ctx, root.kept)));
      TRY(ttm(ctx, j, root.buf));
    }
    if (root.kept.size() == 2) {
      ctx->ops[{root.kept[0], root.kept[1]}] = root.buf;  // N = 3: the root is the operator
    } else {
      TRY(pp_descend(ctx, root, assign[j]));
      dfree(ctx, root.buf);
    }
  }
  if ((int)ctx->ops.size() != N * (N - 1) / 2) return fail(ctx, CPD_ERR_INTERNAL, "missing PP operators");
  // M_p^(n) from a pair operator containing n
  for (int n = 0; n < N; n++) {
    int o = n == 0 ? 1 : 0;
    int a = std::min(n, o), b = std::max(n, o);
    TRY(dalloc(ctx, &ctx->Mp[n], ext(ctx, n) * ctx->R));
    TRY(dalloc(ctx, &ctx->Mt[n], ext(ctx, n) * ctx->R));
    TRY(dalloc(ctx, &ctx->Mt2[n], ext(ctx, n) * ctx->R));
    TRY(mttv(ctx, ctx->ops[{a, b}], {a, b}, o, ctx->Ap[o], ctx->Mp[n], 0));
  }
  CU(cudaStreamSynchronize(ctx->st));
  drain_timers(ctx);
  ctx->pp_valid = true;
  ctx->pp_regime = true;
  ctx->pp_fresh = true;
  for (int n = 0; n < N; n++) ctx->dA2[n] = 0.0;
  ctx->have_dA = true;
  return CPD_OK;
}

cpd_status pp_approx_sweep(cpd_ctx* ctx, double* fitness_out, int* still_valid) {
  TRY(check_ctx(ctx));
  UserSync us_(ctx, true);
  if (!ctx->pp_valid || !ctx->pp_regime) return fail(ctx, CPD_ERR_STATE, "pp_approx_sweep needs a valid pp_init");
  const int N = ctx->N;
  // operator [s_a, s_b, R] of the pair {n, i}: contract the axis of mode i with dA^(i) (Eq. 6)
  auto spec = [&](int n, int i, double* bytes) {
    const int a = std::min(n, i), b = std::max(n, i);
    cpd::MttvSpec sp;
    sp.X = ctx->ops[{a, b}];
    sp.v = ctx->dA[i];
    sp.K = ext(ctx, i);
    sp.pre = n < i ? ext(ctx, n) : 1;
    sp.post = n < i ? 1 : ext(ctx, n);
    *bytes += 8.0 * ((double)ext(ctx, a) * ext(ctx, b) * ctx->R + (double)ext(ctx, i) * ctx->R);
    return sp;
  };
  // M~_loc^(n) = M_p^(n) + Σ_{i≠n} U^(n,i) (Eqs. 5-6).  Only U^(n,n-1) waits for update n-1;
  // the other N-2 streams of mode n (their dA are final once update n-2 is done) are issued on
  // st3 one mode ahead, into Mt[n] = M_p^(n) + Σ_indep U, and the main stream adds U^(n,n-1).
  // Fixed summation order: ((M_p + Σ_indep U in ascending i) + U^(n,n-1)).
  double* const* Mcur = ctx->mt_par ? ctx->Mt2.data() : ctx->Mt.data();
  double* const* Mnxt = ctx->mt_par ? ctx->Mt.data() : ctx->Mt2.data();
  // the independent streams of mode nx (all i != nx, nx-1) on the filler stream into M[nx]
  // first sweep after pp_init: dA = 0 for every mode not yet updated in this sweep (Alg. 2 line 7), so
  // U^(n,i) = 0 exactly (Eq. 6) for those i and M~ starts as M_p: mode 0 entirely, mode 1's filler part
  bool fresh = ctx->pp_fresh;  // cleared after the mode loop: the speculation for the NEXT sweep sees dA != 0
  ctx->pp_fresh = false;
  auto side = [&](int nx, double* const* M) -> cpd_status {
    if (fresh && nx == 1) {
      CU(cudaEventRecord(ctx->ev_pp_a, ctx->st));
      CU(cudaStreamWaitEvent(ctx->st3, ctx->ev_pp_a, 0));
      CU(cudaMemcpyAsync(M[nx], ctx->Mp[nx], sizeof(double) * ext(ctx, nx) * ctx->R, cudaMemcpyDeviceToDevice,
                         ctx->st3));
      CU(cudaEventRecord(ctx->ev_pp_side[nx], ctx->st3));
      return CPD_OK;
    }
    cpd::MttvSpec sp[CPD_MAX_ORDER];
    int J = 0;
    double bytes = 0.0;
    for (int i = 0; i < N; i++)
      if (i != nx && i != nx - 1) sp[J++] = spec(nx, i, &bytes);
    CU(cudaEventRecord(ctx->ev_pp_a, ctx->st));  // update nx-2 (and everything before) enqueued
    CU(cudaStreamWaitEvent(ctx->st3, ctx->ev_pp_a, 0));
    CU(cpd::launch_mttv_multi(sp, J, ctx->R, ctx->Mp[nx], M[nx], 0, ctx->ws_mttv3, kMttvWs, ctx->st3, nullptr,
                                    filler_occ3(), filler_waves()));
    CU(cudaEventRecord(ctx->ev_pp_side[nx], ctx->st3));
    ctx->filler[0] += bytes + 8.0 * 2 * ext(ctx, nx) * ctx->R;
    ctx->filler[1] += 1;
    return CPD_OK;
  };
  static const bool no_spec = getenv("CPD_NO_PP_SPEC") != nullptr;
  static const bool no_spec0 = getenv("CPD_NO_PP_SPEC0") != nullptr;
  const bool spec0 = N > 2 && !no_spec && !no_spec0 && !rs_map_of(ctx, 0);
  for (int n = 0; n < N; n++) {
    const int nx = n + 1;
    if (nx < N && N > 2) {
      if (nx == 1 && ctx->pp_spec) ctx->pp_spec = false;  // started at the end of the last sweep
      else TRY(side(nx, Mcur));
    }
    if (n == N - 1 && spec0) {
      // the next sweep's M~^(0) without its last term: M_p^(0) + Σ_{i<N-1} U^(0,i) (those dA are final
      // once update N-2 is done), on the filler stream while mode N-1 streams
      cpd::MttvSpec sp[CPD_MAX_ORDER];
      int J = 0;
      double bytes = 0.0;
      for (int i = 1; i < N - 1; i++) sp[J++] = spec(0, i, &bytes);
      CU(cudaEventRecord(ctx->ev_pp_a, ctx->st));
      CU(cudaStreamWaitEvent(ctx->st3, ctx->ev_pp_a, 0));
      CU(cpd::launch_mttv_multi(sp, J, ctx->R, ctx->Mp[0], Mnxt[0], 0, ctx->ws_mttv3, kMttvWs, ctx->st3, nullptr,
                                    filler_occ3(), filler_waves()));
      ctx->filler[0] += bytes + 8.0 * 2 * ext(ctx, 0) * ctx->R;
      ctx->filler[1] += 1;
    }
    double* Mt = Mcur[n];
    cpd::MttvSpec sp[CPD_MAX_ORDER];
    int J = 0;
    double bytes = 0.0;
    // the critical stream's K-split reduction is done by the fused update that consumes M~ (one launch
    // and its gap fewer on the serial chain); experiment switch CPD_NO_DEFER_REDUCE
    static const bool no_defer = getenv("CPD_NO_DEFER_REDUCE") != nullptr;
    cpd::MPending pend;
    // the launch that completes M~_loc^(n) stores it into the owners' slots under the fused RS
    const cpd::OutMap* mp = rs_map_of(ctx, n);
    if (n == 0 && ctx->pp_spec0) {
      // M~^(0) was completed on the filler stream at the end of the last sweep (all its dA final)
      CU(cudaStreamWaitEvent(ctx->st, ctx->ev_pp_side[0], 0));
      ctx->pp_spec0 = false;
    } else if (n == 0 && fresh && !mp) {
      CU(cudaMemcpyAsync(Mt, ctx->Mp[0], sizeof(double) * ext(ctx, 0) * ctx->R, cudaMemcpyDeviceToDevice, ctx->st));
    } else if (n == 0 || N <= 2) {
      for (int i = 0; i < N; i++)
        if (i != n) sp[J++] = spec(n, i, &bytes);
      PhaseScope ps(ctx, PH_MTTV);
      CU(cpd::launch_mttv_multi(sp, J, ctx->R, ctx->Mp[n], Mt, 0, ctx->ws_mttv, kMttvWs, ctx->st, mp));
      ctx->counters[2] += 8.0 * 2 * ext(ctx, n) * ctx->R;
    } else {
      sp[J++] = spec(n, n - 1, &bytes);
      CU(cudaStreamWaitEvent(ctx->st, ctx->ev_pp_side[n], 0));
      PhaseScope ps(ctx, PH_MTTV);
      const bool defer = !no_defer && !mp && ctx->slice[n].world == 1 && use_fused(ctx, n, true);
      CU(cpd::launch_mttv_multi(sp, J, ctx->R, nullptr, Mt, 1, ctx->ws_mttv, kMttvWs, ctx->st, mp, false, 0,
                                defer ? &pend : nullptr));
      ctx->counters[2] += 8.0 * 2 * ext(ctx, n) * ctx->R;
    }
    ctx->counters[2] += bytes;
    ctx->counters[3] += 1;
    TRY(update_mode(ctx, n, Mt, true, rs_map_of(ctx, n) != nullptr, &pend));
  }
  // speculation: the next sweep's mode-1 independent streams need only this sweep's final dA,
  // so they start now and overlap the end of this sweep and the host round trip; this sweep's
  // M~ (readable through cpd_get_last_mttkrp) stays intact in the other buffer set
  fresh = false;
  // Mode 0 of the next sweep needs only this sweep's final dA as well: its last term U^(0,N-1) completes
  // the M~^(0) started during mode N-1, first on the filler stream, so the next sweep starts with its
  // first update (not with the fused reduce-scatter, whose slots must be written by the consuming sweep)
  if (N > 2 && !no_spec) {
    if (spec0) {
      cpd::MttvSpec sp[1];
      double bytes = 0.0;
      sp[0] = spec(0, N - 1, &bytes);
      CU(cudaEventRecord(ctx->ev_pp_a, ctx->st));
      CU(cudaStreamWaitEvent(ctx->st3, ctx->ev_pp_a, 0));
      CU(cpd::launch_mttv_multi(sp, 1, ctx->R, nullptr, Mnxt[0], 1, ctx->ws_mttv3, kMttvWs, ctx->st3, nullptr,
                                    filler_occ3(), filler_waves()));
      CU(cudaEventRecord(ctx->ev_pp_side[0], ctx->st3));
      ctx->filler[0] += bytes + 8.0 * 2 * ext(ctx, 0) * ctx->R;
      ctx->filler[1] += 1;
      ctx->pp_spec0 = true;
    }
    TRY(side(1, Mnxt));
    ctx->pp_spec = true;
  }
  ctx->mt_par ^= 1;
  TRY(finish_sweep(ctx, fitness_out));
  if (still_valid) *still_valid = pp_cond(ctx) ? 1 : 0;
  return CPD_OK;
}

cpd_status fitness(cpd_ctx* ctx, double* f_out) {
  if (!ctx || !f_out) return CPD_ERR_INVALID_ARG;
  if (!ctx->have_fit) return fail(ctx, CPD_ERR_STATE, "no completed sweep");
  *f_out = ctx->last_f;
  return CPD_OK;
}

cpd_status cpd_pp_condition(cpd_ctx* ctx, int* ok) {
  if (!ctx || !ok) return CPD_ERR_INVALID_ARG;
  *ok = ctx->have_dA ? (pp_cond(ctx) ? 1 : 0) : 0;
  return CPD_OK;
}

// the GLOBAL s_n x R matrix from this rank's block rows (valid on every rank of the slice):
// all-gathered over the fibre of mode n0 (fibre ranks are ordered by x_n)
static cpd_status gather_rows(cpd_ctx* ctx, int n0, const double* src_block, double* host_out) {
  const int R = ctx->R;
  const int64_t e = ext(ctx, n0) * R;
  cpd::Comm& fb = ctx->fiber[n0];
  if (fb.world == 1) {
    CU(cudaMemcpyAsync(host_out, src_block, sizeof(double) * e, cudaMemcpyDeviceToHost, ctx->st));
  } else {
    if (!ctx->gather_tmp) {
      int64_t mx = 0;
      for (int n = 0; n < ctx->N; n++) mx = std::max(mx, ctx->shape[n]);
      TRY(dalloc(ctx, &ctx->gather_tmp, mx * R));
    }
    CM(cpd::comm_all_gather(fb, src_block, ctx->gather_tmp, e, &m_));
    CU(cudaMemcpyAsync(host_out, ctx->gather_tmp, sizeof(double) * ctx->shape[n0] * R, cudaMemcpyDeviceToHost,
                       ctx->st));
  }
  CU(cudaStreamSynchronize(ctx->st));
  return CPD_OK;
}

cpd_status cpd_get_factor(cpd_ctx* ctx, int n0, double* host_out) {
  TRY(check_ctx(ctx));
  UserSync us_(ctx);
  if (n0 < 0 || n0 >= ctx->N || !host_out) return fail(ctx, CPD_ERR_INVALID_ARG, "bad mode");
  return gather_rows(ctx, n0, ctx->A[n0], host_out);
}

cpd_status cpd_get_last_mttkrp(cpd_ctx* ctx, int n0, double* host_out) {
  TRY(check_ctx(ctx));
  UserSync us_(ctx);
  if (n0 < 0 || n0 >= ctx->N || !host_out) return fail(ctx, CPD_ERR_INVALID_ARG, "bad mode");
  const int64_t ro = rows_own(ctx, n0), off = own_off(ctx, n0);
  if (ctx->Mlast_src[n0])
    CU(cudaMemcpyAsync(ctx->Mlast[n0] + off * ctx->R, ctx->Mlast_src[n0] + off * ctx->R,
                       sizeof(double) * ro * ctx->R, cudaMemcpyDeviceToDevice, ctx->st));
  // own rows (after the reduce-scatter) -> the block (slice) -> the global matrix (fibre)
  if (ctx->slice[n0].world > 1)
    CM(cpd::comm_all_gather(ctx->slice[n0], ctx->Mlast[n0] + off * ctx->R, ctx->Mlast[n0], ro * ctx->R, &m_));
  return gather_rows(ctx, n0, ctx->Mlast[n0], host_out);
}

cpd_status cpd_get_phase_ms(cpd_ctx* ctx, double out[5]) {
  if (!ctx || !out) return CPD_ERR_INVALID_ARG;
  cudaStreamSynchronize(ctx->st);
  cudaStreamSynchronize(ctx->st3);
  drain_timers(ctx, true);
  for (int i = 0; i < 5; i++) out[i] = ctx->phase_ms[i];
  return CPD_OK;
}

cpd_status cpd_last_sweep_status(const cpd_ctx* ctx, int* flags, double* radicand_rel) {
  if (!ctx || !flags) return CPD_ERR_INVALID_ARG;
  *flags = ctx->last_flags;
  if (radicand_rel) *radicand_rel = ctx->last_rad_rel;
  return CPD_OK;
}

cpd_status cpd_ttm_engine(const cpd_ctx* ctx, int* engine) {
  if (!ctx || !engine) return CPD_ERR_INVALID_ARG;
  *engine = ctx->engine;
  return CPD_OK;
}

cpd_status cpd_get_counters(cpd_ctx* ctx, double out[6]) {
  if (!ctx || !out) return CPD_ERR_INVALID_ARG;
  for (int i = 0; i < 5; i++) out[i] = ctx->counters[i];
  out[5] = (double)cpd::g_launches.load();
  return CPD_OK;
}

cpd_status cpd_get_ttm_bytes(cpd_ctx* ctx, double* out) {
  if (!ctx || !out) return CPD_ERR_INVALID_ARG;
  *out = ctx->ttm_bytes;
  return CPD_OK;
}

cpd_status cpd_get_memory(cpd_ctx* ctx, double out[3]) {
  if (!ctx || !out) return CPD_ERR_INVALID_ARG;
  out[0] = ctx->node_peak;
  out[1] = ctx->node_live;
  out[2] = ctx->Td ? 7.0 * (double)cpd::digit_plane_bytes(ctx->T_elems, ext(ctx, ctx->N - 1)) : 0.0;
  return CPD_OK;
}

cpd_status cpd_get_filler_counters(cpd_ctx* ctx, double out[2]) {
  if (!ctx || !out) return CPD_ERR_INVALID_ARG;
  out[0] = ctx->filler[0];
  out[1] = ctx->filler[1];
  return CPD_OK;
}

cpd_status cpd_set_profile_level(cpd_ctx* ctx, int level) {
  if (!ctx || level < 0 || level > 2) return CPD_ERR_INVALID_ARG;
  cudaStreamSynchronize(ctx->st);
  cudaStreamSynchronize(ctx->st3);
  drain_timers(ctx, true);
  ctx->opts.profile_phases = level;
  return CPD_OK;
}

cpd_status cpd_reset_counters(cpd_ctx* ctx) {
  if (!ctx) return CPD_ERR_INVALID_ARG;
  cudaStreamSynchronize(ctx->st);
  cudaStreamSynchronize(ctx->st3);
  drain_timers(ctx, true);
  for (int i = 0; i < 5; i++) ctx->phase_ms[i] = ctx->counters[i] = 0.0;
  ctx->filler[0] = ctx->filler[1] = 0.0;
  ctx->node_peak = ctx->node_live;
  ctx->ttm_bytes = 0.0;
  return CPD_OK;
}

cpd_status cpd_debug_get_pp_operator(cpd_ctx* ctx, int a0, int b0, double* host_out) {
  TRY(check_ctx(ctx));
  UserSync us_(ctx);
  if (!ctx->pp_valid) return fail(ctx, CPD_ERR_STATE, "no PP operators");
  if (a0 < 0 || b0 <= a0 || b0 >= ctx->N || !host_out) return fail(ctx, CPD_ERR_INVALID_ARG, "bad pair");
  auto it = ctx->ops.find({a0, b0});
  if (it == ctx->ops.end()) return fail(ctx, CPD_ERR_INTERNAL, "operator missing");
  int64_t e = ext(ctx, a0) * ext(ctx, b0) * ctx->R;
  CU(cudaMemcpyAsync(host_out, it->second, sizeof(double) * e, cudaMemcpyDeviceToHost, ctx->st));
  CU(cudaStreamSynchronize(ctx->st));
  return CPD_OK;
}

// ---------------- generators and single-kernel entry points ----------------

cpd_status cpd_gen_tensor_block(double* T_dev, int N, const int64_t* shape, const int64_t* lo, const int64_t* hi,
                                int kind, const double* const* At_host, int Rt, double noise_std, uint64_t seed,
                                void* stream) {
  cpd_ctx* ctx = nullptr;
  if (!T_dev || !shape || !lo || !hi || N < 1 || N > CPD_MAX_ORDER)
    return fail(ctx, CPD_ERR_INVALID_ARG, "bad generator arguments");
  cpd::BlockGeo bg{};
  bg.N = N;
  for (int n = 0; n < N; n++) {
    if (lo[n] < 0 || hi[n] <= lo[n] || hi[n] > shape[n]) return fail(ctx, CPD_ERR_INVALID_ARG, "bad block range");
    bg.shape[n] = shape[n];
    bg.lo[n] = lo[n];
    bg.ext[n] = hi[n] - lo[n];
  }
  cudaStream_t st = (cudaStream_t)stream;
  int64_t Q = 1;
  for (int n = 0; n < N - 1; n++) Q *= bg.ext[n];
  const int64_t w = bg.ext[N - 1];
  auto cuerr = [&](cudaError_t e) {
    g_init_error = cudaGetErrorString(e);
    return CPD_ERR_CUDA;
  };
  cudaError_t e;
  if (kind == 0 && Rt > 0) {
    if (!At_host) return fail(ctx, CPD_ERR_INVALID_ARG, "kind 0 needs factors");
    // Kruskal part of the block: KRP of the block rows of modes 0..N-2 times A_N[lo:hi]^T
    std::vector<double*> Ad(N - 1, nullptr);
    double *KR = nullptr, *Bt = nullptr;
    for (int n = 0; n < N - 1; n++) {
      if ((e = cudaMalloc(&Ad[n], sizeof(double) * bg.ext[n] * Rt)) != cudaSuccess) return cuerr(e);
      if ((e = cudaMemcpy(Ad[n], At_host[n] + lo[n] * Rt, sizeof(double) * bg.ext[n] * Rt,
                          cudaMemcpyHostToDevice)) != cudaSuccess)
        return cuerr(e);
    }
    // B = A_N[lo:hi]^T  (Rt x w) so that T[q, z] = Σ_r KR[q, r] B[r, z]
    std::vector<double> bt((size_t)Rt * w);
    for (int64_t z = 0; z < w; z++)
      for (int r = 0; r < Rt; r++) bt[(size_t)r * w + z] = At_host[N - 1][(lo[N - 1] + z) * Rt + r];
    if ((e = cudaMalloc(&Bt, sizeof(double) * bt.size())) != cudaSuccess) return cuerr(e);
    if ((e = cudaMemcpy(Bt, bt.data(), sizeof(double) * bt.size(), cudaMemcpyHostToDevice)) != cudaSuccess)
      return cuerr(e);
    if ((e = cudaMalloc(&KR, sizeof(double) * Q * Rt)) != cudaSuccess) return cuerr(e);
    if ((e = cpd::launch_krp(Ad.data(), bg.ext, N - 1, Rt, KR, st)) != cudaSuccess) return cuerr(e);
    if ((e = cpd::launch_ttm(KR, Q, Rt, 1, Bt, (int)w, T_dev, 0, st)) != cudaSuccess) return cuerr(e);
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return cuerr(e);
    cudaFree(KR);
    cudaFree(Bt);
    for (auto p : Ad) cudaFree(p);
  } else if (kind == 0) {
    if ((e = cudaMemsetAsync(T_dev, 0, sizeof(double) * Q * w, st)) != cudaSuccess) return cuerr(e);
  }
  if (kind == 1 || noise_std != 0.0) {
    if ((e = cpd::launch_noise(T_dev, bg, kind, noise_std, seed, st)) != cudaSuccess) return cuerr(e);
  }
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return cuerr(e);
  return CPD_OK;
}

cpd_status cpd_gen_tensor(double* T_dev, int N, const int64_t* shape, int64_t lo, int64_t hi, int kind,
                          const double* const* At_host, int Rt, double noise_std, uint64_t seed,
                          void* stream) {
  if (!shape || N < 1 || N > CPD_MAX_ORDER) return fail(nullptr, CPD_ERR_INVALID_ARG, "bad generator arguments");
  int64_t l[CPD_MAX_ORDER], h[CPD_MAX_ORDER];
  for (int n = 0; n < N; n++) {
    l[n] = 0;
    h[n] = shape[n];
  }
  l[N - 1] = lo;
  h[N - 1] = hi;
  return cpd_gen_tensor_block(T_dev, N, shape, l, h, kind, At_host, Rt, noise_std, seed, stream);
}

cpd_status cpd_ttm(const double* T_dev, int64_t pre, int64_t K, int64_t post, const double* A_dev, int R,
                   double* out_dev, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cpd::launch_ttm(T_dev, pre, K, post, A_dev, R, out_dev, 0, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    g_init_error = cudaGetErrorString(e);
    return CPD_ERR_CUDA;
  }
  return CPD_OK;
}

cpd_status cpd_ttm_i8(const double* T_dev, int64_t pre, int64_t K, int64_t post, const double* A_dev, int R,
                      double* out_dev, int use_digits, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (K > cpd::kMaxKI8 || R < 1 || R > 256) {
    g_init_error = "cpd_ttm_i8: K or R out of range";
    return CPD_ERR_INVALID_ARG;
  }
  const size_t wsb = cpd::ttm_i8_workspace_bytes(K, R);
  void* ws = nullptr;
  double* part = nullptr;
  int* ex = nullptr;
  cudaError_t e = cudaMallocAsync(&ws, wsb, st);
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&part, sizeof(double) * cpd::kNormBlocks, st);
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&ex, sizeof(int), st);
  if (e == cudaSuccess) e = cpd::launch_absmax_exp(T_dev, pre * K * post, part, ex, st);
  uint8_t* Td = nullptr;
  cpd::DigitView dv;
  if (e == cudaSuccess && use_digits) {
    // T viewed as [pre, K, post]: innermost extent post (or K when post == 1)
    dv.w = post > 1 ? post : K;
    dv.ipad = cpd::digit_inner_pad(dv.w);
    dv.plane_stride = cpd::digit_plane_bytes(pre * K * post, dv.w);
    e = cudaMallocAsync((void**)&Td, (size_t)7 * dv.plane_stride, st);
    if (e == cudaSuccess) e = cpd::launch_slice_digits(T_dev, pre * K * post, dv.w, ex, Td, st);
    dv.planes = Td;
  }
  if (e == cudaSuccess)
    e = cpd::launch_ttm_i8(T_dev, pre, K, post, A_dev, R, out_dev, 0, ex, ws, wsb, st, Td ? &dv : nullptr);
  if (Td) cudaFreeAsync(Td, st);
  if (ws) cudaFreeAsync(ws, st);
  if (part) cudaFreeAsync(part, st);
  if (ex) cudaFreeAsync(ex, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    g_init_error = cudaGetErrorString(e);
    return CPD_ERR_CUDA;
  }
  return CPD_OK;
}

// debug: T's digit planes (7 x digit_plane_bytes(n, w) bytes) into out_dev (device)
cpd_status cpd_debug_slice_digits(const double* T_dev, int64_t n, int64_t w, uint8_t* out_dev, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  double* part = nullptr;
  int* ex = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&part, sizeof(double) * cpd::kNormBlocks, st);
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&ex, sizeof(int), st);
  if (e == cudaSuccess) e = cpd::launch_absmax_exp(T_dev, n, part, ex, st);
  if (e == cudaSuccess) e = cpd::launch_slice_digits(T_dev, n, w, ex, out_dev, st);
  if (part) cudaFreeAsync(part, st);
  if (ex) cudaFreeAsync(ex, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    g_init_error = cudaGetErrorString(e);
    return CPD_ERR_CUDA;
  }
  return CPD_OK;
}

cpd_status cpd_mttv(const double* X_dev, int64_t pre, int64_t K, int64_t post, int R, const double* v_dev,
                    double* out_dev, int beta, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  double* ws = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&ws, sizeof(double) * kMttvWs, st);
  if (e == cudaSuccess) e = cpd::launch_mttv(X_dev, pre, K, post, R, v_dev, out_dev, beta, ws, kMttvWs, st);
  if (ws) cudaFreeAsync(ws, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    g_init_error = cudaGetErrorString(e);
    return CPD_ERR_CUDA;
  }
  return CPD_OK;
}

}  // extern "C"
