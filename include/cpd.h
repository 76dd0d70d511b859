/*
 * cpd.h -- C ABI of libcpd.so: the B200 hot path of MSDT / pairwise-perturbation
 * CP-ALS (Ma & Solomonik, arXiv 2010.12056).
 *
 * Citations: "P:n" = PAPER.md line n (section / equation / algorithm named beside it).
 *
 * Problem statement (Alg. 1; Alg. 2): an order-N dense tensor
 * T in R^{s_1 x ... x s_N}, a CP rank R, factor matrices A^(n) in R^{s_n x R}; CP-ALS
 * updates each A^(n) from the normal equations A^(n) Γ^(n) = M^(n), with
 * the MTTKRP M^(n) computed by the multi-sweep dimension tree (MSDT, §III),
 * by the standard dimension tree (DT), or approximated by pairwise
 * perturbation (PP, §II-C Eqs. 4-8, Alg. 2).
 *
 * Conventions (apply to every entry point):
 *  - Modes are 0-based in the ABI (the paper's are 1-based).
 *  - Layout: T is row-major (last mode fastest), float64.  Factor matrices are s_n x R
 *    row-major float64 (R fastest).  Intermediates live on the device in the layout
 *    [kept modes ascending ..., R] (R innermost).
 *  - Multi-GPU (Alg. 3, Alg. 4) on a processor grid I_1 x .. x I_N
 *    (cpd_opts.grid; default the 1-D grid 1x..x1xP).  Rank r has grid coordinates
 *    (x_1..x_N), r = row-major index (last mode fastest), and holds the block
 *    T[x_1 b_1 : (x_1+1) b_1, ..., x_N b_N : (x_N+1) b_N], b_n = s_n / I_n, row-major and
 *    contiguous (1-D default: the slab T[..., p*s_N/P : (p+1)*s_N/P]).  s_n % I_n == 0 and
 *    b_n % (P / I_n) == 0 (reading Q20: no padding).  With world > 1 every call is
 *    collective: all ranks make the same sequence of calls.  The library owns its NCCL
 *    communicators (the world and, per mode, Proc-Slice(x_n) and the fibre of x_n, split
 *    with ncclCommSplit).
 *  - Ownership: T is BORROWED (device pointer, read-only, must outlive the ctx).
 *    Factors are copied in.  Outputs are copied into caller buffers.  All device
 *    workspaces (tree intermediates, PP operators) belong to the ctx and are freed by
 *    cpd_destroy.
 *  - Blocking: every call returns after its stream work has completed; scalars written
 *    to *_out are host values.
 *  - Errors: every function returns cpd_status; nothing throws across the ABI and
 *    nothing exits.  After CPD_ERR_CUDA or CPD_ERR_NCCL the ctx is poisoned and only
 *    cpd_destroy is valid.  cpd_last_error() gives a message.  There is no CPU fallback:
 *    without a usable sm_100 device cp_als_init fails with CPD_ERR_CUDA.
 */
#ifndef CPD_H
#define CPD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct cpd_ctx cpd_ctx; /* opaque; owns all device state */

typedef enum {
  CPD_OK = 0,
  CPD_ERR_INVALID_ARG = 1, /* bad shape/rank/ε/mode index, s_N % world != 0, R > CPD_MAX_RANK */
  CPD_ERR_STATE = 2,       /* e.g. pp_approx_sweep without a valid pp_init */
  CPD_ERR_NUMERIC = 3,     /* Γ not SPD (Cholesky failed), non-finite values */
  CPD_ERR_CUDA = 4,        /* CUDA runtime error (ctx poisoned) */
  CPD_ERR_NCCL = 5,        /* NCCL error (ctx poisoned) */
  CPD_ERR_OOM = 6,         /* device allocation failed */
  CPD_ERR_INTERNAL = 7     /* scheduler invariant violated (stale intermediate) */
} cpd_status;

#define CPD_MAX_ORDER 8
#define CPD_MAX_RANK 1024     /* R <= 128: fused update with Γ^-1 (one CTA); R <= 232: packed Cholesky in one
                                 CTA's shared memory + row solves; beyond: Γ^-1 by a grid-wide blocked
                                 Gauss-Jordan and x = M Γ^-1 as a DMMA GEMM */
#define CPD_NCCL_ID_BYTES 128

typedef struct {
  uint32_t struct_size;       /* = sizeof(cpd_opts); ABI versioning */
  int device;                 /* CUDA device ordinal used by this ctx */
  int rank, world;            /* this rank and the number of ranks (= prod(grid)) */
  const void* nccl_unique_id; /* CPD_NCCL_ID_BYTES bytes from cpd_nccl_unique_id on rank 0,
                                 broadcast by the caller; NULL iff world == 1 */
  void* stream;               /* caller's cudaStream_t (NULL = the legacy default stream).  The library
                                 runs on streams it owns (its main stream one priority level above the
                                 default; a highest-priority side stream for Γ^-1 / W; a lowest-priority
                                 filler stream for PP operator streams); every call is ordered after the
                                 work already enqueued on `stream` and `stream` after the call's work */
  double pp_eps;              /* ε in (0,1) for still_valid / cpd_pp_condition (Alg. 2 line 5) */
  int reuse_root_in_pp_init;  /* P:384 footnote: reuse a still-valid MSDT root in pp_init (default 1) */
  int profile_phases;         /* CUDA-event timers: 0 off; 1 TTM and mTTV launches only (the roofline
                                 kernels, low overhead); 2 every phase (TTM, mTTV, solve, hadamard,
                                 other; the P:748 breakdown) */
  void* local_group;          /* NULL: NCCL (one process per GPU).  Else a cpd_local_group of `world`
                                 ranks in ONE process on ONE device, each rank's calls made from its own
                                 host thread (verification of the 1-D partition on a single GPU) */
  int ttm_impl;               /* first-level TTM engine (DESIGN.md §6 K2 / K2i):
                                 CPD_TTM_DMMA (0) = FP64 tensor cores (mma.sync .f64, DMMA);
                                 CPD_TTM_INT8 (1) = FP64 operands as 54-bit fixed point split into 7
                                   int8 digits, exact int8 x int8 -> int32 products on the tcgen05
                                   tensor cores (cpd_ttm_i8); T's digits are computed once at init
                                   (7 extra bytes per element when memory allows);
                                 CPD_TTM_AUTO (2, default) = INT8 when max|T| <= 256 rms(T), i.e. when
                                   its norm-wise error bound 2^-55 max|T|/rms(T) is FP64-class, else DMMA.
                                 Modes with s_j > 16384 always use DMMA. */
  int grid[CPD_MAX_ORDER];    /* processor grid I_1..I_N (Alg. 3 line 1); all 0 = the 1-D default
                                 1 x .. x 1 x world; entries beyond N must be 0 */
  int fused_rs;               /* 0 (default): the partial MTTKRP of each mode is reduce-scattered in
                                 Proc-Slice(x_n) by a collective (ncclReduceScatter).  1: fused epilogue
                                 (SURVEY f2): the kernel that completes the local partial M^(n) / M~^(n)
                                 stores each owner's rows straight into that owner's receive buffer
                                 (NCCL: a symmetric window from ncclMemAlloc + ncclCommWindowRegister,
                                 addressed through ncclGetPeerPointer over NVLink; local group: the
                                 same device), then a stream-ordered barrier and a fixed-order sum of
                                 the received slots.  Needs <= 8 ranks per slice. */
  int msdt_levels;            /* upper-level fusion: l in [1, N-2] (0 = 1).  Each MSDT
                                 root contracts a cyclic block of l modes of T at once (one pass over T with
                                 the Khatri-Rao product of their factors) and serves the next N-l updates, so
                                 the largest tree node holds s^(N-l) R instead of s^(N-1) R elements, for N/(N-l)
                                 instead of N/(N-1) passes over T per sweep.  l = 1 is the paper's MSDT.  Affects
                                 msdt_sweep only (DT and pp_init keep first-level TTMs). */
} cpd_opts;

#define CPD_TTM_DMMA 0
#define CPD_TTM_INT8 1
#define CPD_TTM_AUTO 2
/* engine a ctx uses (cpd_ttm_engine) */
#define CPD_ENGINE_DMMA 0
#define CPD_ENGINE_INT8_DIGITS 1   /* T's digit planes streamed by TMA */
#define CPD_ENGINE_INT8_CONVERT 2  /* T converted to digits inside each TTM (no memory for the planes) */

typedef struct cpd_local_group cpd_local_group;
/* In-process group for `world` (1..8) ranks sharing one device (see cpd_opts.local_group):
 * collectives become fixed-order device sums over the ranks' buffers.  Destroy after every
 * ctx that uses it. */
cpd_status cpd_local_group_create(int world, cpd_local_group** out);
cpd_status cpd_local_group_destroy(cpd_local_group* g);

/* Fill *o with defaults: device 0, rank 0, world 1, no NCCL id, default caller stream,
 * pp_eps 0.1, reuse_root_in_pp_init 1, profile_phases 0, ttm_impl CPD_TTM_AUTO. */
cpd_status cpd_opts_default(cpd_opts* o);

/* NCCL unique id for a multi-GPU ctx (call on rank 0, broadcast the 128 bytes). */
cpd_status cpd_nccl_unique_id(void* out /* CPD_NCCL_ID_BYTES */);

/* Create a ctx (Alg. 1 line 2 / Alg. 3 lines 4-9).
 *  N: order, 3 <= N <= CPD_MAX_ORDER.  shape: global s_1..s_N (each >= 1).
 *  R: rank, 1 <= R <= CPD_MAX_RANK.
 *  T_local_dev: BORROWED device pointer to this rank's row-major block
 *    [s_1/I_1, ..., s_N/I_N] (float64, read-only; 1-D default [s_1, ..., s_{N-1}, s_N/world]).
 *  A0_host: N host pointers, each the GLOBAL s_n x R row-major initial factor (copied).
 *  Computes ||T||^2 once (all-reduced), S^(n) = A^(n)T A^(n), MSDT phase 0.
 */
cpd_status cp_als_init(cpd_ctx** out, int N, const int64_t* shape, int R,
                       const double* T_local_dev, const double* const* A0_host,
                       const cpd_opts* opts);

/* One exact CP-ALS sweep, modes 0..N-1 (Alg. 1 lines 5-9), MTTKRPs from the
 * multi-sweep dimension tree (§III, Fig. 2): first-level TTM roots T x_j A^(j) for
 * j = N-1, N-2, ..., 0 cyclically, each serving the N-1 following updates; lower
 * levels by batched TTV.  Any factor change not made by msdt_sweep
 * restarts the cycle.  Sets dA^(n) = the one-sweep update (Alg. 2 line 18).
 * *fitness_out = 1 - r with r from Eq. 3 (reading Q1: ||T||^2). */
cpd_status msdt_sweep(cpd_ctx* ctx, double* fitness_out);

/* One exact sweep with the standard binary dimension tree (Fig. 1a):
 * root T x_{N} serves modes 1..ceil(N/2), root T x_1 serves the rest. */
cpd_status dt_sweep(cpd_ctx* ctx, double* fitness_out);

/* PP initialisation (Alg. 2 lines 6-9; Alg. 4 line 2, no communication):
 * A_p <- A, dA <- 0, pair operators M_p^(a,b) (Eq. 4 with A_p) for all a<b
 * stored as [s_a, s_b, R] (mode N local), and M_p^(n). */
cpd_status pp_init(cpd_ctx* ctx);

/* One PP approximated sweep (Alg. 2 lines 11-16; Eqs. 5-8; Alg. 4 lines
 * 4-16): M~^(n) = M_p^(n) + Σ_i U^(n,i) + V^(n), solve, dA^(n) = A^(n) - A_p^(n).
 * *still_valid = [∀i ||dA^(i)||_F < ε ||A^(i)||_F] after the sweep (Alg. 2 line 10).
 * The library never refuses a sweep because of ε (the driver may force a schedule).
 * Returns CPD_ERR_STATE without a valid pp_init. */
cpd_status pp_approx_sweep(cpd_ctx* ctx, double* fitness_out, int* still_valid);

/* f = 1 - r of the last completed sweep (Eq. 3). CPD_ERR_STATE before any sweep. */
cpd_status fitness(cpd_ctx* ctx, double* f_out);

/* ∀i ||dA^(i)||_F < ε ||A^(i)||_F for the current dA regime (Alg. 2 line 5). */
cpd_status cpd_pp_condition(cpd_ctx* ctx, int* ok);

/* Copy the GLOBAL factor A^(n0) (s_n x R row-major) to host (gathers mode N-1 rows). */
cpd_status cpd_get_factor(cpd_ctx* ctx, int n0, double* host_out);

/* Copy the M^(n0) (or M~^(n0)) used in the last update of mode n0 to host: the
 * GLOBAL s_n x R matrix (after reduction over ranks / gathered for the last mode). */
cpd_status cpd_get_last_mttkrp(cpd_ctx* ctx, int n0, double* host_out);

/* Replace all factors (N host pointers, global s_n x R); recomputes S; invalidates
 * the MSDT root and the PP state. */
cpd_status cpd_set_factors(cpd_ctx* ctx, const double* const* A_host);

/* Accumulated device time per phase since init (requires opts.profile_phases):
 * out[0]=TTM, out[1]=mTTV (incl. PP U-stream), out[2]=solve, out[3]=hadamard/Gram,
 * out[4]=other (P:748 categories). */
cpd_status cpd_get_phase_ms(cpd_ctx* ctx, double out[5]);

/* Algorithmic-work ledger since init: out[0]=TTM flops (2*rows*K*R per launch),
 * out[1]=TTM launches, out[2]=mTTV/PP-stream bytes (8*(elements read+written)) of the launches on
 * the library's main stream (the ones the mTTV timer brackets; see cpd_get_filler_counters for the
 * overlapped PP filler-stream launches), out[3]=those launches, out[4]=first-level TTMs (roots)
 * built, out[5]=kernels launched by libcpd.so in this process (all kernels, monotone; not reset). */
cpd_status cpd_get_counters(cpd_ctx* ctx, double out[6]);

/* Algorithmic HBM bytes of the first-level TTMs and block contractions since init or the last
 * cpd_reset_counters (the roofline numerator of the TTM, DESIGN.md §6/§9): per launch, T read once (7 B per
 * element on the digit planes, 8 B as FP64), the FP64 output written once, the factor (or the block's
 * Khatri-Rao product) read.  Divide by cpd_get_counters' out[1] for bytes per launch. */
cpd_status cpd_get_ttm_bytes(cpd_ctx* ctx, double* out);

/* Auxiliary-memory ledger (Table 1's aux-memory column; the upper-level-fusion trade-off,
 * P:700-702): out[0] = high-water mark of the library's intermediate device buffers (dimension-tree
 * nodes, PP operators, block Khatri-Rao products) since init or the last cpd_reset_counters, in bytes;
 * out[1] = bytes live now; out[2] = bytes of T's int8 digit planes (0 unless the digit engine is used). */
cpd_status cpd_get_memory(cpd_ctx* ctx, double out[3]);

/* Ledger of the PP operator streams (Eq. 6) issued on the low-priority filler stream (the ones whose
 * dA is already final, and the next sweep's speculative ones): out[0] = bytes (8*(elements read +
 * written)), out[1] = launches.  These overlap the main stream and are NOT in cpd_get_counters'
 * out[2..3], which (with the mTTV timer of cpd_get_phase_ms) cover the main-stream launches only. */
cpd_status cpd_get_filler_counters(cpd_ctx* ctx, double out[2]);

/* Change the timer level of opts.profile_phases (0, 1, 2) between calls. */
cpd_status cpd_set_profile_level(cpd_ctx* ctx, int level);

/* Zero the phase timers and counters. */
cpd_status cpd_reset_counters(cpd_ctx* ctx);

/* M_p^(a0,b0) as [s_a/I_a, s_b/I_b, R], the local (block-partial) operator (a0 < b0):
 * checks pp_init directly against the oracle's operators (small configs). */
cpd_status cpd_debug_get_pp_operator(cpd_ctx* ctx, int a0, int b0, double* host_out);

/* Message for the last error on ctx (ctx may be NULL: thread-local init error). */
const char* cpd_last_error(const cpd_ctx* ctx);

/* Free everything owned by ctx (valid on a poisoned ctx; NULL is a no-op). */
cpd_status cpd_destroy(cpd_ctx* ctx);

/* ---- input generation and single-kernel entry points (bench / tests) ---------------- */

/* Write this rank's slab of the synthetic tensor (synth/__init__.py recipe):
 *   kind 0: T(i) = Σ_r Π_n At^(n)(i_n, r) + noise_std * normal(seed, i)
 *   kind 1: T(i) = uniform(seed, i)
 * i = GLOBAL row-major linear index; normal/uniform from the SplitMix64 counter hash.
 * shape: global; slab [lo, hi) of the last mode; At_host: N host arrays s_n x Rt
 * (ignored for kind 1).  Writes (hi-lo)*Π_{n<N-1} s_n doubles at T_dev. */
cpd_status cpd_gen_tensor(double* T_dev, int N, const int64_t* shape, int64_t lo, int64_t hi,
                          int kind, const double* const* At_host, int Rt, double noise_std,
                          uint64_t seed, void* stream);

/* The block [lo_n, hi_n) per mode of the same synthetic tensor (N-D processor grid): T_dev
 * receives Π (hi_n - lo_n) doubles, row-major; element values depend only on the global index. */
cpd_status cpd_gen_tensor_block(double* T_dev, int N, const int64_t* shape, const int64_t* lo,
                                const int64_t* hi, int kind, const double* const* At_host, int Rt,
                                double noise_std, uint64_t seed, void* stream);

/* First-level TTM: out[p, m, r] = Σ_y T[p, y, m] A[y, r] with T viewed as
 * [pre, K, post]; out is [pre*post, R] row-major.  All device pointers; synchronous. */
cpd_status cpd_ttm(const double* T_dev, int64_t pre, int64_t K, int64_t post,
                   const double* A_dev, int R, double* out_dev, void* stream);

/* The contents of the borrowed T changed (same pointer and shape, e.g. a new tensor uploaded
 * into the same buffer): recompute ||T||^2, the TTM engine's exponent and digit
 * planes, and drop every cached tree node and PP operator (the MSDT cycle restarts; the
 * next sweep is a regular one).  Collective when world > 1. */
cpd_status cpd_set_tensor(cpd_ctx* ctx);

/* Status of the last completed sweep's fitness (Eq. 3): *flags bit 0 is set when the
 * radicand ||T||^2 + <Γ^(N),S^(N)> - 2<M^(N),A^(N)> fell below -1e-8 ||T||^2 -- not rounding:
 * M (an approximated M~) and A are inconsistent, as after a PP sweep forced outside the ε regime
 * (Alg. 2 line 10), and the reported fitness is the clamped value 1.  *radicand_rel (may be NULL)
 * = radicand / ||T||^2.  Host values, no device work. */
cpd_status cpd_last_sweep_status(const cpd_ctx* ctx, int* flags, double* radicand_rel);

/* *engine = the first-level TTM engine this ctx chose at init (CPD_ENGINE_*). */
cpd_status cpd_ttm_engine(const cpd_ctx* ctx, int* engine);

/* The same first-level TTM on the INT8 tensor cores (tcgen05.mma kind::i8): both FP64 operands
 * are converted to 54-bit fixed point (one exponent for T = ceil(log2 max|T|), one per column of
 * A) and split into 7 signed 8-bit digits; the 28 most significant digit-pair products are
 * exact int32 tensor-core sums, recombined in FP64 (DESIGN.md §6 K2i).  Norm-wise error of
 * the order of FP64 rounding relative to max|T|·|A|.  K <= 16384, 1 <= R <= 256; otherwise
 * CPD_ERR_INVALID_ARG.  use_digits != 0: T's digit planes are sliced first (7 bytes per
 * element, as cp_als_init does once) and streamed by TMA where the layout allows it; 0: T is
 * converted inside the TTM.  Synchronous; allocates its workspace on `stream`. */
cpd_status cpd_ttm_i8(const double* T_dev, int64_t pre, int64_t K, int64_t post,
                      const double* A_dev, int R, double* out_dev, int use_digits, void* stream);

/* Batched TTV: out[p, c] = beta*out[p, c] + Σ_y X[p, y, c] v[y, c % R],
 * X viewed as [pre, K, C] with C = post*R; beta in {0, 1}.  Synchronous. */
cpd_status cpd_mttv(const double* X_dev, int64_t pre, int64_t K, int64_t post, int R,
                    const double* v_dev, double* out_dev, int beta, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* CPD_H */
