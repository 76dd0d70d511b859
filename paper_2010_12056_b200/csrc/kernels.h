// Internal launchers of libcpd.so (sm_100a).  Citations: P:n = PAPER.md line n.
#pragma once
#include <cstdlib>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>

namespace cpd {

// number of kernels libcpd.so has launched (all launchers add to it)
extern std::atomic<long long> g_launches;

// ---- first-level TTM on FP64 tensor cores (DMMA, mma.sync .f64), P:320-322 ----------
// out[i, n] = beta*out[i, n] + Σ_y X[addr(i, y)] * B[y, n],   i < pre*post, n < ncols
// addr(i, y) = (i / post) * K * post + (i % post) + y * post   (X viewed as [pre, K, post])
// B is K x ncols row-major (ld = ncols); out is (pre*post) x ncols row-major.
cudaError_t launch_ttm(const double* X, int64_t pre, int64_t K, int64_t post, const double* B,
                       int ncols, double* out, int beta, cudaStream_t st);

// ---- the same first-level TTM on the INT8 tensor cores (tcgen05 kind::i8, exact integer
// slicing of both FP64 operands; ttm_i8.cu).  Xexp: device int with 2^Xexp > max|X|
// (launch_absmax_exp); ws: ttm_i8_workspace_bytes(min(K, kMaxKI8), ncols) bytes (sliced B + exponents).
// K <= kMaxKI8 (int32 accumulators) per launch: longer K only on the digit planes, as chunks accumulated
// with beta = 1; ncols <= 1024.
constexpr int64_t kMaxKI8 = 16384;
size_t ttm_i8_workspace_bytes(int64_t K, int ncols);
// X's 7 int8 digit planes (launch_slice_digits): X viewed as [n / w, w] (w = innermost extent),
// plane a of element (row, c) at planes[a * plane_stride + row * ipad + c], ipad = digit_inner_pad(w)
struct DigitView {
  const uint8_t* planes = nullptr;
  int64_t w = 0, ipad = 0, plane_stride = 0;
};
inline int64_t digit_inner_pad(int64_t w) {
  static const int64_t pad = getenv("CPD_DIGIT_PAD") ? atoi(getenv("CPD_DIGIT_PAD")) : 16;  // 16 | 32 | 64 | 128
  return (w + pad - 1) / pad * pad;
}
// dv (may be null): when its layout serves this TTM view, the TTM streams the digit planes
// instead of converting X
cudaError_t launch_ttm_i8(const double* X, int64_t pre, int64_t K, int64_t post, const double* B, int ncols,
                          double* out, int beta, const int* Xexp, void* ws, size_t ws_bytes, cudaStream_t st,
                          const DigitView* dv = nullptr);
// Contraction of T with a Khatri-Rao product over a block of modes (upper-level fusion) on the
// digit planes, as ONE GEMM whose K index is (slab p, q): the digit view is [P][Mrows][Qp] (Qp bytes per row,
// a multiple of 16: the flattened, innermost-padded suffix of the block; P = the flattened prefix of a
// block that wraps around from mode N to mode 1, else 1), Bpad is [P][32*ceil(Qp/32)][ncols] with zero
// rows at pad positions (launch_krp_block).  out (Mrows x ncols) = beta*out + Σ_{p,q} digits(p,i,q) Bpad.
// Launches of <= kMaxKI8 K rows accumulate with beta = 1.  cudaErrorNotSupported: layout not served.
// ws: ttm_i8_workspace_bytes(kMaxKI8, ncols) bytes.
cudaError_t launch_ttm_i8_block(int64_t P, int64_t Mrows, int64_t Qp, const double* Bpad, int ncols, double* out,
                                int beta, const int* Xexp, void* ws, size_t ws_bytes, cudaStream_t st,
                                const DigitView& dv);
// Khatri-Rao product of the factors of a block of modes, scattered into a zero-padded row layout:
// out[(Σ_c y_c stride_c) * R + r] = Π_c A_c[y_c * R + r] for y_c < ext_c (the first mode slowest in the
// enumeration; the row strides place it).  rows_total: rows of out (zeroed first when `pad`).
struct KrpSpec {
  int n;
  const double* A[8];
  int64_t ext[8], stride[8];
};
cudaError_t launch_krp_block(const KrpSpec& sp, int R, double* out, int64_t rows_total, bool pad, cudaStream_t st);
// bytes between digit planes (a multiple of 64); the planes buffer holds 7 * digit_plane_bytes(n, w)
inline int64_t digit_plane_stride(int64_t n) { return (n + 63) / 64 * 64; }
inline int64_t digit_plane_bytes(int64_t n, int64_t w) { return digit_plane_stride(n / w * digit_inner_pad(w)); }
cudaError_t launch_slice_digits(const double* X, int64_t n, int64_t w, const int* Xexp, uint8_t* planes,
                                cudaStream_t st);
// *e_out = e with 2^e > max|x_i| (0 if x == 0), *max_out = max|x_i| if given; partial: kNormBlocks doubles
cudaError_t launch_absmax_exp(const double* x, int64_t n, double* partial, int* e_out, cudaStream_t st,
                              double* max_out = nullptr);

// ---- batched TTV (mTTV) stream, P:320-322 ----------------------------------------------
// out[p, c] = beta*out[p, c] + Σ_y X[(p*K + y)*C + c] * v[y*R + c % R],  C = post*R
// ws (ws_elems doubles, may be null): K-split partials when the (p, chunk) grid is too small
cudaError_t launch_mttv(const double* X, int64_t pre, int64_t K, int64_t post, int R,
                        const double* v, double* out, int beta, double* ws, int64_t ws_elems,
                        cudaStream_t st);

// Several contractions with the same output shape summed into one output (the N-1
// U-streams of a PP mode, Eq. 6): out = base + Σ_jobs contraction_j (base may be null:
// then out = beta*out + Σ).  One launch plus one fixed-order reduce.
struct MttvSpec {
  const double* X;
  const double* v;
  int64_t pre, K, post;
};
// Fused reduce-scatter epilogue (Alg. 3 line 14, Alg. 4 line 9): the final value of
// output element e (the local partial MTTKRP, read-modify-write of `out` when beta = 1) is
// stored at dst[e / chunk] + e % chunk instead of out + e -- this rank's slot in the receive
// buffer of the owner of those rows (a peer's memory over NVLink, or the same device for the
// local group).  nq == 0: plain output.
struct OutMap {
  double* dst[8];
  int64_t chunk;
  int nq;
};
// The K-split partials of an mTTV launch whose fixed-order reduction (mttv_reduce_kernel's arithmetic:
// out[e] = (base ? base[e] : beta ? out[e] : 0) + Σ_k ws[k n + e], k ascending) is left to the kernel that
// consumes out -- the fused factor update on the PP critical chain (one launch fewer per mode).  slots = 0:
// nothing pending (out is final).
struct MPending {
  const double* ws = nullptr;
  int slots = 0;
  int64_t n = 0;
  const double* base = nullptr;
  int beta = 0;
};
// occ3: at most 3 resident CTAs per SM (for launches that overlap latency-critical kernels)
// defer (may be null): a K-split launch without OutMap leaves its reduction to the consumer (*defer)
cudaError_t launch_mttv_multi(const MttvSpec* specs, int J, int R, const double* base, double* out, int beta,
                              double* ws, int64_t ws_elems, cudaStream_t st, const OutMap* map = nullptr,
                              bool occ3 = false, int waves_override = 0, MPending* defer = nullptr);
// Two single-mode contractions of one node in one read (PP-init multi-output descent):
// X viewed as [P][K1][Q][K2][C] (C = trailing extents x R), out1 = contract K1 -> [P][Q][K2][C],
// out2 = contract K2 -> [P][K1][Q][C]; ws: ceil(K1/32) x |out1| doubles of partials when K1 > 32.
cudaError_t launch_mttv_dual(const double* X, int64_t P, int64_t K1, int64_t Q, int64_t K2, int64_t C, int R,
                             const double* v1, const double* v2, double* out1, double* out2, double* ws,
                             int64_t ws_elems, cudaStream_t st);
// dst[e] = Σ_{q < nq} src[q * n + e], q in fixed order (the owner's sum of the received slots)
cudaError_t launch_slot_sum(const double* src, int nq, int64_t n, double* dst, cudaStream_t st);

// ---- synthetic tensor (synth/__init__.py recipe) ------------------------------------
// T[q, z] += std*normal(seed, g) (kind 0) or T = uniform(seed, g) (kind 1) with
// g = q*sN + lo + z the global index, T viewed as [Q, w] (w = hi - lo).
struct BlockGeo {  // a block of a row-major tensor: global shape, first index and extent per mode
  int N;
  int64_t shape[8], lo[8], ext[8];
};
cudaError_t launch_noise(double* T, const BlockGeo& b, int kind, double stdv, uint64_t seed, cudaStream_t st);
// KR[q, r] = Π_{n<N-1} A_n[i_n(q), r]  (Khatri-Rao rows, first mode slowest)
cudaError_t launch_krp(const double* const* A_dev, const int64_t* shape, int nf, int R,
                       double* KR, cudaStream_t st);

// ---- reductions ---------------------------------------------------------------------------
// dst[0] = Σ x_i^2 over n elements (deterministic two-pass; partial needs kNormBlocks doubles)
constexpr int kNormBlocks = 148 * 4;
cudaError_t launch_norm2(const double* x, int64_t n, double* partial, double* dst, cudaStream_t st);
// dst[0] = Σ x_i y_i (single CTA, fixed order) for small arrays; y == nullptr -> Σ x_i^2
cudaError_t launch_dot(const double* x, const double* y, int64_t n, double* dst, cudaStream_t st);

// ---- small dense R x R work (latency-bound) -----------------------------------------------
// G1[a][b] = Σ_i X[i][a] Y1[i][b] (S = A^T A) and, if Y2, G2 = X^T Y2 (dS = A^T dA,
// Eq. 8) in the same pass; rows split over up to 16 CTAs (ws: 2*16*R*R doubles),
// partials summed in a fixed order.
cudaError_t launch_gram(const double* X, const double* Y1, const double* Y2, int64_t rows, int R,
                        double* G1, double* G2, double* ws, int64_t ws_elems, cudaStream_t st);
// Γ^(n) = ∗_{k≠n} S^(k) (Eq. 1) and its Cholesky factor, packed column-major lower, into
// Lp (R(R+1)/2, then the R reciprocal diagonal entries).  status[0] = 0 ok, 1 not SPD.
cudaError_t launch_gamma_chol(const double* S_all, int N, int n, int R, double* Lp, int* status,
                              cudaStream_t st);
// Γ^(n) (Eq. 1) and Ginv = Γ^{-1} (dense R x R) by Gauss-Jordan without pivoting (SPD);
// status[0] = 1 if a pivot is not positive (Γ not SPD).  One CTA, R^2 doubles of shared memory.
// W (optional): also the PP second-order sum W^(n) of Eq. 7 (as launch_pp_w) from S_all, dS_all.
// R beyond one CTA's shared memory: the blocked Gauss-Jordan over a cooperative grid with Γ in
// global memory; ws holds gamma_inverse_big_ws(R) doubles
size_t gamma_inverse_big_ws(int R);
cudaError_t launch_gamma_inverse_big(const double* S_all, int N, int n, int R, double* ws, double* Ginv,
                                     int* status, cudaStream_t st);
cudaError_t launch_gamma_inverse(const double* S_all, int N, int n, int R, double* Ginv, int* status,
                                 cudaStream_t st, const double* dS_all = nullptr, double* W = nullptr);
// Ginv = Γ^{-1} = L^{-T} L^{-1} (dense R x R, exactly symmetric) from the packed factor; one CTA,
// R(R+1)/2 + R + R^2 doubles of shared memory (R <= kUpdMaxR)
cudaError_t launch_chol_inverse(const double* Lp, int R, double* Ginv, cudaStream_t st);
// X[i,:] = M[i,:] Γ^{-1} via L (forward + backward substitution per row), rows x R.
cudaError_t launch_trisolve(const double* Lp, const double* M, int64_t rows, int R, double* X,
                            cudaStream_t st);
// W = Σ_{i<j; i,j≠n} dS_i ∗ dS_j ∗ ∗_{k∉{i,j,n}} S_k (Eq. 7)
cudaError_t launch_pp_w(const double* S_all, const double* dS_all, int N, int n, int R, double* W,
                        cudaStream_t st);
// z = x - y (n elements)
cudaError_t launch_sub(const double* x, const double* y, double* z, int64_t n, cudaStream_t st);
// dA = A - base; *o_dA2 = Σ dA^2, *o_A2 = Σ A^2, *o_MA = Σ M A (if M); one launch, last-block
// fixed-order reduction (part: 3*64 doubles, counter: zero-initialised, self-resetting)
cudaError_t launch_update_stats(const double* A, const double* base, double* dA, const double* M, int64_t n,
                                double* part, unsigned int* counter, double* o_dA2, double* o_A2, double* o_MA,
                                cudaStream_t st);

// ---- fused factor update (update.cu): V term (PP), row solve, dA, statistics, S and dS ----
// Cooperative launch (grid sync between the row solves and the Gram reduction); the solve is
// x = y Ginv with Ginv = Γ^{-1} from launch_chol_inverse ("A = M Γ†").  A holds the
// old rows on entry (read as a_old for V and, if base == nullptr, as the dA base) and the new
// rows on exit.  W (PP) may be null (else M += A_old W is written back); dS may be null;
// S == nullptr skips the Gram phase.
// R <= kUpdMaxR.
constexpr int kUpdMaxR = 128;  // Γ^{-1} + the packed factor fit one CTA's shared memory
constexpr int kUpdMaxBlocks = 148;
// part: 3 * kUpdMaxBlocks doubles; gpart: kUpdMaxBlocks * 2 * R * R doubles (per-CTA Gram partials).
// st_src/st_dst (optional): *st_dst = *st_src at kernel start (status hand-over between streams).
// S_all (R <= 32): Γ^{-1} (and W from S_all, dS_all when W != null -- W then only selects PP) are
// formed inside the launch from the Grams of mode != nmode; SPD verdict to *st_local.
size_t update_fused_smem(int R, bool pp, int RB);
int update_fused_blocks(int64_t rows);
cudaError_t launch_update_fused(int R, int64_t rows, const double* Ginv, const double* W, double* M, double* A,
                                const double* base, double* dA, double* S, double* dS, double* part, double* gpart,
                                double* o_dA2, double* o_A2, double* o_MA, const int* st_src, int* st_dst,
                                cudaStream_t st, const double* S_all = nullptr, const double* dS_all = nullptr,
                                int N = 0, int nmode = 0, int* st_local = nullptr, const MPending* pend = nullptr);

}  // namespace cpd
