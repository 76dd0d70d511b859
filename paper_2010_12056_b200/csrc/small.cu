// Small dense R x R work of each factor update (latency-bound; "the cost of
// solving linear systems is often small"): Gram matrices, dS (Eq. 8), the
// Hadamard chain Γ^(n) (Eq. 1) with its Cholesky factorisation, the row-wise normal-
// equation solve A^(n) = M^(n) Γ^(n)^{-1} (Alg. 1 line 7; reading Q3: Cholesky),
// the PP second-order Hadamard sum W^(n) of Eq. 7, and the per-update
// statistics (dA = A - base, ||dA||^2, ||A||^2, <M, A>) for Alg. 2 line 5 and Eq. 3.
// All reductions run in a fixed order (deterministic; no floating-point atomics).
#include <cooperative_groups.h>

#include "kernels.h"

#define CPD_MAXR 232

namespace cpd {
namespace {

// ---------------- Gram: G1 = X^T Y1 (and G2 = X^T Y2), row-split partials ----------------
constexpr int GT = 16;   // output tile
constexpr int GK = 32;   // rows per smem chunk
__global__ void __launch_bounds__(GT* GT)
    gram_partial_kernel(const double* __restrict__ X, const double* __restrict__ Y1,
                        const double* __restrict__ Y2, int64_t rows, int R, int64_t rows_per_split,
                        double* __restrict__ P1, double* __restrict__ P2) {
  __shared__ double xs[GK][GT + 1], y1s[GK][GT + 1], y2s[GK][GT + 1];
  const int tx = threadIdx.x % GT, ty = threadIdx.x / GT;
  const int a0 = blockIdx.y * GT, b0 = blockIdx.x * GT;
  const int64_t r0 = (int64_t)blockIdx.z * rows_per_split;
  const int64_t r1 = min(rows, r0 + rows_per_split);
  const bool two = Y2 != nullptr;
  double s1 = 0.0, s2 = 0.0;
  for (int64_t i0 = r0; i0 < r1; i0 += GK) {
    for (int e = threadIdx.x; e < GK * GT; e += GT * GT) {
      int r = e / GT, c = e % GT;
      int64_t i = i0 + r;
      bool okr = i < r1;
      xs[r][c] = (okr && a0 + c < R) ? X[i * R + a0 + c] : 0.0;
      y1s[r][c] = (okr && b0 + c < R) ? Y1[i * R + b0 + c] : 0.0;
      if (two) y2s[r][c] = (okr && b0 + c < R) ? Y2[i * R + b0 + c] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int r = 0; r < GK; r++) {
      double xv = xs[r][ty];
      s1 = fma(xv, y1s[r][tx], s1);
      if (two) s2 = fma(xv, y2s[r][tx], s2);
    }
    __syncthreads();
  }
  if (a0 + ty < R && b0 + tx < R) {
    const int64_t RR = (int64_t)R * R;
    P1[blockIdx.z * RR + (a0 + ty) * R + b0 + tx] = s1;
    if (two) P2[blockIdx.z * RR + (a0 + ty) * R + b0 + tx] = s2;
  }
}

__global__ void gram_reduce_kernel(const double* __restrict__ P1, const double* __restrict__ P2, int ks,
                                   int64_t RR, double* __restrict__ G1, double* __restrict__ G2) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < RR; e += (int64_t)gridDim.x * blockDim.x) {
    double s = P1[e];
    for (int k = 1; k < ks; k++) s += P1[k * RR + e];
    G1[e] = s;
    if (P2) {
      double t = P2[e];
      for (int k = 1; k < ks; k++) t += P2[k * RR + e];
      G2[e] = t;
    }
  }
}

// --------- Γ = ∗_{k≠n} S_k, Cholesky (right-looking), packed column-major lower ---------
// element (i, j), i >= j, at col_start(j) + (i - j), col_start(j) = j*R - j*(j-1)/2;
// the R reciprocals of the diagonal follow the packed factor.
__device__ __forceinline__ int pk(int i, int j, int R) { return j * R - (j * (j - 1)) / 2 + (i - j); }

// Blocked (NB = 32) right-to-left panel Cholesky, one CTA.  Per panel [c0, c0+nb):
//  (1) panel update  A(i,j) -= Σ_{m<c0} L(i,m) L(j,m)   (all threads, 4x2 register tiles)
//  (2) diagonal block factorised by warp 0 in registers (lane r holds row r; column k is
//      broadcast with shuffles whose source lane / register are compile-time constants)
//  (3) rows below: L(i,c0+j) solved against the diagonal block (thread per row, registers)
// Only step (2) is sequential, so a panel costs ~3 barriers instead of 32.
constexpr int NB = 16;  // panel width: keeps the unrolled register code small (i-cache)
constexpr int CH_THREADS = 256;
__global__ void __launch_bounds__(CH_THREADS)
    gamma_chol_kernel(const double* __restrict__ S_all, int N, int n, int R, double* __restrict__ Lp,
                      int* status) {
  extern __shared__ double L[];
  const int total = R * (R + 1) / 2;
  double* iv = L + total;  // reciprocals of the diagonal
  __shared__ int bad;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5, nw = CH_THREADS / 32;
  const int64_t RR = (int64_t)R * R;
  if (tid == 0) bad = 0;
  // Γ = ∗_{k≠n} S_k in ascending k (Eq. 1), lower part
  for (int j = warp; j < R; j += nw) {
    const int cs = pk(j, j, R);
    for (int i = j + lane; i < R; i += 32) {
      double gv = 1.0;
      bool first = true;
      for (int k = 0; k < N; k++) {
        if (k == n) continue;
        double sv = S_all[k * RR + (int64_t)i * R + j];
        gv = first ? sv : gv * sv;
        first = false;
      }
      L[cs + (i - j)] = gv;
    }
  }
  __syncthreads();
  for (int c0 = 0; c0 < R; c0 += NB) {
    const int nb = min(NB, R - c0);
    // (1) panel update from the finished columns m < c0
    if (c0 > 0) {
      const int nti = (R - c0 + 3) / 4, ntj = (nb + 1) / 2;
      for (int t = tid; t < nti * ntj; t += CH_THREADS) {
        const int ti = t / ntj, tj = t - ti * ntj;
        const int i0 = c0 + 4 * ti, j0 = c0 + 2 * tj;
        if (i0 + 3 < j0) continue;
        double acc[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
        int cs = -0;  // cs(m) = pk(m,m) - m: L(i,m) = L[cs + i]
        for (int m = 0; m < c0; m++) {
          const double lj0 = L[cs + j0];
          const double lj1 = (j0 + 1 < c0 + nb) ? L[cs + j0 + 1] : 0.0;
#pragma unroll
          for (int q = 0; q < 4; q++) {
            const double li = (i0 + q < R) ? L[cs + i0 + q] : 0.0;
            acc[q][0] = fma(li, lj0, acc[q][0]);
            acc[q][1] = fma(li, lj1, acc[q][1]);
          }
          cs += R - m - 1;
        }
#pragma unroll
        for (int q = 0; q < 4; q++)
#pragma unroll
          for (int c = 0; c < 2; c++) {
            const int i = i0 + q, j = j0 + c;
            if (i < R && j < c0 + nb && i >= j) L[pk(i, j, R)] -= acc[q][c];
          }
      }
      __syncthreads();
    }
    // (2) diagonal block: lane r holds row r (columns 0..r) of the block
    if (warp == 0) {
      double row[NB];
      const int r = lane;
#pragma unroll
      for (int j = 0; j < NB; j++) row[j] = (j <= r && r < nb) ? L[pk(c0 + r, c0 + j, R)] : 0.0;
      int badl = 0;
#pragma unroll
      for (int k = 0; k < NB; k++) {
        if (k < nb) {
          const double akk = __shfl_sync(0xffffffffu, row[k], k);
          if (!(akk > 0.0) || !isfinite(akk)) badl = 1;
          // one long-latency op per pivot on the sequential path: 1/sqrt, then sqrt = a * (1/sqrt a)
          const double inv = rsqrt(akk), d = akk * inv;
          const double lrk = (r > k) ? row[k] * inv : (r == k ? d : row[k]);
          row[k] = lrk;
#pragma unroll
          for (int j = k + 1; j < NB; j++) {
            const double ljk = __shfl_sync(0xffffffffu, row[k], j);  // L(j,k), on lane j
            if (j <= r && j < nb) row[j] = fma(-lrk, ljk, row[j]);
          }
        }
      }
      if (r < nb) {
#pragma unroll
        for (int j = 0; j < NB; j++)
          if (j <= r) L[pk(c0 + r, c0 + j, R)] = row[j];
        iv[c0 + r] = 1.0 / row[r];  // off the sequential path
      }
      if (badl && lane == 0) bad = 1;
    }
    __syncthreads();
    // (3) rows below the block: x L_blk^T = a  (thread per row, column-oriented)
    for (int i = c0 + nb + tid; i < R; i += CH_THREADS) {
      double x[NB];
#pragma unroll
      for (int j = 0; j < NB; j++) x[j] = j < nb ? L[pk(i, c0 + j, R)] : 0.0;
#pragma unroll
      for (int j = 0; j < NB; j++) {
        if (j < nb) {
          x[j] *= iv[c0 + j];
          const int cj = pk(c0 + j, c0 + j, R);
#pragma unroll
          for (int m = j + 1; m < NB; m++)
            if (m < nb) x[m] = fma(-L[cj + (m - j)], x[j], x[m]);
        }
      }
#pragma unroll
      for (int j = 0; j < NB; j++)
        if (j < nb) L[pk(i, c0 + j, R)] = x[j];
    }
    __syncthreads();
    if (bad) break;
  }
  for (int e = tid; e < total + R; e += CH_THREADS) Lp[e] = L[e];
  if (tid == 0) status[0] = bad;
}

// --------- X = M Γ^{-1} with Γ = L L^T, TR rows per CTA, blocked by 32 columns -------------
// forward  Y L^T = M : Y(:,j) = (M(:,j) - Σ_{m<j} Y(:,m) L(j,m)) / L(j,j)
// backward X L   = Y : X(:,j) = (Y(:,j) - Σ_{m>j} X(:,m) L(m,j)) / L(j,j)
// Per panel: (a) the off-panel sums for every (row, column) pair in parallel, (b) the 32x32
// diagonal block solved per row in registers (thread per row).
__global__ void __launch_bounds__(256)
    trisolve_tile_kernel(const double* __restrict__ Lp, const double* __restrict__ M, int64_t rows, int R,
                         int TR, double* __restrict__ X) {
  extern __shared__ double sm[];
  const int total = R * (R + 1) / 2;
  double* L = sm;
  const double* iv = sm + total;
  double* Ys = sm + total + R;  // TR x R, row-major: M, then Y, then X in place
  const int tid = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.x * TR;
  const int tr = (int)min((int64_t)TR, rows - r0);
  for (int e = tid; e < total + R; e += blockDim.x) sm[e] = Lp[e];
  for (int e = tid; e < tr * R; e += blockDim.x) Ys[e] = M[r0 * R + e];
  __syncthreads();
  // forward
  for (int c0 = 0; c0 < R; c0 += NB) {
    const int nb = min(NB, R - c0);
    if (c0 > 0) {
      for (int t = tid; t < tr * nb; t += blockDim.x) {
        const int r = t / nb, j = c0 + (t - r * nb);
        const double* yr = Ys + r * R;
        double s = 0.0;
        int cs = 0;  // L(j,m) = L[cs(m) + j]
        for (int m = 0; m < c0; m++) {
          s = fma(yr[m], L[cs + j], s);
          cs += R - m - 1;
        }
        Ys[r * R + j] -= s;
      }
      __syncthreads();
    }
    if (tid < tr) {
      double* yr = Ys + tid * R;
      double x[NB];
#pragma unroll
      for (int j = 0; j < NB; j++) x[j] = j < nb ? yr[c0 + j] : 0.0;
#pragma unroll
      for (int j = 0; j < NB; j++) {
        if (j < nb) {
          x[j] *= iv[c0 + j];
          const int cj = pk(c0 + j, c0 + j, R);
#pragma unroll
          for (int m = j + 1; m < NB; m++)
            if (m < nb) x[m] = fma(-L[cj + (m - j)], x[j], x[m]);
        }
      }
#pragma unroll
      for (int j = 0; j < NB; j++)
        if (j < nb) yr[c0 + j] = x[j];
    }
    __syncthreads();
  }
  // backward (panels in descending order)
  const int npan = (R + NB - 1) / NB;
  for (int p = npan - 1; p >= 0; p--) {
    const int c0 = p * NB, nb = min(NB, R - c0), c1 = c0 + nb;
    if (c1 < R) {
      for (int t = tid; t < tr * nb; t += blockDim.x) {
        const int r = t / nb, j = c0 + (t - r * nb);
        const double* xr = Ys + r * R;
        const int cj = pk(j, j, R) - j;  // L(m,j) = L[cj + m]
        double s = 0.0;
        for (int m = c1; m < R; m++) s = fma(xr[m], L[cj + m], s);
        Ys[r * R + j] -= s;
      }
      __syncthreads();
    }
    if (tid < tr) {
      double* xr = Ys + tid * R;
      double x[NB];
#pragma unroll
      for (int j = 0; j < NB; j++) x[j] = j < nb ? xr[c0 + j] : 0.0;
#pragma unroll
      for (int j = NB - 1; j >= 0; j--) {
        if (j < nb) {
          x[j] *= iv[c0 + j];
#pragma unroll
          for (int m = 0; m < j; m++) x[m] = fma(-L[pk(c0 + j, c0 + m, R)], x[j], x[m]);
        }
      }
#pragma unroll
      for (int j = 0; j < NB; j++)
        if (j < nb) xr[c0 + j] = x[j];
    }
    __syncthreads();
  }
  for (int e = tid; e < tr * R; e += blockDim.x) X[r0 * R + e] = Ys[e];
}

// --------- W = Σ_{i<j; i,j≠n} dS_i ∗ dS_j ∗ ∗_{k∉{i,j,n}} S_k ---------------------------
__global__ void pp_w_kernel(const double* __restrict__ S_all, const double* __restrict__ dS_all,
                            int N, int n, int R, double* __restrict__ W) {
  const int64_t RR = (int64_t)R * R;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < RR;
       e += (int64_t)gridDim.x * blockDim.x) {
    double w = 0.0;
    for (int i = 0; i < N; i++) {
      if (i == n) continue;
      for (int j = i + 1; j < N; j++) {
        if (j == n) continue;
        double term = dS_all[i * RR + e] * dS_all[j * RR + e];
        for (int k = 0; k < N; k++)
          if (k != i && k != j && k != n) term *= S_all[k * RR + e];
        w += term;
      }
    }
    W[e] = w;
  }
}

// --------- per-update statistics with a last-block fixed-order reduction ------------------
// dA = A - base; out[0] = Σ dA^2, out[1] = Σ A^2, out[2] = Σ M A (if M)
constexpr int ST_BLOCKS = 64;
__global__ void __launch_bounds__(256)
    update_stats_kernel(const double* __restrict__ A, const double* __restrict__ base, double* __restrict__ dA,
                        const double* __restrict__ M, int64_t n, double* __restrict__ part,
                        unsigned int* counter, double* o_dA2, double* o_A2, double* o_MA) {
  __shared__ double red[3][8];
  __shared__ bool last;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double a = A[i];
    double d = a - base[i];
    dA[i] = d;
    s0 = fma(d, d, s0);
    s1 = fma(a, a, s1);
    if (M) s2 = fma(M[i], a, s2);
  }
  for (int o = 16; o > 0; o >>= 1) {
    s0 += __shfl_xor_sync(0xffffffffu, s0, o);
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    red[0][w] = s0;
    red[1][w] = s1;
    red[2][w] = s2;
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    double s = red[threadIdx.x][0];
    for (int k = 1; k < 8; k++) s += red[threadIdx.x][k];
    part[blockIdx.x * 3 + threadIdx.x] = s;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (last && threadIdx.x < 3) {
    __threadfence();
    volatile const double* vp = part;
    double s = vp[threadIdx.x];
    for (unsigned b = 1; b < gridDim.x; b++) s += vp[b * 3 + threadIdx.x];
    if (threadIdx.x == 0) *o_dA2 = s;
    if (threadIdx.x == 1) *o_A2 = s;
    if (threadIdx.x == 2 && M) *o_MA = s;
    if (threadIdx.x == 0) *counter = 0u;
  }
}

// --------- Γ^{-1} = L^{-T} L^{-1} from the packed factor (Alg. 1 line 7 "M Γ†") ---------
// L^{-1} column by column (thread per column: Linv(i,j) = -Σ_{k=j}^{i-1} L(i,k) Linv(k,j) / L(i,i)),
// then Ginv(a,b) = Σ_{k >= max(a,b)} Linv(k,a) Linv(k,b) in ascending k (exactly symmetric).
__global__ void __launch_bounds__(256)
    chol_inverse_kernel(const double* __restrict__ Lp, int R, double* __restrict__ Ginv) {
  extern __shared__ double sm[];
  const int total = R * (R + 1) / 2;
  double* L = sm;                // packed factor
  const double* iv = sm + total; // reciprocal diagonal
  double* Li = sm + total + R;   // R x R dense, Linv(i, j) at Li[i * R + j]
  for (int e = threadIdx.x; e < total + R; e += blockDim.x) L[e] = Lp[e];
  __syncthreads();
  for (int j = threadIdx.x; j < R; j += blockDim.x) {
    for (int i = 0; i < j; i++) Li[i * R + j] = 0.0;
    Li[j * R + j] = iv[j];
    for (int i = j + 1; i < R; i++) {
      double s = 0.0;
      for (int k = j; k < i; k++) s = fma(L[pk(i, k, R)], Li[k * R + j], s);
      Li[i * R + j] = -s * iv[i];
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    const int a = e / R, b = e - a * R;
    double s = 0.0;
    for (int k = max(a, b); k < R; k++) s = fma(Li[k * R + a], Li[k * R + b], s);
    Ginv[e] = s;
  }
}

// --------- Γ^{(n)} = ∗_{k≠n} S^(k) (Eq. 1) and Γ^{-1} by in-place Gauss-Jordan (SPD: no pivoting;
// every pivot is a Schur complement diagonal, > 0 iff Γ is SPD -> status), one CTA ---------
// Blocked by 16 (R padded with the identity to Rp = 16 * ceil(R / 16) <= 128), Γ in shared
// memory.  Block step K = [k0, k0 + 16):
//   P = A[K,K]^{-1}                  one warp: 16 scalar pivots, lane j holds column j
//   Rb = P A[K,:],  Cb = A[:,K]      (old column block)
//   A[I,J] -= Cb[I] Rb[J],  A[I,K] = -Cb[I] P,  A[K,J] = Rb[J],  A[K,K] = P   (I, J != K)
// -- the same pivots, in the same order, as the scalar Gauss-Jordan; the rank-16 updates run
// on all threads with 4 x 4 register tiles (3 barriers per block step instead of one per pivot).
constexpr int kGjThreads = 512;
constexpr int kGjB = 16;

__global__ void __launch_bounds__(kGjThreads)
    gamma_inverse_kernel(const double* __restrict__ S_all, int N, int n, int R, double* __restrict__ Ginv,
                         int* status, int dbg, const double* __restrict__ dS_all, double* __restrict__ W) {
  extern __shared__ double gsm[];
  const int Rp = (R + kGjB - 1) / kGjB * kGjB;
  const int LDA = Rp + 1;
  double* A = gsm;                        // Rp x LDA
  double* Rb = A + (size_t)Rp * LDA;      // 16 x Rp: P A[K,:]
  double* Cb = Rb + kGjB * Rp;            // 16 x Rp: Cb[m * Rp + i] = A[i, k0 + m] (old)
  double* P = Cb + kGjB * Rp;             // 16 x 16
  __shared__ int bad;
  __shared__ double pr[2][kGjB], pc[2][kGjB];  // pivot row / column of the 16 x 16 block
  const int tid = threadIdx.x;
  const int64_t RR = (int64_t)R * R;
  if (tid == 0) bad = 0;
  // PP: the second-order Hadamard sum W^(n) of Eq. 7 (pp_w_kernel's arithmetic) in the same launch, by
  // the CTAs 1.. (each a slice of the R^2 elements) while CTA 0 inverts Γ -- off the Γ^{-1} latency
  if (W && gridDim.x > 1 && blockIdx.x > 0) {
    const int64_t per = (RR + gridDim.x - 2) / (gridDim.x - 1);
    const int64_t lo = (blockIdx.x - 1) * per, hi = min(RR, lo + per);
    for (int64_t e = lo + tid; e < hi; e += kGjThreads) {
      double w = 0.0;
      for (int i = 0; i < N; i++) {
        if (i == n) continue;
        for (int j = i + 1; j < N; j++) {
          if (j == n) continue;
          double term = dS_all[i * RR + e] * dS_all[j * RR + e];
          for (int k = 0; k < N; k++)
            if (k != i && k != j && k != n) term *= S_all[k * RR + e];
          w += term;
        }
      }
      W[e] = w;
    }
    return;
  }
  if (W && gridDim.x == 1) {
    for (int64_t e = tid; e < RR; e += kGjThreads) {
      double w = 0.0;
      for (int i = 0; i < N; i++) {
        if (i == n) continue;
        for (int j = i + 1; j < N; j++) {
          if (j == n) continue;
          double term = dS_all[i * RR + e] * dS_all[j * RR + e];
          for (int k = 0; k < N; k++)
            if (k != i && k != j && k != n) term *= S_all[k * RR + e];
          w += term;
        }
      }
      W[e] = w;
    }
  }
#pragma unroll 4
  for (int e = tid; e < Rp * Rp; e += kGjThreads) {
    const int i = e / Rp, j = e - i * Rp;
    double gv = (i == j) ? 1.0 : 0.0;  // padding: identity (does not touch the R x R block)
    if (i < R && j < R) {
      bool first = true;
      for (int k = 0; k < N; k++) {
        if (k == n) continue;
        const double sv = S_all[k * RR + (int64_t)i * R + j];
        gv = first ? sv : gv * sv;
        first = false;
      }
    }
    A[i * LDA + j] = gv;
  }
  __syncthreads();
  const int ntj = Rp / 4, ntiles = ntj * (Rp / 8);
  for (int k0 = 0; k0 < Rp; k0 += kGjB) {
    // ---- P = A[K,K]^{-1}: 256 threads, thread (i, j) holds element (i, j); pivot row and
    // column through double-buffered shared memory, one barrier per pivot ----
    {
      const int i = tid >> 4, j = tid & 15;
      const bool act = tid < kGjB * kGjB && !(dbg & 1);
      double a = act ? A[(k0 + i) * LDA + k0 + j] : 0.0;
      if (act && i == 0) pr[0][j] = a;
      if (act && j == 0) pc[0][i] = a;
      __syncthreads();
#pragma unroll 1
      for (int p = 0; p < kGjB; p++) {
        const int b = p & 1;
        if (act) {
          const double piv = pr[b][p];
          const double inv = __drcp_rn(piv);  // IEEE reciprocal (= 1.0 / piv)
          if (tid == 0 && (!(piv > 0.0) || !isfinite(piv))) bad = 1;
          const double r = pr[b][j] * inv, c = pc[b][i];
          if (i == p) a = (j == p) ? inv : r;
          else a = (j == p) ? -c * inv : fma(-c, r, a);
          if (i == p + 1) pr[b ^ 1][j] = a;
          if (j == p + 1) pc[b ^ 1][i] = a;
        }
        __syncthreads();
      }
      if (act) P[i * kGjB + j] = a;
    }
    __syncthreads();
    // ---- Rb = P A[K,:] (old rows K), Cb = A[:,K] (old) ----
    for (int e = tid; e < kGjB * Rp; e += kGjThreads) {
      if (dbg & 2) break;
      const int m = e / Rp, c = e - m * Rp;
      double acc = 0.0;
#pragma unroll
      for (int q = 0; q < kGjB; q++) acc = fma(P[m * kGjB + q], A[(k0 + q) * LDA + c], acc);
      Rb[m * Rp + c] = acc;
      Cb[m * Rp + c] = A[c * LDA + k0 + m];
    }
    __syncthreads();
    // ---- rank-16 update, 8 x 4 register tiles: rows 8 ti .. 8 ti + 7, columns tj + ntj q
    // (lanes hold consecutive columns: conflict-free shared-memory rows; 12 loads per 32 FMAs) ----
    for (int t = tid; t < ntiles; t += kGjThreads) {
      if (dbg & 4) break;
      const int i0 = (t / ntj) * 8, tj = t % ntj;
      const bool rowK = i0 >= k0 && i0 < k0 + kGjB;
      int jq[4];
      bool colK[4];
#pragma unroll
      for (int q = 0; q < 4; q++) {
        jq[q] = tj + ntj * q;
        colK[q] = jq[q] >= k0 && jq[q] < k0 + kGjB;
      }
      double acc[8][4];
      if (rowK) {
#pragma unroll
        for (int p = 0; p < 8; p++)
#pragma unroll
          for (int q = 0; q < 4; q++)
            acc[p][q] = colK[q] ? P[(i0 - k0 + p) * kGjB + jq[q] - k0] : Rb[(i0 - k0 + p) * Rp + jq[q]];
      } else {
#pragma unroll
        for (int p = 0; p < 8; p++)
#pragma unroll
          for (int q = 0; q < 4; q++) acc[p][q] = colK[q] ? 0.0 : A[(i0 + p) * LDA + jq[q]];
#pragma unroll 2
        for (int m = 0; m < kGjB; m++) {
          double cv[8], rv[4];
#pragma unroll
          for (int p = 0; p < 8; p++) cv[p] = Cb[m * Rp + i0 + p];
#pragma unroll
          for (int q = 0; q < 4; q++) rv[q] = colK[q] ? P[m * kGjB + jq[q] - k0] : Rb[m * Rp + jq[q]];
#pragma unroll
          for (int p = 0; p < 8; p++)
#pragma unroll
            for (int q = 0; q < 4; q++) acc[p][q] = fma(-cv[p], rv[q], acc[p][q]);
        }
      }
#pragma unroll
      for (int p = 0; p < 8; p++)
#pragma unroll
        for (int q = 0; q < 4; q++) A[(i0 + p) * LDA + jq[q]] = acc[p][q];
    }
    __syncthreads();
  }
  for (int e = tid; e < R * R; e += kGjThreads) {
    const int i = e / R, j = e - i * R;
    Ginv[e] = A[i * LDA + j];
  }
  if (tid == 0) status[0] = bad;
}

// --------- large R (beyond one CTA's shared memory): the same blocked Gauss-Jordan over the
// whole grid, Γ in global memory (L2-resident: R = 1024 is 8 MB).  Per block step K:
//   every CTA inverts the 16 x 16 pivot block A[K,K] itself (element-parallel, in shared
//   memory: the same P everywhere, no extra grid barrier);
//   Rb = P A[K,:] and Cb = A[:,K] by all threads -> grid sync;
//   A[I,J] -= Cb[I] Rb[J], A[I,K] = -Cb[I] P, A[K,J] = Rb[J], A[K,K] = P -> grid sync.
// Same pivots and the same per-element operation order as the single-CTA kernel.
__global__ void __launch_bounds__(256)
    gamma_inverse_big_kernel(const double* __restrict__ S_all, int N, int n, int R, double* __restrict__ A,
                             double* __restrict__ Rb, double* __restrict__ Cb, double* __restrict__ Ginv,
                             int* status) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const int Rp = (R + kGjB - 1) / kGjB * kGjB;
  const int64_t RR = (int64_t)R * R;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  __shared__ double P[kGjB * kGjB];
  __shared__ double pr[2][kGjB], pc[2][kGjB];
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  for (int64_t e = gt; e < (int64_t)Rp * Rp; e += nthr) {
    const int i = (int)(e / Rp), j = (int)(e - (int64_t)i * Rp);
    double gv = (i == j) ? 1.0 : 0.0;
    if (i < R && j < R) {
      bool first = true;
      for (int k = 0; k < N; k++) {
        if (k == n) continue;
        const double sv = S_all[k * RR + (int64_t)i * R + j];
        gv = first ? sv : gv * sv;
        first = false;
      }
    }
    A[e] = gv;
  }
  grid.sync();
  for (int k0 = 0; k0 < Rp; k0 += kGjB) {
    {  // pivot block inverse, redundantly in every CTA
      const int i = threadIdx.x >> 4, j = threadIdx.x & 15;
      double a = A[(int64_t)(k0 + i) * Rp + k0 + j];
      if (i == 0) pr[0][j] = a;
      if (j == 0) pc[0][i] = a;
      __syncthreads();
#pragma unroll 1
      for (int p = 0; p < kGjB; p++) {
        const int b = p & 1;
        const double piv = pr[b][p];
        const double inv = __drcp_rn(piv);
        if (threadIdx.x == 0 && (!(piv > 0.0) || !isfinite(piv))) bad = 1;
        const double r = pr[b][j] * inv, c = pc[b][i];
        if (i == p) a = (j == p) ? inv : r;
        else a = (j == p) ? -c * inv : fma(-c, r, a);
        if (i == p + 1) pr[b ^ 1][j] = a;
        if (j == p + 1) pc[b ^ 1][i] = a;
        __syncthreads();
      }
      P[i * kGjB + j] = a;
      __syncthreads();
    }
    for (int64_t e = gt; e < (int64_t)kGjB * Rp; e += nthr) {
      const int m = (int)(e / Rp), c = (int)(e - (int64_t)m * Rp);
      double acc = 0.0;
#pragma unroll
      for (int q = 0; q < kGjB; q++) acc = fma(P[m * kGjB + q], A[(int64_t)(k0 + q) * Rp + c], acc);
      Rb[e] = acc;
      Cb[e] = A[(int64_t)c * Rp + k0 + m];
    }
    grid.sync();
    for (int64_t e = gt; e < (int64_t)Rp * Rp; e += nthr) {
      const int i = (int)(e / Rp), j = (int)(e - (int64_t)i * Rp);
      const bool rowK = i >= k0 && i < k0 + kGjB, colK = j >= k0 && j < k0 + kGjB;
      double v;
      if (rowK) {
        v = colK ? P[(i - k0) * kGjB + j - k0] : Rb[(int64_t)(i - k0) * Rp + j];
      } else {
        v = colK ? 0.0 : A[e];
#pragma unroll
        for (int m = 0; m < kGjB; m++)
          v = fma(-Cb[(int64_t)m * Rp + i], colK ? P[m * kGjB + j - k0] : Rb[(int64_t)m * Rp + j], v);
      }
      A[e] = v;
    }
    grid.sync();
  }
  for (int64_t e = gt; e < RR; e += nthr) {
    const int i = (int)(e / R), j = (int)(e - (int64_t)i * R);
    Ginv[e] = A[(int64_t)i * Rp + j];
  }
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) status[0] = bad;
}

size_t gamma_inverse_smem(int R) {
  const size_t Rp = (size_t)(R + kGjB - 1) / kGjB * kGjB;
  return sizeof(double) * (Rp * (Rp + 1) + 2 * kGjB * Rp + kGjB * kGjB);
}

// opt a kernel in to the largest dynamic shared memory the device allows
template <typename K>
cudaError_t opt_in_smem(K kern) {
  int dev = 0, optin = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaFuncAttributes fa;
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, kern);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes);
  return e;
}

}  // namespace

size_t gamma_inverse_big_ws(int R) {
  const size_t Rp = (size_t)(R + kGjB - 1) / kGjB * kGjB;
  return Rp * Rp + 2 * kGjB * Rp;
}

cudaError_t launch_gamma_inverse_big(const double* S_all, int N, int n, int R, double* ws, double* Ginv,
                                     int* status, cudaStream_t st) {
  if (R < 1) return cudaErrorInvalidValue;
  const int Rp = (R + kGjB - 1) / kGjB * kGjB;
  double* A = ws;
  double* Rb = ws + (size_t)Rp * Rp;
  double* Cb = Rb + (size_t)kGjB * Rp;
  int dev = 0, nsm = 148, per = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, gamma_inverse_big_kernel, 256, 0);
  int blocks = std::max(1, std::min(nsm * std::max(per, 1), (int)(((int64_t)Rp * Rp + 255) / 256)));
  void* args[] = {&S_all, &N, &n, &R, &A, &Rb, &Cb, &Ginv, &status};
  g_launches++;
  return cudaLaunchCooperativeKernel((void*)gamma_inverse_big_kernel, blocks, 256, args, 0, st);
}


cudaError_t launch_gram(const double* X, const double* Y1, const double* Y2, int64_t rows, int R,
                        double* G1, double* G2, double* ws, int64_t ws_elems, cudaStream_t st) {
  const int nt = (R + GT - 1) / GT;
  const int64_t RR = (int64_t)R * R;
  int ks = (296 + nt * nt - 1) / (nt * nt);
  int64_t max_by_rows = (rows + 63) / 64;
  if (ks > max_by_rows) ks = (int)max_by_rows;
  if (ks > 16) ks = 16;
  const int per = Y2 ? 2 : 1;
  if (ws == nullptr || (int64_t)ks * RR * per > ws_elems) ks = 1;
  if (ks < 1) ks = 1;
  int64_t rps = (rows + ks - 1) / ks;
  dim3 grid(nt, nt, ks);
  g_launches++;
  if (ks == 1) {
    gram_partial_kernel<<<grid, GT * GT, 0, st>>>(X, Y1, Y2, rows, R, rps, G1, G2);
    return cudaGetLastError();
  }
  double* P1 = ws;
  double* P2 = Y2 ? ws + ks * RR : nullptr;
  gram_partial_kernel<<<grid, GT * GT, 0, st>>>(X, Y1, Y2, rows, R, rps, P1, P2);
  g_launches++;
  int blocks = (int)((RR + 255) / 256);
  gram_reduce_kernel<<<blocks, 256, 0, st>>>(P1, P2, ks, RR, G1, G2);
  return cudaGetLastError();
}

cudaError_t launch_gamma_chol(const double* S_all, int N, int n, int R, double* Lp, int* status,
                              cudaStream_t st) {
  size_t smem = sizeof(double) * ((size_t)R * (R + 1) / 2 + R);
  static bool attr = false;  // one process per GPU: set the opt-in once
  if (!attr) {
    cudaError_t e = opt_in_smem(gamma_chol_kernel);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  g_launches++;
  gamma_chol_kernel<<<1, CH_THREADS, smem, st>>>(S_all, N, n, R, Lp, status);
  return cudaGetLastError();
}

cudaError_t launch_gamma_inverse(const double* S_all, int N, int n, int R, double* Ginv, int* status,
                                 cudaStream_t st, const double* dS_all, double* W) {
  if (R < 1 || R > 128) return cudaErrorInvalidValue;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = opt_in_smem(gamma_inverse_kernel);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  g_launches++;
  static const int dbg = getenv("CPD_GJ_DBG") ? atoi(getenv("CPD_GJ_DBG")) : 0;  // profiling switches
  // W (PP) by extra CTAs beside the inverting CTA 0 (experiment switch CPD_GJ_W1: all in CTA 0)
  static const bool w1 = getenv("CPD_GJ_W1") != nullptr;
  const int grid = (W && !w1) ? 1 + (int)std::min<int64_t>(16, ((int64_t)R * R + 2047) / 2048) : 1;
  gamma_inverse_kernel<<<grid, kGjThreads, gamma_inverse_smem(R), st>>>(S_all, N, n, R, Ginv, status, dbg, dS_all, W);
  return cudaGetLastError();
}

cudaError_t launch_chol_inverse(const double* Lp, int R, double* Ginv, cudaStream_t st) {
  const size_t smem = sizeof(double) * ((size_t)R * (R + 1) / 2 + R + (size_t)R * R);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = opt_in_smem(chol_inverse_kernel);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  g_launches++;
  chol_inverse_kernel<<<1, 256, smem, st>>>(Lp, R, Ginv);
  return cudaGetLastError();
}

cudaError_t launch_trisolve(const double* Lp, const double* M, int64_t rows, int R, double* X,
                            cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  const size_t lbytes = sizeof(double) * ((size_t)R * (R + 1) / 2 + R);
  // rows per CTA: spread over the SMs, bounded by shared memory (227 KB)
  int64_t tr = (rows + 147) / 148;
  int64_t tr_max = ((int64_t)227 * 1024 - (int64_t)lbytes) / (8 * (int64_t)R);
  if (tr > tr_max) tr = tr_max;
  if (tr > 64) tr = 64;
  if (tr < 1) tr = 1;
  size_t smem = lbytes + sizeof(double) * tr * R;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = opt_in_smem(trisolve_tile_kernel);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  int64_t blocks = (rows + tr - 1) / tr;
  g_launches++;
  trisolve_tile_kernel<<<(unsigned)blocks, 256, smem, st>>>(Lp, M, rows, R, (int)tr, X);
  return cudaGetLastError();
}

cudaError_t launch_pp_w(const double* S_all, const double* dS_all, int N, int n, int R, double* W,
                        cudaStream_t st) {
  int64_t RR = (int64_t)R * R;
  int blocks = (int)((RR + 255) / 256);
  g_launches++;
  pp_w_kernel<<<blocks, 256, 0, st>>>(S_all, dS_all, N, n, R, W);
  return cudaGetLastError();
}

cudaError_t launch_update_stats(const double* A, const double* base, double* dA, const double* M, int64_t n,
                                double* part, unsigned int* counter, double* o_dA2, double* o_A2, double* o_MA,
                                cudaStream_t st) {
  int64_t blocks = (n + 255) / 256;
  if (blocks > ST_BLOCKS) blocks = ST_BLOCKS;
  if (blocks < 1) blocks = 1;
  g_launches++;
  update_stats_kernel<<<(unsigned)blocks, 256, 0, st>>>(A, base, dA, M, n, part, counter, o_dA2, o_A2, o_MA);
  return cudaGetLastError();
}

}  // namespace cpd
