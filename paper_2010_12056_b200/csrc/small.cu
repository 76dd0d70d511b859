// Small dense R x R work of each factor update (latency-bound; "the cost of
// solving linear systems is often small"): Gram matrices, dS (Eq. 8), the
// Hadamard chain Γ^(n) (Eq. 1) with its Cholesky factorisation, the row-wise normal-
// equation solve A^(n) = M^(n) Γ^(n)^{-1} (Alg. 1 line 7; reading Q3: Cholesky),
// the PP second-order Hadamard sum W^(n) of Eq. 7, and the per-update
// statistics (dA = A - base, ||dA||^2, ||A||^2, <M, A>) for Alg. 2 line 5 and Eq. 3.
// All reductions run in a fixed order (deterministic; no floating-point atomics).
#include "kernels.h"

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

__global__ void __launch_bounds__(1024)
    gamma_chol_kernel(const double* __restrict__ S_all, int N, int n, int R, double* __restrict__ Lp,
                      int* status) {
  extern __shared__ double L[];
  __shared__ int bad;
  const int tid = threadIdx.x;
  if (tid == 0) bad = 0;
  const int total = R * (R + 1) / 2;
  const int64_t RR = (int64_t)R * R;
  // Γ (lower part), Hadamard product in ascending k (Eq. 1); coalesced over j
  for (int idx = tid; idx < R * R; idx += blockDim.x) {
    int i = idx / R, j = idx - i * R;
    if (j > i) continue;
    double gv = 1.0;
    bool first = true;
    for (int k = 0; k < N; k++) {
      if (k == n) continue;
      double sv = S_all[k * RR + idx];
      gv = first ? sv : gv * sv;
      first = false;
    }
    L[pk(i, j, R)] = gv;
  }
  __syncthreads();
  const int tx = tid % 32, ty = tid / 32, nty = blockDim.x / 32;
  for (int k = 0; k < R; k++) {
    double d = L[pk(k, k, R)];
    if (!(d > 0.0) || !isfinite(d)) {
      if (tid == 0) bad = 1;
      break;  // uniform: every thread read the same d
    }
    d = sqrt(d);
    const double inv = 1.0 / d;
    // column k below the diagonal: L(i,k) = A(i,k) * (1/L(k,k)) (LAPACK dpotf2 scales by
    // the reciprocal); the trailing update recomputes the scaled L(i,k), L(j,k) it needs so
    // the column can be scaled after the same barrier
    for (int j = k + 1 + ty; j < R; j += nty) {
      double ljk = L[pk(j, k, R)] * inv;
      for (int i = j + tx; i < R; i += 32) {
        double lik = L[pk(i, k, R)] * inv;
        L[pk(i, j, R)] -= lik * ljk;
      }
    }
    __syncthreads();
    for (int i = k + 1 + tid; i < R; i += blockDim.x) L[pk(i, k, R)] *= inv;
    if (tid == 0) {
      L[pk(k, k, R)] = d;
      Lp[total + k] = inv;
    }
    __syncthreads();
  }
  for (int e = tid; e < total; e += blockDim.x) Lp[e] = L[e];
  if (tid == 0) status[0] = bad;
}

// --------- X[i,:] = M[i,:] Γ^{-1}: L y = m (column sweep), L^T x = y (dot sweep) ---------
// One warp per row; lane holds entries j = lane + 32q.
template <int RQ>
__global__ void __launch_bounds__(1024)
    trisolve_kernel(const double* __restrict__ Lp, const double* __restrict__ M, int64_t rows, int R,
                    double* __restrict__ X) {
  extern __shared__ double L[];
  const int total = R * (R + 1) / 2 + R;
  for (int e = threadIdx.x; e < total; e += blockDim.x) L[e] = Lp[e];
  __syncthreads();
  const double* invd = L + (total - R);
  const int lane = threadIdx.x & 31;
  const int64_t wglob = blockIdx.x * (int64_t)(blockDim.x / 32) + (threadIdx.x >> 5);
  const int64_t wstride = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t row = wglob; row < rows; row += wstride) {
    double m[RQ];
#pragma unroll
    for (int q = 0; q < RQ; q++) {
      int j = lane + 32 * q;
      m[q] = j < R ? M[row * R + j] : 0.0;
    }
    // forward: y_k = m_k / L_kk ; m_j -= L_jk y_k (j > k)
#pragma unroll
    for (int q = 0; q < RQ; q++) {
      for (int kk = 0; kk < 32; kk++) {
        int k = 32 * q + kk;
        if (k >= R) break;
        double yk = __shfl_sync(0xffffffffu, m[q], kk) * invd[k];
        if (lane == kk) m[q] = yk;
        const int cs = pk(k, k, R);
#pragma unroll
        for (int q2 = q; q2 < RQ; q2++) {
          int j = lane + 32 * q2;
          if (j > k && j < R) m[q2] = fma(-L[cs + (j - k)], yk, m[q2]);
        }
      }
    }
    // backward: x_k = (y_k - Σ_{j>k} L_jk x_j) / L_kk
#pragma unroll
    for (int q = RQ - 1; q >= 0; q--) {
      for (int kk = 31; kk >= 0; kk--) {
        int k = 32 * q + kk;
        if (k >= R) continue;
        const int cs = pk(k, k, R);
        double part = 0.0;
#pragma unroll
        for (int q2 = q; q2 < RQ; q2++) {
          int j = lane + 32 * q2;
          if (j > k && j < R) part = fma(L[cs + (j - k)], m[q2], part);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        double yk = __shfl_sync(0xffffffffu, m[q], kk);
        double xk = (yk - part) * invd[k];
        if (lane == kk) m[q] = xk;
      }
    }
#pragma unroll
    for (int q = 0; q < RQ; q++) {
      int j = lane + 32 * q;
      if (j < R) X[row * R + j] = m[q];
    }
  }
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

}  // namespace

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
  size_t smem = sizeof(double) * (size_t)R * (R + 1) / 2;
  cudaError_t e = cudaFuncSetAttribute(gamma_chol_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  g_launches++;
  gamma_chol_kernel<<<1, 1024, smem, st>>>(S_all, N, n, R, Lp, status);
  return cudaGetLastError();
}

template <int RQ>
static cudaError_t trisolve_rq(const double* Lp, const double* M, int64_t rows, int R, double* X,
                               cudaStream_t st) {
  size_t smem = sizeof(double) * ((size_t)R * (R + 1) / 2 + R);
  auto kern = trisolve_kernel<RQ>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  // spread rows over all SMs: warps per block chosen so that ~148 blocks cover the rows
  int64_t wpb = (rows + 147) / 148;
  if (wpb < 1) wpb = 1;
  if (wpb > 32) wpb = 32;
  int64_t blocks = (rows + wpb - 1) / wpb;
  if (blocks > 148) blocks = 148;
  g_launches++;
  kern<<<(unsigned)blocks, (unsigned)(32 * wpb), smem, st>>>(Lp, M, rows, R, X);
  return cudaGetLastError();
}

cudaError_t launch_trisolve(const double* Lp, const double* M, int64_t rows, int R, double* X,
                            cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  switch ((R + 31) / 32) {
    case 1: return trisolve_rq<1>(Lp, M, rows, R, X, st);
    case 2: return trisolve_rq<2>(Lp, M, rows, R, X, st);
    case 3: return trisolve_rq<3>(Lp, M, rows, R, X, st);
    case 4: return trisolve_rq<4>(Lp, M, rows, R, X, st);
    case 5: return trisolve_rq<5>(Lp, M, rows, R, X, st);
    case 6: return trisolve_rq<6>(Lp, M, rows, R, X, st);
    case 7: return trisolve_rq<7>(Lp, M, rows, R, X, st);
    case 8: return trisolve_rq<8>(Lp, M, rows, R, X, st);
  }
  return cudaErrorInvalidValue;
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
