// Small dense R x R work of each factor update (latency-bound; "the cost of
// solving linear systems is often small"): Gram matrices, dS (Eq. 8), the
// Hadamard chain Γ^(n) (Eq. 1) with its Cholesky factorisation, the row-wise normal-
// equation solve A^(n) = M^(n) Γ^(n)^{-1} (Alg. 1 line 7; reading Q3: Cholesky),
// and the PP second-order Hadamard sum W^(n) of Eq. 7.
// All reductions run in a fixed order (deterministic; no atomics).
#include "kernels.h"

namespace cpd {
namespace {

// ---------------- Gram: G[a][b] = Σ_i X[i][a] Y[i][b] ------------------------------------
constexpr int GT = 16;   // output tile
constexpr int GK = 32;   // rows per smem chunk
__global__ void __launch_bounds__(GT* GT)
    gram_kernel(const double* __restrict__ X, const double* __restrict__ Y, int64_t rows, int R,
                double* __restrict__ G) {
  __shared__ double xs[GK][GT + 1], ys[GK][GT + 1];
  const int tx = threadIdx.x % GT, ty = threadIdx.x / GT;
  const int a0 = blockIdx.y * GT, b0 = blockIdx.x * GT;
  double s = 0.0;
  for (int64_t i0 = 0; i0 < rows; i0 += GK) {
    for (int e = threadIdx.x; e < GK * GT; e += GT * GT) {
      int r = e / GT, c = e % GT;
      int64_t i = i0 + r;
      xs[r][c] = (i < rows && a0 + c < R) ? X[i * R + a0 + c] : 0.0;
      ys[r][c] = (i < rows && b0 + c < R) ? Y[i * R + b0 + c] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int r = 0; r < GK; r++) s = fma(xs[r][ty], ys[r][tx], s);
    __syncthreads();
  }
  if (a0 + ty < R && b0 + tx < R) G[(a0 + ty) * R + b0 + tx] = s;
}

// --------- Γ = ∗_{k≠n} S_k, Cholesky (right-looking), packed column-major lower ---------
// element (i, j), i >= j, at col_start(j) + (i - j), col_start(j) = j*R - j*(j-1)/2
__device__ __forceinline__ int pk(int i, int j, int R) { return j * R - (j * (j - 1)) / 2 + (i - j); }

__global__ void __launch_bounds__(1024)
    gamma_chol_kernel(const double* __restrict__ S_all, int N, int n, int R, double* __restrict__ Lp,
                      int* status) {
  extern __shared__ double L[];
  __shared__ int bad;
  const int tid = threadIdx.x;
  if (tid == 0) bad = 0;
  const int total = R * (R + 1) / 2;
  // build Γ (lower part) in packed storage, Hadamard product in ascending k (Eq. 1)
  for (int j = 0; j < R; j++) {
    for (int i = j + tid; i < R; i += blockDim.x) {
      double gv = 1.0;
      bool first = true;
      for (int k = 0; k < N; k++) {
        if (k == n) continue;
        double sv = S_all[(size_t)k * R * R + (size_t)i * R + j];
        gv = first ? sv : gv * sv;
        first = false;
      }
      L[pk(i, j, R)] = gv;
    }
  }
  __syncthreads();
  const int tx = tid % 32, ty = tid / 32, nty = blockDim.x / 32;
  for (int k = 0; k < R; k++) {
    // diagonal + column scale
    double d = L[pk(k, k, R)];
    if (!(d > 0.0) || !isfinite(d)) {
      if (tid == 0) bad = 1;
      break;  // uniform across the block (all threads read the same d)
    }
    d = sqrt(d);
    __syncthreads();
    if (tid == 0) L[pk(k, k, R)] = d;
    for (int i = k + 1 + tid; i < R; i += blockDim.x) L[pk(i, k, R)] /= d;
    __syncthreads();
    // trailing update A(i,j) -= L(i,k) L(j,k), k < j <= i
    for (int j = k + 1 + ty; j < R; j += nty) {
      double ljk = L[pk(j, k, R)];
      for (int i = j + tx; i < R; i += 32) L[pk(i, j, R)] -= L[pk(i, k, R)] * ljk;
    }
    __syncthreads();
  }
  __syncthreads();
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
  const int total = R * (R + 1) / 2;
  for (int e = threadIdx.x; e < total; e += blockDim.x) L[e] = Lp[e];
  __syncthreads();
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
        double yk = __shfl_sync(0xffffffffu, m[q], kk) / L[pk(k, k, R)];
        if (lane == kk) m[q] = yk;
#pragma unroll
        for (int q2 = q; q2 < RQ; q2++) {
          int j = lane + 32 * q2;
          if (j > k && j < R) m[q2] = fma(-L[pk(j, k, R)], yk, m[q2]);
        }
      }
    }
    // backward: x_k = (y_k - Σ_{j>k} L_jk x_j) / L_kk
#pragma unroll
    for (int q = RQ - 1; q >= 0; q--) {
      for (int kk = 31; kk >= 0; kk--) {
        int k = 32 * q + kk;
        if (k >= R) continue;
        double part = 0.0;
#pragma unroll
        for (int q2 = q; q2 < RQ; q2++) {
          int j = lane + 32 * q2;
          if (j > k && j < R) part = fma(L[pk(j, k, R)], m[q2], part);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        double yk = __shfl_sync(0xffffffffu, m[q], kk);
        double xk = (yk - part) / L[pk(k, k, R)];
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

}  // namespace

cudaError_t launch_gram(const double* X, const double* Y, int64_t rows, int R, double* G,
                        cudaStream_t st) {
  dim3 grid((R + GT - 1) / GT, (R + GT - 1) / GT);
  g_launches++;
  gram_kernel<<<grid, GT * GT, 0, st>>>(X, Y, rows, R, G);
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
  size_t smem = sizeof(double) * (size_t)R * (R + 1) / 2;
  auto kern = trisolve_kernel<RQ>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int threads = 1024;
  int64_t warps_needed = rows;
  int64_t blocks = (warps_needed + 31) / 32;
  if (blocks > 148) blocks = 148;
  if (blocks < 1) blocks = 1;
  g_launches++;
  kern<<<(unsigned)blocks, threads, smem, st>>>(Lp, M, rows, R, X);
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

}  // namespace cpd
