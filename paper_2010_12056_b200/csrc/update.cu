// Fused factor update of one mode (Alg. 1 lines 7-8; Eq. 1; PP:
// Eqs. 5/7/8 P:386-409): one cooperative launch instead of V-term GEMM + row solve +
// statistics + Gram partials + Gram reduce (five latency-bound launches).
//
// Phase 1 (warp per row, lanes own columns c = lane + 32 u):
//   m   = M[i]  (+ a_old W  for PP: V^(n) = A^(n) W^(n), Eq. 7, with the pre-update row)
//   x   = m Γ^{-1} ("M Γ†"), Γ^{-1} = L^{-T} L^{-1} formed from the Cholesky factor on the
//         side stream (launch_chol_inverse) while the MTTKRP streamed; a mat-vec per row,
//         y_k broadcast by shuffles, independent FMAs per lane
//   A[i] = x, dA[i] = x - base[i] (base = the row before the update, or A_p in PP),
//   partial sums of |dA|^2, |A|^2 and <m, x> (Eq. 3 needs <M^(N), A^(N)>) per CTA.
// grid.sync()
// Phase 2: S = A^T A and dS = A^T dA (Eq. 8) over all rows, one output element per
//   thread, rows in ascending order (deterministic; S exactly symmetric); CTA 0 reduces the
//   statistics partials in CTA order.
#include <cooperative_groups.h>

#include <cstdlib>

#include "kernels.h"

namespace cpd {
namespace {

namespace cg = cooperative_groups;

constexpr int UPD_THREADS = 256;


// dst[0..n) = src[0..n): 8 independent loads in flight per thread
__device__ __forceinline__ void fill_smem(double* dst, const double* __restrict__ src, int n, int tid) {
  int e = tid;
  for (; e + 7 * UPD_THREADS < n; e += 8 * UPD_THREADS) {
    double v[8];
#pragma unroll
    for (int q = 0; q < 8; q++) v[q] = __ldg(src + e + q * UPD_THREADS);
#pragma unroll
    for (int q = 0; q < 8; q++) dst[e + q * UPD_THREADS] = v[q];
  }
  for (; e < n; e += UPD_THREADS) dst[e] = __ldg(src + e);
}

// Γ^{-1} of a 32 x 32 SPD matrix held by ONE warp, lane j holding column j (col[i] = Γ[i][j]):
// Gauss-Jordan without pivoting (every pivot is a Schur-complement diagonal of an SPD matrix,
// > 0 iff Γ is SPD -> bad), the pivot column broadcast by shuffles; fully unrolled, so the column
// stays in registers.  Rows / columns beyond R are padded with the identity (pivots 1, untouched).
__device__ __forceinline__ void gj32_warp(double (&col)[32], int lane, bool& bad) {
#pragma unroll
  for (int p = 0; p < 32; p++) {
    const double piv = __shfl_sync(0xffffffffu, col[p], p);
    const double inv = __drcp_rn(piv);  // IEEE reciprocal (= 1.0 / piv)
    if (!(piv > 0.0) || !isfinite(piv)) bad = true;
    const double r = col[p] * inv;      // new row p, column lane (j != p)
#pragma unroll
    for (int i = 0; i < 32; i++) {
      if (i == p) continue;
      const double c = __shfl_sync(0xffffffffu, col[i], p);  // old Γ[i][p]
      col[i] = (lane == p) ? -c * inv : fma(-c, r, col[i]);
    }
    col[p] = (lane == p) ? inv : r;
  }
}

// out[c] = Σ_k v[k] Mat[k, c] for the row v held by a warp (lane owns v[lane + 32 u]) and the
// columns c = lane + 32 u: v_k broadcast by one shuffle per k (block u of k is static), two
// independent FMA chains (even / odd k) summed at the end -- a fixed order
template <int U>
__device__ __forceinline__ void rowvec_mat(const double (&v)[U], const double* __restrict__ Mat, int R, int lane,
                                           double (&out)[U]) {
  double e[U], o[U];
#pragma unroll
  for (int u = 0; u < U; u++) e[u] = o[u] = 0.0;
#pragma unroll
  for (int ub = 0; ub < U; ub++) {
    const int kmax = min(32, R - 32 * ub);
#pragma unroll 4
    for (int kk = 0; kk < 32; kk += 2) {
      if (kk >= kmax) break;
      const int k = 32 * ub + kk;
      const double v0 = __shfl_sync(0xffffffffu, v[ub], kk);
      const double v1 = __shfl_sync(0xffffffffu, v[ub], kk + 1);
      const bool has1 = kk + 1 < kmax;
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int c = lane + 32 * u;
        if (c < R) {
          e[u] = fma(v0, Mat[k * R + c], e[u]);
          if (has1) o[u] = fma(v1, Mat[(k + 1) * R + c], o[u]);
        }
      }
    }
  }
#pragma unroll
  for (int u = 0; u < U; u++) out[u] = e[u] + o[u];
}

// phase 2b: S, dS = Σ over the nparts CTA partials in CTA order (deterministic; S exactly symmetric);
// gt / nthr: this thread's index in, and the size of, the grid doing the reduction; t0 >= 0 for the
// threads 0..2 of one CTA (the scalar sums)
__device__ __forceinline__ void reduce_partials(const double* __restrict__ gpart, const double* __restrict__ part,
                                                unsigned nparts, int64_t nout, int64_t RR, int64_t gt, int64_t nthr,
                                                int t0, double* __restrict__ S, double* __restrict__ dS,
                                                double* __restrict__ o_dA2, double* __restrict__ o_A2,
                                                double* __restrict__ o_MA) {
  // 4 lanes per output when the grid has the threads (lane q sums the CTA partials c = q mod 4 in
  // ascending c, then ((s0 + s1) + (s2 + s3))): a fixed order either way
  if (nout * 4 <= nthr) {
    const int64_t e = gt >> 2;
    const int q = (int)(gt & 3);
    double acc = 0.0;
    if (e < nout) {
      unsigned c = q;
      for (; c + 12 < nparts; c += 16) {
        double v[4];
#pragma unroll
        for (int t = 0; t < 4; t++) v[t] = gpart[(int64_t)(c + 4 * t) * nout + e];
#pragma unroll
        for (int t = 0; t < 4; t++) acc += v[t];
      }
      for (; c < nparts; c += 4) acc += gpart[(int64_t)c * nout + e];
    }
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
    if (e < nout && q == 0) {
      if (e < RR) S[e] = acc;
      else dS[e - RR] = acc;
    }
  } else {
    for (int64_t e = gt; e < nout; e += nthr) {
      // CTA partials in CTA order; 16 independent loads in flight per batch
      double acc = gpart[e];
      unsigned c = 1;
      for (; c + 16 <= nparts; c += 16) {
        double v[16];
#pragma unroll
        for (int q = 0; q < 16; q++) v[q] = gpart[(int64_t)(c + q) * nout + e];
#pragma unroll
        for (int q = 0; q < 16; q++) acc += v[q];
      }
      for (; c < nparts; c++) acc += gpart[(int64_t)c * nout + e];
      if (e < RR) S[e] = acc;
      else dS[e - RR] = acc;
    }
  }
  if (t0 >= 0 && t0 < 3) {
    double s = part[t0];
    for (unsigned b = 1; b < nparts; b++) s += part[b * 3 + t0];
    if (t0 == 0) *o_dA2 = s;
    if (t0 == 1) *o_A2 = s;
    if (t0 == 2 && o_MA) *o_MA = s;
  }
}

template <int U, bool SPLIT>
__global__ void __launch_bounds__(UPD_THREADS)
    update_fused_kernel(int R, int64_t rows, const double* __restrict__ Gi, const double* __restrict__ W,
                        double* __restrict__ M, double* __restrict__ A, const double* __restrict__ base,
                        double* __restrict__ dA, double* __restrict__ S, double* __restrict__ dS,
                        double* __restrict__ part, double* __restrict__ gpart, int RB,
                        double* __restrict__ o_dA2, double* __restrict__ o_A2, double* __restrict__ o_MA,
                        const int* __restrict__ st_src, int* __restrict__ st_dst,
                        const double* __restrict__ S_all, const double* __restrict__ dS_all, int N, int nmode,
                        int* __restrict__ st_local, MPending pend, int shfl) {
  extern __shared__ double sm[];
  double* G = sm;                 // R x R: Γ^{-1}
  double* Ws = sm + R * R;        // R x R (PP only)
  double* Xs = Ws + (W ? R * R : 0);  // RB x R: this CTA's new rows
  double* Ds = Xs + RB * R;           // RB x R: their dA
  // DMMA row phase: y (and a_old) of the CTA's rows, RBp = RB rounded up to 8, row stride LDY
  const int RBp = (RB + 7) & ~7, Rq = (R + 7) & ~7, LDY = Rq + 4;
  double* Ys = Ds + RB * R;           // RBp x LDY
  double* Ao = Ys + RBp * LDY;        // RBp x LDY
  __shared__ double red[3][UPD_THREADS / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // the side stream's SPD verdict for this Γ^{-1}, handed to the main stream's status slot
  if (st_dst && blockIdx.x == 0 && tid == 0) *st_dst = *st_src;
  if constexpr (U != 1) {
    fill_smem(G, Gi, R * R, tid);
    if (W) fill_smem(Ws, W, R * R, tid);
  } else if (S_all) {
    // R <= 32: Γ^{(n)} = ∗_{k≠n} S^(k) (Eq. 1) and its inverse formed here by warp 0 (gj32_warp),
    // and for PP W^(n) of Eq. 7 by the other warps -- no side-stream launches on the chain
    const int64_t RR = (int64_t)R * R;
    if (warp == 0) {
      double col[32];
      bool bad = false;
#pragma unroll
      for (int i = 0; i < 32; i++) {
        double g = (i == lane) ? 1.0 : 0.0;
        if (i < R && lane < R) {
          bool first = true;
          for (int k = 0; k < N; k++) {
            if (k == nmode) continue;
            const double sv = S_all[k * RR + i * R + lane];
            g = first ? sv : g * sv;
            first = false;
          }
        }
        col[i] = g;
      }
      gj32_warp(col, lane, bad);
#pragma unroll
      for (int i = 0; i < 32; i++)
        if (i < R && lane < R) G[i * R + lane] = col[i];
      const unsigned any_bad = __ballot_sync(0xffffffffu, bad);
      if (st_local && blockIdx.x == 0 && lane == 0) *st_local = any_bad ? 1 : 0;
    } else if (W) {
      for (int64_t e = tid - 32; e < RR; e += UPD_THREADS - 32) {  // pp_w_kernel's arithmetic
        double w = 0.0;
        for (int i = 0; i < N; i++) {
          if (i == nmode) continue;
          for (int j = i + 1; j < N; j++) {
            if (j == nmode) continue;
            double term = dS_all[i * RR + e] * dS_all[j * RR + e];
            for (int k = 0; k < N; k++)
              if (k != i && k != j && k != nmode) term *= S_all[k * RR + e];
            w += term;
          }
        }
        Ws[e] = w;
      }
    }
  } else {
    fill_smem(G, Gi, R * R, tid);
    if (W) fill_smem(Ws, W, R * R, tid);
  }
  __syncthreads();

  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  // this CTA owns rows [r0, r0 + RB); warp w solves rows r0 + w, r0 + w + 8, ...
  const int64_t r0 = (int64_t)blockIdx.x * RB;
  const int nrows = (int)max((int64_t)0, min((int64_t)RB, rows - r0));
  if (!shfl) {
    // Row phase on the FP64 tensor cores: the CTA's rows are m8 tiles, (M [+ A_old W]) Γ^{-1} as two small
    // GEMMs of mma.m8n8k4.f64 (one warp per 8 x 8 output tile, k in steps of 4), then the elementwise
    // dA / statistics / writes.  (CPD_UPD_SHFL: the warp-per-row shuffle mat-vecs below.)
    const int fr = lane >> 2, fc = lane & 3;
    for (int e = tid; e < RBp * Rq; e += UPD_THREADS) {
      const int lr = e / Rq, c = e - lr * Rq;
      double y = 0.0, ao = 0.0;
      if (lr < nrows && c < R) {
        const int64_t g = (r0 + lr) * R + c;
        if (pend.slots > 0) {  // the mTTV's K-split reduction, in mttv_reduce_kernel's order
          double sv = pend.base ? pend.base[g] : (pend.beta ? M[g] : 0.0);
          for (int k = 0; k < pend.slots; k++) sv += pend.ws[k * pend.n + g];
          y = sv;
          if (!W) M[g] = sv;
        } else {
          y = M[g];
        }
        ao = A[g];
      }
      Ys[lr * LDY + c] = y;
      Ao[lr * LDY + c] = ao;
    }
    __syncthreads();
    const int nt = (RBp / 8) * (Rq / 8);
    // C(8x8 tile) += X(rows, k) Mat(k, cols) over k < R; X from shared memory (stride LDY), Mat R x R
    auto tile_mma = [&](const double* X, const double* Mat, int m0, int n0, double& c0, double& c1) {
      for (int k0 = 0; k0 < R; k0 += 4) {
        const int k = k0 + fc;
        const double a = k < R ? X[(m0 + fr) * LDY + k] : 0.0;
        const double b = (k < R && n0 + fr < R) ? Mat[k * R + n0 + fr] : 0.0;
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c0), "+d"(c1)
                     : "d"(a), "d"(b));
      }
    };
    if (W) {  // y += a_old W (Eq. 7's V), written back so M~ = M_p + ΣU + V stays readable
      for (int t = warp; t < nt; t += UPD_THREADS / 32) {
        const int m0 = (t / (Rq / 8)) * 8, n0 = (t % (Rq / 8)) * 8;
        const int lr = m0 + fr, c = n0 + 2 * fc;
        double c0 = Ys[lr * LDY + c], c1 = Ys[lr * LDY + c + 1];
        tile_mma(Ao, Ws, m0, n0, c0, c1);
        __syncwarp();
        Ys[lr * LDY + c] = c0;
        Ys[lr * LDY + c + 1] = c1;
        if (lr < nrows) {
          if (c < R) M[(r0 + lr) * R + c] = c0;
          if (c + 1 < R) M[(r0 + lr) * R + c + 1] = c1;
        }
      }
      __syncthreads();
    }
    // x = y Γ^{-1} into Xs
    for (int t = warp; t < nt; t += UPD_THREADS / 32) {
      const int m0 = (t / (Rq / 8)) * 8, n0 = (t % (Rq / 8)) * 8;
      double c0 = 0.0, c1 = 0.0;
      tile_mma(Ys, G, m0, n0, c0, c1);
      const int lr = m0 + fr, c = n0 + 2 * fc;
      if (lr < nrows) {
        if (c < R) Xs[lr * R + c] = c0;
        if (c + 1 < R) Xs[lr * R + c + 1] = c1;
      }
    }
    __syncthreads();
    for (int e = tid; e < nrows * R; e += UPD_THREADS) {
      const int lr = e / R, c = e - lr * R;
      const int64_t g = (r0 + lr) * R + c;
      const double x = Xs[e];
      const double b = base ? base[g] : Ao[lr * LDY + c];
      const double d = x - b;
      A[g] = x;
      dA[g] = d;
      Ds[e] = d;
      s0 = fma(d, d, s0);
      s1 = fma(x, x, s1);
      s2 = fma(Ys[lr * LDY + c], x, s2);
    }
  }
  for (int lr = warp; shfl && lr < nrows; lr += UPD_THREADS / 32) {
    const int64_t i = r0 + lr;
    double y[U], ao[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int c = lane + 32 * u;
      if (pend.slots > 0 && c < R) {
        // the mTTV's K-split reduction, in mttv_reduce_kernel's order, then M~ materialised
        const int64_t e = i * R + c;
        double s = pend.base ? pend.base[e] : (pend.beta ? M[e] : 0.0);
        for (int k = 0; k < pend.slots; k++) s += pend.ws[k * pend.n + e];
        y[u] = s;
        if (!W) M[e] = s;
      } else {
        y[u] = c < R ? M[i * R + c] : 0.0;
      }
      ao[u] = c < R ? A[i * R + c] : 0.0;
    }
    if (W) {  // y += a_old W
      double v[U];
      rowvec_mat<U>(ao, Ws, R, lane, v);
#pragma unroll
      for (int u = 0; u < U; u++) {
        y[u] += v[u];
        const int c = lane + 32 * u;
        if (c < R) M[i * R + c] = y[u];  // keep M~ = M_p + ΣU + V readable (cpd_get_last_mttkrp)
      }
    }
    double mm[U];
#pragma unroll
    for (int u = 0; u < U; u++) mm[u] = y[u];
    // x = y Γ^{-1}: lanes own output columns, y_k broadcast by shuffles (independent FMAs)
    double x[U];
    rowvec_mat<U>(y, G, R, lane, x);
#pragma unroll
    for (int u = 0; u < U; u++) y[u] = x[u];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int c = lane + 32 * u;
      if (c < R) {
        const double b = base ? base[i * R + c] : ao[u];
        const double d = y[u] - b;
        A[i * R + c] = y[u];
        dA[i * R + c] = d;
        Xs[lr * R + c] = y[u];
        Ds[lr * R + c] = d;
        s0 = fma(d, d, s0);
        s1 = fma(y[u], y[u], s1);
        s2 = fma(mm[u], y[u], s2);
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    s0 += __shfl_xor_sync(0xffffffffu, s0, o);
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
  }
  if (lane == 0) {
    red[0][warp] = s0;
    red[1][warp] = s1;
    red[2][warp] = s2;
  }
  __syncthreads();
  if (tid < 3) {
    double s = red[tid][0];
    for (int w = 1; w < UPD_THREADS / 32; w++) s += red[tid][w];
    part[blockIdx.x * 3 + tid] = s;
  }
  // phase 2a: this CTA's partial Grams over its rows (ascending), from shared memory
  const int64_t RR = (int64_t)R * R;
  const int64_t nout = S ? (dS ? 2 * RR : RR) : 0;
  __syncthreads();
  // (a, b) of output e = tid + UPD_THREADS j stepped incrementally (one division per thread: the
  // per-element e / R was ~14 % of the kernel's stall samples at R = 100)
  {
    const int step_a = UPD_THREADS / R, step_b = UPD_THREADS - step_a * R;
    int a = tid / R, b = tid - (tid / R) * R;  // for f = e mod RR; a runs past R into the dS half
    for (int64_t e = tid; e < nout; e += UPD_THREADS) {
      const bool second = a >= R;
      const double* Y = second ? Ds : Xs;
      const int aa = second ? a - R : a;
      double acc = 0.0;
#pragma unroll 8
      for (int r = 0; r < nrows; r++) acc = fma(Xs[r * R + aa], Y[r * R + b], acc);
      gpart[(int64_t)blockIdx.x * nout + e] = acc;
      a += step_a;
      b += step_b;
      if (b >= R) {
        b -= R;
        a++;
      }
    }
  }
  if constexpr (SPLIT) return;  // phase 2b in update_reduce_kernel (a second, ordinary launch)
  cg::this_grid().sync();
  reduce_partials(gpart, part, gridDim.x, nout, RR, (int64_t)blockIdx.x * UPD_THREADS + tid,
                  (int64_t)gridDim.x * UPD_THREADS, blockIdx.x == 0 ? tid : -1, S, dS, o_dA2, o_A2, o_MA);
}

__global__ void __launch_bounds__(UPD_THREADS)
    update_reduce_kernel(const double* __restrict__ gpart, const double* __restrict__ part, unsigned nparts,
                         int64_t nout, int64_t RR, double* __restrict__ S, double* __restrict__ dS,
                         double* __restrict__ o_dA2, double* __restrict__ o_A2, double* __restrict__ o_MA) {
  reduce_partials(gpart, part, nparts, nout, RR, (int64_t)blockIdx.x * UPD_THREADS + threadIdx.x,
                  (int64_t)gridDim.x * UPD_THREADS, blockIdx.x == 0 ? (int)threadIdx.x : -1, S, dS, o_dA2, o_A2,
                  o_MA);
}


// SPLIT (experiment switch CPD_UPD_SPLIT): the row phase as an ordinary launch (its CTAs start as SMs
// free up, no co-residency, no grid barrier) and the partial-sum reduction as a second launch
template <int U>
cudaError_t coop_launch(int blocks, size_t smem, void** args, cudaStream_t st, bool split) {
  static bool attr = false, attr_s = false;  // per instantiation
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(update_fused_kernel<U, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         227 * 1024 - 2048);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  if (!attr_s) {
    cudaError_t e = cudaFuncSetAttribute(update_fused_kernel<U, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         227 * 1024 - 2048);
    if (e != cudaSuccess) return e;
    attr_s = true;
  }
  g_launches++;
  if (!split)
    return cudaLaunchCooperativeKernel((void*)update_fused_kernel<U, false>, blocks, UPD_THREADS, args, smem, st);
  return cudaLaunchKernel((void*)update_fused_kernel<U, true>, blocks, UPD_THREADS, args, smem, st);
}

}  // namespace

size_t update_fused_smem(int R, bool pp, int RB) {
  // Γ^{-1}, W (PP), this CTA's rows and their dA, the DMMA row phase's y and a_old tiles
  const size_t RBp = (RB + 7) & ~7, LDY = ((R + 7) & ~7) + 4;
  return sizeof(double) * ((size_t)R * R + (pp ? (size_t)R * R : 0) + 2 * (size_t)RB * R + 2 * RBp * LDY);
}

int update_fused_blocks(int64_t rows) {
  // experiment switch CPD_UPD_BLOCKS: cap on the cooperative grid (fewer CTAs: less Γ^-1 / W staging
  // and fewer Gram partials, and fewer SMs to wait for while filler-stream kernels occupy the GPU)
  static const int cap = getenv("CPD_UPD_BLOCKS") ? std::max(1, std::min(kUpdMaxBlocks, atoi(getenv("CPD_UPD_BLOCKS"))))
                                                  : kUpdMaxBlocks;
  return (int)std::min<int64_t>(cap, (rows + 7) / 8);
}

cudaError_t launch_update_fused(int R, int64_t rows, const double* Ginv, const double* W, double* M, double* A,
                                const double* base, double* dA, double* S, double* dS, double* part, double* gpart,
                                double* o_dA2, double* o_A2, double* o_MA, const int* st_src, int* st_dst,
                                cudaStream_t st, const double* S_all, const double* dS_all, int N, int nmode,
                                int* st_local, const MPending* pendp) {
  if (S_all && R > 32) return cudaErrorInvalidValue;
  MPending pend = pendp ? *pendp : MPending{};
  static int shfl = getenv("CPD_UPD_SHFL") ? 1 : 0;  // experiment switch: the warp-per-row shuffle row phase
  if (R > kUpdMaxR || rows <= 0) return cudaErrorInvalidValue;
  const int blocks = update_fused_blocks(rows);
  int RB = (int)((rows + blocks - 1) / blocks);
  const size_t smem = update_fused_smem(R, W != nullptr, RB);
  if (smem > 227 * 1024 - 2048) return cudaErrorInvalidValue;
  void* args[] = {&R,     &rows,   &Ginv,   &W,      &M,      &A,    &base,  &dA,    &S,       &dS,
                  &part,  &gpart,  &RB,     &o_dA2,  &o_A2,   &o_MA, &st_src, &st_dst, &S_all, &dS_all,
                  &N,     &nmode,  &st_local, &pend, &shfl};
  static const bool split = getenv("CPD_UPD_SPLIT") != nullptr;
  cudaError_t e = cudaErrorInvalidValue;
  switch ((R + 31) / 32) {
    case 1: e = coop_launch<1>(blocks, smem, args, st, split); break;
    case 2: e = coop_launch<2>(blocks, smem, args, st, split); break;
    case 3: e = coop_launch<3>(blocks, smem, args, st, split); break;
    case 4: e = coop_launch<4>(blocks, smem, args, st, split); break;
    case 5: e = coop_launch<5>(blocks, smem, args, st, split); break;
  }
  if (e != cudaSuccess || !split) return e;
  const int64_t RR = (int64_t)R * R;
  const int64_t nout = S ? (dS ? 2 * RR : RR) : 0;
  int64_t rb = (4 * nout + UPD_THREADS - 1) / UPD_THREADS;
  if (rb < 1) rb = 1;
  if (rb > 4 * kUpdMaxBlocks) rb = 4 * kUpdMaxBlocks;
  g_launches++;
  update_reduce_kernel<<<(unsigned)rb, UPD_THREADS, 0, st>>>(gpart, part, (unsigned)blocks, nout, RR, S, dS, o_dA2,
                                                             o_A2, o_MA);
  return cudaGetLastError();
}

}  // namespace cpd
