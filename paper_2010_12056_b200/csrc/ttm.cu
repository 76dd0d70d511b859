// First-level TTM of the (multi-sweep) dimension tree on FP64 tensor cores.
//
// P:320-322 (§II-D): "The first level contractions (contractions between the input
// tensor and one factor matrix) are done via TTM ... generally the most time-consuming
// part of ALS"; "TTM is the major bottleneck".  Eq. 4 with one
// contracted mode j:  M^({1..N}\j)(..., r) = Σ_{i_j} T(..., i_j, ...) A^(j)(i_j, r).
//
// B200 design: FP64 has no tcgen05 kind on sm_100a; the FP64
// tensor path is the warp-level DMMA (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4), measured
// at 37.1 TFLOP/s = 148 SM x 128 flop/clk x 1.965 GHz (profiles/r01_peaks_fp64.json).
// T is viewed as [pre, K, post]; the GEMM rows i = (p, m) are either K-contiguous
// (post == 1, contract the last kept mode) or M-contiguous (post > 1, contract a
// leading/middle mode -- a batched GEMM over p with no transposed copy of T, unlike the
// paper's stored transposes).  Each CTA owns a 128-row M tile and BN = 8*NF
// columns of R (whole R when R <= 128), so T streams from HBM once; a 4-stage cp.async
// pipeline stages T and factor tiles in padded shared memory (conflict-free 64-bit
// fragment loads), 8 warps each issue 2*NF independent DMMAs per k4 step.
#include "kernels.h"

namespace cpd {
namespace {


__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp16(void* dst, const void* src, bool valid) {
  // 16-byte async copy, L2 only (.cg); zero-fill when !valid
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
               "r"(valid ? 16 : 0));
}
__device__ __forceinline__ void cp8(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
               "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int NF>
struct Smem {
  // Tile shapes per accumulator width (measured on the BASELINE shapes, tools/bench_ttm.cu):
  //   NF <= 4 : BM  64, BK 32, 2 stages, 4 CTAs/SM  (short K, e.g. C4 K = 64: CTAs overlap)
  //   NF <= 8 : BM 128, BK 32, 2 stages, 2 CTAs/SM  (C2: 89 % of the DMMA peak)
  //   NF > 8  : BM  64, BK 16, 4 stages, 2 CTAs/SM  (> 128 registers per thread)
  static constexpr int BK = NF <= 8 ? 32 : 16;
  static constexpr int STAGES = NF <= 8 ? 2 : 4;
  static constexpr int BM = (NF <= 4 || NF > 8) ? 64 : 128;
  static constexpr int THREADS = 2 * BM;  // 16 rows per warp
  static constexpr int MIN_BLOCKS = NF <= 4 ? 4 : 2;
  static constexpr int LDA_MC = BM + 4;  // [BK][BM+4]: (t*LDA + g) mod 16 distinct
  static constexpr int LDA_KC = BK + 4;  // [BM][BK+4]: (g*LDA + t) mod 16 distinct for g,t < 4
  static constexpr int BN = 8 * NF;
  static constexpr int LDB = ((BN + 15) / 16) * 16 + 4;
  static constexpr int A_ELEMS = (BM * LDA_KC > BK * LDA_MC) ? BM * LDA_KC : BK * LDA_MC;
  static constexpr int B_ELEMS = BK * LDB;
  static constexpr int STAGE = A_ELEMS + B_ELEMS;
  static constexpr size_t BYTES = sizeof(double) * STAGE * STAGES;
};

// MC: post > 1 (M-contiguous rows); VEC2: 16-byte chunks (requires post even for MC,
// K even for KC, ncols even for B).
template <int NF, bool MC, bool VEC2, bool BVEC2>
__global__ void __launch_bounds__(Smem<NF>::THREADS, Smem<NF>::MIN_BLOCKS)
    ttm_dmma_kernel(const double* __restrict__ X, int64_t pre, int64_t K, int64_t post,
                    const double* __restrict__ B, int ncols, int ntiles_n,
                    double* __restrict__ out, int beta) {
  using S = Smem<NF>;
  constexpr int BN = S::BN;
  constexpr int STAGES = S::STAGES;
  constexpr int BK = S::BK;
  constexpr int LDA_KC = S::LDA_KC;
  constexpr int LDA_MC = S::LDA_MC;
  constexpr int BM = S::BM;
  constexpr int THREADS = S::THREADS;
  constexpr int HB = BM / 2;  // MC 16-byte chunks per k-row
  extern __shared__ __align__(16) double smem[];
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;

  const int64_t Mrows = pre * post;
  const int64_t mtile = blockIdx.x / ntiles_n;
  const int ntile = blockIdx.x % ntiles_n;
  const int64_t i0 = mtile * BM;
  const int n0 = ntile * BN;
  const int64_t nk = (K + BK - 1) / BK;

  // ---- per-thread constant parts of the T addresses ----
  // KC: CPR chunks (k pairs, or single k) per row; thread: chunk tid%CPR, rows tid/CPR + RSTEP*q
  // MC: row pair 2*(tid%64) (or row tid%128), k-rows tid/64 + 4q (or tid/128 + 2q)
  constexpr int CPR = VEC2 ? BK / 2 : BK;
  constexpr int RSTEP = THREADS / CPR;
  constexpr int NQ = MC ? (VEC2 ? BK / (THREADS / HB) : BK / (THREADS / BM)) : BM / RSTEP;
  int64_t abase[MC ? 1 : NQ];
  bool arow_ok[MC ? 1 : NQ];
  if constexpr (!MC) {
#pragma unroll
    for (int q = 0; q < NQ; q++) {
      int r = tid / CPR + RSTEP * q;
      int64_t i = i0 + r;
      arow_ok[q] = i < Mrows;
      abase[q] = (arow_ok[q] ? i : 0) * K;
    }
  } else {
    int r = VEC2 ? 2 * (tid % HB) : (tid % BM);
    int64_t i = i0 + r;
    arow_ok[0] = i < Mrows;
    int64_t ii = arow_ok[0] ? i : 0;
    int64_t p = ii / post, m = ii - p * post;
    abase[0] = p * K * post + m;
  }

  auto load_stage = [&](int slot, int64_t kt) {
    double* As = smem + slot * S::STAGE;
    double* Bs = As + S::A_ELEMS;
    const int64_t k0 = kt * BK;
    if constexpr (!MC) {
#pragma unroll
      for (int q = 0; q < NQ; q++) {
        if constexpr (VEC2) {
          int r = tid / CPR + RSTEP * q, c = tid % CPR;
          int64_t k = k0 + 2 * c;
          bool ok = arow_ok[q] && k < K;
          cp16(As + r * LDA_KC + 2 * c, X + abase[q] + (ok ? k : 0), ok);
        } else {
          int r = tid / CPR + RSTEP * q, c = tid % CPR;
          int64_t k = k0 + c;
          bool ok = arow_ok[q] && k < K;
          cp8(As + r * LDA_KC + c, X + abase[q] + (ok ? k : 0), ok);
        }
      }
    } else {
#pragma unroll
      for (int q = 0; q < NQ; q++) {
        if constexpr (VEC2) {
          int y = tid / HB + (THREADS / HB) * q, c = tid % HB;
          int64_t k = k0 + y;
          bool ok = arow_ok[0] && k < K;
          cp16(As + y * LDA_MC + 2 * c, X + abase[0] + (ok ? k * post : 0), ok);
        } else {
          int y = tid / BM + (THREADS / BM) * q, c = tid % BM;
          int64_t k = k0 + y;
          bool ok = arow_ok[0] && k < K;
          cp8(As + y * LDA_MC + c, X + abase[0] + (ok ? k * post : 0), ok);
        }
      }
    }
    // B tile: BK x BN from B[k0.., n0..]
    if constexpr (BVEC2) {
      constexpr int BCPR = BN / 2;  // chunks per k-row
      for (int e = tid; e < BK * BCPR; e += THREADS) {
        int y = e / BCPR, c = e % BCPR;
        int64_t k = k0 + y;
        int n = n0 + 2 * c;
        bool ok = k < K && n < ncols;
        cp16(Bs + y * S::LDB + 2 * c, B + (ok ? k * ncols + n : 0), ok);
      }
    } else {
      for (int e = tid; e < BK * BN; e += THREADS) {
        int y = e / BN, c = e % BN;
        int64_t k = k0 + y;
        int n = n0 + c;
        bool ok = k < K && n < ncols;
        cp8(Bs + y * S::LDB + c, B + (ok ? k * ncols + n : 0), ok);
      }
    }
  };

  double acc[2][NF][2];
#pragma unroll
  for (int h = 0; h < 2; h++)
#pragma unroll
    for (int f = 0; f < NF; f++) acc[h][f][0] = acc[h][f][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; s++) {
    if (s < nk) load_stage(s, s);
    cp_commit();
  }

  const int wrow = warp * 16;
  for (int64_t kt = 0; kt < nk; kt++) {
    cp_wait<STAGES - 2>();
    __syncthreads();
    {
      int64_t nt = kt + STAGES - 1;
      if (nt < nk) load_stage((int)(nt % STAGES), nt);
      cp_commit();
    }
    const double* As = smem + (int)(kt % STAGES) * S::STAGE;
    const double* Bs = As + S::A_ELEMS;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double a_lo, a_hi;
      if constexpr (!MC) {
        a_lo = As[(wrow + g) * LDA_KC + kk + t];
        a_hi = As[(wrow + 8 + g) * LDA_KC + kk + t];
      } else {
        a_lo = As[(kk + t) * LDA_MC + wrow + g];
        a_hi = As[(kk + t) * LDA_MC + wrow + 8 + g];
      }
      double b[NF];
#pragma unroll
      for (int f = 0; f < NF; f++) b[f] = Bs[(kk + t) * S::LDB + 8 * f + g];
#pragma unroll
      for (int f = 0; f < NF; f++) {
        dmma(acc[0][f][0], acc[0][f][1], a_lo, b[f]);
        dmma(acc[1][f][0], acc[1][f][1], a_hi, b[f]);
      }
    }
  }
  cp_wait<0>();

  // ---- epilogue: rows wrow+g (+8), cols 8f + 2t, 2t+1 ----
#pragma unroll
  for (int h = 0; h < 2; h++) {
    int64_t i = i0 + wrow + 8 * h + g;
    if (i >= Mrows) continue;
    double* orow = out + i * ncols;
#pragma unroll
    for (int f = 0; f < NF; f++) {
      int n = n0 + 8 * f + 2 * t;
      double v0 = acc[h][f][0], v1 = acc[h][f][1];
      if (BVEC2 && n + 1 < ncols) {
        double2* p2 = reinterpret_cast<double2*>(orow + n);
        if (beta) {
          double2 o = *p2;
          v0 += o.x;
          v1 += o.y;
        }
        *p2 = make_double2(v0, v1);
      } else {
        if (n < ncols) orow[n] = beta ? orow[n] + v0 : v0;
        if (n + 1 < ncols) orow[n + 1] = beta ? orow[n + 1] + v1 : v1;
      }
    }
  }
}

template <int NF, bool MC, bool VEC2, bool BVEC2>
cudaError_t launch_nf(const double* X, int64_t pre, int64_t K, int64_t post, const double* B,
                      int ncols, int ntiles_n, double* out, int beta, cudaStream_t st) {
  auto kern = ttm_dmma_kernel<NF, MC, VEC2, BVEC2>;
  size_t smem = Smem<NF>::BYTES;
  static bool attr_set = false;  // per instantiation
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  constexpr int BM = Smem<NF>::BM;
  int64_t mt = (pre * post + BM - 1) / BM;
  int64_t grid = mt * ntiles_n;
  if (grid > 0x7fffffff) return cudaErrorInvalidConfiguration;
  g_launches++;
  kern<<<(unsigned)grid, Smem<NF>::THREADS, smem, st>>>(X, pre, K, post, B, ncols, ntiles_n, out, beta);
  return cudaGetLastError();
}

template <int NF>
cudaError_t dispatch_layout(const double* X, int64_t pre, int64_t K, int64_t post, const double* B,
                            int ncols, int ntiles_n, double* out, int beta, cudaStream_t st) {
  const bool mc = post > 1;
  const bool bvec = (ncols % 2) == 0;
  const bool avec = mc ? (post % 2) == 0 : (K % 2) == 0;
#define CPD_TTM_CASE(MC_, V_, BV_)                                                          \
  if (mc == MC_ && avec == V_ && bvec == BV_)                                               \
    return launch_nf<NF, MC_, V_, BV_>(X, pre, K, post, B, ncols, ntiles_n, out, beta, st);
  CPD_TTM_CASE(false, true, true)
  CPD_TTM_CASE(false, true, false)
  CPD_TTM_CASE(false, false, true)
  CPD_TTM_CASE(false, false, false)
  CPD_TTM_CASE(true, true, true)
  CPD_TTM_CASE(true, true, false)
  CPD_TTM_CASE(true, false, true)
  CPD_TTM_CASE(true, false, false)
#undef CPD_TTM_CASE
  return cudaErrorInvalidValue;
}

}  // namespace

cudaError_t launch_ttm(const double* X, int64_t pre, int64_t K, int64_t post, const double* B,
                       int ncols, double* out, int beta, cudaStream_t st) {
  if (pre <= 0 || post <= 0 || ncols <= 0) return cudaSuccess;
  if (K <= 0) return cudaErrorInvalidValue;
#ifndef CPD_TTM_MAXNF
#define CPD_TTM_MAXNF 16
#endif
  int nf_total = (ncols + 7) / 8;
  int ntiles = (nf_total + CPD_TTM_MAXNF - 1) / CPD_TTM_MAXNF;
  int nf = (nf_total + ntiles - 1) / ntiles;
  switch (nf) {
    case 1: return dispatch_layout<1>(X, pre, K, post, B, ncols, ntiles, out, beta, st);
    case 2: return dispatch_layout<2>(X, pre, K, post, B, ncols, ntiles, out, beta, st);
    case 3: return dispatch_layout<3>(X, pre, K, post, B, ncols, ntiles, out, beta, st);
    case 4: return dispatch_layout<4>(X, pre, K, post, B, ncols, ntiles, out, beta, st);
    case 5: return dispatch_layout<5>(X, pre, K, post, B, ncols, ntiles, out, beta, st);
    case 6: return dispatch_layout<6>(X, pre, K, post, B, ncols, ntiles, out, beta, st);
    case 7: return dispatch_layout<7>(X, pre, K, post, B, ncols, ntiles, out, beta, st);
    case 8: return dispatch_layout<8>(X, pre, K, post, B, ncols, ntiles, out, beta, st);
    case 9: return dispatch_layout<9>(X, pre, K, post, B, ncols, ntiles, out, beta, st);
    case 10: return dispatch_layout<10>(X, pre, K, post, B, ncols, ntiles, out, beta, st);
    case 11: return dispatch_layout<11>(X, pre, K, post, B, ncols, ntiles, out, beta, st);
    case 12: return dispatch_layout<12>(X, pre, K, post, B, ncols, ntiles, out, beta, st);
    case 13: return dispatch_layout<13>(X, pre, K, post, B, ncols, ntiles, out, beta, st);
    case 14: return dispatch_layout<14>(X, pre, K, post, B, ncols, ntiles, out, beta, st);
    case 15: return dispatch_layout<15>(X, pre, K, post, B, ncols, ntiles, out, beta, st);
    case 16: return dispatch_layout<16>(X, pre, K, post, B, ncols, ntiles, out, beta, st);
  }
  return cudaErrorInvalidValue;
}


namespace {
__global__ void krp_block_kernel(KrpSpec sp, int R, double* __restrict__ out, int64_t total) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e % R);
    int64_t rest = e / R, row = 0;
    double v = 1.0;
    for (int c = sp.n - 1; c >= 0; c--) {  // last mode fastest
      const int64_t y = rest % sp.ext[c];
      rest /= sp.ext[c];
      row += y * sp.stride[c];
      v *= sp.A[c][y * R + r];
    }
    out[row * R + r] = v;
  }
}
}  // namespace

cudaError_t launch_krp_block(const KrpSpec& sp, int R, double* out, int64_t rows_total, bool pad, cudaStream_t st) {
  if (sp.n < 1 || sp.n > 8 || R < 1) return cudaErrorInvalidValue;
  int64_t total = R;
  for (int c = 0; c < sp.n; c++) total *= sp.ext[c];
  if (pad) {
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(double) * (size_t)rows_total * R, st);
    if (e != cudaSuccess) return e;
  }
  g_launches++;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
  krp_block_kernel<<<blocks, 256, 0, st>>>(sp, R, out, total);
  return cudaGetLastError();
}

}  // namespace cpd
