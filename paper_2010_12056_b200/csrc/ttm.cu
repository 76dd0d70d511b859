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
//
// Default staging (ttm_dmma_tma_kernel; aligned shapes): the T and factor tiles arrive by TMA
// (cp.async.bulk.tensor, 128-byte swizzle, 16-double-wide boxes, out-of-range rows / k / columns
// zero-filled by the copy engine) on full/empty mbarriers, issued by warp 0; the fragment rows and
// columns a lane owns are permuted so that the swizzled tiles are read without bank conflicts.
// The cp.async kernel below serves the unaligned shapes (odd K / ncols / post, small post % 16 != 0, tiny tensors)
// and CPD_DMMA_NO_TMA=1.
#include <cuda.h>
#include <cudaTypedefs.h>

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


// ---------------------------------------------------------------------------------------------
// TMA-staged variant.  Shared-memory stage = A boxes then B boxes, every box [rows][16 doubles]
// with the 128-byte swizzle (16-byte chunk c of row r stored at chunk c ^ (r & 7)):
//   KC (post == 1): BK/16 boxes [BM tile rows][16 k]    of the 2-D map {K, Mrows}
//   MC (post  > 1): BM/16 boxes [BK k][16 m]            of the 3-D map {post, K, pre}; tile rows in the
//                   padded row space i' = p*post16 + m, so a box never straddles two p
//   B:              ceil(BN/16) boxes [BK k][16 n]      of the 2-D map {ncols, K}
// A DMMA step uses k = kk..kk+3 (lane t -> k = kk + t).  Which tile row is "fragment row g" and
// which column is "fragment column g" is free as long as the epilogue stores to the same places:
//   KC rows   r = 16 w + 2 g + h              (h = lo / hi fragment of warp w)
//   MC rows   m = 16 w + 8 g1 + 4 h + 2 g2 + g0
//   columns   n = 16 (f>>1) + 8 g1 + 4 (f&1) + 2 g2 + g0   (fragment pair f, f^1 = one 16-column box;
//             the odd last fragment of an odd NF keeps n = 16 (f>>1) + g)
// With these a half-warp (g < 4 or g >= 4, all t) touches 16 distinct 8-byte banks and the two
// half-warps pair up on them: two wavefronts per 64-bit fragment load, the minimum.
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE_%=;\nbra WAIT_%=;\nDONE_%=:\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_2d(uint32_t dst, const CUtensorMap* tm, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(dst), "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_3d(uint32_t dst, const CUtensorMap* tm, int c0, int c1, int c2, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(dst), "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}

template <int NF, bool O3 = false>
struct SmemT {
  using S = Smem<NF>;
  // O3 (NF 9..14, e.g. R = 100, 200: NF = 13; grids of several waves): 3 stages and 3 CTAs/SM = 12 warps/SM
  // (4 stages x 2 CTAs = 8 warps/SM left the DMMA pipe 87 % active on C5).  Small grids (the R x R update
  // GEMMs) keep the 4-stage configuration: they are latency-bound and measured slower with 3 stages.
  static constexpr bool OCC3 = O3 && NF > 8 && NF <= 14;
  static constexpr int BK = S::BK, BM = S::BM, THREADS = S::THREADS;
  static constexpr int STAGES = OCC3 ? 3 : S::STAGES;
  static constexpr int MIN_BLOCKS = OCC3 ? 3 : S::MIN_BLOCKS;
  static constexpr int NB16 = (8 * NF + 15) / 16;        // B boxes per stage
  static constexpr int A_BYTES = BM * BK * 8;
  static constexpr int BBOX_BYTES = BK * 128;
  static constexpr int STAGE_BYTES = A_BYTES + NB16 * BBOX_BYTES;  // a multiple of 1024
  static constexpr size_t BYTES = (size_t)STAGE_BYTES * STAGES + 1024 /* alignment slack */ + 16 * STAGES;
};

template <int NF, bool MC, bool O3>
__global__ void __launch_bounds__(SmemT<NF, O3>::THREADS, SmemT<NF, O3>::MIN_BLOCKS)
    ttm_dmma_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                        int64_t pre, int64_t K, int64_t post, int64_t post16, int ncols, int ntiles_n,
                        double* __restrict__ out, int beta) {
  // MC: the tile rows live in a padded row space i' = p * post16 + m (post16 = post rounded up to 16), so a
  // 16-row box never straddles two p; rows m >= post are zero-filled by TMA and skipped by the epilogue
  using ST = SmemT<NF, O3>;
  constexpr int BK = ST::BK, BM = ST::BM, STAGES = ST::STAGES, BN = 8 * NF;
  constexpr int NWARPS = ST::THREADS / 32;
  constexpr int NA = MC ? BM / 16 : BK / 16;             // A boxes per stage
  constexpr int ABOX_BYTES = MC ? BK * 128 : BM * 128;
  constexpr int NFP = NF & ~1;                           // fragments with the paired column map
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw));
  const uint32_t base = (raw + 1023u) & ~1023u;                  // swizzle atoms are 1024-byte aligned
  const uint8_t* sbase = smem_raw + (base - raw);                // the same place, for the fragment loads
  const uint32_t full0 = base + ST::STAGE_BYTES * STAGES, empty0 = full0 + 8 * STAGES;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int g0 = g & 1, g1 = (g >> 1) & 1, g2 = g >> 2;

  const int64_t Mrows = pre * (MC ? post16 : post);
  const int64_t mtile = blockIdx.x / ntiles_n;
  const int ntile = blockIdx.x % ntiles_n;
  const int64_t i0 = mtile * BM;
  const int n0 = ntile * BN;
  const int nk = (int)((K + BK - 1) / BK);

  if (tid == 0) {
    for (int s = 0; s < STAGES; s++) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, NWARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // warp 0: lane l < NA + NB16 issues box l of stage kt
  auto issue = [&](int kt) {
    const int slot = kt % STAGES;
    const uint32_t bar = full0 + 8 * slot, dst = base + slot * ST::STAGE_BYTES;
    if (kt >= STAGES) mbar_wait(empty0 + 8 * slot, ((kt / STAGES) - 1) & 1);
    if (lane == 0) mbar_arrive_expect_tx(bar, ST::STAGE_BYTES);
    __syncwarp();
    const int k0 = kt * BK;
    if (lane < NA) {
      if constexpr (!MC) {
        tma_2d(dst + lane * ABOX_BYTES, &tmA, k0 + 16 * lane, (int)i0, bar);
      } else {
        const int64_t i = i0 + 16 * lane;
        const int64_t p = i / post16;
        tma_3d(dst + lane * ABOX_BYTES, &tmA, (int)(i - p * post16), k0, (int)p, bar);
      }
    } else if (lane < NA + ST::NB16) {
      const int j = lane - NA;
      tma_2d(dst + ST::A_BYTES + j * ST::BBOX_BYTES, &tmB, n0 + 16 * j, k0, bar);
    }
  };

  double acc[2][NF][2];
#pragma unroll
  for (int h = 0; h < 2; h++)
#pragma unroll
    for (int f = 0; f < NF; f++) acc[h][f][0] = acc[h][f][1] = 0.0;

  if (warp == 0)
    for (int s = 0; s < STAGES - 1 && s < nk; s++) issue(s);

  // per-thread parts of the swizzled fragment addresses (bytes inside a box)
  //   KC A: row r = 16 w + 2 g + h, k = kk + t: chunk ((kk & 15) >> 1) + (t >> 1), half t & 1
  //   MC A / B: row k = kk + t (k & 7 = (kk & 4) + t), 16-byte chunk of the column, half g0
  const uint32_t a_kc = (uint32_t)((16 * warp + 2 * g) * 128 + ((t & 1) << 3));
  const uint32_t rk = (uint32_t)(t * 128 + (g0 << 3));

  for (int kt = 0; kt < nk; kt++) {
    if (warp == 0 && kt + STAGES - 1 < nk) issue(kt + STAGES - 1);
    const int slot = kt % STAGES;
    mbar_wait(full0 + 8 * slot, (kt / STAGES) & 1);
    const uint8_t* As = sbase + slot * ST::STAGE_BYTES;
    const uint8_t* Bs = As + ST::A_BYTES;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double a[2];
#pragma unroll
      for (int h = 0; h < 2; h++) {
        uint32_t ad;
        if constexpr (!MC) {
          const uint32_t chunk = (uint32_t)((((kk & 15) >> 1) + (t >> 1)) ^ ((2 * g + h) & 7));
          ad = (kk >> 4) * ABOX_BYTES + a_kc + h * 128 + (chunk << 4);
        } else {
          const uint32_t chunk = (uint32_t)((4 * g1 + 2 * h + g2) ^ ((kk & 4) + t));
          ad = warp * ABOX_BYTES + kk * 128 + rk + (chunk << 4);
        }
        a[h] = *reinterpret_cast<const double*>(As + ad);
      }
      double b[NF];
#pragma unroll
      for (int f = 0; f < NF; f++) {
        const uint32_t cn = f < NFP ? (uint32_t)(4 * g1 + 2 * (f & 1) + g2) : (uint32_t)(g >> 1);
        const uint32_t chunk = cn ^ (uint32_t)((kk & 4) + t);
        const uint32_t ad = (f >> 1) * ST::BBOX_BYTES + kk * 128 + rk + (chunk << 4);
        b[f] = *reinterpret_cast<const double*>(Bs + ad);
      }
#pragma unroll
      for (int f = 0; f < NF; f++) {
        dmma(acc[0][f][0], acc[0][f][1], a[0], b[f]);
        dmma(acc[1][f][0], acc[1][f][1], a[1], b[f]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty0 + 8 * slot);
  }

  // ---- epilogue: the lane's rows (h = 0, 1) and column pairs under the permuted maps ----
#pragma unroll
  for (int h = 0; h < 2; h++) {
    const int rloc = MC ? 16 * warp + 8 * g1 + 4 * h + 2 * g2 + g0 : 16 * warp + 2 * g + h;
    int64_t i = i0 + rloc;
    if (i >= Mrows) continue;
    if constexpr (MC) {
      const int64_t p = i / post16, m = i - p * post16;
      if (m >= post) continue;
      i = p * post + m;
    }
    double* orow = out + i * ncols;
#pragma unroll
    for (int f = 0; f < NF; f++) {
      const int n = n0 + 16 * (f >> 1) + (f < NFP ? 8 * (t & 1) + 4 * (f & 1) + 2 * (t >> 1) : 2 * t);
      double v0 = acc[h][f][0], v1 = acc[h][f][1];
      if (n + 1 < ncols) {  // ncols even: n, n + 1 both valid, 16-byte aligned
        double2* p2 = reinterpret_cast<double2*>(orow + n);
        if (beta) {
          double2 o = *p2;
          v0 += o.x;
          v1 += o.y;
        }
        *p2 = make_double2(v0, v1);
      }
    }
  }
}

PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

template <int NF, bool MC, bool O3>
cudaError_t run_tma(const CUtensorMap& tmA, const CUtensorMap& tmB, int64_t grid, int64_t pre, int64_t K,
                    int64_t post, int64_t post16, int ncols, int ntiles_n, double* out, int beta, cudaStream_t st) {
  using ST = SmemT<NF, O3>;
  auto kern = ttm_dmma_tma_kernel<NF, MC, O3>;
  static bool attr_set = false;  // per instantiation
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ST::BYTES);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  g_launches++;
  kern<<<(unsigned)grid, ST::THREADS, ST::BYTES, st>>>(tmA, tmB, pre, K, post, post16, ncols, ntiles_n, out, beta);
  return cudaGetLastError();
}

// returns cudaErrorNotSupported when the shape does not qualify (the caller falls back to cp.async)
template <int NF>
cudaError_t launch_tma(const double* X, int64_t pre, int64_t K, int64_t post, const double* B, int ncols,
                       int ntiles_n, double* out, int beta, cudaStream_t st) {
  using ST = SmemT<NF>;
  static const bool off = getenv("CPD_DMMA_NO_TMA") && atoi(getenv("CPD_DMMA_NO_TMA"));
  const bool mc = post > 1;
  const int64_t post16 = (post + 15) / 16 * 16;
  const int64_t Mrows = pre * (mc ? post16 : post);  // MC: padded row space (see the kernel)
  if (off || (ncols & 1) || ncols < 16 || K < ST::BK || Mrows < ST::BM || Mrows > 0x7fffffff ||
      K > 0x7fffffff || (reinterpret_cast<uintptr_t>(X) & 15) || (reinterpret_cast<uintptr_t>(B) & 15) ||
      (reinterpret_cast<uintptr_t>(out) & 15))
    return cudaErrorNotSupported;
  // TMA strides are multiples of 16 bytes; MC rows padded per p to 16: at most 25 % zero rows
  if (mc ? ((post & 1) || (post % 16 != 0 && post < 64)) : (K % 2 != 0)) return cudaErrorNotSupported;
  auto enc = tmap_encoder();
  if (!enc) return cudaErrorNotSupported;
  CUtensorMap tmA, tmB;
  CUresult r;
  if (!mc) {
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)Mrows};
    cuuint64_t strides[1] = {(cuuint64_t)K * 8};
    cuuint32_t box[2] = {16, (cuuint32_t)ST::BM}, es[2] = {1, 1};
    r = enc(&tmA, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(X), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    cuuint64_t dims[3] = {(cuuint64_t)post, (cuuint64_t)K, (cuuint64_t)pre};
    cuuint64_t strides[2] = {(cuuint64_t)post * 8, (cuuint64_t)K * post * 8};
    cuuint32_t box[3] = {16, (cuuint32_t)ST::BK, 1}, es[3] = {1, 1, 1};
    r = enc(&tmA, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(X), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (r != CUDA_SUCCESS) return cudaErrorNotSupported;
  {
    cuuint64_t dims[2] = {(cuuint64_t)ncols, (cuuint64_t)K};
    cuuint64_t strides[1] = {(cuuint64_t)ncols * 8};
    cuuint32_t box[2] = {16, (cuuint32_t)ST::BK}, es[2] = {1, 1};
    r = enc(&tmB, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(B), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (r != CUDA_SUCCESS) return cudaErrorNotSupported;
  const int64_t grid = (Mrows + ST::BM - 1) / ST::BM * ntiles_n;
  if (grid > 0x7fffffff) return cudaErrorInvalidConfiguration;
  if constexpr (NF > 8 && NF <= 14) {
    static const bool no_occ3 = getenv("CPD_DMMA_NO_OCC3") && atoi(getenv("CPD_DMMA_NO_OCC3"));
    if (!no_occ3 && grid >= 4 * 148 * 3)  // several waves of 3 CTAs/SM
      return mc ? run_tma<NF, true, true>(tmA, tmB, grid, pre, K, post, post16, ncols, ntiles_n, out, beta, st)
                : run_tma<NF, false, true>(tmA, tmB, grid, pre, K, post, post16, ncols, ntiles_n, out, beta, st);
  }
  return mc ? run_tma<NF, true, false>(tmA, tmB, grid, pre, K, post, post16, ncols, ntiles_n, out, beta, st)
            : run_tma<NF, false, false>(tmA, tmB, grid, pre, K, post, post16, ncols, ntiles_n, out, beta, st);
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
  {
    cudaError_t e = launch_tma<NF>(X, pre, K, post, B, ncols, ntiles_n, out, beta, st);
    if (e != cudaErrorNotSupported) return e;
  }
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
  // N tiles of at most maxnf 8-column fragments (CPD_DMMA_MAXNF, experiment switch; default CPD_TTM_MAXNF)
  static const int maxnf = [] {
    int v = getenv("CPD_DMMA_MAXNF") ? atoi(getenv("CPD_DMMA_MAXNF")) : CPD_TTM_MAXNF;
    return v < 1 ? 1 : (v > 16 ? 16 : v);
  }();
  int nf_total = (ncols + 7) / 8;
  int ntiles = (nf_total + maxnf - 1) / maxnf;
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
