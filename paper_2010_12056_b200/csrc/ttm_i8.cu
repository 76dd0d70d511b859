// First-level TTM with FP64 operands on the 5th-generation INT8 tensor cores
// (tcgen05.mma kind::i8, TMEM accumulators): exact integer slicing of both operands.
//
// Operation (same as launch_ttm, Eq. 4 with one contracted mode):
//   out[i, c] = beta*out[i, c] + Σ_k X[addr(i, k)] B[k, c],  X viewed as [pre, K, post].
//
// Arithmetic (DESIGN.md §6 "K2i"):  with 2^eX > max|X| (one exponent for the whole tensor,
// computed once) and 2^F_c > max_k |B[k, c]| (per column),
//   x = X 2^(54-eX),  b = B 2^(54-F_c)  rounded to integers, |x|, |b| < 2^54,
// each written in 7 signed base-256 digits  x = Σ_{a=0..6} s_a 256^a,  s_a ∈ [-128, 127]
// (bias trick: the bytes of x + 0x0080808080808080, each xor 0x80).  Then
//   Σ_k x b = Σ_{a,b} 256^(a+b) Σ_k s^x_a s^b_b,
// the inner sums are exact int8 x int8 -> int32 tensor-core products, and the pairs with
// a + b >= 6 (28 of 49, the "diagonals" D_d, d = a + b - 6 = 0..6) are kept:
//   out = 2^(eX + F_c - 60) Σ_d D_d 256^d.
// Truncation: inputs to 54 bits below the tensor maximum, dropped pairs below 2^-46 of a
// single top-digit product -- a norm-wise error of the order of FP64 rounding for the
// workloads here (parity against the oracle at 1e-10 in tests/test_gpu_parity.py).
// int32 range: |D_d| <= 7 * 128^2 * K < 2^31 for K <= 16384 (launcher checks).
//
// Kernel: persistent, one CTA per SM (TMEM fully used: 7 diagonals x Rp columns).
//   warps 0-7  converters: cp.async FP64 tile rows -> smem ring (thread-private slots),
//              -> int64 -> 7 digit planes in the UMMA K-major canonical layout (no swizzle),
//              thread 0 also bulk-copies the pre-sliced B digits of the K step;
//   warp 8     TMEM allocator + single-thread MMA issuer: per K32 step, for a = 6..0,
//              D[0 .. a] += S^x_a · [S^b_{6-a} | ... | S^b_6]  (one MMA, N = (a+1) Rp,
//              split at 256): the concatenated B planes land on consecutive diagonals;
//   warps 9-12 epilogue: tcgen05.ld of the 7 diagonals, exact int64 partial recombination,
//              FP64 scale, 32-byte vector stores.
#include <algorithm>

#include "kernels.h"

namespace cpd {
namespace {

constexpr int kBM = 128;
constexpr int kND = 7;
constexpr int kDS = 3;                       // digit-plane stages
constexpr int kFS = 3;                       // FP64 staging stages
constexpr int kConv = 256;                   // converter threads
constexpr int kThreads = kConv + 32 + 128;
constexpr int kRpMax = 64;
constexpr int kAPlane = kBM * 32;            // bytes of one digit plane per K32 step
constexpr int kAStage = kND * kAPlane;       // 28672
constexpr int kBStage = kND * kRpMax * 32;   // 14336 (max)
constexpr int kDStage = kAStage + kBStage;
constexpr int kFStage = kConv * 16 * 8;      // 32768: 16 doubles per converter thread
constexpr int kSmemData = kDS * kDStage + kFS * kFStage;
constexpr int kSmem = kSmemData + 128;
constexpr uint64_t kBias = 0x0080808080808080ull;

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint32_t bar, uint32_t bytes) {
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
__device__ __forceinline__ void cp16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0));
}
__device__ __forceinline__ void cp8(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}
// 4x4 byte transpose: o[b] = (w0[b], w1[b], w2[b], w3[b])
__device__ __forceinline__ void transpose4(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3, uint32_t o[4]) {
  uint32_t t0 = prmt(w0, w1, 0x5140), t1 = prmt(w0, w1, 0x7362);
  uint32_t t2 = prmt(w2, w3, 0x5140), t3 = prmt(w2, w3, 0x7362);
  o[0] = prmt(t0, t2, 0x5410);
  o[1] = prmt(t0, t2, 0x7632);
  o[2] = prmt(t1, t3, 0x5410);
  o[3] = prmt(t1, t3, 0x7632);
}
// UMMA shared-memory descriptor, K-major, no swizzle: ((8,m),2):((16 B, sbo),lbo)
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
// instruction descriptor: kind::i8, D s32, A/B signed int8, both K-major, M = 128
__device__ __forceinline__ uint32_t idesc(int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(kBM >> 4) << 24);
}
__device__ __forceinline__ void mma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}
__device__ __forceinline__ double pow2(int e) {  // 2^e for normal range
  return __longlong_as_double((long long)(1023 + e) << 52);
}

struct Geo {
  int64_t pre, K, post, Mrows;
  int ncols, Rn, Rp, ntn;   // columns, columns per N tile, padded, number of N tiles
  int64_t nmt, ntiles;      // M tiles, total tiles
  int nkc;                  // K32 steps
};

template <bool MC, bool VEC>
__global__ void __launch_bounds__(kThreads, 1)
    ttm_i8_kernel(const double* __restrict__ X, Geo g, const uint8_t* __restrict__ Bimg,
                  const int* __restrict__ Fexp, const int* __restrict__ Xexp, double* __restrict__ out, int beta) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* dring = smem;                               // kDS digit stages
  uint8_t* fring = smem + kDS * kDStage;               // kFS FP64 stages
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kSmemData);
  const uint32_t full0 = su32(bars), empty0 = su32(bars + kDS);
  const uint32_t tfull = su32(bars + 2 * kDS), tempty = su32(bars + 2 * kDS + 1);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 2 * kDS + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int Bbytes = kND * g.Rp * 32;

  if (tid == 0) {
    for (int s = 0; s < kDS; s++) {
      mbar_init(full0 + 8 * s, kConv);
      mbar_init(empty0 + 8 * s, 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 128);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 8) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  const int64_t my_tiles = g.ntiles > blockIdx.x ? (g.ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t iters = my_tiles * g.nkc;

  if (warp < 8) {
    // ===================== converters =====================
    const int row = MC ? (tid & 127) : (tid >> 1);
    const int h = MC ? (tid >> 7) : (tid & 1);
    const double scale = pow2(54 - *Xexp);
    auto issue = [&](int64_t it) {
      const int fs = (int)(it % kFS);
      const uint32_t fb = su32(fring + fs * kFStage) + tid * 16;
      if (it < iters) {
        const int64_t tile = blockIdx.x + (it / g.nkc) * gridDim.x;
        const int kc = (int)(it % g.nkc);
        const int64_t mt = tile / g.ntn;
        const int64_t i = mt * kBM + row;
        const bool rok = i < g.Mrows;
        const int64_t k0 = (int64_t)kc * 32 + 16 * h;
        if constexpr (!MC) {
          const double* src = X + (rok ? i : 0) * g.K;
#pragma unroll
          for (int q = 0; q < 8; q++) {
            const int64_t k = k0 + 2 * q;
            if constexpr (VEC) {
              const bool ok = rok && k < g.K;  // K even: pairs never straddle the end
              cp16(fb + q * (kConv * 16), src + (ok ? k : 0), ok);
            } else {
              cp8(fb + q * (kConv * 16), src + (rok && k < g.K ? k : 0), rok && k < g.K);
              cp8(fb + q * (kConv * 16) + 8, src + (rok && k + 1 < g.K ? k + 1 : 0), rok && k + 1 < g.K);
            }
          }
        } else {
          const int64_t ii = rok ? i : 0;
          const int64_t p = ii / g.post, m = ii - p * g.post;
          const double* src = X + p * g.K * g.post + m;
#pragma unroll
          for (int q = 0; q < 16; q++) {
            const int64_t k = k0 + q;
            const bool ok = rok && k < g.K;
            cp8(fb + (q >> 1) * (kConv * 16) + (q & 1) * 8, src + (ok ? k * g.post : 0), ok);
          }
        }
      }
      cp_commit();
    };
#pragma unroll 1
    for (int q = 0; q < kFS - 1; q++) issue(q);
#pragma unroll 1
    for (int64_t it = 0; it < iters; it++) {
      issue(it + kFS - 1);
      cp_wait<kFS - 1>();
      const int fs = (int)(it % kFS);
      const double2* fp = reinterpret_cast<const double2*>(fring + fs * kFStage) + tid;
      uint32_t lo[16], hi[16];
#pragma unroll
      for (int q = 0; q < 8; q++) {
        const double2 v = fp[q * kConv];
        const long long a0 = __double2ll_rn(v.x * scale) + (long long)kBias;
        const long long a1 = __double2ll_rn(v.y * scale) + (long long)kBias;
        lo[2 * q] = (uint32_t)a0;
        hi[2 * q] = (uint32_t)((unsigned long long)a0 >> 32);
        lo[2 * q + 1] = (uint32_t)a1;
        hi[2 * q + 1] = (uint32_t)((unsigned long long)a1 >> 32);
      }
      const int s = (int)(it % kDS);
      const uint32_t round = (uint32_t)(it / kDS);
      mbar_wait(empty0 + 8 * s, (round & 1) ^ 1);
      uint8_t* st = dring + s * kDStage;
      // plane a, this thread's 16 k-bytes of row `row`, K half h
      const int off = (row >> 3) * 256 + h * 128 + (row & 7) * 16;
      uint32_t pl[8][4];
#pragma unroll
      for (int w = 0; w < 4; w++) {
        uint32_t o[4];
        transpose4(lo[4 * w], lo[4 * w + 1], lo[4 * w + 2], lo[4 * w + 3], o);
#pragma unroll
        for (int b = 0; b < 4; b++) pl[b][w] = o[b] ^ 0x80808080u;
        transpose4(hi[4 * w], hi[4 * w + 1], hi[4 * w + 2], hi[4 * w + 3], o);
#pragma unroll
        for (int b = 0; b < 4; b++) pl[4 + b][w] = o[b] ^ 0x80808080u;
      }
#pragma unroll
      for (int a = 0; a < kND; a++)
        *reinterpret_cast<uint4*>(st + a * kAPlane + off) = make_uint4(pl[a][0], pl[a][1], pl[a][2], pl[a][3]);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      if (tid == 0) {
        const int64_t tile = blockIdx.x + (it / g.nkc) * gridDim.x;
        const int nt = (int)(tile % g.ntn);
        const int kc = (int)(it % g.nkc);
        const uint8_t* src = Bimg + ((int64_t)nt * g.nkc + kc) * Bbytes;
        mbar_arrive_tx(full0 + 8 * s, Bbytes);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                su32(st + kAStage)),
            "l"(src), "r"(Bbytes), "r"(full0 + 8 * s)
            : "memory");
      } else {
        mbar_arrive(full0 + 8 * s);
      }
    }
    cp_wait<0>();
  } else if (warp == 8) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      int64_t it = 0;
      for (int64_t tt = 0; tt < my_tiles; tt++) {
        mbar_wait(tempty, ((uint32_t)tt & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        for (int kc = 0; kc < g.nkc; kc++, it++) {
          const int s = (int)(it % kDS);
          mbar_wait(full0 + 8 * s, (uint32_t)(it / kDS) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t abase = su32(dring + s * kDStage), bbase = abase + kAStage;
#pragma unroll 1
          for (int a = kND - 1; a >= 0; a--) {
            const uint32_t acc = (kc > 0 || a < kND - 1) ? 1u : 0u;
            const uint64_t ad = sdesc(abase + a * kAPlane, 128, 256);
            const int b0 = kND - 1 - a;  // first B plane: diagonal 0
            const int n = (a + 1) * g.Rp;
            const uint32_t bstart = bbase + b0 * g.Rp * 32;
            const int n1 = n > 256 ? 256 : n;
            mma_i8(tmem, ad, sdesc(bstart, 128, 256), idesc(n1), acc);
            if (n > 256) mma_i8(tmem + 256, ad, sdesc(bstart + 256 * 32, 128, 256), idesc(n - 256), acc);
          }
          mma_commit(empty0 + 8 * s);
        }
        mma_commit(tfull);
      }
    }
    __syncwarp();
  } else {
    // ===================== epilogue =====================
    const int q = warp & 3;  // TMEM lane quarter of this warp
    const int r = q * 32 + lane;
    const int ex = *Xexp;
    for (int64_t tt = 0; tt < my_tiles; tt++) {
      const int64_t tile = blockIdx.x + tt * gridDim.x;
      const int64_t mt = tile / g.ntn;
      const int nt = (int)(tile % g.ntn);
      const int64_t i = mt * kBM + r;
      const int n0 = nt * g.Rn;
      mbar_wait(tfull, (uint32_t)tt & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      for (int c0 = 0; c0 < g.Rp; c0 += 8) {
        uint32_t D[kND][8];
#pragma unroll
        for (int d = 0; d < kND; d++) {
          const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + d * g.Rp + c0;
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                       : "=r"(D[d][0]), "=r"(D[d][1]), "=r"(D[d][2]), "=r"(D[d][3]), "=r"(D[d][4]),
                         "=r"(D[d][5]), "=r"(D[d][6]), "=r"(D[d][7])
                       : "r"(ta));
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        const int cmax = min(8, min(g.Rn - c0, g.ncols - n0 - c0));
        if (i < g.Mrows && cmax > 0) {
          double v[8];
#pragma unroll
          for (int j = 0; j < 8; j++) {
            // Σ_d D_d 256^d: exact int64 partial sums of three diagonals, two FP64 roundings
            const long long l0 = (long long)(int)D[0][j] + ((long long)(int)D[1][j] << 8) +
                                 ((long long)(int)D[2][j] << 16);
            const long long l1 = (long long)(int)D[3][j] + ((long long)(int)D[4][j] << 8) +
                                 ((long long)(int)D[5][j] << 16);
            const double t = fma((double)(int)D[6][j], 281474976710656.0 /* 2^48 */, (double)l1 * 16777216.0);
            v[j] = (t + (double)l0) * pow2(ex + Fexp[n0 + c0 + j] - 60);
          }
          double* orow = out + i * g.ncols + n0 + c0;
          if (cmax == 8 && !beta && ((reinterpret_cast<uintptr_t>(orow) & 31) == 0)) {
            asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(orow), "d"(v[0]), "d"(v[1]), "d"(v[2]),
                         "d"(v[3]) : "memory");
            asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(orow + 4), "d"(v[4]), "d"(v[5]), "d"(v[6]),
                         "d"(v[7]) : "memory");
          } else {
#pragma unroll
            for (int j = 0; j < 8; j++)
              if (j < cmax) orow[j] = beta ? orow[j] + v[j] : v[j];
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(tempty);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 8) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// ---- operand preparation ----
// per-column exponent of B: 2^F > max_k |B[k, c]| (F = 0 for a zero column)
__global__ void col_exp_kernel(const double* __restrict__ B, int64_t K, int ncols, int* __restrict__ F) {
  const int c = blockIdx.x;
  double m = 0.0;
  for (int64_t k = threadIdx.x; k < K; k += blockDim.x) m = fmax(m, fabs(B[k * ncols + c]));
  __shared__ double red[32];
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); w++) m = fmax(m, red[w]);
    int e = 0;
    if (m > 0.0) frexp(m, &e);
    F[c] = e;
  }
}

// B digit image: [nt][kc][plane b][Rp rows x 32 B, K-major canonical layout]
__global__ void b_image_kernel(const double* __restrict__ B, int64_t K, Geo g, const int* __restrict__ F,
                               uint8_t* __restrict__ img) {
  const int64_t total = (int64_t)g.ntn * g.nkc * g.Rp * 32;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int kb = (int)(e & 31);
    const int64_t rr = e >> 5;
    const int r = (int)(rr % g.Rp);
    const int64_t rest = rr / g.Rp;
    const int kc = (int)(rest % g.nkc);
    const int nt = (int)(rest / g.nkc);
    const int64_t k = (int64_t)kc * 32 + kb;
    const int c = nt * g.Rn + r;
    unsigned long long u = kBias;  // digits 0
    if (k < K && r < g.Rn && c < g.ncols) {
      const double x = B[k * g.ncols + c] * pow2(54 - F[c]);
      u = (unsigned long long)(__double2ll_rn(x) + (long long)kBias);
    }
    uint8_t* base = img + (((int64_t)nt * g.nkc + kc) * kND) * (g.Rp * 32);
    const int off = (r >> 3) * 256 + (kb >> 4) * 128 + (r & 7) * 16 + (kb & 15);
#pragma unroll
    for (int b = 0; b < kND; b++) base[b * (g.Rp * 32) + off] = (uint8_t)(((u >> (8 * b)) & 0xFF) ^ 0x80);
  }
}

__global__ void absmax_partial_kernel(const double* __restrict__ x, int64_t n, double* __restrict__ part) {
  double m = 0.0;
  const int64_t n2 = n / 2;
  const double2* x2 = reinterpret_cast<const double2*>(x);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n2; e += (int64_t)gridDim.x * blockDim.x) {
    const double2 v = x2[e];
    m = fmax(m, fmax(fabs(v.x), fabs(v.y)));
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && (n & 1)) m = fmax(m, fabs(x[n - 1]));
  __shared__ double red[32];
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); w++) m = fmax(m, red[w]);
    part[blockIdx.x] = m;
  }
}
__global__ void absmax_final_kernel(const double* __restrict__ part, int nb, int* __restrict__ e_out) {
  double m = 0.0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) m = fmax(m, part[b]);
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (threadIdx.x == 0) {
    int e = 0;
    if (m > 0.0) frexp(m, &e);
    *e_out = e;
  }
}

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

Geo make_geo(int64_t pre, int64_t K, int64_t post, int ncols) {
  Geo g;
  g.pre = pre;
  g.K = K;
  g.post = post;
  g.Mrows = pre * post;
  g.ncols = ncols;
  g.ntn = (ncols + kRpMax - 1) / kRpMax;
  g.Rn = (ncols + g.ntn - 1) / g.ntn;
  g.Rp = (g.Rn + 15) / 16 * 16;
  g.nmt = (g.Mrows + kBM - 1) / kBM;
  g.ntiles = g.nmt * g.ntn;
  g.nkc = (int)((K + 31) / 32);
  return g;
}

template <bool MC, bool VEC>
cudaError_t run_i8(int grid, const double* X, const Geo& g, const uint8_t* Bimg, const int* F, const int* Xexp,
                   double* out, int beta, cudaStream_t st) {
  static bool attr = false;  // per instantiation
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(ttm_i8_kernel<MC, VEC>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  ttm_i8_kernel<MC, VEC><<<grid, kThreads, kSmem, st>>>(X, g, Bimg, F, Xexp, out, beta);
  return cudaGetLastError();
}

}  // namespace

size_t ttm_i8_workspace_bytes(int64_t K, int ncols) {
  Geo g = make_geo(1, K, 1, ncols);
  return (size_t)g.ntn * g.nkc * kND * g.Rp * 32 + 256 * sizeof(int);
}

cudaError_t launch_absmax_exp(const double* x, int64_t n, double* partial, int* e_out, cudaStream_t st) {
  g_launches += 2;
  absmax_partial_kernel<<<kNormBlocks, 256, 0, st>>>(x, n, partial);
  absmax_final_kernel<<<1, 32, 0, st>>>(partial, kNormBlocks, e_out);
  return cudaGetLastError();
}

cudaError_t launch_ttm_i8(const double* X, int64_t pre, int64_t K, int64_t post, const double* B, int ncols,
                          double* out, int beta, const int* Xexp, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (pre <= 0 || post <= 0 || ncols <= 0) return cudaSuccess;
  if (K <= 0 || K > kMaxKI8 || ncols > 256) return cudaErrorInvalidValue;
  Geo g = make_geo(pre, K, post, ncols);
  const size_t img = (size_t)g.ntn * g.nkc * kND * g.Rp * 32;
  if (ws_bytes < img + 256 * sizeof(int)) return cudaErrorInvalidValue;
  uint8_t* Bimg = static_cast<uint8_t*>(ws);
  int* F = reinterpret_cast<int*>(static_cast<uint8_t*>(ws) + img);
  g_launches += 3;
  col_exp_kernel<<<ncols, 256, 0, st>>>(B, K, ncols, F);
  {
    int64_t total = (int64_t)g.ntn * g.nkc * g.Rp * 32;
    int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 8);
    b_image_kernel<<<blocks, 256, 0, st>>>(B, K, g, F, Bimg);
  }
  const bool mc = post > 1;
  const bool vec = !mc && (K % 2) == 0 && ((uintptr_t)X % 16) == 0;
  const int grid = (int)std::min<int64_t>(g.ntiles, sm_count());
  if (mc) return run_i8<true, false>(grid, X, g, Bimg, F, Xexp, out, beta, st);
  if (vec) return run_i8<false, true>(grid, X, g, Bimg, F, Xexp, out, beta, st);
  return run_i8<false, false>(grid, X, g, Bimg, F, Xexp, out, beta, st);
}

}  // namespace cpd
