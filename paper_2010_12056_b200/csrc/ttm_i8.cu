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
#include <cstdlib>

#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstring>

#include "kernels.h"

namespace cpd {
namespace {

constexpr int kBM = 128;
constexpr int kND = 7;
constexpr int kRpMax = 64;
constexpr int kAPlane = kBM * 32;            // bytes of one digit plane per K32 step
constexpr int kAStage = kND * kAPlane;       // 28672
constexpr int kBStage = kND * kRpMax * 32;   // 14336 (max)
constexpr int kDStage = kAStage + kBStage;   // 43008
constexpr int kFStage = kBM * 32 * 8;        // 32768: one 128 x 32 FP64 tile
// loader variants: register loads (generic shapes) or TMA tiles into an FP64 smem ring
enum { L_KC = 0, L_MC = 2, L_KC_TMA = 3, L_MC_TMA = 4 };
template <int L>
struct Cfg {
  static constexpr bool MC = (L == L_MC || L == L_MC_TMA);
  static constexpr bool TMA = L >= L_KC_TMA;
  static constexpr int NCW = TMA ? 16 : 8;           // converter warps
  static constexpr int NDS = TMA ? 3 : 5;            // digit stages
  static constexpr int NFS = TMA ? 3 : 0;            // FP64 stages
  static constexpr int THREADS = NCW * 32 + 128;     // + 4 epilogue warps (the first also issues MMAs)
  static constexpr int FOFF = NDS * kDStage;         // FP64 ring offset (1024-aligned)
  static constexpr int DATA = FOFF + NFS * kFStage;
  static constexpr int SMEM = DATA + 256;
  static constexpr int MAXREG = TMA ? 96 : 168;      // 5 resp. 3 warps per SMSP register file
};
static_assert(Cfg<L_KC_TMA>::FOFF % 1024 == 0, "swizzled TMA boxes need 1024-byte alignment");
static_assert(Cfg<L_KC_TMA>::SMEM <= 232448, "smem");
static_assert(Cfg<L_KC>::SMEM <= 232448, "smem");
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
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE_%=;\nbra WAIT_%=;\nDONE_%=:\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
// blocking form: the thread is suspended until the phase completes (or the time hint passes)
__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@P1 bra DONE_%=;\nbra WAIT_%=;\nDONE_%=:\n}\n" ::"r"(bar),
      "r"(parity), "r"(1000000)
      : "memory");
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
__device__ __forceinline__ void mma_commit_mc(uint32_t bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
      "h"(mask)
      : "memory");
}
__device__ __forceinline__ double pow2(int e) {  // 2^e for normal range
  return __longlong_as_double((long long)(1023 + e) << 52);
}
// exact integer -> FP64 without the conversion unit: x + 1.5 2^52 written into the mantissa, valid for
// |x| < 2^51 (ping-pong epilogue: C4 digit TTM 1-2 % faster than with I2F.F64, A/B on one box)
__device__ __forceinline__ double i2d_exact(long long x) {
  return __longlong_as_double(x + 0x4338000000000000LL) - 6755399441055744.0;
}
__device__ __forceinline__ double i2d_exact(int x) {  // 2^52 + 2^31 + x, any int32
  return __hiloint2double(0x43300000, (int)((unsigned)x ^ 0x80000000u)) - 4503601774854144.0;
}

struct Geo {
  int64_t pre, K, post, Mrows;
  int ncols, Rn, Rp, ntn;   // columns, columns per N tile, padded, number of N tiles
  int bstride;              // bytes of one (N tile, K32 step) block of the B digit image
  int64_t nmt, ntiles;      // M tiles, total tiles
  int nkc;                  // K32 steps
  // padded-digit MC tiling (D_MCP): rows (p, mo, m), m < w in blocks of 128
  int64_t w = 0, Mo = 0, ipad = 0;
  int wb = 0;
  // flattened padded MC tiling (D_MCF): the (Mo, ipad) rows of one prefix are contiguous, so tiles run
  // over postF = Mo * ipad in steps of 128 (pad positions m >= w are skipped in the epilogue)
  int64_t postF = 0;
  // digit kernel: CTAs per cluster (1, or 2: a pair takes two N tiles of one M tile and the A box
  // is TMA-multicast to both -- T's digits leave HBM/L2 once per pair)
  int cl = 1;
  // K chunks (a contraction longer than kMaxKI8 runs as several launches accumulating with beta = 1):
  // kofs = first K index of this launch (added to the K coordinate of every box), Kfull = K extent of
  // the tensor map (0: K).  D_KCW (block contraction, upper-level fusion): the digit view is
  // [P2 slabs][Mrows][Qp bytes] and K step kc reads slab p0 + kc / nkq at offset kofs + 32 (kc % nkq)
  int64_t kofs = 0, Kfull = 0;
  int nkq = 0;
  int64_t p0 = 0, P2 = 1, Qp = 0;
};

// tile tt of this CTA (digit kernel) -> M tile, N tile
__device__ __forceinline__ void tile_of(const Geo& g, int64_t tt, int64_t& mt, int& nt) {
  if (g.cl == 1) {
    const int64_t tile = blockIdx.x + tt * gridDim.x;
    mt = tile / g.ntn;
    nt = (int)(tile % g.ntn);
  } else {  // cluster tile ct = (M tile, group of cl consecutive N tiles); rank = N tile in the group
    const int ng = g.ntn / g.cl;
    const int64_t ct = blockIdx.x / g.cl + tt * (gridDim.x / g.cl);
    mt = ct / ng;
    nt = (int)(ct - mt * ng) * g.cl + (int)(blockIdx.x % g.cl);
  }
}
__device__ __forceinline__ int64_t tiles_of_cta(const Geo& g) {
  if (g.cl == 1) return g.ntiles > blockIdx.x ? (g.ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t cid = blockIdx.x / g.cl, ncl = gridDim.x / g.cl, nct = g.nmt * (g.ntn / g.cl);
  return nct > cid ? (nct - 1 - cid) / ncl + 1 : 0;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// 128-byte swizzle of the TMA KC boxes: 16-byte chunk c of row r is stored at c ^ (r % 8)
__device__ __forceinline__ int swz(int row, int c) { return row * 128 + ((c ^ (row & 7)) << 4); }

template <int L, int RP>
__global__ void __maxnreg__(Cfg<L>::MAXREG)
    ttm_i8_kernel(const double* __restrict__ X, Geo g, const uint8_t* __restrict__ Bimg,
                  const int* __restrict__ Fexp, const int* __restrict__ Xexp, double* __restrict__ out, int beta,
                  int dbg, const __grid_constant__ CUtensorMap tmap) {
  using C = Cfg<L>;
  constexpr bool MC = C::MC;
  constexpr int NDS = C::NDS, NFS = C::NFS;
  constexpr int Rp = RP;  // padded columns per N tile (16, 32, 48 or 64): MMA shapes are compile-time
  constexpr int Bbytes = kND * Rp * 32;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* dring = smem;                               // NDS digit stages
  uint8_t* fring = smem + C::FOFF;                     // NFS FP64 stages (TMA variants)
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::DATA);
  const uint32_t full0 = su32(bars), empty0 = su32(bars + NDS);
  const uint32_t tfull = su32(bars + 2 * NDS), tempty = su32(bars + 2 * NDS + 1);
  const uint32_t ffull0 = su32(bars + 2 * NDS + 2), fempty0 = su32(bars + 2 * NDS + 2 + NFS);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 2 * NDS + 2 + 2 * NFS);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int MMAW = C::NCW;  // TMEM allocator, MMA issuer (lane 0), epilogue quarter 0

  if (tid == 0) {
    for (int s = 0; s < NDS; s++) {
      mbar_init(full0 + 8 * s, C::NCW);   // one arrival per converter warp
      mbar_init(empty0 + 8 * s, 1);
    }
    for (int f = 0; f < NFS; f++) {
      mbar_init(ffull0 + 8 * f, 1);
      mbar_init(fempty0 + 8 * f, C::NCW);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 128);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if constexpr (C::TMA) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
  }
  if (warp == MMAW) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  const int64_t my_tiles = g.ntiles > blockIdx.x ? (g.ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t iters = my_tiles * g.nkc;

  if (warp < C::NCW) {
    // ===================== converters =====================
    const double scale = pow2(54 - *Xexp);
    int64_t tile = blockIdx.x;
    int kc = 0, s = 0;
    uint32_t dpar = 1;  // parity of the digit-stage round we wait for (first round passes)
    // x: this thread's NV consecutive-k values of one row -> digits, stores, arrive
    auto emit = [&](const double* x, int NV, int row, int kb0) {
      if (dbg & 16) mbar_wait_sleep(empty0 + 8 * s, dpar); else mbar_wait(empty0 + 8 * s, dpar);
      uint8_t* st = dring + s * kDStage;
      if (tid == 0 && !(dbg & 8)) {  // the factor digits of this K step: bulk copy, overlapping the conversion
        const int nt = (int)(tile % g.ntn);
        const uint8_t* src = Bimg + ((int64_t)nt * g.nkc + kc) * Bbytes;
        mbar_expect_tx(full0 + 8 * s, Bbytes);  // tx only: thread 0 arrives after its own stores
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                su32(st + kAStage)),
            "l"(src), "r"(Bbytes), "r"(full0 + 8 * s)
            : "memory");
      }
      // plane a of row `row`, bytes kb0.. of the K32 step (UMMA K-major canonical, no swizzle)
      const int off = (row >> 3) * 256 + (kb0 >> 4) * 128 + (row & 7) * 16 + (kb0 & 15);
      // groups of 8 values: int64 fixed point + bias, byte transpose, 7 x 8-byte stores
      for (int hf = 0; hf < NV / 8; hf++) {
        if (dbg & 4) break;
        uint32_t lo[8], hi[8];
#pragma unroll
        for (int q = 0; q < 8; q++) {
          const long long a = __double2ll_rn(x[8 * hf + q] * scale) + (long long)kBias;
          lo[q] = (uint32_t)a;
          hi[q] = (uint32_t)((unsigned long long)a >> 32);
        }
        uint32_t pl[7][2];
#pragma unroll
        for (int w = 0; w < 2; w++) {
          uint32_t o[4];
          transpose4(lo[4 * w], lo[4 * w + 1], lo[4 * w + 2], lo[4 * w + 3], o);
#pragma unroll
          for (int b = 0; b < 4; b++) pl[b][w] = o[b] ^ 0x80808080u;
          transpose4(hi[4 * w], hi[4 * w + 1], hi[4 * w + 2], hi[4 * w + 3], o);
#pragma unroll
          for (int b = 0; b < 3; b++) pl[4 + b][w] = o[b] ^ 0x80808080u;
        }
#pragma unroll
        for (int a = 0; a < kND; a++)
          *reinterpret_cast<uint2*>(st + a * kAPlane + off + 8 * hf) = make_uint2(pl[a][0], pl[a][1]);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // own stores -> async proxy
      __syncwarp();
      if (lane == 0) mbar_arrive(full0 + 8 * s);
      if (++s == NDS) {
        s = 0;
        dpar ^= 1;
      }
      if (++kc == g.nkc) {
        kc = 0;
        tile += gridDim.x;
      }
    };

    if constexpr (C::TMA) {
      // ---- TMA loader (thread 0 issues K steps NFS-1 ahead) + 16 converter warps ----
      const int row = tid & 127, part = tid >> 7;  // 8 consecutive k of one row per K step
      int64_t l_tile = blockIdx.x, l_it = 0;
      int l_kc = 0, l_f = 0;
      uint32_t l_par = 1;
      auto issue = [&]() {  // thread 0: next FP64 tile into the ring
        if (l_it >= iters) return;
        if (dbg & 16) mbar_wait_sleep(fempty0 + 8 * l_f, l_par); else mbar_wait(fempty0 + 8 * l_f, l_par);
        const uint32_t dst = su32(fring + l_f * kFStage), bar = ffull0 + 8 * l_f;
        if (!(dbg & 2)) {
          mbar_arrive_expect_tx(bar, kFStage);
          const int64_t i0 = (l_tile / g.ntn) * kBM;
          const int k0 = l_kc * 32;
          if constexpr (!MC) {
            for (int hb = 0; hb < 2; hb++)
              asm volatile(
                  "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
                  "[%4];" ::"r"(dst + hb * (kFStage / 2)),
                  "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(k0 + 16 * hb), "r"((int)i0), "r"(bar)
                  : "memory");
          } else {
            const int64_t p = i0 / g.post, m0 = i0 - p * g.post;
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
                "[%5];" ::"r"(dst),
                "l"(reinterpret_cast<uint64_t>(&tmap)), "r"((int)m0), "r"(k0), "r"((int)p), "r"(bar)
                : "memory");
          }
        } else {
          mbar_arrive(bar);
        }
        l_it++;
        if (++l_f == NFS) {
          l_f = 0;
          l_par ^= 1;
        }
        if (++l_kc == g.nkc) {
          l_kc = 0;
          l_tile += gridDim.x;
        }
      };
      if (tid == 0)
        for (int q = 0; q < NFS - 1; q++) issue();
      int f = 0;
      uint32_t fpar = 0;
#pragma unroll 1
      for (int64_t it = 0; it < iters; it++) {
        if (tid == 0) issue();
        if (dbg & 16) mbar_wait_sleep(ffull0 + 8 * f, fpar); else mbar_wait(ffull0 + 8 * f, fpar);
        const uint8_t* fb = fring + f * kFStage;
        double x[8];
        if constexpr (!MC) {
          // box part>>1 holds k 16*(part>>1).., row-major 128-byte rows, 128B-swizzled
          const uint8_t* box = fb + (part >> 1) * (kFStage / 2);
#pragma unroll
          for (int c = 0; c < 4; c++) {
            const double2 v = *reinterpret_cast<const double2*>(box + swz(row, (part & 1) * 4 + c));
            x[2 * c] = v.x;
            x[2 * c + 1] = v.y;
          }
        } else {
#pragma unroll
          for (int q = 0; q < 8; q++) x[q] = reinterpret_cast<const double*>(fb)[(8 * part + q) * kBM + row];
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(fempty0 + 8 * f);
        if (++f == NFS) {
          f = 0;
          fpar ^= 1;
        }
        emit(x, 8, row, 8 * part);
      }
    } else {
      // ---- register loader: 16 values per thread, two K steps ahead (three named buffers) ----
      const int row = MC ? (tid & 127) : (tid >> 1);
      const int h = MC ? (tid >> 7) : (tid & 1);
      int64_t l_tile = blockIdx.x, l_it = 0;
      int l_kc = 0;
      const double* l_src = X;
      bool l_rok = false;
      auto new_tile = [&]() {  // base of this thread's row in tile l_tile
        const int64_t mt = l_tile / g.ntn;
        const int64_t i = mt * kBM + row;
        l_rok = i < g.Mrows;
        const int64_t ii = l_rok ? i : 0;
        if constexpr (!MC) {
          l_src = X + ii * g.K;
        } else {
          const int64_t p = ii / g.post, m = ii - p * g.post;
          l_src = X + p * g.K * g.post + m;
        }
      };
      if (iters > 0) new_tile();
      auto load = [&](double (&x)[16]) {
        if (l_it < iters) {
          const int64_t k0 = (int64_t)l_kc * 32 + 16 * h;
          if constexpr (!MC) {
#pragma unroll
            for (int q = 0; q < 16; q++) x[q] = (l_rok && k0 + q < g.K) ? __ldg(l_src + k0 + q) : 0.0;
          } else {
            const double* src = l_src + k0 * g.post;
#pragma unroll
            for (int q = 0; q < 16; q++) x[q] = (l_rok && k0 + q < g.K) ? __ldg(src + q * g.post) : 0.0;
          }
          l_it++;
          if (++l_kc == g.nkc) {
            l_kc = 0;
            l_tile += gridDim.x;
            if (l_it < iters) new_tile();
          }
        }
      };
      double xa[16], xb[16], xc[16];
      load(xa);
      load(xb);
#pragma unroll 1
      for (int64_t it = 0; it < iters; it += 3) {
        load(xc);
        emit(xa, 16, row, 16 * h);
        if (it + 1 >= iters) break;
        load(xa);
        emit(xb, 16, row, 16 * h);
        if (it + 2 >= iters) break;
        load(xb);
        emit(xc, 16, row, 16 * h);
      }
    }
  } else {
    // ===================== epilogue (4 warps; the first also issues the MMAs) =====================
    const int q = warp & 3;  // TMEM lane quarter of this warp
    const int r = q * 32 + lane;
    const int ex = *Xexp;
    int s = 0;  // MMA issuer: digit stage and its parity
    uint32_t fpar = 0;
    for (int64_t tt = 0; tt < my_tiles; tt++) {
      const int64_t tile = blockIdx.x + tt * gridDim.x;
      const int64_t mt = tile / g.ntn;
      const int nt = (int)(tile % g.ntn);
      const int64_t i = mt * kBM + r;
      const int n0 = nt * g.Rn;
      if (warp == MMAW) {
        if (lane == 0) {
          mbar_wait_sleep(tempty, ((uint32_t)tt & 1) ^ 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          for (int kc = 0; kc < g.nkc; kc++) {
            mbar_wait(full0 + 8 * s, fpar);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t abase = su32(dring + s * kDStage);
            const uint64_t ad0 = sdesc(abase, 128, 256), bd0 = sdesc(abase + kAStage, 128, 256);
            if (!(dbg & 1)) {
#pragma unroll
              for (int a = kND - 1; a >= 0; a--) {
                const uint32_t acc = (kc > 0 || a < kND - 1) ? 1u : 0u;
                const int n = (a + 1) * Rp;                                  // diagonals 0..a
                const uint64_t ad = ad0 + (uint64_t)((a * kAPlane) >> 4);
                const uint64_t bd = bd0 + (uint64_t)(((kND - 1 - a) * Rp * 32) >> 4);  // B planes 6-a..6
                mma_i8(tmem, ad, bd, idesc(n > 256 ? 256 : n), acc);
                if (n > 256) mma_i8(tmem + 256, ad, bd + ((256 * 32) >> 4), idesc(n - 256), acc);
              }
            }
            mma_commit(empty0 + 8 * s);
            if (++s == NDS) {
              s = 0;
              fpar ^= 1;
            }
          }
          mma_commit(tfull);
        }
        __syncwarp();
      }
      mbar_wait_sleep(tfull, (uint32_t)tt & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      for (int c0 = 0; c0 < Rp; c0 += 8) {
        uint32_t D[kND][8];
#pragma unroll
        for (int d = 0; d < kND; d++) {
          const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + d * Rp + c0;
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
  if (warp == MMAW) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
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
    uint8_t* base = img + ((int64_t)nt * g.nkc + kc) * g.bstride;
    const int off = (r >> 3) * 256 + (kb >> 4) * 128 + (r & 7) * 16 + (kb & 15);
#pragma unroll
    for (int b = 0; b < kND; b++) base[b * (g.Rp * 32) + off] = (uint8_t)(((u >> (8 * b)) & 0xFF) ^ 0x80);
  }
  // Rp % 16 == 8: 8 zero rows after plane 6 -- the last MMA of each T digit is rounded up to a
  // multiple of 16 columns and reads them (zero products on the next diagonal's columns)
  const int pad = g.bstride - kND * g.Rp * 32;
  if (pad > 0) {
    const int64_t nb = (int64_t)g.ntn * g.nkc * pad;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nb; e += (int64_t)gridDim.x * blockDim.x)
      img[(e / pad) * g.bstride + kND * g.Rp * 32 + e % pad] = 0;
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
__global__ void absmax_final_kernel(const double* __restrict__ part, int nb, int* __restrict__ e_out,
                                    double* __restrict__ m_out) {
  double m = 0.0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) m = fmax(m, part[b]);
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (threadIdx.x == 0) {
    int e = 0;
    if (m > 0.0) frexp(m, &e);
    *e_out = e;
    if (m_out) *m_out = m;
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

// rp8: the digit kernel also takes N tiles padded to a multiple of 8 (Rp = 40, 56) instead of 16
// (R = 100 as 2 x 52 columns, R = 200 as 4 x 52: 56-column tiles do 11 % fewer MMA columns than 64)
Geo make_geo(int64_t pre, int64_t K, int64_t post, int ncols, bool rp8) {
  Geo g;
  g.pre = pre;
  g.K = K;
  g.post = post;
  g.Mrows = pre * post;
  g.ncols = ncols;
  static const int rpmax = getenv("CPD_I8_RPMAX") ? std::min(kRpMax, std::max(16, atoi(getenv("CPD_I8_RPMAX")) / 16 * 16)) : kRpMax;
  g.ntn = (ncols + rpmax - 1) / rpmax;
  g.Rn = (ncols + g.ntn - 1) / g.ntn;
  if (g.ntn > 1) g.Rn = std::min(rpmax, (g.Rn + 3) / 4 * 4);  // 32-byte aligned column blocks
  g.ntn = (ncols + g.Rn - 1) / g.Rn;
  g.Rp = (g.Rn + 15) / 16 * 16;
  static const bool no_rp8 = getenv("CPD_I8_NO_RP8") != nullptr;  // experiment switch
  if (rp8 && !no_rp8 && (g.Rn + 7) / 8 * 8 < g.Rp && g.Rp > 32) g.Rp = (g.Rn + 7) / 8 * 8;
  g.bstride = kND * g.Rp * 32 + (g.Rp % 16 ? 256 : 0);
  g.nmt = (g.Mrows + kBM - 1) / kBM;
  g.ntiles = g.nmt * g.ntn;
  g.nkc = (int)((K + 31) / 32);
  return g;
}

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
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

// TMA descriptor of T for the loader variant: KC = 2-D [Mrows][K] in 16 x 128 boxes with
// the 128-byte swizzle; MC = 3-D [pre][K][post] in 128 x 32 x 1 boxes (post % 128 == 0)
bool make_tmap(int L, const double* X, const Geo& g, CUtensorMap* tm) {
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  CUresult r;
  if (L == L_KC_TMA) {
    cuuint64_t dims[2] = {(cuuint64_t)g.K, (cuuint64_t)g.Mrows};
    cuuint64_t strides[1] = {(cuuint64_t)g.K * 8};
    cuuint32_t box[2] = {16, (cuuint32_t)kBM}, es[2] = {1, 1};
    r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(X), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    cuuint64_t dims[3] = {(cuuint64_t)g.post, (cuuint64_t)g.K, (cuuint64_t)g.pre};
    cuuint64_t strides[2] = {(cuuint64_t)g.post * 8, (cuuint64_t)g.K * g.post * 8};
    cuuint32_t box[3] = {(cuuint32_t)kBM, 32, 1}, es[3] = {1, 1, 1};
    r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(X), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  return r == CUDA_SUCCESS;
}

template <int L, int RP>
cudaError_t run_i8(int grid, const double* X, const Geo& g, const uint8_t* Bimg, const int* F, const int* Xexp,
                   double* out, int beta, const CUtensorMap& tm, cudaStream_t st) {
  static const int dbg = getenv("CPD_I8_DBG") ? atoi(getenv("CPD_I8_DBG")) : 0;  // profiling switches
  static bool attr = false;  // per instantiation
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(ttm_i8_kernel<L, RP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Cfg<L>::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  ttm_i8_kernel<L, RP><<<grid, Cfg<L>::THREADS, Cfg<L>::SMEM, st>>>(X, g, Bimg, F, Xexp, out, beta, dbg, tm);
  return cudaGetLastError();
}

template <int RP>
cudaError_t dispatch_i8(int L, int grid, const double* X, const Geo& g, const uint8_t* Bimg, const int* F,
                        const int* Xexp, double* out, int beta, const CUtensorMap& tm, cudaStream_t st) {
  switch (L) {
    case L_KC: return run_i8<L_KC, RP>(grid, X, g, Bimg, F, Xexp, out, beta, tm, st);
    case L_MC: return run_i8<L_MC, RP>(grid, X, g, Bimg, F, Xexp, out, beta, tm, st);
    case L_KC_TMA: return run_i8<L_KC_TMA, RP>(grid, X, g, Bimg, F, Xexp, out, beta, tm, st);
    case L_MC_TMA: return run_i8<L_MC_TMA, RP>(grid, X, g, Bimg, F, Xexp, out, beta, tm, st);
  }
  return cudaErrorInvalidValue;
}

// ============================================================================================
// Digit-plane variant: T's 7 int8 digit planes are computed ONCE (T is read-only for the
// whole decomposition, like the paper's stored transposed copies of T) and the
// TTM streams them with TMA straight into the UMMA operand layout -- no per-sweep conversion.
// Planes are stored plane-major, each with T's row-major layout (7 bytes per element).
//   KC (contract the last kept mode, K contiguous): 3-D map {K, Mrows, 7}, box {32, 128, 7},
//      128 rows x 32 bytes per plane, 32-byte swizzle = UMMA K-major SWIZZLE_32B;
//   MC (post % 128 == 0): 4-D map {post, K, pre, 7}, box {128, 32, 1, 7}: 32 k-rows x 128 m
//      bytes per plane, 128-byte swizzle = UMMA MN-major SWIZZLE_128B.
// Warps: 0 TMA producer, 1 TMEM allocator + MMA issuer, 2-9 epilogue (two per lane quarter).
// ============================================================================================
// loader layouts of the digit kernel: KC, or MC with an MN atom of 128 / 64 / 32 bytes
// (post % 128 == 0, or post == 64 / 32 with 2 / 4 consecutive prefix indices per tile), or
// D_MCP: MC over padded digit rows (innermost extent w not a multiple of 16, or post % 128 != 0):
// tiles (p, mo, 128-block of the innermost mode), 5-D map {w, Mo, K, pre, 7}
// D_MCF: MC over padded digit rows with Mo = post / w > 1 and Mo * ipad % 128 == 0: the same boxes as
// D_MC128 over the flattened (Mo, ipad) extent -- 4 % of pad rows instead of D_MCP's per-row 128-blocks
// (C3, w = 200, ipad = 208: 208 MMA rows per 200 instead of 256)
// D_KCW: KC over a [P2][Mrows][Qp] view -- the K index is (slab p, q): the contraction of a block of
// modes with a Khatri-Rao product (upper-level fusion), wrapping blocks included
enum { D_KC = 0, D_MC128 = 1, D_MC64 = 2, D_MC32 = 3, D_MCP = 4, D_MCF = 5, D_KCW = 6 };
constexpr int kStagesD = 5;
constexpr int kEpiWarps = 16;                        // 4 per TMEM lane quarter
constexpr int kThreadsD = 32 * (2 + kEpiWarps);
constexpr int kMaxColsI8 = 1024;  // output columns (R) of one TTM: column scales in shared memory
constexpr int kSmemD = kStagesD * kDStage + 256 + kMaxColsI8 * 8;  // stages, barriers, column scales
static_assert(kSmemD <= 232448, "smem");

// UMMA descriptor with a swizzle layout type (2 = 128B, 4 = 64B, 6 = 32B), base offset 0
__device__ __forceinline__ uint64_t sdesc_sw(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return sdesc(addr, lbo, sbo) | ((uint64_t)layout << 61);
}

// DRAIN epilogue of one warp: rows r (TMEM lane quarter base tq), columns c_lo .. c_lo + CQ.
// Per tile and 8-column chunk: the 7 diagonals in one batch of tcgen05.ld (one wait per chunk: the
// TMEM load latency is paid CQ/8 times per tile, not once per diagonal pair), exact int64 partial
// sums, the FP64 value; then release the accumulator (tempty), and the global stores overlap the
// next tile's MMAs.
template <int L, int Rp, int CQ>
__device__ __forceinline__ void epilogue_drain(const Geo& g, uint32_t tq, int c_lo, int r, int64_t my_tiles,
                                               double* __restrict__ out, int beta, const double* colscale,
                                               uint32_t tfull0, uint32_t tempty0, int dbg) {
  constexpr int NCH = CQ / 8;
  const bool active = c_lo < Rp;  // warp-uniform
  for (int64_t tt = 0; tt < my_tiles; tt++) {
    int64_t mt;
    int nt;
    tile_of(g, tt, mt, nt);
    int64_t i = mt * kBM + r;
    bool row_ok = i < g.Mrows;
    if constexpr (L == D_MCP) {
      const int64_t pm = mt / g.wb;
      const int64_t mb0 = (mt - pm * g.wb) * kBM;
      const int64_t m = min(mb0, g.ipad - kBM) + r;
      i = pm * g.w + m;
      row_ok = m >= mb0 && m < g.w;
    } else if constexpr (L == D_MCF) {
      const int64_t f = mt * kBM + r, p = f / g.postF, fm = f - p * g.postF;
      const int64_t mo = fm / g.ipad, m = fm - mo * g.ipad;
      i = p * g.post + mo * g.w + m;
      row_ok = m < g.w;
    }
    const int n0 = nt * g.Rn;
    if (dbg & 128) mbar_wait(tfull0, (uint32_t)tt & 1);  // profiling switch 128: spin instead of suspend
    else mbar_wait_sleep(tfull0, (uint32_t)tt & 1);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    double v[NCH][8];
    if (active && !(dbg & 256)) {  // profiling switch 256: release the accumulator without draining it
#pragma unroll
      for (int ch = 0; ch < NCH; ch++) {
        uint32_t D[kND][8];
#pragma unroll
        for (int d = 0; d < kND; d++)
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                       : "=r"(D[d][0]), "=r"(D[d][1]), "=r"(D[d][2]), "=r"(D[d][3]), "=r"(D[d][4]), "=r"(D[d][5]),
                         "=r"(D[d][6]), "=r"(D[d][7])
                       : "r"(tq + d * Rp + c_lo + 8 * ch));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        const int c0 = c_lo + 8 * ch;
        const int cmax = max(1, min(8, min(g.Rn - c0, g.ncols - n0 - c0)));
#pragma unroll
        for (int j = 0; j < 8; j++) {
          // Σ_d D_d 256^d: exact int64 partial sums of diagonals 0-2 and 3-6 (|l1| < 2^56), one rounding
          // of l1, then the FP64 value (hardware conversions: the bias conversion of the ping-pong
          // epilogue measured 4 % slower here, C3 MC launches 6.57 -> 6.85 ms)
          const long long l0 = (long long)(int)D[0][j] + ((long long)(int)D[1][j] << 8) +
                               ((long long)(int)D[2][j] << 16);
          const long long l1 = (long long)(int)D[3][j] + ((long long)(int)D[4][j] << 8) +
                               ((long long)(int)D[5][j] << 16) + ((long long)(int)D[6][j] << 24);
          v[ch][j] = fma((double)l1, 16777216.0 /* 2^24 */, (double)l0) * colscale[n0 + c0 + min(j, cmax - 1)];
        }
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    mbar_arrive(tempty0);
    if (!active || (dbg & (32 | 256))) continue;
#pragma unroll
    for (int ch = 0; ch < NCH; ch++) {
      const int c0 = c_lo + 8 * ch;
      const int cmax = min(8, min(g.Rn - c0, g.ncols - n0 - c0));
      if (!row_ok || cmax <= 0) continue;
      double* orow = out + i * g.ncols + n0 + c0;
      const uintptr_t al = reinterpret_cast<uintptr_t>(orow) & 31;
      if (cmax == 8 && !beta && al == 0) {
        asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(orow), "d"(v[ch][0]), "d"(v[ch][1]),
                     "d"(v[ch][2]), "d"(v[ch][3]) : "memory");
        asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(orow + 4), "d"(v[ch][4]), "d"(v[ch][5]),
                     "d"(v[ch][6]), "d"(v[ch][7]) : "memory");
      } else if (cmax == 8 && !beta && (al & 15) == 0) {
#pragma unroll
        for (int j = 0; j < 8; j += 2)
          asm volatile("st.global.v2.f64 [%0], {%1,%2};" ::"l"(orow + j), "d"(v[ch][j]), "d"(v[ch][j + 1]) : "memory");
      } else {
#pragma unroll
        for (int j = 0; j < 8; j++)
          if (j < cmax) orow[j] = beta ? orow[j] + v[ch][j] : v[ch][j];
      }
    }
  }
}

template <int L, int RP>
__global__ void __launch_bounds__(kThreadsD, 1)
    ttm_i8d_kernel(Geo g, const uint8_t* __restrict__ Bimg, const int* __restrict__ Fexp,
                   const int* __restrict__ Xexp, double* __restrict__ out, int beta,
                   const __grid_constant__ CUtensorMap tmap, int dbg) {
  constexpr int Rp = RP;
  constexpr int Bbytes = kND * Rp * 32 + (Rp % 16 ? 256 : 0);  // + 8 zero rows when Rp % 16 == 8
  static_assert(Bbytes <= kBStage, "B stage");
  constexpr int NDS = kStagesD;
  // TMEM accumulator buffers: 7 diagonals x Rp columns each; two (ping-pong) when they fit
  constexpr int NACC = (2 * kND * Rp <= 512 && kND * Rp <= 256) ? 2 : 1;
  constexpr int MCW = (L == D_MC128 || L == D_MCP || L == D_MCF) ? 128 : L == D_MC64 ? 64 : 32;  // MN atom bytes
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NDS * kDStage);
  const uint32_t full0 = su32(bars), empty0 = su32(bars + NDS);
  const uint32_t tfull0 = su32(bars + 2 * NDS), tempty0 = su32(bars + 2 * NDS + 2);
  // DRAIN (one accumulator set, 7 Rp > 256 columns): the epilogue first moves the diagonals into
  // exact int64 partial sums in registers and releases the accumulator, then does the FP64
  // recombination and the global stores while the MMA warp already runs the next tile
  constexpr bool DRAIN = NACC == 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 2 * NDS + 4);
  double* colscale = reinterpret_cast<double*>(smem + NDS * kDStage + 256);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < NDS; s++) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, g.cl);  // one MMA commit per CTA of the cluster
    }
    for (int b = 0; b < 2; b++) {
      mbar_init(tfull0 + 8 * b, 1);
      mbar_init(tempty0 + 8 * b, 32 * kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
  }
  {
    const int ex = *Xexp;  // 2^(e_X + F_c - 60) per output column c
    for (int c = tid; c < g.ncols; c += blockDim.x) colscale[c] = pow2(ex + Fexp[c] - 60);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if (g.cl > 1) cluster_sync_all();  // peers' barriers initialised before any multicast
  else __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  const int64_t my_tiles = tiles_of_cta(g);
  const uint16_t cmask = (uint16_t)((1u << g.cl) - 1);

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      int s = 0;
      uint32_t par = 1;
      for (int64_t tt = 0; tt < my_tiles; tt++) {
        int64_t mt;
        int nt;
        tile_of(g, tt, mt, nt);
        const int64_t i0 = mt * kBM;
        int p = 0, m0 = 0, mo = 0;
        if constexpr (L == D_MCP) {
          // the last block of the innermost mode is shifted back to end at w: boxes never
          // overhang the tensor edge (an overhanging MN-major box corrupted loads on sm_100a)
          const int64_t pm = mt / g.wb;
          m0 = (int)min((mt - pm * g.wb) * kBM, g.ipad - kBM);  // 16-byte aligned start
          p = (int)(pm / g.Mo);
          mo = (int)(pm - (int64_t)p * g.Mo);
        } else if constexpr (L == D_MCF) {
          p = (int)(i0 / g.postF);
          m0 = (int)(i0 - (int64_t)p * g.postF);
        } else if constexpr (L != D_KC && L != D_KCW) {
          p = (int)(i0 / g.post);
          m0 = (int)(i0 - (int64_t)p * g.post);
        }
        for (int kc = 0; kc < g.nkc; kc++) {
          mbar_wait(empty0 + 8 * s, par);
          const uint32_t st = su32(smem + s * kDStage), bar = full0 + 8 * s;
          int kk = (int)g.kofs + kc * 32;  // K coordinate of this step
          if constexpr (L == D_KCW) {
            const int sl = kc / g.nkq;
            kk = (int)g.kofs + (kc - sl * g.nkq) * 32;
            p = (int)g.p0 + sl;
          }
          if (dbg & 2) {  // profiling: no loads
            mbar_arrive(bar);
            if (++s == NDS) {
              s = 0;
              par ^= 1;
            }
            continue;
          }
          mbar_arrive_expect_tx(bar, ((dbg & 8) ? 0 : kAStage) + ((dbg & 4) ? 0 : Bbytes));
          if (dbg & 8) {  // profiling: no A loads
          } else if (g.cl > 1) {
            // A box multicast to every CTA of the cluster (same smem offset, each CTA's full[s]) by the
            // cluster's rank 0 (rotating the issuer with the K step measured slower: C3 loads 4.2 -> 5.1 ms)
            if (blockIdx.x % g.cl == 0) {
              if constexpr (L == D_KC) {
                asm volatile(
                    "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster "
                    "[%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(st),
                    "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(kk), "r"((int)i0), "r"(0), "r"(bar), "h"(cmask)
                    : "memory");
              } else if constexpr (L == D_KCW) {
                asm volatile(
                    "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster "
                    "[%0], [%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(st),
                    "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(kk), "r"((int)i0), "r"(p), "r"(0), "r"(bar), "h"(cmask)
                    : "memory");
              } else if (L == D_MCP && g.Mo > 1) {
                asm volatile(
                    "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster "
                    "[%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;" ::"r"(st),
                    "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(m0), "r"(mo), "r"(kk), "r"(p), "r"(0), "r"(bar),
                    "h"(cmask)
                    : "memory");
              } else {
                asm volatile(
                    "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster "
                    "[%0], [%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(st),
                    "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(m0), "r"(kk), "r"(p), "r"(0), "r"(bar), "h"(cmask)
                    : "memory");
              }
            }
          } else if constexpr (L == D_KC) {
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
                "%4}], [%5];" ::"r"(st),
                "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(kk), "r"((int)i0), "r"(0), "r"(bar)
                : "memory");
          } else if constexpr (L == D_KCW) {
            asm volatile(
                "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
                "%4, %5}], [%6];" ::"r"(st),
                "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(kk), "r"((int)i0), "r"(p), "r"(0), "r"(bar)
                : "memory");
          } else if (L == D_MCP && g.Mo == 1) {
            asm volatile(
                "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
                "%4, %5}], [%6];" ::"r"(st),
                "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(m0), "r"(kk), "r"(p), "r"(0), "r"(bar)
                : "memory");
          } else if constexpr (L == D_MCP) {
            asm volatile(
                "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
                "%4, %5, %6}], [%7];" ::"r"(st),
                "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(m0), "r"(mo), "r"(kk), "r"(p), "r"(0), "r"(bar)
                : "memory");
          } else {
            asm volatile(
                "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
                "%4, %5}], [%6];" ::"r"(st),
                "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(m0), "r"(kk), "r"(p), "r"(0), "r"(bar)
                : "memory");
          }
          const uint8_t* bsrc = Bimg + ((int64_t)nt * g.nkc + kc) * Bbytes;
          if (!(dbg & 4))  // profiling switch 4: no B loads
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    st + kAStage),
                "l"(bsrc), "r"(Bbytes), "r"(bar)
                : "memory");
          if (++s == NDS) {
            s = 0;
            par ^= 1;
          }
        }
      }
      if (g.cl > 1) {  // every stage's last release (peers' MMA commits) has landed before exit
        for (int q = 0; q < NDS; q++) {
          mbar_wait(empty0 + 8 * s, par);
          if (++s == NDS) {
            s = 0;
            par ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      int s = 0;
      uint32_t par = 0;
      // A: KC K-major SW32 (8-row groups of 256 B); MC MN-major, swizzle = MN atom width:
      // LBO = stride between the G atoms (one prefix index each), SBO = 8 k-rows of the atom
      constexpr bool KMAJ = L == D_KC || L == D_KCW;
      constexpr uint32_t A_LBO = KMAJ ? 16 : 32 * MCW;
      constexpr uint32_t A_SBO = KMAJ ? 256 : 8 * MCW;
      constexpr uint32_t A_LAYOUT = (KMAJ || L == D_MC32) ? 6 : L == D_MC64 ? 4 : 2;
      constexpr uint32_t AMAJ = KMAJ ? 0u : (1u << 15);
      for (int64_t tt = 0; tt < my_tiles; tt++) {
        const int ab = NACC == 2 ? (int)(tt & 1) : 0;
        const uint32_t use = NACC == 2 ? (uint32_t)(tt >> 1) : (uint32_t)tt;  // uses of this buffer so far
        if (dbg & 128) mbar_wait(tempty0 + 8 * ab, (use & 1) ^ 1);
        else mbar_wait_sleep(tempty0 + 8 * ab, (use & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t dcol = tmem + ab * 256;
        for (int kc = 0; kc < g.nkc; kc++) {
          mbar_wait(full0 + 8 * s, par);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t abase = su32(smem + s * kDStage);
          const uint64_t ad0 = sdesc_sw(abase, A_LBO, A_SBO, A_LAYOUT), bd0 = sdesc(abase + kAStage, 128, 256);
#pragma unroll
          for (int a = kND - 1; a >= 0; a--) {
            if (dbg & 1) break;  // profiling: no MMAs
            const uint32_t acc = (kc > 0 || a < kND - 1) ? 1u : 0u;
            // diagonals 0..a; N rounded up to 16 (Rp % 16 == 8): the extra 8 columns multiply the zero rows
            // after plane 6 into diagonal a+1's first columns (+0; a = 6 initialises them at kc = 0)
            const int n = ((a + 1) * Rp + 15) / 16 * 16;
            const uint64_t ad = ad0 + (uint64_t)((a * kAPlane) >> 4);
            const uint64_t bd = bd0 + (uint64_t)(((kND - 1 - a) * Rp * 32) >> 4);  // B planes 6-a..6
            // N > 256 is split in two: at 256 (dbg 64) or in halves (multiples of 16), which keeps
            // both MMAs wide enough that their A + B shared-memory reads stay under 128 B/clk
            const int n1 = n <= 256 ? n : ((dbg & 64) ? 256 : (n / 2 + 15) / 16 * 16);
            mma_i8(dcol, ad, bd, idesc(n1) | AMAJ, acc);
            if (n > n1) mma_i8(dcol + n1, ad, bd + (uint64_t)((n1 * 32) >> 4), idesc(n - n1) | AMAJ, acc);
          }
          if (g.cl > 1) mma_commit_mc(empty0 + 8 * s, cmask);  // release the stage in every CTA
          else mma_commit(empty0 + 8 * s);
          if (++s == NDS) {
            s = 0;
            par ^= 1;
          }
        }
        mma_commit(tfull0 + 8 * ab);
      }
    }
    __syncwarp();
  } else {
    // ===================== epilogue: 16 warps, lane quarter warp % 4, column quarter =====================
    const int q = warp & 3;
    const int cq = (warp - 2) >> 2;  // 0..3
    const int r = q * 32 + lane;
    constexpr int CQ = (Rp / 4 + 7) / 8 * 8;  // columns per epilogue warp, a multiple of 8
    if constexpr (DRAIN) {
      epilogue_drain<L, Rp, CQ>(g, tmem + ((uint32_t)(q * 32) << 16), cq * CQ, r, my_tiles, out, beta, colscale,
                                tfull0, tempty0, dbg);
    } else
    for (int64_t tt = 0; tt < my_tiles; tt++) {
      int64_t mt;
      int nt;
      tile_of(g, tt, mt, nt);
      int64_t i = mt * kBM + r;
      bool row_ok = i < g.Mrows;
      if constexpr (L == D_MCP) {
        const int64_t pm = mt / g.wb;
        const int64_t mb0 = (mt - pm * g.wb) * kBM;      // first row this tile owns
        const int64_t m = min(mb0, g.ipad - kBM) + r;    // row held in TMEM lane r
        i = pm * g.w + m;
        row_ok = m >= mb0 && m < g.w;                     // overlap rows belong to the previous block
      } else if constexpr (L == D_MCF) {
        const int64_t f = mt * kBM + r, p = f / g.postF, fm = f - p * g.postF;
        const int64_t mo = fm / g.ipad, m = fm - mo * g.ipad;
        i = p * g.post + mo * g.w + m;
        row_ok = m < g.w;                                 // pad positions of the innermost mode
      }
      const int n0 = nt * g.Rn;
      const int ab = NACC == 2 ? (int)(tt & 1) : 0;
      const uint32_t use = NACC == 2 ? (uint32_t)(tt >> 1) : (uint32_t)tt;
      if (dbg & 128) mbar_wait(tfull0 + 8 * ab, use & 1);
      else mbar_wait_sleep(tfull0 + 8 * ab, use & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t tbase = tmem + ab * 256 + ((uint32_t)(q * 32) << 16);
#pragma unroll 1
      for (int c0 = cq * CQ; c0 < min(Rp, (cq + 1) * CQ); c0 += 8) {
        if (dbg & 32) break;
        uint32_t D[kND][8];
#pragma unroll
        for (int d = 0; d < kND; d++) {
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                       : "=r"(D[d][0]), "=r"(D[d][1]), "=r"(D[d][2]), "=r"(D[d][3]), "=r"(D[d][4]),
                         "=r"(D[d][5]), "=r"(D[d][6]), "=r"(D[d][7])
                       : "r"(tbase + d * Rp + c0));
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        const int cmax = min(8, min(g.Rn - c0, g.ncols - n0 - c0));
        if (row_ok && cmax > 0) {
          double v[8];
#pragma unroll
          for (int j = 0; j < 8; j++) {
            // Σ_d D_d 256^d: exact int64 partial sums of three diagonals, two FP64 roundings
            const long long l0 = (long long)(int)D[0][j] + ((long long)(int)D[1][j] << 8) +
                                 ((long long)(int)D[2][j] << 16);
            const long long l1 = (long long)(int)D[3][j] + ((long long)(int)D[4][j] << 8) +
                                 ((long long)(int)D[5][j] << 16);
            // |l0|, |l1| < 2^48: exact in FP64 (bias conversion, the same values as the hardware one)
            const double t = fma(i2d_exact((int)D[6][j]), 281474976710656.0 /* 2^48 */, i2d_exact(l1) * 16777216.0);
            v[j] = (t + i2d_exact(l0)) * colscale[n0 + c0 + min(j, cmax - 1)];
          }
          double* orow = out + i * g.ncols + n0 + c0;
          const uintptr_t al = reinterpret_cast<uintptr_t>(orow) & 31;
          if (cmax == 8 && !beta && al == 0) {
            asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(orow), "d"(v[0]), "d"(v[1]), "d"(v[2]),
                         "d"(v[3]) : "memory");
            asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(orow + 4), "d"(v[4]), "d"(v[5]), "d"(v[6]),
                         "d"(v[7]) : "memory");
          } else if (cmax == 8 && !beta && (al & 15) == 0) {
#pragma unroll
            for (int j = 0; j < 8; j += 2)
              asm volatile("st.global.v2.f64 [%0], {%1,%2};" ::"l"(orow + j), "d"(v[j]), "d"(v[j + 1]) : "memory");
          } else {
#pragma unroll
            for (int j = 0; j < 8; j++)
              if (j < cmax) orow[j] = beta ? orow[j] + v[j] : v[j];
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(tempty0 + 8 * ab);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if (g.cl > 1) cluster_sync_all();  // no CTA leaves while a peer may still signal it
  else __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// digit planes of X viewed as [n / w, w]: plane a of element (row, c) = byte a of
// (rint(X 2^(54-eX)) + bias) xor 0x80, stored at planes[a * ps + row * ipad + c]
// (ipad = digit_inner_pad(w); the pad columns stay zero = digit value 0)
__global__ void slice_digits_kernel(const double* __restrict__ X, int64_t n, int64_t w, int64_t ipad, int64_t ps,
                                    const int* __restrict__ Xexp, uint8_t* __restrict__ planes, int slow) {
  const double scale = pow2(54 - *Xexp);
  if (ipad == w && (n % 16) == 0 && !slow) {
    const int64_t n16 = n / 16;
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < n16;
         b += (int64_t)gridDim.x * blockDim.x) {
      const double2* src = reinterpret_cast<const double2*>(X + 16 * b);
      uint32_t wd[7][4];
#pragma unroll
      for (int g4 = 0; g4 < 4; g4++) {
        uint32_t lo[4], hi[4];
#pragma unroll
        for (int q = 0; q < 2; q++) {
          const double2 v = __ldg(src + 2 * g4 + q);
          const long long a0 = __double2ll_rn(v.x * scale) + (long long)kBias;
          const long long a1 = __double2ll_rn(v.y * scale) + (long long)kBias;
          lo[2 * q] = (uint32_t)a0;
          hi[2 * q] = (uint32_t)((unsigned long long)a0 >> 32);
          lo[2 * q + 1] = (uint32_t)a1;
          hi[2 * q + 1] = (uint32_t)((unsigned long long)a1 >> 32);
        }
        uint32_t o[4];
        transpose4(lo[0], lo[1], lo[2], lo[3], o);
#pragma unroll
        for (int a = 0; a < 4; a++) wd[a][g4] = o[a] ^ 0x80808080u;
        transpose4(hi[0], hi[1], hi[2], hi[3], o);
#pragma unroll
        for (int a = 0; a < 3; a++) wd[4 + a][g4] = o[a] ^ 0x80808080u;
      }
#pragma unroll
      for (int a = 0; a < kND; a++)
        *reinterpret_cast<uint4*>(planes + a * ps + 16 * b) = make_uint4(wd[a][0], wd[a][1], wd[a][2], wd[a][3]);
    }
    return;
  }
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = e / w, c = e - row * w;
    const unsigned long long u = (unsigned long long)(__double2ll_rn(X[e] * scale) + (long long)kBias);
#pragma unroll
    for (int a = 0; a < kND; a++) planes[a * ps + row * ipad + c] = (uint8_t)(((u >> (8 * a)) & 0xFF) ^ 0x80);
  }
}

bool make_tmap_digits(int L, const DigitView& dv, const Geo& g, CUtensorMap* tm) {
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  // L2 promotion of the MN-major boxes (rows of 128 / 64 / 32 bytes at large strides)
  static const int promo_env = getenv("CPD_I8_PROMO") ? atoi(getenv("CPD_I8_PROMO")) : 3;
  const CUtensorMapL2promotion promo_mc = promo_env == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                                          : promo_env == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                                          : promo_env == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                                           : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  uint8_t* base = const_cast<uint8_t*>(dv.planes);
  const cuuint64_t ps = (cuuint64_t)dv.plane_stride;
  const cuuint64_t KF = (cuuint64_t)(g.Kfull ? g.Kfull : g.K);  // K extent of the map (K chunks)
  CUresult r;
  if (L == D_KCW) {  // [P2][Mrows][Qp]: slabs of Mrows rows of Qp bytes
    cuuint64_t dims[4] = {(cuuint64_t)g.Qp, (cuuint64_t)g.Mrows, (cuuint64_t)g.P2, (cuuint64_t)kND};
    cuuint64_t strides[3] = {(cuuint64_t)g.Qp, (cuuint64_t)g.Qp * g.Mrows, ps};
    cuuint32_t box[4] = {32, (cuuint32_t)kBM, 1, (cuuint32_t)kND}, es[4] = {1, 1, 1, 1};
    r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else if (L == D_KC) {  // rows of ipad bytes (K = w)
    cuuint64_t dims[3] = {KF, (cuuint64_t)g.Mrows, (cuuint64_t)kND};
    cuuint64_t strides[2] = {(cuuint64_t)dv.ipad, ps};
    cuuint32_t box[3] = {32, (cuuint32_t)kBM, (cuuint32_t)kND}, es[3] = {1, 1, 1};
    r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else if (L == D_MCP) {
    if (g.Mo == 1) {
      cuuint64_t dims[4] = {(cuuint64_t)dv.ipad, KF, (cuuint64_t)g.pre, (cuuint64_t)kND};
      cuuint64_t strides[3] = {(cuuint64_t)dv.ipad, (cuuint64_t)dv.ipad * KF, ps};
      cuuint32_t box[4] = {(cuuint32_t)kBM, 32, 1, (cuuint32_t)kND}, es[4] = {1, 1, 1, 1};
      r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, promo_mc, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
      cuuint64_t dims[5] = {(cuuint64_t)dv.ipad, (cuuint64_t)g.Mo, KF, (cuuint64_t)g.pre, (cuuint64_t)kND};
      cuuint64_t strides[4] = {(cuuint64_t)dv.ipad, (cuuint64_t)dv.ipad * g.Mo, (cuuint64_t)dv.ipad * g.Mo * KF, ps};
      cuuint32_t box[5] = {(cuuint32_t)kBM, 1, 32, 1, (cuuint32_t)kND}, es[5] = {1, 1, 1, 1, 1};
      r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 5, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, promo_mc, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
  } else {  // unpadded: post contiguous (D_MCF: the flattened padded extent postF)
    const int mcw = (L == D_MC128 || L == D_MCF) ? 128 : L == D_MC64 ? 64 : 32;
    const cuuint64_t pe = (cuuint64_t)(L == D_MCF ? g.postF : g.post);
    cuuint64_t dims[4] = {pe, KF, (cuuint64_t)g.pre, (cuuint64_t)kND};
    cuuint64_t strides[3] = {pe, KF * pe, ps};
    cuuint32_t box[4] = {(cuuint32_t)mcw, 32, (cuuint32_t)(kBM / mcw), (cuuint32_t)kND}, es[4] = {1, 1, 1, 1};
    const CUtensorMapSwizzle sw =
        mcw == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : mcw == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B;
    r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
            promo_mc, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  return r == CUDA_SUCCESS;
}

template <int L, int RP>
cudaError_t run_i8d(int grid, const Geo& g, const uint8_t* Bimg, const int* F, const int* Xexp, double* out,
                    int beta, const CUtensorMap& tm, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(ttm_i8d_kernel<L, RP>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemD);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  static const int dbg = getenv("CPD_I8_DBG") ? atoi(getenv("CPD_I8_DBG")) : 0;  // profiling switches
  if (g.cl == 1) {
    ttm_i8d_kernel<L, RP><<<grid, kThreadsD, kSmemD, st>>>(g, Bimg, F, Xexp, out, beta, tm, dbg);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kThreadsD);
  cfg.dynamicSmemBytes = kSmemD;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)g.cl;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, ttm_i8d_kernel<L, RP>, g, Bimg, F, Xexp, out, beta, tm, dbg);
}

}  // namespace

size_t ttm_i8_workspace_bytes(int64_t K, int ncols) {
  Geo g = make_geo(1, K, 1, ncols, false);  // the 16-column padding bounds the 8-column one
  return (size_t)g.ntn * g.nkc * g.bstride + kMaxColsI8 * sizeof(int);
}

cudaError_t launch_absmax_exp(const double* x, int64_t n, double* partial, int* e_out, cudaStream_t st,
                              double* max_out) {
  g_launches += 2;
  absmax_partial_kernel<<<kNormBlocks, 256, 0, st>>>(x, n, partial);
  absmax_final_kernel<<<1, 32, 0, st>>>(partial, kNormBlocks, e_out, max_out);
  return cudaGetLastError();
}

cudaError_t launch_slice_digits(const double* X, int64_t n, int64_t w, const int* Xexp, uint8_t* planes,
                                cudaStream_t st) {
  if (((uintptr_t)X % 16) != 0 || w <= 0 || n % w != 0) return cudaErrorInvalidValue;
  const int64_t ipad = digit_inner_pad(w), ps = digit_plane_bytes(n, w);
  if (ipad != w) {
    cudaError_t e = cudaMemsetAsync(planes, 0, (size_t)kND * ps, st);
    if (e != cudaSuccess) return e;
  }
  g_launches++;
  static const int slow = getenv("CPD_SLOW_SLICE") ? 1 : 0;
  slice_digits_kernel<<<148 * 8, 256, 0, st>>>(X, n, w, ipad, ps, Xexp, planes, slow);
  return cudaGetLastError();
}

// digit-kernel layout for a TTM view [pre, K, post] of a tensor whose digit planes have
// innermost extent w (padded to ipad); -1 if none applies
int digit_layout(int64_t pre, int64_t K, int64_t post, int64_t w, int64_t ipad) {
  if (post == 1) return K == w ? D_KC : -1;
  if (post % w != 0) return -1;
  if (ipad == w) {
    if ((post % kBM) == 0) return D_MC128;
    if (post == 64 && pre % 2 == 0) return D_MC64;
    if (post == 32 && pre % 4 == 0) return D_MC32;
  }
  static const bool no_mcf = getenv("CPD_I8_NO_MCF") != nullptr;  // experiment switch
  if (!no_mcf && ipad != w && post / w > 1 && ((post / w) * ipad) % kBM == 0) return D_MCF;
  return ipad >= kBM ? D_MCP : -1;  // tiles of 128 rows over the innermost mode (no box overhang)
}

namespace {
// one digit-kernel launch of layout Ld over the geometry g (its B image already in Bimg): tile counts of
// the padded layouts, the CTA-pair cluster, the tensor map.  *launched = false: no tensor map (caller
// falls back)
cudaError_t launch_digit_geo(int Ld, Geo gd, const DigitView& dv, const uint8_t* Bimg, const int* F,
                             const int* Xexp, double* out, int beta, cudaStream_t st, bool* launched) {
  *launched = false;
  if (Ld == D_MCP) {
    gd.w = dv.w;
    gd.ipad = dv.ipad;
    gd.Mo = gd.post / dv.w;
    gd.wb = (int)((dv.w + kBM - 1) / kBM);
    gd.nmt = gd.pre * gd.Mo * gd.wb;
    gd.ntiles = gd.nmt * gd.ntn;
  } else if (Ld == D_MCF) {
    gd.w = dv.w;
    gd.ipad = dv.ipad;
    gd.Mo = gd.post / dv.w;
    gd.postF = gd.Mo * dv.ipad;
    gd.nmt = gd.pre * gd.postF / kBM;
    gd.ntiles = gd.nmt * gd.ntn;
  }
  // N tiles of one M tile on one cluster with the A box multicast (2 or 4 N tiles)
  static const bool no_mc = getenv("CPD_I8_NO_MULTICAST") != nullptr;
  // pairs only: a 4-CTA cluster couples four MMA-bound CTAs to the slowest (C5: 53 -> 73 ms)
  static const int cl_env = getenv("CPD_I8_CLUSTER") ? atoi(getenv("CPD_I8_CLUSTER")) : 2;
  if (!no_mc && gd.ntn % 2 == 0 && (cl_env == 2 || cl_env == 4) && gd.ntn % cl_env == 0 &&
      sm_count() % cl_env == 0)
    gd.cl = cl_env;
  // persistent grid: one CTA (pair) per SM, but one SM (pair) left free when that does not raise the most
  // tiles any CTA runs -- the side stream's single-CTA Γ^{-1} launch then finds an SM without delaying a
  // TTM CTA by its duration (C2: 8192 tiles need 56 rounds on 148 or 147 CTAs alike)
  const int64_t units = gd.cl == 1 ? gd.ntiles : gd.nmt * (gd.ntn / gd.cl);
  int64_t slots = sm_count() / gd.cl;
  static const bool no_spare = getenv("CPD_I8_NO_SPARE_SM") != nullptr;  // experiment switch
  if (!no_spare && slots > 1 && (units + slots - 2) / (slots - 1) == (units + slots - 1) / slots) slots--;
  const int gridd = gd.cl * (int)std::min<int64_t>(units, slots);
  CUtensorMap tmd;
  if (!make_tmap_digits(Ld, dv, gd, &tmd)) return cudaSuccess;
  *launched = true;
  g_launches++;
  switch (gd.Rp) {
#define CPD_I8D_CASE(RP_)                                                                         \
  case RP_:                                                                                       \
    switch (Ld) {                                                                                 \
      case D_KC: return run_i8d<D_KC, RP_>(gridd, gd, Bimg, F, Xexp, out, beta, tmd, st);         \
      case D_KCW: return run_i8d<D_KCW, RP_>(gridd, gd, Bimg, F, Xexp, out, beta, tmd, st);       \
      case D_MC128: return run_i8d<D_MC128, RP_>(gridd, gd, Bimg, F, Xexp, out, beta, tmd, st);   \
      case D_MC64: return run_i8d<D_MC64, RP_>(gridd, gd, Bimg, F, Xexp, out, beta, tmd, st);     \
      case D_MC32: return run_i8d<D_MC32, RP_>(gridd, gd, Bimg, F, Xexp, out, beta, tmd, st);     \
      case D_MCF: return run_i8d<D_MCF, RP_>(gridd, gd, Bimg, F, Xexp, out, beta, tmd, st);       \
      default: return run_i8d<D_MCP, RP_>(gridd, gd, Bimg, F, Xexp, out, beta, tmd, st);         \
    }
    CPD_I8D_CASE(16)
    CPD_I8D_CASE(32)
    CPD_I8D_CASE(40)
    CPD_I8D_CASE(48)
    CPD_I8D_CASE(56)
    CPD_I8D_CASE(64)
#undef CPD_I8D_CASE
  }
  return cudaErrorInvalidValue;
}

// column exponents and the B digit image of rows [0, K) of B (one K chunk)
void factor_image(const double* B, int64_t K, const Geo& g, int* F, uint8_t* Bimg, cudaStream_t st) {
  g_launches += 2;
  col_exp_kernel<<<g.ncols, 256, 0, st>>>(B, K, g.ncols, F);
  const int64_t total = (int64_t)g.ntn * g.nkc * g.Rp * 32;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 8);
  b_image_kernel<<<blocks, 256, 0, st>>>(B, K, g, F, Bimg);
}
}  // namespace

cudaError_t launch_ttm_i8(const double* X, int64_t pre, int64_t K, int64_t post, const double* B, int ncols,
                          double* out, int beta, const int* Xexp, void* ws, size_t ws_bytes, cudaStream_t st,
                          const DigitView* dv) {
  if (pre <= 0 || post <= 0 || ncols <= 0) return cudaSuccess;
  if (K <= 0 || ncols > kMaxColsI8) return cudaErrorInvalidValue;
  static const bool no_digits = getenv("CPD_I8_NO_DIGITS") != nullptr;
  const int Ld = dv && dv->planes ? digit_layout(pre, K, post, dv->w, dv->ipad) : -1;
  const bool digits = Ld >= 0 && !no_digits && ((uintptr_t)dv->planes % 16) == 0;
  if (K > kMaxKI8 && !digits) return cudaErrorInvalidValue;
  const int64_t Kc0 = std::min<int64_t>(K, kMaxKI8);
  const size_t img_max = ttm_i8_workspace_bytes(Kc0, ncols) - kMaxColsI8 * sizeof(int);
  if (ws_bytes < img_max + kMaxColsI8 * sizeof(int)) return cudaErrorInvalidValue;
  uint8_t* Bimg = static_cast<uint8_t*>(ws);
  int* F = reinterpret_cast<int*>(static_cast<uint8_t*>(ws) + img_max);
  if (digits) {
    // K chunks of <= kMaxKI8 (|D_d| < 2^31), each its own exponents and image, accumulated with beta = 1
    for (int64_t k0 = 0; k0 < K; k0 += kMaxKI8) {
      const int64_t Kc = std::min<int64_t>(kMaxKI8, K - k0);
      Geo g = make_geo(pre, Kc, post, ncols, true);
      g.kofs = k0;
      g.Kfull = K;
      factor_image(B + k0 * ncols, Kc, g, F, Bimg, st);
      bool launched = false;
      cudaError_t e = launch_digit_geo(Ld, g, *dv, Bimg, F, Xexp, out, beta || k0 > 0, st, &launched);
      if (e != cudaSuccess) return e;
      if (!launched) {
        if (k0 > 0 || K > kMaxKI8) return cudaErrorInvalidValue;
        break;  // converting kernel below
      }
      if (k0 + Kc >= K) return cudaSuccess;
    }
  }
  Geo g = make_geo(pre, K, post, ncols, false);
  factor_image(B, K, g, F, Bimg, st);
  g_launches++;
  // loader: TMA when the layout allows it (16-byte aligned strides; MC tiles must not straddle
  // the prefix index, i.e. post % 128 == 0), else register loads
  static const bool no_tma = getenv("CPD_I8_NO_TMA") != nullptr;
  const bool mc = post > 1;
  const bool aligned = ((uintptr_t)X % 16) == 0;
  int L = mc ? L_MC : L_KC;
  CUtensorMap tm;
  std::memset(&tm, 0, sizeof(tm));
  if (!no_tma && aligned && (mc ? (post % kBM) == 0 : (K % 2) == 0)) {
    const int Lt = mc ? L_MC_TMA : L_KC_TMA;
    if (make_tmap(Lt, X, g, &tm)) L = Lt;
  }
  const int grid = (int)std::min<int64_t>(g.ntiles, sm_count());
  switch (g.Rp) {
    case 16: return dispatch_i8<16>(L, grid, X, g, Bimg, F, Xexp, out, beta, tm, st);
    case 32: return dispatch_i8<32>(L, grid, X, g, Bimg, F, Xexp, out, beta, tm, st);
    case 48: return dispatch_i8<48>(L, grid, X, g, Bimg, F, Xexp, out, beta, tm, st);
    case 64: return dispatch_i8<64>(L, grid, X, g, Bimg, F, Xexp, out, beta, tm, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_ttm_i8_block(int64_t P, int64_t Mrows, int64_t Qp, const double* Bpad, int ncols, double* out,
                                int beta, const int* Xexp, void* ws, size_t ws_bytes, cudaStream_t st,
                                const DigitView& dv) {
  if (P <= 0 || Mrows <= 0 || ncols <= 0) return cudaSuccess;
  if (!dv.planes || Qp <= 0 || Qp % 16 || ((uintptr_t)dv.planes % 16) || ncols > kMaxColsI8)
    return cudaErrorNotSupported;
  const int64_t nkq = (Qp + 31) / 32, Ks = 32 * nkq;  // K rows of Bpad per slab
  const size_t img_max = ttm_i8_workspace_bytes(kMaxKI8, ncols) - kMaxColsI8 * sizeof(int);
  if (ws_bytes < img_max + kMaxColsI8 * sizeof(int)) return cudaErrorInvalidValue;
  uint8_t* Bimg = static_cast<uint8_t*>(ws);
  int* F = reinterpret_cast<int*>(static_cast<uint8_t*>(ws) + img_max);
  auto one = [&](int64_t p0, int64_t np, int64_t q0, int64_t K, int nk, bool first) -> cudaError_t {
    Geo g = make_geo(Mrows, K, 1, ncols, true);
    g.nkq = nk;
    g.p0 = p0;
    g.kofs = q0;
    g.P2 = P;
    g.Qp = Qp;
    const double* Bc = Bpad + (p0 * Ks + q0) * ncols;
    factor_image(Bc, K, g, F, Bimg, st);
    bool launched = false;
    cudaError_t e = launch_digit_geo(D_KCW, g, dv, Bimg, F, Xexp, out, beta || !first, st, &launched);
    if (e == cudaSuccess && !launched) e = cudaErrorNotSupported;
    (void)np;
    return e;
  };
  if (Ks <= kMaxKI8) {  // whole slabs per launch
    const int64_t spc = kMaxKI8 / Ks;
    for (int64_t p0 = 0; p0 < P; p0 += spc) {
      const int64_t np = std::min(spc, P - p0);
      cudaError_t e = one(p0, np, 0, np * Ks, (int)nkq, p0 == 0);
      if (e != cudaSuccess) return e;
    }
  } else {  // slabs longer than one launch: K chunks inside each slab
    for (int64_t p = 0; p < P; p++)
      for (int64_t q0 = 0; q0 < Ks; q0 += kMaxKI8) {
        const int64_t K = std::min<int64_t>(kMaxKI8, Ks - q0);
        cudaError_t e = one(p, 1, q0, K, (int)(K / 32), p == 0 && q0 == 0);
        if (e != cudaSuccess) return e;
      }
  }
  return cudaSuccess;
}

}  // namespace cpd
