// HBM-bound streams: batched TTV (mTTV) levels of the dimension trees and the PP
// first-order corrections, the synthetic-tensor generator, and reductions.
//
// "Other contractions (transforming one intermediate into another
// intermediate) are done via batched TTV"; "the mTTV kernel is vertical
// communication (memory bandwidth) bound"; Eq. 6:
// U^(n,i)(x,k) = Σ_y M_p^(n,i)(x,y,k) dA^(i)(y,k) is the same contraction.
//
// B200 design: intermediates are stored [kept modes..., R] with R
// innermost, so contracting any kept mode reads X as [pre, K, C = post*R] and every
// warp load is a contiguous 512-byte row segment (double2 per lane).  A CTA owns one
// p and 64 columns; its 8 warps split the K rows (fixed interleave) and reduce through
// shared memory in a fixed order (deterministic, no atomics).
#include <algorithm>
#include <cstdlib>

#include "kernels.h"

namespace cpd {
std::atomic<long long> g_launches{0};
namespace {

constexpr int MT_THREADS = 256;
constexpr int MT_COLS = 64;  // columns per CTA (32 lanes x double2)

// One CTA = one work item (job, p, 64-column chunk, K-split); 8 warps interleave the rows
// of the split, 4 rows in flight per warp; fixed-order shared-memory reduction.  A launch
// may carry several jobs with the same output shape (the N-1 U-streams of one PP mode,
// Eq. 6): their partial sums go to ws[slot][p*C + c] and mttv_reduce_kernel adds base
// (M_p^(n)) and the slots in job/split order (deterministic).  A single job with no
// K-split writes out directly (out = beta*out + sum).
struct MttvJob {
  const double* X;
  const double* v;
  int64_t pre, K, C, rps, item0, slot0;
  int nchunks, ks;
  int ppc;  // p values per CTA: 64 / C when the row is narrower than a CTA's 64 columns (C4: C = R = 32)
};
struct MttvJobs {
  MttvJob j[8];
  int J;
  int64_t E;  // output elements (pre*C, same for every job)
};

__device__ __forceinline__ double* map_dst(const OutMap& m, double* out, int64_t e) {
  if (m.nq == 0) return out + e;
  const int64_t q = e / m.chunk;
  double* d = m.dst[0];
#pragma unroll
  for (int k = 1; k < 8; k++) d = (q == k) ? m.dst[k] : d;  // static indices: no local copy of the map
  return d + (e - q * m.chunk);
}

// 4 CTAs (32 warps, 128 loads of 512 bytes) resident per SM: at 80 registers only 3 fit, and the
// stream was latency-bound at ~4.6-5.6 TB/s on the large-node contractions (C3/C4 roots)
template <bool VEC2, bool VV, bool PACK, int OCC>
__global__ void __launch_bounds__(MT_THREADS, PACK ? 3 : OCC)
    mttv_kernel(MttvJobs jobs, int R, double* __restrict__ out, int beta, double* __restrict__ ws, OutMap om) {
  __shared__ double red[8][MT_COLS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // this CTA's job, read from the parameter space with static indices only (a dynamically indexed
  // copy of the job table went to the local stack)
  struct {
    const double* X;
    const double* v;
    int64_t pre, K, C, rps, item0, slot0;
    int nchunks, ks, ppc;
  } jb = {jobs.j[0].X, jobs.j[0].v, jobs.j[0].pre, jobs.j[0].K, jobs.j[0].C, jobs.j[0].rps, jobs.j[0].item0,
          jobs.j[0].slot0, jobs.j[0].nchunks, jobs.j[0].ks, jobs.j[0].ppc};
#pragma unroll
  for (int q = 1; q < 8; q++) {
    const bool sel = q < jobs.J && (int64_t)blockIdx.x >= jobs.j[q].item0;
    jb.X = sel ? jobs.j[q].X : jb.X;
    jb.v = sel ? jobs.j[q].v : jb.v;
    jb.K = sel ? jobs.j[q].K : jb.K;
    jb.C = sel ? jobs.j[q].C : jb.C;
    jb.rps = sel ? jobs.j[q].rps : jb.rps;
    jb.item0 = sel ? jobs.j[q].item0 : jb.item0;
    jb.slot0 = sel ? jobs.j[q].slot0 : jb.slot0;
    jb.nchunks = sel ? jobs.j[q].nchunks : jb.nchunks;
    jb.ks = sel ? jobs.j[q].ks : jb.ks;
    jb.pre = sel ? jobs.j[q].pre : jb.pre;
    jb.ppc = sel ? jobs.j[q].ppc : jb.ppc;
  }
  const int64_t local = (int64_t)blockIdx.x - jb.item0;
  const int split = (int)(local % jb.ks);
  const int64_t rest = local / jb.ks;
  const int ppc = PACK ? jb.ppc : 1;
  const int64_t p = (rest / jb.nchunks) * ppc;  // first p of this CTA
  const int chunk = (int)(rest % jb.nchunks);
  const int64_t K = jb.K, C = jb.C;
  const double* __restrict__ v = jb.v;
  const int64_t k0 = split * jb.rps;
  const int64_t k1 = min(K, k0 + jb.rps);
  // virtual column cv in [0, 64) of the chunk; with ppc > 1 it spans ppc consecutive rows p of width C
  const int64_t cvA = (int64_t)chunk * MT_COLS + (VEC2 ? 2 * lane : lane);
  const int64_t cvB = VEC2 ? cvA + 1 : cvA + 32;
  const int64_t pA = ppc > 1 ? p + cvA / C : p, pB = ppc > 1 ? p + cvB / C : p;
  const int64_t cA = ppc > 1 ? cvA % C : cvA, cB = ppc > 1 ? cvB % C : cvB;
  const bool okA = ppc > 1 ? pA < jb.pre : cA < C, okB = ppc > 1 ? pB < jb.pre : cB < C;
  const int rA = okA ? (int)(cA % R) : 0, rB = okB ? (int)(cB % R) : 0;
  const double* Xp = jb.X + pA * K * C;    // VEC2: cB = cA + 1 lies in the same row (C even)
  const double* XpB = jb.X + pB * K * C;
  double sA = 0.0, sB = 0.0;
  if (okA) {
    int64_t y = k0 + warp;
    for (; y + 24 < k1; y += 32) {
      double a[4], b[4], va[4], vb[4];
      if (VEC2) {
#pragma unroll
        for (int u = 0; u < 4; u++) {
          double2 x2 = __ldcs(reinterpret_cast<const double2*>(Xp + (y + 8 * u) * C + cA));
          a[u] = x2.x;
          b[u] = x2.y;
        }
      } else {
#pragma unroll
        for (int u = 0; u < 4; u++) {
          a[u] = __ldcs(Xp + (y + 8 * u) * C + cA);
          b[u] = okB ? __ldcs(XpB + (y + 8 * u) * C + cB) : 0.0;
        }
      }
      if (VV) {
#pragma unroll
        for (int u = 0; u < 4; u++) {
          double2 v2 = __ldg(reinterpret_cast<const double2*>(v + (y + 8 * u) * R + rA));
          va[u] = v2.x;
          vb[u] = v2.y;
        }
      } else {
#pragma unroll
        for (int u = 0; u < 4; u++) {
          va[u] = __ldg(v + (y + 8 * u) * R + rA);
          vb[u] = okB ? __ldg(v + (y + 8 * u) * R + rB) : 0.0;
        }
      }
#pragma unroll
      for (int u = 0; u < 4; u++) {
        sA = fma(a[u], va[u], sA);
        sB = fma(b[u], vb[u], sB);
      }
    }
    for (; y < k1; y += 8) {
      sA = fma(Xp[y * C + cA], v[y * R + rA], sA);
      if (okB) sB = fma(XpB[y * C + cB], v[y * R + rB], sB);
    }
  }
  if (VEC2) {
    red[warp][2 * lane] = sA;
    red[warp][2 * lane + 1] = sB;
  } else {
    red[warp][lane] = sA;
    red[warp][lane + 32] = sB;
  }
  __syncthreads();
  if (threadIdx.x < MT_COLS) {
    const int64_t cv = (int64_t)chunk * MT_COLS + threadIdx.x;
    if (ppc > 1 ? p + cv / C < jb.pre : cv < C) {
      double s = red[0][threadIdx.x];
#pragma unroll
      for (int w = 1; w < 8; w++) s += red[w][threadIdx.x];
      const int64_t e = p * C + cv;  // rows p.. of width C are contiguous in the output
      if (ws == nullptr) {
        *map_dst(om, out, e) = beta ? out[e] + s : s;
        if (om.nq) __threadfence_system();  // fused RS: the store may target a peer GPU (NVLink)
      } else {
        ws[(jb.slot0 + split) * jobs.E + e] = s;
      }
    }
  }
}

// out[e] = (base ? base[e] : beta*out[e]) + Σ_slot ws[slot*n + e]   (slot order fixed)
__global__ void mttv_reduce_kernel(const double* __restrict__ ws, int slots, int64_t n, const double* __restrict__ base,
                                   double* __restrict__ out, int beta, OutMap om) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    double s = base ? base[e] : (beta ? out[e] : 0.0);
    for (int k = 0; k < slots; k++) s += ws[k * n + e];
    *map_dst(om, out, e) = s;
  }
  if (om.nq) __threadfence_system();  // fused RS: stores to peers complete before the barrier collective
}

// Two contractions of one node in one read (PP-init's multi-output descent, SURVEY a9 "deeper levels
// from each parent in one multi-output pass"): X viewed as [P][K1][Q][K2][C],
//   out1[p][q][k2][c] = Σ_{k1} X[p][k1][q][k2][c] v1[k1][c % R]   (contract K1)
//   out2[p][k1][q][c] = Σ_{k2} X[p][k1][q][k2][c] v2[k2][c % R]   (contract K2).
// A CTA owns (p, q, a block of 32 k1 rows, 64 columns) and walks all k2: out2 of its rows completes
// in registers; out1 gets the block's partial (8 warps x 4 rows, fixed-order shared-memory sum per
// group of 4 k2), written to ws[k1 block] (or straight to out1 when K1 <= 32) and summed over the
// blocks in block order by mttv_reduce_kernel (deterministic).
constexpr int DU_THREADS = 512;             // 16 warps x 2 k1 rows
constexpr int DU_WARPS = DU_THREADS / 32;
constexpr int DU_RPW = 2;                   // k1 rows per warp
constexpr int DU_ROWS = DU_WARPS * DU_RPW;  // k1 rows per CTA (32)
constexpr int DU_K2B = 4;                   // k2 values per shared-memory reduction
template <bool VEC2>
__global__ void __launch_bounds__(DU_THREADS, 2)
    mttv_dual_kernel(const double* __restrict__ X, int64_t P, int64_t K1, int64_t Q, int64_t K2, int64_t C, int R,
                     const double* __restrict__ v1, const double* __restrict__ v2, double* __restrict__ out1,
                     double* __restrict__ out2, double* __restrict__ ws, int nkb) {
  __shared__ double red[DU_K2B][DU_WARPS][MT_COLS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nch = (int)((C + MT_COLS - 1) / MT_COLS);
  int64_t b = blockIdx.x;
  const int ch = (int)(b % nch);
  b /= nch;
  const int kb = (int)(b % nkb);
  b /= nkb;
  const int64_t q = b % Q, p = b / Q;
  const int64_t cA = (int64_t)ch * MT_COLS + (VEC2 ? 2 * lane : lane);
  const int64_t cB = VEC2 ? cA + 1 : cA + 32;
  const bool okA = cA < C, okB = cB < C;
  const int rA = okA ? (int)(cA % R) : 0, rB = okB ? (int)(cB % R) : 0;
  int64_t y[DU_RPW];
  bool yok[DU_RPW];
  const double* xr[DU_RPW];
  double w1a[DU_RPW], w1b[DU_RPW], a2[DU_RPW], b2[DU_RPW];
#pragma unroll
  for (int u = 0; u < DU_RPW; u++) {
    y[u] = (int64_t)kb * DU_ROWS + warp + DU_WARPS * u;
    yok[u] = y[u] < K1;
    xr[u] = X + ((p * K1 + (yok[u] ? y[u] : 0)) * Q + q) * K2 * C;
    w1a[u] = (yok[u] && okA) ? v1[y[u] * R + rA] : 0.0;
    w1b[u] = (yok[u] && okB) ? v1[y[u] * R + rB] : 0.0;
    a2[u] = b2[u] = 0.0;
  }
  const int64_t E1 = P * Q * K2 * C;
  for (int64_t k0 = 0; k0 < K2; k0 += DU_K2B) {
#pragma unroll
    for (int j = 0; j < DU_K2B; j++) {
      const int64_t k2 = k0 + j;
      double pa = 0.0, pb = 0.0;
      if (k2 < K2 && okA) {
        const double v2a = v2[k2 * R + rA], v2b = okB ? v2[k2 * R + rB] : 0.0;
#pragma unroll
        for (int u = 0; u < DU_RPW; u++) {
          if (!yok[u]) continue;
          double xa, xb;
          if (VEC2) {
            const double2 x2 = __ldcs(reinterpret_cast<const double2*>(xr[u] + k2 * C + cA));
            xa = x2.x;
            xb = x2.y;
          } else {
            xa = __ldcs(xr[u] + k2 * C + cA);
            xb = okB ? __ldcs(xr[u] + k2 * C + cB) : 0.0;
          }
          a2[u] = fma(xa, v2a, a2[u]);
          b2[u] = fma(xb, v2b, b2[u]);
          pa = fma(xa, w1a[u], pa);
          pb = fma(xb, w1b[u], pb);
        }
      }
      if (VEC2) {
        red[j][warp][2 * lane] = pa;
        red[j][warp][2 * lane + 1] = pb;
      } else {
        red[j][warp][lane] = pa;
        red[j][warp][lane + 32] = pb;
      }
    }
    __syncthreads();
    if (threadIdx.x < DU_K2B * MT_COLS) {
      const int j = threadIdx.x / MT_COLS, col = threadIdx.x % MT_COLS;  // 4 x 64 outputs
      const int64_t k2 = k0 + j, c = (int64_t)ch * MT_COLS + col;
      if (k2 < K2 && c < C) {
        double s = red[j][0][col];
#pragma unroll
        for (int w = 1; w < DU_WARPS; w++) s += red[j][w][col];
        const int64_t e = ((p * Q + q) * K2 + k2) * C + c;
        if (ws) ws[(int64_t)kb * E1 + e] = s;
        else out1[e] = s;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < DU_RPW; u++) {
    if (!yok[u]) continue;
    double* o = out2 + ((p * K1 + y[u]) * Q + q) * C;
    if (okA) o[cA] = a2[u];
    if (okB) o[cB] = b2[u];
  }
}

__global__ void scatter_copy_kernel(const double* __restrict__ src, int64_t n, OutMap om) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    *map_dst(om, nullptr, e) = src[e];
  __threadfence_system();
}

__global__ void slot_sum_kernel(const double* __restrict__ src, int nq, int64_t n, double* __restrict__ dst) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    double s = src[e];
    for (int q = 1; q < nq; q++) s += src[q * n + e];
    dst[e] = s;
  }
}

// ---- SplitMix64 counter hash (spec in synth/__init__.py) ----
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double hash_u(uint64_t key, uint64_t idx, uint64_t lane) {
  return (double)(splitmix64(key ^ (2ull * idx + lane)) >> 11) * 0x1.0p-53;
}

// T block [lo_0:hi_0, ..., lo_{N-1}:hi_{N-1}] (row-major, local extents b.ext) of a tensor of
// global shape b.shape: element li gets the hash of its GLOBAL row-major linear index
__global__ void noise_kernel(double* __restrict__ T, BlockGeo b, int kind, double stdv, uint64_t key) {
  int64_t n = 1;
  for (int m = 0; m < b.N; m++) n *= b.ext[m];
  for (int64_t li = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; li < n;
       li += (int64_t)gridDim.x * blockDim.x) {
    int64_t rem = li, gidx_s = 0, stride = 1;
    for (int m = b.N - 1; m >= 0; m--) {
      const int64_t c = rem % b.ext[m];
      rem /= b.ext[m];
      gidx_s += (b.lo[m] + c) * stride;
      stride *= b.shape[m];
    }
    const uint64_t gidx = (uint64_t)gidx_s;
    if (kind == 1) {
      T[li] = hash_u(key, gidx, 0);
    } else {
      double u1 = hash_u(key, gidx, 0), u2 = hash_u(key, gidx, 1);
      double zn = sqrt(-2.0 * log1p(-u1)) * cos(2.0 * 3.141592653589793 * u2);
      T[li] += stdv * zn;
    }
  }
}

struct KrpArgs {
  const double* A[8];
  int64_t s[8];
};

__global__ void krp_kernel(KrpArgs a, int nf, int R, int64_t rows, double* __restrict__ KR) {
  const int64_t n = rows * R;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t q = e / R;
    int r = (int)(e - q * R);
    // decode q with the first mode slowest; multiply in ascending mode order
    int64_t idx[8];
    int64_t rem = q;
    for (int m = nf - 1; m >= 0; m--) {
      idx[m] = rem % a.s[m];
      rem /= a.s[m];
    }
    double pr = a.A[0][idx[0] * R + r];
    for (int m = 1; m < nf; m++) pr *= a.A[m][idx[m] * R + r];
    KR[e] = pr;
  }
}

__global__ void norm2_partial_kernel(const double* __restrict__ x, int64_t n, double* partial) {
  __shared__ double red[32];
  double s = 0.0;
  const int64_t n2 = n / 2;
  const double2* x2 = reinterpret_cast<const double2*>(x);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2; i += stride) {
    double2 v = __ldcs(x2 + i);
    s = fma(v.x, v.x, s);
    s = fma(v.y, v.y, s);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && (n & 1)) s = fma(x[n - 1], x[n - 1], s);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = (threadIdx.x < blockDim.x / 32) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
  }
}

// single CTA, fixed order: mode 0: dst = Σ x*y; mode 1: Σ x*x; mode 2: Σ x
__global__ void dot_kernel(const double* __restrict__ x, const double* __restrict__ y, int64_t n,
                           double* dst, int mode) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
    s = mode == 2 ? s + x[i] : fma(x[i], mode == 0 ? y[i] : x[i], s);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = (threadIdx.x < blockDim.x / 32) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) dst[0] = s;
  }
}

__global__ void sub_kernel(const double* __restrict__ x, const double* __restrict__ y,
                           double* __restrict__ z, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    z[i] = x[i] - y[i];
}

}  // namespace

// occ3: the 3-CTAs-per-SM build (80 registers) -- used for the PP filler-stream launches, which
// then leave room on every SM for the critical main-stream kernels (C2 PP sweep 0.645 -> 0.615 ms
// with 3/SM everywhere; the large root contractions of C3/C4 prefer 4/SM)
// experiment switch CPD_MTTV_CARVEOUT: the mTTV kernels prefer the maximum shared-memory carveout, so an
// SM running them never has to drain to host the large-smem update / Γ^-1 kernels of the other streams
// (measured: C2 PP sweep 0.62 -> 0.93 ms -- the smaller L1 costs the streams more; off by default)
template <typename K>
void carveout(K kern) {
  static const bool on = getenv("CPD_MTTV_CARVEOUT") != nullptr;
  if (on) cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
}

void launch_mttv_variant(bool vec2, bool vv, bool pack, bool occ3, unsigned grid, const MttvJobs& jobs, int R,
                         double* out, int beta, double* ws, const OutMap& om, cudaStream_t st) {
  // experiment switch CPD_FILLER_PAD_KB = k: the filler-stream (occ3) launches use the 64-register build
  // with k KB of unused dynamic shared memory per CTA, so the shared memory (not the registers) caps them at
  // 3 CTAs per SM and 16K registers stay free for a main-stream mTTV CTA beside them
  static const int pad_kb = getenv("CPD_FILLER_PAD_KB") ? atoi(getenv("CPD_FILLER_PAD_KB")) : 0;
  const size_t dyn = (occ3 && pad_kb > 0) ? (size_t)pad_kb * 1024 : 0;
  if (dyn) occ3 = false;
#define CPD_MTTV_V(V2, VV_, PK, O)                                                             \
  do {                                                                                         \
    static bool set_ = false;                                                                  \
    if (!set_) {                                                                               \
      carveout(mttv_kernel<V2, VV_, PK, O>);                                                   \
      if (pad_kb > 0)                                                                          \
        cudaFuncSetAttribute(mttv_kernel<V2, VV_, PK, O>,                                      \
                             cudaFuncAttributeMaxDynamicSharedMemorySize, pad_kb * 1024);       \
      set_ = true;                                                                             \
    }                                                                                          \
    mttv_kernel<V2, VV_, PK, O><<<grid, MT_THREADS, dyn, st>>>(jobs, R, out, beta, ws, om);   \
  } while (0)
  if (pack) {
    if (vec2 && vv) CPD_MTTV_V(true, true, true, 3);
    else if (vec2) CPD_MTTV_V(true, false, true, 3);
    else CPD_MTTV_V(false, false, true, 3);
  } else if (occ3) {
    if (vec2 && vv) CPD_MTTV_V(true, true, false, 3);
    else if (vec2) CPD_MTTV_V(true, false, false, 3);
    else CPD_MTTV_V(false, false, false, 3);
  } else {
    if (vec2 && vv) CPD_MTTV_V(true, true, false, 4);
    else if (vec2) CPD_MTTV_V(true, false, false, 4);
    else CPD_MTTV_V(false, false, false, 4);
  }
#undef CPD_MTTV_V
}

cudaError_t launch_slot_sum(const double* src, int nq, int64_t n, double* dst, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  g_launches++;
  slot_sum_kernel<<<(unsigned)blocks, 256, 0, st>>>(src, nq, n, dst);
  return cudaGetLastError();
}

cudaError_t launch_mttv_multi(const MttvSpec* specs, int J, int R, const double* base, double* out, int beta,
                              double* ws, int64_t ws_elems, cudaStream_t st, const OutMap* map, bool occ3,
                              int waves_override, MPending* defer) {
  if (J < 1 || J > 8) return cudaErrorInvalidValue;
  if (defer) *defer = MPending{};
  OutMap om{};
  if (map) om = *map;
  MttvJobs jobs{};
  jobs.J = J;
  jobs.E = specs[0].pre * specs[0].post * R;
  bool vec2 = true, vv = (R % 2) == 0;
  int64_t items = 0, slots = 0;
  for (int q = 0; q < J; q++) {
    const MttvSpec& sp = specs[q];
    MttvJob& jb = jobs.j[q];
    jb.X = sp.X;
    jb.v = sp.v;
    jb.pre = sp.pre;
    jb.K = sp.K;
    jb.C = sp.post * R;
    if (jb.pre * jb.C != jobs.E || jb.K <= 0) return cudaErrorInvalidValue;
    jb.nchunks = (int)((jb.C + MT_COLS - 1) / MT_COLS);
    jb.ppc = 1;
    static const bool no_pack = getenv("CPD_MTTV_NO_PACK") != nullptr;  // experiment switch
    if (!no_pack && jb.C < MT_COLS && MT_COLS % jb.C == 0) {  // several narrow rows per CTA
      jb.ppc = (int)(MT_COLS / jb.C);
      jb.nchunks = 1;
    }
    vec2 = vec2 && (jb.C % 2) == 0 && ((uintptr_t)sp.X % 16) == 0;
    vv = vv && ((uintptr_t)sp.v % 16) == 0;
    const int64_t items0 = (jb.pre + jb.ppc - 1) / jb.ppc * jb.nchunks;
    // split K so the whole grid is >= ~`waves` waves of 4 resident CTAs per SM; every split adds a
    // partial-sum slot and the reduce pass, so the split stops at 2 waves (8 waves measured slower
    // on the C2 PP operator streams: PP sweep 0.736 -> 0.65 ms with at most 2 splits)
    static const int waves_env = getenv("CPD_MTTV_WAVES") ? std::max(1, atoi(getenv("CPD_MTTV_WAVES"))) : 2;
    const int waves = waves_override > 0 ? waves_override : waves_env;
    int64_t ks = (148 * 4 * waves / J + items0 - 1) / items0;
    if (ks > jb.K / 64) ks = jb.K / 64;
    static const int ks_max = getenv("CPD_MTTV_MAXKS") ? atoi(getenv("CPD_MTTV_MAXKS")) : 16;  // experiment switch
    if (ks > ks_max) ks = ks_max;
    if (ks < 1) ks = 1;
    jb.ks = (int)ks;
    jb.rps = (jb.K + ks - 1) / ks;
    jb.item0 = items;
    jb.slot0 = slots;
    items += items0 * ks;
    slots += ks;
  }
  const bool direct = (J == 1 && slots == 1 && base == nullptr);
  if (!direct && (ws == nullptr || slots * jobs.E > ws_elems)) {
    // not enough workspace: fall back to one direct launch per job, no K-split
    if (base) {
      cudaError_t e = cudaMemcpyAsync(out, base, sizeof(double) * jobs.E, cudaMemcpyDeviceToDevice, st);
      if (e != cudaSuccess) return e;
      beta = 1;
    }
    for (int q = 0; q < J; q++) {
      MttvJobs one{};
      one.J = 1;
      one.E = jobs.E;
      one.j[0] = jobs.j[q];
      one.j[0].ks = 1;
      one.j[0].rps = one.j[0].K;
      one.j[0].item0 = 0;
      one.j[0].slot0 = 0;
      int64_t grid = (one.j[0].pre + one.j[0].ppc - 1) / one.j[0].ppc * one.j[0].nchunks;
      g_launches++;
      const OutMap none{};
      launch_mttv_variant(vec2, vv, one.j[0].ppc > 1, occ3, (unsigned)grid, one, R, out, q > 0 ? 1 : beta, nullptr,
                          none, st);
    }
    if (om.nq > 0) {  // the local result, then scattered to the owners' slots
      int64_t blocks = (jobs.E + 255) / 256;
      if (blocks > 148 * 8) blocks = 148 * 8;
      g_launches++;
      scatter_copy_kernel<<<(unsigned)blocks, 256, 0, st>>>(out, jobs.E, om);
    }
    return cudaGetLastError();
  }
  if (items > 0x7fffffff) return cudaErrorInvalidConfiguration;
  double* w = direct ? nullptr : ws;
  g_launches++;
  const OutMap km = direct ? om : OutMap{};
  bool pack = false;  // jobs of one launch share the output size, not C: any packed job selects the variant
  for (int q = 0; q < J; q++) pack = pack || jobs.j[q].ppc > 1;
  launch_mttv_variant(vec2, vv, pack, occ3, (unsigned)items, jobs, R, out, beta, w, km, st);
  if (!direct && defer && om.nq == 0) {
    *defer = MPending{ws, (int)slots, jobs.E, base, beta};
    return cudaGetLastError();
  }
  if (!direct) {
    g_launches++;
    int64_t blocks = (jobs.E + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    mttv_reduce_kernel<<<(unsigned)blocks, 256, 0, st>>>(ws, (int)slots, jobs.E, base, out, beta, om);
  }
  return cudaGetLastError();
}

cudaError_t launch_mttv_dual(const double* X, int64_t P, int64_t K1, int64_t Q, int64_t K2, int64_t C, int R,
                             const double* v1, const double* v2, double* out1, double* out2, double* ws,
                             int64_t ws_elems, cudaStream_t st) {
  if (P <= 0 || Q <= 0 || C <= 0 || K1 <= 0 || K2 <= 0) return cudaSuccess;
  static_assert(DU_THREADS >= DU_K2B * MT_COLS, "one reduction output per thread");
  const int nkb = (int)((K1 + DU_ROWS - 1) / DU_ROWS);
  const int64_t E1 = P * Q * K2 * C;
  if (nkb > 1 && (ws == nullptr || (int64_t)nkb * E1 > ws_elems)) return cudaErrorInvalidValue;
  const int64_t nch = (C + MT_COLS - 1) / MT_COLS;
  const int64_t grid = P * Q * nkb * nch;
  if (grid > 0x7fffffff) return cudaErrorInvalidConfiguration;
  const bool vec2 = (C % 2) == 0 && ((uintptr_t)X % 16) == 0;
  double* w = nkb > 1 ? ws : nullptr;
  g_launches++;
  if (vec2)
    mttv_dual_kernel<true><<<(unsigned)grid, DU_THREADS, 0, st>>>(X, P, K1, Q, K2, C, R, v1, v2, out1, out2, w, nkb);
  else
    mttv_dual_kernel<false><<<(unsigned)grid, DU_THREADS, 0, st>>>(X, P, K1, Q, K2, C, R, v1, v2, out1, out2, w, nkb);
  if (nkb > 1) {
    int64_t blocks = (E1 + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    g_launches++;
    mttv_reduce_kernel<<<(unsigned)blocks, 256, 0, st>>>(ws, nkb, E1, nullptr, out1, 0, OutMap{});
  }
  return cudaGetLastError();
}

cudaError_t launch_mttv(const double* X, int64_t pre, int64_t K, int64_t post, int R,
                        const double* v, double* out, int beta, double* ws, int64_t ws_elems, cudaStream_t st) {
  if (pre <= 0 || post * R <= 0) return cudaSuccess;
  MttvSpec sp{X, v, pre, K, post};
  return launch_mttv_multi(&sp, 1, R, nullptr, out, beta, ws, ws_elems, st);
}

cudaError_t launch_noise(double* T, const BlockGeo& b, int kind, double stdv, uint64_t seed, cudaStream_t st) {
  // key = splitmix64(seed), computed on the host with the same mix
  uint64_t z = seed + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  uint64_t key = z ^ (z >> 31);
  g_launches++;
  noise_kernel<<<148 * 8, 256, 0, st>>>(T, b, kind, stdv, key);
  return cudaGetLastError();
}

cudaError_t launch_krp(const double* const* A_dev, const int64_t* shape, int nf, int R, double* KR,
                       cudaStream_t st) {
  KrpArgs a{};
  int64_t rows = 1;
  for (int m = 0; m < nf; m++) {
    a.A[m] = A_dev[m];
    a.s[m] = shape[m];
    rows *= shape[m];
  }
  g_launches++;
  krp_kernel<<<148 * 8, 256, 0, st>>>(a, nf, R, rows, KR);
  return cudaGetLastError();
}

cudaError_t launch_norm2(const double* x, int64_t n, double* partial, double* dst, cudaStream_t st) {
  g_launches += 2;
  norm2_partial_kernel<<<kNormBlocks, 512, 0, st>>>(x, n, partial);
  dot_kernel<<<1, 1024, 0, st>>>(partial, nullptr, kNormBlocks, dst, 2);
  return cudaGetLastError();
}

cudaError_t launch_dot(const double* x, const double* y, int64_t n, double* dst, cudaStream_t st) {
  g_launches++;
  dot_kernel<<<1, 1024, 0, st>>>(x, y, n, dst, y ? 0 : 1);
  return cudaGetLastError();
}

cudaError_t launch_sub(const double* x, const double* y, double* z, int64_t n, cudaStream_t st) {
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) return cudaSuccess;
  g_launches++;
  sub_kernel<<<(unsigned)blocks, 256, 0, st>>>(x, y, z, n);
  return cudaGetLastError();
}

}  // namespace cpd
