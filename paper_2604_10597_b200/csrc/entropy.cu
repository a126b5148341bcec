// entropy.cu -- sm_100a kernels for the K-bin activation-entropy estimator and the
// on-device chunk rule (reference: proj/include/chunklab/entropy.hpp, chunk.hpp).
//
//   minmax      entropy.hpp:108-114  strided min/max + all-element finite check
//   histogram   entropy.hpp:116-126  exact detail::bin_index binning (bit-exact counts)
//   decide      entropy.hpp:130-164 + chunk.hpp:68-89, 206-218, 256-368
//
// Bit-exactness of the fp32 histogram: the reference bins in fp64 with
// floor((v-lo)/(hi-lo)*K).  The kernel bins in fp32 with a proven error bound
// delta on x = (v-lo_f)*s_f; whenever x lies within delta of an interior bin
// boundary (probability ~2*delta per sample) it recomputes the bin with the
// reference's exact fp64 operation sequence.  Away from boundaries floor(x) equals
// the reference's bin, so counts are bit-exact by construction.
#include <cuda_runtime.h>

#include <cfloat>
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "cl_internal.h"

#ifndef CL_DEVICE_CHECKS
#define CL_DEVICE_CHECKS 0
#endif
// lane_count_u8 counts with shared-memory reductions (1) or read-modify-write pairs (0)
// float4 loads in flight per min/max thread: 4 (C3 0.188 ms) beats 6 (0.200) and 8 (0.196)
#ifndef CL_MM_UNROLL
#define CL_MM_UNROLL 4
#endif
#ifndef CL_HIST_ATOMS
#define CL_HIST_ATOMS 1
#endif
#include "conv_common.cuh"
#include "range.cuh"
#include "tma_map.cuh"

namespace cl {
namespace {

constexpr int kThreads = 256;

__host__ __device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

using range::atomic_max_f64;
using range::finite_f32;
using range::finite_f64;

// detail::bin_index (entropy.hpp:87-94), operation-for-operation in fp64.  The
// int conversion reproduces x86-64 cvttsd2si (out-of-range -> INT_MIN), which is
// what the reference's static_cast<int> does on its build target; it only
// matters for Fixed-range outliers more than 2^31 bins away.
__device__ __forceinline__ int bin_index_exact(double v, double lo, double width, int k) {
  if (!(width > 0.0)) return 0;
  const double x = __dmul_rn(__ddiv_rn(__dsub_rn(v, lo), width), static_cast<double>(k));
  const double f = floor(x);
  int idx;
  if (!(f >= -2147483648.0 && f < 2147483648.0))
    idx = INT_MIN;
  else
    idx = static_cast<int>(f);
  if (idx < 0) idx = 0;
  if (idx >= k) idx = k - 1;
  return idx;
}

// Per-launch binning parameters, derived on device from the (allreduced) range.
//
// Fast path: x' = fma(v, s_f, c_f) approximates X' = (v - lo)*K/width - 0.5, so
// round-to-nearest(x') = floor(X) = the reference bin, unless x' lies within delta
// of a half-integer (X within delta of a bin edge).  delta bounds |x' - X'| for
// |v| <= max(|lo|,|hi|) + width:
//   |x' - X'| <= u*(|v|*S + |c| + |x'|) + |S - s_f|*|v| + |c - c_f|  (u = 2^-24)
// and is doubled; near-edge samples take the reference's exact fp64 path.
struct BinParams {
  double lo, width;  // exact fp64 range
  float s_f, c_f;    // fast-path fp32 affine map x' = v*s_f + c_f
  float thr;         // |x' - round(x')| > thr  <=>  within delta of an edge
  int k;
  int exact_only;    // fast path unusable (pathological fixed range)
};

__device__ BinParams make_bin_params_lohi(double lo, double hi, int k) {
  BinParams p;
  p.lo = lo;
  p.width = __dsub_rn(hi, lo);
  p.k = k;
  p.exact_only = 0;
  if (!(p.width > 0.0)) {  // degenerate range: everything in bin 0 (entropy.hpp:89)
    p.s_f = 0.f;
    p.c_f = 0.25f;  // x' = 0.25: bin 0, never near an edge
    p.thr = 0.5f;
    return p;
  }
  const double S = static_cast<double>(k) / p.width;
  const double c = -(lo * S) - 0.5;
  p.s_f = static_cast<float>(S);
  p.c_f = static_cast<float>(c);
  const double u = 5.9604644775390625e-08;  // 2^-24
  const double M = fmax(fabs(lo), fabs(hi)) + p.width;
  const double err = u * (M * S + fabs(c) + k + 1.0) + fabs(S - static_cast<double>(p.s_f)) * M +
                     fabs(c - static_cast<double>(p.c_f));
  const double delta = 2.0 * err * 1.01 + static_cast<double>(k) * 1e-12;
  const bool ok = isfinite(p.s_f) && isfinite(p.c_f) && p.s_f > 0.f && delta < 0.2 &&
                  fabs(c) < 1e6 && M * S < 1e6;
  p.thr = static_cast<float>(0.5 - delta);
  p.exact_only = ok ? 0 : 1;
  return p;
}

__device__ BinParams make_bin_params(const double* d_range, int range_mode, double fixed_lo,
                                     double fixed_hi, int k) {
  if (range_mode == CL_RANGE_FIXED) return make_bin_params_lohi(fixed_lo, fixed_hi, k);
  return make_bin_params_lohi(-d_range[0], d_range[1], k);
}

// Fast bin: returns n = round(x') and sets *slow when the sample must take the exact
// path.  FIXED adds clamps (fixed-range outliers) and the huge-value guard.
template <bool FIXED>
__device__ __forceinline__ int bin_fast(float v, const BinParams& p, bool* slow) {
  float x = fmaf(v, p.s_f, p.c_f);
  bool big = false;
  if (FIXED) {
    big = !(fabsf(x) < 2.0e9f);
    x = fminf(fmaxf(x, -1.25f), static_cast<float>(p.k) + 0.25f);
  }
  const float t = x + 12582912.0f;  // 1.5*2^23: round-to-nearest into the mantissa
  const float rn = t - 12582912.0f;
  int n = __float_as_int(t) - 0x4B400000;
  // written as !(d <= thr) so NaN / inf samples (flagged by minmax) take the exact path
  *slow = !(fabsf(x - rn) <= p.thr) || big;
  if (FIXED) n = min(max(n, 0), p.k - 1);
  // Dynamic range: a sample outside the supplied range (a caller's d_range that does
  // not cover the data) takes the exact, clamping path (entropy.hpp:91-92)
  if (!FIXED) *slow |= static_cast<uint32_t>(n) >= static_cast<uint32_t>(p.k);
  return n;
}

// Bin with exact fallback (any mode).
__device__ __forceinline__ int bin_f32(float v, const BinParams& p, bool fixed) {
  bool slow;
  int n = fixed ? bin_fast<true>(v, p, &slow) : bin_fast<false>(v, p, &slow);
  if (slow || p.exact_only) n = bin_index_exact(static_cast<double>(v), p.lo, p.width, p.k);
  return n;
}

// ---------------------------------------------------------------------------
// Stage 1: min/max + finite
// ---------------------------------------------------------------------------
template <typename T>
struct Vec4;
template <>
struct Vec4<float> {
  using type = float4;
};
template <>
struct Vec4<double> {
  using type = double2;  // 16 bytes
};

template <int MODE>
__device__ __forceinline__ bool sampled(uint64_t gi, uint64_t stride) {
  if (MODE == 0) return true;
  if (MODE == 1) return (gi & (stride - 1)) == 0;
  return gi % stride == 0;
}

// GATHER: every sampled value is also written to gather[(g0 + i) / stride - first] (first =
// the first sampled global index / stride), so a strided histogram reads n / stride values
// instead of all n (cl_minmax_gather_f32)
template <int MODE, bool GATHER = false>
__global__ void __launch_bounds__(kThreads) minmax_f32_kernel(const float* __restrict__ v,
                                                              uint64_t n, uint64_t g0,
                                                              uint64_t stride, double* range,
                                                              float* __restrict__ gather = nullptr,
                                                              uint64_t first = 0) {
  range::Acc acc;
  const uint64_t head = umin64(n, ((16u - (reinterpret_cast<uintptr_t>(v) & 15u)) & 15u) / 4u);
  const uint64_t n4 = (n - head) / 4;
  const uint64_t tail0 = head + n4 * 4;
  const int sh = MODE == 1 ? __ffsll(static_cast<long long>(stride)) - 1 : 0;
  auto visit = [&](float x, uint64_t i) {
    const bool smp = sampled<MODE>(g0 + i, stride);
    acc.visit(x, smp);
    if (GATHER && smp)
      gather[(MODE == 1 ? (g0 + i) >> sh : (g0 + i) / stride) - first] = x;
  };
  if (blockIdx.x == 0) {
    for (uint64_t i = threadIdx.x; i < head; i += blockDim.x) visit(v[i], i);
    for (uint64_t i = tail0 + threadIdx.x; i < n; i += blockDim.x) visit(v[i], i);
  }
  const float4* v4 = reinterpret_cast<const float4*>(v + head);
  const uint64_t T = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  uint64_t i4 = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  constexpr int kU = CL_MM_UNROLL;  // float4 loads in flight per thread
  for (; i4 + (kU - 1) * T < n4; i4 += kU * T) {
    float4 q[kU];
#pragma unroll
    for (int j = 0; j < kU; ++j) q[j] = __ldcs(v4 + i4 + j * T);
#pragma unroll
    for (int j = 0; j < kU; ++j) {
      const uint64_t i = head + (i4 + j * T) * 4;
      visit(q[j].x, i);
      visit(q[j].y, i + 1);
      visit(q[j].z, i + 2);
      visit(q[j].w, i + 3);
    }
  }
  for (; i4 < n4; i4 += T) {
    const float4 q = __ldcs(v4 + i4);
    const uint64_t i = head + i4 * 4;
    visit(q.x, i);
    visit(q.y, i + 1);
    visit(q.z, i + 2);
    visit(q.w, i + 3);
  }
  range::commit<kThreads>(acc, range);
}

template <int MODE>
__global__ void __launch_bounds__(kThreads) minmax_f64_kernel(const double* __restrict__ v,
                                                              uint64_t n, uint64_t g0,
                                                              uint64_t stride, double* range) {
  double lo = DBL_MAX, hi = -DBL_MAX;
  bool any = false, bad = false;
  const uint64_t T = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += T) {
    const double x = v[i];
    bad |= !finite_f64(x);
    if (sampled<MODE>(g0 + i, stride)) {
      // std::min(lo, x) keeps lo unless x < lo (entropy.hpp:111-112)
      lo = x < lo ? x : lo;
      hi = hi < x ? x : hi;
      any = true;
    }
  }
  for (int o = 16; o; o >>= 1) {
    const double l2 = __shfl_xor_sync(0xffffffffu, lo, o);
    const double h2 = __shfl_xor_sync(0xffffffffu, hi, o);
    lo = l2 < lo ? l2 : lo;
    hi = hi < h2 ? h2 : hi;
  }
  any = __any_sync(0xffffffffu, any);
  bad = __any_sync(0xffffffffu, bad);
  __shared__ double s_lo[kThreads / 32], s_hi[kThreads / 32];
  __shared__ int s_any[kThreads / 32], s_bad[kThreads / 32];
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  if (l == 0) {
    s_lo[w] = lo;
    s_hi[w] = hi;
    s_any[w] = any;
    s_bad[w] = bad;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < kThreads / 32; ++k) {
      lo = s_lo[k] < lo ? s_lo[k] : lo;
      hi = hi < s_hi[k] ? s_hi[k] : hi;
      any |= s_any[k] != 0;
      bad |= s_bad[k] != 0;
    }
    if (any) {
      atomic_max_f64(range + 0, -lo);
      atomic_max_f64(range + 1, hi);
    }
    if (bad) atomic_max_f64(range + 2, 1.0);
  }
}

__global__ void range_init_kernel(double* range) {
  range[0] = -INFINITY;
  range[1] = -INFINITY;
  range[2] = 0.0;
  range[3] = 0.0;
}

// range_init and zeroed counts in one launch (the prefill's first node)
__global__ void __launch_bounds__(256) prefill_init_kernel(double* range,
                                                           unsigned long long* counts, int k) {
  if (threadIdx.x == 0) {
    range[0] = -INFINITY;
    range[1] = -INFINITY;
    range[2] = 0.0;
    range[3] = 0.0;
  }
  for (int b = threadIdx.x; b < k; b += blockDim.x) counts[b] = 0ull;
}

// ---------------------------------------------------------------------------
// Stage 2: histogram, K <= 256.  Each lane owns private counters (no atomics): the
// per-lane read-modify-write chain is broken into pairs (full chunks) or groups of four
// samples: the counters are loaded together, and the stores (in order) carry the
// in-group duplicate count, so the last store to a bin holds the right total.  Input
// is streamed through a shared-memory ring filled by cp.async.bulk (TMA bulk copies)
// issued by a dedicated producer warp; consumers release slots through an mbarrier.  Two
// CTAs per SM: two rings halve the cross-warp gating of slot release, and the producer
// keeps kHistPrefetch more chunks on their way into L2.  Fire-and-forget shared atomics
// on a conflict-free packed layout measured +39% (ATOMS throughput).  Counters are
// flushed (per CTA, then one atomic per bin) before they can overflow.
// ---------------------------------------------------------------------------
// CL_HIST_U8=1 (default): 8-bit lane counters (8 KB per warp) in a bank-exclusive layout
// (lane l's counters for bins 4r..4r+3 are the bytes of word r*32 + l, so every lane of a
// warp always hits its own bank), 8 consumer warps per CTA and a 2-stage ring, flushed
// every 15 chunks.  Measured at C3 (K=256, ms): u16 5 warps x 3 stages 0.251; u8 layouts
// 7x3 0.246, 6x4 0.274, 8x2 0.231, 9x2 0.239 (spills), 10 warps x 8 samples 0.256;
// 8-bit [bin][lane] without the bank-exclusive map 0.262 (4-way conflicts: the shared
// pipe saturates at 91%).  Warps per SM, not ring depth, is what the loop needs.
// CL_HIST_U8=0: 16-bit counters [bin][lane] (16 KB per warp, 2-way bank conflicts), 5 warps.
#ifndef CL_HIST_U8
#define CL_HIST_U8 1
#endif
#ifndef CL_HIST_WARPS
#define CL_HIST_WARPS (CL_HIST_U8 ? 8 : 5)
#endif
constexpr int kHistWarps = CL_HIST_WARPS;             // consumer warps per CTA

constexpr int kHistThreads = (kHistWarps + 1) * 32;  // + producer warp
#ifndef CL_HIST_STAGES
#define CL_HIST_STAGES (CL_HIST_U8 ? 2 : 3)
#endif
constexpr int kStages = CL_HIST_STAGES;
constexpr int kCntBytes = CL_HIST_U8 ? 1 : 2;              // bytes per lane counter
#ifndef CL_HIST_SAMPLES
#define CL_HIST_SAMPLES 16
#endif
constexpr int kLaneSamples = CL_HIST_SAMPLES;               // samples per lane per stage
constexpr int kLaneF4 = kLaneSamples / 4;
constexpr int kChunkFloats = kHistWarps * 32 * kLaneSamples;
constexpr int kChunkBytes = kChunkFloats * 4;
constexpr int kLaneBins = 256;
constexpr int kBinStride = 32 * kCntBytes;                 // bytes per bin row (32 lanes)
constexpr size_t kCounterBytes = size_t(kHistWarps) * kLaneBins * kBinStride;
constexpr size_t kHistSmem = kCounterBytes + size_t(kStages) * kChunkBytes + kLaneBins * 4 +
                             2 * kStages * 8 + 64;
// CTAs that fit one SM's 228 KB (227 KB usable per CTA + 1 KB reserved each)
constexpr int kHistCtasPerSm = static_cast<int>(233472 / (kHistSmem + 1024 + 1024)) > 4
                                   ? 4
                                   : static_cast<int>(233472 / (kHistSmem + 1024 + 1024));
// flush before a counter can overflow: chunks * samples per lane (+ up to 6 head/tail
// samples on block 0, warp 0) stays below 2^(8*kCntBytes)
constexpr int kFlushChunks = CL_HIST_U8 ? 240 / kLaneSamples : 4000;
static_assert(kFlushChunks * kLaneSamples + 6 < (1 << (8 * kCntBytes)), "counter overflow");
using cnt_t = std::conditional_t<CL_HIST_U8 != 0, uint8_t, uint16_t>;

// Byte offset of bin b's counter from the lane's base (counters + warp block + lane's word
// or half-word): u8 bank-exclusive (b/4)*128 + b%4, u16 [bin][lane] b*64.
__device__ __forceinline__ uint32_t cofs(uint32_t b) {
  if (CL_HIST_U8) return (b & ~3u) * 32u + (b & 3u);
  return b * 64u;
}
// Counter byte offset from the start of the counter block, straight from the bits of the
// magic-number rounded t = n + 1.5*2^23 (bits 0x4B400000 + n, 0 <= n < 256, so n's bits
// are the low byte and the exponent bits lie above it): (n & ~3)*32 + (n & 3) plus the
// lane's word and the warp's block (wl = warp*8192 + lane*4) -- LOP3, LOP3, IMAD.
[[maybe_unused]] __device__ __forceinline__ uint32_t cofs_from_tbits(uint32_t tb, uint32_t wl) {
  uint32_t o;
  asm("{\n"
      ".reg .b32 hi, lo;\n"
      "and.b32 hi, %1, 0xfc;\n"
      "lop3.b32 lo, %1, 3, %2, 0xea;\n"  // (tb & 3) | wl: LUT (a & b) | c
      "mad.lo.u32 %0, hi, 32, lo;\n"
      "}\n"
      : "=r"(o)
      : "r"(tb), "r"(wl));
  return o;
}
__device__ __forceinline__ cnt_t& cref(unsigned char* lane_base, int b) {
  return *reinterpret_cast<cnt_t*>(lane_base + cofs(static_cast<uint32_t>(b)));
}
#ifndef CL_HIST_PREFETCH
#define CL_HIST_PREFETCH 3
#endif
constexpr int kHistPrefetch = CL_HIST_PREFETCH;  // chunks prefetched to L2 beyond the ring

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void named_bar(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// Sum of the counters packed in one 32-bit word (two u16 or four u8).
__device__ __forceinline__ uint32_t word_sum(uint32_t w) {
  if (CL_HIST_U8) return __dp4a(w, 0x01010101u, 0u);
  return (w & 0xffffu) + (w >> 16);
}

// Sum this warp's lane-private counters into the CTA histogram and clear them.
__device__ __forceinline__ void flush_warp(cnt_t* cnt, uint32_t* cta_hist, int lane, int k) {
  __syncwarp();
  if (CL_HIST_U8) {
    // row r = bins 4r..4r+3 of all 32 lanes (32 words); lane takes rows lane, lane + 32.
    // Byte lanes are summed pairwise in 16-bit halves (32 * 255 < 65536).
    const uint4* w4 = reinterpret_cast<const uint4*>(cnt);
    for (int r = lane; 4 * r < k; r += 32) {
      uint32_t s02 = 0, s13 = 0;
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        const uint4 w = w4[r * 8 + ((m + lane) & 7)];  // staggered: 4-way, not 32-way
        s02 += (w.x & 0x00ff00ffu) + (w.y & 0x00ff00ffu) + (w.z & 0x00ff00ffu) + (w.w & 0x00ff00ffu);
        s13 += ((w.x >> 8) & 0x00ff00ffu) + ((w.y >> 8) & 0x00ff00ffu) +
               ((w.z >> 8) & 0x00ff00ffu) + ((w.w >> 8) & 0x00ff00ffu);
      }
      const uint32_t c[4] = {s02 & 0xffffu, s13 & 0xffffu, s02 >> 16, s13 >> 16};
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (c[e] && 4 * r + e < k) atomicAdd(cta_hist + 4 * r + e, c[e]);
    }
    __syncwarp();
    uint4* c4 = reinterpret_cast<uint4*>(cnt);
    for (int i = lane; i < ((k + 3) / 4) * 8; i += 32) c4[i] = make_uint4(0, 0, 0, 0);
    __syncwarp();
    return;
  }
  constexpr int kRow4 = kBinStride / 16;  // uint4 per bin row (32 lanes' counters)
  for (int b = lane; b < k; b += 32) {
    const uint4* row = reinterpret_cast<const uint4*>(cnt + b * 32);
    uint32_t sum = 0;
#pragma unroll
    for (int m = 0; m < kRow4; ++m) {
      const uint4 w = row[(m + (lane >> 1)) % kRow4];
      sum += word_sum(w.x) + word_sum(w.y) + word_sum(w.z) + word_sum(w.w);
    }
    if (sum) atomicAdd(cta_hist + b, sum);
  }
  __syncwarp();
  uint4* c4 = reinterpret_cast<uint4*>(cnt);
  for (int i = lane; i < k * kBinStride / 16; i += 32) c4[i] = make_uint4(0, 0, 0, 0);
  __syncwarp();
}

#ifndef CL_HIST_X2
#define CL_HIST_X2 1
#endif
#ifndef CL_HIST_RANGE_CHECK
#define CL_HIST_RANGE_CHECK 1
#endif
__device__ __forceinline__ uint64_t pack_f2(float a, float b) {
  return (static_cast<uint64_t>(__float_as_uint(b)) << 32) | __float_as_uint(a);
}
__device__ __forceinline__ float lo_f(uint64_t v) { return __uint_as_float(static_cast<uint32_t>(v)); }
__device__ __forceinline__ float hi_f(uint64_t v) { return __uint_as_float(static_cast<uint32_t>(v >> 32)); }

__device__ __forceinline__ uint64_t add_mod(uint64_t r, uint64_t d, uint64_t stride) {
  r += d;  // r, d < stride
  return r >= stride ? r - stride : r;
}

// The hot path's binning and counting for one lane's kLaneSamples values (u8 counters,
// bank-exclusive layout): the exact bin of every sample, as bits 0x4B400000 + n of the
// magic-number rounded affine map (near-edge samples re-binned exactly in fp64), then
// pairwise in-order read-modify-writes of the lane's counters.
// POW2K (k a power of two, the default 256): the range check ORs tb ^ 0x4B400000 (= n for
// 0 <= n < 256, with higher bits set for any n outside [0, 256)) into one word per lane,
// one LOP3 per sample, tested against ~(k - 1) once per call.
template <int NS, bool POW2K = false>
__device__ __forceinline__ void lane_count_u8(const float (&val)[NS], const BinParams& p,
                                            unsigned char* cblk, int warp, int lane) {
  // t bits carry the bin (0x4B400000 + n); near-edge samples get the exact bin's bits
  uint32_t tb[NS];
  bool any_slow = p.exact_only != 0;
  [[maybe_unused]] uint32_t rx = 0;
#if CL_HIST_X2
  // the same per-sample fp32 operations on sample pairs (FFMA2 / FADD2: every f32x2
  // lane rounds exactly like the scalar op), half the FMA-pipe instructions
  const uint64_t s2 = pack_f2(p.s_f, p.s_f), c2 = pack_f2(p.c_f, p.c_f);
  const uint64_t mp = pack_f2(12582912.0f, 12582912.0f);
  const uint64_t mn = pack_f2(-12582912.0f, -12582912.0f);
#pragma unroll
  for (int e = 0; e < NS; e += 2) {
    uint64_t x2, t2, r2, d2;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(x2) : "l"(pack_f2(val[e], val[e + 1])), "l"(s2), "l"(c2));
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(t2) : "l"(x2), "l"(mp));
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r2) : "l"(t2), "l"(mn));
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d2) : "l"(x2), "l"(r2));
    any_slow |= !(fabsf(lo_f(d2)) <= p.thr);
    any_slow |= !(fabsf(hi_f(d2)) <= p.thr);
    tb[e] = static_cast<uint32_t>(t2);
    tb[e + 1] = static_cast<uint32_t>(t2 >> 32);
#if CL_HIST_RANGE_CHECK
    // a sample outside the supplied range (a caller's d_range that does not cover the
    // data) rounds to n < 0 or n >= k: take the exact, clamping path (entropy.hpp:91-92)
    // instead of wrapping into bin n mod 256
    if constexpr (POW2K) {
      rx |= (tb[e] ^ 0x4B400000u) | (tb[e + 1] ^ 0x4B400000u);
    } else {
      any_slow |= tb[e] - 0x4B400000u >= static_cast<uint32_t>(p.k);
      any_slow |= tb[e + 1] - 0x4B400000u >= static_cast<uint32_t>(p.k);
    }
#endif
  }
#if CL_HIST_RANGE_CHECK
  if constexpr (POW2K) any_slow |= (rx & ~static_cast<uint32_t>(p.k - 1)) != 0u;
#endif
#else
#pragma unroll
  for (int e = 0; e < NS; ++e) {
    const float x = fmaf(val[e], p.s_f, p.c_f);
    const float t = x + 12582912.0f;
    any_slow |= !(fabsf(x - (t - 12582912.0f)) <= p.thr);
    tb[e] = __float_as_uint(t);
#if CL_HIST_RANGE_CHECK
    any_slow |= tb[e] - 0x4B400000u >= static_cast<uint32_t>(p.k);
#endif
  }
#endif
  if (__any_sync(0xffffffffu, any_slow)) {
#pragma unroll
    for (int e = 0; e < NS; ++e) {
      bool sl;
      bin_fast<false>(val[e], p, &sl);
      if (sl || p.exact_only)
        tb[e] = 0x4B400000u + static_cast<uint32_t>(bin_index_exact(
                                  static_cast<double>(val[e]), p.lo, p.width, p.k));
    }
  }
  // the counter block starts at dynamic shared offset 0, so an offset is an address
  // and the loads / stores below are LDS/STS [R + UR(base)] with no add
  const uint32_t wl = static_cast<uint32_t>(warp) * (kLaneBins * 32) + lane * 4u;
#if CL_HIST_ATOMS
  // one shared-memory reduction per sample on the lane's own word (byte n & 3 of word
  // (n >> 2, lane)): no read-modify-write chain, same-bin samples need no special case;
  // a byte never carries into its neighbour (<= 246 increments between flushes)
  const uint32_t base = smem_u32(cblk);
#pragma unroll
  for (int e = 0; e < NS; ++e) {
    const uint32_t w = base + (tb[e] & 0xFCu) * 32u + wl;
    const uint32_t inc = 1u << ((tb[e] & 3u) << 3);
    // volatile, no memory clobber: the reductions stay in program order among themselves
    // and behind the flush's __syncwarp, without pinning the surrounding loads
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(w), "r"(inc));
  }
#else
#pragma unroll
  for (int g = 0; g < NS / 2; ++g) {
    // plain accesses: the offsets may alias, so the compiler keeps this order
    const uint32_t o0 = cofs_from_tbits(tb[2 * g], wl);
    const uint32_t o1 = cofs_from_tbits(tb[2 * g + 1], wl);
    const uint32_t v0 = cblk[o0];
    const uint32_t v1 = cblk[o1];
    cblk[o0] = static_cast<unsigned char>(v0 + 1u);
    cblk[o1] = static_cast<unsigned char>(v1 + 1u + (o0 == o1 ? 1u : 0u));
  }
#endif
}

template <int MODE, bool FIXED>
__global__ void __launch_bounds__(kHistThreads, kHistCtasPerSm)
    hist_f32_lane_kernel(const float* __restrict__ v, uint64_t n, uint64_t g0, uint64_t stride,
                         int range_mode, double fixed_lo, double fixed_hi, int k,
                         const double* __restrict__ d_range, unsigned long long* d_counts) {
  extern __shared__ __align__(128) unsigned char smem[];
  cnt_t* counters = reinterpret_cast<cnt_t*>(smem);
  unsigned char* ring = smem + kCounterBytes;
  uint32_t* cta_hist = reinterpret_cast<uint32_t*>(ring + size_t(kStages) * kChunkBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(cta_hist + kLaneBins);
  uint64_t* empty = full + kStages;
  __shared__ BinParams sp;

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    sp = make_bin_params(d_range, range_mode, fixed_lo, fixed_hi, k);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, kHistWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  {
    uint4* c4 = reinterpret_cast<uint4*>(smem);
    for (int i = threadIdx.x; i < static_cast<int>(kCounterBytes / 16); i += blockDim.x)
      c4[i] = make_uint4(0, 0, 0, 0);
    for (int i = threadIdx.x; i < kLaneBins; i += blockDim.x) cta_hist[i] = 0;
  }
  __syncthreads();
  const BinParams p = sp;

  // Body = 16B-aligned span of v; head/tail (< 4 elements each) go to block 0.
  const uint64_t head = umin64(n, ((16u - (reinterpret_cast<uintptr_t>(v) & 15u)) & 15u) / 4u);
  const uint64_t body_n = ((n - head) / 4) * 4;
  const float* body = v + head;
  const uint64_t n_chunks = (body_n + kChunkFloats - 1) / kChunkFloats;

  if (warp == kHistWarps) {
    // ---------------- producer warp ----------------
    if (lane == 0) {
      uint32_t it = 0;
      for (uint64_t c = blockIdx.x; c < n_chunks; c += gridDim.x, ++it) {
        const int s = it % kStages;
        const uint32_t phase = (it / kStages) & 1;
        if (it >= kStages) mbar_wait(empty + s, phase ^ 1);
        const uint64_t off = c * kChunkFloats;
        const uint32_t bytes = static_cast<uint32_t>(umin64(kChunkFloats, body_n - off) * 4);
        mbar_expect_tx(full + s, bytes);
        bulk_g2s(ring + size_t(s) * kChunkBytes, body + off, bytes, full + s);
        // the ring holds kStages chunks; keep kHistPrefetch more on their way into L2
        // so ring fills are served from L2 instead of waiting a full DRAM latency
        const uint64_t pc = c + static_cast<uint64_t>(kHistPrefetch) * gridDim.x;
        if (kHistPrefetch > 0 && pc < n_chunks) {
          const uint64_t po = pc * kChunkFloats;
          bulk_prefetch_l2(body + po, static_cast<uint32_t>(umin64(kChunkFloats, body_n - po) * 4));
        }
      }
    }
    return;
  }

  // ---------------- consumer warps ----------------
  // this lane's counter base: bin b's counter is at lane_base + cofs(b)
  unsigned char* lane_base = reinterpret_cast<unsigned char*>(counters + warp * kLaneBins * 32) +
                             lane * (CL_HIST_U8 ? 4 : 2);

  if (blockIdx.x == 0 && warp == 0) {
    for (uint64_t i = lane; i < head; i += 32)
      if (sampled<MODE>(g0 + i, stride)) cref(lane_base, bin_f32(v[i], p, FIXED)) += 1;
    for (uint64_t i = head + body_n + lane; i < n; i += 32)
      if (sampled<MODE>(g0 + i, stride)) cref(lane_base, bin_f32(v[i], p, FIXED)) += 1;
  }

  const uint32_t cbase = smem_u32(lane_base);
  // strided sampling (MODE != 0): residue of this lane's first sample index in the
  // current chunk, advanced incrementally (no per-sample 64-bit modulo)
  // strided sampling (MODE != 0): residue of the chunk's first element's global index,
  // advanced incrementally (no per-chunk 64-bit modulo)
  uint64_t r_chunk = 0, step_chunk = 0;
  if (MODE != 0) {
    r_chunk = (g0 + head + static_cast<uint64_t>(blockIdx.x) * kChunkFloats) % stride;
    step_chunk = (static_cast<uint64_t>(gridDim.x) * kChunkFloats) % stride;
  }
  uint32_t it = 0, since_flush = 0;
  for (uint64_t c = blockIdx.x; c < n_chunks;
       c += gridDim.x, ++it, r_chunk = MODE != 0 ? add_mod(r_chunk, step_chunk, stride) : 0) {
    const int s = it % kStages;
    const uint32_t phase = (it / kStages) & 1;
    mbar_wait(full + s, phase);
    const float4* tile = reinterpret_cast<const float4*>(ring + size_t(s) * kChunkBytes);
    const uint64_t off = c * kChunkFloats;
    const int valid4 = static_cast<int>(umin64(kChunkFloats, body_n - off) / 4);
    if (MODE == 0 && !FIXED && valid4 == kChunkFloats / 4) {
      // ---- hot path: full chunk, every element sampled ----
      float val[kLaneSamples];
#pragma unroll
      for (int j = 0; j < kLaneF4; ++j) {
        const float4 q = tile[j * (kHistWarps * 32) + warp * 32 + lane];
        val[4 * j] = q.x;
        val[4 * j + 1] = q.y;
        val[4 * j + 2] = q.z;
        val[4 * j + 3] = q.w;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + s);
      if constexpr (CL_HIST_U8 != 0) {
        lane_count_u8(val, p, reinterpret_cast<unsigned char*>(counters), warp, lane);
      } else {
        int bin[kLaneSamples];
        bool any_slow = p.exact_only != 0;
#pragma unroll
        for (int e = 0; e < kLaneSamples; ++e) {
          bool sl;
          bin[e] = bin_fast<false>(val[e], p, &sl);
          any_slow |= sl;
        }
        if (__any_sync(0xffffffffu, any_slow)) {
#pragma unroll
          for (int e = 0; e < kLaneSamples; ++e) {
            bool sl;
            bin_fast<false>(val[e], p, &sl);
            if (sl || p.exact_only)
              bin[e] = bin_index_exact(static_cast<double>(val[e]), p.lo, p.width, p.k);
          }
        }
        // pairwise read-modify-write: both counters loaded, then stored in order with
        // the second carrying the pair's duplicate
#pragma unroll
        for (int g = 0; g < kLaneSamples / 2; ++g) {
          const int b0 = bin[2 * g], b1 = bin[2 * g + 1];
          const uint32_t a0 = cbase + cofs(static_cast<uint32_t>(b0));
          const uint32_t a1 = cbase + cofs(static_cast<uint32_t>(b1));
          uint32_t v0, v1;
          asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v0) : "r"(a0) : "memory");
          asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v1) : "r"(a1) : "memory");
          v1 += 1u + (b0 == b1 ? 1u : 0u);
          v0 += 1u;
          asm volatile("st.shared.u16 [%0], %1;" ::"r"(a0), "h"(static_cast<uint16_t>(v0)) : "memory");
          asm volatile("st.shared.u16 [%0], %1;" ::"r"(a1), "h"(static_cast<uint16_t>(v1)) : "memory");
        }
      }
      if (++since_flush == kFlushChunks) {
        flush_warp(counters + warp * kLaneBins * 32, cta_hist, lane, k);
        since_flush = 0;
      }
      continue;
    }
    if (MODE != 0) {
      // ---- strided sampling: gather the chunk's samples, sample m to lane m % (32W) ----
      // Sample m sits at chunk offset first + m*stride, so every lane holds a sample (no
      // lane idles on a float4 without one, as a float4-per-lane split does at stride 8);
      // at most kLaneSamples/2 per lane (stride >= 2).
      const uint64_t valid = static_cast<uint64_t>(valid4) * 4u;
      const uint64_t first = r_chunk == 0 ? 0 : stride - r_chunk;
      const float* ringf = reinterpret_cast<const float*>(tile);
      constexpr int kMaxPer = kLaneSamples / 2;
      const uint32_t m0 = static_cast<uint32_t>(warp * 32 + lane);
      float sv[kMaxPer];
      uint32_t have = 0;
#pragma unroll
      for (int t = 0; t < kMaxPer; ++t) {
        const uint64_t o = first + static_cast<uint64_t>(m0 + t * kHistWarps * 32) * stride;
        sv[t] = 0.f;
        if (o < valid) {
          sv[t] = ringf[o];
          have |= 1u << t;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + s);
#pragma unroll
      for (int t = 0; t < kMaxPer; ++t) {
        if (have & (1u << t)) {
          const int b = bin_f32(sv[t], p, FIXED);
          cref(lane_base, b) = static_cast<cnt_t>(cref(lane_base, b) + 1u);
        }
      }
      if (++since_flush == kFlushChunks) {
        flush_warp(counters + warp * kLaneBins * 32, cta_hist, lane, k);
        since_flush = 0;
      }
      continue;
    }

    // ---- every element sampled: partial chunk, or the fixed-range mode ----
    float val[kLaneSamples];
    uint32_t inc = 0;  // bit e: sample e is valid
#pragma unroll
    for (int j = 0; j < kLaneF4; ++j) {
      const int idx = j * (kHistWarps * 32) + warp * 32 + lane;
      float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
      if (idx < valid4) {
        q = tile[idx];
        inc |= 0xfu << (4 * j);
      }
      val[4 * j] = q.x;
      val[4 * j + 1] = q.y;
      val[4 * j + 2] = q.z;
      val[4 * j + 3] = q.w;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + s);

    int bin[kLaneSamples];
    uint32_t slow = 0;
#pragma unroll
    for (int e = 0; e < kLaneSamples; ++e) {
      bool sl;
      bin[e] = bin_fast<FIXED>(val[e], p, &sl);
      slow |= (sl ? 1u : 0u) << e;
    }
    slow &= inc;
    if (p.exact_only) slow = inc;
    if (__any_sync(0xffffffffu, slow != 0)) {
#pragma unroll
      for (int e = 0; e < kLaneSamples; ++e)
        if (slow & (1u << e)) bin[e] = bin_index_exact(static_cast<double>(val[e]), p.lo, p.width, p.k);
    }
#pragma unroll
    for (int e = 0; e < kLaneSamples; ++e)
      if (!(inc & (1u << e))) bin[e] = 0;  // +0 on bin 0: harmless in the grouped RMW
#pragma unroll
    for (int g = 0; g < kLaneF4; ++g) {
      const int b0 = bin[4 * g], b1 = bin[4 * g + 1], b2 = bin[4 * g + 2], b3 = bin[4 * g + 3];
      const uint32_t i0 = (inc >> (4 * g)) & 1u, i1 = (inc >> (4 * g + 1)) & 1u;
      const uint32_t i2 = (inc >> (4 * g + 2)) & 1u, i3 = (inc >> (4 * g + 3)) & 1u;
      const uint32_t v0 = cref(lane_base, b0), v1 = cref(lane_base, b1);
      const uint32_t v2 = cref(lane_base, b2), v3 = cref(lane_base, b3);
      const uint32_t n1 = v1 + i1 + (b1 == b0 ? i0 : 0u);
      const uint32_t n2 = v2 + i2 + (b2 == b0 ? i0 : 0u) + (b2 == b1 ? i1 : 0u);
      const uint32_t n3 = v3 + i3 + (b3 == b0 ? i0 : 0u) + (b3 == b1 ? i1 : 0u) + (b3 == b2 ? i2 : 0u);
      cref(lane_base, b0) = static_cast<cnt_t>(v0 + i0);
      cref(lane_base, b1) = static_cast<cnt_t>(n1);
      cref(lane_base, b2) = static_cast<cnt_t>(n2);
      cref(lane_base, b3) = static_cast<cnt_t>(n3);
    }
    if (++since_flush == kFlushChunks) {
      flush_warp(counters + warp * kLaneBins * 32, cta_hist, lane, k);
      since_flush = 0;
    }
  }
  flush_warp(counters + warp * kLaneBins * 32, cta_hist, lane, k);
  named_bar(1, kHistWarps * 32);
  for (int b = threadIdx.x; b < k; b += kHistWarps * 32)
    if (cta_hist[b]) atomicAdd(d_counts + b, static_cast<unsigned long long>(cta_hist[b]));
}

// ---- Histogram, register-fed (the hot path: K <= 256, stride 1, Dynamic range) ----
// One CTA per SM of kRegWarps consumer warps and no shared ring: a warp streams 2 KB
// warp-chunks (lane l takes float4 j*32 + l, every LDG.128 covers 512 contiguous bytes),
// loading chunk c + 1 into registers while it bins chunk c, with lane 0 keeping
// CL_HIST_REG_PF chunks of its stream on their way into L2.  Shared memory holds only the
// counters (16 x 8 KB).  Binning and counting are lane_count_u8, as in the ring kernel.
// The ring kernel's consumers spent 12% of their stall samples waiting on the full
// barrier; here the next chunk is already in flight in registers.  C3 (ms): ring kernel
// 0.2212; register-fed with L2 prefetch distance 0 / 1 / 2 / 3 / 4 / 6 / 12 chunks:
// 0.219 / 0.211 / 0.194 / 0.193 / 0.197 / 0.197 / 0.203 (118 registers, no spills).
#ifndef CL_HIST_REG
#define CL_HIST_REG 1
#endif
#ifndef CL_HIST_REG_PF
#define CL_HIST_REG_PF 3
#endif
// ---------------------------------------------------------------------------
// Stage 3: entropy + rule + policy (one CTA, or the histogram's last CTA).
// ---------------------------------------------------------------------------
struct DecideArgs {
  const unsigned long long* counts;  // may be null (host-features mode)
  const double* range;
  int k;
  double epsilon;
  int range_mode;
  double fixed_lo, fixed_hi;
  uint64_t n_samples;
  cl_rule_spec rule;
  uint64_t seq_len;
  int features_mode;  // 0: entropy from counts; 1: host features; 2: token entropy
  cl_features f;
  const double* token;  // mode 2: cl_token_entropy output {raw, normalized, n, nonfinite}
};

__device__ __forceinline__ int ilog2_pow2(int v) { return 31 - __clz(v); }

// select_chunk (chunk.hpp:68-89) in fp64.  Returns 0 or CL_DEV_SIGNAL.
__device__ int device_select_chunk(double signal, int c_min, int c_max, double h_ref, int* chunk,
                                   double* r_out, double* margin) {
  if (!(signal >= 0.0)) return CL_DEV_SIGNAL;
  double r = __ddiv_rn(signal, h_ref);
  if (1.0 < r) r = 1.0;
  const double target = __dadd_rn(static_cast<double>(c_min),
                                  __dmul_rn(r, static_cast<double>(c_max - c_min)));
  const double l2 = log2(target);
  const double e = floor(__dadd_rn(l2, 0.5));  // round_half_up (common.hpp:35)
  const double frac = __dsub_rn(__dadd_rn(l2, 0.5), e);
  *margin = fmin(frac, 1.0 - frac);
  const double pow2 = exp2(e);
  int c = static_cast<int>(pow2);
  c = c < c_min ? c_min : (c > c_max ? c_max : c);
  *chunk = c;
  *r_out = r;
  return 0;
}

// snap_to_buckets (chunk.hpp:206-218): nearest by |log2| distance, ties toward
// the larger bucket.  All operands are powers of two, so log2 is exact.
__device__ int device_snap(int chunk, const cl_rule_spec& rule) {
  int best = rule.buckets[0];
  int best_dist = INT_MAX;
  const int lc = ilog2_pow2(chunk);
  for (int i = 0; i < rule.n_buckets; ++i) {
    const int b = rule.buckets[i];
    int d = ilog2_pow2(b) - lc;
    d = d < 0 ? -d : d;
    if (d < best_dist || (d == best_dist && b > best)) {
      best = b;
      best_dist = d;
    }
  }
  return best;
}

__device__ int decide_simple(const DecideArgs& a, int kind, int static_chunk, double entropy,
                             cl_decision& out) {
  const cl_rule_spec& rule = a.rule;
  out.r = 0.0;
  out.signal_nats = 0.0;
  switch (kind) {
    case CL_POL_STATIC:
      out.chunk = static_chunk;
      out.source = 0;
      return 0;
    case CL_POL_MIDPOINT: {
      const int n = rule.n_buckets;
      int idx = (n + 1) / 2;
      if (idx > n - 1) idx = n - 1;
      out.chunk = rule.buckets[idx];
      out.source = 1;
      return 0;
    }
    case CL_POL_FULL_HIST:
    case CL_POL_SAMPLED_HIST:
    case CL_POL_TOKEN_HIST:
    case CL_POL_RULE: {
      int c;
      double r;
      const int st = device_select_chunk(entropy, rule.c_min, rule.c_max, rule.h_ref_nats, &c,
                                         &r, &out.margin);
      if (st) return st;
      out.chunk = kind == CL_POL_RULE ? c : device_snap(c, rule);
      out.r = r;
      out.signal_nats = entropy;
      out.source = kind;  // CL_POL_* doubles as the source_policy tag code
      return 0;
    }
    case CL_POL_LEARNED_TABLE: {
      const uint64_t L = a.features_mode == 1 ? a.f.seq_len : a.seq_len;
      out.chunk = L < rule.threshold_tokens ? rule.short_chunk : rule.long_chunk;
      out.signal_nats = static_cast<double>(L);
      out.source = 4;
      return 0;
    }
  }
  return 0;
}

// The decision of one CTA (blockDim.x >= kThreads; the first kThreads threads form the
// bin terms).  COHERENT: counts were accumulated by other CTAs of the same grid (the
// histogram's last CTA), so they are read from L2.
template <bool COHERENT>
__device__ void decide_block(const DecideArgs& a, cl_decision* d_out) {
  __shared__ double terms[kThreads];
  cl_decision out = {};
  out.margin = 1.0;
  double entropy = 0.0;
  int status = 0;
  if (a.features_mode == 0) {
    const bool bad = a.range[2] != 0.0;
    // masses[b] = counts[b] * (1/n) (entropy.hpp:130-133); terms p*log(p+eps)
    const double inv_n = __ddiv_rn(1.0, static_cast<double>(a.n_samples));
    double raw = 0.0;
    for (int base = 0; base < a.k; base += kThreads) {
      // any block size: threads stride over the kThreads term slots
      for (int i = threadIdx.x; i < kThreads; i += blockDim.x) {
        const int b = base + i;
        double t = 0.0;
        if (b < a.k) {
          const unsigned long long cb = COHERENT ? __ldcg(a.counts + b) : a.counts[b];
          const double pm = __dmul_rn(static_cast<double>(cb), inv_n);
          if (pm > 0.0) t = __dmul_rn(pm, log(__dadd_rn(pm, a.epsilon)));
        }
        terms[i] = t;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        // raw -= p*log(p+eps) in bin order (entropy.hpp:154-156).  Empty bins hold +0.0
        // and raw - (+0.0) == raw bit for bit, so they are subtracted too: the chain reads
        // shared memory only (no per-bin global count load and branch)
        const int m = min(kThreads, a.k - base);
#pragma unroll 8
        for (int i = 0; i < m; ++i) raw = __dsub_rn(raw, terms[i]);
      }
      __syncthreads();
    }
    if (threadIdx.x != 0) return;
    out.raw_nats = raw;
    out.normalized = __ddiv_rn(raw, log(static_cast<double>(a.k)));
    out.bin_count = a.k;
    out.sample_count = a.n_samples;
    if (a.range_mode == CL_RANGE_FIXED) {
      out.lo = a.fixed_lo;
      out.hi = a.fixed_hi;
    } else {
      out.lo = -a.range[0];
      out.hi = a.range[1];
    }
    entropy = raw;
    if (bad) status = CL_DEV_NON_FINITE;
    else if (a.n_samples == 0) status = CL_DEV_NO_SAMPLES;
  } else if (a.features_mode == 2) {
    if (threadIdx.x != 0) return;
    entropy = a.token[0];
    out.raw_nats = a.token[0];
    out.normalized = a.token[1];
    out.sample_count = static_cast<uint64_t>(a.token[2]);
    out.bin_count = a.k;
    out.lo = out.hi = 0.0;  // one range per position: none to report
    if (a.token[3] != 0.0) status = CL_DEV_NON_FINITE;
  } else {
    if (threadIdx.x != 0) return;
  }

  if (status == 0) {
    const cl_rule_spec& rule = a.rule;
    double e_inner = entropy;
    if (a.features_mode == 1) {
      const int kind = rule.kind == CL_POL_GUARDED ? rule.inner_kind : rule.kind;
      e_inner = kind == CL_POL_SAMPLED_HIST ? a.f.sampled_entropy_nats
                : kind == CL_POL_TOKEN_HIST ? a.f.token_entropy_nats
                                            : a.f.full_entropy_nats;
    }
    if (rule.kind != CL_POL_GUARDED) {
      status = decide_simple(a, rule.kind, rule.static_chunk, e_inner, out);
    } else {
      // GuardedPolicy (chunk.hpp:344-358)
      status = decide_simple(a, rule.inner_kind, rule.inner_static_chunk, e_inner, out);
      if (!status) {
        int delta = ilog2_pow2(out.chunk) - ilog2_pow2(rule.safe_chunk);
        delta = delta < 0 ? -delta : delta;
        if (delta >= rule.min_delta_buckets) {
          out.source += CL_SRC_GUARDED;
        } else {
          out.chunk = rule.safe_chunk;
          out.source = CL_SRC_GUARDED_FALLBACK;
        }
      }
    }
  }
  out.status = status;
  *d_out = out;
}

__global__ void __launch_bounds__(kThreads) decide_kernel(DecideArgs a, cl_decision* d_out) {
  decide_block<false>(a, d_out);
}

constexpr int kRegWarps = 16;
constexpr int kRegChunk = 32 * kLaneSamples;  // floats per warp-chunk
constexpr size_t kRegSmem = size_t(kRegWarps) * kLaneBins * kBinStride + kLaneBins * 4 + 64;

// FUSE: the CTA that finishes last (an arrival ticket in the stream workspace, 0 on
// entry and reset here by the last CTA) also runs the decision, so the single-GPU
// prefill has no separate decide launch.
// POW2K: k is a power of two (the default 256), the one-LOP3 range check of lane_count_u8
template <bool FUSE, bool POW2K>
__global__ void __launch_bounds__(kRegWarps * 32, 1)
    hist_f32_reg_kernel(const float* __restrict__ v, uint64_t n, int range_mode, double fixed_lo,
                        double fixed_hi, int k, const double* __restrict__ d_range,
                        unsigned long long* d_counts, DecideArgs da, cl_decision* d_out,
                        unsigned long long* ticket) {
  extern __shared__ __align__(128) unsigned char smem[];
  cnt_t* counters = reinterpret_cast<cnt_t*>(smem);
  uint32_t* cta_hist = reinterpret_cast<uint32_t*>(smem + size_t(kRegWarps) * kLaneBins * kBinStride);
  __shared__ BinParams sp;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) sp = make_bin_params(d_range, range_mode, fixed_lo, fixed_hi, k);
  {
    uint4* c4 = reinterpret_cast<uint4*>(smem);
    for (int i = threadIdx.x; i < static_cast<int>(size_t(kRegWarps) * kLaneBins * kBinStride / 16);
         i += blockDim.x)
      c4[i] = make_uint4(0, 0, 0, 0);
    for (int i = threadIdx.x; i < kLaneBins; i += blockDim.x) cta_hist[i] = 0;
  }
  __syncthreads();
  const BinParams p = sp;
  unsigned char* lane_base = reinterpret_cast<unsigned char*>(counters + warp * kLaneBins * 32) + lane * 4;

  const uint64_t head = umin64(n, ((16u - (reinterpret_cast<uintptr_t>(v) & 15u)) & 15u) / 4u);
  const float* body = v + head;
  const uint64_t nwc = (n - head) / kRegChunk;  // full warp-chunks
  const uint64_t tail0 = head + nwc * kRegChunk;
  if (blockIdx.x == 0 && warp == 0) {
    for (uint64_t i = lane; i < head; i += 32) cref(lane_base, bin_f32(v[i], p, false)) += 1;
    for (uint64_t i = tail0 + lane; i < n; i += 32) cref(lane_base, bin_f32(v[i], p, false)) += 1;
    // up to 3 + 16 samples per lane: flush now so the chunk loop's budget is untouched
    flush_warp(counters + warp * kLaneBins * 32, cta_hist, lane, k);
  }
  const uint64_t wstride = static_cast<uint64_t>(gridDim.x) * kRegWarps;
  uint64_t c = static_cast<uint64_t>(blockIdx.x) * kRegWarps + warp;
  if (lane == 0) {
#pragma unroll 1
    for (int d = 0; d < CL_HIST_REG_PF; ++d) {
      const uint64_t pc = c + d * wstride;
      if (pc < nwc) bulk_prefetch_l2(body + pc * kRegChunk, kRegChunk * 4);
    }
  }
  // (a two-buffer ping-pong that avoids copying the chunk in flight into val measured
  // slower: C3 0.250 vs 0.211 ms)
  float4 nx[kLaneF4];
  if (c < nwc) {
    const float4* src = reinterpret_cast<const float4*>(body + c * kRegChunk);
#pragma unroll
    for (int j = 0; j < kLaneF4; ++j) nx[j] = __ldcs(src + j * 32 + lane);
  }
  uint32_t since_flush = 0;
  for (; c < nwc; c += wstride) {
    float val[kLaneSamples];
#pragma unroll
    for (int j = 0; j < kLaneF4; ++j) {
      val[4 * j] = nx[j].x;
      val[4 * j + 1] = nx[j].y;
      val[4 * j + 2] = nx[j].z;
      val[4 * j + 3] = nx[j].w;
    }
    const uint64_t cn = c + wstride;
    if (cn < nwc) {
      const float4* src = reinterpret_cast<const float4*>(body + cn * kRegChunk);
#pragma unroll
      for (int j = 0; j < kLaneF4; ++j) nx[j] = __ldcs(src + j * 32 + lane);
    }
    if (lane == 0) {
      const uint64_t pc = c + CL_HIST_REG_PF * wstride;
      if (pc < nwc) bulk_prefetch_l2(body + pc * kRegChunk, kRegChunk * 4);
    }
    lane_count_u8<kLaneSamples, POW2K>(val, p, reinterpret_cast<unsigned char*>(counters), warp,
                                       lane);
    if (++since_flush == kFlushChunks) {
      flush_warp(counters + warp * kLaneBins * 32, cta_hist, lane, k);
      since_flush = 0;
    }
  }
  flush_warp(counters + warp * kLaneBins * 32, cta_hist, lane, k);
  __syncthreads();
  for (int b = threadIdx.x; b < k; b += blockDim.x)
    if (cta_hist[b]) atomicAdd(d_counts + b, static_cast<unsigned long long>(cta_hist[b]));
  if constexpr (FUSE) {
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned long long old = atomicAdd(ticket, 1ull);
#if CL_DEVICE_CHECKS
      if (old >= gridDim.x) {  // a dirty ticket: the decision would never be written
        printf("CL_DCHECK failed: histogram arrival ticket %llu >= grid %u\n", old, gridDim.x);
        __trap();
      }
#endif
      last = old == gridDim.x - 1;
    }
    __syncthreads();
    if (last) {
      __threadfence();
      decide_block<true>(da, d_out);
      if (threadIdx.x == 0) *ticket = 0ull;
    }
  }
}


// Producer fusion with a Fixed range ("deeper kernel fusion of the
// entropy estimator"): the conv1d (+ SiLU) that produces u bins every u it writes.  With a
// Fixed range the bin edges are known before u exists (entropy.hpp:116-119), so u is
// never read back for the histogram: x is read once, u written once, counts come out of
// the same pass.  The conv arithmetic is conv1d.cu's (conv_common.cuh: identical bits of
// u) in its warp-coalesced layout (a warp unit = kCHWQ 32-quad blocks of one row, lane l
// holding quad l of each), so a full unit is exactly kLaneSamples values per lane: the
// hot path's lane_count_u8 (u8 lane counters, exact fp64 fallback near edges and for
// clipped outliers).  Every element is also checked for finiteness (validate_tensor,
// entropy.hpp:42) into d_range[2].  Needs L % 128 == 0, 16-byte aligned x / u, K <= 256.
constexpr int kCHWarps = 8;
constexpr int kCHWQ = 4;  // = conv1d.cu kWQ
static_assert(kCHWQ * 4 == kLaneSamples, "a full warp unit is one lane_count_u8 call");
constexpr size_t kCHSmem = size_t(kCHWarps) * kLaneBins * kBinStride + kLaneBins * 4;

template <int W>
__global__ void __launch_bounds__(kCHWarps * 32)
    conv_hist_fixed_kernel(const float* __restrict__ x, const float* __restrict__ wts,
                           const float* __restrict__ cbias, float* __restrict__ u, uint64_t rows,
                           uint64_t dim, uint64_t L, int silu, double fixed_lo, double fixed_hi,
                           int k, unsigned long long* d_counts, double* d_range) {
  extern __shared__ __align__(128) unsigned char smem[];
  cnt_t* counters = reinterpret_cast<cnt_t*>(smem);
  uint32_t* cta_hist = reinterpret_cast<uint32_t*>(smem + size_t(kCHWarps) * kLaneBins * kBinStride);
  __shared__ BinParams sp;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) sp = make_bin_params_lohi(fixed_lo, fixed_hi, k);
  {
    uint4* c4 = reinterpret_cast<uint4*>(smem);
    for (int i = threadIdx.x; i < static_cast<int>(size_t(kCHWarps) * kLaneBins * kBinStride / 16);
         i += blockDim.x)
      c4[i] = make_uint4(0, 0, 0, 0);
    for (int i = threadIdx.x; i < kLaneBins; i += blockDim.x) cta_hist[i] = 0;
  }
  __syncthreads();
  const BinParams p = sp;
  unsigned char* lane_base =
      reinterpret_cast<unsigned char*>(counters + warp * kLaneBins * 32) + lane * 4;
  const uint64_t qpr = L / 4;
  const uint64_t runs_per_row = qpr / (32 * kCHWQ);
  const uint64_t tail_blocks = (qpr / 32) % kCHWQ;
  const uint64_t units_per_row = runs_per_row + (tail_blocks ? 1 : 0);
  const uint64_t units = rows * units_per_row;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  float4* u4 = reinterpret_cast<float4*>(u);
  const uint64_t warps = static_cast<uint64_t>(gridDim.x) * kCHWarps;
  bool bad = false;
  uint32_t since_flush = 0;
  for (uint64_t unit = static_cast<uint64_t>(blockIdx.x) * kCHWarps + warp; unit < units;
       unit += warps) {
    const uint64_t row = unit / units_per_row;
    const uint64_t ur = unit - row * units_per_row;
    const int nb = ur < runs_per_row ? kCHWQ : static_cast<int>(tail_blocks);
    const uint64_t qb = row * qpr + ur * 32 * kCHWQ;
    const uint64_t d = row % dim;
    float4 in[kCHWQ];
#pragma unroll
    for (int m = 0; m < kCHWQ; ++m)
      in[m] = m < nb ? __ldcs(x4 + qb + m * 32 + lane) : make_float4(0.f, 0.f, 0.f, 0.f);
    float4 prev31 = make_float4(0.f, 0.f, 0.f, 0.f);
    if (ur > 0) prev31 = __ldg(x4 + qb - 1);
    float wk[W];
#pragma unroll
    for (int kk = 0; kk < W; ++kk) wk[kk] = __ldg(wts + d * W + kk);
    const float bias = cbias ? __ldg(cbias + d) : 0.f;
    float val[kLaneSamples];
#pragma unroll
    for (int m = 0; m < kCHWQ; ++m) {
      if (m >= nb) break;
      float o[4];
      conv_block<W>(in[m], prev31, lane, wk, bias, silu != 0, o);
      __stcs(u4 + qb + m * 32 + lane, make_float4(o[0], o[1], o[2], o[3]));
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        val[4 * m + i] = o[i];
        bad |= !range::finite_f32(o[i]);
      }
    }
    if (nb == kCHWQ) {
      lane_count_u8(val, p, reinterpret_cast<unsigned char*>(counters), warp, lane);
    } else {
#pragma unroll
      for (int m = 0; m < kCHWQ; ++m) {
        if (m >= nb) break;
#pragma unroll
        for (int i = 0; i < 4; ++i) cref(lane_base, bin_f32(val[4 * m + i], p, true)) += 1;
      }
    }
    if (++since_flush == kFlushChunks) {
      flush_warp(counters + warp * kLaneBins * 32, cta_hist, lane, k);
      since_flush = 0;
    }
  }
  flush_warp(counters + warp * kLaneBins * 32, cta_hist, lane, k);
  bad = __any_sync(0xffffffffu, bad);
  __syncthreads();
  for (int b = threadIdx.x; b < k; b += blockDim.x)
    if (cta_hist[b]) atomicAdd(d_counts + b, static_cast<unsigned long long>(cta_hist[b]));
  if (bad && lane == 0) range::atomic_max_f64(d_range + 2, 1.0);
}

// ---------------------------------------------------------------------------
// Lean entropy kernels, for co-scheduling under another call's scan (the pipelined
// prefill: call i+1's min/max + histogram run while call i's MUFU-bound scan leaves half of
// HBM idle; bench.py "pipelined").  Sized to fit beside a resident scan CTA (448 threads x
// 128 registers, ~149 KB of shared memory): 4 warps x <= 64 registers = 8192 registers
// and ~66 KB of shared memory, one CTA per SM.  The loads in flight live in a
// cp.async.bulk ring (kLeanStages x 4 KB) instead of registers; warp 0's lane 0 refills it.
// Dynamic range, stride 1, K <= 256 (the calibrated rule's configuration); results equal
// cl_minmax_f32 + cl_histogram_decide_f32 bit for bit.
// ---------------------------------------------------------------------------
constexpr int kLeanWarps = 4;
constexpr int kLeanSamples = 8;                             // per lane per chunk
constexpr int kLeanChunk = kLeanWarps * 32 * kLeanSamples;  // 1024 floats = 4 KB
constexpr int kLeanStages = 8;
constexpr size_t kLeanRing = size_t(kLeanStages) * kLeanChunk * 4;  // 32 KB
constexpr size_t kLeanMmSmem = kLeanRing + 2 * kLeanStages * 8 + 128;
constexpr size_t kLeanHistSmem =
    size_t(kLeanWarps) * kLaneBins * kBinStride + kLeanRing + kLaneBins * 4 + 2 * kLeanStages * 8 + 128;
constexpr int kLeanFlush = 240 / kLeanSamples;  // u8 counters: flush before 255

// The ring: chunk i of this CTA (global chunk blockIdx.x + i * gridDim.x) in stage i % S.
struct LeanRing {
  float* buf;
  uint64_t* full;
  uint64_t* empty;
  const float* body;
  uint64_t n_chunks;
  __device__ uint64_t chunk(uint64_t i) const { return blockIdx.x + i * gridDim.x; }
  __device__ void issue(uint64_t i) {  // one thread
    const uint64_t c = chunk(i);
    if (c >= n_chunks) return;
    const int st = static_cast<int>(i % kLeanStages);
    if (i >= static_cast<uint64_t>(kLeanStages))
      mbar_wait(empty + st, static_cast<uint32_t>((i / kLeanStages - 1) & 1));
    mbar_expect_tx(full + st, kLeanChunk * 4);
    bulk_g2s(buf + size_t(st) * kLeanChunk, body + c * kLeanChunk, kLeanChunk * 4, full + st);
  }
  __device__ const float* wait(uint64_t i) {
    const int st = static_cast<int>(i % kLeanStages);
    mbar_wait(full + st, static_cast<uint32_t>((i / kLeanStages) & 1));
    return buf + size_t(st) * kLeanChunk;
  }
  __device__ void release(uint64_t i, int lane) {
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + static_cast<int>(i % kLeanStages));
  }
};

__device__ __forceinline__ LeanRing lean_ring_setup(unsigned char* ring_base, const float* body,
                                                    uint64_t n_chunks) {
  LeanRing r;
  r.buf = reinterpret_cast<float*>(ring_base);
  r.full = reinterpret_cast<uint64_t*>(ring_base + kLeanRing);
  r.empty = r.full + kLeanStages;
  r.body = body;
  r.n_chunks = n_chunks;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kLeanStages; ++i) {
      mbar_init(r.full + i, 1);
      mbar_init(r.empty + i, kLeanWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kLeanWarps * 32, 8)
    minmax_lean_kernel(const float* __restrict__ v, uint64_t n, double* range) {
  extern __shared__ __align__(128) unsigned char lsm[];
  range::Acc acc;
  const int lane = threadIdx.x % 32, warp = threadIdx.x / 32;
  const uint64_t head = umin64(n, ((16u - (reinterpret_cast<uintptr_t>(v) & 15u)) & 15u) / 4u);
  const float* body = v + head;
  const uint64_t n_chunks = (n - head) / kLeanChunk;
  const uint64_t tail0 = head + n_chunks * kLeanChunk;
  if (blockIdx.x == 0) {
    for (uint64_t i = threadIdx.x; i < head; i += blockDim.x) acc.visit(v[i], true);
    for (uint64_t i = tail0 + threadIdx.x; i < n; i += blockDim.x) acc.visit(v[i], true);
  }
  LeanRing ring = lean_ring_setup(lsm, body, n_chunks);
  const uint64_t mine = blockIdx.x < n_chunks ? (n_chunks - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  if (threadIdx.x == 0)
    for (uint64_t i = 0; i + 1 < kLeanStages && i < mine; ++i) ring.issue(i);
  for (uint64_t i = 0; i < mine; ++i) {
    if (threadIdx.x == 0) ring.issue(i + kLeanStages - 1);
    const float4* c4 = reinterpret_cast<const float4*>(ring.wait(i));
    const float4 a = c4[warp * 64 + lane], b = c4[warp * 64 + 32 + lane];
    ring.release(i, lane);
    acc.visit(a.x, true), acc.visit(a.y, true), acc.visit(a.z, true), acc.visit(a.w, true);
    acc.visit(b.x, true), acc.visit(b.y, true), acc.visit(b.z, true), acc.visit(b.w, true);
  }
  range::commit<kLeanWarps * 32>(acc, range);
}

// (min 8 blocks per SM caps the registers at 65536 / (128 * 8) = 64)
__global__ void __launch_bounds__(kLeanWarps * 32, 8)
    hist_lean_kernel(const float* __restrict__ v, uint64_t n, int k,
                     const double* __restrict__ d_range, unsigned long long* d_counts,
                     DecideArgs da, cl_decision* d_out, unsigned long long* ticket) {
  extern __shared__ __align__(128) unsigned char lsm[];
  cnt_t* counters = reinterpret_cast<cnt_t*>(lsm);
  uint32_t* cta_hist =
      reinterpret_cast<uint32_t*>(lsm + size_t(kLeanWarps) * kLaneBins * kBinStride);
  unsigned char* ring_base = reinterpret_cast<unsigned char*>(cta_hist + kLaneBins);
  __shared__ BinParams sp;
  __shared__ bool last;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) sp = make_bin_params(d_range, CL_RANGE_DYNAMIC, 0.0, 0.0, k);
  {
    uint4* c4 = reinterpret_cast<uint4*>(lsm);
    for (int i = threadIdx.x; i < static_cast<int>(size_t(kLeanWarps) * kLaneBins * kBinStride / 16);
         i += blockDim.x)
      c4[i] = make_uint4(0, 0, 0, 0);
    for (int i = threadIdx.x; i < kLaneBins; i += blockDim.x) cta_hist[i] = 0;
  }
  const uint64_t head = umin64(n, ((16u - (reinterpret_cast<uintptr_t>(v) & 15u)) & 15u) / 4u);
  const float* body = v + head;
  const uint64_t n_chunks = (n - head) / kLeanChunk;
  const uint64_t tail0 = head + n_chunks * kLeanChunk;
  LeanRing ring = lean_ring_setup(ring_base, body, n_chunks);  // (its __syncthreads publishes sp)
  const BinParams p = sp;
  unsigned char* lane_base =
      reinterpret_cast<unsigned char*>(counters + warp * kLaneBins * 32) + lane * 4;
  if (blockIdx.x == 0 && warp == 0) {
    for (uint64_t i = lane; i < head; i += 32) cref(lane_base, bin_f32(v[i], p, false)) += 1;
    for (uint64_t i = tail0 + lane; i < n; i += 32) cref(lane_base, bin_f32(v[i], p, false)) += 1;
    flush_warp(counters + warp * kLaneBins * 32, cta_hist, lane, k);
  }
  const uint64_t mine = blockIdx.x < n_chunks ? (n_chunks - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  if (threadIdx.x == 0)
    for (uint64_t i = 0; i + 1 < kLeanStages && i < mine; ++i) ring.issue(i);
  int since = 0;
  for (uint64_t i = 0; i < mine; ++i) {
    if (threadIdx.x == 0) ring.issue(i + kLeanStages - 1);
    const float4* c4 = reinterpret_cast<const float4*>(ring.wait(i));
    const float4 a = c4[warp * 64 + lane], b = c4[warp * 64 + 32 + lane];
    ring.release(i, lane);
    const float val[kLeanSamples] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    lane_count_u8(val, p, reinterpret_cast<unsigned char*>(counters), warp, lane);
    if (++since == kLeanFlush) {
      flush_warp(counters + warp * kLaneBins * 32, cta_hist, lane, k);
      since = 0;
    }
  }
  flush_warp(counters + warp * kLaneBins * 32, cta_hist, lane, k);
  __syncthreads();
  for (int b = threadIdx.x; b < k; b += blockDim.x)
    if (cta_hist[b]) atomicAdd(d_counts + b, static_cast<unsigned long long>(cta_hist[b]));
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1ull) == gridDim.x - 1;
  __syncthreads();
  if (last) {
    __threadfence();
    decide_block<true>(da, d_out);
    if (threadIdx.x == 0) *ticket = 0ull;
  }
}

// K > 256 (or f64 input): shared-memory atomics on a CTA histogram.
template <typename T, int MODE>
__global__ void __launch_bounds__(kThreads)
    hist_atomic_kernel(const T* __restrict__ v, uint64_t n, uint64_t g0, uint64_t stride,
                       int range_mode, double fixed_lo, double fixed_hi, int k,
                       const double* __restrict__ d_range, unsigned long long* d_counts,
                       int use_smem) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem_raw);
  __shared__ BinParams sp;
  if (threadIdx.x == 0) sp = make_bin_params(d_range, range_mode, fixed_lo, fixed_hi, k);
  if (use_smem)
    for (int i = threadIdx.x; i < k; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  const BinParams p = sp;
  const uint64_t nthr = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += nthr) {
    if (!sampled<MODE>(g0 + i, stride)) continue;
    int b;
    if constexpr (sizeof(T) == 4)
      b = bin_f32(v[i], p, range_mode == CL_RANGE_FIXED);
    else
      b = bin_index_exact(v[i], p.lo, p.width, k);
    if (use_smem)
      atomicAdd(hist + b, 1u);
    else
      atomicAdd(d_counts + b, 1ull);
  }
  if (use_smem) {
    __syncthreads();
    for (int i = threadIdx.x; i < k; i += blockDim.x)
      if (hist[i]) atomicAdd(d_counts + i, static_cast<unsigned long long>(hist[i]));
  }
}

// ---------------------------------------------------------------------------
// token_entropy (entropy.hpp:180-210): the tensor read as (channels, length), one
// compute_histogram per position t over its channel slice (slice index c sampled iff
// c % stride == 0; Dynamic range of the slice's samples or the Fixed range), and the
// per-position raw entropies averaged in position order.
//
// Four stream-ordered stages (the multi-GPU protocol inserts its two collectives
// between them, exactly as for the global histogram).  fp32 inputs with K <= 256 and
// 16-byte aligned rows take the lane-per-position kernels further down
// (token_minmax_lane_kernel, token_hist_lane_kernel); the tiled kernels here serve fp64,
// K > 256 and unaligned inputs:
//   1. token_minmax: blocks own a tile of 32 positions (8 x float4) x a share of the channels;
//      a thread loads 16 contiguous bytes of one channel row per step (a warp covers 4
//      channel rows x 128 B), keeps per-position min/max + the finite flag, and the
//      block folds them into trange [2][L] = {-lo, hi} with fp64 atomic max.
//   2. token_hist: same tiling, per-position bin parameters from trange, an
//      [32][K] u32 shared-memory histogram flushed into counts [L][K] (global
//      atomics straight into counts when the tile does not fit shared memory).
//   3. token_entropy: a warp per position, estimate_entropy in fp64, bin order.
//   4. token_finalize: the ordered mean over positions.
// Channel indices are global (channel_offset + c) so a row-sharded tensor samples the
// same slice entries as the whole one.
// ---------------------------------------------------------------------------
constexpr int kTokMaxSmemHist = 64 * 1024;

template <typename T>
struct TokVec {
  static constexpr int kV = 16 / sizeof(T);  // elements per 16-byte load
};

struct TokArgs {
  uint64_t channels, length, offset, stride;
  int k;
  int vec;  // 1: vector loads (length % kV == 0, aligned), 0: scalar
};

// Per-thread walk over this block's channel share with the sampled test kept as an
// incremental c_global % stride.
struct ChanWalk {
  uint64_t c, end, cm, step_mod, stride;
  __device__ ChanWalk(uint64_t c0, uint64_t end_, uint64_t offset, uint64_t step, uint64_t st)
      : c(c0), end(end_), cm((offset + c0) % st), step_mod(step % st), stride(st) {}
  __device__ __forceinline__ bool ok() const { return c < end; }
  __device__ __forceinline__ bool sampled() const { return cm == 0; }
  __device__ __forceinline__ void next(uint64_t step) {
    c += step;
    cm += step_mod;
    if (cm >= stride) cm -= stride;
  }
};

__device__ __forceinline__ void tok_channel_share(uint64_t channels, uint64_t* c0,
                                                  uint64_t* c1) {
  const uint64_t per = (channels + gridDim.y - 1) / gridDim.y;
  *c0 = per * blockIdx.y;
  *c1 = umin64(channels, *c0 + per);
}

// thread -> (position group g of 8, channel lane cl of 32); a group is kV positions for
// vector loads (8 x kV = 32 for fp32) or 1 position for scalar loads.
template <typename T, int VEC>
__global__ void __launch_bounds__(kThreads) token_minmax_kernel(const T* __restrict__ v,
                                                                TokArgs a, double* trange,
                                                                double* flag) {
  constexpr int kV = VEC ? TokVec<T>::kV : 1;
  constexpr int kTile = 8 * kV;
  const int g = threadIdx.x % 8, cl = threadIdx.x / 8;
  const uint64_t t0 = static_cast<uint64_t>(blockIdx.x) * kTile + g * kV;
  uint64_t c0, c1;
  tok_channel_share(a.channels, &c0, &c1);
  double lo[kV], hi[kV];
#pragma unroll
  for (int e = 0; e < kV; ++e) {
    lo[e] = INFINITY;
    hi[e] = -INFINITY;
  }
  bool bad = false;
  if (t0 < a.length) {
    for (ChanWalk w(c0 + cl, c1, a.offset, kThreads / 8, a.stride); w.ok(); w.next(kThreads / 8)) {
      const T* row = v + w.c * a.length + t0;
      T x[kV];
      if (VEC) {
        *reinterpret_cast<typename Vec4<T>::type*>(x) =
            __ldcs(reinterpret_cast<const typename Vec4<T>::type*>(row));
      } else {
        x[0] = row[0];
      }
#pragma unroll
      for (int e = 0; e < kV; ++e) {
        const double d = static_cast<double>(x[e]);
        bad |= !finite_f64(d);
        if (w.sampled()) {
          lo[e] = fmin(lo[e], d);
          hi[e] = fmax(hi[e], d);
        }
      }
    }
  }
  // lanes g, g+8, g+16, g+24 of a warp share positions: fold them, then across warps
#pragma unroll
  for (int e = 0; e < kV; ++e) {
    for (int o = 8; o < 32; o <<= 1) {
      lo[e] = fmin(lo[e], __shfl_xor_sync(0xffffffffu, lo[e], o));
      hi[e] = fmax(hi[e], __shfl_xor_sync(0xffffffffu, hi[e], o));
    }
  }
  bad = __any_sync(0xffffffffu, bad);
  __shared__ double s_lo[kThreads / 32][kTile], s_hi[kThreads / 32][kTile];
  __shared__ int s_bad[kThreads / 32];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (lane < 8) {
#pragma unroll
    for (int e = 0; e < kV; ++e) {
      s_lo[warp][lane * kV + e] = lo[e];
      s_hi[warp][lane * kV + e] = hi[e];
    }
  }
  if (lane == 0) s_bad[warp] = bad;
  __syncthreads();
  if (threadIdx.x < kTile) {
    const uint64_t t = static_cast<uint64_t>(blockIdx.x) * kTile + threadIdx.x;
    double l = s_lo[0][threadIdx.x], h = s_hi[0][threadIdx.x];
    for (int w = 1; w < kThreads / 32; ++w) {
      l = fmin(l, s_lo[w][threadIdx.x]);
      h = fmax(h, s_hi[w][threadIdx.x]);
    }
    if (t < a.length && h >= l) {
      atomic_max_f64(trange + t, -l);
      atomic_max_f64(trange + a.length + t, h);
    }
  }
  if (threadIdx.x == 0) {
    int b = 0;
    for (int w = 0; w < kThreads / 32; ++w) b |= s_bad[w];
    if (b) atomic_max_f64(flag, 1.0);
  }
}

template <typename T, int VEC, bool FIXED, bool SMEM>
__global__ void __launch_bounds__(kThreads) token_hist_kernel(const T* __restrict__ v,
                                                              TokArgs a, const double* trange,
                                                              double fixed_lo, double fixed_hi,
                                                              unsigned int* counts) {
  constexpr int kV = VEC ? TokVec<T>::kV : 1;
  constexpr int kTile = 8 * kV;
  extern __shared__ unsigned int thist[];  // [kTile][k] when SMEM
  __shared__ BinParams bp[kTile];
  const int k = a.k;
  const uint64_t tb = static_cast<uint64_t>(blockIdx.x) * kTile;
  if (SMEM)
    for (int i = threadIdx.x; i < kTile * k; i += kThreads) thist[i] = 0u;
  if (threadIdx.x < kTile) {
    const uint64_t t = tb + threadIdx.x;
    bp[threadIdx.x] = FIXED ? make_bin_params_lohi(fixed_lo, fixed_hi, k)
                    : t < a.length ? make_bin_params_lohi(-trange[t], trange[a.length + t], k)
                                   : make_bin_params_lohi(0.0, 0.0, k);
  }
  __syncthreads();
  const int g = threadIdx.x % 8, cl = threadIdx.x / 8;
  const uint64_t t0 = tb + g * kV;
  uint64_t c0, c1;
  tok_channel_share(a.channels, &c0, &c1);
  if (t0 < a.length) {
    BinParams P[kV];
#pragma unroll
    for (int e = 0; e < kV; ++e) P[e] = bp[g * kV + e];
    for (ChanWalk w(c0 + cl, c1, a.offset, kThreads / 8, a.stride); w.ok(); w.next(kThreads / 8)) {
      if (!w.sampled()) continue;
      const T* row = v + w.c * a.length + t0;
      T x[kV];
      if (VEC) {
        *reinterpret_cast<typename Vec4<T>::type*>(x) =
            __ldcs(reinterpret_cast<const typename Vec4<T>::type*>(row));
      } else {
        x[0] = row[0];
      }
#pragma unroll
      for (int e = 0; e < kV; ++e) {
        int bin;
        if (sizeof(T) == 4)
          bin = bin_f32(static_cast<float>(x[e]), P[e], FIXED);
        else
          bin = bin_index_exact(static_cast<double>(x[e]), P[e].lo, P[e].width, k);
        if (SMEM)
          atomicAdd(thist + (g * kV + e) * k + bin, 1u);
        else
          atomicAdd(counts + (t0 + e) * k + bin, 1u);
      }
    }
  }
  if (!SMEM) return;
  __syncthreads();
  for (int i = threadIdx.x; i < kTile * k; i += kThreads) {
    const uint64_t t = tb + i / k;
    if (t < a.length && thist[i]) atomicAdd(counts + t * k + (i % k), thist[i]);
  }
}

// ---- fp32 fast path (K <= 256, 16-byte aligned rows): lane-per-position kernels ----
// The tiled kernels above give every (position, bin) counter to many threads, so each
// sample is a shared-memory atomic (ATOMS throughput bound).  Here a lane owns positions:
//   min/max  a lane holds 4 consecutive positions (one float4 per channel row), a warp
//            streams 512 contiguous bytes of one row per load, the block's 8 warps split
//            the channel share and fold their ranges in shared memory;
//   hist     a lane owns ONE position and lane-private 16-bit counters [bin][lane] (16 KB
//            per warp, no atomics; in-order pairwise read-modify-write as in the global
//            histogram), a warp reads 128 contiguous bytes of one channel row per load;
//            the block's 4 warps are summed at the end and added to counts [L][K].
// Work items are (position tile, channel split) pairs walked grid-stride by resident
// blocks.  Channels are sampled by global index (channel_offset + c) % stride == 0 (the
// minmax pass still reads every channel: the finite check covers all values).
constexpr int kTokMmWarps = 8;              // min/max: warps per block, 128 positions
constexpr int kTokHWarps = 4;               // hist: warps per block, 32 positions
#ifndef CL_TOK_MM_ROWS
#define CL_TOK_MM_ROWS 8
#endif
#ifndef CL_TOK_H_UNROLL
#define CL_TOK_H_UNROLL 24
#endif
// Measured at C3 (u 8x4096x8192 as 32768 channels x 8192 positions): min/max 0.31-0.33 ms
// for 4, 8 or 16 rows per batch with one 128-position slice per block, 0.25 with 2-4
// slices side by side (the block reads 1-2 KB of a row at a time: DRAM locality), 0.26
// with 8; histogram 0.98 / 0.72 / 0.53 / 0.47 / 0.77 ms for 4 / 8 /
// 16 / 24 / 32 rows (32: 182 registers, 2 blocks per SM).  Loads in flight, not
// instructions, bound the histogram: a lane reads 4 bytes of a row, a warp 128 bytes.
// Giving the block's warps 2 or 4 adjacent 32-position slices (256 / 512 contiguous bytes
// of a row per block step, as in the min/max kernel) measured slower: 0.51 / 0.56 ms; so
// did bulk L2 prefetches of each warp's row segments 1-4 batches ahead: 0.59-0.61 ms.
#ifndef CL_TOK_MM_COLS
#define CL_TOK_MM_COLS 4
#endif
constexpr int kTokMmRows = CL_TOK_MM_ROWS;  // min/max: channel rows per batch
constexpr int kTokMmCols = CL_TOK_MM_COLS;  // min/max: 128-position slices per block tile
constexpr int kTokHUnroll = CL_TOK_H_UNROLL;  // hist: channel rows per batch (2 in flight)
constexpr int kTokHMaxPerFlush = 65000;     // u16 counters: flush before overflow
// Token histogram kernel: the TMA-fed one (default, CL_TOK_TMA=1) or the LDG-fed lane
// kernel (CL_TOK_TMA=0).  Measured at C3 (channels 32768, L 8192, K 256;
// profiles/r2f_token_ab.txt): lane 0.537 ms; TMA first version 0.670 ms (ALU-bound: 64% of the
// ALU pipe, 42 instructions per 32-sample step -- per-row sampling masks, pair-layout
// addressing); with the stride-1 mask computed once, [bin][lane] addressing and constant
// increments for full boxes: below.
// min/max CTAs per SM (8 x 256 threads: a C1-sized input is one batch of 4 float4 loads per
// thread, all in flight at once) and the register-fed histogram's minimum chunks per warp
#ifndef CL_MM_CTAS_PER_SM
#define CL_MM_CTAS_PER_SM 4
#endif
#ifndef CL_HIST_MIN_CHUNKS
#define CL_HIST_MIN_CHUNKS 1
#endif
#ifndef CL_TOK_TMA
#define CL_TOK_TMA 1
#endif
#ifndef CL_TOK_QUAD
#define CL_TOK_QUAD 1
#endif
#ifndef CL_TOK_RED
#define CL_TOK_RED 1
#endif

__device__ __forceinline__ void tok_item_split(uint64_t item, uint64_t tiles, uint64_t splits,
                                               uint64_t channels, uint64_t* tile,
                                               uint64_t* c0, uint64_t* c1) {
  *tile = item % tiles;
  const uint64_t sp = item / tiles;
  const uint64_t per = (channels + splits - 1) / splits;
  *c0 = sp * per;
  *c1 = umin64(channels, *c0 + per);
}

__global__ void __launch_bounds__(kTokMmWarps * 32) token_minmax_lane_kernel(
    const float* __restrict__ v, TokArgs a, uint64_t tiles, uint64_t splits, double* trange,
    double* flag) {
  __shared__ float s_lo[kTokMmWarps][128], s_hi[kTokMmWarps][128];
  __shared__ int s_bad;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) s_bad = 0;
  bool bad = false;
  for (uint64_t item = blockIdx.x; item < tiles * splits; item += gridDim.x) {
    uint64_t tile, c0, c1;
    tok_item_split(item, tiles, splits, a.channels, &tile, &c0, &c1);
    // kTokMmCols 128-position column slices per tile; the kTokMmWarps / kTokMmCols warps
    // of a slice split the item's channels
    constexpr int kSliceWarps = kTokMmWarps / kTokMmCols;
    const int col = warp / kSliceWarps, wsl = warp % kSliceWarps;
    const uint64_t t0 = (tile * kTokMmCols + col) * 128 + lane * 4;
    float lo[4] = {INFINITY, INFINITY, INFINITY, INFINITY};
    float hi[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
    if (t0 < a.length) {
      const uint64_t per = (c1 - c0 + kSliceWarps - 1) / kSliceWarps;
      const uint64_t w0 = umin64(c1, c0 + wsl * per), w1 = umin64(c1, w0 + per);
      uint64_t cm = (a.offset + w0) % a.stride;  // (offset + c) % stride, incremental
      uint64_t c = w0;
      const float* rp = v + w0 * a.length + t0;
      // one batch of rows in flight ahead of the one being reduced
      float4 qn[kTokMmRows];
      if (c + kTokMmRows <= w1) {
#pragma unroll
        for (int i = 0; i < kTokMmRows; ++i) {
          qn[i] = __ldcs(reinterpret_cast<const float4*>(rp));
          rp += a.length;
        }
      }
      for (; c + kTokMmRows <= w1; c += kTokMmRows) {
        float4 q[kTokMmRows];
#pragma unroll
        for (int i = 0; i < kTokMmRows; ++i) q[i] = qn[i];
        if (c + 2 * kTokMmRows <= w1) {
#pragma unroll
          for (int i = 0; i < kTokMmRows; ++i) {
            qn[i] = __ldcs(reinterpret_cast<const float4*>(rp));
            rp += a.length;
          }
        }
#pragma unroll
        for (int i = 0; i < kTokMmRows; ++i) {
          const float x[4] = {q[i].x, q[i].y, q[i].z, q[i].w};
          const bool smp = cm == 0;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            bad |= !(fabsf(x[e]) <= FLT_MAX);
            if (smp) {
              lo[e] = x[e] < lo[e] ? x[e] : lo[e];  // std::min keeps lo unless x < lo
              hi[e] = hi[e] < x[e] ? x[e] : hi[e];
            }
          }
          if (++cm == a.stride) cm = 0;
        }
      }
      for (; c < w1; ++c) {
        const float4 q = __ldcs(reinterpret_cast<const float4*>(v + c * a.length + t0));
        const float x[4] = {q.x, q.y, q.z, q.w};
        const bool smp = cm == 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          bad |= !(fabsf(x[e]) <= FLT_MAX);
          if (smp) {
            lo[e] = x[e] < lo[e] ? x[e] : lo[e];
            hi[e] = hi[e] < x[e] ? x[e] : hi[e];
          }
        }
        if (++cm == a.stride) cm = 0;
      }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      s_lo[warp][lane * 4 + e] = lo[e];
      s_hi[warp][lane * 4 + e] = hi[e];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 128 * kTokMmCols; i += blockDim.x) {
      const int cs = i / 128, p = i % 128;
      const uint64_t t = (tile * kTokMmCols + cs) * 128 + p;
      float l = s_lo[cs * kSliceWarps][p], h = s_hi[cs * kSliceWarps][p];
      for (int w = 1; w < kSliceWarps; ++w) {
        l = s_lo[cs * kSliceWarps + w][p] < l ? s_lo[cs * kSliceWarps + w][p] : l;
        h = h < s_hi[cs * kSliceWarps + w][p] ? s_hi[cs * kSliceWarps + w][p] : h;
      }
      if (t < a.length && h >= l) {
        atomic_max_f64(trange + t, -static_cast<double>(l));
        atomic_max_f64(trange + a.length + t, static_cast<double>(h));
      }
    }
    __syncthreads();
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) s_bad = 1;
  __syncthreads();
  if (threadIdx.x == 0 && s_bad) atomic_max_f64(flag, 1.0);
}

// u16 counters of (warp w, bin b, lane l): lane l owns the 32-bit word (b/2)*32 + l of its
// warp's 16 KB block, even bin in the low half, odd in the high -- every lane addresses
// only its own bank (the earlier [bin][lane] halves put a lane pair in one bank with
// different words whenever their bins differed with equal parity: 48% of shared wavefronts
// were conflicts, ncu, profiles/r2f_token_ncu.txt).
__device__ __forceinline__ uint32_t tok_cidx(int w, int b, int lane) {  // in u16 units
  return static_cast<uint32_t>(w) * 8192u + ((static_cast<uint32_t>(b) >> 1) * 32u + lane) * 2u +
         (static_cast<uint32_t>(b) & 1u);
}

// Adds the block's 4 warps' counters for its 32 positions into counts [L][K] and clears
// them: warp w sums bins w, w+4, ... over the warps for position (tile*32 + lane).
__device__ __forceinline__ void tok_flush(uint16_t* cnt, uint64_t t, bool t_ok, int k,
                                          unsigned int* counts) {
  __syncthreads();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int b = warp; b < k; b += kTokHWarps) {
    uint32_t sum = 0;
#pragma unroll
    for (int w = 0; w < kTokHWarps; ++w) sum += cnt[tok_cidx(w, b, lane)];
    if (sum && t_ok) atomicAdd(counts + t * k + b, sum);
  }
  __syncthreads();
  uint4* c4 = reinterpret_cast<uint4*>(cnt);
  for (int i = threadIdx.x; i < kTokHWarps * 256 * 32 * 2 / 16; i += blockDim.x)
    c4[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();
}

template <bool FIXED>
__global__ void __launch_bounds__(kTokHWarps * 32) token_hist_lane_kernel(
    const float* __restrict__ v, TokArgs a, uint64_t tiles, uint64_t splits,
    const double* trange, double fixed_lo, double fixed_hi, unsigned int* counts) {
  extern __shared__ __align__(16) uint16_t tcnt[];  // [warp][128 bin pairs][32 lanes][2]
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int k = a.k;
  {
    uint4* c4 = reinterpret_cast<uint4*>(tcnt);
    for (int i = threadIdx.x; i < kTokHWarps * 256 * 32 * 2 / 16; i += blockDim.x)
      c4[i] = make_uint4(0, 0, 0, 0);
  }
  __syncthreads();
  const uint32_t cbase = static_cast<uint32_t>(__cvta_generic_to_shared(tcnt)) +
                         static_cast<uint32_t>(warp) * (256 * 32 * 2) + lane * 4u;
  for (uint64_t item = blockIdx.x; item < tiles * splits; item += gridDim.x) {
    uint64_t tile, c0, c1;
    tok_item_split(item, tiles, splits, a.channels, &tile, &c0, &c1);
    const uint64_t t = tile * 32 + lane;
    const bool t_ok = t < a.length;
    const BinParams P = FIXED ? make_bin_params_lohi(fixed_lo, fixed_hi, k)
                        : t_ok ? make_bin_params_lohi(-trange[t], trange[a.length + t], k)
                               : make_bin_params_lohi(0.0, 0.0, k);
    // this warp's sampled channels: c = cf + i*stride, cf the first sampled one >= w0
    const uint64_t per = (c1 - c0 + kTokHWarps - 1) / kTokHWarps;
    const uint64_t w0 = umin64(c1, c0 + warp * per), w1 = umin64(c1, w0 + per);
    const uint64_t r = (a.offset + w0) % a.stride;
    const uint64_t cf = w0 + (r == 0 ? 0 : a.stride - r);
    const uint64_t n = cf < w1 ? (w1 - cf + a.stride - 1) / a.stride : 0;
    // block-uniform trip count (an upper bound on every warp's n), so the flush's
    // __syncthreads below is reached by all warps together
    const uint64_t n_blk = per / a.stride + 1;
    const float* col = v + (t_ok ? t : 0);
    const uint64_t rstep = a.stride * a.length;  // elements between sampled rows
    const uint32_t inc = t_ok ? 1u : 0u;
    uint32_t since = 0;
    // loads run one batch ahead of the binning: 2 x kTokHUnroll rows in flight per lane;
    // full batches (the common case) carry no per-sample predicates
    float xn[kTokHUnroll];
    {
      const float* q = col + cf * a.length;
#pragma unroll
      for (int u = 0; u < kTokHUnroll; ++u) {
        xn[u] = static_cast<uint64_t>(u) < n ? __ldcs(q) : 0.f;
        q += rstep;
      }
    }
    for (uint64_t i = 0; i < n_blk; i += kTokHUnroll) {
      float x[kTokHUnroll];
#pragma unroll
      for (int u = 0; u < kTokHUnroll; ++u) x[u] = xn[u];
      const float* q = col + (cf + (i + kTokHUnroll) * a.stride) * a.length;
      if (i + 2 * kTokHUnroll <= n) {
#pragma unroll
        for (int u = 0; u < kTokHUnroll; ++u) {
          xn[u] = __ldcs(q);
          q += rstep;
        }
      } else {
#pragma unroll
        for (int u = 0; u < kTokHUnroll; ++u) {
          xn[u] = i + kTokHUnroll + u < n ? __ldcs(q) : 0.f;
          q += rstep;
        }
      }
      int bin[kTokHUnroll];
      bool any_slow = P.exact_only != 0;
#pragma unroll
      for (int u = 0; u < kTokHUnroll; ++u) {
        bool sl;
        bin[u] = bin_fast<FIXED>(x[u], P, &sl);
        any_slow |= sl;
      }
      if (__any_sync(0xffffffffu, any_slow)) {
#pragma unroll
        for (int u = 0; u < kTokHUnroll; ++u) {
          bool sl;
          bin_fast<FIXED>(x[u], P, &sl);
          if (sl || P.exact_only)
            bin[u] = bin_index_exact(static_cast<double>(x[u]), P.lo, P.width, k);
        }
      }
      const bool full = i + kTokHUnroll <= n;
#pragma unroll
      for (int g = 0; g < kTokHUnroll / 2; ++g) {
        const uint32_t i0 = (full || i + 2 * g < n) ? inc : 0u;
        const uint32_t i1 = (full || i + 2 * g + 1 < n) ? inc : 0u;
        const int b0 = bin[2 * g], b1 = bin[2 * g + 1];
        const uint32_t a0 = cbase + (static_cast<uint32_t>(b0) & ~1u) * 64u + (b0 & 1) * 2u;
        const uint32_t a1 = cbase + (static_cast<uint32_t>(b1) & ~1u) * 64u + (b1 & 1) * 2u;
        uint32_t v0, v1;
        asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v0) : "r"(a0) : "memory");
        asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v1) : "r"(a1) : "memory");
        v0 += i0;
        v1 += i1 + (b0 == b1 ? i0 : 0u);
        asm volatile("st.shared.u16 [%0], %1;" ::"r"(a0), "h"(static_cast<uint16_t>(v0)) : "memory");
        asm volatile("st.shared.u16 [%0], %1;" ::"r"(a1), "h"(static_cast<uint16_t>(v1)) : "memory");
      }
      since += kTokHUnroll;
      // flush before a 16-bit counter can overflow (block-uniform condition)
      if (since >= kTokHMaxPerFlush && i + kTokHUnroll < n_blk) {
        tok_flush(tcnt, t, t_ok, k, counts);
        since = 0;
      }
    }
    tok_flush(tcnt, t, t_ok, k, counts);
  }
}

// TMA-fed token histogram (the fp32 / K <= 256 hot path of token_entropy stage 2).  A block
// owns a tile of 128 positions and a channel range; its producer warp streams boxes of
// {128 positions x kTokBoxRows channel rows} (8 KB) through a kTokStages-deep shared-memory
// ring with cp.async.bulk.tensor, so the loads in flight per SM no longer live in consumer
// registers (the LDG-fed lane kernel above sat on long-scoreboard stalls at 12 warps per SM,
// profiles/r2f_token_ncu.txt).  Consumer warp w owns positions 32w .. 32w+31 of the tile (lane
// = position) with private u16 counters in the bank-exclusive pair layout (tok_cidx), reads
// its 32 floats of each sampled row from the stage (conflict-free), bins them exactly like the
// lane kernel, and at the end of the item adds its counters into counts [L][K] (atomics; the
// positions of different warps are disjoint, so no block reduction).
constexpr int kTokTWarps = 4;                      // consumer warps: 128 positions
constexpr int kTokBoxRows = 16;                    // channel rows per box
constexpr int kTokStages = 5;                      // ring depth (2 blocks fit an SM)
constexpr int kTokBoxBytes = 128 * kTokBoxRows * 4;  // 8 KB
constexpr size_t kTokTSmem = size_t(kTokTWarps) * 256 * 32 * 2 + size_t(kTokStages) * kTokBoxBytes +
                             2 * kTokStages * 8 + 1024;

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

template <bool FIXED>
__global__ void __launch_bounds__((kTokTWarps + 1) * 32) token_hist_tma_kernel(
    const __grid_constant__ CUtensorMap map, TokArgs a, uint64_t tiles, uint64_t splits,
    const double* trange, double fixed_lo, double fixed_hi, unsigned int* counts) {
  extern __shared__ __align__(128) unsigned char tsm[];
  unsigned char* base = tsm + ((1024u - (smem_u32(tsm) & 1023u)) & 1023u);
  uint16_t* tcnt = reinterpret_cast<uint16_t*>(base);  // [warp][256 bins][32 lanes]
  unsigned char* ring = base + size_t(kTokTWarps) * 256 * 32 * 2;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + size_t(kTokStages) * kTokBoxBytes);
  uint64_t* empty = full + kTokStages;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int k = a.k;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kTokStages; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, kTokTWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  {
    uint4* c4 = reinterpret_cast<uint4*>(tcnt);
    for (int i = threadIdx.x; i < kTokTWarps * 256 * 32 * 2 / 16; i += blockDim.x)
      c4[i] = make_uint4(0, 0, 0, 0);
  }
  __syncthreads();
  const uint64_t n_items = tiles * splits;
  const uint64_t per_split = (a.channels + splits - 1) / splits;
  if (warp == kTokTWarps) {
    // ---------------- producer ----------------
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map)));
      uint32_t it = 0;
      for (uint64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
        const uint64_t tile = item % tiles, c0 = (item / tiles) * per_split;
        const uint64_t c1 = umin64(a.channels, c0 + per_split);
        for (uint64_t c = c0; c < c1; c += kTokBoxRows, ++it) {
          const int st = it % kTokStages;
          // (a nanosleep backoff instead of this wait measured no different, r2n)
          if (it >= static_cast<uint32_t>(kTokStages)) mbar_wait(empty + st, ((it / kTokStages) - 1) & 1);
          mbar_expect_tx(full + st, kTokBoxBytes);
          tma_load_3d(ring + size_t(st) * kTokBoxBytes, &map, static_cast<int>(tile * 128),
                      static_cast<int>(c), 0, full + st);
        }
      }
    }
    return;
  }
  // ---------------- consumers ----------------
  const uint32_t cbase = smem_u32(tcnt) + static_cast<uint32_t>(warp) * (256 * 32 * 2) + lane * 2u;
  uint32_t it = 0;
  for (uint64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
    const uint64_t tile = item % tiles, c0 = (item / tiles) * per_split;
    const uint64_t c1 = umin64(a.channels, c0 + per_split);
    const uint64_t t = tile * 128 + warp * 32 + lane;
    const bool t_ok = t < a.length;
    const BinParams P = FIXED ? make_bin_params_lohi(fixed_lo, fixed_hi, k)
                        : t_ok ? make_bin_params_lohi(-trange[t], trange[a.length + t], k)
                               : make_bin_params_lohi(0.0, 0.0, k);
    uint64_t cm = (a.offset + c0) % a.stride;  // (offset + c) % stride of the box's first row
    uint32_t since = 0;
    for (uint64_t c = c0; c < c1; c += kTokBoxRows, ++it) {
      const int st = it % kTokStages;
      mbar_wait(full + st, (it / kTokStages) & 1);
      const float* box = reinterpret_cast<const float*>(ring + size_t(st) * kTokBoxBytes);
      const int rows = static_cast<int>(umin64(kTokBoxRows, c1 - c));
      float x[kTokBoxRows];
#pragma unroll
      for (int r = 0; r < kTokBoxRows; ++r) x[r] = box[r * 128 + warp * 32 + lane];
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + st);  // the stage's values are in registers
      // bit r: row r is one of this item's channels and sampled (stride 1: all of them)
      uint32_t smp;
      if (a.stride == 1) {
        smp = rows == kTokBoxRows ? 0xFFFFu : (1u << rows) - 1u;
      } else {
        smp = 0;
#pragma unroll
        for (int r = 0; r < kTokBoxRows; ++r) {
          smp |= (r < rows && cm == 0 ? 1u : 0u) << r;
          if (++cm == a.stride) cm = 0;
        }
      }
      if (!t_ok) smp = 0;
      // every row is binned (exactly where needed), so every bin is in [0, k): rows outside
      // the item or unsampled only add 0
      int bin[kTokBoxRows];
      bool any_slow = P.exact_only != 0;
#pragma unroll
      for (int r = 0; r < kTokBoxRows; ++r) {
        bool sl;
        bin[r] = bin_fast<FIXED>(x[r], P, &sl);
        any_slow |= sl;
      }
      if (__any_sync(0xffffffffu, any_slow)) {
#pragma unroll
        for (int r = 0; r < kTokBoxRows; ++r) {
          bool sl;
          bin_fast<FIXED>(x[r], P, &sl);
          if (sl || P.exact_only) bin[r] = bin_index_exact(static_cast<double>(x[r]), P.lo, P.width, k);
        }
      }
      // u16 counters [bin][lane] (address = base + bin * 64: one IMAD; the lane pair sharing
      // a bank word conflicts only on different bins of equal parity -- this loop is
      // ALU-bound, not shared-memory-bound, ncu r2f)
      if (CL_TOK_RED) {
        // one shared-memory reduction per sample on the 32-bit word the lane shares with
        // its neighbour: this lane's u16 half is 1 << 16 * (lane & 1) (<= 65000 counts
        // between flushes, so a half never carries); no read-modify-write chain
        const uint32_t wbase = cbase & ~3u;
        const uint32_t inc1 = 1u << ((lane & 1) * 16);
        if (__all_sync(0xffffffffu, smp == 0xFFFFu)) {
#pragma unroll
          for (int r = 0; r < kTokBoxRows; ++r)
            asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(wbase + static_cast<uint32_t>(bin[r]) * 64u), "r"(inc1));
        } else {
#pragma unroll
          for (int r = 0; r < kTokBoxRows; ++r)
            if ((smp >> r) & 1u)
              asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(wbase + static_cast<uint32_t>(bin[r]) * 64u), "r"(inc1));
        }
      } else if (CL_TOK_QUAD && __all_sync(0xffffffffu, smp == 0xFFFFu)) {
        // full box, every row sampled (stride 1): constant increments, four samples per
        // read-modify-write round (all four loads, then the stores in sample order, each
        // carrying the earlier samples of its bin: the last store to a bin holds the
        // bin's whole multiplicity) -- the per-lane RMW chain is 4 rounds per box, not 8
#pragma unroll
        for (int g = 0; g < kTokBoxRows / 4; ++g) {
          const int b0 = bin[4 * g], b1 = bin[4 * g + 1], b2 = bin[4 * g + 2], b3 = bin[4 * g + 3];
          const uint32_t a0 = cbase + static_cast<uint32_t>(b0) * 64u;
          const uint32_t a1 = cbase + static_cast<uint32_t>(b1) * 64u;
          const uint32_t a2 = cbase + static_cast<uint32_t>(b2) * 64u;
          const uint32_t a3 = cbase + static_cast<uint32_t>(b3) * 64u;
          uint32_t v0, v1, v2, v3;
          asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v0) : "r"(a0) : "memory");
          asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v1) : "r"(a1) : "memory");
          asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v2) : "r"(a2) : "memory");
          asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v3) : "r"(a3) : "memory");
          v0 += 1u;
          v1 += 1u + (b0 == b1);
          v2 += 1u + (b0 == b2) + (b1 == b2);
          v3 += 1u + (b0 == b3) + (b1 == b3) + (b2 == b3);
          asm volatile("st.shared.u16 [%0], %1;" ::"r"(a0), "h"(static_cast<uint16_t>(v0)) : "memory");
          asm volatile("st.shared.u16 [%0], %1;" ::"r"(a1), "h"(static_cast<uint16_t>(v1)) : "memory");
          asm volatile("st.shared.u16 [%0], %1;" ::"r"(a2), "h"(static_cast<uint16_t>(v2)) : "memory");
          asm volatile("st.shared.u16 [%0], %1;" ::"r"(a3), "h"(static_cast<uint16_t>(v3)) : "memory");
        }
      } else if (__all_sync(0xffffffffu, smp == 0xFFFFu)) {
        // full box, every row sampled (stride 1): constant increments
#pragma unroll
        for (int g = 0; g < kTokBoxRows / 2; ++g) {
          const int b0 = bin[2 * g], b1 = bin[2 * g + 1];
          const uint32_t a0 = cbase + static_cast<uint32_t>(b0) * 64u;
          const uint32_t a1 = cbase + static_cast<uint32_t>(b1) * 64u;
          uint32_t v0, v1;
          asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v0) : "r"(a0) : "memory");
          asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v1) : "r"(a1) : "memory");
          v1 += b0 == b1 ? 2u : 1u;
          asm volatile("st.shared.u16 [%0], %1;" ::"r"(a0), "h"(static_cast<uint16_t>(v0 + 1u)) : "memory");
          asm volatile("st.shared.u16 [%0], %1;" ::"r"(a1), "h"(static_cast<uint16_t>(v1)) : "memory");
        }
      } else
#pragma unroll
      for (int g = 0; g < kTokBoxRows / 2; ++g) {
        const uint32_t i0 = (smp >> (2 * g)) & 1u;
        const uint32_t i1 = (smp >> (2 * g + 1)) & 1u;
        const int b0 = bin[2 * g], b1 = bin[2 * g + 1];
        const uint32_t a0 = cbase + static_cast<uint32_t>(b0) * 64u;
        const uint32_t a1 = cbase + static_cast<uint32_t>(b1) * 64u;
        uint32_t v0, v1;
        asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v0) : "r"(a0) : "memory");
        asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v1) : "r"(a1) : "memory");
        v0 += i0;
        v1 += i1 + (b0 == b1 ? i0 : 0u);
        asm volatile("st.shared.u16 [%0], %1;" ::"r"(a0), "h"(static_cast<uint16_t>(v0)) : "memory");
        asm volatile("st.shared.u16 [%0], %1;" ::"r"(a1), "h"(static_cast<uint16_t>(v1)) : "memory");
      }
      since += kTokBoxRows;
      if (since > kTokHMaxPerFlush - kTokBoxRows || c + kTokBoxRows >= c1) {
        // this warp's 32 positions into counts [L][K], counters cleared (warp-local)
        __syncwarp();
        if (t_ok) {
          // four counters in flight per step (the loads no longer wait on each other)
          int b = 0;
          for (; b + 4 <= k; b += 4) {
            uint32_t v[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) v[q] = tcnt[(warp * 256 + b + q) * 32 + lane];
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (v[q]) atomicAdd(counts + t * k + b + q, v[q]);
          }
          for (; b < k; ++b) {
            const uint32_t v = tcnt[(warp * 256 + b) * 32 + lane];
            if (v) atomicAdd(counts + t * k + b, v);
          }
        }
        __syncwarp();
        uint4* c4 = reinterpret_cast<uint4*>(tcnt + warp * 256 * 32);
        for (int i = lane; i < 256 * 32 * 2 / 16; i += 32) c4[i] = make_uint4(0, 0, 0, 0);
        __syncwarp();
        since = 0;
      }
    }
  }
}

// estimate_entropy per position (entropy.hpp:149-164): warp w of the block -> position
// blockIdx.x * 8 + w; masses = count * (1/n), terms subtracted in bin order.
__global__ void __launch_bounds__(kThreads) token_entropy_kernel(const unsigned int* counts,
                                                                 uint64_t length, int k,
                                                                 uint64_t n_per_pos, double eps,
                                                                 double* raw_t) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint64_t t = static_cast<uint64_t>(blockIdx.x) * (kThreads / 32) + warp;
  if (t >= length) return;
  const double inv_n = __ddiv_rn(1.0, static_cast<double>(n_per_pos));
  const unsigned int* hw = counts + t * k;
  double raw = 0.0;
  for (int base = 0; base < k; base += 32) {
    const int b = base + lane;
    const unsigned int cnt = b < k ? hw[b] : 0u;
    double term = 0.0;
    if (cnt) {
      const double pm = __dmul_rn(static_cast<double>(cnt), inv_n);
      term = __dmul_rn(pm, log(__dadd_rn(pm, eps)));
    }
    const int m = min(32, k - base);
    for (int i = 0; i < m; ++i) {
      const double ti = __shfl_sync(0xffffffffu, term, i);
      const unsigned ci = __shfl_sync(0xffffffffu, cnt, i);
      if (ci) raw = __dsub_rn(raw, ti);
    }
  }
  if (lane == 0) raw_t[t] = raw;
}

// raw_nats = (sum_t raw_t in position order) / L; normalized = raw_nats / log K.  The sum
// must be the reference's left-to-right fp64 chain, so one thread adds; the block stages
// raw_t through shared memory so those adds wait on shared-memory loads, not DRAM.
constexpr int kFinThreads = 1024;
constexpr int kFinChunk = 4096;  // doubles per staged chunk (32 KB)

__global__ void __launch_bounds__(kFinThreads) token_finalize_kernel(
    const double* __restrict__ raw_t, uint64_t length, uint64_t samples_per_pos, int k,
    const double* flag, double* out) {
  __shared__ double buf[kFinChunk];
  double sum = 0.0;
  for (uint64_t base = 0; base < length; base += kFinChunk) {
    const int m = static_cast<int>(umin64(kFinChunk, length - base));
    __syncthreads();
    for (int i = threadIdx.x; i < m; i += kFinThreads) buf[i] = raw_t[base + i];
    __syncthreads();
    if (threadIdx.x == 0) {
      int i = 0;
      for (; i + 8 <= m; i += 8) {
        double v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = buf[i + j];
#pragma unroll
        for (int j = 0; j < 8; ++j) sum = __dadd_rn(sum, v[j]);
      }
      for (; i < m; ++i) sum = __dadd_rn(sum, buf[i]);
    }
  }
  if (threadIdx.x != 0) return;
  const double raw = __ddiv_rn(sum, static_cast<double>(length));
  out[0] = raw;
  out[1] = __ddiv_rn(raw, log(static_cast<double>(k)));
  out[2] = static_cast<double>(samples_per_pos * length);
  out[3] = flag ? *flag : 0.0;
}

__global__ void token_range_init_kernel(double* trange, uint64_t length) {
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < 2 * length;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    trange[i] = -INFINITY;
}

__global__ void entropy_masses_kernel(const double* masses, int k, double eps, double* out) {
  __shared__ double terms[kThreads];
  double raw = 0.0;
  for (int base = 0; base < k; base += kThreads) {
    const int b = base + threadIdx.x;
    double t = 0.0;
    if (b < k) {
      const double pm = masses[b];
      if (pm > 0.0) t = __dmul_rn(pm, log(__dadd_rn(pm, eps)));
    }
    terms[threadIdx.x] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
      const int m = min(kThreads, k - base);
      for (int i = 0; i < m; ++i) {
        const double pm = masses[base + i];
        if (pm > 0.0) raw = __dsub_rn(raw, terms[i]);
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[0] = raw;
    out[1] = __ddiv_rn(raw, log(static_cast<double>(k)));
  }
}

int grid_for(uint64_t work_items, int per_block, int num_sms, int blocks_per_sm) {
  const uint64_t need = (work_items + per_block - 1) / per_block;
  const uint64_t cap = static_cast<uint64_t>(num_sms) * blocks_per_sm;
  return static_cast<int>(need < 1 ? 1 : (need < cap ? need : cap));
}

int stride_mode(uint64_t stride) {
  if (stride == 1) return 0;
  if ((stride & (stride - 1)) == 0) return 1;
  return 2;
}

}  // namespace

cudaError_t launch_range_init(double* d_range, cudaStream_t s) {
  range_init_kernel<<<1, 1, 0, s>>>(d_range);
  return cudaGetLastError();
}

cudaError_t launch_prefill_init(double* d_range, uint64_t* d_counts, int k, cudaStream_t s) {
  prefill_init_kernel<<<1, 256, 0, s>>>(d_range, reinterpret_cast<unsigned long long*>(d_counts),
                                        k);
  return cudaGetLastError();
}

cudaError_t launch_minmax_f32(const float* v, uint64_t n, uint64_t g0, uint64_t stride,
                              double* d_range, int num_sms, cudaStream_t s, int* launches) {
  if (n == 0) return cudaSuccess;
  static const int per_sm = [] {
    const char* e = getenv("CL_MM_CTAS_PER_SM");
    return e ? atoi(e) : CL_MM_CTAS_PER_SM;
  }();
  const int grid = grid_for(n / 4 + 1, kThreads * 4, num_sms, per_sm);
  switch (stride_mode(stride)) {
    case 0: minmax_f32_kernel<0><<<grid, kThreads, 0, s>>>(v, n, g0, stride, d_range); break;
    case 1: minmax_f32_kernel<1><<<grid, kThreads, 0, s>>>(v, n, g0, stride, d_range); break;
    default: minmax_f32_kernel<2><<<grid, kThreads, 0, s>>>(v, n, g0, stride, d_range); break;
  }
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_minmax_gather_f32(const float* v, uint64_t n, uint64_t g0, uint64_t stride,
                                     double* d_range, float* d_samples, int num_sms,
                                     cudaStream_t s, int* launches) {
  if (n == 0) return cudaSuccess;
  const int grid = grid_for(n / 4 + 1, kThreads * 4, num_sms, CL_MM_CTAS_PER_SM);
  const uint64_t first = (g0 + stride - 1) / stride;
  switch (stride_mode(stride)) {
    case 0:
      minmax_f32_kernel<0, true><<<grid, kThreads, 0, s>>>(v, n, g0, stride, d_range, d_samples, first);
      break;
    case 1:
      minmax_f32_kernel<1, true><<<grid, kThreads, 0, s>>>(v, n, g0, stride, d_range, d_samples, first);
      break;
    default:
      minmax_f32_kernel<2, true><<<grid, kThreads, 0, s>>>(v, n, g0, stride, d_range, d_samples, first);
      break;
  }
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_minmax_f64(const double* v, uint64_t n, uint64_t g0, uint64_t stride,
                              double* d_range, int num_sms, cudaStream_t s, int* launches) {
  if (n == 0) return cudaSuccess;
  const int grid = grid_for(n, kThreads * 4, num_sms, 4);
  switch (stride_mode(stride)) {
    case 0: minmax_f64_kernel<0><<<grid, kThreads, 0, s>>>(v, n, g0, stride, d_range); break;
    case 1: minmax_f64_kernel<1><<<grid, kThreads, 0, s>>>(v, n, g0, stride, d_range); break;
    default: minmax_f64_kernel<2><<<grid, kThreads, 0, s>>>(v, n, g0, stride, d_range); break;
  }
  ++*launches;
  return cudaGetLastError();
}

DecideArgs make_decide_args(const uint64_t* d_counts, const double* d_range,
                            const cl_hist_spec& spec, uint64_t n_samples,
                            const cl_rule_spec& rule, uint64_t seq_len,
                            const cl_features* features) {
  DecideArgs a{};
  a.counts = reinterpret_cast<const unsigned long long*>(d_counts);
  a.range = d_range;
  a.k = spec.bin_count;
  a.epsilon = spec.epsilon;
  a.range_mode = spec.range_mode;
  a.fixed_lo = spec.fixed_lo;
  a.fixed_hi = spec.fixed_hi;
  a.n_samples = n_samples;
  a.rule = rule;
  a.seq_len = seq_len;
  a.features_mode = features ? 1 : 0;
  if (features) a.f = *features;
  return a;
}

// The histogram; with fuse != null and the register-fed kernel applicable, that
// kernel's last CTA also writes the decision (*fused = true; no launch_decide needed).
cudaError_t launch_histogram_f32(const float* v, uint64_t n, uint64_t g0,
                                 const cl_hist_spec& spec, const double* d_range,
                                 uint64_t* d_counts, int num_sms, cudaStream_t s,
                                 int* launches, const HistFuse* fuse, bool* fused) {
  if (fused) *fused = false;
  if (n == 0) return cudaSuccess;
  const uint64_t stride = spec.sample_stride;
  const int k = spec.bin_count;
  auto* counts = reinterpret_cast<unsigned long long*>(d_counts);
  const int mode = stride_mode(stride);
  if (k <= 256 && n >= 4096) {
    const uint64_t chunks = n / kChunkFloats + 1;
    const uint64_t ctas = static_cast<uint64_t>(num_sms) * kHistCtasPerSm;
    const int grid = static_cast<int>(chunks < ctas ? chunks : ctas);
    const bool fixed = spec.range_mode == CL_RANGE_FIXED;
    auto launch = [&](auto kern) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(kHistSmem));
      kern<<<grid, kHistThreads, kHistSmem, s>>>(v, n, g0, stride, spec.range_mode,
                                                 spec.fixed_lo, spec.fixed_hi, k, d_range,
                                                 counts);
    };
    if (CL_HIST_REG && !fixed && mode == 0 && CL_HIST_U8) {
      const bool fz = fuse != nullptr && g0 == 0;
      const uint64_t wchunks = n / kRegChunk + 1;
      // small inputs: give every warp at least a few chunks -- each warp pays a full 8 KB
      // counter flush (and each CTA 256 global atomics) however little it bins
      static const uint64_t min_chunks = [] {
        const char* e = getenv("CL_HIST_MIN_CHUNKS");
        return e ? static_cast<uint64_t>(atoi(e)) : uint64_t(CL_HIST_MIN_CHUNKS);
      }();
      const uint64_t per_cta = uint64_t(kRegWarps) * (min_chunks < 1 ? 1 : min_chunks);
      const uint64_t gmax = (wchunks + per_cta - 1) / per_cta;
      const int rgrid = static_cast<int>(gmax < static_cast<uint64_t>(num_sms) ? gmax : num_sms);
      DecideArgs da{};
      cl_decision* d_out = nullptr;
      if (fz) {
        da = make_decide_args(d_counts, d_range, spec, fuse->n_samples, *fuse->rule,
                              fuse->seq_len, nullptr);
        d_out = fuse->d_out;
      }
      const bool pow2k = (k & (k - 1)) == 0;
      auto kern = fz ? (pow2k ? hist_f32_reg_kernel<true, true> : hist_f32_reg_kernel<true, false>)
                     : (pow2k ? hist_f32_reg_kernel<false, true> : hist_f32_reg_kernel<false, false>);
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(kRegSmem));
      kern<<<rgrid, kRegWarps * 32, kRegSmem, s>>>(v, n, spec.range_mode, spec.fixed_lo,
                                                   spec.fixed_hi, k, d_range, counts, da, d_out,
                                                   fz ? fuse->ticket : nullptr);
      if (fused) *fused = fz;
    } else if (fixed) {
      if (mode == 0) launch(hist_f32_lane_kernel<0, true>);
      else if (mode == 1) launch(hist_f32_lane_kernel<1, true>);
      else launch(hist_f32_lane_kernel<2, true>);
    } else {
      if (mode == 0) launch(hist_f32_lane_kernel<0, false>);
      else if (mode == 1) launch(hist_f32_lane_kernel<1, false>);
      else launch(hist_f32_lane_kernel<2, false>);
    }
  } else {
    const int use_smem = k <= 16384 ? 1 : 0;
    const size_t smem = use_smem ? static_cast<size_t>(k) * 4 : 0;
    const int grid = grid_for(n, kThreads * 8, num_sms, 4);
    if (smem > 48 * 1024) {
      cudaFuncSetAttribute(hist_atomic_kernel<float, 0>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
      cudaFuncSetAttribute(hist_atomic_kernel<float, 1>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
      cudaFuncSetAttribute(hist_atomic_kernel<float, 2>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    }
    if (mode == 0)
      hist_atomic_kernel<float, 0><<<grid, kThreads, smem, s>>>(
          v, n, g0, stride, spec.range_mode, spec.fixed_lo, spec.fixed_hi, k, d_range, counts,
          use_smem);
    else if (mode == 1)
      hist_atomic_kernel<float, 1><<<grid, kThreads, smem, s>>>(
          v, n, g0, stride, spec.range_mode, spec.fixed_lo, spec.fixed_hi, k, d_range, counts,
          use_smem);
    else
      hist_atomic_kernel<float, 2><<<grid, kThreads, smem, s>>>(
          v, n, g0, stride, spec.range_mode, spec.fixed_lo, spec.fixed_hi, k, d_range, counts,
          use_smem);
  }
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_histogram_f64(const double* v, uint64_t n, uint64_t g0,
                                 const cl_hist_spec& spec, const double* d_range,
                                 uint64_t* d_counts, int num_sms, cudaStream_t s,
                                 int* launches) {
  if (n == 0) return cudaSuccess;
  const uint64_t stride = spec.sample_stride;
  const int k = spec.bin_count;
  auto* counts = reinterpret_cast<unsigned long long*>(d_counts);
  const int use_smem = k <= 16384 ? 1 : 0;
  const size_t smem = use_smem ? static_cast<size_t>(k) * 4 : 0;
  const int grid = grid_for(n, kThreads * 8, num_sms, 4);
  if (smem > 48 * 1024) {
    cudaFuncSetAttribute(hist_atomic_kernel<double, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         65536);
    cudaFuncSetAttribute(hist_atomic_kernel<double, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         65536);
    cudaFuncSetAttribute(hist_atomic_kernel<double, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         65536);
  }
  const int mode = stride_mode(stride);
  if (mode == 0)
    hist_atomic_kernel<double, 0><<<grid, kThreads, smem, s>>>(
        v, n, g0, stride, spec.range_mode, spec.fixed_lo, spec.fixed_hi, k, d_range, counts,
        use_smem);
  else if (mode == 1)
    hist_atomic_kernel<double, 1><<<grid, kThreads, smem, s>>>(
        v, n, g0, stride, spec.range_mode, spec.fixed_lo, spec.fixed_hi, k, d_range, counts,
        use_smem);
  else
    hist_atomic_kernel<double, 2><<<grid, kThreads, smem, s>>>(
        v, n, g0, stride, spec.range_mode, spec.fixed_lo, spec.fixed_hi, k, d_range, counts,
        use_smem);
  ++*launches;
  return cudaGetLastError();
}

// The conv + Fixed-range histogram epilogue, when it applies (returns false otherwise;
// the caller then runs cl_conv1d_f32 + the histogram).
bool launch_conv_hist_fixed(const float* x, const float* w, const float* bias, float* u,
                            uint64_t batch, uint64_t dim, uint64_t L, int width, int silu,
                            const cl_hist_spec& spec, uint64_t* d_counts, double* d_range,
                            int num_sms, cudaStream_t s, cudaError_t* err) {
  *err = cudaSuccess;
  if (!CL_HIST_U8 || spec.range_mode != CL_RANGE_FIXED || spec.sample_stride != 1 ||
      spec.bin_count > kLaneBins || L % 128 != 0 || width < 1 || width > 4 ||
      (reinterpret_cast<uintptr_t>(x) & 15u) || (reinterpret_cast<uintptr_t>(u) & 15u))
    return false;
  const uint64_t rows = batch * dim;
  const uint64_t units = rows * ((L / 4) / (32 * kCHWQ) + ((L / 4 / 32) % kCHWQ ? 1 : 0));
  const uint64_t want = (units + kCHWarps - 1) / kCHWarps;
  const uint64_t cap = static_cast<uint64_t>(num_sms) * 3;  // 3 x 65 KB per SM
  const int grid = static_cast<int>(want < cap ? (want < 1 ? 1 : want) : cap);
  auto* counts = reinterpret_cast<unsigned long long*>(d_counts);
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(kCHSmem));
    kern<<<grid, kCHWarps * 32, kCHSmem, s>>>(x, w, bias, u, rows, dim, L, silu, spec.fixed_lo,
                                              spec.fixed_hi, spec.bin_count, counts, d_range);
  };
  switch (width) {
    case 1: go(conv_hist_fixed_kernel<1>); break;
    case 2: go(conv_hist_fixed_kernel<2>); break;
    case 3: go(conv_hist_fixed_kernel<3>); break;
    default: go(conv_hist_fixed_kernel<4>); break;
  }
  *err = cudaGetLastError();
  return true;
}

// The lean (co-schedulable) min/max and histogram + decision, one CTA per SM; returns
// false when the configuration is not the one they serve (the caller falls back).
bool launch_entropy_lean(const float* v, uint64_t n, const cl_hist_spec& spec,
                         const cl_rule_spec& rule, uint64_t seq_len, double* d_range,
                         uint64_t* d_counts, cl_decision* d_out, unsigned long long* ticket,
                         int num_sms, cudaStream_t s, cudaError_t* err) {
  *err = cudaSuccess;
  if (!CL_HIST_U8 || spec.range_mode != CL_RANGE_DYNAMIC || spec.sample_stride != 1 ||
      spec.bin_count > kLaneBins || n < uint64_t(kLeanChunk) * 8)
    return false;
  const int grid = num_sms;
  cudaFuncSetAttribute(minmax_lean_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(kLeanMmSmem));
  cudaFuncSetAttribute(hist_lean_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(kLeanHistSmem));
  cudaFuncSetAttribute(minmax_lean_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                       cudaSharedmemCarveoutMaxShared);
  cudaFuncSetAttribute(hist_lean_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                       cudaSharedmemCarveoutMaxShared);
  minmax_lean_kernel<<<grid, kLeanWarps * 32, kLeanMmSmem, s>>>(v, n, d_range);
  if ((*err = cudaGetLastError()) != cudaSuccess) return true;
  const DecideArgs da = make_decide_args(d_counts, d_range, spec, n, rule, seq_len, nullptr);
  hist_lean_kernel<<<grid, kLeanWarps * 32, kLeanHistSmem, s>>>(
      v, n, spec.bin_count, d_range, reinterpret_cast<unsigned long long*>(d_counts), da, d_out,
      ticket);
  *err = cudaGetLastError();
  return true;
}

cudaError_t launch_decide(const uint64_t* d_counts, const double* d_range,
                          const cl_hist_spec& spec, uint64_t n_samples, const cl_rule_spec& rule,
                          uint64_t seq_len, const cl_features* features, cl_decision* d_out,
                          cudaStream_t s) {
  const DecideArgs a =
      make_decide_args(d_counts, d_range, spec, n_samples, rule, seq_len, features);
  decide_kernel<<<1, kThreads, 0, s>>>(a, d_out);
  return cudaGetLastError();
}

cudaError_t launch_decide_token(const double* d_token, const cl_hist_spec& spec,
                                const cl_rule_spec& rule, uint64_t seq_len, cl_decision* d_out,
                                cudaStream_t s) {
  DecideArgs a{};
  a.k = spec.bin_count;
  a.epsilon = spec.epsilon;
  a.range_mode = spec.range_mode;
  a.rule = rule;
  a.seq_len = seq_len;
  a.features_mode = 2;
  a.token = d_token;
  decide_kernel<<<1, kThreads, 0, s>>>(a, d_out);
  return cudaGetLastError();
}

cudaError_t launch_entropy_from_masses(const double* d_masses, int k, double eps, double* d_out,
                                       cudaStream_t s) {
  entropy_masses_kernel<<<1, kThreads, 0, s>>>(d_masses, k, eps, d_out);
  return cudaGetLastError();
}

namespace {
template <typename T>
bool tok_vec_ok(const T* v, uint64_t length) {
  return length % TokVec<T>::kV == 0 && (reinterpret_cast<uintptr_t>(v) & 15u) == 0;
}

template <typename T>
dim3 tok_grid(uint64_t channels, uint64_t length, bool vec, int num_sms) {
  const uint64_t tile = vec ? 8 * TokVec<T>::kV : 8;
  const uint64_t tiles = (length + tile - 1) / tile;
  // channel shares so the grid covers ~4 blocks per SM, each share >= 64 channels
  uint64_t splits = (static_cast<uint64_t>(num_sms) * 4 + tiles - 1) / tiles;
  const uint64_t max_splits = (channels + 63) / 64;
  if (splits > max_splits) splits = max_splits;
  if (splits < 1) splits = 1;
  if (splits > 65535) splits = 65535;
  return dim3(static_cast<unsigned>(tiles), static_cast<unsigned>(splits));
}
}  // namespace

cudaError_t launch_token_range_init(double* d_trange, double* d_flag, uint64_t length,
                                    cudaStream_t s) {
  token_range_init_kernel<<<64, kThreads, 0, s>>>(d_trange, length);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return cudaMemsetAsync(d_flag, 0, sizeof(double), s);
}

// (position tiles, channel splits) for the lane kernels: enough items for ~4 per resident
// block, each split >= 256 channels
void tok_lane_items(uint64_t channels, uint64_t length, uint64_t tile, int resident,
                    uint64_t* tiles, uint64_t* splits) {
  *tiles = (length + tile - 1) / tile;
  uint64_t sp = (static_cast<uint64_t>(resident) * 4 + *tiles - 1) / *tiles;
  const uint64_t max_sp = (channels + 255) / 256;
  if (sp > max_sp) sp = max_sp;
  *splits = sp < 1 ? 1 : sp;
}

bool tok_lane_ok(const float* v, uint64_t length, int k) {
  return k <= 256 && length % 4 == 0 && (reinterpret_cast<uintptr_t>(v) & 15u) == 0;
}
template <typename T>
bool tok_lane_ok(const T*, uint64_t, int) {
  return false;
}

template <typename T>
cudaError_t launch_token_minmax(const T* v, uint64_t channels, uint64_t length, uint64_t offset,
                                uint64_t stride, double* d_trange, double* d_flag, int num_sms,
                                cudaStream_t s) {
  if (tok_lane_ok(v, length, 0)) {
    const TokArgs a{channels, length, offset, stride, 0, 1};
    uint64_t tiles, splits;
    const int resident = num_sms * 2;  // 2 blocks of 8 warps per SM
    tok_lane_items(channels, length, 128 * kTokMmCols, resident, &tiles, &splits);
    const uint64_t items = tiles * splits;
    const unsigned grid = static_cast<unsigned>(items < static_cast<uint64_t>(resident) ? items : resident);
    token_minmax_lane_kernel<<<grid, kTokMmWarps * 32, 0, s>>>(
        reinterpret_cast<const float*>(v), a, tiles, splits, d_trange, d_flag);
    return cudaGetLastError();
  }
  const bool vec = tok_vec_ok(v, length);
  const TokArgs a{channels, length, offset, stride, 0, vec ? 1 : 0};
  const dim3 grid = tok_grid<T>(channels, length, vec, num_sms);
  if (vec)
    token_minmax_kernel<T, 1><<<grid, kThreads, 0, s>>>(v, a, d_trange, d_flag);
  else
    token_minmax_kernel<T, 0><<<grid, kThreads, 0, s>>>(v, a, d_trange, d_flag);
  return cudaGetLastError();
}

template <typename T, int VEC, bool FIXED>
cudaError_t launch_token_hist_v(const T* v, const TokArgs& a, const double* d_trange,
                                const cl_hist_spec& spec, unsigned int* d_counts, dim3 grid,
                                cudaStream_t s) {
  constexpr int kTile = 8 * (VEC ? TokVec<T>::kV : 1);
  const size_t smem = static_cast<size_t>(kTile) * a.k * sizeof(unsigned int);
  if (smem <= kTokMaxSmemHist) {
    auto kern = token_hist_kernel<T, VEC, FIXED, true>;
    if (smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(smem));
      if (e != cudaSuccess) return e;
    }
    kern<<<grid, kThreads, smem, s>>>(v, a, d_trange, spec.fixed_lo, spec.fixed_hi, d_counts);
  } else {
    token_hist_kernel<T, VEC, FIXED, false><<<grid, kThreads, 0, s>>>(
        v, a, d_trange, spec.fixed_lo, spec.fixed_hi, d_counts);
  }
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_token_hist(const T* v, uint64_t channels, uint64_t length, uint64_t offset,
                              const cl_hist_spec& spec, const double* d_trange,
                              unsigned int* d_counts, int num_sms, cudaStream_t s) {
  if (CL_TOK_TMA && tok_lane_ok(v, length, spec.bin_count) && length <= (1ull << 31) &&
      channels <= (1ull << 31) && get_encode()) {
    const TokArgs a{channels, length, offset, spec.sample_stride, spec.bin_count, 1};
    CUtensorMap map;
    if (!make_map(&map, reinterpret_cast<const float*>(v), length, channels, 1, 128, kTokBoxRows,
                  0))
      return cudaErrorInvalidValue;
    const int resident = num_sms * 2;  // 2 blocks (64 KB counters + 40 KB ring) per SM
    // channel splits: every item ends with a flush of its 128 x K counters (LDS + a global
    // atomic per nonzero bin), and the items run in rounds of `resident` blocks, so pick the
    // split count minimising rounds x (channels per item + flush cost in channel
    // equivalents); at least a few boxes per item
    const uint64_t tiles = (length + 127) / 128;
    static const uint64_t flush_cost = [] {
      const char* e = getenv("CL_TOK_FLUSH_COST");
      return e ? static_cast<uint64_t>(atoi(e)) : uint64_t(256);
    }();
    const uint64_t max_sp = (channels + 4 * kTokBoxRows - 1) / (4 * kTokBoxRows);
    const uint64_t hi_sp = (8 * static_cast<uint64_t>(resident) + tiles - 1) / tiles;
    uint64_t splits = 1, best = ~0ull;
    for (uint64_t sp = 1; sp <= hi_sp && sp <= (max_sp < 1 ? 1 : max_sp); ++sp) {
      const uint64_t rounds = (tiles * sp + resident - 1) / resident;
      const uint64_t cost = rounds * ((channels + sp - 1) / sp + flush_cost);
      if (cost < best) {
        best = cost;
        splits = sp;
      }
    }
    const uint64_t items = tiles * splits;
    const unsigned grid = static_cast<unsigned>(items < static_cast<uint64_t>(resident) ? items : resident);
    const bool fixed = spec.range_mode == CL_RANGE_FIXED;
    auto kern = fixed ? token_hist_tma_kernel<true> : token_hist_tma_kernel<false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kTokTSmem));
    if (e != cudaSuccess) return e;
    kern<<<grid, (kTokTWarps + 1) * 32, kTokTSmem, s>>>(map, a, tiles, splits, d_trange,
                                                        spec.fixed_lo, spec.fixed_hi, d_counts);
    return cudaGetLastError();
  }
  if (tok_lane_ok(v, length, spec.bin_count)) {
    const TokArgs a{channels, length, offset, spec.sample_stride, spec.bin_count, 1};
    uint64_t tiles, splits;
    const int resident = num_sms * 3;  // 3 blocks of 4 warps (64 KB of counters) per SM
    tok_lane_items(channels, length, 32, resident, &tiles, &splits);
    const uint64_t items = tiles * splits;
    const unsigned grid = static_cast<unsigned>(items < static_cast<uint64_t>(resident) ? items : resident);
    const size_t smem = size_t(kTokHWarps) * 256 * 32 * 2;
    const bool fixed = spec.range_mode == CL_RANGE_FIXED;
    auto kern = fixed ? token_hist_lane_kernel<true> : token_hist_lane_kernel<false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    kern<<<grid, kTokHWarps * 32, smem, s>>>(reinterpret_cast<const float*>(v), a, tiles, splits,
                                            d_trange, spec.fixed_lo, spec.fixed_hi, d_counts);
    return cudaGetLastError();
  }
  const bool vec = tok_vec_ok(v, length);
  const TokArgs a{channels, length, offset, spec.sample_stride, spec.bin_count, vec ? 1 : 0};
  const dim3 grid = tok_grid<T>(channels, length, vec, num_sms);
  const bool fixed = spec.range_mode == CL_RANGE_FIXED;
  if (vec)
    return fixed ? launch_token_hist_v<T, 1, true>(v, a, d_trange, spec, d_counts, grid, s)
                 : launch_token_hist_v<T, 1, false>(v, a, d_trange, spec, d_counts, grid, s);
  return fixed ? launch_token_hist_v<T, 0, true>(v, a, d_trange, spec, d_counts, grid, s)
               : launch_token_hist_v<T, 0, false>(v, a, d_trange, spec, d_counts, grid, s);
}

cudaError_t launch_token_entropy(const unsigned int* d_counts, uint64_t length,
                                 uint64_t n_per_pos, const cl_hist_spec& spec,
                                 const double* d_flag, double* d_raw_t, double* d_out,
                                 cudaStream_t s) {
  const uint64_t blocks = (length + kThreads / 32 - 1) / (kThreads / 32);
  token_entropy_kernel<<<static_cast<unsigned>(blocks), kThreads, 0, s>>>(
      d_counts, length, spec.bin_count, n_per_pos, spec.epsilon, d_raw_t);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  token_finalize_kernel<<<1, kFinThreads, 0, s>>>(d_raw_t, length, n_per_pos, spec.bin_count,
                                                  d_flag, d_out);
  return cudaGetLastError();
}

template cudaError_t launch_token_minmax<float>(const float*, uint64_t, uint64_t, uint64_t,
                                                uint64_t, double*, double*, int, cudaStream_t);
template cudaError_t launch_token_minmax<double>(const double*, uint64_t, uint64_t, uint64_t,
                                                 uint64_t, double*, double*, int, cudaStream_t);
template cudaError_t launch_token_hist<float>(const float*, uint64_t, uint64_t, uint64_t,
                                              const cl_hist_spec&, const double*, unsigned int*,
                                              int, cudaStream_t);
template cudaError_t launch_token_hist<double>(const double*, uint64_t, uint64_t, uint64_t,
                                               const cl_hist_spec&, const double*,
                                               unsigned int*, int, cudaStream_t);

}  // namespace cl
