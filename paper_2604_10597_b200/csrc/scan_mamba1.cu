// scan_mamba1.cu -- fused Mamba-1 selective scan for sm_100a (fp32).
//
// Semantics (mamba_ssm selective_scan_fn, the paper's kernel),
// recurrence core identical to chunklab::scan_window (scan.hpp:77-100) under the
// mapping a = exp(delta'*A), x = delta'*u, b/c = B/C (SURVEY.md finding 1):
//   delta' = softplus(delta + bias)            (identity above 20, mamba_ssm)
//   h_s    = exp(delta'*A[c,s]) * h_s + B[b,s,t] * (delta'*u)     s = 0..N-1
//   y      = (sum_s C[b,s,t]*h_s + D[c]*u) * z*sigmoid(z)
//
// Kernels:
//   * rowpair_ws_kernel (the hot path, N = 16): warp-specialised.  Consumer warps own
//     16-row tiles (two lanes per (b, c) row, 8 states each in FFMA2 register pairs);
//     producer warps feed each consumer a 2-stage TMA ring of 16-timestep boxes
//     (u / delta / z with 64B swizzle, one interleaved [B^T | C^T] box).  y is stored
//     from registers.  Work items are (row tile, L-segment) pairs with segment length
//     = the chunk chosen by the device rule (read from device memory, rounded up to
//     whole boxes), dispatched segment-major through an atomic ticket; the state carry
//     between consecutive segments of a tile is a chained scan (flag + release /
//     acquire), so chunking never changes a single floating-point operation: outputs
//     are bit-identical for every chunk size.
//   * rowseq_tma_kernel: one lane per row (32-row tiles), each warp feeding its own
//     TMA ring and TMA-storing y; kept as a selectable variant (CL_SCAN_CFG=1..3).
//   * generic_kernel: any N <= 64, any alignment; one thread per row, direct loads.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <cstdlib>
#include <mutex>

#include "cl_internal.h"

namespace cl {
namespace {

constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// ---- canonical elementwise math ----
// Every Mamba-1 path (generic scan, TMA scans, decode) evaluates softplus, SiLU and, for
// N = 16, C.h with exactly these operation sequences, so the paths agree bit for bit
// and a prefill followed by decode steps equals a longer prefill bit for bit (the
// paper's passive-vs-routed claim is bitwise output equality).  The
// FFMA2 versions further down (softplus2 / silu2 / the lane-pair C.h) are these
// functions applied per lane of a register pair.

// softplus(x) = max(x,0) + log1p(exp(-|x|)): one MUFU.EX2 and a degree-9 minimax
// polynomial for log1p on [0,1] (max rel err 2e-7; equals x to fp32 above 20).
__device__ __forceinline__ float softplus_canon(float a) {
  const float e = ex2_approx(-fabsf(a) * kLog2e);
  float q = 0.005253826278033571f;
  q = fmaf(q, e, -0.02959069552080005f);
  q = fmaf(q, e, 0.07836660226277938f);
  q = fmaf(q, e, -0.13675328086246433f);
  q = fmaf(q, e, 0.19111774195698683f);
  q = fmaf(q, e, -0.24844483411506615f);
  q = fmaf(q, e, 0.33319289806287417f);
  q = fmaf(q, e, -0.49999502673812024f);
  q = fmaf(q, e, 0.9999999706625772f);
  return fmaf(q, e, fmaxf(a, 0.f));
}

// z * sigmoid(z): one MUFU.EX2, reciprocal by 3 Newton steps from the bit-trick seed.
__device__ __forceinline__ float silu_canon(float z) {
  const float e = ex2_approx(fmaxf(z, -80.f) * -kLog2e);
  const float d = e + 1.f;
  float r = __int_as_float(0x7EF311C7 - __float_as_int(d));
  const float nd = d * -1.f;
#pragma unroll
  for (int it = 0; it < 3; ++it) {
    const float en = fmaf(nd, r, 1.f);
    r = fmaf(r, en, r);
  }
  return z * r;
}

// y = sum_s c[s] h[s] for N = 16 in the lane-pair kernel's order: lane half hf holds
// states 8hf..8hf+7 and accumulates, as FFMA2 chains started from +0,
//   ya = (s0,s1) then (s4,s5),   yb = (s2,s3) then (s6,s7)
// then L_hf = (ya.lo + yb.lo) + (ya.hi + yb.hi); y = L_0 + L_1.  Every step is an
// explicit fused multiply-add or a plain add of two values that are not products, so no
// compiler can contract it differently on different paths.
__device__ __forceinline__ float cdot16_canon(const float* c, const float* h) {
  float L[2];
#pragma unroll
  for (int hf = 0; hf < 2; ++hf) {
    const float* cc = c + 8 * hf;
    const float* hh = h + 8 * hf;
    const float ya_lo = fmaf(cc[4], hh[4], fmaf(cc[0], hh[0], 0.f));
    const float ya_hi = fmaf(cc[5], hh[5], fmaf(cc[1], hh[1], 0.f));
    const float yb_lo = fmaf(cc[6], hh[6], fmaf(cc[2], hh[2], 0.f));
    const float yb_hi = fmaf(cc[7], hh[7], fmaf(cc[3], hh[3], 0.f));
    L[hf] = __fadd_rn(__fadd_rn(ya_lo, yb_lo), __fadd_rn(ya_hi, yb_hi));
  }
  return __fadd_rn(L[0], L[1]);
}

__device__ __forceinline__ int read_chunk(const cl_decision* d, int fixed_chunk, int* status) {
  if (d) {
    *status = d->status;
    return d->chunk;
  }
  *status = 0;
  return fixed_chunk;
}

// ---------------------------------------------------------------------------
// Generic kernel
// ---------------------------------------------------------------------------
struct GenericArgs {
  const float *u, *delta, *A, *B, *C, *D, *z, *bias, *h0;
  float *out, *h_last;
  uint64_t batch, dim, L;
  int N;
  int softplus;
  const cl_decision* decision;
};

template <int NS>
__global__ void __launch_bounds__(128) generic_kernel(GenericArgs a) {
  if (a.decision && a.decision->status != 0) return;
  const uint64_t row = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (row >= a.batch * a.dim) return;
  const int N = NS > 0 ? NS : a.N;
  const uint64_t b = row / a.dim, c = row % a.dim;
  float h[NS > 0 ? NS : 64];
  float A2[NS > 0 ? NS : 64];
#pragma unroll
  for (int s = 0; s < (NS > 0 ? NS : 64); ++s) {
    if (s < N) {
      h[s] = a.h0 ? a.h0[row * N + s] : 0.f;
      A2[s] = a.A[c * N + s] * kLog2e;
    }
  }
  const float bias = a.bias ? a.bias[c] : 0.f;
  const float Dc = a.D ? a.D[c] : 0.f;
  const float* Bb = a.B + b * N * a.L;
  const float* Cb = a.C + b * N * a.L;
  for (uint64_t t = 0; t < a.L; ++t) {
    const float u = a.u[row * a.L + t];
    float dt = a.delta[row * a.L + t] + bias;
    if (a.softplus) dt = softplus_canon(dt);
    const float x = __fmul_rn(dt, u);
    float y = 0.f;
    if (NS == 16) {
      float cv[16];
#pragma unroll
      for (int s = 0; s < 16; ++s) {
        const float dA = ex2_approx(A2[s] * dt);
        h[s] = fmaf(dA, h[s], __fmul_rn(Bb[s * a.L + t], x));
        cv[s] = Cb[s * a.L + t];
      }
      y = cdot16_canon(cv, h);
    } else {
#pragma unroll
      for (int s = 0; s < (NS > 0 ? NS : 64); ++s) {
        if (s < N) {
          const float dA = ex2_approx(A2[s] * dt);
          h[s] = fmaf(dA, h[s], __fmul_rn(Bb[s * a.L + t], x));
          y = fmaf(Cb[s * a.L + t], h[s], y);
        }
      }
    }
    y = fmaf(Dc, u, y);
    if (a.z) y *= silu_canon(a.z[row * a.L + t]);
    a.out[row * a.L + t] = y;
  }
  if (a.h_last) {
#pragma unroll
    for (int s = 0; s < (NS > 0 ? NS : 64); ++s)
      if (s < N) a.h_last[row * N + s] = h[s];
  }
}

// ---------------------------------------------------------------------------
// Decode step: one token through the recurrence, state updated in
// place -- mamba_ssm's selective_state_update(state, x, dt, A, B, C, D, z, dt_bias,
// dt_softplus) semantics, with the canonical math above so that prefill(L) followed by
// decode steps reproduces prefill(L + k) bit for bit.  One thread per (b, d) row.
// ---------------------------------------------------------------------------
struct DecodeArgs {
  float* state;  // (batch, dim, N), in/out
  const float *x, *dt, *A, *B, *C, *D, *z, *dt_bias;
  float* out;  // (batch, dim)
  uint64_t batch, dim;
  int N;
  int softplus;
};

template <int NS>
__global__ void __launch_bounds__(128) decode_kernel(DecodeArgs a) {
  const uint64_t row = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (row >= a.batch * a.dim) return;
  const int N = NS > 0 ? NS : a.N;
  const uint64_t b = row / a.dim, c = row - b * a.dim;
  float dt = a.dt[row] + (a.dt_bias ? a.dt_bias[c] : 0.f);
  if (a.softplus) dt = softplus_canon(dt);
  const float u = a.x[row];
  const float xx = __fmul_rn(dt, u);
  float* st = a.state + row * N;
  const float* Bb = a.B + b * N;
  const float* Cb = a.C + b * N;
  float y = 0.f;
  if (NS == 16) {
    float h[16], cv[16];
#pragma unroll
    for (int s = 0; s < 16; ++s) {
      const float dA = ex2_approx((a.A[c * 16 + s] * kLog2e) * dt);
      h[s] = fmaf(dA, st[s], __fmul_rn(Bb[s], xx));
      cv[s] = Cb[s];
    }
    y = cdot16_canon(cv, h);
#pragma unroll
    for (int s = 0; s < 16; ++s) st[s] = h[s];
  } else {
    for (int s = 0; s < N; ++s) {
      const float dA = ex2_approx((a.A[c * N + s] * kLog2e) * dt);
      const float h = fmaf(dA, st[s], __fmul_rn(Bb[s], xx));
      y = fmaf(Cb[s], h, y);
      st[s] = h;
    }
  }
  y = fmaf(a.D ? a.D[c] : 0.f, u, y);
  if (a.z) y *= silu_canon(a.z[row]);
  a.out[row] = y;
}

// ---------------------------------------------------------------------------
// TMA kernels (N = 16): shared helpers, then the 32-row row-sequential kernel
// ---------------------------------------------------------------------------
constexpr int kN = 16;
constexpr int kRows = 32;  // rows per tile = lanes per warp

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
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
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
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0,
                                             int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(src))
      : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read_le1() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned int* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned int* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// two 64-bit words per access (each word single-copy atomic: a tag and its value)
__device__ __forceinline__ void ld_relaxed_u64x2(const unsigned long long* p,
                                                 unsigned long long& a, unsigned long long& b) {
  asm volatile("ld.relaxed.gpu.global.v2.b64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
__device__ __forceinline__ void st_relaxed_u64x2(unsigned long long* p, unsigned long long a,
                                                 unsigned long long b) {
  asm volatile("st.relaxed.gpu.global.v2.b64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}

// ---- packed fp32x2 (FFMA2) helpers: a 64-bit register pair holds two fp32 lanes ----
typedef unsigned long long f2_t;
__device__ __forceinline__ f2_t pk(float lo, float hi) {
  f2_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void upk(f2_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ f2_t fma2(f2_t a, f2_t b, f2_t c) {
  f2_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ f2_t mul2(f2_t a, f2_t b) {
  f2_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2_t add2(f2_t a, f2_t b) {
  f2_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

// softplus for a pair, branch-free: max(x,0) + log1p(exp(-|x|)), log1p by a degree-9
// minimax polynomial on [0,1] (max rel err 2e-7 in fp32).  Equals x to fp32 precision
// above 20, matching mamba_ssm's threshold.
__device__ __forceinline__ f2_t softplus2(f2_t x) {
  float a, b;
  upk(x, a, b);
  const f2_t e = pk(ex2_approx(-fabsf(a) * kLog2e), ex2_approx(-fabsf(b) * kLog2e));
  f2_t q = pk(0.005253826278033571f, 0.005253826278033571f);
  q = fma2(q, e, pk(-0.02959069552080005f, -0.02959069552080005f));
  q = fma2(q, e, pk(0.07836660226277938f, 0.07836660226277938f));
  q = fma2(q, e, pk(-0.13675328086246433f, -0.13675328086246433f));
  q = fma2(q, e, pk(0.19111774195698683f, 0.19111774195698683f));
  q = fma2(q, e, pk(-0.24844483411506615f, -0.24844483411506615f));
  q = fma2(q, e, pk(0.33319289806287417f, 0.33319289806287417f));
  q = fma2(q, e, pk(-0.49999502673812024f, -0.49999502673812024f));
  q = fma2(q, e, pk(0.9999999706625772f, 0.9999999706625772f));
  return fma2(q, e, pk(fmaxf(a, 0.f), fmaxf(b, 0.f)));
}

// z * sigmoid(z) for a pair: one MUFU.EX2 per lane, reciprocal by Newton iterations
// on the FMA pipe (3 steps from the bit-trick seed: rel err < 1e-7).
__device__ __forceinline__ f2_t silu2(f2_t z) {
  float a, b;
  upk(z, a, b);
  const f2_t e =
      pk(ex2_approx(fmaxf(a, -80.f) * -kLog2e), ex2_approx(fmaxf(b, -80.f) * -kLog2e));
  const f2_t d = add2(e, pk(1.f, 1.f));
  float dl, dh;
  upk(d, dl, dh);
  f2_t r = pk(__int_as_float(0x7EF311C7 - __float_as_int(dl)),
              __int_as_float(0x7EF311C7 - __float_as_int(dh)));
  const f2_t one = pk(1.f, 1.f);
  const f2_t nd = mul2(d, pk(-1.f, -1.f));
#pragma unroll
  for (int it = 0; it < 3; ++it) {
    const f2_t e = fma2(nd, r, one);
    r = fma2(r, e, r);
  }
  return mul2(z, r);
}

struct TmaArgs {
  const float *A, *D, *bias, *h0;
  float* out;              // y, for the direct-store (warp-specialised) kernel
  float* h_last;
  float* carry;            // [n_tiles][32][16]
  unsigned int* flags;     // [n_tiles] completed segments
  unsigned long long* tcarry;  // [n_tiles][16][16] {tag << 32 | h bits} (rowpair_ws_kernel)
  unsigned int epoch;          // tag of segment s's carry-in = epoch + s
  int stage_params;            // A / bias / D 16-byte aligned: the producer stages a full
                               // tile's rows of them into shared memory with the item's first box
  unsigned int* ticket;    // work counter
  uint64_t batch, dim, L;
  int tiles_per_batch;
  int n_tiles;
  const cl_decision* decision;
  int fixed_chunk;
};

struct Item {
  int tile, seg, nbox;
  int t0;
};

// Geometry: BOX timesteps per TMA box (32/16/8 -> 128B/64B/32B swizzle),
// WARPS independent warps per CTA, STAGES-deep per-warp TMA ring.
template <int BOX>
struct Geo {
  static constexpr int kTileBytes = kRows * BOX * 4;            // u / delta / z / y
  static constexpr int kBCBytes = BOX * kN * 4;                 // B^T or C^T  [BOX][16]
  static constexpr int kStageBytes = 3 * kTileBytes + 2 * kBCBytes;
  // 16B-chunk j (4 timesteps) of row r inside a swizzled [32 x BOX] box
  static __device__ __forceinline__ int swz(int r, int j) {
    if (BOX == 32) return r * 128 + ((j ^ (r & 7)) << 4);        // SWIZZLE_128B
    if (BOX == 16) return r * 64 + ((j ^ ((r >> 1) & 3)) << 4);  // SWIZZLE_64B
    return r * 32 + ((j ^ ((r >> 2) & 1)) << 4);                 // SWIZZLE_32B
  }
};

template <int BOX, int STAGES>
constexpr int warp_bytes() {
  return STAGES * Geo<BOX>::kStageBytes + 2 * Geo<BOX>::kTileBytes;  // + 2 y staging buffers
}

template <int BOX, int WARPS, int STAGES, bool SP, bool HZ>
__global__ void __launch_bounds__(WARPS * 32, 1)
    rowseq_tma_kernel(const __grid_constant__ CUtensorMap map_u,
                      const __grid_constant__ CUtensorMap map_dt,
                      const __grid_constant__ CUtensorMap map_z,
                      const __grid_constant__ CUtensorMap map_out,
                      const __grid_constant__ CUtensorMap map_Bt,
                      const __grid_constant__ CUtensorMap map_Ct, TmaArgs a) {
  using G = Geo<BOX>;
  int status;
  const int chunk = read_chunk(a.decision, a.fixed_chunk, &status);
  if (status != 0) return;
  int seg_len = chunk < BOX ? BOX : chunk;
  seg_len = (seg_len + BOX - 1) / BOX * BOX;
  const int L = static_cast<int>(a.L);
  const int n_seg = (L + seg_len - 1) / seg_len;
  const int n_items = n_seg * a.n_tiles;

  extern __shared__ unsigned char smem_raw[];
  // align to 1024 B (128B swizzle atom) with pointer arithmetic on the __shared__
  // base, so every access below stays in the shared window (LDS/STS, not generic LD)
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  constexpr int kWB = warp_bytes<BOX, STAGES>();
  unsigned char* wbase = smem + size_t(warp) * kWB;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + size_t(WARPS) * kWB) + warp * 4;
  int meta_item[STAGES], meta_box[STAGES];

  if (lane == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(bars + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_u)));
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_dt)));
    if (HZ) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_z)));
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_Bt)));
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_Ct)));
  }
  __syncwarp();

  auto decode = [&](int id) {
    Item it;
    it.seg = id / a.n_tiles;
    it.tile = id % a.n_tiles;
    it.t0 = it.seg * seg_len;
    const int len = min(seg_len, L - it.t0);
    it.nbox = (len + BOX - 1) / BOX;
    return it;
  };
  auto claim = [&]() {
    int id = 0;
    if (lane == 0) id = static_cast<int>(atomicAdd(a.ticket, 1u));
    return __shfl_sync(0xffffffffu, id, 0);
  };

  int p_item = claim();
  int p_box = 0;
  Item p_it = decode(p_item);
  auto produce = [&](int slot) {
    meta_item[slot] = -1;
    if (p_item >= n_items) return;
    const Item it = p_it;
    meta_item[slot] = p_item;
    meta_box[slot] = p_box;
    if (lane == 0) {
      unsigned char* st = wbase + slot * G::kStageBytes;
      const int b = it.tile / a.tiles_per_batch;
      const int r0 = (it.tile % a.tiles_per_batch) * kRows;
      const int t = it.t0 + p_box * BOX;
      mbar_expect_tx(bars + slot, HZ ? G::kStageBytes : G::kStageBytes - G::kTileBytes);
      tma_load_3d(st, &map_u, t, r0, b, bars + slot);
      tma_load_3d(st + G::kTileBytes, &map_dt, t, r0, b, bars + slot);
      if (HZ) tma_load_3d(st + 2 * G::kTileBytes, &map_z, t, r0, b, bars + slot);
      tma_load_3d(st + 3 * G::kTileBytes, &map_Bt, 0, t, b, bars + slot);
      tma_load_3d(st + 3 * G::kTileBytes + G::kBCBytes, &map_Ct, 0, t, b, bars + slot);
    }
    if (++p_box == it.nbox) {
      p_box = 0;
      p_item = claim();
      p_it = decode(p_item);
    }
  };

  for (int s = 0; s < STAGES; ++s) produce(s);

  unsigned char* ybuf0 = wbase + STAGES * G::kStageBytes;
  f2_t h2[kN / 2], A2p[kN / 2];
  float bias = 0.f, Dc = 0.f;
  Item cur{};
  int row = 0;
  bool row_valid = false;
  for (int iter = 0;; ++iter) {
    const int slot = iter % STAGES;
    const int item = meta_item[slot];
    if (item < 0) break;
    const int box = meta_box[slot];
    if (box == 0) {
      cur = decode(item);
      const int b = cur.tile / a.tiles_per_batch;
      const int c = (cur.tile % a.tiles_per_batch) * kRows + lane;
      row_valid = c < static_cast<int>(a.dim);
      const int cc = row_valid ? c : 0;
      row = b * static_cast<int>(a.dim) + cc;
#pragma unroll
      for (int s = 0; s < kN; s += 4) {
        const float4 q = *reinterpret_cast<const float4*>(a.A + size_t(cc) * kN + s);
        A2p[s / 2] = pk(q.x * kLog2e, q.y * kLog2e);
        A2p[s / 2 + 1] = pk(q.z * kLog2e, q.w * kLog2e);
      }
      bias = a.bias ? a.bias[cc] : 0.f;
      Dc = a.D ? a.D[cc] : 0.f;
      const float* src = nullptr;
      if (cur.seg == 0) {
        src = a.h0 ? a.h0 + size_t(row) * kN : nullptr;
      } else {
        // chained carry from segment seg-1 of this tile
        if (lane == 0)
          while (ld_acquire(a.flags + cur.tile) < static_cast<unsigned>(cur.seg)) __nanosleep(64);
        __syncwarp();
        src = a.carry + (size_t(cur.tile) * kRows + lane) * kN;
      }
#pragma unroll
      for (int s = 0; s < kN; s += 4) {
        float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
        if (src) q = __ldcg(reinterpret_cast<const float4*>(src + s));
        h2[s / 2] = pk(q.x, q.y);
        h2[s / 2 + 1] = pk(q.z, q.w);
      }
    }

    mbar_wait(bars + slot, (iter / STAGES) & 1);
    // y staging is double-buffered: this buffer is free once the store issued two
    // boxes ago has read it (at most the newest store may still be in flight)
    unsigned char* ybuf = ybuf0 + (iter & 1) * G::kTileBytes;
    if (lane == 0) bulk_wait_read_le1();
    __syncwarp();
    unsigned char* st = wbase + slot * G::kStageBytes;
    const unsigned char* sB = st + 3 * G::kTileBytes;
    const unsigned char* sC = sB + G::kBCBytes;
    const int tbox = cur.t0 + box * BOX;
    const int valid = min(BOX, L - tbox);  // multiple of 4 (L % 4 == 0)
    const f2_t bias2 = pk(bias, bias);
#pragma unroll
    for (int j = 0; j < BOX / 4; ++j) {
      if (4 * j >= valid) break;
      const int off = G::swz(lane, j);
      const float4 u4 = *reinterpret_cast<const float4*>(st + off);
      const float4 d4 = *reinterpret_cast<const float4*>(st + G::kTileBytes + off);
      // elementwise prologue for the 4 timesteps, packed in pairs
      f2_t dt01 = add2(pk(d4.x, d4.y), bias2), dt23 = add2(pk(d4.z, d4.w), bias2);
      if (SP) {
        dt01 = softplus2(dt01);
        dt23 = softplus2(dt23);
      }
      const f2_t x01 = mul2(dt01, pk(u4.x, u4.y)), x23 = mul2(dt23, pk(u4.z, u4.w));
      float dt[4], xs[4];
      upk(dt01, dt[0], dt[1]);
      upk(dt23, dt[2], dt[3]);
      upk(x01, xs[0], xs[1]);
      upk(x23, xs[2], xs[3]);
      float yy[4];
      // phase A: the 4x16 transition factors exp(dt*A) do not depend on the state,
      // so they are all issued up front (MUFU-paced, independent)
      f2_t dA[4][kN / 2];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const f2_t dd = pk(dt[k], dt[k]);
#pragma unroll
        for (int i = 0; i < kN / 2; ++i) {
          float al, ah;
          upk(mul2(A2p[i], dd), al, ah);
          dA[k][i] = pk(ex2_approx(al), ex2_approx(ah));
        }
      }
      // phase B: recurrence h = dA*h + B*x and y = C.h, FFMA2 on state pairs
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int t = 4 * j + k;
        const ulonglong2* Bt = reinterpret_cast<const ulonglong2*>(sB + t * kN * 4);
        const ulonglong2* Ct = reinterpret_cast<const ulonglong2*>(sC + t * kN * 4);
        const f2_t xx = pk(xs[k], xs[k]);
        // canonical FFMA2 chains per half (cdot16_canon): pairs 0,2 / 1,3 and 4,6 / 5,7
        f2_t ya0 = 0ull, yb0 = 0ull, ya1 = 0ull, yb1 = 0ull;
#pragma unroll
        for (int q = 0; q < kN / 4; ++q) {
          const ulonglong2 bq = Bt[q];
          const ulonglong2 cq = Ct[q];
          h2[2 * q] = fma2(dA[k][2 * q], h2[2 * q], mul2(bq.x, xx));
          h2[2 * q + 1] = fma2(dA[k][2 * q + 1], h2[2 * q + 1], mul2(bq.y, xx));
          if (q < 2) {
            ya0 = fma2(cq.x, h2[2 * q], ya0);
            yb0 = fma2(cq.y, h2[2 * q + 1], yb0);
          } else {
            ya1 = fma2(cq.x, h2[2 * q], ya1);
            yb1 = fma2(cq.y, h2[2 * q + 1], yb1);
          }
        }
        float l0a, l0b, l1a, l1b;
        upk(add2(ya0, yb0), l0a, l0b);
        upk(add2(ya1, yb1), l1a, l1b);
        yy[k] = (l0a + l0b) + (l1a + l1b);
      }
      const float uu[4] = {u4.x, u4.y, u4.z, u4.w};
      f2_t y01 = fma2(pk(Dc, Dc), pk(uu[0], uu[1]), pk(yy[0], yy[1]));
      f2_t y23 = fma2(pk(Dc, Dc), pk(uu[2], uu[3]), pk(yy[2], yy[3]));
      if (HZ) {
        const float4 z4 = *reinterpret_cast<const float4*>(st + 2 * G::kTileBytes + off);
        y01 = mul2(y01, silu2(pk(z4.x, z4.y)));
        y23 = mul2(y23, silu2(pk(z4.z, z4.w)));
      }
      float o0, o1, o2, o3;
      upk(y01, o0, o1);
      upk(y23, o2, o3);
      *reinterpret_cast<float4*>(ybuf + off) = make_float4(o0, o1, o2, o3);
    }
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) {
      const int b = cur.tile / a.tiles_per_batch;
      const int r0 = (cur.tile % a.tiles_per_batch) * kRows;
      tma_store_3d(&map_out, ybuf, tbox, r0, b);
    }

    if (box == cur.nbox - 1) {
      float hs[kN];
#pragma unroll
      for (int i = 0; i < kN / 2; ++i) upk(h2[i], hs[2 * i], hs[2 * i + 1]);
      if (cur.seg == n_seg - 1) {
        if (a.h_last && row_valid) {
#pragma unroll
          for (int s = 0; s < kN; s += 4)
            *reinterpret_cast<float4*>(a.h_last + size_t(row) * kN + s) =
                make_float4(hs[s], hs[s + 1], hs[s + 2], hs[s + 3]);
        }
      } else {
        float* cw = a.carry + (size_t(cur.tile) * kRows + lane) * kN;
#pragma unroll
        for (int s = 0; s < kN; s += 4)
          __stcg(reinterpret_cast<float4*>(cw + s),
                 make_float4(hs[s], hs[s + 1], hs[s + 2], hs[s + 3]));
        __threadfence();
        __syncwarp();
        if (lane == 0) st_release(a.flags + cur.tile, static_cast<unsigned>(cur.seg + 1));
      }
    }
    // every lane has consumed this slot: refill it for iteration iter + STAGES
    __syncwarp();
    produce(slot);
  }
  if (lane == 0) bulk_wait_all();
  __syncwarp();
}

// ---------------------------------------------------------------------------
// Warp-specialised lane-pair kernel (the hot path).
//
// Layout: a consumer warp owns a 16-row tile; lanes (2r, 2r+1) share row r and hold
// states 0-7 / 8-15 as FFMA2 register pairs.  That doubles the independent row
// chains of the 32-row kernel for the same shape (the chained-segment schedule caps
// busy warps at the tile count: 2048 tiles at C3 = 13.8 warps per SM), at the cost
// of one 64-bit shuffle pair per 4 timesteps.
//
// Roles: WARPS consumer warps only compute; NPROD producer warps run the consumers'
// TMA rings (lane l of producer p owns consumer p*ceil(WARPS/NPROD) + l): ticket
// claims, expect_tx and the four tile loads per box (u, delta, z and one interleaved
// [B | C] box).  Measured on C3: issuing TMA from the compute warps cost ~10% of
// the scan, one producer warp could not keep up with 14 consumers (its per-lane
// TMA issue serialises through uniform registers), two can.  y is stored straight
// from registers (8 B per lane per 4 timesteps, st.global.cs): the four stores of a
// box complete each 64-byte row segment in L2 within microseconds, and dropping the
// y staging buffer, proxy fence and TMA store saved another ~3%.
// ---------------------------------------------------------------------------
constexpr int kRowsP = 16;
#ifndef CL_PROD_SLEEP_NS
#define CL_PROD_SLEEP_NS 32
#endif

template <int BOX>
struct GeoP {
  static constexpr int kTileBytes = kRowsP * BOX * 4;  // u / delta / z: [16 rows][BOX]
  static constexpr int kBCBytes = BOX * 2 * kN * 4;    // [BOX][B 0..15 | C 0..15]
  static constexpr int kStageBytes = 3 * kTileBytes + kBCBytes;
  // per-item parameters staged with an item's first box: A rows [16][16], bias [16], D [16]
  static constexpr int kParamBytes = kRowsP * kN * 4 + 2 * kRowsP * 4;
};
constexpr int kStagedFlag = 1 << 30;  // meta.y bit: this item's parameters are in shared memory

__device__ __forceinline__ f2_t shfl_xor2(f2_t v, int m) {
  float lo, hi;
  upk(v, lo, hi);
  return pk(__shfl_xor_sync(0xffffffffu, lo, m), __shfl_xor_sync(0xffffffffu, hi, m));
}

// One 16-row x BOX-timestep box: lane (r, hf) owns row r's states 8hf..8hf+7.  Reads
// u / delta / z / [B | C] from the TMA stage `st`, advances the carried state h2 and
// stores y for timesteps (4j + 2hf, 4j + 2hf + 1) of row r to ydst (nullptr: pad row).
template <int BOX, bool SP, bool HZ>
__device__ __forceinline__ void pair_box(const unsigned char* st, float* ydst, int r, int hf,
                                         int valid, float bias, float Dc,
                                         const f2_t (&A2p)[kN / 4], f2_t (&h2)[kN / 4]) {
  using G = GeoP<BOX>;
  constexpr int kP = kN / 4;
  constexpr int kBCRow = 2 * kN * 4;
  const unsigned char* sB = st + 3 * G::kTileBytes + 32 * hf;  // this lane's 8 states
  const unsigned char* sC = sB + kN * 4;
  const f2_t bias2 = pk(bias, bias);
  // fully unrolled over the box's 4-timestep groups: straight-line code lets the
  // scheduler interleave group j+1's exponentials with group j's FFMA2 chains
#pragma unroll
  for (int j = 0; j < BOX / 4; ++j) {
    if (4 * j >= valid) break;
    const int off = Geo<BOX>::swz(r, j);
    const float4 u4 = *reinterpret_cast<const float4*>(st + off);
    const float4 d4 = *reinterpret_cast<const float4*>(st + G::kTileBytes + off);
    // softplus of timesteps (2hf, 2hf+1) here, the other pair from the partner lane
    f2_t mine = add2(hf ? pk(d4.z, d4.w) : pk(d4.x, d4.y), bias2);
    if (SP) mine = softplus2(mine);
    const f2_t other = shfl_xor2(mine, 1);
    const f2_t dt01 = hf ? other : mine, dt23 = hf ? mine : other;
    const f2_t x01 = mul2(dt01, pk(u4.x, u4.y)), x23 = mul2(dt23, pk(u4.z, u4.w));
    float dt[4], xs[4];
    upk(dt01, dt[0], dt[1]);
    upk(dt23, dt[2], dt[3]);
    upk(x01, xs[0], xs[1]);
    upk(x23, xs[2], xs[3]);
    // the 4x8 transition factors exp(dt*A) do not depend on the state: issue them all
    f2_t dA[4][kP];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const f2_t dd = pk(dt[k], dt[k]);
#pragma unroll
      for (int i = 0; i < kP; ++i) {
        float al, ah;
        upk(mul2(A2p[i], dd), al, ah);
        dA[k][i] = pk(ex2_approx(al), ex2_approx(ah));
      }
    }
    float yp[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int t = 4 * j + k;
      const ulonglong2* Bt = reinterpret_cast<const ulonglong2*>(sB + t * kBCRow);
      const ulonglong2* Ct = reinterpret_cast<const ulonglong2*>(sC + t * kBCRow);
      const f2_t xx = pk(xs[k], xs[k]);
      f2_t ya = 0ull, yb = 0ull;  // canonical FFMA2 chains (cdot16_canon)
#pragma unroll
      for (int q = 0; q < kP / 2; ++q) {
        const ulonglong2 bq = Bt[q];
        const ulonglong2 cq = Ct[q];
        h2[2 * q] = fma2(dA[k][2 * q], h2[2 * q], mul2(bq.x, xx));
        h2[2 * q + 1] = fma2(dA[k][2 * q + 1], h2[2 * q + 1], mul2(bq.y, xx));
        ya = fma2(cq.x, h2[2 * q], ya);
        yb = fma2(cq.y, h2[2 * q + 1], yb);
      }
      float a0, a1;
      upk(add2(ya, yb), a0, a1);
      yp[k] = a0 + a1;
    }
    // lane hf finalises timesteps (2hf, 2hf+1): swap the partial sums it does not own
    const f2_t keep = hf ? pk(yp[2], yp[3]) : pk(yp[0], yp[1]);
    const f2_t give = hf ? pk(yp[0], yp[1]) : pk(yp[2], yp[3]);
    const f2_t ysum = add2(keep, shfl_xor2(give, 1));
    const f2_t u2 = hf ? pk(u4.z, u4.w) : pk(u4.x, u4.y);
    f2_t yo = fma2(pk(Dc, Dc), u2, ysum);
    if (HZ) {
      const float4 z4 = *reinterpret_cast<const float4*>(st + 2 * G::kTileBytes + off);
      yo = mul2(yo, silu2(hf ? pk(z4.z, z4.w) : pk(z4.x, z4.y)));
    }
    if (ydst) {
      float y0, y1;
      upk(yo, y0, y1);
      __stcs(reinterpret_cast<float2*>(ydst + 4 * j + 2 * hf), make_float2(y0, y1));
    }
  }
}

// pair_box for a full box (valid == BOX), software-pipelined by one 4-timestep group:
// group j+1's serial prologue (LDS of u / delta / z, bias add, softplus -- one MUFU then
// a 9-deep FFMA2 chain -- the partner-lane shuffle and the SiLU(z) gate) is issued between group j's
// exponentials and its recurrence, so its latency hides under group j's MUFU work
// instead of stalling the MUFU pipe at every group boundary.  Same operations on the
// same values as pair_box, so the outputs are bit-identical.
template <int BOX, bool SP, bool HZ>
__device__ __forceinline__ void pair_box_pipe(const unsigned char* st, float* ydst, int r,
                                              int hf, float bias, float Dc,
                                              const f2_t (&A2p)[kN / 4], f2_t (&h2)[kN / 4]) {
  using G = GeoP<BOX>;
  constexpr int kP = kN / 4;
  constexpr int kG = BOX / 4;
  constexpr int kBCRow = 2 * kN * 4;
  const unsigned char* sB = st + 3 * G::kTileBytes + 32 * hf;
  const unsigned char* sC = sB + kN * 4;
  const f2_t bias2 = pk(bias, bias);
  // prologue of group j: dt (4 timesteps, softplus'd), x = dt*u, and this lane's u pair
  auto prep = [&](int j, float (&dt)[4], float (&xs)[4], f2_t& u2, f2_t& g2) {
    const int off = Geo<BOX>::swz(r, j);
    const float4 u4 = *reinterpret_cast<const float4*>(st + off);
    const float4 d4 = *reinterpret_cast<const float4*>(st + G::kTileBytes + off);
    f2_t mine = add2(hf ? pk(d4.z, d4.w) : pk(d4.x, d4.y), bias2);
    if (SP) mine = softplus2(mine);
    const f2_t other = shfl_xor2(mine, 1);
    const f2_t dt01 = hf ? other : mine, dt23 = hf ? mine : other;
    const f2_t x01 = mul2(dt01, pk(u4.x, u4.y)), x23 = mul2(dt23, pk(u4.z, u4.w));
    upk(dt01, dt[0], dt[1]);
    upk(dt23, dt[2], dt[3]);
    upk(x01, xs[0], xs[1]);
    upk(x23, xs[2], xs[3]);
    u2 = hf ? pk(u4.z, u4.w) : pk(u4.x, u4.y);
    if (HZ) {
      const float4 z4 = *reinterpret_cast<const float4*>(st + 2 * G::kTileBytes + off);
      g2 = silu2(hf ? pk(z4.z, z4.w) : pk(z4.x, z4.y));
    }
  };
  float dt[4], xs[4];
  f2_t u2, g2 = 0ull;
  prep(0, dt, xs, u2, g2);
#pragma unroll
  for (int j = 0; j < kG; ++j) {
    f2_t dA[4][kP];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const f2_t dd = pk(dt[k], dt[k]);
#pragma unroll
      for (int i = 0; i < kP; ++i) {
        float al, ah;
        upk(mul2(A2p[i], dd), al, ah);
        dA[k][i] = pk(ex2_approx(al), ex2_approx(ah));
      }
    }
    float ndt[4], nxs[4];
    f2_t nu2 = 0ull, ng2 = 0ull;
    if (j + 1 < kG) prep(j + 1, ndt, nxs, nu2, ng2);
    float yp[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int t = 4 * j + k;
      const ulonglong2* Bt = reinterpret_cast<const ulonglong2*>(sB + t * kBCRow);
      const ulonglong2* Ct = reinterpret_cast<const ulonglong2*>(sC + t * kBCRow);
      const f2_t xx = pk(xs[k], xs[k]);
      f2_t ya = 0ull, yb = 0ull;  // canonical FFMA2 chains (cdot16_canon)
#pragma unroll
      for (int q = 0; q < kP / 2; ++q) {
        const ulonglong2 bq = Bt[q];
        const ulonglong2 cq = Ct[q];
        h2[2 * q] = fma2(dA[k][2 * q], h2[2 * q], mul2(bq.x, xx));
        h2[2 * q + 1] = fma2(dA[k][2 * q + 1], h2[2 * q + 1], mul2(bq.y, xx));
        ya = fma2(cq.x, h2[2 * q], ya);
        yb = fma2(cq.y, h2[2 * q + 1], yb);
      }
      float a0, a1;
      upk(add2(ya, yb), a0, a1);
      yp[k] = a0 + a1;
    }
    const f2_t keep = hf ? pk(yp[2], yp[3]) : pk(yp[0], yp[1]);
    const f2_t give = hf ? pk(yp[0], yp[1]) : pk(yp[2], yp[3]);
    const f2_t ysum = add2(keep, shfl_xor2(give, 1));
    f2_t yo = fma2(pk(Dc, Dc), u2, ysum);
    if (HZ) yo = mul2(yo, g2);
    if (ydst) {
      float y0, y1;
      upk(yo, y0, y1);
      __stcs(reinterpret_cast<float2*>(ydst + 4 * j + 2 * hf), make_float2(y0, y1));
    }
    if (j + 1 < kG) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        dt[k] = ndt[k];
        xs[k] = nxs[k];
      }
      u2 = nu2;
      g2 = ng2;
    }
  }
}

// Per consumer warp and stage: full[s] (producer arrive.expect_tx + TMA bytes) and
// empty[s] (consumer lane 0 arrive after its last shared-memory read of the stage).
// The meta words (item, box) travel through shared memory under full[s]'s release.
template <int BOX, int WARPS, int STAGES, bool SP, bool HZ, int NPROD, int PIPE>
__global__ void __launch_bounds__((WARPS + NPROD) * 32, 1)
    rowpair_ws_kernel(const __grid_constant__ CUtensorMap map_u,
                      const __grid_constant__ CUtensorMap map_dt,
                      const __grid_constant__ CUtensorMap map_z,
                      const __grid_constant__ CUtensorMap map_bc, TmaArgs a) {
  using G = GeoP<BOX>;
  int status;
  const int chunk = read_chunk(a.decision, a.fixed_chunk, &status);
  if (status != 0) return;
  int seg_len = chunk < BOX ? BOX : chunk;
  seg_len = (seg_len + BOX - 1) / BOX * BOX;
  const int L = static_cast<int>(a.L);
  const int n_seg = (L + seg_len - 1) / seg_len;
  const int n_items = n_seg * a.n_tiles;

  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  constexpr int kWB = STAGES * G::kStageBytes;
  unsigned char* params = smem + size_t(WARPS) * kWB;  // [WARPS][STAGES][kParamBytes]
  uint64_t* full = reinterpret_cast<uint64_t*>(params + size_t(WARPS) * STAGES * G::kParamBytes);
  uint64_t* empty = full + WARPS * STAGES;                                  // [WARPS][STAGES]
  int2* meta = reinterpret_cast<int2*>(empty + WARPS * STAGES);              // [WARPS][STAGES]

  if (threadIdx.x < WARPS * STAGES) {
    mbar_init(full + threadIdx.x, 1);
    mbar_init(empty + threadIdx.x, 1);
  }
  if (threadIdx.x == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();

  auto decode = [&](int id) {
    Item it;
    it.seg = id / a.n_tiles;
    it.tile = id % a.n_tiles;
    it.t0 = it.seg * seg_len;
    const int len = min(seg_len, L - it.t0);
    it.nbox = (len + BOX - 1) / BOX;
    return it;
  };

  if (warp >= WARPS) {
    // ---------------- producers ----------------
    constexpr int kPer = (WARPS + NPROD - 1) / NPROD;
    const int w = (warp - WARPS) * kPer + lane;
    bool live = lane < kPer && w < WARPS;
    if (lane == 0 && warp == WARPS) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_u)));
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_dt)));
      if (HZ) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_z)));
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_bc)));
    }
    // boxes go through each consumer's ring in ticket order
    int p_item = live ? static_cast<int>(atomicAdd(a.ticket, 1u)) : 0;
    Item p_it = decode(p_item);
    int p_b = p_it.tile / a.tiles_per_batch, p_r0 = (p_it.tile % a.tiles_per_batch) * kRowsP;
    int p_box = 0, n_issued = 0;
    unsigned char* wbase = smem + size_t(w < WARPS ? w : 0) * kWB;
    while (__any_sync(0xffffffffu, live)) {
      bool issued = false;
      if (live) {
        const int slot = n_issued % STAGES;
        const bool free = n_issued < STAGES ||
                          mbar_test(empty + w * STAGES + slot, ((n_issued / STAGES) - 1) & 1);
        if (free) {
          uint64_t* bar = full + w * STAGES + slot;
          if (p_item >= n_items) {
            meta[w * STAGES + slot] = make_int2(-1, 0);
            mbar_arrive(bar);
            live = false;
          } else {
            unsigned char* st = wbase + slot * G::kStageBytes;
            const int t = p_it.t0 + p_box * BOX;
            const bool stage = p_box == 0 && a.stage_params &&
                               p_r0 + kRowsP <= static_cast<int>(a.dim);
            meta[w * STAGES + slot] = make_int2(p_item, p_box | (stage ? kStagedFlag : 0));
            uint32_t tx = HZ ? G::kStageBytes : G::kStageBytes - G::kTileBytes;
            if (stage) tx += kRowsP * kN * 4 + (a.bias ? kRowsP * 4 : 0) + (a.D ? kRowsP * 4 : 0);
            mbar_expect_tx(bar, tx);
            if (stage) {
              unsigned char* pp = params + (size_t(w) * STAGES + slot) * G::kParamBytes;
              bulk_g2s(pp, a.A + size_t(p_r0) * kN, kRowsP * kN * 4, bar);
              if (a.bias) bulk_g2s(pp + kRowsP * kN * 4, a.bias + p_r0, kRowsP * 4, bar);
              if (a.D) bulk_g2s(pp + kRowsP * kN * 4 + kRowsP * 4, a.D + p_r0, kRowsP * 4, bar);
            }
            tma_load_3d(st, &map_u, t, p_r0, p_b, bar);
            tma_load_3d(st + G::kTileBytes, &map_dt, t, p_r0, p_b, bar);
            if (HZ) tma_load_3d(st + 2 * G::kTileBytes, &map_z, t, p_r0, p_b, bar);
            tma_load_3d(st + 3 * G::kTileBytes, &map_bc, 0, t, p_b, bar);
            if (++p_box == p_it.nbox) {
              p_box = 0;
              p_item = static_cast<int>(atomicAdd(a.ticket, 1u));
              p_it = decode(p_item);
              p_b = p_it.tile / a.tiles_per_batch;
              p_r0 = (p_it.tile % a.tiles_per_batch) * kRowsP;
            }
          }
          ++n_issued;
          issued = true;
        }
      }
      if (!__any_sync(0xffffffffu, issued)) __nanosleep(CL_PROD_SLEEP_NS);
    }
    return;
  }

  // ---------------- consumers ----------------
  const int r = lane >> 1, hf = lane & 1;
  const unsigned char* wbase = smem + size_t(warp) * kWB;
  uint64_t* wfull = full + warp * STAGES;
  uint64_t* wempty = empty + warp * STAGES;
  const int2* wmeta = meta + warp * STAGES;
  constexpr int kP = kN / 4;
  f2_t h2[kP], A2p[kP];
  float bias = 0.f, Dc = 0.f;
  Item cur{};
  int row = 0;
  bool row_valid = false;
  for (int iter = 0;; ++iter) {
    const int slot = iter % STAGES;
    mbar_wait(wfull + slot, (iter / STAGES) & 1);
    const int2 m = wmeta[slot];
    if (m.x < 0) break;
    const int box = m.y & ~kStagedFlag;
    if (box == 0) {
      cur = decode(m.x);
      const int b = cur.tile / a.tiles_per_batch;
      const int c = (cur.tile % a.tiles_per_batch) * kRowsP + r;
      row_valid = c < static_cast<int>(a.dim);
      const int cc = row_valid ? c : 0;
      row = b * static_cast<int>(a.dim) + cc;
      if (m.y & kStagedFlag) {
        // staged by the producer with this box (shared memory: no global round trip)
        const unsigned char* pp = params + (size_t(warp) * STAGES + slot) * G::kParamBytes;
#pragma unroll
        for (int s = 0; s < kN / 2; s += 4) {
          const float4 q = *reinterpret_cast<const float4*>(pp + (r * kN + 8 * hf + s) * 4);
          A2p[s / 2] = pk(q.x * kLog2e, q.y * kLog2e);
          A2p[s / 2 + 1] = pk(q.z * kLog2e, q.w * kLog2e);
        }
        bias = a.bias ? reinterpret_cast<const float*>(pp + kRowsP * kN * 4)[r] : 0.f;
        Dc = a.D ? reinterpret_cast<const float*>(pp + kRowsP * kN * 4 + kRowsP * 4)[r] : 0.f;
      } else {
#pragma unroll
        for (int s = 0; s < kN / 2; s += 4) {
          const float4 q = *reinterpret_cast<const float4*>(a.A + size_t(cc) * kN + 8 * hf + s);
          A2p[s / 2] = pk(q.x * kLog2e, q.y * kLog2e);
          A2p[s / 2 + 1] = pk(q.z * kLog2e, q.w * kLog2e);
        }
        bias = a.bias ? a.bias[cc] : 0.f;
        Dc = a.D ? a.D[cc] : 0.f;
      }
      const float* src = nullptr;
      if (cur.seg == 0) {
        src = a.h0 ? a.h0 + size_t(row) * kN + 8 * hf : nullptr;
      }
      if (cur.seg == 0) {
#pragma unroll
        for (int s = 0; s < kN / 2; s += 4) {
          float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
          if (src) q = __ldcg(reinterpret_cast<const float4*>(src + s));
          h2[s / 2] = pk(q.x, q.y);
          h2[s / 2 + 1] = pk(q.z, q.w);
        }
      } else {
        // chained carry from segment seg-1 of this tile: every word carries its own tag,
        // so a lane polls its 8 words with relaxed loads -- no flag, no acquire / release
        // (the writer's release would also wait for all of its y stores to land)
        const unsigned long long* w64 =
            a.tcarry + (size_t(cur.tile) * kRowsP + r) * kN + 8 * hf;
        const unsigned want = a.epoch + static_cast<unsigned>(cur.seg);
        unsigned long long w[kN / 2];
        for (;;) {
          bool ok = true;
#pragma unroll
          for (int i = 0; i < kN / 2; i += 2) {
            ld_relaxed_u64x2(w64 + i, w[i], w[i + 1]);
            ok &= static_cast<unsigned>(w[i] >> 32) == want;
            ok &= static_cast<unsigned>(w[i + 1] >> 32) == want;
          }
          if (__all_sync(0xffffffffu, ok)) break;
          __nanosleep(64);
        }
#pragma unroll
        for (int i = 0; i < kP; ++i)
          h2[i] = pk(__uint_as_float(static_cast<unsigned>(w[2 * i])),
                     __uint_as_float(static_cast<unsigned>(w[2 * i + 1])));
      }
    }

    const int tbox = cur.t0 + box * BOX;
    float* ydst = row_valid ? a.out + size_t(row) * a.L + tbox : nullptr;
    if (PIPE == 1 && tbox + BOX <= L)
      pair_box_pipe<BOX, SP, HZ>(wbase + slot * G::kStageBytes, ydst, r, hf, bias, Dc, A2p, h2);
    else
      pair_box<BOX, SP, HZ>(wbase + slot * G::kStageBytes, ydst, r, hf, min(BOX, L - tbox), bias,
                            Dc, A2p, h2);
    __syncwarp();
    if (lane == 0) mbar_arrive(wempty + slot);  // stage consumed: producer may refill

    if (box == cur.nbox - 1) {
      float hs[kN / 2];
#pragma unroll
      for (int i = 0; i < kP; ++i) upk(h2[i], hs[2 * i], hs[2 * i + 1]);
      if (cur.seg == n_seg - 1) {
        if (a.h_last && row_valid) {
          float* dst = a.h_last + size_t(row) * kN + 8 * hf;
          __stcg(reinterpret_cast<float4*>(dst), make_float4(hs[0], hs[1], hs[2], hs[3]));
          __stcg(reinterpret_cast<float4*>(dst + 4), make_float4(hs[4], hs[5], hs[6], hs[7]));
        }
      } else {
        unsigned long long* w64 = a.tcarry + (size_t(cur.tile) * kRowsP + r) * kN + 8 * hf;
        const unsigned long long tag =
            static_cast<unsigned long long>(a.epoch + static_cast<unsigned>(cur.seg + 1)) << 32;
#pragma unroll
        for (int i = 0; i < kN / 2; i += 2)
          st_relaxed_u64x2(w64 + i, tag | __float_as_uint(hs[i]), tag | __float_as_uint(hs[i + 1]));
      }
    }
  }
}

// (b, N, L) -> (b, L, N) for B and C, so a timestep's 16 state coefficients are one
// contiguous 64-byte row: the scan then reads them as FFMA2 register pairs.
__global__ void __launch_bounds__(256) transpose_bc_kernel(const float* __restrict__ B,
                                                           const float* __restrict__ C,
                                                           float* __restrict__ Bt,
                                                           float* __restrict__ Ct, int L,
                                                           int row_stride) {
  __shared__ float tile[kN][33];
  const float* src = blockIdx.z ? C : B;
  float* dst = blockIdx.z ? Ct : Bt;
  const int b = blockIdx.y, t0 = blockIdx.x * 32;
  const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;  // ty 0..7
  for (int s = ty; s < kN; s += 8) {
    const int t = t0 + tx;
    tile[s][tx] = t < L ? src[(size_t(b) * kN + s) * L + t] : 0.f;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 32 * kN; e += 256) {
    const int tt = e / kN, s = e % kN;
    const int t = t0 + tt;
    if (t < L) dst[(size_t(b) * L + t) * row_stride + s] = tile[s][tt];
  }
}

// ---------------------------------------------------------------------------
// host side: tensor maps through the driver entry point (no libcuda link)
// ---------------------------------------------------------------------------
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn get_encode() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

bool make_map(CUtensorMap* m, const float* base, uint64_t d0, uint64_t d1, uint64_t d2,
              uint32_t box0, uint32_t box1, int swizzle_bytes) {
  EncodeFn enc = get_encode();
  if (!enc) return false;
  const cuuint64_t dims[3] = {d0, d1, d2};
  const cuuint64_t strides[2] = {d0 * 4, d0 * d1 * 4};
  const cuuint32_t box[3] = {box0, box1, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUtensorMapSwizzle sw = swizzle_bytes == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                                : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                      : CU_TENSOR_MAP_SWIZZLE_NONE;
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box,
             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

bool tma_eligible(const cl_mamba1_args& a) {
  if (a.d_state != kN) return false;
  if (a.seq_len % 4 != 0) return false;
  if (a.seq_len > (1u << 30) || a.dim > (1u << 30) || a.batch > (1u << 30)) return false;
  const void* ps[] = {a.u, a.delta, a.out, a.B, a.C, a.A};
  for (const void* p : ps)
    if (!aligned16(p)) return false;
  if (a.z && !aligned16(a.z)) return false;
  if (a.h0 && !aligned16(a.h0)) return false;
  if (a.h_last && !aligned16(a.h_last)) return false;
  return get_encode() != nullptr;
}

template <typename T>
int grow(cl_ctx* ctx, T** ptr, size_t* have, size_t need, const char* what) {
  if (*have >= need) return CL_OK;
  if (*ptr) cudaFree(*ptr);
  *ptr = nullptr;
  *have = 0;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(ptr), need);
  if (e != cudaSuccess) return cuda_fail(ctx, e, what);
  *have = need;
  return CL_OK;
}

// ---- kernel table (CL_SCAN_CFG=<index> selects a row, for experiments) ----
enum ScanKind { kWarpSpecPair = 0, kRowSeq = 1, kWarpSpecPairNoPipe = 2 };
struct ScanCfg {
  int kind, box, warps, stages;
};
constexpr ScanCfg kCfgs[] = {
    // 12 consumer + 2 producer warps per SM (C3, C4): three consumers on every SM
    // sub-partition, so every warp gets the same share of its SMSP's MUFU quarter.
    // Measured at C3 (scan ms): 12 consumers 1.357; 13: 1.373; 14 (4/4/3/3 per SMSP):
    // 1.404 -- the uneven sub-partitions made warps wait on each other's carries (ncu:
    // carry-spin samples 2.7% -> 0.3%); 16 (capped at 96 registers, spills): 1.726;
    // 12 x 3 stages 1.371; 8 consumers 1.497; 12 with 1 producer 1.572, with 3: 1.371.
    // 16 consumers + a producer warpgroup that hands its registers over with setmaxnreg
    // (consumers 112, producers 24; no hot-loop spills): 1.654 -- more warps per SMSP do
    // not buy MUFU issue once each has fewer registers for the group pipeline.
    {kWarpSpecPair, 16, 12, 2},
    {kRowSeq, 32, 4, 3},         // 32-row tiles, self-fed TMA rings
    {kRowSeq, 16, 8, 3},
    {kRowSeq, 16, 7, 3},
    // few 16-row tiles (C1: 96, C2: 128): fewer consumers per CTA so the tiles spread over
    // all SMs instead of packing 12 to an SM (one producer, deeper ring)
    {kWarpSpecPair, 16, 1, 4},
    {kWarpSpecPair, 16, 2, 4},
    {kWarpSpecPair, 16, 4, 4},
    {kWarpSpecPair, 16, 7, 3},
    {kWarpSpecPairNoPipe, 16, 12, 2},  // 8: row 0 without the group software pipeline (A/B)
    {kWarpSpecPair, 16, 14, 2},        // 9: 14 consumers (the previous default)
    // A quad layout for few tiles (a warp pair per 16-row tile, four lanes per row, each
    // lane's chain a canonical ya / yb, bitwise equal to the lane pair) was measured
    // slower: C1 0.26 vs 0.17 ms, C2 0.49 vs 0.30 -- the per-lane elementwise work
    // (softplus, SiLU, exchanges) does not shrink with the lane's state count, so the
    // instruction count went up 1.8x on latency-bound lone warps (commit history).
    {kWarpSpecPair, 32, 1, 4},  // 10: few tiles, 32-timestep boxes (half the per-box overhead)
    {kWarpSpecPair, 32, 2, 4},  // 11
    {kWarpSpecPair, 32, 4, 3},  // 12
    {kWarpSpecPair, 32, 8, 2},  // 13
    {kWarpSpecPair, 32, 6, 3},  // 14
};
constexpr int kDefaultCfg = 0;

// producers per CTA: two keep up with 12-14 consumers (one feeding 12 costs +16%), one with up to 7
template <int WARPS>
constexpr int producers_for() {
  return WARPS >= 8 ? 2 : 1;
}

template <typename K>
cudaError_t set_smem(K kern, size_t smem) {
  return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(smem));
}

int grid_for(int n_tiles, int warps, int num_sms) {
  const int max_useful = (n_tiles + warps - 1) / warps;
  return max_useful < num_sms ? (max_useful < 1 ? 1 : max_useful) : num_sms;
}

template <int BOX, int WARPS, int STAGES, bool SP, bool HZ, int PIPE = 1, int NP = 0>
cudaError_t launch_ws(const CUtensorMap (&m)[6], const TmaArgs& t, int num_sms, cudaStream_t s) {
  constexpr int kProducers = NP > 0 ? NP : producers_for<WARPS>();
  auto kern = rowpair_ws_kernel<BOX, WARPS, STAGES, SP, HZ, kProducers, PIPE>;
  const size_t smem = size_t(WARPS) * STAGES * (GeoP<BOX>::kStageBytes + GeoP<BOX>::kParamBytes) +
                      1024 + size_t(WARPS) * STAGES * (16 + 8);
  cudaError_t e = set_smem(kern, smem);
  if (e != cudaSuccess) return e;
  kern<<<grid_for(t.n_tiles, WARPS, num_sms), (WARPS + kProducers) * 32, smem, s>>>(
      m[0], m[1], m[2], m[4], t);
  return cudaGetLastError();
}

template <int BOX, int WARPS, int STAGES, bool SP, bool HZ>
cudaError_t launch_rowseq(const CUtensorMap (&m)[6], const TmaArgs& t, int num_sms,
                          cudaStream_t s) {
  auto kern = rowseq_tma_kernel<BOX, WARPS, STAGES, SP, HZ>;
  const size_t smem = size_t(WARPS) * warp_bytes<BOX, STAGES>() + 1024 + 256;
  cudaError_t e = set_smem(kern, smem);
  if (e != cudaSuccess) return e;
  kern<<<grid_for(t.n_tiles, WARPS, num_sms), WARPS * 32, smem, s>>>(m[0], m[1], m[2], m[3],
                                                                      m[4], m[5], t);
  return cudaGetLastError();
}

// softplus / z-gate are compile-time switches: four instantiations per geometry
template <bool WS, int BOX, int WARPS, int STAGES>
cudaError_t dispatch(bool sp, bool hz, const CUtensorMap (&m)[6], const TmaArgs& t, int n,
                     cudaStream_t s) {
  if constexpr (WS) {
    if (sp && hz) return launch_ws<BOX, WARPS, STAGES, true, true>(m, t, n, s);
    if (sp) return launch_ws<BOX, WARPS, STAGES, true, false>(m, t, n, s);
    if (hz) return launch_ws<BOX, WARPS, STAGES, false, true>(m, t, n, s);
    return launch_ws<BOX, WARPS, STAGES, false, false>(m, t, n, s);
  } else {
    if (sp && hz) return launch_rowseq<BOX, WARPS, STAGES, true, true>(m, t, n, s);
    if (sp) return launch_rowseq<BOX, WARPS, STAGES, true, false>(m, t, n, s);
    if (hz) return launch_rowseq<BOX, WARPS, STAGES, false, true>(m, t, n, s);
    return launch_rowseq<BOX, WARPS, STAGES, false, false>(m, t, n, s);
  }
}

// CL_SCAN_CFG=<row> forces a kCfgs row (experiments); otherwise the warp-specialised
// kernel with the fewest consumers per CTA that still puts every 16-row tile on its own
// SM (12 consumers once there are more than 7 tiles per SM).
constexpr int kNumCfgs = static_cast<int>(sizeof(kCfgs) / sizeof(kCfgs[0]));

int scan_cfg_index(uint64_t pair_tiles, int num_sms, int variant) {
  if (variant >= CL_SCAN_CONFIG_BASE) return variant - CL_SCAN_CONFIG_BASE;
  static const int forced = [] {
    const char* e = getenv("CL_SCAN_CFG");
    if (!e) return -1;
    const int v = atoi(e);
    return v >= 0 && v < static_cast<int>(sizeof(kCfgs) / sizeof(kCfgs[0])) ? v : -1;
  }();
  if (forced >= 0) return forced;
  const uint64_t per_sm = (pair_tiles + num_sms - 1) / num_sms;
  // Below ~11 tiles per SM, 32-timestep boxes (half the per-box pipeline fill and barrier
  // round trips) with the fewest consumers per CTA that still cover the tiles in about one
  // wave.  Measured (scan ms, tools/cfg_ab.py): C1 (96 tiles) 0.167 -> 0.152 (row 11);
  // C2 (128) 0.301 -> 0.269 (11); 512 tiles 0.327 -> 0.309 (12); 768: 0.453 -> 0.388 (12);
  // 1280: 0.634 -> 0.521 (13); 1792 and C3's 2048 stay with row 0 (0.649 vs 0.708, 1.376
  // vs 1.530 for row 13).
  if (per_sm <= 2) return 11;
  if (per_sm <= 6) return 12;
  if (per_sm <= 10) return 13;
  return kDefaultCfg;  // 12 consumers
}

}  // namespace

int scan_mamba1(cl_ctx* ctx, const cl_mamba1_args& a, const cl_decision* d_decision,
                int fixed_chunk, int variant, cudaStream_t s) {
  const bool tma_ok = tma_eligible(a);
  if (variant >= CL_SCAN_CONFIG_BASE && variant - CL_SCAN_CONFIG_BASE >= kNumCfgs)
    return fail(ctx, CL_E_INVALID, "scan variant: no such kernel configuration");
  if ((variant == CL_SCAN_ROWSEQ_TMA || variant >= CL_SCAN_CONFIG_BASE) && !tma_ok)
    return fail(ctx, CL_E_INVALID, "scan variant rowseq_tma needs d_state 16, L % 4 == 0 and 16-byte aligned buffers");
  const bool use_tma = variant == CL_SCAN_ROWSEQ_TMA || variant >= CL_SCAN_CONFIG_BASE ||
                       (variant == CL_SCAN_AUTO && tma_ok);
  if (use_tma) {
    const uint64_t pair_tiles = ((a.dim + kRowsP - 1) / kRowsP) * a.batch;
    const int cfg_idx = scan_cfg_index(pair_tiles, ctx->num_sms, variant);
    const ScanCfg cfg = kCfgs[cfg_idx];
    const bool ws = cfg.kind != kRowSeq;
    const uint64_t L = a.seq_len, D = a.dim, Bt = a.batch;
    const int rows_per_tile = ws ? kRowsP : kRows;
    const int tiles_per_batch = static_cast<int>((D + rows_per_tile - 1) / rows_per_tile);
    const int n_tiles = tiles_per_batch * static_cast<int>(Bt);
    const size_t work_bytes = (size_t(n_tiles) + 32) * sizeof(unsigned int);
    const size_t carry_bytes = size_t(n_tiles) * rows_per_tile * kN * sizeof(float);
    const size_t bc_bytes = 2 * size_t(Bt) * L * kN * sizeof(float);
    cl_workspace* w = workspace(ctx, s);  // scratch of this stream only
    if (!w) return CL_E_CUDA;
    int rc = grow(ctx, &w->d_work, &w->work_bytes, work_bytes, "cudaMalloc(scan work)");
    if (!rc && !ws)
      rc = grow(ctx, &w->d_carry, &w->carry_bytes, carry_bytes, "cudaMalloc(carry)");
    if (!rc) rc = grow(ctx, &w->d_bct, &w->bct_bytes, bc_bytes, "cudaMalloc(B/C transpose)");
    if (rc) return rc;
    unsigned int epoch = 0;
    if (ws) {
      // tagged carry words: zeroed when (re)allocated or when the epoch would wrap; each
      // launch takes tags epoch + 1 .. epoch + (segments <= boxes), above every older tag
      const size_t tcarry_bytes = size_t(n_tiles) * kRowsP * kN * sizeof(unsigned long long);
      const bool fresh = w->tcarry_bytes < tcarry_bytes;
      rc = grow(ctx, &w->d_tcarry, &w->tcarry_bytes, tcarry_bytes, "cudaMalloc(tagged carry)");
      if (rc) return rc;
      const unsigned span = static_cast<unsigned>((L + cfg.box - 1) / cfg.box) + 2u;
      if (fresh || w->carry_epoch == 0 || w->carry_epoch > 0xFFFFFFFFu - span) {
        cudaError_t e = cudaMemsetAsync(w->d_tcarry, 0, w->tcarry_bytes, s);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMemsetAsync(tagged carry)");
        w->carry_epoch = 1;
      }
      epoch = w->carry_epoch;
      w->carry_epoch += span;
    }
    // B^T / C^T: interleaved per timestep ([B | C], 128 B rows, one TMA box) for the
    // warp-specialised kernel, two separate (b, L, 16) arrays for the row kernel
    float* d_Bt = w->d_bct;
    float* d_Ct = ws ? w->d_bct + kN : w->d_bct + size_t(Bt) * L * kN;
    const int box = cfg.box;
    const int sw = box == 32 ? 128 : (box == 16 ? 64 : 32);
    CUtensorMap m[6];  // u, delta, z, out, B^T (or [B|C]), C^T
    std::memset(m, 0, sizeof(m));
    bool ok = make_map(&m[0], a.u, L, D, Bt, box, rows_per_tile, sw) &&
              make_map(&m[1], a.delta, L, D, Bt, box, rows_per_tile, sw) &&
              make_map(&m[2], a.z ? a.z : a.u, L, D, Bt, box, rows_per_tile, sw) &&
              make_map(&m[3], a.out, L, D, Bt, box, rows_per_tile, sw);
    if (ok && ws) ok = make_map(&m[4], d_Bt, 2 * kN, L, Bt, 2 * kN, box, 0);
    if (ok && !ws)
      ok = make_map(&m[4], d_Bt, kN, L, Bt, kN, box, 0) &&
           make_map(&m[5], d_Ct, kN, L, Bt, kN, box, 0);
    if (!ok) return fail(ctx, CL_E_CUDA, "cuTensorMapEncodeTiled failed");
    cudaError_t e = cudaMemsetAsync(w->d_work, 0, work_bytes, s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMemsetAsync(scan work)");
    const dim3 tgrid(static_cast<unsigned>((L + 31) / 32), static_cast<unsigned>(Bt), 2);
    transpose_bc_kernel<<<tgrid, 256, 0, s>>>(a.B, a.C, d_Bt, d_Ct, static_cast<int>(L),
                                              ws ? 2 * kN : kN);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(ctx, e, "transpose_bc_kernel launch");
    ++ctx->launches;
    TmaArgs t{};
    t.out = a.out;
    t.A = a.A;
    t.D = a.D;
    t.bias = a.delta_bias;
    t.h0 = a.h0;
    t.h_last = a.h_last;
    t.carry = w->d_carry;
    t.tcarry = w->d_tcarry;
    t.epoch = epoch;
    t.stage_params = aligned16(a.A) && (!a.delta_bias || aligned16(a.delta_bias)) &&
                     (!a.D || aligned16(a.D));
    t.ticket = w->d_work;
    t.flags = w->d_work + 32;
    t.batch = Bt;
    t.dim = D;
    t.L = L;
    t.tiles_per_batch = tiles_per_batch;
    t.n_tiles = n_tiles;
    t.decision = d_decision;
    t.fixed_chunk = fixed_chunk;
    const bool sp = a.delta_softplus != 0, hz = a.z != nullptr;
    const int n = ctx->num_sms;
    switch (cfg_idx) {
      case 1: e = dispatch<false, 32, 4, 3>(sp, hz, m, t, n, s); break;
      case 2: e = dispatch<false, 16, 8, 3>(sp, hz, m, t, n, s); break;
      case 3: e = dispatch<false, 16, 7, 3>(sp, hz, m, t, n, s); break;
      case 4: e = dispatch<true, 16, 1, 4>(sp, hz, m, t, n, s); break;
      case 5: e = dispatch<true, 16, 2, 4>(sp, hz, m, t, n, s); break;
      case 6: e = dispatch<true, 16, 4, 4>(sp, hz, m, t, n, s); break;
      case 7: e = dispatch<true, 16, 7, 3>(sp, hz, m, t, n, s); break;
      case 8:
        e = sp && hz ? launch_ws<16, 12, 2, true, true, 0>(m, t, n, s)
                     : dispatch<true, 16, 12, 2>(sp, hz, m, t, n, s);
        break;
      case 9: e = dispatch<true, 16, 14, 2>(sp, hz, m, t, n, s); break;
      case 10: e = dispatch<true, 32, 1, 4>(sp, hz, m, t, n, s); break;
      case 11: e = dispatch<true, 32, 2, 4>(sp, hz, m, t, n, s); break;
      case 12: e = dispatch<true, 32, 4, 3>(sp, hz, m, t, n, s); break;
      case 13: e = dispatch<true, 32, 8, 2>(sp, hz, m, t, n, s); break;
      case 14: e = dispatch<true, 32, 6, 3>(sp, hz, m, t, n, s); break;
      default: e = dispatch<true, 16, 12, 2>(sp, hz, m, t, n, s); break;
    }
    if (e != cudaSuccess) return cuda_fail(ctx, e, "scan kernel launch");
    ++ctx->launches;
    return CL_OK;
  }
  if (a.d_state < 1 || a.d_state > 64)
    return fail(ctx, CL_E_INVALID, "d_state must lie in [1, 64]");
  GenericArgs g{};
  g.u = a.u;
  g.delta = a.delta;
  g.A = a.A;
  g.B = a.B;
  g.C = a.C;
  g.D = a.D;
  g.z = a.z;
  g.bias = a.delta_bias;
  g.h0 = a.h0;
  g.out = a.out;
  g.h_last = a.h_last;
  g.batch = a.batch;
  g.dim = a.dim;
  g.L = a.seq_len;
  g.N = static_cast<int>(a.d_state);
  g.softplus = a.delta_softplus;
  g.decision = d_decision;
  const uint64_t rows = a.batch * a.dim;
  const unsigned grid = static_cast<unsigned>((rows + 127) / 128);
  if (a.d_state == 16)
    generic_kernel<16><<<grid, 128, 0, s>>>(g);
  else
    generic_kernel<0><<<grid, 128, 0, s>>>(g);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(ctx, e, "generic_kernel launch");
  ++ctx->launches;
  (void)fixed_chunk;
  return CL_OK;
}

int state_update_f32(cl_ctx* ctx, const cl_state_update_args& a, cudaStream_t s) {
  DecodeArgs d{a.state, a.x, a.dt, a.A, a.B, a.C, a.D, a.z, a.dt_bias, a.out,
               a.batch, a.dim, static_cast<int>(a.d_state), a.dt_softplus};
  const uint64_t rows = a.batch * a.dim;
  if (rows == 0) return CL_OK;
  const unsigned grid = static_cast<unsigned>((rows + 127) / 128);
  if (a.d_state == 16)
    decode_kernel<16><<<grid, 128, 0, s>>>(d);
  else
    decode_kernel<0><<<grid, 128, 0, s>>>(d);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(ctx, e, "decode_kernel launch");
  ++ctx->launches;
  return CL_OK;
}

}  // namespace cl
