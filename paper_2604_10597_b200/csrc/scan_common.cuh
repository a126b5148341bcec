// scan_common.cuh -- device and host building blocks shared by the fused Mamba-1 scan
// kernels (scan_mamba1.cu: chained-carry kernels; scan_lookback.cu: the L-parallel
// kernel for few-row shapes).  Everything is in an anonymous namespace: each
// translation unit gets its own copy (device code is inlined anyway).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "cl_internal.h"
#include "tma_map.cuh"

// Device-side invariant checks (A/B builds with -DCL_DEVICE_CHECKS=1; compute-sanitizer is
// closed on this pool): a failed check prints and traps.
#ifndef CL_DEVICE_CHECKS
#define CL_DEVICE_CHECKS 0
#endif
#define CL_DCHECK(cond)                                                                 \
  do {                                                                                  \
    if (CL_DEVICE_CHECKS && !(cond)) {                                                  \
      printf("CL_DCHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__,   \
             #cond, blockIdx.x, threadIdx.x);                                           \
      __trap();                                                                         \
    }                                                                                   \
  } while (0)

namespace cl {
namespace {

constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// ---- exponentials of the elementwise terms (softplus, SiLU) ----
// ex2.approx (MUFU) by default.  CL_ELEM_MUFU=0 moves the two elementwise exponentials
// per element to the FMA pipe: 2^x = p(f) * 2^n, n = rint(x) by the 1.5 * 2^23 magic add,
// f = x - n exactly, p a degree-5 minimax polynomial for 2^f on [-1/2, 1/2] (max rel err
// 1.5e-7; ex2.approx's is 2.4e-7), 2^n added into the exponent field, x clamped below at
// -125, NaN kept.  It takes the scan from 18 to 16 MUFU per element, and is SLOWER:
// C3 scan 1.414 vs 1.351 ms (profiles/r2d_elem_exp_ab.txt) -- the longer dependent chain
// sits in every group's prologue, and the FMA pipe is already half busy.
#ifndef CL_ELEM_MUFU
#define CL_ELEM_MUFU 1
#endif
constexpr float kE2c0 = 1.0000001192092896f, kE2c1 = 0.6931469440460205f,
                kE2c2 = 0.24022120237350464f, kE2c3 = 0.05550713092088699f,
                kE2c4 = 0.009675540961325169f, kE2c5 = 0.001327647129073739f;

__device__ __forceinline__ float max_nan(float a, float b) {
  float y;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(y) : "f"(a), "f"(b));
  return y;
}

__device__ __forceinline__ float exp2_elem(float x) {
#if CL_ELEM_MUFU
  return ex2_approx(x);
#else
  x = max_nan(x, -125.f);
  const float t = __fadd_rn(x, 12582912.f);
  const float f = __fadd_rn(x, -__fadd_rn(t, -12582912.f));
  float p = fmaf(kE2c5, f, kE2c4);
  p = fmaf(p, f, kE2c3);
  p = fmaf(p, f, kE2c2);
  p = fmaf(p, f, kE2c1);
  p = fmaf(p, f, kE2c0);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
#endif
}

// ---- exponentials of the state transitions, dA = 2^(A log2e dt) ----
// MUFU by default.  CL_STATE_POLY=m (0..4) computes the states s with ((s & 7) >> 1) < m
// -- m of every lane's 4 state pairs -- on the FMA pipe instead: n = rint(x) by the
// 1.5 * 2^23 magic add, f = x - n exactly, 2^f = 1 + f q(f) with q a degree-4 polynomial
// (minimax relative error of 2^f with the constant term pinned to 1 so dA -> 1 exactly as
// dt -> 0: 6.8e-8, 2.2e-7 after fp32 rounding; ex2.approx: 2.4e-7), 2^n added into the
// exponent field, x clamped to [-125, 127] (NaN kept).  Every kernel picks the same
// function for the same state, so all paths stay bitwise consistent.  A/B in
// profiles/r2k_state_poly_ab.txt.
#ifndef CL_STATE_POLY
#define CL_STATE_POLY 0
#endif
constexpr float kSq1 = 0.6931465864181519f, kSq2 = 0.24022166430950165f,
                kSq3 = 0.055510472506284714f, kSq4 = 0.009674952365458012f,
                kSq5 = 0.0013202981790527701f;

__device__ __forceinline__ float min_nan(float a, float b) {
  float y;
  asm("min.NaN.f32 %0, %1, %2;" : "=f"(y) : "f"(a), "f"(b));
  return y;
}

__device__ __forceinline__ bool state_on_fma(int s) { return ((s & 7) >> 1) < CL_STATE_POLY; }

__device__ __forceinline__ float exp2_state_poly(float x) {
  x = min_nan(max_nan(x, -125.f), 127.f);
  const float t = __fadd_rn(x, 12582912.f);
  const float f = __fadd_rn(x, -__fadd_rn(t, -12582912.f));
  float q = fmaf(kSq5, f, kSq4);
  q = fmaf(q, f, kSq3);
  q = fmaf(q, f, kSq2);
  q = fmaf(q, f, kSq1);
  const float p = fmaf(q, f, 1.f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

// dA of state s (scalar kernels: generic scan, decode)
__device__ __forceinline__ float state_exp2(float x, int s) {
  return state_on_fma(s) ? exp2_state_poly(x) : ex2_approx(x);
}

// ---- canonical elementwise math ----
// Every Mamba-1 path (generic scan, TMA scans, decode) evaluates softplus, SiLU and, for
// N = 16, C.h with exactly these operation sequences, so the paths agree bit for bit
// and a prefill followed by decode steps equals a longer prefill bit for bit (the
// paper's passive-vs-routed claim is bitwise output equality).  The
// FFMA2 versions further down (softplus2 / silu2 / the lane-pair C.h) are these
// functions applied per lane of a register pair.

// softplus(x) = max(x,0) + log1p(exp(-|x|)): one exponential (exp2_elem) and a degree-9
// minimax polynomial for log1p on [0,1] (max rel err 2e-7; equals x to fp32 above 20).
__device__ __forceinline__ float softplus_canon(float a) {
  const float e = exp2_elem(-fabsf(a) * kLog2e);
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

// z * sigmoid(z): one exponential (exp2_elem), reciprocal by 3 Newton steps from the
// bit-trick seed.
__device__ __forceinline__ float silu_canon(float z) {
  const float e = exp2_elem(fmaxf(z, -80.f) * -kLog2e);
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
        const float dA = state_exp2(A2[s] * dt, s);
        h[s] = fmaf(dA, h[s], __fmul_rn(Bb[s * a.L + t], x));
        cv[s] = Cb[s * a.L + t];
      }
      y = cdot16_canon(cv, h);
    } else {
#pragma unroll
      for (int s = 0; s < (NS > 0 ? NS : 64); ++s) {
        if (s < N) {
          const float dA = state_exp2(A2[s] * dt, s);
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
      const float dA = state_exp2((a.A[c * 16 + s] * kLog2e) * dt, s);
      h[s] = fmaf(dA, st[s], __fmul_rn(Bb[s], xx));
      cv[s] = Cb[s];
    }
    y = cdot16_canon(cv, h);
#pragma unroll
    for (int s = 0; s < 16; ++s) st[s] = h[s];
  } else {
    for (int s = 0; s < N; ++s) {
      const float dA = state_exp2((a.A[c * N + s] * kLog2e) * dt, s);
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
// exp2_elem on both lanes of a pair (FFMA2 / FADD2: each lane rounds exactly like the
// scalar sequence, so the pair and scalar paths agree bit for bit)
__device__ __forceinline__ f2_t exp2_elem2(float xa, float xb) {
#if CL_ELEM_MUFU
  return pk(ex2_approx(xa), ex2_approx(xb));
#else
  const f2_t x = pk(max_nan(xa, -125.f), max_nan(xb, -125.f));
  const f2_t t = add2(x, pk(12582912.f, 12582912.f));
  const f2_t n = add2(t, pk(-12582912.f, -12582912.f));
  float nl, nh;
  upk(n, nl, nh);
  const f2_t f = add2(x, pk(-nl, -nh));
  f2_t p = fma2(pk(kE2c5, kE2c5), f, pk(kE2c4, kE2c4));
  p = fma2(p, f, pk(kE2c3, kE2c3));
  p = fma2(p, f, pk(kE2c2, kE2c2));
  p = fma2(p, f, pk(kE2c1, kE2c1));
  p = fma2(p, f, pk(kE2c0, kE2c0));
  float pl, ph, tl, th;
  upk(p, pl, ph);
  upk(t, tl, th);
  return pk(__int_as_float(__float_as_int(pl) + (__float_as_int(tl) << 23)),
            __int_as_float(__float_as_int(ph) + (__float_as_int(th) << 23)));
#endif
}

// dA of the state pair (s0, s0 + 1), s0 even, i = (s0 & 7) >> 1 (compile-time in the
// unrolled pair loops); per lane the same operations as state_exp2
__device__ __forceinline__ f2_t state_exp2_pair(f2_t x2, int i) {
  float xa, xb;
  upk(x2, xa, xb);
  if (i >= CL_STATE_POLY) return pk(ex2_approx(xa), ex2_approx(xb));
  const f2_t x = pk(min_nan(max_nan(xa, -125.f), 127.f), min_nan(max_nan(xb, -125.f), 127.f));
  const f2_t t = add2(x, pk(12582912.f, 12582912.f));
  const f2_t n = add2(t, pk(-12582912.f, -12582912.f));
  float nl, nh;
  upk(n, nl, nh);
  const f2_t f = add2(x, pk(-nl, -nh));
  f2_t q = fma2(pk(kSq5, kSq5), f, pk(kSq4, kSq4));
  q = fma2(q, f, pk(kSq3, kSq3));
  q = fma2(q, f, pk(kSq2, kSq2));
  q = fma2(q, f, pk(kSq1, kSq1));
  const f2_t p = fma2(q, f, pk(1.f, 1.f));
  float pl, ph, tl, th;
  upk(p, pl, ph);
  upk(t, tl, th);
  return pk(__int_as_float(__float_as_int(pl) + (__float_as_int(tl) << 23)),
            __int_as_float(__float_as_int(ph) + (__float_as_int(th) << 23)));
}

__device__ __forceinline__ f2_t softplus2(f2_t x) {
  float a, b;
  upk(x, a, b);
  const f2_t e = exp2_elem2(-fabsf(a) * kLog2e, -fabsf(b) * kLog2e);
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
  const f2_t e = exp2_elem2(fmaxf(a, -80.f) * -kLog2e, fmaxf(b, -80.f) * -kLog2e);
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

// ---------------------------------------------------------------------------
// lane-pair building blocks (a consumer warp owns a 16-row tile; lanes (2r, 2r+1) share
// row r, states 0-7 / 8-15 in FFMA2 register pairs)
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

// Self-resetting work ticket: ticket[0] is the item counter, ticket[1] counts finished
// claimers; the last of `claimers` warps (after its final claim) zeroes both.  Every
// claiming lane ends with exactly one claim past the last item, so a ticket that started
// at 0 ends at n_items + claiming lanes (checked in CL_DEVICE_CHECKS builds: a dirty
// ticket would have skipped items and left consumers waiting for carries).
// In a captured graph the last claimer also advances the workspace's launch counter (every
// CTA read it at its start, and every CTA has started once all claimers retired).
__device__ __forceinline__ void ticket_retire(unsigned int* ticket, unsigned claimers, int lane,
                                              unsigned expect_final,
                                              unsigned int* launch_counter = nullptr) {
  if (lane == 0) {
    __threadfence();
    if (atomicAdd(ticket + 1, 1u) == claimers - 1) {
      CL_DCHECK(atomicAdd(ticket, 0u) == expect_final);
      atomicExch(ticket, 0u);
      atomicExch(ticket + 1, 0u);
      if (launch_counter) atomicAdd(launch_counter, 1u);
    }
  }
}

// Tag of a launch's words: the host's epoch (eager; always < 0x80000000), or in a captured
// graph 0x80000000 | the device-side launch counter -- every replay of every graph captured
// on the stream gets its own tag (2^31 launches before one could repeat), so the graph
// needs no in-graph memset of the tagged words.
constexpr unsigned kGraphEpochA = 0x80000000u;
__device__ __forceinline__ unsigned launch_epoch(unsigned host_epoch, const unsigned int* counter) {
  if (!counter) return host_epoch;
  return kGraphEpochA | (__ldcg(counter) & 0x7FFFFFFFu);
}

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
    const float2 d2 = *reinterpret_cast<const float2*>(st + G::kTileBytes + off + 8 * hf);
    // softplus of timesteps (2hf, 2hf+1) here, the other pair from the partner lane
    f2_t mine = add2(pk(d2.x, d2.y), bias2);
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
        dA[k][i] = state_exp2_pair(mul2(A2p[i], dd), i);
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
      const float2 z2 = *reinterpret_cast<const float2*>(st + 2 * G::kTileBytes + off + 8 * hf);
      yo = mul2(yo, silu2(pk(z2.x, z2.y)));
    }
    if (ydst) {
      float y0, y1;
      upk(yo, y0, y1);
      CL_DCHECK(4 * j + 2 * hf + 1 < valid);
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
    // this lane's delta pair (timesteps 2hf, 2hf + 1): an 8-byte load, no select
    const float2 d2 = *reinterpret_cast<const float2*>(st + G::kTileBytes + off + 8 * hf);
    f2_t mine = add2(pk(d2.x, d2.y), bias2);
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
      const float2 z2 = *reinterpret_cast<const float2*>(st + 2 * G::kTileBytes + off + 8 * hf);
      g2 = silu2(pk(z2.x, z2.y));
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
        dA[k][i] = state_exp2_pair(mul2(A2p[i], dd), i);
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

// ---------------------------------------------------------------------------
// host side: tensor maps through the driver entry point (no libcuda link)
// ---------------------------------------------------------------------------
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


}  // namespace
}  // namespace cl

namespace cl {
// ---- the L-parallel kernel (scan_lookback.cu), launched by scan_mamba1() ----
struct LookbackLaunch {
  const float *A, *D, *bias, *h0;
  float* out;
  float* h_last;
  unsigned long long* agg;  // [n_tiles][n_seg][16][18] tagged words
  unsigned int epoch;
  unsigned int* launch_counter;  // captured graphs: the device-side launch counter (else null)
  int stage_params;
  unsigned int* ticket;
  uint64_t batch, dim, L;
  int tiles_per_batch, n_tiles, seg_len, n_seg;
  const cl_decision* decision;
};
constexpr int kLookbackCfgs = 6;
int lookback_warps(int cfg);
int lookback_box(int cfg);
cudaError_t launch_lookback(int cfg, bool sp, bool hz, const CUtensorMap* maps,
                            const LookbackLaunch& p, int num_sms, cudaStream_t s);
}  // namespace cl
