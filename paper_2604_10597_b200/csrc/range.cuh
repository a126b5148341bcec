// range.cuh -- the stage-1 range protocol shared by every kernel that produces it
// (minmax_f32/f64 in entropy.cu, the fused conv1d epilogue in conv1d.cu).
//
// d_range holds 4 doubles {-lo, hi, nonfinite, 0}; every field only ever grows, so
// partial results from blocks, kernels and ranks combine with MAX (atomics here,
// ncclAllReduce(MAX) across GPUs).  lo/hi cover the sampled elements (global flat
// index % stride == 0, entropy.hpp:108-114); nonfinite covers every element
// (validate_tensor, entropy.hpp:42).
#pragma once

#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>

namespace cl {
namespace range {

__device__ __forceinline__ bool finite_f32(float x) {
  return (__float_as_uint(x) & 0x7f800000u) != 0x7f800000u;
}
__device__ __forceinline__ bool finite_f64(double x) {
  return (__double_as_longlong(x) & 0x7ff0000000000000ll) != 0x7ff0000000000000ll;
}

__device__ __forceinline__ void atomic_max_f64(double* addr, double v) {
  unsigned long long* a = reinterpret_cast<unsigned long long*>(addr);
  unsigned long long old = *a;
  while (__longlong_as_double(static_cast<long long>(old)) < v) {
    const unsigned long long assumed = old;
    old = atomicCAS(a, assumed, static_cast<unsigned long long>(__double_as_longlong(v)));
    if (old == assumed) break;
  }
}

// Per-thread accumulator for fp32 producers.
struct Acc {
  float lo = FLT_MAX, hi = -FLT_MAX;
  bool any = false, bad = false;
  __device__ __forceinline__ void visit(float x, bool is_sampled) {
    bad |= !finite_f32(x);
    if (is_sampled) {
      lo = fminf(lo, x);
      hi = fmaxf(hi, x);
      any = true;
    }
  }
};

// Block reduce (blockDim.x == THREADS) and one atomic per field per block.
template <int THREADS>
__device__ __forceinline__ void commit(Acc a, double* range) {
  for (int o = 16; o; o >>= 1) {
    a.lo = fminf(a.lo, __shfl_xor_sync(0xffffffffu, a.lo, o));
    a.hi = fmaxf(a.hi, __shfl_xor_sync(0xffffffffu, a.hi, o));
  }
  a.any = __any_sync(0xffffffffu, a.any);
  a.bad = __any_sync(0xffffffffu, a.bad);
  __shared__ float s_lo[THREADS / 32], s_hi[THREADS / 32];
  __shared__ int s_any[THREADS / 32], s_bad[THREADS / 32];
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  if (l == 0) {
    s_lo[w] = a.lo;
    s_hi[w] = a.hi;
    s_any[w] = a.any;
    s_bad[w] = a.bad;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < THREADS / 32; ++k) {
      a.lo = fminf(a.lo, s_lo[k]);
      a.hi = fmaxf(a.hi, s_hi[k]);
      a.any |= s_any[k] != 0;
      a.bad |= s_bad[k] != 0;
    }
    if (a.any) {
      atomic_max_f64(range + 0, -static_cast<double>(a.lo));
      atomic_max_f64(range + 1, static_cast<double>(a.hi));
    }
    if (a.bad) atomic_max_f64(range + 2, 1.0);
  }
}

}  // namespace range
}  // namespace cl
