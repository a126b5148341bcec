// conv_common.cuh -- the depthwise causal conv1d (+ SiLU) arithmetic of the producer of u,
// shared by conv1d.cu (conv with the range epilogue) and entropy.cu (conv with the
// Fixed-range histogram epilogue), so both produce the identical bits of u.
//   u[b,d,t] = act(bias[d] + sum_{k<W} weight[d,k] * x[b,d,t-(W-1)+k]),  x[.,.,<0] = 0
// accumulated in fp32 from bias in k order with fused multiply-adds.
#pragma once

#include <cuda_runtime.h>

namespace cl {
namespace {

__device__ __forceinline__ float conv_act(float v, bool silu) {
  // SiLU: v * sigmoid(v); MUFU exp + fast divide (a few ulp).  The exponent is clamped
  // at 88 so the denominator stays finite (< 2^128) for v < -88, where the quotient
  // is then 0 (the limit of v * sigmoid(v))
  return silu ? __fdividef(v, 1.f + __expf(fminf(-v, 88.f))) : v;
}

// One 32-quad block of a row in the warp-coalesced layout: lane l holds quad l (`in`); the
// previous quad comes from lane l-1 by shuffle, for lane 0 from `prev31` (the previous
// block's lane 31, or the zero padding / one load at a run start), which is then advanced
// to this block's lane 31.  All 32 lanes must call it.
template <int W>
__device__ __forceinline__ void conv_block(const float4& in, float4& prev31, int lane,
                                           const float (&wk)[W], float bias, bool silu,
                                           float (&o)[4]) {
  float4 pv;
  pv.y = __shfl_up_sync(0xffffffffu, in.y, 1);
  pv.z = __shfl_up_sync(0xffffffffu, in.z, 1);
  pv.w = __shfl_up_sync(0xffffffffu, in.w, 1);
  if (lane == 0) pv = prev31;
  prev31.y = __shfl_sync(0xffffffffu, in.y, 31);
  prev31.z = __shfl_sync(0xffffffffu, in.z, 31);
  prev31.w = __shfl_sync(0xffffffffu, in.w, 31);
  const float xs[8] = {0.f, pv.y, pv.z, pv.w, in.x, in.y, in.z, in.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float s = bias;
#pragma unroll
    for (int k = 0; k < W; ++k) s = fmaf(wk[k], xs[4 + i - (W - 1) + k], s);
    o[i] = conv_act(s, silu);
  }
}

}  // namespace
}  // namespace cl
