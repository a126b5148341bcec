// conv1d.cu -- producer fusion: Mamba-1's depthwise causal conv1d +
// SiLU, which produces the scan input u, with the entropy stage-1 epilogue folded in.
//
// Semantics (causal_conv1d_fn(x, weight, bias, activation="silu"), the producer of u in
// the paper's MambaMixer):
//   u[b,d,t] = act(bias[d] + sum_{k<W} weight[d,k] * x[b,d,t-(W-1)+k]),  x[.,.,<0] = 0
// accumulated in fp32 from bias in k order with fused multiply-adds, act = SiLU or
// identity.  Parity unpinned (the reference has no convolution); tests check it
// against an fp64 restatement.
//
// Epilogue: the same range protocol as cl_minmax_f32 (range.cuh) over the produced u
// -- strided min/max at global flat indices, finite check of every element -- so
// cl_conv1d_f32 + cl_histogram_f32 + cl_decide gives the identical decision to
// cl_minmax_f32 over a separately produced u, while u is read from HBM once instead of
// twice.  HBM-bound: reads x (4 B/elem), writes u (4 B/elem).
#include <cuda_runtime.h>

#include <cstdint>

#include "cl_internal.h"
#include "conv_common.cuh"
#include "range.cuh"

namespace cl {
namespace {

constexpr int kConvThreads = 256;

template <int MODE>
__device__ __forceinline__ bool sampled(uint64_t gi, uint64_t stride) {
  if (MODE == 0) return true;
  if (MODE == 1) return (gi & (stride - 1)) == 0;
  return gi % stride == 0;
}

__device__ __forceinline__ float act(float v, bool silu) { return conv_act(v, silu); }

// Grid-stride cursor over (row, position-in-row, channel) without a 64-bit division per
// step: the stride is decomposed once per thread.
struct Cursor {
  uint64_t row, t, d;          // current row, index within the row, channel = row % dim
  uint64_t s_row, s_t, s_d;    // the grid stride as (rows, positions, channels)
  uint64_t per_row, dim;
  __device__ Cursor(uint64_t start, uint64_t stride, uint64_t per_row_, uint64_t dim_)
      : per_row(per_row_), dim(dim_) {
    row = start / per_row;
    t = start - row * per_row;
    d = row % dim;
    s_row = stride / per_row;
    s_t = stride - s_row * per_row;
    s_d = s_row % dim;
  }
  __device__ __forceinline__ void advance() {
    row += s_row;
    t += s_t;
    d += s_d;
    if (t >= per_row) {
      t -= per_row;
      ++row;
      ++d;
    }
    while (d >= dim) d -= dim;
  }
};

struct ConvArgs {
  const float* x;
  const float* w;     // [dim][W]
  const float* bias;  // [dim] or null
  float* u;
  uint64_t rows, dim, L;
  uint64_t g0, stride;
  int width;
  int silu;
  double* range;  // null: no epilogue
};

// Vector path (L % 4 == 0, 16-byte aligned x and u): one thread per run of QPT
// consecutive float4 quads of a row.  The causal halo (the last W-1 inputs before the
// run) is one extra float4 per run; inside the run it is carried in registers, and the
// channel's weights are loaded once per run.  All QPT loads are issued before any math.
template <int W, int QPT, int MODE>
__global__ void __launch_bounds__(kConvThreads) conv1d_vec_kernel(ConvArgs a) {
  range::Acc acc;
  const uint64_t qpr = a.L / 4;      // quads per row
  const uint64_t runs = qpr / QPT;   // runs per row
  const float4* x4 = reinterpret_cast<const float4*>(a.x);
  float4* u4 = reinterpret_cast<float4*>(a.u);
  for (Cursor c(static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x,
                static_cast<uint64_t>(gridDim.x) * blockDim.x, runs, a.dim);
       c.row < a.rows; c.advance()) {
    const uint64_t q0 = c.row * qpr + c.t * QPT;
    float4 in[QPT + 1];
    in[0] = c.t ? __ldg(x4 + q0 - 1) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int j = 0; j < QPT; ++j) in[j + 1] = __ldcs(x4 + q0 + j);
    float wk[W];
#pragma unroll
    for (int k = 0; k < W; ++k) wk[k] = __ldg(a.w + c.d * W + k);
    const float bias = a.bias ? __ldg(a.bias + c.d) : 0.f;
    const uint64_t gi0 = a.g0 + c.row * a.L + c.t * QPT * 4;
#pragma unroll
    for (int j = 0; j < QPT; ++j) {
      const float xs[8] = {in[j].x, in[j].y, in[j].z, in[j].w,
                           in[j + 1].x, in[j + 1].y, in[j + 1].z, in[j + 1].w};
      float o[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float s = bias;
#pragma unroll
        for (int k = 0; k < W; ++k) s = fmaf(wk[k], xs[4 + i - (W - 1) + k], s);
        o[i] = act(s, a.silu != 0);
      }
      __stcs(u4 + q0 + j, make_float4(o[0], o[1], o[2], o[3]));
      if (a.range) {
#pragma unroll
        for (int i = 0; i < 4; ++i) acc.visit(o[i], sampled<MODE>(gi0 + 4 * j + i, a.stride));
      }
    }
  }
  if (a.range) range::commit<kConvThreads>(acc, a.range);
}

// Warp-coalesced path (L a multiple of 128, 16-byte aligned x and u): a warp owns runs
// of kWQ consecutive 32-quad blocks of one row (2 KB of x per block group); lane l takes
// quad l of each block, so every load and store instruction covers 512 contiguous bytes.
// The causal halo of a quad (the previous quad's last W-1 inputs) comes from lane l-1 by
// shuffle, and from the previous block's lane 31 (or one load / the zero padding at the
// row start) for lane 0.
constexpr int kWQ = 4;  // 32-quad blocks per warp run (4 x 16 B in flight per lane)

template <int W, int MODE>
__global__ void __launch_bounds__(kConvThreads) conv1d_warp_kernel(ConvArgs a) {
  range::Acc acc;
  const int lane = threadIdx.x % 32;
  const uint64_t qpr = a.L / 4;                  // quads per row (a multiple of 32)
  const uint64_t runs_per_row = qpr / (32 * kWQ);  // whole runs per row
  const uint64_t tail_blocks = (qpr / 32) % kWQ;   // 32-quad blocks after the last run
  const uint64_t units_per_row = runs_per_row + (tail_blocks ? 1 : 0);
  const uint64_t units = a.rows * units_per_row;
  const float4* x4 = reinterpret_cast<const float4*>(a.x);
  float4* u4 = reinterpret_cast<float4*>(a.u);
  const uint64_t warps = static_cast<uint64_t>(gridDim.x) * (blockDim.x / 32);
  for (uint64_t unit = static_cast<uint64_t>(blockIdx.x) * (blockDim.x / 32) + threadIdx.x / 32;
       unit < units; unit += warps) {
    const uint64_t row = unit / units_per_row;
    const uint64_t ur = unit - row * units_per_row;
    const int nb = ur < runs_per_row ? kWQ : static_cast<int>(tail_blocks);
    const uint64_t qb = row * qpr + ur * 32 * kWQ;  // first quad of the run
    const uint64_t d = row % a.dim;
    float4 in[kWQ];
#pragma unroll
    for (int m = 0; m < kWQ; ++m)
      in[m] = m < nb ? __ldcs(x4 + qb + m * 32 + lane) : make_float4(0.f, 0.f, 0.f, 0.f);
    // halo of the run's first quad: the quad before it in the row (zero at the row start)
    float4 prev31 = make_float4(0.f, 0.f, 0.f, 0.f);
    if (ur > 0) prev31 = __ldg(x4 + qb - 1);
    float wk[W];
#pragma unroll
    for (int k = 0; k < W; ++k) wk[k] = __ldg(a.w + d * W + k);
    const float bias = a.bias ? __ldg(a.bias + d) : 0.f;
#pragma unroll
    for (int m = 0; m < kWQ; ++m) {
      if (m >= nb) break;
      // previous quad: lane-1's, or for lane 0 the last quad of the previous block
      float o[4];
      conv_block<W>(in[m], prev31, lane, wk, bias, a.silu != 0, o);
      const uint64_t q = qb + m * 32 + lane;
      __stcs(u4 + q, make_float4(o[0], o[1], o[2], o[3]));
      if (a.range) {
        const uint64_t gi = a.g0 + q * 4;
#pragma unroll
        for (int i = 0; i < 4; ++i) acc.visit(o[i], sampled<MODE>(gi + i, a.stride));
      }
    }
  }
  if (a.range) range::commit<kConvThreads>(acc, a.range);
}

// Scalar path: any L, any alignment, W <= 4.
template <int MODE>
__global__ void __launch_bounds__(kConvThreads) conv1d_scalar_kernel(ConvArgs a) {
  range::Acc acc;
  for (Cursor c(static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x,
                static_cast<uint64_t>(gridDim.x) * blockDim.x, a.L, a.dim);
       c.row < a.rows; c.advance()) {
    const uint64_t row = c.row, t = c.t, d = c.d;
    const uint64_t i = row * a.L + t;
    float s = a.bias ? a.bias[d] : 0.f;
    for (int k = 0; k < a.width; ++k) {
      const int64_t tt = static_cast<int64_t>(t) - (a.width - 1) + k;
      const float xv = tt >= 0 ? a.x[row * a.L + static_cast<uint64_t>(tt)] : 0.f;
      s = fmaf(a.w[d * a.width + k], xv, s);
    }
    const float o = act(s, a.silu != 0);
    a.u[i] = o;
    if (a.range) acc.visit(o, sampled<MODE>(a.g0 + i, a.stride));
  }
  if (a.range) range::commit<kConvThreads>(acc, a.range);
}

template <int W, int MODE>
void launch_vec(const ConvArgs& a, dim3 grid, cudaStream_t s) {
  if ((a.L / 4) % 4 == 0)
    conv1d_vec_kernel<W, 4, MODE><<<grid, kConvThreads, 0, s>>>(a);
  else
    conv1d_vec_kernel<W, 1, MODE><<<grid, kConvThreads, 0, s>>>(a);
}

template <int MODE>
cudaError_t launch_mode(const ConvArgs& a, bool vec, int num_sms, cudaStream_t s) {
  const uint64_t work = vec ? a.rows * (a.L / 4) : a.rows * a.L;
  uint64_t blocks = (work + kConvThreads - 1) / kConvThreads;
  const uint64_t cap = static_cast<uint64_t>(num_sms) * 8;  // 8 x 256 threads per SM
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  const dim3 grid(static_cast<unsigned>(blocks));
  if (!vec) {
    conv1d_scalar_kernel<MODE><<<grid, kConvThreads, 0, s>>>(a);
  } else if (a.L % 128 == 0) {
    switch (a.width) {
      case 1: conv1d_warp_kernel<1, MODE><<<grid, kConvThreads, 0, s>>>(a); break;
      case 2: conv1d_warp_kernel<2, MODE><<<grid, kConvThreads, 0, s>>>(a); break;
      case 3: conv1d_warp_kernel<3, MODE><<<grid, kConvThreads, 0, s>>>(a); break;
      default: conv1d_warp_kernel<4, MODE><<<grid, kConvThreads, 0, s>>>(a); break;
    }
  } else {
    switch (a.width) {
      case 1: launch_vec<1, MODE>(a, grid, s); break;
      case 2: launch_vec<2, MODE>(a, grid, s); break;
      case 3: launch_vec<3, MODE>(a, grid, s); break;
      default: launch_vec<4, MODE>(a, grid, s); break;
    }
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_conv1d_f32(const float* x, const float* w, const float* bias, float* u,
                              uint64_t batch, uint64_t dim, uint64_t L, int width, int silu,
                              uint64_t g0, uint64_t stride, double* d_range, int num_sms,
                              cudaStream_t s) {
  ConvArgs a{x, w, bias, u, batch * dim, dim, L, g0, stride, width, silu, d_range};
  if (a.rows * L == 0) return cudaSuccess;
  const bool vec = L % 4 == 0 && (reinterpret_cast<uintptr_t>(x) & 15u) == 0 &&
                   (reinterpret_cast<uintptr_t>(u) & 15u) == 0;
  if (stride == 1) return launch_mode<0>(a, vec, num_sms, s);
  if ((stride & (stride - 1)) == 0) return launch_mode<1>(a, vec, num_sms, s);
  return launch_mode<2>(a, vec, num_sms, s);
}

}  // namespace cl
