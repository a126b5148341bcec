// scan_mamba1.cu -- fused Mamba-1 selective scan for sm_100a (fp32).
//
// Semantics (mamba_ssm selective_scan_fn, the paper's kernel),
// recurrence core identical to chunklab::scan_window (scan.hpp:77-100) under the
// mapping a = exp(delta'*A), x = delta'*u, b/c = B/C (SURVEY.md finding 1):
//   delta' = softplus(delta + bias)            (identity above 20, mamba_ssm)
//   h_s    = exp(delta'*A[c,s]) * h_s + B[b,s,t] * (delta'*u)     s = 0..N-1
//   y      = (sum_s C[b,s,t]*h_s + D[c]*u) * z*sigmoid(z)
//
// Two kernels:
//   * rowseq_tma_kernel (the hot path, N = 16): one thread owns one (b, c) row
//     and keeps its 16 states in registers.  A warp owns a 32-row tile; each
//     warp runs its own 3-stage TMA pipeline (cp.async.bulk.tensor, 128B
//     swizzle) over 32-timestep boxes of u / delta / z and the tile's B / C
//     boxes, writes y in place of u and TMA-stores it.  Work items are
//     (row tile, L-segment) pairs with segment length = the chunk chosen by the
//     device rule (read from device memory, rounded up to whole boxes),
//     dispatched in segment-major order through an atomic ticket; the state
//     carry between consecutive segments of a tile is a chained scan (flag +
//     release/acquire), so chunking never changes a single floating-point
//     operation: outputs are bit-identical for every chunk size.
//   * generic_kernel: any N <= 64, any alignment; one thread per row, direct loads.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
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

__device__ __forceinline__ float softplus_f32(float x) {
  return x <= 20.f ? log1pf(__expf(x)) : x;
}

__device__ __forceinline__ float silu_f32(float z) { return __fdividef(z, 1.f + __expf(-z)); }

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
    if (a.softplus) dt = softplus_f32(dt);
    const float x = dt * u;
    float y = 0.f;
#pragma unroll
    for (int s = 0; s < (NS > 0 ? NS : 64); ++s) {
      if (s < N) {
        const float dA = ex2_approx(dt * A2[s]);
        h[s] = fmaf(dA, h[s], Bb[s * a.L + t] * x);
        y = fmaf(Cb[s * a.L + t], h[s], y);
      }
    }
    y = fmaf(Dc, u, y);
    if (a.z) y *= silu_f32(a.z[row * a.L + t]);
    a.out[row * a.L + t] = y;
  }
  if (a.h_last) {
#pragma unroll
    for (int s = 0; s < (NS > 0 ? NS : 64); ++s)
      if (s < N) a.h_last[row * N + s] = h[s];
  }
}

// ---------------------------------------------------------------------------
// TMA row-sequential kernel (N = 16)
// ---------------------------------------------------------------------------
constexpr int kN = 16;
constexpr int kBox = 32;       // timesteps per box (128 B rows, SWIZZLE_128B)
constexpr int kRows = 32;      // rows per tile = lanes per warp
constexpr int kWarps = 4;      // independent warps per CTA
constexpr int kStages = 3;
constexpr int kTileBytes = kRows * kBox * 4;  // 4 KB (u / delta / z / y)
constexpr int kBCBytes = kN * kBox * 4;       // 2 KB (B or C)
constexpr int kStageBytes = 3 * kTileBytes + 2 * kBCBytes;  // 16 KB
constexpr int kWarpBytes = kStages * kStageBytes + kTileBytes;  // 48 KB in + 4 KB y staging
constexpr size_t kTmaSmem = size_t(kWarps) * kWarpBytes + 1024 /*align*/ + 256 /*barriers*/;

struct TmaArgs {
  const float *A, *D, *bias, *h0;
  float* h_last;
  float* carry;            // [n_tiles][32][16]
  unsigned int* flags;     // [n_tiles] completed segments
  unsigned int* ticket;    // work counter
  uint64_t batch, dim, L;
  int tiles_per_batch;
  int n_tiles;
  int softplus;
  int has_z;
  const cl_decision* decision;
  int fixed_chunk;
};

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
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
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
__device__ __forceinline__ void bulk_wait_read_all() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
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

// 128B-swizzled float4 chunk j of row r inside a [32 rows x 32 floats] box.
__device__ __forceinline__ int swz(int r, int j) { return r * 128 + ((j ^ (r & 7)) << 4); }

struct Item {
  int tile, seg, nbox;
  int t0;
};

__global__ void __launch_bounds__(kWarps * 32, 1)
    rowseq_tma_kernel(const __grid_constant__ CUtensorMap map_u,
                      const __grid_constant__ CUtensorMap map_dt,
                      const __grid_constant__ CUtensorMap map_z,
                      const __grid_constant__ CUtensorMap map_out,
                      const __grid_constant__ CUtensorMap map_B,
                      const __grid_constant__ CUtensorMap map_C, TmaArgs a) {
  int status;
  const int chunk = read_chunk(a.decision, a.fixed_chunk, &status);
  if (status != 0) return;
  int seg_len = chunk < kBox ? kBox : chunk;
  seg_len = (seg_len + kBox - 1) / kBox * kBox;
  const int L = static_cast<int>(a.L);
  const int n_seg = (L + seg_len - 1) / seg_len;
  const int n_items = n_seg * a.n_tiles;

  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  unsigned char* wbase = smem + size_t(warp) * kWarpBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + size_t(kWarps) * kWarpBytes) + warp * 4;
  // per-slot metadata (item index, box) kept in registers of every lane
  int meta_item[kStages], meta_box[kStages];

  if (lane == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(bars + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (warp == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_u)));
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_dt)));
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_z)));
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_B)));
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_C)));
    }
  }
  __syncwarp();

  auto decode = [&](int id) {
    Item it;
    it.seg = id / a.n_tiles;
    it.tile = id % a.n_tiles;
    it.t0 = it.seg * seg_len;
    const int len = min(seg_len, L - it.t0);
    it.nbox = (len + kBox - 1) / kBox;
    return it;
  };
  auto claim = [&]() {
    int id = 0;
    if (lane == 0) id = static_cast<int>(atomicAdd(a.ticket, 1u));
    return __shfl_sync(0xffffffffu, id, 0);
  };

  // producer cursor
  int p_item = claim();
  int p_box = 0;
  auto produce = [&](int slot) {
    meta_item[slot] = -1;
    if (p_item >= n_items) return;
    const Item it = decode(p_item);
    meta_item[slot] = p_item;
    meta_box[slot] = p_box;
    if (lane == 0) {
      unsigned char* st = wbase + slot * kStageBytes;
      const int b = it.tile / a.tiles_per_batch;
      const int r0 = (it.tile % a.tiles_per_batch) * kRows;
      const int t = it.t0 + p_box * kBox;
      mbar_expect_tx(bars + slot, a.has_z ? kStageBytes : kStageBytes - kTileBytes);
      tma_load_3d(st, &map_u, t, r0, b, bars + slot);
      tma_load_3d(st + kTileBytes, &map_dt, t, r0, b, bars + slot);
      if (a.has_z) tma_load_3d(st + 2 * kTileBytes, &map_z, t, r0, b, bars + slot);
      tma_load_3d(st + 3 * kTileBytes, &map_B, t, 0, b, bars + slot);
      tma_load_3d(st + 3 * kTileBytes + kBCBytes, &map_C, t, 0, b, bars + slot);
    }
    if (++p_box == it.nbox) {
      p_box = 0;
      p_item = claim();
    }
  };

  for (int s = 0; s < kStages; ++s) produce(s);

  unsigned char* ybuf = wbase + kStages * kStageBytes;
  float h[kN], A2[kN];
  float bias = 0.f, Dc = 0.f;
  Item cur{};
  int row = 0;
  bool row_valid = false;
  for (int iter = 0;; ++iter) {
    const int slot = iter % kStages;
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
        A2[s] = q.x * kLog2e;
        A2[s + 1] = q.y * kLog2e;
        A2[s + 2] = q.z * kLog2e;
        A2[s + 3] = q.w * kLog2e;
      }
      bias = a.bias ? a.bias[cc] : 0.f;
      Dc = a.D ? a.D[cc] : 0.f;
      if (cur.seg == 0) {
#pragma unroll
        for (int s = 0; s < kN; ++s) h[s] = 0.f;
        if (a.h0) {
#pragma unroll
          for (int s = 0; s < kN; s += 4) {
            const float4 q = *reinterpret_cast<const float4*>(a.h0 + size_t(row) * kN + s);
            h[s] = q.x;
            h[s + 1] = q.y;
            h[s + 2] = q.z;
            h[s + 3] = q.w;
          }
        }
      } else {
        // chained carry from segment seg-1 of this tile
        if (lane == 0)
          while (ld_acquire(a.flags + cur.tile) < static_cast<unsigned>(cur.seg)) __nanosleep(64);
        __syncwarp();
        const float* cr = a.carry + (size_t(cur.tile) * kRows + lane) * kN;
#pragma unroll
        for (int s = 0; s < kN; s += 4) {
          const float4 q = __ldcg(reinterpret_cast<const float4*>(cr + s));
          h[s] = q.x;
          h[s + 1] = q.y;
          h[s + 2] = q.z;
          h[s + 3] = q.w;
        }
      }
    }

    mbar_wait(bars + slot, (iter / kStages) & 1);
    // the y staging buffer is free once the previous box's store has read it
    if (lane == 0) bulk_wait_read_all();
    __syncwarp();
    unsigned char* st = wbase + slot * kStageBytes;
    const float* sB = reinterpret_cast<const float*>(st + 3 * kTileBytes);
    const float* sC = reinterpret_cast<const float*>(st + 3 * kTileBytes + kBCBytes);
    const int tbox = cur.t0 + box * kBox;
    const int valid = min(kBox, L - tbox);  // multiple of 4 (L % 4 == 0)
    for (int j = 0; j < valid / 4; ++j) {
      const int off = swz(lane, j);
      const float4 u4 = *reinterpret_cast<const float4*>(st + off);
      const float4 d4 = *reinterpret_cast<const float4*>(st + kTileBytes + off);
      float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
      if (a.has_z) z4 = *reinterpret_cast<const float4*>(st + 2 * kTileBytes + off);
      const float uu[4] = {u4.x, u4.y, u4.z, u4.w};
      const float dd[4] = {d4.x, d4.y, d4.z, d4.w};
      const float zz[4] = {z4.x, z4.y, z4.z, z4.w};
      float yy[4];
      float4 Bq[kN], Cq[kN];
#pragma unroll
      for (int s = 0; s < kN; ++s) {
        Bq[s] = *reinterpret_cast<const float4*>(sB + s * kBox + 4 * j);
        Cq[s] = *reinterpret_cast<const float4*>(sC + s * kBox + 4 * j);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        float dt = dd[k] + bias;
        if (a.softplus) dt = softplus_f32(dt);
        const float x = dt * uu[k];
        float y = 0.f;
#pragma unroll
        for (int s = 0; s < kN; ++s) {
          const float bs = k == 0 ? Bq[s].x : (k == 1 ? Bq[s].y : (k == 2 ? Bq[s].z : Bq[s].w));
          const float cs = k == 0 ? Cq[s].x : (k == 1 ? Cq[s].y : (k == 2 ? Cq[s].z : Cq[s].w));
          const float dA = ex2_approx(dt * A2[s]);
          h[s] = fmaf(dA, h[s], bs * x);
          y = fmaf(cs, h[s], y);
        }
        y = fmaf(Dc, uu[k], y);
        if (a.has_z) y *= silu_f32(zz[k]);
        yy[k] = y;
      }
      *reinterpret_cast<float4*>(ybuf + off) = make_float4(yy[0], yy[1], yy[2], yy[3]);
    }
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) {
      const int b = cur.tile / a.tiles_per_batch;
      const int r0 = (cur.tile % a.tiles_per_batch) * kRows;
      tma_store_3d(&map_out, ybuf, tbox, r0, b);
    }

    if (box == cur.nbox - 1) {
      if (cur.seg == n_seg - 1) {
        if (a.h_last && row_valid) {
#pragma unroll
          for (int s = 0; s < kN; s += 4)
            *reinterpret_cast<float4*>(a.h_last + size_t(row) * kN + s) =
                make_float4(h[s], h[s + 1], h[s + 2], h[s + 3]);
        }
      } else {
        float* cw = a.carry + (size_t(cur.tile) * kRows + lane) * kN;
#pragma unroll
        for (int s = 0; s < kN; s += 4)
          __stcg(reinterpret_cast<float4*>(cw + s), make_float4(h[s], h[s + 1], h[s + 2], h[s + 3]));
        __threadfence();
        __syncwarp();
        if (lane == 0) st_release(a.flags + cur.tile, static_cast<unsigned>(cur.seg + 1));
      }
    }
    // every lane has consumed this slot: refill it for iteration iter + kStages
    produce(slot);
  }
  if (lane == 0) bulk_wait_all();
  __syncwarp();
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
              uint32_t box0, uint32_t box1, bool swizzle) {
  EncodeFn enc = get_encode();
  if (!enc) return false;
  const cuuint64_t dims[3] = {d0, d1, d2};
  const cuuint64_t strides[2] = {d0 * 4, d0 * d1 * 4};
  const cuuint32_t box[3] = {box0, box1, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box,
             estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
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

int ensure_scratch(cl_ctx* ctx, size_t work_bytes, size_t carry_bytes) {
  if (ctx->work_bytes < work_bytes) {
    if (ctx->d_work) cudaFree(ctx->d_work);
    ctx->d_work = nullptr;
    ctx->work_bytes = 0;
    cudaError_t e = cudaMalloc(&ctx->d_work, work_bytes);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMalloc(scan work)");
    ctx->work_bytes = work_bytes;
  }
  if (ctx->carry_bytes < carry_bytes) {
    if (ctx->d_carry) cudaFree(ctx->d_carry);
    ctx->d_carry = nullptr;
    ctx->carry_bytes = 0;
    cudaError_t e = cudaMalloc(&ctx->d_carry, carry_bytes);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMalloc(scan carry)");
    ctx->carry_bytes = carry_bytes;
  }
  return CL_OK;
}

}  // namespace

int scan_mamba1(cl_ctx* ctx, const cl_mamba1_args& a, const cl_decision* d_decision,
                int fixed_chunk, int variant, cudaStream_t s) {
  const bool tma_ok = tma_eligible(a);
  if (variant == CL_SCAN_ROWSEQ_TMA && !tma_ok)
    return fail(ctx, CL_E_INVALID, "scan variant rowseq_tma needs d_state 16, L % 4 == 0 and 16-byte aligned buffers");
  const bool use_tma = variant == CL_SCAN_ROWSEQ_TMA || (variant == CL_SCAN_AUTO && tma_ok);
  if (use_tma) {
    CUtensorMap mu, mdt, mz, mout, mB, mC;
    const uint64_t L = a.seq_len, D = a.dim, Bt = a.batch;
    bool ok = make_map(&mu, a.u, L, D, Bt, kBox, kRows, true) &&
              make_map(&mdt, a.delta, L, D, Bt, kBox, kRows, true) &&
              make_map(&mout, a.out, L, D, Bt, kBox, kRows, true) &&
              make_map(&mB, a.B, L, kN, Bt, kBox, kN, false) &&
              make_map(&mC, a.C, L, kN, Bt, kBox, kN, false);
    if (ok) ok = make_map(&mz, a.z ? a.z : a.u, L, D, Bt, kBox, kRows, true);
    if (!ok) return fail(ctx, CL_E_CUDA, "cuTensorMapEncodeTiled failed");
    const int tiles_per_batch = static_cast<int>((D + kRows - 1) / kRows);
    const int n_tiles = tiles_per_batch * static_cast<int>(Bt);
    const size_t work_bytes = (size_t(n_tiles) + 32) * sizeof(unsigned int);
    const size_t carry_bytes = size_t(n_tiles) * kRows * kN * sizeof(float);
    int rc = ensure_scratch(ctx, work_bytes, carry_bytes);
    if (rc) return rc;
    cudaError_t e = cudaMemsetAsync(ctx->d_work, 0, work_bytes, s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMemsetAsync(scan work)");
    TmaArgs t{};
    t.A = a.A;
    t.D = a.D;
    t.bias = a.delta_bias;
    t.h0 = a.h0;
    t.h_last = a.h_last;
    t.carry = ctx->d_carry;
    t.ticket = ctx->d_work;
    t.flags = ctx->d_work + 32;
    t.batch = Bt;
    t.dim = D;
    t.L = L;
    t.tiles_per_batch = tiles_per_batch;
    t.n_tiles = n_tiles;
    t.softplus = a.delta_softplus;
    t.has_z = a.z != nullptr;
    t.decision = d_decision;
    t.fixed_chunk = fixed_chunk;
    static bool attr = false;
    if (!attr) {
      e = cudaFuncSetAttribute(rowseq_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(kTmaSmem));
      if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaFuncSetAttribute(rowseq_tma)");
      attr = true;
    }
    // persistent: one CTA (4 independent warps) per SM, capped by the tile count
    int grid = ctx->num_sms;
    const int max_useful = (n_tiles + kWarps - 1) / kWarps;
    if (max_useful < grid) grid = max_useful < 1 ? 1 : max_useful;
    rowseq_tma_kernel<<<grid, kWarps * 32, kTmaSmem, s>>>(mu, mdt, mz, mout, mB, mC, t);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(ctx, e, "rowseq_tma_kernel launch");
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

}  // namespace cl
