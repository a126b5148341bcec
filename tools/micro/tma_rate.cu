// Microbenchmark: TMA op throughput per SM for small boxes (the scan's access shape).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_rate tma_rate.cu -lcuda
//
// Each warp's lane 0 streams `ops` loads through a STAGES-deep smem ring (mbarrier per
// slot) over its own rows of a (rows x L) fp32 tensor, like the scan's per-warp ring.
// Reports ops/us/SM and GB/s.  Modes:
//   0: 3-D tensor box  R rows x 16 fp32 (64 B rows)
//   1: 1-D bulk copy   R x 64 bytes contiguous
//   2: 3-D tensor box  R rows x 32 fp32 (128 B rows)
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE, int R, int STAGES>
__global__ void kern(const __grid_constant__ CUtensorMap map, const float* src, int L, int rows,
                     int ops, int warps) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = sm + ((1024u - (sa(sm) & 1023u)) & 1023u);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  constexpr int kBytes = MODE == 2 ? R * 128 : R * 64;
  unsigned char* ring = base + warp * STAGES * kBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + warps * STAGES * kBytes) + warp * STAGES;
  if (lane == 0)
    for (int s = 0; s < STAGES; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(bars + s)));
  __syncwarp();
  const int gw = blockIdx.x * warps + warp;
  const int row0 = (gw * R) % rows;
  const int tstep = MODE == 2 ? 32 : 16;
  for (int i = 0; i < ops; ++i) {
    const int s = i % STAGES;
    if (i >= STAGES) {
      const uint32_t par = ((i / STAGES) - 1) & 1;
      asm volatile(
          "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
              sa(bars + s)),
          "r"(par)
          : "memory");
    }
    __syncwarp();
    if (lane == 0) {
      const int t = (i * tstep) % L;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(bars + s)),
                   "r"(kBytes)
                   : "memory");
      if (MODE == 1) {
        const float* g = src + (size_t(row0) * L + size_t(i) * R * 16) % (size_t(rows) * L);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                sa(ring + s * kBytes)),
            "l"(g), "r"(kBytes), "r"(sa(bars + s))
            : "memory");
      } else {
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
                sa(ring + s * kBytes)),
            "l"(reinterpret_cast<uint64_t>(&map)), "r"(t), "r"(row0), "r"(0), "r"(sa(bars + s))
            : "memory");
      }
    }
  }
  for (int i = ops; i < ops + STAGES; ++i) {
    const int s = i % STAGES;
    const uint32_t par = ((i / STAGES) - 1) & 1;
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
            sa(bars + s)),
        "r"(par)
        : "memory");
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);

template <int MODE, int R, int STAGES>
void run(const char* name, float* d, int L, int rows, int warps, int ops, EncodeFn enc) {
  CUtensorMap m;
  const uint32_t bx = MODE == 2 ? 32 : 16;
  cuuint64_t dims[3] = {(cuuint64_t)L, (cuuint64_t)rows, 1};
  cuuint64_t str[2] = {(cuuint64_t)L * 4, (cuuint64_t)L * rows * 4};
  cuuint32_t box[3] = {bx, R, 1}, es[3] = {1, 1, 1};
  enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      MODE == 2 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  constexpr int kBytes = MODE == 2 ? R * 128 : R * 64;
  const size_t smem = size_t(warps) * STAGES * kBytes + 1024 + warps * STAGES * 8;
  cudaFuncSetAttribute(kern<MODE, R, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<MODE, R, STAGES><<<148, warps * 32, smem>>>(m, d, L, rows, 8, warps);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<MODE, R, STAGES><<<148, warps * 32, smem>>>(m, d, L, rows, ops, warps);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double nops = 148.0 * warps * ops;
  printf("%-28s warps %2d stages %d rows %5d: %.3f ms  %.1f ops/us/SM  %.0f GB/s  (%s)\n", name,
         warps, STAGES, rows, ms, nops / (ms * 1e3) / 148, nops * kBytes / (ms * 1e6),
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  const int L = 8192;
  float* d;
  const int big_rows = 32768;  // 1 GiB: DRAM-resident
  cudaMalloc(&d, size_t(big_rows) * L * 4);
  cudaMemset(d, 0, size_t(big_rows) * L * 4);
  for (int rows : {big_rows, 512}) {  // 512 rows = 16 MiB: L2-resident
    for (int w : {4, 8, 14}) {
      run<0, 16, 2>("tensor 16x64B", d, L, rows, w, 2000, enc);
      run<1, 16, 2>("bulk1d 1KB", d, L, rows, w, 2000, enc);
      run<2, 16, 2>("tensor 16x128B", d, L, rows, w, 2000, enc);
      run<0, 16, 6>("tensor 16x64B", d, L, rows, w, 2000, enc);
    }
  }
  return 0;
}
