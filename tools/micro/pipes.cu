// Microbenchmark: sustained MUFU.EX2 / FFMA2 / FFMA throughput and mixes on one B200.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipes pipes.cu
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) { u64 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }

// M = MUFU per iteration, F = FFMA2 per iteration, S = scalar FFMA per iteration; 8 independent chains
template <int M, int F, int S>
__global__ void kern(float* out, int iters) {
  float a[8]; u64 b[8]; float c[8];
  for (int i = 0; i < 8; ++i) { a[i] = -0.001f * (threadIdx.x + i); b[i] = (u64)__float_as_uint(1.0f + 1e-7f * i) | ((u64)__float_as_uint(1.0f) << 32); c[i] = 1.0f + i * 1e-6f; }
  const u64 m = (u64)__float_as_uint(0.9999f) | ((u64)__float_as_uint(0.9999f) << 32);
  const u64 ad = (u64)__float_as_uint(1e-6f) | ((u64)__float_as_uint(1e-6f) << 32);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
#pragma unroll
      for (int q = 0; q < M; ++q) a[k] = ex2(a[k]) - 1.0f;
#pragma unroll
      for (int q = 0; q < F; ++q) b[k] = fma2(b[k], m, ad);
#pragma unroll
      for (int q = 0; q < S; ++q) c[k] = fmaf(c[k], 0.9999f, 1e-6f);
    }
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i] + __uint_as_float((unsigned)b[i]) + c[i];
  if (s == 12345.f) out[0] = s;
}

template <int M, int F, int S>
void run(const char* name, int threads) {
  float* d; cudaMalloc(&d, 4);
  int iters = 4000;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<M, F, S><<<148 * 4, threads>>>(d, 10);
  cudaEventRecord(e0);
  kern<M, F, S><<<148 * 4, threads>>>(d, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double warps = 148.0 * 4 * threads / 32;
  double per_sm_cycle = 1.965e9 * ms / 1e3;  // assume max clock
  double lanes = warps * 32 * iters * 8.0;
  printf("%-26s thr=%4d  %8.3f ms  MUFU/clk/SM=%6.2f  FFMA2/clk/SM=%6.2f (lane-pairs)  FFMA/clk/SM=%6.2f\n", name, threads, ms,
         lanes * M / per_sm_cycle / 148, lanes * F / per_sm_cycle / 148, lanes * S / per_sm_cycle / 148);
}
int main() {
  for (int t : {128, 256}) {
    run<1, 0, 0>("mufu only", t);
    run<0, 1, 0>("ffma2 only", t);
    run<0, 0, 1>("ffma only", t);
    run<1, 2, 0>("1 mufu : 2 ffma2", t);
    run<1, 3, 0>("1 mufu : 3 ffma2", t);
    run<1, 4, 0>("1 mufu : 4 ffma2", t);
    run<1, 0, 4>("1 mufu : 4 ffma", t);
    run<1, 0, 8>("1 mufu : 8 ffma", t);
  }
  return 0;
}
