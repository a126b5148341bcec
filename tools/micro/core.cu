// Register-only replica of the scan's core per lane: 8 state pairs x T timesteps per
// iteration: arg = A2*dt (FMUL2), dA = 2x MUFU.EX2, bx = B*x (FMUL2), h = dA*h + bx (FFMA2),
// y += C*h (FFMA2).  Variants: ORDER 0 = per-timestep (as written in the kernel),
// ORDER 1 = all MUFU for T timesteps first.  Reports MUFU/clk/SM.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ u64 pk(float a, float b) { u64 r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ void upk(u64 v, float& a, float& b) { asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); }
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) { u64 r; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
__device__ __forceinline__ u64 mul2(u64 a, u64 b) { u64 r; asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ u64 add2(u64 a, u64 b) { u64 r; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }

template <int P, int T, int ORDER, int SMEM = 0>
__global__ void __launch_bounds__(256) core(float* out, int iters, float seed) {
  __shared__ __align__(16) float sBC[2][64][16];
  for (int i = threadIdx.x; i < 2 * 64 * 16; i += blockDim.x) (&sBC[0][0][0])[i] = 0.01f * (i % 37);
  __syncthreads();
  u64 h[P], A[P], Bv[P], Cv[P];
  for (int i = 0; i < P; ++i) {
    h[i] = pk(0.f, 0.f);
    A[i] = pk(-1.4f * (i + 1), -1.5f * (i + 1));
    Bv[i] = pk(0.3f + i * 0.01f, 0.2f);
    Cv[i] = pk(0.1f, 0.2f - i * 0.01f);
  }
  float dt = 0.01f + threadIdx.x * 1e-5f + seed, x = 0.5f;
  float yacc = 0.f;
  for (int it = 0; it < iters; ++it) {
    float dts[T], xs[T];
#pragma unroll
    for (int k = 0; k < T; ++k) { dts[k] = dt + k * 1e-4f; xs[k] = x - k * 1e-3f; }
    if (ORDER == 1) {
      u64 dA[T][P];
#pragma unroll
      for (int k = 0; k < T; ++k)
#pragma unroll
        for (int i = 0; i < P; ++i) {
          float a, b; upk(mul2(A[i], pk(dts[k], dts[k])), a, b); dA[k][i] = pk(ex2(a), ex2(b));
        }
#pragma unroll
      for (int k = 0; k < T; ++k) {
        u64 ya = 0, yb = 0;
#pragma unroll
        for (int i = 0; i < P; i += 2) {
          h[i] = fma2(dA[k][i], h[i], mul2(Bv[i], pk(xs[k], xs[k])));
          h[i + 1] = fma2(dA[k][i + 1], h[i + 1], mul2(Bv[i + 1], pk(xs[k], xs[k])));
          ya = fma2(Cv[i], h[i], ya); yb = fma2(Cv[i + 1], h[i + 1], yb);
        }
        float a, b; upk(add2(ya, yb), a, b); yacc += a + b;
      }
    } else {
#pragma unroll
      for (int k = 0; k < T; ++k) {
        u64 ya = 0, yb = 0;
        if (SMEM) {
          const int t = (it * T + k) & 63;
          const ulonglong2* Bq = reinterpret_cast<const ulonglong2*>(&sBC[0][t][0]);
          const ulonglong2* Cq = reinterpret_cast<const ulonglong2*>(&sBC[1][t][0]);
#pragma unroll
          for (int q = 0; q < P / 2; ++q) { ulonglong2 b = Bq[q], c = Cq[q]; Bv[2*q] = b.x; Bv[2*q+1] = b.y; Cv[2*q] = c.x; Cv[2*q+1] = c.y; }
        }
#pragma unroll
        for (int i = 0; i < P; i += 2) {
          float a0, b0, a1, b1;
          upk(mul2(A[i], pk(dts[k], dts[k])), a0, b0);
          upk(mul2(A[i + 1], pk(dts[k], dts[k])), a1, b1);
          h[i] = fma2(pk(ex2(a0), ex2(b0)), h[i], mul2(Bv[i], pk(xs[k], xs[k])));
          h[i + 1] = fma2(pk(ex2(a1), ex2(b1)), h[i + 1], mul2(Bv[i + 1], pk(xs[k], xs[k])));
          ya = fma2(Cv[i], h[i], ya); yb = fma2(Cv[i + 1], h[i + 1], yb);
        }
        float a, b; upk(add2(ya, yb), a, b); yacc += a + b;
      }
    }
    dt += 1e-7f; x *= 0.9999f;
  }
  float s = yacc; for (int i = 0; i < P; ++i) { float a, b; upk(h[i], a, b); s += a + b; }
  if (s == 1234.5f) out[0] = s;
}

template <int P, int T, int ORDER, int SMEM = 0>
void run(const char* name, int threads, int blocks_per_sm) {
  float* d; cudaMalloc(&d, 4);
  const int iters = 2000;
  core<P, T, ORDER, SMEM><<<148 * blocks_per_sm, threads>>>(d, 5, 0.f);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  core<P, T, ORDER, SMEM><<<148 * blocks_per_sm, threads>>>(d, iters, 0.f);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double mufu = 148.0 * blocks_per_sm * threads * (double)iters * T * P * 2;
  printf("%-22s P=%d T=%d warps/SM=%2d  %.3f ms  MUFU/clk/SM=%5.2f\n", name, P, T,
         threads / 32 * blocks_per_sm, ms, mufu / (ms * 1e-3 * 1.965e9) / 148);
}
int main() {
  run<8, 4, 0, 0>("row regs-BC", 128, 2);
  run<8, 4, 0, 1>("row smem-BC", 128, 2);
  run<4, 4, 0, 0>("pair regs-BC", 128, 4);
  run<4, 4, 0, 1>("pair smem-BC", 128, 4);
  run<8, 4, 0, 1>("row smem-BC", 128, 1);
  return 0;
  run<16, 4, 0>("2row, per-timestep", 128, 1);
  run<16, 4, 1>("2row, MUFU-first", 128, 1);
  run<16, 4, 0>("2row, per-timestep", 128, 2);
  run<8, 8, 0>("row T8, per-timestep", 128, 2);
  run<8, 8, 1>("row T8, MUFU-first", 128, 2);
  return 0;
  for (int wps : {4, 8, 12, 16}) {
    run<4, 4, 0>("pair, per-timestep", 128, wps / 4);
    run<4, 4, 1>("pair, MUFU-first", 128, wps / 4);
    run<8, 4, 0>("row, per-timestep", 128, wps / 4);
    run<8, 4, 1>("row, MUFU-first", 128, wps / 4);
  }
  return 0;
}
