// Latency probe of the decision's parts on one CTA (clock64 segments): fp64 terms
// p*log(p+eps) by 256 threads, the in-order 256-term fp64 subtraction chain by one thread,
// and the rule's log2 / exp2.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 decide_lat.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(const unsigned long long* counts, double n, double* out, long long* t) {
  __shared__ double terms[256];
  long long t0 = clock64();
  const double inv_n = __ddiv_rn(1.0, n);
  const double pm = __dmul_rn(static_cast<double>(__ldcg(counts + threadIdx.x)), inv_n);
  terms[threadIdx.x] = pm > 0.0 ? __dmul_rn(pm, log(__dadd_rn(pm, 1e-12))) : 0.0;
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) {
    double raw = 0.0;
#pragma unroll 8
    for (int i = 0; i < 256; ++i) raw = __dsub_rn(raw, terms[i]);
    long long t2 = clock64();
    const double l2 = log2(__dadd_rn(32.0, raw * 100.0));
    const double e = floor(l2 + 0.5);
    const double p2 = exp2(e);
    long long t3 = clock64();
    out[0] = raw + p2;
    t[0] = t1 - t0; t[1] = t2 - t1; t[2] = t3 - t2;
  }
}
int main() {
  unsigned long long h[256];
  for (int i = 0; i < 256; ++i) h[i] = 1000 + i * 37;
  unsigned long long* d; double* o; long long* t;
  cudaMalloc(&d, sizeof h); cudaMalloc(&o, 8); cudaMalloc(&t, 24);
  cudaMemcpy(d, h, sizeof h, cudaMemcpyHostToDevice);
  for (int r = 0; r < 3; ++r) {
    probe<<<1, 256>>>(d, 1e6, o, t);
    long long ht[3];
    cudaMemcpy(ht, t, 24, cudaMemcpyDeviceToHost);
    printf("terms %lld cycles, chain %lld cycles, rule %lld cycles\n", ht[0], ht[1], ht[2]);
  }
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int r = 0; r < 100; ++r) probe<<<1, 256>>>(d, 1e6, o, t);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("back-to-back launch %.2f us\n", ms * 10);
  return 0;
}
