// scan_f64.cu -- fp64 reference-mode recurrence on sm_100a, bit-identical to
// chunklab::scan_sequential / scan_chunked (proj/include/chunklab/scan.hpp:77-136).
//
// One thread per channel walks t in order; per (t, c) the state lanes are
// updated in s order with the reference's exact operation sequence
//     h = a*h + b*x ;  out += c*h ;  y = out + d*x
// using __dmul_rn/__dadd_rn so nvcc cannot contract into FMA (the reference's
// x86-64 build has no FMA, SURVEY.md finding 3).  Channels are independent in
// scan_window (the c loop carries nothing), so running them in parallel does
// not change any per-element operation order.  Chunking repartitions the t
// loop only; the carried state is the same registers, so chunked == sequential.
#include <cuda_runtime.h>

#include "cl_internal.h"

namespace cl {
namespace {

struct F64Args {
  uint64_t channels, n, L;
  const double *a, *b, *c, *d, *x;
  int at, bt, ct;
  const double* h0;
  double* y;
  double* h;
};

__device__ __forceinline__ void window_step(const F64Args& p, uint64_t ch, uint64_t t,
                                            double* h) {
  const uint64_t n = p.n;
  const double* a_ct = p.at ? p.a + (t * p.channels + ch) * n : p.a + ch * n;
  const double* b_t = p.bt ? p.b + t * n : p.b;
  const double* c_t = p.ct ? p.c + t * n : p.c;
  const double x = p.x[ch * p.L + t];
  double out = 0.0;
  for (uint64_t s = 0; s < n; ++s) {
    h[s] = __dadd_rn(__dmul_rn(a_ct[s], h[s]), __dmul_rn(b_t[s], x));
    out = __dadd_rn(out, __dmul_rn(c_t[s], h[s]));
  }
  p.y[ch * p.L + t] = __dadd_rn(out, __dmul_rn(p.d[ch], x));
}

// Register-resident state for the common small N; generic N keeps the state in
// the output buffer (global, L1-resident).
template <int N>
__global__ void scan_f64_kernel(F64Args p, uint64_t chunk) {
  const uint64_t ch = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (ch >= p.channels) return;
  if constexpr (N > 0) {
    double h[N];
#pragma unroll
    for (int s = 0; s < N; ++s) h[s] = p.h0 ? p.h0[ch * N + s] : 0.0;
    for (uint64_t t0 = 0; t0 < p.L; t0 += chunk) {
      const uint64_t t1 = t0 + chunk < p.L ? t0 + chunk : p.L;
      for (uint64_t t = t0; t < t1; ++t) {
        const double* a_ct = p.at ? p.a + (t * p.channels + ch) * N : p.a + ch * N;
        const double* b_t = p.bt ? p.b + t * N : p.b;
        const double* c_t = p.ct ? p.c + t * N : p.c;
        const double x = p.x[ch * p.L + t];
        double out = 0.0;
#pragma unroll
        for (int s = 0; s < N; ++s) {
          h[s] = __dadd_rn(__dmul_rn(a_ct[s], h[s]), __dmul_rn(b_t[s], x));
          out = __dadd_rn(out, __dmul_rn(c_t[s], h[s]));
        }
        p.y[ch * p.L + t] = __dadd_rn(out, __dmul_rn(p.d[ch], x));
      }
    }
#pragma unroll
    for (int s = 0; s < N; ++s) p.h[ch * N + s] = h[s];
  } else {
    double* h = p.h + ch * p.n;
    for (uint64_t s = 0; s < p.n; ++s) h[s] = p.h0 ? p.h0[ch * p.n + s] : 0.0;
    for (uint64_t t0 = 0; t0 < p.L; t0 += chunk) {
      const uint64_t t1 = t0 + chunk < p.L ? t0 + chunk : p.L;
      for (uint64_t t = t0; t < t1; ++t) window_step(p, ch, t, h);
    }
  }
}

}  // namespace

cudaError_t launch_scan_f64(const cl_scan_params_f64& q, const double* d_h0, uint64_t chunk,
                            double* d_y, double* d_h, cudaStream_t s) {
  F64Args p;
  p.channels = q.channels;
  p.n = q.state_dim;
  p.L = q.seq_len;
  p.a = q.a;
  p.b = q.b;
  p.c = q.c;
  p.d = q.d;
  p.x = q.x;
  p.at = q.a_len == q.seq_len * q.channels * q.state_dim;
  p.bt = q.b_len == q.seq_len * q.state_dim;
  p.ct = q.c_len == q.seq_len * q.state_dim;
  p.h0 = d_h0;
  p.y = d_y;
  p.h = d_h;
  if (chunk == 0) chunk = q.seq_len;
  const int threads = 64;
  const unsigned grid = static_cast<unsigned>((q.channels + threads - 1) / threads);
  switch (q.state_dim) {
    case 1: scan_f64_kernel<1><<<grid, threads, 0, s>>>(p, chunk); break;
    case 2: scan_f64_kernel<2><<<grid, threads, 0, s>>>(p, chunk); break;
    case 4: scan_f64_kernel<4><<<grid, threads, 0, s>>>(p, chunk); break;
    case 8: scan_f64_kernel<8><<<grid, threads, 0, s>>>(p, chunk); break;
    case 16: scan_f64_kernel<16><<<grid, threads, 0, s>>>(p, chunk); break;
    default: scan_f64_kernel<0><<<grid, threads, 0, s>>>(p, chunk); break;
  }
  return cudaGetLastError();
}

}  // namespace cl
