// Concurrency contract of the drop-in (reference SPEC.md:86: every function is pure and
// "safely shareable across threads"): the drop-in routes all calls through one
// process-wide context, so
//   (1) compute_histogram / estimate_entropy / scan_chunked from 4 host threads at once
//       must return exactly what a single thread computes, and
//   (2) two prefills (entropy -> device rule -> fused scan) on two CUDA streams of that
//       one context, in flight at the same time, must produce the bits each produces
//       alone (per-stream workspaces: scan work ticket, tagged carry, B/C transpose,
//       fused-histogram arrival ticket).
// Exit code 0 and "threads ok" on success.
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

#include "chunklab/chunk.hpp"
#include "chunklab/entropy.hpp"
#include "chunklab/mamba1.hpp"
#include "chunklab/scan.hpp"
#include "chunklab/synthetic.hpp"

using namespace chunklab;

static int g_fail = 0;
#define EXPECT(c)                                                        \
  do {                                                                   \
    if (!(c)) {                                                          \
      ++g_fail;                                                          \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);           \
    }                                                                    \
  } while (0)

static void cuda_ok(cudaError_t e) {
  if (e != cudaSuccess) {
    std::printf("CUDA error: %s\n", cudaGetErrorString(e));
    std::exit(2);
  }
}

struct HostCase {
  ActivationTensor t;
  HistogramSpec spec;
  Histogram h;
  EntropyEstimate e;
  ScanParams p;
  std::vector<double> y, hl;
};

static void host_threads() {
  constexpr int kThreads = 4, kIters = 6;
  std::vector<HostCase> cases(kThreads);
  for (int i = 0; i < kThreads; ++i) {
    SyntheticSpec syn;
    syn.distribution = i % 2 ? Distribution::StandardNormal : Distribution::Laplace;
    syn.seed = 100 + i;
    syn.shape = {64, 1000 + 37 * i};
    cases[i].t = generate_activations(syn);
    cases[i].spec.sample_stride = 1 + i;  // strided and unstrided calls interleave
    cases[i].h = compute_histogram(cases[i].t, cases[i].spec);
    cases[i].e = estimate_entropy(cases[i].h, cases[i].spec.epsilon);
    cases[i].p = random_scan_params(7 + i, 8, 4, 300 + 50 * i, true);
    auto [o, st] = scan_chunked(cases[i].p, ScanState{}, 64);
    cases[i].y = o.y;
    cases[i].hl = st.h;
  }
  std::atomic<int> mismatches{0};
  std::vector<std::thread> th;
  for (int i = 0; i < kThreads; ++i) {
    th.emplace_back([&, i] {
      for (int it = 0; it < kIters; ++it) {
        const HostCase& c = cases[i];
        const Histogram h = compute_histogram(c.t, c.spec);
        const EntropyEstimate e = estimate_entropy(h, c.spec.epsilon);
        if (h.masses != c.h.masses || h.lo != c.h.lo || h.hi != c.h.hi ||
            h.sample_count != c.h.sample_count || e.raw_nats != c.e.raw_nats)
          ++mismatches;
        auto [o, st] = scan_chunked(c.p, ScanState{}, 64);
        if (o.y != c.y || st.h != c.hl) ++mismatches;
        // error strings stay per thread while other threads succeed
        try {
          compute_histogram(ActivationTensor{{1.0, std::nan("")}, {2}}, c.spec);
          ++mismatches;
        } catch (const invalid_input& ex) {
          if (std::strcmp(ex.what(), "non-finite input") != 0) ++mismatches;
        }
      }
    });
  }
  for (auto& t : th) t.join();
  EXPECT(mismatches.load() == 0);
  std::printf("host threads: %d threads x %d iterations, %d mismatches\n", kThreads, kIters,
              mismatches.load());
}

struct Layer {
  std::vector<float> u, dt, A, B, C, D, z, bias;
  uint64_t batch, dim, L;
  float *du, *ddt, *dA, *dB, *dC, *dD, *dz, *dbias, *dout, *dh;
  void make(uint64_t b, uint64_t d, uint64_t l, unsigned seed) {
    batch = b, dim = d, L = l;
    std::mt19937_64 g(seed);
    std::normal_distribution<float> n01;
    std::uniform_real_distribution<float> un(-1.f, 1.f);
    auto fill = [&](std::vector<float>& v, size_t n, float scale) {
      v.resize(n);
      for (auto& x : v) x = scale * n01(g);
    };
    fill(u, b * d * l, 1.f);
    fill(dt, b * d * l, 0.1f);
    fill(B, b * 16 * l, 1.f);
    fill(C, b * 16 * l, 1.f);
    fill(z, b * d * l, 1.f);
    A.resize(d * 16);
    for (uint64_t c = 0; c < d; ++c)
      for (int s = 0; s < 16; ++s) A[c * 16 + s] = -(s + 1) * (1.f + 0.1f * un(g));
    D.resize(d);
    bias.resize(d);
    for (uint64_t c = 0; c < d; ++c) {
      D[c] = 1.f + 0.1f * n01(g);
      const float t = std::exp(std::log(1e-3f) + (un(g) + 1.f) * 0.5f * std::log(100.f));
      bias[c] = std::log(std::expm1(t));
    }
    auto up = [](const std::vector<float>& v, float** p) {
      cuda_ok(cudaMalloc(p, v.size() * 4));
      cuda_ok(cudaMemcpy(*p, v.data(), v.size() * 4, cudaMemcpyHostToDevice));
    };
    up(u, &du), up(dt, &ddt), up(A, &dA), up(B, &dB), up(C, &dC), up(D, &dD), up(z, &dz);
    up(bias, &dbias);
    cuda_ok(cudaMalloc(&dout, b * d * l * 4));
    cuda_ok(cudaMalloc(&dh, b * d * 16 * 4));
  }
  Mamba1Args args() const {
    Mamba1Args a{};
    a.u = du, a.delta = ddt, a.A = dA, a.B = dB, a.C = dC, a.D = dD, a.z = dz;
    a.delta_bias = dbias, a.out = dout, a.h_last = dh;
    a.batch = batch, a.dim = dim, a.seq_len = L, a.d_state = 16, a.delta_softplus = 1;
    return a;
  }
  std::vector<float> out() const {
    std::vector<float> y(batch * dim * L + batch * dim * 16);
    cuda_ok(cudaMemcpy(y.data(), dout, batch * dim * L * 4, cudaMemcpyDeviceToHost));
    cuda_ok(cudaMemcpy(y.data() + batch * dim * L, dh, batch * dim * 16 * 4,
                       cudaMemcpyDeviceToHost));
    return y;
  }
};

static void two_streams() {
  // two shapes that take different scan kernels (few tiles / many tiles) and different
  // segment counts, so a shared ticket or carry would be visible
  Layer a, b;
  a.make(1, 768, 2048, 1);
  b.make(4, 1024, 1024, 2);
  HistogramSpec spec;
  Prefill pa(spec, nullptr, ChunkBounds{32, 512}, CalibrationRef::log_k(256));
  Prefill pb(spec, nullptr, ChunkBounds{32, 512}, CalibrationRef::log_k(256));
  cudaStream_t sa, sb;
  cuda_ok(cudaStreamCreateWithFlags(&sa, cudaStreamNonBlocking));
  cuda_ok(cudaStreamCreateWithFlags(&sb, cudaStreamNonBlocking));
  // alone
  pa.run(a.args(), sa);
  cuda_ok(cudaStreamSynchronize(sa));
  const std::vector<float> ya = a.out();
  const int ca = pa.decision().chunk;
  pb.run(b.args(), sb);
  cuda_ok(cudaStreamSynchronize(sb));
  const std::vector<float> yb = b.out();
  const int cb = pb.decision().chunk;
  // together, many times
  int bad = 0;
  for (int it = 0; it < 20; ++it) {
    cuda_ok(cudaMemset(a.dout, 0, a.batch * a.dim * a.L * 4));
    cuda_ok(cudaMemset(b.dout, 0, b.batch * b.dim * b.L * 4));
    pa.run(a.args(), sa);
    pb.run(b.args(), sb);
    cuda_ok(cudaStreamSynchronize(sa));
    cuda_ok(cudaStreamSynchronize(sb));
    if (a.out() != ya || b.out() != yb || pa.decision().chunk != ca || pb.decision().chunk != cb)
      ++bad;
  }
  EXPECT(bad == 0);
  std::printf("two streams: 20 concurrent prefill pairs, %d differ from the lone runs\n", bad);
  // the same from two host threads, each driving its own stream
  bad = 0;
  std::atomic<int> tbad{0};
  std::thread t1([&] {
    for (int it = 0; it < 10; ++it) {
      pa.run(a.args(), sa);
      cuda_ok(cudaStreamSynchronize(sa));
      if (a.out() != ya) ++tbad;
    }
  });
  std::thread t2([&] {
    for (int it = 0; it < 10; ++it) {
      pb.run(b.args(), sb);
      cuda_ok(cudaStreamSynchronize(sb));
      if (b.out() != yb) ++tbad;
    }
  });
  t1.join();
  t2.join();
  EXPECT(tbad.load() == 0);
  std::printf("two threads x two streams: %d differ\n", tbad.load());
}

int main() {
  host_threads();
  two_streams();
  std::printf(g_fail ? "threads FAILED (%d)\n" : "threads ok\n", g_fail);
  return g_fail ? 1 : 0;
}
