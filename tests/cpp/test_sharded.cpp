// Multi-GPU entry point through the C++ drop-in (chunklab::ShardedPrefill ->
// cl_prefill_sharded_f32) on ONE B200: each "rank" is a host thread with its own CUDA
// stream and its own local tensors, and the two allreduces are host-staged (D2H, host
// barrier, combine, H2D) -- no kernel ever waits on another rank's kernel, so running the
// ranks on one GPU is safe.  Checked against the single-GPU prefill of the whole tensor:
//   * range, counts and the decision record: bit for bit, on every rank;
//   * every rank's output rows and h_last: <= 1e-6 normwise (the local row count can
//     select a different scan kernel than the whole tensor does; same kernel => same bits).
// Plans: batch split (C3/C4-style) and d_inner split (C1/C2-style, incl. B = 2), Dynamic
// stride 1, Guarded{Sampled stride 8}, and TokenHistogram.  Then world = 1 through REAL
// NCCL (ncclCommInitAll on one device, cl_collectives_nccl): bitwise equal to single-GPU.
// Prints "sharded ok" on success.
#include <cuda_runtime.h>
#include <nccl.h>

#include <barrier>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <random>
#include <thread>
#include <vector>

#include "chunklab/chunk.hpp"
#include "chunklab/mamba1.hpp"

using namespace chunklab;

static int g_fail = 0;
#define EXPECT(c)                                              \
  do {                                                         \
    if (!(c)) {                                                \
      ++g_fail;                                                \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
    }                                                          \
  } while (0)

static void ok(cudaError_t e) {
  if (e != cudaSuccess) {
    std::printf("CUDA error: %s\n", cudaGetErrorString(e));
    std::exit(2);
  }
}

struct Host {  // global tensors
  uint64_t B, D, L;
  std::vector<float> u, dt, A, Bm, Cm, Dv, z, bias;
};

static Host make(uint64_t B, uint64_t D, uint64_t L, unsigned seed) {
  Host h{B, D, L};
  std::mt19937_64 g(seed);
  std::normal_distribution<float> n01;
  std::uniform_real_distribution<float> un(-1.f, 1.f);
  auto fill = [&](std::vector<float>& v, size_t n, float s) {
    v.resize(n);
    for (auto& x : v) x = s * n01(g);
  };
  fill(h.u, B * D * L, 1.f);
  fill(h.dt, B * D * L, 0.1f);
  fill(h.Bm, B * 16 * L, 1.f);
  fill(h.Cm, B * 16 * L, 1.f);
  fill(h.z, B * D * L, 1.f);
  h.A.resize(D * 16);
  for (uint64_t c = 0; c < D; ++c)
    for (int s = 0; s < 16; ++s) h.A[c * 16 + s] = -(s + 1) * (1.f + 0.1f * un(g));
  h.Dv.resize(D);
  h.bias.resize(D);
  for (uint64_t c = 0; c < D; ++c) {
    h.Dv[c] = 1.f + 0.1f * n01(g);
    const float t = std::exp(std::log(1e-3f) + (un(g) + 1.f) * 0.5f * std::log(100.f));
    h.bias[c] = std::log(std::expm1(t));
  }
  return h;
}

struct Dev {  // one rank's local tensors on the device
  uint64_t b, d, L;
  float *u, *dt, *A, *B, *C, *D, *z, *bias, *out, *h;
  Dev(const Host& g, const cl_shard& s) : b(s.b1 - s.b0), d(s.d1 - s.d0), L(g.L) {
    std::vector<float> u_, dt_, z_, B_, C_, A_, D_, bias_;
    for (uint64_t bb = s.b0; bb < s.b1; ++bb) {
      for (uint64_t c = s.d0; c < s.d1; ++c) {
        const size_t o = (bb * g.D + c) * L;
        u_.insert(u_.end(), g.u.begin() + o, g.u.begin() + o + L);
        dt_.insert(dt_.end(), g.dt.begin() + o, g.dt.begin() + o + L);
        z_.insert(z_.end(), g.z.begin() + o, g.z.begin() + o + L);
      }
      B_.insert(B_.end(), g.Bm.begin() + bb * 16 * L, g.Bm.begin() + (bb + 1) * 16 * L);
      C_.insert(C_.end(), g.Cm.begin() + bb * 16 * L, g.Cm.begin() + (bb + 1) * 16 * L);
    }
    A_.assign(g.A.begin() + s.d0 * 16, g.A.begin() + s.d1 * 16);
    D_.assign(g.Dv.begin() + s.d0, g.Dv.begin() + s.d1);
    bias_.assign(g.bias.begin() + s.d0, g.bias.begin() + s.d1);
    auto up = [](const std::vector<float>& v, float** p) {
      ok(cudaMalloc(p, v.size() * 4));
      ok(cudaMemcpy(*p, v.data(), v.size() * 4, cudaMemcpyHostToDevice));
    };
    up(u_, &u), up(dt_, &dt), up(z_, &z), up(B_, &B), up(C_, &C), up(A_, &A), up(D_, &D);
    up(bias_, &bias);
    ok(cudaMalloc(&out, b * d * L * 4));
    ok(cudaMalloc(&h, b * d * 16 * 4));
  }
  ~Dev() {
    for (float* p : {u, dt, A, B, C, D, z, bias, out, h}) cudaFree(p);
  }
  Mamba1Args args() const {
    Mamba1Args a{};
    a.u = u, a.delta = dt, a.A = A, a.B = B, a.C = C, a.D = D, a.z = z, a.delta_bias = bias;
    a.out = out, a.h_last = h, a.batch = b, a.dim = d, a.seq_len = L, a.d_state = 16;
    a.delta_softplus = 1;
    return a;
  }
  std::vector<float> y() const {
    std::vector<float> v(b * d * L);
    ok(cudaMemcpy(v.data(), out, v.size() * 4, cudaMemcpyDeviceToHost));
    return v;
  }
  std::vector<float> hl() const {
    std::vector<float> v(b * d * 16);
    ok(cudaMemcpy(v.data(), h, v.size() * 4, cudaMemcpyDeviceToHost));
    return v;
  }
};

// Host-staged allreduce shared by `world` rank threads.
struct Staging {
  int world;
  std::barrier<> bar;
  std::vector<std::vector<unsigned char>> slot;
  explicit Staging(int w) : world(w), bar(w), slot(w) {}
};
struct RankHook {
  Staging* st;
  int rank;
};

template <typename T, typename Op>
static int staged(T* d, size_t n, void* stream, void* user, Op op) {
  auto* rh = static_cast<RankHook*>(user);
  Staging& st = *rh->st;
  auto s = static_cast<cudaStream_t>(stream);
  std::vector<unsigned char>& mine = st.slot[rh->rank];
  mine.resize(n * sizeof(T));
  if (cudaMemcpyAsync(mine.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return CL_E_CUDA;
  st.bar.arrive_and_wait();
  std::vector<T> acc(n);
  std::memcpy(acc.data(), st.slot[0].data(), n * sizeof(T));
  for (int r = 1; r < st.world; ++r) {
    const T* o = reinterpret_cast<const T*>(st.slot[r].data());
    for (size_t i = 0; i < n; ++i) acc[i] = op(acc[i], o[i]);
  }
  st.bar.arrive_and_wait();  // every rank has read every slot
  if (cudaMemcpyAsync(d, acc.data(), n * sizeof(T), cudaMemcpyHostToDevice, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return CL_E_CUDA;
  return CL_OK;
}
static int h_max_f64(double* d, size_t n, void* s, void* u) {
  return staged(d, n, s, u, [](double a, double b) { return a < b ? b : a; });
}
static int h_sum_u64(uint64_t* d, size_t n, void* s, void* u) {
  return staged(d, n, s, u, [](uint64_t a, uint64_t b) { return a + b; });
}
static int h_sum_u32(uint32_t* d, size_t n, void* s, void* u) {
  return staged(d, n, s, u, [](uint32_t a, uint32_t b) { return a + b; });
}

struct Record {
  cl_decision dec;
  std::vector<uint64_t> counts;
  double range[4];
};

static Record read(const Prefill& p, int k, bool token) {
  Record r{};
  ok(cudaDeviceSynchronize());
  ok(cudaMemcpy(&r.dec, p.device_decision(), sizeof(cl_decision), cudaMemcpyDeviceToHost));
  if (!token) {
    r.counts.resize(k);
    ok(cudaMemcpy(r.counts.data(), p.device_counts(), k * 8, cudaMemcpyDeviceToHost));
    ok(cudaMemcpy(r.range, p.device_range(), 32, cudaMemcpyDeviceToHost));
  }
  return r;
}

static double rel(const std::vector<float>& a, const std::vector<float>& b) {
  double num = 0, den = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    num += (double(a[i]) - b[i]) * (double(a[i]) - b[i]);
    den += double(b[i]) * b[i];
  }
  return std::sqrt(num / (den > 0 ? den : 1));
}

struct Case {
  const char* name;
  uint64_t B, D, L;
  int world;
  int policy;  // 0 rule, 1 guarded sampled stride 8, 2 token histogram
};

static void run_case(const Case& c) {
  const Host g = make(c.B, c.D, c.L, 11 + c.world);
  HistogramSpec spec;
  std::unique_ptr<SchedulerPolicy> pol;
  ChunkBounds bounds{32, 512};
  const std::vector<int> buckets = {128, 256, 512, 1024, 2048};
  if (c.policy == 1) {
    spec.sample_stride = 8;
    SchedulerPolicy inner{SampledHistogramPolicy{8}, buckets};
    pol = std::make_unique<SchedulerPolicy>(
        SchedulerPolicy{GuardedPolicy{std::make_shared<SchedulerPolicy>(inner), 512, 2}, buckets});
    bounds = ChunkBounds{128, 2048};
  } else if (c.policy == 2) {
    pol = std::make_unique<SchedulerPolicy>(SchedulerPolicy{TokenHistogramPolicy{}, buckets});
    bounds = ChunkBounds{128, 2048};
  }
  const CalibrationRef cal = CalibrationRef::log_k(256);
  // single GPU, whole tensor
  const cl_shard whole = ShardedPrefill::plan(c.B, c.D, 0, 1);
  Dev full(g, whole);
  Prefill ref(spec, pol.get(), bounds, cal);
  ref.run(full.args());
  const Record rr = read(ref, 256, c.policy == 2);
  const std::vector<float> yref = full.y(), href = full.hl();
  // world ranks as threads
  Staging st(c.world);
  std::vector<Record> recs(c.world);
  std::vector<double> yerr(c.world), herr(c.world);
  std::vector<int> bitwise(c.world);
  std::vector<std::thread> th;
  for (int r = 0; r < c.world; ++r) {
    th.emplace_back([&, r] {
      const cl_shard sh = ShardedPrefill::plan(c.B, c.D, r, c.world);
      Dev loc(g, sh);
      RankHook rh{&st, r};
      cl_collectives coll{h_max_f64, h_sum_u64, h_sum_u32, &rh};
      cudaStream_t s;
      ok(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
      ShardedPrefill sp(spec, pol.get(), bounds, cal, sh, coll);
      sp.run(loc.args(), s);
      ok(cudaStreamSynchronize(s));
      recs[r] = read(sp, 256, c.policy == 2);
      // the rank's rows of the single-GPU output
      std::vector<float> ysub, hsub;
      for (uint64_t b = sh.b0; b < sh.b1; ++b)
        for (uint64_t d = sh.d0; d < sh.d1; ++d) {
          const size_t o = (b * c.D + d);
          ysub.insert(ysub.end(), yref.begin() + o * c.L, yref.begin() + (o + 1) * c.L);
          hsub.insert(hsub.end(), href.begin() + o * 16, href.begin() + (o + 1) * 16);
        }
      const std::vector<float> y = loc.y(), h = loc.hl();
      yerr[r] = rel(y, ysub);
      herr[r] = rel(h, hsub);
      bitwise[r] = y == ysub && h == hsub;
      ok(cudaStreamDestroy(s));
    });
  }
  for (auto& t : th) t.join();
  for (int r = 0; r < c.world; ++r) {
    const Record& q = recs[r];
    EXPECT(std::memcmp(&q.dec, &rr.dec, sizeof(cl_decision)) == 0);
    EXPECT(q.counts == rr.counts);
    if (c.policy != 2) EXPECT(std::memcmp(q.range, rr.range, 24) == 0);
    EXPECT(yerr[r] <= 1e-6 && herr[r] <= 1e-6);
    std::printf("  %s rank %d/%d: chunk %d raw %.17g, y rel %.2e, h rel %.2e, bitwise %d\n",
                c.name, r, c.world, q.dec.chunk, q.dec.raw_nats, yerr[r], herr[r], bitwise[r]);
  }
}

static void nccl_world1() {
  const Host g = make(2, 128, 1024, 5);
  HistogramSpec spec;
  const CalibrationRef cal = CalibrationRef::log_k(256);
  const cl_shard whole = ShardedPrefill::plan(2, 128, 0, 1);
  Dev a(g, whole), b(g, whole);
  Prefill ref(spec, nullptr, ChunkBounds{32, 512}, cal);
  ref.run(a.args());
  const Record rr = read(ref, 256, false);
  ncclComm_t comm;
  int dev = 0;
  if (ncclCommInitAll(&comm, 1, &dev) != ncclSuccess) {
    std::printf("FAIL ncclCommInitAll\n");
    ++g_fail;
    return;
  }
  ShardedPrefill sp(spec, nullptr, ChunkBounds{32, 512}, cal, whole, ShardedPrefill::nccl(comm));
  sp.run(b.args());
  const Record q = read(sp, 256, false);
  EXPECT(std::memcmp(&q.dec, &rr.dec, sizeof(cl_decision)) == 0);
  EXPECT(q.counts == rr.counts);
  EXPECT(a.y() == b.y() && a.hl() == b.hl());
  std::printf("  nccl world 1: chunk %d, bitwise %d\n", q.dec.chunk, int(a.y() == b.y()));
  ncclCommDestroy(comm);
}

int main() {
  const Case cases[] = {
      {"batch-split", 4, 96, 1024, 2, 0},
      {"batch-split-guarded-s8", 4, 64, 2048, 4, 1},
      {"dim-split", 1, 256, 2048, 2, 0},
      {"dim-split-B2", 2, 64, 512, 4, 0},
      {"dim-split-token", 1, 128, 512, 2, 2},
      {"batch-split-token", 2, 64, 256, 2, 2},
  };
  for (const Case& c : cases) run_case(c);
  nccl_world1();
  std::printf(g_fail ? "sharded FAILED (%d)\n" : "sharded ok\n", g_fail);
  return g_fail ? 1 : 0;
}
