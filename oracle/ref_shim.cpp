// ref_shim.cpp -- C-ABI shim over the REFERENCE's own headers (TEST INFRASTRUCTURE ONLY).
//
// Compiled in place against /root/reference/proj/include (never copied) by
// oracle/Makefile into oracle/_ref/libchunklab_ref.so.  It exposes the
// reference's hot-path functions with plain-C signatures so that
//   * tests can pin the C restatement (chunklab_oracle.c) bit-for-bit against
//     the reference itself, and generate tests/golden/ fixtures, and
//   * bench.py --impl reference can time the reference's own CPU path.
// Nothing in the product path loads this library.
#include <chunklab/chunk.hpp>
#include <chunklab/entropy.hpp>
#include <chunklab/scan.hpp>
#include <chunklab/synthetic.hpp>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

using namespace chunklab;

namespace {
thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

struct RefHistSpec {  // layout-identical to or_hist_spec / cl_hist_spec
  int bin_count;
  double epsilon;
  int range_mode;
  double fixed_lo, fixed_hi;
  uint64_t sample_stride;
};

HistogramSpec to_spec(const RefHistSpec* s) {
  HistogramSpec h;
  h.bin_count = s->bin_count;
  h.epsilon = s->epsilon;
  h.range_mode = s->range_mode ? RangeMode::Fixed : RangeMode::Dynamic;
  h.fixed_lo = s->fixed_lo;
  h.fixed_hi = s->fixed_hi;
  h.sample_stride = s->sample_stride;
  return h;
}

struct RefPolicy {  // layout-identical to or_policy
  int kind;
  int static_chunk;
  int inner_kind;
  int inner_static_chunk;
  int safe_chunk;
  int min_delta_buckets;
  uint64_t threshold_tokens;
  int short_chunk, long_chunk;
  int n_buckets;
  int buckets[16];
};

struct RefFeatures {  // layout-identical to or_features
  int has_full_entropy;
  double full_entropy_nats;
  int has_sampled_entropy;
  double sampled_entropy_nats;
  int has_seq_len;
  uint64_t seq_len;
};

PolicyVariant simple_variant(int kind, int static_chunk, const RefPolicy* p) {
  switch (kind) {
    case 0: return StaticPolicy{static_chunk};
    case 1: return NoEntropyMidpointPolicy{};
    case 2: return FullHistogramPolicy{};
    case 3: return SampledHistogramPolicy{8};
    case 4: return LearnedTablePolicy{p->threshold_tokens, p->short_chunk, p->long_chunk};
    default: throw invalid_input("unsupported policy kind");
  }
}

int source_code(const std::string& tag) {
  static const char* names[] = {"static", "no_entropy_midpoint", "full_histogram",
                                "sampled_histogram", "learned_table"};
  if (tag == "guarded[fallback]") return 32;
  for (int i = 0; i < 5; ++i) {
    if (tag == names[i]) return i;
    if (tag == std::string("guarded[") + names[i] + "]") return 16 + i;
  }
  return -1;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_generate_activations(int dist, double laplace_scale, double nonzero_fraction,
                             uint64_t seed, uint64_t n, double* out) {
  return guarded([&] {
    SyntheticSpec s;
    s.distribution = static_cast<Distribution>(dist);
    s.laplace_scale = laplace_scale;
    s.nonzero_fraction = nonzero_fraction;
    s.seed = seed;
    s.shape = {static_cast<std::size_t>(n)};
    ActivationTensor t = generate_activations(s);
    std::memcpy(out, t.values.data(), n * sizeof(double));
  });
}

// compute_histogram(ActivationTensor) (entropy.hpp:140-145) -> masses, lo, hi, n.
int ref_compute_histogram(const double* values, uint64_t n, const RefHistSpec* spec,
                          double* masses, double* lo, double* hi, uint64_t* count) {
  return guarded([&] {
    ActivationTensor t;
    t.values.assign(values, values + n);
    t.shape = {static_cast<std::size_t>(n)};
    Histogram h = compute_histogram(t, to_spec(spec));
    std::memcpy(masses, h.masses.data(), h.masses.size() * sizeof(double));
    *lo = h.lo;
    *hi = h.hi;
    *count = h.sample_count;
  });
}

// Same over float values widened to double (io.hpp:19-44 semantics).
int ref_compute_histogram_f32(const float* values, uint64_t n, const RefHistSpec* spec,
                              double* masses, double* lo, double* hi, uint64_t* count) {
  return guarded([&] {
    ActivationTensor t;
    t.values.resize(n);
    for (uint64_t i = 0; i < n; ++i) t.values[i] = static_cast<double>(values[i]);
    t.shape = {static_cast<std::size_t>(n)};
    Histogram h = compute_histogram(t, to_spec(spec));
    std::memcpy(masses, h.masses.data(), h.masses.size() * sizeof(double));
    *lo = h.lo;
    *hi = h.hi;
    *count = h.sample_count;
  });
}

// token_entropy(tensor (channels, length), spec) (entropy.hpp:180-210).
int ref_token_entropy(const double* values, uint64_t channels, uint64_t length,
                      const RefHistSpec* spec, double* raw, double* norm, uint64_t* count) {
  return guarded([&] {
    ActivationTensor t;
    t.values.assign(values, values + channels * length);
    t.shape = {static_cast<std::size_t>(channels), static_cast<std::size_t>(length)};
    EntropyEstimate e = token_entropy(t, to_spec(spec));
    *raw = e.raw_nats;
    *norm = e.normalized;
    *count = e.sample_count;
  });
}

int ref_estimate_entropy(const double* masses, int k, double eps, double* raw, double* norm) {
  return guarded([&] {
    Histogram h;
    h.masses.assign(masses, masses + k);
    EntropyEstimate e = estimate_entropy(h, eps);
    *raw = e.raw_nats;
    *norm = e.normalized;
  });
}

int ref_select_chunk(double signal, int c_min, int c_max, double h_ref, int* chunk,
                     double* r) {
  return guarded([&] {
    CalibrationRef cal{CalibrationMode::LegacyFixed, h_ref};
    ChunkDecision d = select_chunk(signal, ChunkBounds{c_min, c_max}, cal);
    *chunk = d.chunk;
    *r = d.r;
  });
}

int ref_schedule(const RefPolicy* p, const RefFeatures* f, int c_min, int c_max, double h_ref,
                 int* chunk, double* r, double* signal, int* source) {
  return guarded([&] {
    SchedulerPolicy pol;
    pol.bucket_set.assign(p->buckets, p->buckets + p->n_buckets);
    if (p->kind == 5) {
      GuardedPolicy g;
      auto inner = std::make_shared<SchedulerPolicy>();
      inner->bucket_set = pol.bucket_set;
      inner->variant = simple_variant(p->inner_kind, p->inner_static_chunk, p);
      g.inner = inner;
      g.safe_chunk = p->safe_chunk;
      g.min_delta_buckets = p->min_delta_buckets;
      pol.variant = g;
    } else {
      pol.variant = simple_variant(p->kind, p->static_chunk, p);
    }
    ScheduleFeatures feat;
    if (f->has_full_entropy) {
      EntropyEstimate e;
      e.raw_nats = f->full_entropy_nats;
      feat.full_entropy = e;
    }
    if (f->has_sampled_entropy) {
      EntropyEstimate e;
      e.raw_nats = f->sampled_entropy_nats;
      feat.sampled_entropy = e;
    }
    if (f->has_seq_len) feat.seq_len = static_cast<std::size_t>(f->seq_len);
    CalibrationRef cal{CalibrationMode::LegacyFixed, h_ref};
    ChunkDecision d = schedule(pol, feat, ChunkBounds{c_min, c_max}, cal);
    *chunk = d.chunk;
    *r = d.r;
    *signal = d.signal_nats;
    *source = source_code(d.source_policy);
  });
}

// scan_sequential / scan_chunked (scan.hpp:113-136).  chunk == 0 -> sequential.
int ref_scan(uint64_t channels, uint64_t state_dim, uint64_t seq_len, const double* a,
             uint64_t a_len, const double* b, uint64_t b_len, const double* c, uint64_t c_len,
             const double* d, uint64_t d_len, const double* x, uint64_t x_len, const double* h0,
             uint64_t chunk, double* y, double* h_out) {
  return guarded([&] {
    ScanParams p;
    p.channels = channels;
    p.state_dim = state_dim;
    p.seq_len = seq_len;
    p.a.assign(a, a + a_len);
    p.b.assign(b, b + b_len);
    p.c.assign(c, c + c_len);
    p.d.assign(d, d + d_len);
    p.x.assign(x, x + x_len);
    ScanState s0;
    if (h0) s0.h.assign(h0, h0 + channels * state_dim);
    auto res = chunk == 0 ? scan_sequential(p, s0) : scan_chunked(p, s0, chunk);
    std::memcpy(y, res.first.y.data(), res.first.y.size() * sizeof(double));
    std::memcpy(h_out, res.second.h.data(), res.second.h.size() * sizeof(double));
  });
}

int ref_random_scan_params(uint64_t seed, uint64_t channels, uint64_t state_dim,
                           uint64_t seq_len, int tv, double* a, double* b, double* c, double* d,
                           double* x) {
  return guarded([&] {
    ScanParams p = random_scan_params(seed, channels, state_dim, seq_len, tv != 0);
    std::memcpy(a, p.a.data(), p.a.size() * sizeof(double));
    std::memcpy(b, p.b.data(), p.b.size() * sizeof(double));
    std::memcpy(c, p.c.data(), p.c.size() * sizeof(double));
    std::memcpy(d, p.d.data(), p.d.size() * sizeof(double));
    std::memcpy(x, p.x.data(), p.x.size() * sizeof(double));
  });
}

// Mamba-1 selective scan expressed through the reference recurrence
// (SURVEY.md finding 1): per batch, scan_sequential with time-varying
// a[t][c][s] = exp(delta'(c,t) * A[c,s]), b/c = B/C[b,:,t], x = delta'*u, d = 0;
// then y = y_ref + D*u and the SiLU(z) gate.  Rows [row_begin,row_end) must lie
// in one batch.  Float inputs are widened to double (io.hpp:19-44).  Used as
// the --impl reference CPU path; `threads` partitions the rows.
int ref_mamba1_rows_f32(const float* u, const float* delta, const float* A, const float* Bm,
                        const float* Cm, const float* Dv, const float* z,
                        const float* delta_bias, int delta_softplus, uint64_t batch,
                        uint64_t dim, uint64_t N, uint64_t L, uint64_t row_begin,
                        uint64_t row_end, int threads, double* y, double* h_last) {
  return guarded([&] {
    if (row_end <= row_begin) return;
    if (row_begin / dim != (row_end - 1) / dim)
      throw invalid_input("row range must lie in one batch");
    const uint64_t bb = row_begin / dim;
    const uint64_t rows = row_end - row_begin;
    if (threads < 1) threads = 1;
    if (static_cast<uint64_t>(threads) > rows) threads = static_cast<int>(rows);
    auto work = [&](uint64_t r0, uint64_t r1) {
      const uint64_t ch = r1 - r0;
      ScanParams p;
      p.channels = ch;
      p.state_dim = N;
      p.seq_len = L;
      p.a.resize(L * ch * N);
      p.b.resize(L * N);
      p.c.resize(L * N);
      p.d.assign(ch, 0.0);
      p.x.resize(ch * L);
      std::vector<double> dt(ch * L);
      for (uint64_t k = 0; k < ch; ++k) {
        const uint64_t row = r0 + k, cc = row % dim;
        const double bias = delta_bias ? static_cast<double>(delta_bias[cc]) : 0.0;
        for (uint64_t t = 0; t < L; ++t) {
          double v = static_cast<double>(delta[row * L + t]) + bias;
          if (delta_softplus) v = v <= 20.0 ? std::log1p(std::exp(v)) : v;
          dt[k * L + t] = v;
          p.x[k * L + t] = v * static_cast<double>(u[row * L + t]);
        }
      }
      for (uint64_t t = 0; t < L; ++t) {
        for (uint64_t k = 0; k < ch; ++k) {
          const uint64_t cc = (r0 + k) % dim;
          for (uint64_t s = 0; s < N; ++s)
            p.a[(t * ch + k) * N + s] =
                std::exp(dt[k * L + t] * static_cast<double>(A[cc * N + s]));
        }
        for (uint64_t s = 0; s < N; ++s) {
          p.b[t * N + s] = static_cast<double>(Bm[(bb * N + s) * L + t]);
          p.c[t * N + s] = static_cast<double>(Cm[(bb * N + s) * L + t]);
        }
      }
      auto res = scan_sequential(p, ScanState{});
      for (uint64_t k = 0; k < ch; ++k) {
        const uint64_t row = r0 + k, cc = row % dim;
        const double dskip = Dv ? static_cast<double>(Dv[cc]) : 0.0;
        for (uint64_t t = 0; t < L; ++t) {
          const double uu = static_cast<double>(u[row * L + t]);
          double yy = res.first.y[k * L + t] + dskip * uu;
          if (z) {
            const double zz = static_cast<double>(z[row * L + t]);
            yy = yy * (zz / (1.0 + std::exp(-zz)));
          }
          y[(row - row_begin) * L + t] = yy;
        }
        if (h_last)
          for (uint64_t s = 0; s < N; ++s)
            h_last[(row - row_begin) * N + s] = res.second.h[k * N + s];
      }
    };
    std::vector<std::thread> pool;
    const uint64_t per = (rows + threads - 1) / threads;
    for (int i = 0; i < threads; ++i) {
      const uint64_t r0 = row_begin + i * per;
      const uint64_t r1 = std::min(row_end, r0 + per);
      if (r0 >= r1) break;
      pool.emplace_back(work, r0, r1);
    }
    for (auto& th : pool) th.join();
  });
}

}  // extern "C"
