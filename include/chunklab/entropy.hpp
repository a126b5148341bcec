// chunklab/entropy.hpp -- drop-in for the reference's K-bin entropy estimator
// (/root/reference/proj/include/chunklab/entropy.hpp), computed on the B200.
//
//   compute_histogram        entropy.hpp:101-145  -> cl_compute_histogram_host (counts bit-exact)
//   estimate_entropy         entropy.hpp:149-164  -> cl_estimate_entropy_host
//   estimate_tensor_entropy  entropy.hpp:168-174
//   token_entropy            entropy.hpp:180-210  -> one device histogram per position
//   update_ema               entropy.hpp:214-227  (scalar arithmetic)
#pragma once

#include <cstddef>
#include <span>
#include <vector>

#include "chunklab/common.hpp"

namespace chunklab {

struct ActivationTensor {
  std::vector<double> values;
  std::vector<std::size_t> shape;
  std::size_t size() const { return values.size(); }
};

// Shape checks of validate_tensor (entropy.hpp:34-41), host-side.
inline void validate_tensor_shape(const ActivationTensor& t) {
  if (t.shape.empty()) throw invalid_input("empty shape");
  std::size_t n = 1;
  for (const std::size_t e : t.shape) {
    if (e == 0) throw invalid_input("zero shape extent");
    n *= e;
  }
  if (n != t.values.size()) throw invalid_input("shape/value count mismatch");
}

namespace detail {
// validate_tensor's value check (entropy.hpp:42) over every value, on the device
inline void require_all_finite(std::span<const double> values) {
  int ok = 1;
  b200::check(cl_all_finite_host(b200::Runtime::get().ctx(), values.data(), values.size(), &ok));
  if (!ok) throw invalid_input("non-finite input");
}
}  // namespace detail

// validate_tensor (entropy.hpp:34-43): shape checks in the reference's order, then the
// finite check over every value (a min/max pass on the GPU, cl_all_finite_host).
inline void validate_tensor(const ActivationTensor& t) {
  validate_tensor_shape(t);
  detail::require_all_finite(t.values);
}

enum class RangeMode { Dynamic, Fixed };

struct HistogramSpec {
  int bin_count = 256;
  double epsilon = 1e-8;
  RangeMode range_mode = RangeMode::Dynamic;
  double fixed_lo = 0.0;
  double fixed_hi = 0.0;
  std::size_t sample_stride = 1;
};

namespace detail {
inline cl_hist_spec to_c(const HistogramSpec& s) {
  cl_hist_spec c{};
  c.bin_count = s.bin_count;
  c.epsilon = s.epsilon;
  c.range_mode = s.range_mode == RangeMode::Fixed ? CL_RANGE_FIXED : CL_RANGE_DYNAMIC;
  c.fixed_lo = s.fixed_lo;
  c.fixed_hi = s.fixed_hi;
  c.sample_stride = s.sample_stride;
  return c;
}
}  // namespace detail

inline void validate_spec(const HistogramSpec& s) {
  const cl_hist_spec c = detail::to_c(s);
  b200::check(cl_validate_hist_spec(b200::Runtime::get().ctx(), &c));
}

struct Histogram {
  std::vector<double> masses;
  double lo = 0.0;
  double hi = 0.0;
  std::size_t sample_count = 0;
  int bin_count() const { return static_cast<int>(masses.size()); }
};

struct EntropyEstimate {
  double raw_nats = 0.0;
  double normalized = 0.0;
  int bin_count = 0;
  double epsilon = 0.0;
  std::size_t sample_stride = 1;
  std::size_t sample_count = 0;
};

inline Histogram compute_histogram(std::span<const double> values, const HistogramSpec& spec) {
  validate_spec(spec);
  if (values.empty()) throw invalid_input("no samples");
  Histogram h;
  h.masses.assign(static_cast<std::size_t>(spec.bin_count), 0.0);
  const cl_hist_spec c = detail::to_c(spec);
  std::uint64_t n = 0;
  b200::check(cl_compute_histogram_host(b200::Runtime::get().ctx(), values.data(), values.size(),
                                        &c, nullptr, h.masses.data(), &h.lo, &h.hi, &n));
  h.sample_count = static_cast<std::size_t>(n);
  return h;
}

inline Histogram compute_histogram(const ActivationTensor& tensor, const HistogramSpec& spec) {
  if (tensor.values.empty()) throw invalid_input("no samples");
  validate_tensor(tensor);
  return compute_histogram(std::span<const double>(tensor.values), spec);
}

inline EntropyEstimate estimate_entropy(const Histogram& hist, double epsilon) {
  EntropyEstimate e;
  b200::check(cl_estimate_entropy_host(b200::Runtime::get().ctx(), hist.masses.data(),
                                       hist.bin_count(), epsilon, &e.raw_nats, &e.normalized));
  e.bin_count = hist.bin_count();
  e.epsilon = epsilon;
  e.sample_count = hist.sample_count;
  return e;
}

inline EntropyEstimate estimate_tensor_entropy(const ActivationTensor& tensor,
                                               const HistogramSpec& spec) {
  EntropyEstimate e = estimate_entropy(compute_histogram(tensor, spec), spec.epsilon);
  e.sample_stride = spec.sample_stride;
  return e;
}

// entropy.hpp:180-210: mean over positions of the per-position histogram entropy, one
// device call (cl_token_entropy_host: a block per 8 positions, both passes on the GPU).
inline EntropyEstimate token_entropy(const ActivationTensor& tensor, const HistogramSpec& spec) {
  validate_tensor(tensor);
  validate_spec(spec);
  if (tensor.shape.size() < 2)
    throw invalid_input("token entropy needs a (channels, length) tensor");
  const std::size_t length = tensor.shape.back();
  const std::size_t channels = tensor.values.size() / length;
  const cl_hist_spec cs = detail::to_c(spec);
  EntropyEstimate e;
  std::uint64_t samples = 0;
  b200::check(cl_token_entropy_host(b200::Runtime::get().ctx(), tensor.values.data(), channels,
                                    length, &cs, &e.raw_nats, &e.normalized, &samples));
  e.bin_count = spec.bin_count;
  e.epsilon = spec.epsilon;
  e.sample_stride = spec.sample_stride;
  e.sample_count = samples;
  return e;
}

struct EmaState {
  double current = 0.0;
  double decay = 0.85;
  std::uint64_t update_count = 0;
};

inline EmaState update_ema(const EmaState& state, double new_h) {
  if (!(state.decay >= 0.0 && state.decay < 1.0))
    throw invalid_input("ema decay must lie in [0,1)");
  EmaState next = state;
  next.current = state.decay * state.current + (1.0 - state.decay) * new_h;
  next.update_count = state.update_count + 1;
  return next;
}

}  // namespace chunklab
