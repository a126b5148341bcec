// chunklab/scan.hpp -- drop-in for the reference recurrence
// (/root/reference/proj/include/chunklab/scan.hpp).  scan_sequential / scan_chunked
// run the fp64 reference-mode kernel on the B200 (cl_scan_f64_host): the operation
// order of scan_window (scan.hpp:77-100) is kept without FMA contraction, so the
// outputs are bit-identical to the reference for every chunk size.
#pragma once

#include <cstddef>
#include <utility>
#include <vector>

#include "chunklab/common.hpp"
#include "chunklab/rng.hpp"

namespace chunklab {

struct ScanParams {
  std::size_t channels = 0;
  std::size_t state_dim = 0;
  std::size_t seq_len = 0;
  std::vector<double> a;  // d*state or L*d*state [t][c][s]
  std::vector<double> b;  // state or L*state [t][s]
  std::vector<double> c;  // state or L*state [t][s]
  std::vector<double> d;  // channels
  std::vector<double> x;  // [c][t]

  bool a_time_varying() const { return a.size() == seq_len * channels * state_dim; }
  bool b_time_varying() const { return b.size() == seq_len * state_dim; }
  bool c_time_varying() const { return c.size() == seq_len * state_dim; }
};

struct ScanState {
  std::vector<double> h;
};

struct ScanOutput {
  std::vector<double> y;
};

// scan.hpp:54-68, the shape part (the scan call checks finiteness on the device)
inline void validate_scan_shapes(const ScanParams& p) {
  if (p.channels == 0 || p.state_dim == 0 || p.seq_len == 0) throw invalid_input("shape mismatch");
  const std::size_t cs = p.channels * p.state_dim;
  const bool ok = (p.a.size() == cs || p.a.size() == p.seq_len * cs) &&
                  (p.b.size() == p.state_dim || p.b.size() == p.seq_len * p.state_dim) &&
                  (p.c.size() == p.state_dim || p.c.size() == p.seq_len * p.state_dim) &&
                  p.d.size() == p.channels && p.x.size() == p.channels * p.seq_len;
  if (!ok) throw invalid_input("shape mismatch");
}

namespace detail {
inline bool all_finite_on_device(const std::vector<double>& v) {
  int ok = 1;
  b200::check(cl_all_finite_host(b200::Runtime::get().ctx(), v.data(), v.size(), &ok));
  return ok != 0;
}
}  // namespace detail

// validate_scan_params (scan.hpp:54-69): the shape checks, then "non-finite input" if
// any of a, b, c, d, x holds a NaN or infinity (checked by a min/max pass on the GPU).
inline void validate_scan_params(const ScanParams& p) {
  validate_scan_shapes(p);
  if (!detail::all_finite_on_device(p.a) || !detail::all_finite_on_device(p.b) ||
      !detail::all_finite_on_device(p.c) || !detail::all_finite_on_device(p.d) ||
      !detail::all_finite_on_device(p.x))
    throw invalid_input("non-finite input");
}

namespace detail {
inline std::pair<ScanOutput, ScanState> run_scan(const ScanParams& p, const ScanState& h0,
                                                 std::size_t chunk) {
  validate_scan_shapes(p);
  if (!h0.h.empty() && h0.h.size() != p.channels * p.state_dim)
    throw invalid_input("shape mismatch");
  cl_scan_params_f64 q{};
  q.channels = p.channels;
  q.state_dim = p.state_dim;
  q.seq_len = p.seq_len;
  q.a = p.a.data();
  q.b = p.b.data();
  q.c = p.c.data();
  q.d = p.d.data();
  q.x = p.x.data();
  q.a_len = p.a.size();
  q.b_len = p.b.size();
  q.c_len = p.c.size();
  q.d_len = p.d.size();
  q.x_len = p.x.size();
  ScanOutput out;
  ScanState st;
  out.y.resize(p.channels * p.seq_len);
  st.h.resize(p.channels * p.state_dim);
  b200::check(cl_scan_f64_host(b200::Runtime::get().ctx(), &q,
                               h0.h.empty() ? nullptr : h0.h.data(), chunk, out.y.data(),
                               st.h.data()));
  return {std::move(out), std::move(st)};
}
}  // namespace detail

inline std::pair<ScanOutput, ScanState> scan_sequential(const ScanParams& p, const ScanState& h0) {
  return detail::run_scan(p, h0, 0);
}

inline std::pair<ScanOutput, ScanState> scan_chunked(const ScanParams& p, const ScanState& h0,
                                                     std::size_t chunk) {
  validate_scan_shapes(p);
  if (chunk < 1) throw invalid_input("chunk must be >= 1");
  return detail::run_scan(p, h0, chunk);
}

// Seeded parameters (scan.hpp:140-163): same stream layout as the reference.
inline ScanParams random_scan_params(std::uint64_t seed, std::size_t channels,
                                     std::size_t state_dim, std::size_t seq_len,
                                     bool time_varying = true) {
  Rng rng(seed);
  ScanParams p;
  p.channels = channels;
  p.state_dim = state_dim;
  p.seq_len = seq_len;
  p.a.resize(time_varying ? seq_len * channels * state_dim : channels * state_dim);
  const std::size_t nbc = time_varying ? seq_len * state_dim : state_dim;
  for (double& v : p.a) v = rng.uniform(0.5, 0.995);
  p.b.resize(nbc);
  for (double& v : p.b) v = rng.normal();
  p.c.resize(nbc);
  const double inv = std::sqrt(static_cast<double>(state_dim));
  for (double& v : p.c) v = rng.normal() / inv;
  p.d.resize(channels);
  for (double& v : p.d) v = 0.1 * rng.normal();
  p.x.resize(channels * seq_len);
  for (double& v : p.x) v = rng.normal();
  return p;
}

}  // namespace chunklab
