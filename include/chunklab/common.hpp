// chunklab/common.hpp -- drop-in for /root/reference/proj/include/chunklab/common.hpp
// (B200 build).  Same names and semantics; the compute entry points of the other
// headers forward to libchunklab_b200.so (include/chunklab_capi.h).
#pragma once

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <span>
#include <stdexcept>
#include <string>

#include "chunklab_capi.h"

namespace chunklab {

// common.hpp:12-18 -- stable messages surfaced verbatim.
class invalid_input : public std::invalid_argument {
 public:
  using std::invalid_argument::invalid_argument;
};

// common.hpp:20-46 (scalar helpers used by the API contracts)
inline constexpr bool is_power_of_two(std::uint64_t v) { return v && !(v & (v - 1)); }

inline int log2_exact(std::uint64_t v) {
  int e = -1;
  do {
    ++e;
    v >>= 1;
  } while (v);
  return e;
}

inline double round_half_up(double x) { return std::floor(x + 0.5); }

inline bool all_finite(std::span<const double> xs) {
  for (const double x : xs)
    if (!std::isfinite(x)) return false;
  return true;
}

inline std::size_t ceil_div(std::size_t num, std::size_t den) { return (num + den - 1) / den; }

namespace b200 {

// One C-ABI context per process (device from $CHUNKLAB_DEVICE, default 0).
class Runtime {
 public:
  static Runtime& get() {
    static Runtime rt;
    return rt;
  }
  cl_ctx* ctx() {
    std::call_once(once_, [this] {
      const char* d = std::getenv("CHUNKLAB_DEVICE");
      const int dev = d ? std::atoi(d) : 0;
      rc_ = cl_ctx_create(dev, &ctx_);
      if (rc_ != CL_OK) err_ = cl_last_error(nullptr);
    });
    if (rc_ != CL_OK) throw std::runtime_error("chunklab B200 runtime unavailable: " + err_);
    return ctx_;
  }
  ~Runtime() {
    if (ctx_) cl_ctx_destroy(ctx_);
  }

 private:
  Runtime() = default;
  std::once_flag once_;
  cl_ctx* ctx_ = nullptr;
  int rc_ = CL_OK;
  std::string err_;
};

// Map a C-ABI status onto the reference's exception types.
inline void check(int rc) {
  if (rc == CL_OK) return;
  cl_ctx* c = Runtime::get().ctx();
  const std::string msg = cl_last_error(c);
  if (rc == CL_E_INVALID || rc == CL_E_DEVICE) throw invalid_input(msg);
  throw std::runtime_error(msg);
}

}  // namespace b200
}  // namespace chunklab
