// capi.cu -- the extern "C" boundary (include/chunklab_capi.h) over the sm_100a kernels.
// Host-side validation reproduces the reference's invalid_input messages verbatim
// (entropy.hpp:34-62, chunk.hpp:34-181, scan.hpp:54-69, :102-109, :127).
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "cl_internal.h"

namespace cl {

namespace {
// cl_last_error is per calling thread (errno-style): contexts are shared between host
// threads (the drop-in's process-wide context), so a per-context string would race.
thread_local std::string g_error;
}  // namespace

int fail(cl_ctx*, int code, const std::string& msg) {
  g_error = msg;
  return code;
}

const std::string& thread_error() { return g_error; }

int zero_now(cl_ctx* ctx, void* p, size_t bytes) {
  std::lock_guard<std::recursive_mutex> lk(ctx->host_mu);  // own_stream is the host path's
  CaptureRelaxed relax;
  cudaError_t e = cudaMemsetAsync(p, 0, bytes, ctx->own_stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->own_stream);
  return e == cudaSuccess ? CL_OK : cuda_fail(ctx, e, "zero scratch");
}

unsigned long long capture_id_of(cudaStream_t stream) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  unsigned long long id = 0;
  if (cudaStreamGetCaptureInfo(stream, &cs, &id) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return cs == cudaStreamCaptureStatusActive ? id : 0;
}

cl_workspace* workspace(cl_ctx* ctx, cudaStream_t stream) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  unsigned long long capture_id = 0;
  if (cudaStreamGetCaptureInfo(stream, &cs, &capture_id) != cudaSuccess) {
    cudaGetLastError();
    cs = cudaStreamCaptureStatusNone;
  }
  // Everything captured on one stream shares one captured workspace (distinct from the
  // stream's eager one): the graphs of a step (e.g. per-stage graphs replayed in order)
  // then pass state the way eager launches on that stream do.  Like any scratch, it must
  // not be used by two replays at once -- the same rule that already holds for replaying
  // one graph on two streams concurrently.
  const unsigned long long captured = cs == cudaStreamCaptureStatusActive ? 1ull : 0ull;
  (void)capture_id;
  const auto key = std::make_pair(stream, captured);
  std::lock_guard<std::mutex> lk(ctx->ws_mu);
  auto it = ctx->ws.find(key);
  if (it != ctx->ws.end()) return it->second;
  auto* w = new cl_workspace();
  w->captured = captured != 0;
  cudaError_t e;
  {
    CaptureRelaxed relax;
    e = cudaMalloc(&w->d_hist_ticket, sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMalloc(&w->d_epoch, 4 * sizeof(unsigned int));
  }
  if (e != cudaSuccess) {
    cudaFree(w->d_hist_ticket);
    cudaFree(w->d_epoch);
    delete w;
    cuda_fail(ctx, e, "cudaMalloc(stream workspace)");
    return nullptr;
  }
  if (zero_now(ctx, w->d_hist_ticket, sizeof(unsigned long long)) ||
      zero_now(ctx, w->d_epoch, 4 * sizeof(unsigned int))) {
    cudaFree(w->d_hist_ticket);
    cudaFree(w->d_epoch);
    delete w;
    return nullptr;
  }
  ctx->ws.emplace(key, w);
  return w;
}

namespace {
void free_workspace(cl_workspace* w) {
  cudaFree(w->d_work);
  cudaFree(w->d_carry);
  cudaFree(w->d_tcarry);
  cudaFree(w->d_bct);
  cudaFree(w->d_agg);
  cudaFree(w->d_hist_ticket);
  cudaFree(w->d_epoch);
  cudaFree(w->d_token_raw);
  cudaFree(w->d_token_range);
  cudaFree(w->d_token_counts);
  cudaFree(w->d_samples);
  for (void* p : w->retired) cudaFree(p);
  delete w;
}
}  // namespace

int cuda_fail(cl_ctx* ctx, cudaError_t e, const char* where) {
  return fail(ctx, CL_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

bool is_pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }

int validate_spec(cl_ctx* ctx, const cl_hist_spec* s) {
  if (!s) return fail(ctx, CL_E_INVALID, "null spec");
  if (s->bin_count < 2) return fail(ctx, CL_E_INVALID, "degenerate spec");
  if (!(s->epsilon > 0.0)) return fail(ctx, CL_E_INVALID, "epsilon must be positive");
  if (s->sample_stride < 1) return fail(ctx, CL_E_INVALID, "stride must be >= 1");
  if (s->range_mode == CL_RANGE_FIXED && !(s->fixed_lo < s->fixed_hi))
    return fail(ctx, CL_E_INVALID, "fixed range requires lo < hi");
  if (s->bin_count > kMaxBinsScratch) return fail(ctx, CL_E_INVALID, "bin_count too large");
  return CL_OK;
}

int validate_bounds(cl_ctx* ctx, int c_min, int c_max) {
  if (c_min <= 0 || c_max <= 0 || !is_pow2(c_min) || !is_pow2(c_max) || c_min > c_max)
    return fail(ctx, CL_E_INVALID, "invalid chunk bounds");
  return CL_OK;
}

bool member(const cl_rule_spec* r, int c) {
  for (int i = 0; i < r->n_buckets; ++i)
    if (r->buckets[i] == c) return true;
  return false;
}

// validate_bucket_set / validate_policy (chunk.hpp:149-181) + bounds + h_ref.
int validate_rule(cl_ctx* ctx, const cl_rule_spec* r) {
  if (!r) return fail(ctx, CL_E_INVALID, "null rule");
  const bool needs_buckets = r->kind != CL_POL_RULE;
  if (needs_buckets) {
    if (r->n_buckets < 1) return fail(ctx, CL_E_INVALID, "bucket_set must be non-empty");
    if (r->n_buckets > 16) return fail(ctx, CL_E_INVALID, "bucket_set too large");
    int prev = 0;
    for (int i = 0; i < r->n_buckets; ++i) {
      const int b = r->buckets[i];
      if (b <= 0 || !is_pow2(b) || b <= prev)
        return fail(ctx, CL_E_INVALID, "bucket_set must be strictly increasing powers of two");
      prev = b;
    }
  }
  switch (r->kind) {
    case CL_POL_STATIC:
      if (!member(r, r->static_chunk))
        return fail(ctx, CL_E_INVALID, "static chunk not in bucket_set");
      break;
    case CL_POL_GUARDED:
      if (r->inner_kind == CL_POL_GUARDED || r->inner_kind == CL_POL_RULE ||
          r->inner_kind < 0 || r->inner_kind > CL_POL_TOKEN_HIST)
        return fail(ctx, CL_E_INVALID, "guarded policy needs an inner policy");
      if (!member(r, r->safe_chunk)) return fail(ctx, CL_E_INVALID, "safe chunk not in bucket_set");
      if (r->min_delta_buckets < 0)
        return fail(ctx, CL_E_INVALID, "min_delta_buckets must be >= 0");
      if (r->inner_kind == CL_POL_STATIC && !member(r, r->inner_static_chunk))
        return fail(ctx, CL_E_INVALID, "static chunk not in bucket_set");
      if (r->inner_kind == CL_POL_LEARNED_TABLE &&
          (!member(r, r->short_chunk) || !member(r, r->long_chunk)))
        return fail(ctx, CL_E_INVALID, "learned-table chunk not in bucket_set");
      break;
    case CL_POL_LEARNED_TABLE:
      if (!member(r, r->short_chunk) || !member(r, r->long_chunk))
        return fail(ctx, CL_E_INVALID, "learned-table chunk not in bucket_set");
      break;
    case CL_POL_MIDPOINT:
    case CL_POL_FULL_HIST:
    case CL_POL_SAMPLED_HIST:
    case CL_POL_TOKEN_HIST:
    case CL_POL_RULE:
      break;
    default:
      return fail(ctx, CL_E_INVALID, "unknown policy kind");
  }
  int rc = validate_bounds(ctx, r->c_min, r->c_max);
  if (rc) return rc;
  if (!(r->h_ref_nats > 0.0)) return fail(ctx, CL_E_INVALID, "h_ref must be positive");
  return CL_OK;
}

const char* device_error_message(int code) {
  switch (code) {
    case CL_DEV_NON_FINITE: return "non-finite input";
    case CL_DEV_NO_SAMPLES: return "no samples";
    case CL_DEV_SIGNAL: return "signal must be >= 0";
    default: return "device error";
  }
}

// Host-path device staging: the context's upload buffer, grown on demand and reused, so a
// host call does no cudaMalloc / cudaFree once warm.  Callers hold ctx->host_mu.
template <typename T>
struct DevBuf {
  cl_ctx* ctx;
  T* p = nullptr;
  explicit DevBuf(cl_ctx* c) : ctx(c) {}
  cudaError_t alloc(size_t n) {
    const size_t need = n * sizeof(T) + 16;
    if (ctx->stage_bytes < need) {
      cudaFree(ctx->d_stage);
      ctx->d_stage = nullptr;
      ctx->stage_bytes = 0;
      cudaError_t e = cudaMalloc(&ctx->d_stage, need);
      if (e != cudaSuccess) return e;
      ctx->stage_bytes = need;
    }
    p = static_cast<T*>(ctx->d_stage);
    return cudaSuccess;
  }
};

int check_launch(cl_ctx* ctx, cudaError_t e, const char* where) {
  return e == cudaSuccess ? CL_OK : cuda_fail(ctx, e, where);
}

uint64_t samples_of(uint64_t n, uint64_t stride) { return n == 0 ? 0 : (n + stride - 1) / stride; }

}  // namespace
}  // namespace cl

using namespace cl;

#ifndef CL_HIST_FUSE
#define CL_HIST_FUSE 1
#endif

extern "C" {

int cl_abi_version(void) { return CL_ABI_VERSION; }

int cl_ctx_create(int device, cl_ctx** out) {
  if (!out) return CL_E_INVALID;
  *out = nullptr;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    g_error = "no CUDA device available: the chunklab B200 path has no CPU fallback";
    return CL_E_CUDA;
  }
  if (device < 0 || device >= n) {
    g_error = "invalid device ordinal";
    return CL_E_INVALID;
  }
  auto* ctx = new cl_ctx();
  ctx->device = device;
  DeviceGuard g(device);
  cudaDeviceProp prop;
  e = cudaGetDeviceProperties(&prop, device);
  if (e != cudaSuccess) {
    g_error = cudaGetErrorString(e);
    delete ctx;
    return CL_E_CUDA;
  }
  if (prop.major < 10) {
    g_error = "libchunklab_b200 is built for sm_100a (Blackwell); found sm_" +
                     std::to_string(prop.major) + std::to_string(prop.minor);
    delete ctx;
    return CL_E_CUDA;
  }
  ctx->num_sms = prop.multiProcessorCount;
  if ((e = cudaMalloc(&ctx->d_scratch_range, 4 * sizeof(double))) != cudaSuccess ||
      (e = cudaMalloc(&ctx->d_scratch_counts, kMaxBinsScratch * sizeof(uint64_t))) != cudaSuccess ||
      (e = cudaMalloc(&ctx->d_scratch_decision, sizeof(cl_decision))) != cudaSuccess ||
      (e = cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking)) != cudaSuccess) {
    g_error = cudaGetErrorString(e);
    cl_ctx_destroy(ctx);
    return CL_E_CUDA;
  }
  *out = ctx;
  return CL_OK;
}

int cl_ctx_destroy(cl_ctx* ctx) {
  if (!ctx) return CL_OK;
  DeviceGuard g(ctx->device);
  // cudaFree synchronises the device, so no workspace is freed under a running kernel
  if (ctx->own_stream) cudaStreamSynchronize(ctx->own_stream);
  cudaFree(ctx->d_scratch_range);
  cudaFree(ctx->d_scratch_counts);
  cudaFree(ctx->d_scratch_decision);
  cudaFree(ctx->d_token_out);
  cudaFree(ctx->d_stage);
  for (auto& kv : ctx->ws) free_workspace(kv.second);
  ctx->ws.clear();
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  delete ctx;
  return CL_OK;
}

const char* cl_last_error(const cl_ctx*) { return g_error.c_str(); }

uint64_t cl_launch_count(const cl_ctx* ctx) { return ctx ? ctx->launches.load() : 0; }

int cl_validate_hist_spec(cl_ctx* ctx, const cl_hist_spec* spec) { return validate_spec(ctx, spec); }
int cl_validate_rule(cl_ctx* ctx, const cl_rule_spec* rule) { return validate_rule(ctx, rule); }

// ---------------------------------------------------------------- device path
int cl_range_init(cl_ctx* ctx, double* d_range, void* stream) {
  if (!ctx || !d_range) return fail(ctx, CL_E_INVALID, "null argument");
  DeviceGuard g(ctx->device);
  ++ctx->launches;
  return check_launch(ctx, launch_range_init(d_range, static_cast<cudaStream_t>(stream)),
                      "range_init");
}

int cl_minmax_f32(cl_ctx* ctx, const float* d_values, uint64_t n, uint64_t global_offset,
                  uint64_t stride, double* d_range, void* stream) {
  if (!ctx || (!d_values && n) || !d_range) return fail(ctx, CL_E_INVALID, "null argument");
  if (stride < 1) return fail(ctx, CL_E_INVALID, "stride must be >= 1");
  DeviceGuard g(ctx->device);
  int l = 0;
  cudaError_t e = launch_minmax_f32(d_values, n, global_offset, stride, d_range, ctx->num_sms,
                                    static_cast<cudaStream_t>(stream), &l);
  ctx->launches += l;
  return check_launch(ctx, e, "minmax_f32");
}

uint64_t cl_samples_in(uint64_t global_offset, uint64_t n, uint64_t stride) {
  if (stride == 0) return 0;
  const uint64_t first = (global_offset + stride - 1) / stride;
  const uint64_t end = (global_offset + n + stride - 1) / stride;  // multiples below g0 + n
  return end > first ? end - first : 0;
}

int cl_minmax_gather_f32(cl_ctx* ctx, const float* d_values, uint64_t n, uint64_t global_offset,
                         uint64_t stride, double* d_range, float* d_samples, void* stream) {
  if (!ctx || (!d_values && n) || !d_range || (!d_samples && n))
    return fail(ctx, CL_E_INVALID, "null argument");
  if (stride < 1) return fail(ctx, CL_E_INVALID, "stride must be >= 1");
  DeviceGuard g(ctx->device);
  int l = 0;
  cudaError_t e = launch_minmax_gather_f32(d_values, n, global_offset, stride, d_range, d_samples,
                                           ctx->num_sms, static_cast<cudaStream_t>(stream), &l);
  ctx->launches += l;
  return check_launch(ctx, e, "minmax_gather_f32");
}

int cl_minmax_f64(cl_ctx* ctx, const double* d_values, uint64_t n, uint64_t global_offset,
                  uint64_t stride, double* d_range, void* stream) {
  if (!ctx || (!d_values && n) || !d_range) return fail(ctx, CL_E_INVALID, "null argument");
  if (stride < 1) return fail(ctx, CL_E_INVALID, "stride must be >= 1");
  DeviceGuard g(ctx->device);
  int l = 0;
  cudaError_t e = launch_minmax_f64(d_values, n, global_offset, stride, d_range, ctx->num_sms,
                                    static_cast<cudaStream_t>(stream), &l);
  ctx->launches += l;
  return check_launch(ctx, e, "minmax_f64");
}

int cl_conv1d_f32(cl_ctx* ctx, const float* d_x, const float* d_weight, const float* d_bias,
                  float* d_u, uint64_t batch, uint64_t dim, uint64_t seq_len, int width,
                  int silu, uint64_t global_offset, uint64_t stride, double* d_range,
                  void* stream) {
  const uint64_t n = batch * dim * seq_len;
  if (!ctx || (n && (!d_x || !d_weight || !d_u))) return fail(ctx, CL_E_INVALID, "null argument");
  if (width < 1 || width > 4) return fail(ctx, CL_E_INVALID, "conv width must lie in [1, 4]");
  if (stride < 1) return fail(ctx, CL_E_INVALID, "stride must be >= 1");
  DeviceGuard g(ctx->device);
  cudaError_t e = launch_conv1d_f32(d_x, d_weight, d_bias, d_u, batch, dim, seq_len, width,
                                    silu, global_offset, stride, d_range, ctx->num_sms,
                                    static_cast<cudaStream_t>(stream));
  if (n) ++ctx->launches;
  return check_launch(ctx, e, "conv1d_f32");
}

int cl_counts_zero(cl_ctx* ctx, uint64_t* d_counts, int bin_count, void* stream) {
  if (!ctx || !d_counts || bin_count < 1) return fail(ctx, CL_E_INVALID, "null argument");
  DeviceGuard g(ctx->device);
  return check_launch(ctx,
                      cudaMemsetAsync(d_counts, 0, size_t(bin_count) * sizeof(uint64_t),
                                      static_cast<cudaStream_t>(stream)),
                      "counts_zero");
}

int cl_prefill_init(cl_ctx* ctx, double* d_range, uint64_t* d_counts, int bin_count,
                    void* stream) {
  if (!ctx || !d_range || !d_counts || bin_count < 1) return fail(ctx, CL_E_INVALID, "null argument");
  DeviceGuard g(ctx->device);
  ++ctx->launches;
  return check_launch(ctx,
                      launch_prefill_init(d_range, d_counts, bin_count,
                                          static_cast<cudaStream_t>(stream)),
                      "prefill_init");
}

int cl_prefill_init_prepare_f32(cl_ctx* ctx, double* d_range, uint64_t* d_counts, int bin_count,
                                const cl_mamba1_args* a, void* stream) {
  if (!ctx || !d_range || !d_counts || bin_count < 1 || !a)
    return fail(ctx, CL_E_INVALID, "null argument");
  if (a->batch == 0 || a->dim == 0 || a->seq_len == 0 || a->d_state == 0)
    return fail(ctx, CL_E_INVALID, "shape mismatch");
  if (!a->B || !a->C) return fail(ctx, CL_E_INVALID, "null argument");
  DeviceGuard g(ctx->device);
  return scan_prepare_with_init(ctx, *a, d_range, d_counts, bin_count,
                                static_cast<cudaStream_t>(stream));
}

int cl_histogram_f32(cl_ctx* ctx, const float* d_values, uint64_t n, uint64_t global_offset,
                     const cl_hist_spec* spec, const double* d_range, uint64_t* d_counts,
                     void* stream) {
  int rc = validate_spec(ctx, spec);
  if (rc) return rc;
  if ((!d_values && n) || !d_range || !d_counts) return fail(ctx, CL_E_INVALID, "null argument");
  DeviceGuard g(ctx->device);
  int l = 0;
  cudaError_t e = launch_histogram_f32(d_values, n, global_offset, *spec, d_range, d_counts,
                                       ctx->num_sms, static_cast<cudaStream_t>(stream), &l);
  ctx->launches += l;
  return check_launch(ctx, e, "histogram_f32");
}

int cl_histogram_f64(cl_ctx* ctx, const double* d_values, uint64_t n, uint64_t global_offset,
                     const cl_hist_spec* spec, const double* d_range, uint64_t* d_counts,
                     void* stream) {
  int rc = validate_spec(ctx, spec);
  if (rc) return rc;
  if ((!d_values && n) || !d_range || !d_counts) return fail(ctx, CL_E_INVALID, "null argument");
  DeviceGuard g(ctx->device);
  int l = 0;
  cudaError_t e = launch_histogram_f64(d_values, n, global_offset, *spec, d_range, d_counts,
                                       ctx->num_sms, static_cast<cudaStream_t>(stream), &l);
  ctx->launches += l;
  return check_launch(ctx, e, "histogram_f64");
}

int cl_histogram_decide_f32(cl_ctx* ctx, const float* d_values, uint64_t n,
                            const cl_hist_spec* spec, const double* d_range, uint64_t* d_counts,
                            const cl_rule_spec* rule, uint64_t seq_len, cl_decision* d_decision,
                            void* stream) {
  int rc = validate_spec(ctx, spec);
  if (rc) return rc;
  rc = validate_rule(ctx, rule);
  if (rc) return rc;
  if (!d_values || !d_range || !d_counts || !d_decision)
    return fail(ctx, CL_E_INVALID, "null argument");
  if (n == 0) return fail(ctx, CL_E_INVALID, "no samples");
  bool fused = false;
  {
    DeviceGuard g(ctx->device);
    cl_workspace* w = workspace(ctx, static_cast<cudaStream_t>(stream));
    if (!w) return CL_E_CUDA;
    const HistFuse fz{samples_of(n, spec->sample_stride), rule, seq_len, d_decision,
                      w->d_hist_ticket};
    int l = 0;
    cudaError_t e = launch_histogram_f32(d_values, n, 0, *spec, d_range, d_counts, ctx->num_sms,
                                         static_cast<cudaStream_t>(stream), &l,
                                         CL_HIST_FUSE ? &fz : nullptr, &fused);
    ctx->launches += l;
    if ((rc = check_launch(ctx, e, "histogram_f32"))) return rc;
  }
  if (fused) return CL_OK;
  return cl_decide(ctx, d_counts, d_range, spec, samples_of(n, spec->sample_stride), rule,
                   seq_len, d_decision, stream);
}

int cl_entropy_lean_f32(cl_ctx* ctx, const float* d_values, uint64_t n, const cl_hist_spec* spec,
                        const cl_rule_spec* rule, uint64_t seq_len, uint64_t* d_counts,
                        double* d_range, cl_decision* d_decision, void* stream) {
  int rc = validate_spec(ctx, spec);
  if (rc) return rc;
  if ((rc = validate_rule(ctx, rule))) return rc;
  if (!d_values || !d_range || !d_counts || !d_decision)
    return fail(ctx, CL_E_INVALID, "null argument");
  if (n == 0) return fail(ctx, CL_E_INVALID, "no samples");
  if ((rc = cl_prefill_init(ctx, d_range, d_counts, spec->bin_count, stream))) return rc;
  cudaError_t e = cudaSuccess;
  bool lean;
  {
    DeviceGuard g(ctx->device);
    cl_workspace* w = workspace(ctx, static_cast<cudaStream_t>(stream));
    if (!w) return CL_E_CUDA;
    lean = launch_entropy_lean(d_values, n, *spec, *rule, seq_len, d_range, d_counts, d_decision,
                               w->d_hist_ticket, ctx->num_sms, static_cast<cudaStream_t>(stream),
                               &e);
  }
  if ((rc = check_launch(ctx, e, "entropy_lean"))) return rc;
  if (lean) {
    ctx->launches += 2;
    return CL_OK;
  }
  if ((rc = cl_minmax_f32(ctx, d_values, n, 0, spec->sample_stride, d_range, stream))) return rc;
  return cl_histogram_decide_f32(ctx, d_values, n, spec, d_range, d_counts, rule, seq_len,
                                 d_decision, stream);
}

int cl_decide(cl_ctx* ctx, const uint64_t* d_counts, const double* d_range,
              const cl_hist_spec* spec, uint64_t n_samples_total, const cl_rule_spec* rule,
              uint64_t seq_len, cl_decision* d_decision, void* stream) {
  int rc = validate_spec(ctx, spec);
  if (rc) return rc;
  rc = validate_rule(ctx, rule);
  if (rc) return rc;
  if (!d_counts || !d_range || !d_decision) return fail(ctx, CL_E_INVALID, "null argument");
  if (n_samples_total == 0) return fail(ctx, CL_E_INVALID, "no samples");
  DeviceGuard g(ctx->device);
  ++ctx->launches;
  return check_launch(ctx,
                      launch_decide(d_counts, d_range, *spec, n_samples_total, *rule, seq_len,
                                    nullptr, d_decision, static_cast<cudaStream_t>(stream)),
                      "decide");
}

extern "C++" {
namespace {
int validate_token(cl_ctx* ctx, const cl_hist_spec* spec, uint64_t channels, uint64_t length) {
  int rc = validate_spec(ctx, spec);
  if (rc) return rc;
  if (channels == 0 || length == 0) return fail(ctx, CL_E_INVALID, "no samples");
  if (spec->bin_count > 4096)
    return fail(ctx, CL_E_INVALID, "token entropy supports bin_count <= 4096");
  return CL_OK;
}

template <typename P>
int grow_bytes(cl_ctx* ctx, P** ptr, size_t* have, size_t need, cl_workspace* w = nullptr) {
  return grow_scratch(ctx, w, ptr, have, need, "cudaMalloc(token entropy scratch)");
}

int grow_token(cl_ctx* ctx, cl_workspace* w, uint64_t length, int k) {
  int rc = grow_bytes(ctx, &w->d_token_raw, &w->token_raw_bytes, length * sizeof(double), w);
  if (!rc)
    rc = grow_bytes(ctx, &w->d_token_range, &w->token_range_bytes,
                    (2 * length + 1) * sizeof(double), w);
  if (!rc)
    rc = grow_bytes(ctx, &w->d_token_counts, &w->token_counts_bytes,
                    length * static_cast<size_t>(k) * sizeof(unsigned int), w);
  return rc;
}

// the four stages over one device tensor with the stream workspace's scratch
template <typename T>
cudaError_t token_pipeline(cl_ctx* ctx, cl_workspace* w, const T* d_values, uint64_t channels,
                           uint64_t length, const cl_hist_spec& spec, double* d_out,
                           cudaStream_t s) {
  double* trange = w->d_token_range;
  double* flag = w->d_token_range + 2 * length;
  cudaError_t e = launch_token_range_init(trange, flag, length, s);
  if (e == cudaSuccess)
    e = launch_token_minmax<T>(d_values, channels, length, 0, spec.sample_stride, trange, flag,
                               ctx->num_sms, s);
  if (e == cudaSuccess)
    e = cudaMemsetAsync(w->d_token_counts, 0,
                        length * static_cast<size_t>(spec.bin_count) * sizeof(unsigned int), s);
  if (e == cudaSuccess)
    e = launch_token_hist<T>(d_values, channels, length, 0, spec, trange, w->d_token_counts,
                             ctx->num_sms, s);
  if (e == cudaSuccess)
    e = launch_token_entropy(w->d_token_counts, length, samples_of(channels, spec.sample_stride),
                             spec, flag, w->d_token_raw, d_out, s);
  ctx->launches += 5;
  return e;
}
}  // namespace
}  // extern "C++"

int cl_token_range_init(cl_ctx* ctx, double* d_trange, uint64_t length, void* stream) {
  if (!ctx || !d_trange) return fail(ctx, CL_E_INVALID, "null argument");
  DeviceGuard g(ctx->device);
  ++ctx->launches;
  return check_launch(ctx,
                      launch_token_range_init(d_trange, d_trange + 2 * length, length,
                                              static_cast<cudaStream_t>(stream)),
                      "token_range_init");
}

int cl_token_minmax_f32(cl_ctx* ctx, const float* d_values, uint64_t channels, uint64_t length,
                        uint64_t channel_offset, uint64_t stride, double* d_trange,
                        void* stream) {
  if (!ctx || !d_trange || (!d_values && channels && length))
    return fail(ctx, CL_E_INVALID, "null argument");
  if (stride < 1) return fail(ctx, CL_E_INVALID, "stride must be >= 1");
  if (channels == 0 || length == 0) return CL_OK;
  DeviceGuard g(ctx->device);
  ++ctx->launches;
  return check_launch(ctx,
                      launch_token_minmax<float>(d_values, channels, length, channel_offset,
                                                 stride, d_trange, d_trange + 2 * length,
                                                 ctx->num_sms,
                                                 static_cast<cudaStream_t>(stream)),
                      "token_minmax_f32");
}

int cl_token_histogram_f32(cl_ctx* ctx, const float* d_values, uint64_t channels, uint64_t length,
                           uint64_t channel_offset, const cl_hist_spec* spec,
                           const double* d_trange, uint32_t* d_counts, void* stream) {
  if (!ctx) return CL_E_INVALID;
  int rc = validate_spec(ctx, spec);
  if (rc) return rc;
  if (spec->bin_count > 4096)
    return fail(ctx, CL_E_INVALID, "token entropy supports bin_count <= 4096");
  if (!d_trange || !d_counts || (!d_values && channels && length))
    return fail(ctx, CL_E_INVALID, "null argument");
  if (channels == 0 || length == 0) return CL_OK;
  DeviceGuard g(ctx->device);
  ++ctx->launches;
  return check_launch(ctx,
                      launch_token_hist<float>(d_values, channels, length, channel_offset, *spec,
                                               d_trange, d_counts, ctx->num_sms,
                                               static_cast<cudaStream_t>(stream)),
                      "token_histogram_f32");
}

int cl_token_entropy_counts(cl_ctx* ctx, const uint32_t* d_counts, const double* d_trange,
                            uint64_t length, uint64_t samples_per_position,
                            const cl_hist_spec* spec, double* d_out, void* stream) {
  if (!ctx) return CL_E_INVALID;
  int rc = validate_spec(ctx, spec);
  if (rc) return rc;
  if (!d_counts || !d_trange || !d_out) return fail(ctx, CL_E_INVALID, "null argument");
  if (length == 0 || samples_per_position == 0) return fail(ctx, CL_E_INVALID, "no samples");
  DeviceGuard g(ctx->device);
  cl_workspace* w = workspace(ctx, static_cast<cudaStream_t>(stream));
  if (!w) return CL_E_CUDA;
  if ((rc = grow_bytes(ctx, &w->d_token_raw, &w->token_raw_bytes, length * sizeof(double), w)))
    return rc;
  ctx->launches += 2;
  return check_launch(ctx,
                      launch_token_entropy(d_counts, length, samples_per_position, *spec,
                                           d_trange + 2 * length, w->d_token_raw, d_out,
                                           static_cast<cudaStream_t>(stream)),
                      "token_entropy");
}

int cl_token_entropy_f32(cl_ctx* ctx, const float* d_values, uint64_t channels, uint64_t length,
                         const cl_hist_spec* spec, double* d_out, void* stream) {
  if (!ctx) return CL_E_INVALID;
  int rc = validate_token(ctx, spec, channels, length);
  if (rc) return rc;
  if (!d_values || !d_out) return fail(ctx, CL_E_INVALID, "null argument");
  DeviceGuard g(ctx->device);
  cl_workspace* w = workspace(ctx, static_cast<cudaStream_t>(stream));
  if (!w) return CL_E_CUDA;
  if ((rc = grow_token(ctx, w, length, spec->bin_count))) return rc;
  return check_launch(ctx,
                      token_pipeline<float>(ctx, w, d_values, channels, length, *spec, d_out,
                                            static_cast<cudaStream_t>(stream)),
                      "token_entropy_f32");
}

int cl_decide_token(cl_ctx* ctx, const double* d_token, const cl_hist_spec* spec,
                    const cl_rule_spec* rule, uint64_t seq_len, cl_decision* d_out,
                    void* stream) {
  int rc = validate_spec(ctx, spec);
  if (rc) return rc;
  if ((rc = validate_rule(ctx, rule))) return rc;
  if (!d_token || !d_out) return fail(ctx, CL_E_INVALID, "null argument");
  const int kind = rule->kind == CL_POL_GUARDED ? rule->inner_kind : rule->kind;
  if (kind == CL_POL_FULL_HIST || kind == CL_POL_SAMPLED_HIST || kind == CL_POL_RULE)
    return fail(ctx, CL_E_INVALID, "token decision needs a token_histogram policy");
  DeviceGuard g(ctx->device);
  ++ctx->launches;
  return check_launch(ctx,
                      launch_decide_token(d_token, *spec, *rule, seq_len, d_out,
                                          static_cast<cudaStream_t>(stream)),
                      "decide_token");
}

int cl_selective_scan_f32(cl_ctx* ctx, const cl_mamba1_args* args, const cl_decision* d_decision,
                          int fixed_chunk, int variant, void* stream) {
  if (!ctx || !args) return fail(ctx, CL_E_INVALID, "null argument");
  const cl_mamba1_args& a = *args;
  if (a.batch == 0 || a.dim == 0 || a.seq_len == 0 || a.d_state == 0)
    return fail(ctx, CL_E_INVALID, "shape mismatch");
  if (!a.u || !a.delta || !a.A || !a.B || !a.C || !a.out)
    return fail(ctx, CL_E_INVALID, "null argument");
  if (!d_decision && fixed_chunk < 1) return fail(ctx, CL_E_INVALID, "chunk must be >= 1");
  DeviceGuard g(ctx->device);
  return scan_mamba1(ctx, a, d_decision, fixed_chunk, variant, static_cast<cudaStream_t>(stream));
}

int cl_scan_plan_f32(cl_ctx* ctx, const cl_mamba1_args* args, int variant, cl_scan_plan* out) {
  if (!ctx || !args || !out) return fail(ctx, CL_E_INVALID, "null argument");
  return scan_plan(ctx, *args, variant, out);
}

int cl_selective_state_update_f32(cl_ctx* ctx, const cl_state_update_args* args, void* stream) {
  if (!ctx || !args) return fail(ctx, CL_E_INVALID, "null argument");
  const cl_state_update_args& a = *args;
  if (a.batch == 0 || a.dim == 0 || a.d_state == 0) return fail(ctx, CL_E_INVALID, "shape mismatch");
  if (a.d_state > 64) return fail(ctx, CL_E_INVALID, "d_state must lie in [1, 64]");
  if (!a.state || !a.x || !a.dt || !a.A || !a.B || !a.C || !a.out)
    return fail(ctx, CL_E_INVALID, "null argument");
  DeviceGuard g(ctx->device);
  return state_update_f32(ctx, a, static_cast<cudaStream_t>(stream));
}

int cl_prefill_f32(cl_ctx* ctx, const cl_mamba1_args* args, const cl_hist_spec* spec,
                   const cl_rule_spec* rule, uint64_t* d_counts, double* d_range,
                   cl_decision* d_decision, void* stream) {
  if (!ctx || !args) return fail(ctx, CL_E_INVALID, "null argument");
  int rc = validate_spec(ctx, spec);
  if (rc) return rc;
  rc = validate_rule(ctx, rule);
  if (rc) return rc;
  const uint64_t n = args->batch * args->dim * args->seq_len;
  if (n == 0) return fail(ctx, CL_E_INVALID, "no samples");
  const int kind = rule->kind == CL_POL_GUARDED ? rule->inner_kind : rule->kind;
  if (kind == CL_POL_TOKEN_HIST) {
    // TokenHistogram: token_entropy over u as (batch*dim, seq_len), result staged in
    // d_range (4 doubles, the token_entropy output layout); d_counts unused
    if ((rc = cl_token_entropy_f32(ctx, args->u, args->batch * args->dim, args->seq_len, spec,
                                   d_range, stream)))
      return rc;
    if ((rc = cl_decide_token(ctx, d_range, spec, rule, args->seq_len, d_decision, stream)))
      return rc;
    return cl_selective_scan_f32(ctx, args, d_decision, 0, CL_SCAN_AUTO, stream);
  }
  if ((rc = cl_prefill_init_prepare_f32(ctx, d_range, d_counts, spec->bin_count, args, stream)))
    return rc;
  if (spec->sample_stride >= CL_GATHER_MIN_STRIDE) {
    // strided sampling: min/max gathers the samples, the histogram reads only them
    // (stride 8 at C4: 1.125 + 0.125 reads of u instead of 2)
    cl_workspace* w = workspace(ctx, static_cast<cudaStream_t>(stream));
    if (!w) return CL_E_CUDA;
    const uint64_t m = cl_samples_in(0, n, spec->sample_stride);
    if ((rc = grow_scratch(ctx, w, &w->d_samples, &w->samples_bytes, m * sizeof(float),
                           "cudaMalloc(gathered samples)")))
      return rc;
    if ((rc = cl_minmax_gather_f32(ctx, args->u, n, 0, spec->sample_stride, d_range, w->d_samples,
                                   stream)))
      return rc;
    cl_hist_spec s1 = *spec;
    s1.sample_stride = 1;
    if ((rc = cl_histogram_decide_f32(ctx, w->d_samples, m, &s1, d_range, d_counts, rule,
                                       args->seq_len, d_decision, stream)))
      return rc;
    return cl_selective_scan_f32(ctx, args, d_decision, 0, CL_SCAN_AUTO, stream);
  }
  if ((rc = cl_minmax_f32(ctx, args->u, n, 0, spec->sample_stride, d_range, stream))) return rc;
  if ((rc = cl_histogram_decide_f32(ctx, args->u, n, spec, d_range, d_counts, rule,
                                     args->seq_len, d_decision, stream)))
    return rc;
  return cl_selective_scan_f32(ctx, args, d_decision, 0, CL_SCAN_AUTO, stream);
}

int cl_prefill_from_conv_f32(cl_ctx* ctx, const cl_conv_args* conv, const cl_mamba1_args* args,
                             const cl_hist_spec* spec, const cl_rule_spec* rule,
                             uint64_t* d_counts, double* d_range, cl_decision* d_decision,
                             void* stream) {
  if (!ctx || !conv || !args) return fail(ctx, CL_E_INVALID, "null argument");
  int rc = validate_spec(ctx, spec);
  if (rc) return rc;
  if ((rc = validate_rule(ctx, rule))) return rc;
  const uint64_t n = args->batch * args->dim * args->seq_len;
  if (n == 0) return fail(ctx, CL_E_INVALID, "no samples");
  if (!conv->x || !conv->weight || !args->u) return fail(ctx, CL_E_INVALID, "null argument");
  if (conv->width < 1 || conv->width > 4)
    return fail(ctx, CL_E_INVALID, "conv width must lie in [1, 4]");
  float* u = const_cast<float*>(args->u);  // the conv's output buffer
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int kind = rule->kind == CL_POL_GUARDED ? rule->inner_kind : rule->kind;
  if (kind == CL_POL_TOKEN_HIST) {
    if ((rc = cl_conv1d_f32(ctx, conv->x, conv->weight, conv->bias, u, args->batch, args->dim,
                            args->seq_len, conv->width, conv->silu, 0, 1, nullptr, stream)))
      return rc;
    return cl_prefill_f32(ctx, args, spec, rule, d_counts, d_range, d_decision, stream);
  }
  if ((rc = cl_prefill_init_prepare_f32(ctx, d_range, d_counts, spec->bin_count, args, stream)))
    return rc;
  if (spec->range_mode == CL_RANGE_FIXED) {
    cudaError_t e = cudaSuccess;
    bool fused;
    {
      DeviceGuard g(ctx->device);
      fused = launch_conv_hist_fixed(conv->x, conv->weight, conv->bias, u, args->batch, args->dim,
                                     args->seq_len, conv->width, conv->silu, *spec, d_counts,
                                     d_range, ctx->num_sms, s, &e);
    }
    if ((rc = check_launch(ctx, e, "conv_hist_fixed"))) return rc;
    if (fused) {
      ++ctx->launches;
    } else {
      // conv with the range epilogue (its finite flag), then the histogram pass
      if ((rc = cl_conv1d_f32(ctx, conv->x, conv->weight, conv->bias, u, args->batch, args->dim,
                              args->seq_len, conv->width, conv->silu, 0, spec->sample_stride,
                              d_range, stream)) ||
          (rc = cl_histogram_f32(ctx, u, n, 0, spec, d_range, d_counts, stream)))
        return rc;
    }
    if ((rc = cl_decide(ctx, d_counts, d_range, spec, samples_of(n, spec->sample_stride), rule,
                        args->seq_len, d_decision, stream)))
      return rc;
  } else {
    if ((rc = cl_conv1d_f32(ctx, conv->x, conv->weight, conv->bias, u, args->batch, args->dim,
                            args->seq_len, conv->width, conv->silu, 0, spec->sample_stride,
                            d_range, stream)) ||
        (rc = cl_histogram_decide_f32(ctx, u, n, spec, d_range, d_counts, rule, args->seq_len,
                                      d_decision, stream)))
      return rc;
  }
  return cl_selective_scan_f32(ctx, args, d_decision, 0, CL_SCAN_AUTO, stream);
}

int cl_decision_check(cl_ctx* ctx, const cl_decision* d_decision, cl_decision* h_out,
                      void* stream) {
  if (!ctx || !d_decision) return fail(ctx, CL_E_INVALID, "null argument");
  DeviceGuard g(ctx->device);
  cl_decision tmp;
  cl_decision* dst = h_out ? h_out : &tmp;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemcpyAsync(dst, d_decision, sizeof(cl_decision), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "decision_check");
  if (dst->status != CL_DEV_OK) return fail(ctx, CL_E_DEVICE, device_error_message(dst->status));
  return CL_OK;
}

int cl_scan_f64(cl_ctx* ctx, const cl_scan_params_f64* p, const double* d_h0, uint64_t chunk,
                double* d_y, double* d_h, void* stream) {
  if (!ctx || !p || !d_y || !d_h) return fail(ctx, CL_E_INVALID, "null argument");
  // validate_scan_params (scan.hpp:54-69), shape part; finiteness is the host path's job.
  if (p->channels == 0 || p->state_dim == 0 || p->seq_len == 0)
    return fail(ctx, CL_E_INVALID, "shape mismatch");
  const uint64_t cs = p->channels * p->state_dim;
  if ((p->a_len != cs && p->a_len != p->seq_len * cs) ||
      (p->b_len != p->state_dim && p->b_len != p->seq_len * p->state_dim) ||
      (p->c_len != p->state_dim && p->c_len != p->seq_len * p->state_dim) ||
      p->d_len != p->channels || p->x_len != p->channels * p->seq_len)
    return fail(ctx, CL_E_INVALID, "shape mismatch");
  DeviceGuard g(ctx->device);
  ++ctx->launches;
  return check_launch(
      ctx, launch_scan_f64(*p, d_h0, chunk, d_y, d_h, static_cast<cudaStream_t>(stream)),
      "scan_f64");
}

// ------------------------------------------------------------------ host path
int cl_all_finite_host(cl_ctx* ctx, const double* h_values, uint64_t n, int* h_all_finite) {
  if (!ctx) return CL_E_INVALID;
  if ((n && !h_values) || !h_all_finite) return fail(ctx, CL_E_INVALID, "null argument");
  *h_all_finite = 1;
  if (n == 0) return CL_OK;
  DeviceGuard g(ctx->device);
  std::lock_guard<std::recursive_mutex> lk(ctx->host_mu);
  cudaStream_t s = ctx->own_stream;
  DevBuf<double> dv(ctx);
  cudaError_t e = dv.alloc(n);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMalloc");
  if ((e = cudaMemcpyAsync(dv.p, h_values, n * sizeof(double), cudaMemcpyHostToDevice, s)) !=
      cudaSuccess)
    return cuda_fail(ctx, e, "cudaMemcpyAsync");
  int rc;
  if ((rc = cl_range_init(ctx, ctx->d_scratch_range, s))) return rc;
  if ((rc = cl_minmax_f64(ctx, dv.p, n, 0, 1, ctx->d_scratch_range, s))) return rc;
  double range[4];
  if ((e = cudaMemcpyAsync(range, ctx->d_scratch_range, sizeof range, cudaMemcpyDeviceToHost,
                           s)) != cudaSuccess ||
      (e = cudaStreamSynchronize(s)) != cudaSuccess)
    return cuda_fail(ctx, e, "finite readback");
  *h_all_finite = range[2] == 0.0;
  return CL_OK;
}

int cl_compute_histogram_host(cl_ctx* ctx, const double* h_values, uint64_t n,
                              const cl_hist_spec* spec, uint64_t* h_counts, double* h_masses,
                              double* h_lo, double* h_hi, uint64_t* h_sample_count) {
  if (!ctx) return CL_E_INVALID;
  int rc = validate_spec(ctx, spec);
  if (rc) return rc;
  if (n == 0) return fail(ctx, CL_E_INVALID, "no samples");
  // The span overload visits values[0], values[stride], ... only (entropy.hpp:108-114):
  // gather that subsequence so the device pass -- including its finite check -- sees
  // exactly the values the reference visits; binning then runs at stride 1.
  std::vector<double> gathered;
  cl_hist_spec sp = *spec;
  if (spec->sample_stride > 1) {
    gathered.reserve(samples_of(n, spec->sample_stride));
    for (uint64_t i = 0; i < n; i += spec->sample_stride) gathered.push_back(h_values[i]);
    h_values = gathered.data();
    n = gathered.size();
    sp.sample_stride = 1;
  }
  DeviceGuard g(ctx->device);
  std::lock_guard<std::recursive_mutex> lk(ctx->host_mu);
  cudaStream_t s = ctx->own_stream;
  DevBuf<double> dv(ctx);
  cudaError_t e = dv.alloc(n);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMalloc");
  if ((e = cudaMemcpyAsync(dv.p, h_values, n * sizeof(double), cudaMemcpyHostToDevice, s)) !=
      cudaSuccess)
    return cuda_fail(ctx, e, "cudaMemcpyAsync");
  double* d_range = ctx->d_scratch_range;
  uint64_t* d_counts = ctx->d_scratch_counts;
  if ((rc = cl_range_init(ctx, d_range, s))) return rc;
  if ((rc = cl_minmax_f64(ctx, dv.p, n, 0, 1, d_range, s))) return rc;
  double range[4];
  if ((e = cudaMemcpyAsync(range, d_range, sizeof range, cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
      (e = cudaStreamSynchronize(s)) != cudaSuccess)
    return cuda_fail(ctx, e, "minmax readback");
  // entropy.hpp:110: the reference throws on the first non-finite sampled value
  if (range[2] != 0.0) return fail(ctx, CL_E_INVALID, "non-finite input");
  if ((rc = cl_counts_zero(ctx, d_counts, sp.bin_count, s))) return rc;
  if ((rc = cl_histogram_f64(ctx, dv.p, n, 0, &sp, d_range, d_counts, s))) return rc;
  std::vector<uint64_t> counts(sp.bin_count);
  if ((e = cudaMemcpyAsync(counts.data(), d_counts, counts.size() * sizeof(uint64_t),
                           cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
      (e = cudaStreamSynchronize(s)) != cudaSuccess)
    return cuda_fail(ctx, e, "counts readback");
  const uint64_t ns = n;
  if (h_counts) std::memcpy(h_counts, counts.data(), counts.size() * sizeof(uint64_t));
  if (h_masses) {
    // masses[b] = counts[b] * (1/n) (entropy.hpp:130-133); exact IEEE ops on the host
    // are identical to the device's, kept here to avoid another round trip.
    const double inv_n = 1.0 / static_cast<double>(ns);
    for (int b = 0; b < sp.bin_count; ++b) h_masses[b] = static_cast<double>(counts[b]) * inv_n;
  }
  if (h_lo) *h_lo = sp.range_mode == CL_RANGE_FIXED ? sp.fixed_lo : -range[0];
  if (h_hi) *h_hi = sp.range_mode == CL_RANGE_FIXED ? sp.fixed_hi : range[1];
  if (h_sample_count) *h_sample_count = ns;
  return CL_OK;
}

int cl_token_entropy_host(cl_ctx* ctx, const double* h_values, uint64_t channels,
                          uint64_t length, const cl_hist_spec* spec, double* h_raw,
                          double* h_normalized, uint64_t* h_sample_count) {
  if (!ctx) return CL_E_INVALID;
  int rc = validate_token(ctx, spec, channels, length);
  if (rc) return rc;
  if (!h_values) return fail(ctx, CL_E_INVALID, "null argument");
  DeviceGuard g(ctx->device);
  std::lock_guard<std::recursive_mutex> lk(ctx->host_mu);
  cudaStream_t s = ctx->own_stream;
  cl_workspace* w = workspace(ctx, s);
  if (!w) return CL_E_CUDA;
  const uint64_t n = channels * length;
  DevBuf<double> dv(ctx);
  cudaError_t e = dv.alloc(n);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMalloc");
  if ((rc = grow_bytes(ctx, &ctx->d_token_out, &ctx->token_out_bytes, 4 * sizeof(double))))
    return rc;
  if ((rc = grow_token(ctx, w, length, spec->bin_count))) return rc;
  if ((e = cudaMemcpyAsync(dv.p, h_values, n * sizeof(double), cudaMemcpyHostToDevice, s)) !=
      cudaSuccess)
    return cuda_fail(ctx, e, "cudaMemcpyAsync");
  if ((e = token_pipeline<double>(ctx, w, dv.p, channels, length, *spec, ctx->d_token_out, s)) !=
      cudaSuccess)
    return cuda_fail(ctx, e, "token_entropy_f64");
  double out[4];
  if ((e = cudaMemcpyAsync(out, ctx->d_token_out, sizeof out, cudaMemcpyDeviceToHost, s)) !=
          cudaSuccess ||
      (e = cudaStreamSynchronize(s)) != cudaSuccess)
    return cuda_fail(ctx, e, "token entropy readback");
  if (out[3] != 0.0) return fail(ctx, CL_E_INVALID, "non-finite input");
  if (h_raw) *h_raw = out[0];
  if (h_normalized) *h_normalized = out[1];
  if (h_sample_count) *h_sample_count = static_cast<uint64_t>(out[2]);
  return CL_OK;
}

int cl_estimate_entropy_host(cl_ctx* ctx, const double* h_masses, int bin_count, double epsilon,
                             double* h_raw, double* h_normalized) {
  if (!ctx) return CL_E_INVALID;
  if (bin_count < 2) return fail(ctx, CL_E_INVALID, "degenerate spec");
  if (!(epsilon > 0.0)) return fail(ctx, CL_E_INVALID, "epsilon must be positive");
  DeviceGuard g(ctx->device);
  std::lock_guard<std::recursive_mutex> lk(ctx->host_mu);
  cudaStream_t s = ctx->own_stream;
  DevBuf<double> dm(ctx);
  cudaError_t e = dm.alloc(size_t(bin_count) + 2);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMalloc");
  if ((e = cudaMemcpyAsync(dm.p, h_masses, bin_count * sizeof(double), cudaMemcpyHostToDevice,
                           s)) != cudaSuccess)
    return cuda_fail(ctx, e, "cudaMemcpyAsync");
  double* d_out = dm.p + bin_count;
  ++ctx->launches;
  if ((e = launch_entropy_from_masses(dm.p, bin_count, epsilon, d_out, s)) != cudaSuccess)
    return cuda_fail(ctx, e, "entropy kernel");
  double out[2];
  if ((e = cudaMemcpyAsync(out, d_out, sizeof out, cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
      (e = cudaStreamSynchronize(s)) != cudaSuccess)
    return cuda_fail(ctx, e, "entropy readback");
  if (h_raw) *h_raw = out[0];
  if (h_normalized) *h_normalized = out[1];
  return CL_OK;
}

int cl_schedule_host(cl_ctx* ctx, const cl_rule_spec* rule, const cl_features* features,
                     cl_decision* h_out) {
  if (!ctx) return CL_E_INVALID;
  int rc = validate_rule(ctx, rule);
  if (rc) return rc;
  if (!features || !h_out) return fail(ctx, CL_E_INVALID, "null argument");
  // missing-feature checks (chunk.hpp:197-201), in Scheduler::decide order
  const int kind = rule->kind == CL_POL_GUARDED ? rule->inner_kind : rule->kind;
  if (kind == CL_POL_FULL_HIST && !features->has_full_entropy)
    return fail(ctx, CL_E_INVALID, "missing feature: full_entropy");
  if (kind == CL_POL_SAMPLED_HIST && !features->has_sampled_entropy)
    return fail(ctx, CL_E_INVALID, "missing feature: sampled_entropy");
  if (kind == CL_POL_RULE && !features->has_full_entropy)
    return fail(ctx, CL_E_INVALID, "missing feature: full_entropy");
  if (kind == CL_POL_LEARNED_TABLE && !features->has_seq_len)
    return fail(ctx, CL_E_INVALID, "missing feature: seq_len");
  if (kind == CL_POL_TOKEN_HIST && !features->has_token_entropy)
    return fail(ctx, CL_E_INVALID, "missing feature: token_entropy");
  DeviceGuard g(ctx->device);
  std::lock_guard<std::recursive_mutex> lk(ctx->host_mu);
  cudaStream_t s = ctx->own_stream;
  cl_hist_spec spec{256, 1e-8, 0, 0.0, 0.0, 1};
  ++ctx->launches;
  cudaError_t e = launch_decide(nullptr, ctx->d_scratch_range, spec, 1, *rule,
                                features->has_seq_len ? features->seq_len : 0, features,
                                ctx->d_scratch_decision, s);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "decide");
  rc = cl_decision_check(ctx, ctx->d_scratch_decision, h_out, s);
  if (rc == CL_E_DEVICE) return fail(ctx, CL_E_INVALID, std::string(thread_error()));
  return rc;
}

int cl_scan_f64_host(cl_ctx* ctx, const cl_scan_params_f64* h, const double* h_h0,
                     uint64_t chunk, double* h_y, double* h_h) {
  if (!ctx || !h) return fail(ctx, CL_E_INVALID, "null argument");
  if (h->channels == 0 || h->state_dim == 0 || h->seq_len == 0)
    return fail(ctx, CL_E_INVALID, "shape mismatch");
  const uint64_t cs = h->channels * h->state_dim;
  if ((h->a_len != cs && h->a_len != h->seq_len * cs) ||
      (h->b_len != h->state_dim && h->b_len != h->seq_len * h->state_dim) ||
      (h->c_len != h->state_dim && h->c_len != h->seq_len * h->state_dim) ||
      h->d_len != h->channels || h->x_len != h->channels * h->seq_len)
    return fail(ctx, CL_E_INVALID, "shape mismatch");
  DeviceGuard g(ctx->device);
  std::lock_guard<std::recursive_mutex> lk(ctx->host_mu);
  cudaStream_t s = ctx->own_stream;
  const size_t total = h->a_len + h->b_len + h->c_len + h->d_len + h->x_len + cs;
  DevBuf<double> buf(ctx);
  cudaError_t e = buf.alloc(total + h->x_len + cs);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMalloc");
  double* p = buf.p;
  cl_scan_params_f64 d = *h;
  const double* srcs[5] = {h->a, h->b, h->c, h->d, h->x};
  const uint64_t lens[5] = {h->a_len, h->b_len, h->c_len, h->d_len, h->x_len};
  const double** dsts[5] = {&d.a, &d.b, &d.c, &d.d, &d.x};
  for (int k = 0; k < 5; ++k) {
    if ((e = cudaMemcpyAsync(p, srcs[k], lens[k] * sizeof(double), cudaMemcpyHostToDevice, s)) !=
        cudaSuccess)
      return cuda_fail(ctx, e, "cudaMemcpyAsync");
    *dsts[k] = p;
    p += lens[k];
  }
  double* d_h0 = nullptr;
  if (h_h0) {
    d_h0 = p;
    if ((e = cudaMemcpyAsync(d_h0, h_h0, cs * sizeof(double), cudaMemcpyHostToDevice, s)) !=
        cudaSuccess)
      return cuda_fail(ctx, e, "cudaMemcpyAsync");
    p += cs;
  }
  double* d_y = p;
  p += h->x_len;
  double* d_hout = p;
  // validate_scan_params / initial_state finiteness (scan.hpp:70-72, :111) on device
  int rc = cl_range_init(ctx, ctx->d_scratch_range, s);
  if (rc) return rc;
  for (int k = 0; k < 5; ++k)
    if ((rc = cl_minmax_f64(ctx, *dsts[k], lens[k], 0, 1, ctx->d_scratch_range, s))) return rc;
  double range[4];
  if ((e = cudaMemcpyAsync(range, ctx->d_scratch_range, sizeof range, cudaMemcpyDeviceToHost, s)) !=
          cudaSuccess ||
      (e = cudaStreamSynchronize(s)) != cudaSuccess)
    return cuda_fail(ctx, e, "finite check");
  if (range[2] != 0.0) return fail(ctx, CL_E_INVALID, "non-finite input");
  if (d_h0) {
    if ((rc = cl_minmax_f64(ctx, d_h0, cs, 0, 1, ctx->d_scratch_range, s))) return rc;
    if ((e = cudaMemcpyAsync(range, ctx->d_scratch_range, sizeof range, cudaMemcpyDeviceToHost,
                             s)) != cudaSuccess ||
        (e = cudaStreamSynchronize(s)) != cudaSuccess)
      return cuda_fail(ctx, e, "finite check");
    if (range[2] != 0.0) return fail(ctx, CL_E_INVALID, "non-finite input");
  }
  rc = cl_scan_f64(ctx, &d, d_h0, chunk, d_y, d_hout, s);
  if (rc) return rc;
  if ((e = cudaMemcpyAsync(h_y, d_y, h->x_len * sizeof(double), cudaMemcpyDeviceToHost, s)) !=
          cudaSuccess ||
      (e = cudaMemcpyAsync(h_h, d_hout, cs * sizeof(double), cudaMemcpyDeviceToHost, s)) !=
          cudaSuccess ||
      (e = cudaStreamSynchronize(s)) != cudaSuccess)
    return cuda_fail(ctx, e, "scan readback");
  return CL_OK;
}

}  // extern "C"
