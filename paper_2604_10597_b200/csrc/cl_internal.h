// cl_internal.h -- internal declarations shared by the C-ABI implementation and the kernels.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <map>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "chunklab_capi.h"

// Device scratch that a launch sequence on ONE stream owns.  Kernels on the same stream
// are ordered, so they may reuse it; two streams never share one (a scan's work ticket,
// tagged carry and B/C transpose, or the fused histogram's arrival ticket, would race).
struct cl_workspace {
  unsigned int* d_work = nullptr;  // scan work counters / flags (grown on demand)
  size_t work_bytes = 0;
  bool ticket_dirty = false;  // the last scan on this stream left d_work non-zero
  float* d_carry = nullptr;  // scan segment carry of the row kernel (grown on demand)
  size_t carry_bytes = 0;
  // tagged segment carry of the warp-specialised scan: 64-bit words {tag, h}; tags are
  // epoch + segment with the epoch advanced past every launch's tags, so stale words from
  // earlier launches never match (zeroed on allocation and on epoch wrap)
  unsigned long long* d_tcarry = nullptr;
  size_t tcarry_bytes = 0;
  unsigned int carry_epoch = 0;
  float* d_bct = nullptr;  // B^T / C^T (b, L, N) for the TMA scan (grown on demand)
  size_t bct_bytes = 0;
  // d_bct already holds the interleaved [B | C] re-layout of these inputs, written by
  // cl_prefill_init_prepare_f32 earlier on this stream; the next scan with the same B, C,
  // batch and L consumes it (and clears it) instead of launching its own transpose
  // (in a captured workspace only within the same capture: a graph's replays cannot know
  // what another graph's replays left in d_bct)
  bool bct_ready = false;
  const float* bct_B = nullptr;
  const float* bct_C = nullptr;
  uint64_t bct_batch = 0, bct_L = 0;
  unsigned long long bct_capture = 0;  // capture id of the prepare (0: eager)
  // L-parallel scan: per-(tile, segment) aggregates {tag, h~_end[16], sum dt} words
  unsigned long long* d_agg = nullptr;
  size_t agg_bytes = 0;
  unsigned int agg_epoch = 0;
  // arrival ticket of the fused histogram -> decision launch: 0 between launches (the
  // last CTA resets it), never visible to callers
  unsigned long long* d_hist_ticket = nullptr;
  // captured workspaces: device-side launch counters ([1]: L-parallel aggregate tags),
  // advanced by each launch's last work claimer, so every replay of every graph captured on
  // the stream tags its words differently and no in-graph memset is needed
  unsigned int* d_epoch = nullptr;
  // created inside a CUDA-graph capture: its buffers are baked into that graph, which
  // may replay many times, so per-launch state (tagged-carry epochs) is reset in-graph
  bool captured = false;
  std::vector<void*> retired;  // buffers outgrown during a capture (freed with the ctx)
  // device-path token_entropy scratch
  double* d_token_raw = nullptr;
  size_t token_raw_bytes = 0;
  double* d_token_range = nullptr;
  size_t token_range_bytes = 0;
  unsigned int* d_token_counts = nullptr;
  size_t token_counts_bytes = 0;
  // strided prefill: the sampled values gathered by cl_minmax_gather_f32
  float* d_samples = nullptr;
  size_t samples_bytes = 0;
};

struct cl_ctx {
  int device = 0;
  int num_sms = 148;
  std::atomic<uint64_t> launches{0};
  // one workspace per (stream handle, captured?): the stream's eager workspace and one for
  // everything captured on that stream; created on first use, freed with the context
  std::mutex ws_mu;
  std::map<std::pair<cudaStream_t, unsigned long long>, cl_workspace*> ws;
  // The host path (*_host) and its scratch: serialised per context, so the drop-in C++
  // API (one process-wide context) stays reentrant and thread-safe (reference SPEC.md:86).
  std::recursive_mutex host_mu;
  double* d_scratch_range = nullptr;   // 4 doubles
  uint64_t* d_scratch_counts = nullptr;  // up to kMaxBinsScratch
  cl_decision* d_scratch_decision = nullptr;
  double* d_token_out = nullptr;
  size_t token_out_bytes = 0;
  void* d_stage = nullptr;  // host-path upload buffer (grown on demand, reused across calls)
  size_t stage_bytes = 0;
  cudaStream_t own_stream = nullptr;
};

namespace cl {

constexpr int kMaxBinsScratch = 1 << 16;

// Set the calling thread's error message (cl_last_error) and return the code.
int fail(cl_ctx* ctx, int code, const std::string& msg);
int cuda_fail(cl_ctx* ctx, cudaError_t e, const char* where);
const std::string& thread_error();

// Zero a freshly allocated device buffer right now, outside any stream capture (on the
// context's own stream, synchronised), so graphs never replay an initialisation memset.
int zero_now(cl_ctx* ctx, void* p, size_t bytes);

// Zero a freshly allocated device buffer right now, outside any stream capture (on the
// context's own stream, synchronised), so graphs never replay an initialisation memset.
int zero_now(cl_ctx* ctx, void* p, size_t bytes);

// The workspace of `stream` (created on first use); nullptr + error on allocation failure.
// Inside a stream capture: the stream's captured workspace (shared by its captures).
cl_workspace* workspace(cl_ctx* ctx, cudaStream_t stream);
// id of the capture in progress on the stream, 0 when the stream is not capturing
unsigned long long capture_id_of(cudaStream_t stream);

// cudaMalloc is not allowed while a stream captures in the default (global) mode; a
// library may switch the calling thread to relaxed mode around its own allocations.
struct CaptureRelaxed {
  cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
  CaptureRelaxed() { cudaThreadExchangeStreamCaptureMode(&mode); }
  ~CaptureRelaxed() { cudaThreadExchangeStreamCaptureMode(&mode); }
};

template <typename T>
int grow_scratch(cl_ctx* ctx, cl_workspace* w, T** ptr, size_t* have, size_t need,
                 const char* what) {
  if (*have >= need) return 0;
  CaptureRelaxed relax;
  if (*ptr) {
    if (w && w->captured) w->retired.push_back(*ptr);  // no cudaFree inside a capture
    else cudaFree(*ptr);
  }
  *ptr = nullptr;
  *have = 0;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(ptr), need);
  if (e != cudaSuccess) return cuda_fail(ctx, e, what);
  *have = need;
  return 0;
}

// ---- kernel launchers (defined in the .cu files) ----
// entropy.cu
cudaError_t launch_range_init(double* d_range, cudaStream_t s);
cudaError_t launch_prefill_init(double* d_range, uint64_t* d_counts, int k, cudaStream_t s);
cudaError_t launch_minmax_f32(const float* v, uint64_t n, uint64_t g0, uint64_t stride,
                              double* d_range, int num_sms, cudaStream_t s, int* launches);
cudaError_t launch_minmax_f64(const double* v, uint64_t n, uint64_t g0, uint64_t stride,
                              double* d_range, int num_sms, cudaStream_t s, int* launches);
cudaError_t launch_minmax_gather_f32(const float* v, uint64_t n, uint64_t g0, uint64_t stride,
                                     double* d_range, float* d_samples, int num_sms,
                                     cudaStream_t s, int* launches);
// Histogram + decision in one launch (single-GPU prefill): the decision's inputs
// beyond the histogram's own.
struct HistFuse {
  uint64_t n_samples;
  const cl_rule_spec* rule;
  uint64_t seq_len;
  cl_decision* d_out;
  unsigned long long* ticket;  // the stream workspace's arrival ticket (0 on entry and exit)
};
cudaError_t launch_histogram_f32(const float* v, uint64_t n, uint64_t g0,
                                 const cl_hist_spec& spec, const double* d_range,
                                 uint64_t* d_counts, int num_sms, cudaStream_t s,
                                 int* launches, const HistFuse* fuse = nullptr,
                                 bool* fused = nullptr);
cudaError_t launch_histogram_f64(const double* v, uint64_t n, uint64_t g0,
                                 const cl_hist_spec& spec, const double* d_range,
                                 uint64_t* d_counts, int num_sms, cudaStream_t s,
                                 int* launches);
cudaError_t launch_decide(const uint64_t* d_counts, const double* d_range,
                          const cl_hist_spec& spec, uint64_t n_samples, const cl_rule_spec& rule,
                          uint64_t seq_len, const cl_features* features_or_null,
                          cl_decision* d_out, cudaStream_t s);
cudaError_t launch_decide_token(const double* d_token, const cl_hist_spec& spec,
                                const cl_rule_spec& rule, uint64_t seq_len, cl_decision* d_out,
                                cudaStream_t s);
cudaError_t launch_token_range_init(double* d_trange, double* d_flag, uint64_t length,
                                    cudaStream_t s);
template <typename T>
cudaError_t launch_token_minmax(const T* v, uint64_t channels, uint64_t length, uint64_t offset,
                                uint64_t stride, double* d_trange, double* d_flag, int num_sms,
                                cudaStream_t s);
template <typename T>
cudaError_t launch_token_hist(const T* v, uint64_t channels, uint64_t length, uint64_t offset,
                              const cl_hist_spec& spec, const double* d_trange,
                              unsigned int* d_counts, int num_sms, cudaStream_t s);
cudaError_t launch_token_entropy(const unsigned int* d_counts, uint64_t length,
                                 uint64_t n_per_pos, const cl_hist_spec& spec,
                                 const double* d_flag, double* d_raw_t, double* d_out,
                                 cudaStream_t s);
cudaError_t launch_entropy_from_masses(const double* d_masses, int k, double eps, double* d_out,
                                       cudaStream_t s);
bool launch_entropy_lean(const float* v, uint64_t n, const cl_hist_spec& spec,
                         const cl_rule_spec& rule, uint64_t seq_len, double* d_range,
                         uint64_t* d_counts, cl_decision* d_out, unsigned long long* ticket,
                         int num_sms, cudaStream_t s, cudaError_t* err);
bool launch_conv_hist_fixed(const float* x, const float* w, const float* bias, float* u,
                            uint64_t batch, uint64_t dim, uint64_t L, int width, int silu,
                            const cl_hist_spec& spec, uint64_t* d_counts, double* d_range,
                            int num_sms, cudaStream_t s, cudaError_t* err);
// conv1d.cu
cudaError_t launch_conv1d_f32(const float* x, const float* w, const float* bias, float* u,
                              uint64_t batch, uint64_t dim, uint64_t L, int width, int silu,
                              uint64_t g0, uint64_t stride, double* d_range, int num_sms,
                              cudaStream_t s);
// scan_f64.cu
cudaError_t launch_scan_f64(const cl_scan_params_f64& p, const double* d_h0, uint64_t chunk,
                            double* d_y, double* d_h, cudaStream_t s);
// scan_mamba1.cu
int scan_mamba1(cl_ctx* ctx, const cl_mamba1_args& a, const cl_decision* d_decision,
                int fixed_chunk, int variant, cudaStream_t s);
int state_update_f32(cl_ctx* ctx, const cl_state_update_args& a, cudaStream_t s);
int scan_plan(cl_ctx* ctx, const cl_mamba1_args& a, int variant, cl_scan_plan* p);
int scan_prepare_with_init(cl_ctx* ctx, const cl_mamba1_args& a, double* d_range,
                           uint64_t* d_counts, int bin_count, cudaStream_t s);

}  // namespace cl
