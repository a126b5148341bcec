// chunklab/mamba1.hpp -- additive extension of the drop-in API: the paper's prefill
// path on the B200 with device pointers, no host sync between
// the entropy estimate, the chunk decision and the fused Mamba-1 scan.
//
//   Prefill pf(spec, rule);           // scratch for counts / range / decision
//   pf.run(args, stream);             // minmax -> histogram -> decide -> scan
//   ChunkDecision d = pf.decision();  // sync point; throws deferred device errors
//
// selective_scan(args, chunk, stream) is mamba_ssm's selective_scan_fn with an
// explicit chunk (the paper's patched fwd_with_chunk_size);
// selective_state_update(args, stream) its one-token decode step (bitwise consistent
// with the scan); causal_conv1d(...) the conv1d + SiLU producer of u, optionally with
// the entropy min/max pass fused into it (d_range != nullptr).
#pragma once

#include <cuda_runtime.h>

#include "chunklab/chunk.hpp"
#include "chunklab/common.hpp"
#include "chunklab/entropy.hpp"

namespace chunklab {

using Mamba1Args = cl_mamba1_args;

inline void selective_scan(const Mamba1Args& args, int chunk, cudaStream_t stream = nullptr) {
  b200::check(cl_selective_scan_f32(b200::Runtime::get().ctx(), &args, nullptr, chunk,
                                    CL_SCAN_AUTO, stream));
}

using StateUpdateArgs = cl_state_update_args;

inline void selective_state_update(const StateUpdateArgs& args, cudaStream_t stream = nullptr) {
  b200::check(cl_selective_state_update_f32(b200::Runtime::get().ctx(), &args, stream));
}

inline void causal_conv1d(const float* d_x, const float* d_weight, const float* d_bias,
                          float* d_u, std::uint64_t batch, std::uint64_t dim,
                          std::uint64_t seq_len, int width, bool silu,
                          double* d_range = nullptr, std::uint64_t stride = 1,
                          cudaStream_t stream = nullptr) {
  b200::check(cl_conv1d_f32(b200::Runtime::get().ctx(), d_x, d_weight, d_bias, d_u, batch, dim,
                            seq_len, width, silu ? 1 : 0, 0, stride, d_range, stream));
}

class Prefill {
 public:
  // policy == nullptr: the bare calibrated rule select_chunk(H, bounds, cal)
  Prefill(const HistogramSpec& spec, const SchedulerPolicy* policy, const ChunkBounds& bounds,
          const CalibrationRef& cal)
      : spec_(detail::to_c(spec)) {
    rule_ = detail::base_rule(bounds, cal.h_ref_nats);
    if (!policy) {
      rule_.kind = CL_POL_RULE;
    } else {
      validate_policy(*policy);
      rule_.n_buckets = static_cast<int>(policy->bucket_set.size());
      for (int i = 0; i < rule_.n_buckets && i < 16; ++i) rule_.buckets[i] = policy->bucket_set[i];
      fill(policy->variant, /*inner=*/false);
    }
    cl_ctx* c = b200::Runtime::get().ctx();
    b200::check(cl_validate_hist_spec(c, &spec_));
    b200::check(cl_validate_rule(c, &rule_));
    check_cuda(cudaMalloc(&d_counts_, sizeof(std::uint64_t) * spec.bin_count));
    check_cuda(cudaMalloc(&d_range_, 4 * sizeof(double)));
    check_cuda(cudaMalloc(&d_decision_, sizeof(cl_decision)));
  }
  ~Prefill() {
    cudaFree(d_counts_);
    cudaFree(d_range_);
    cudaFree(d_decision_);
  }
  Prefill(const Prefill&) = delete;
  Prefill& operator=(const Prefill&) = delete;

  void run(const Mamba1Args& args, cudaStream_t stream = nullptr) {
    b200::check(cl_prefill_f32(b200::Runtime::get().ctx(), &args, &spec_, &rule_, d_counts_,
                               d_range_, d_decision_, stream));
    stream_ = stream;
  }

  // The prefill with its producer fused (cl_prefill_from_conv_f32): args.u is the buffer
  // the conv writes u = act(conv1d(conv.x)) into; the min/max (Dynamic range) or the whole
  // histogram (Fixed range) runs in the conv's epilogue.  Same bits as causal_conv1d + run.
  void run_from_conv(const cl_conv_args& conv, const Mamba1Args& args,
                     cudaStream_t stream = nullptr) {
    b200::check(cl_prefill_from_conv_f32(b200::Runtime::get().ctx(), &conv, &args, &spec_,
                                         &rule_, d_counts_, d_range_, d_decision_, stream));
    stream_ = stream;
  }

  ChunkDecision decision(EntropyEstimate* entropy = nullptr) const {
    cl_decision d{};
    b200::check(cl_decision_check(b200::Runtime::get().ctx(), d_decision_, &d, stream_));
    if (entropy) {
      entropy->raw_nats = d.raw_nats;
      entropy->normalized = d.normalized;
      entropy->bin_count = d.bin_count;
      entropy->sample_count = d.sample_count;
    }
    ChunkDecision out;
    out.chunk = d.chunk;
    out.r = d.r;
    out.source_policy = detail::source_tag(d.source);
    out.signal_nats = d.signal_nats;
    return out;
  }

  const cl_decision* device_decision() const { return d_decision_; }
  const std::uint64_t* device_counts() const { return d_counts_; }
  const double* device_range() const { return d_range_; }

 protected:
  static void check_cuda(cudaError_t e) {
    if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
  }
  void fill(const PolicyVariant& v, bool inner) {
    int kind;
    if (const auto* s = std::get_if<StaticPolicy>(&v)) {
      kind = CL_POL_STATIC;
      (inner ? rule_.inner_static_chunk : rule_.static_chunk) = s->chunk;
    } else if (std::holds_alternative<NoEntropyMidpointPolicy>(v)) {
      kind = CL_POL_MIDPOINT;
    } else if (std::holds_alternative<FullHistogramPolicy>(v)) {
      kind = CL_POL_FULL_HIST;
    } else if (std::holds_alternative<SampledHistogramPolicy>(v)) {
      kind = CL_POL_SAMPLED_HIST;
    } else if (std::holds_alternative<TokenHistogramPolicy>(v)) {
      kind = CL_POL_TOKEN_HIST;
    } else if (const auto* l = std::get_if<LearnedTablePolicy>(&v)) {
      kind = CL_POL_LEARNED_TABLE;
      rule_.threshold_tokens = l->threshold_tokens;
      rule_.short_chunk = l->short_chunk;
      rule_.long_chunk = l->long_chunk;
    } else if (const auto* g = std::get_if<GuardedPolicy>(&v)) {
      if (inner) throw invalid_input("nested guarded policies are not supported on the device path");
      kind = CL_POL_GUARDED;
      rule_.safe_chunk = g->safe_chunk;
      rule_.min_delta_buckets = g->min_delta_buckets;
      fill(g->inner->variant, /*inner=*/true);
    } else {
      throw invalid_input("policy needs host-side features; use Scheduler::decide");
    }
    (inner ? rule_.inner_kind : rule_.kind) = kind;
  }

  cl_hist_spec spec_{};
  cl_rule_spec rule_{};
  std::uint64_t* d_counts_ = nullptr;
  double* d_range_ = nullptr;
  cl_decision* d_decision_ = nullptr;
  cudaStream_t stream_ = nullptr;
};

// One rank of a row-sharded prefill (one process -- or thread -- per GPU):
// the rank owns `shard` of the global (batch, d_inner, L) tensors and `args` describe its
// local tensors.  run() is cl_prefill_sharded_f32: the two allreduces (range MAX, counts
// SUM) go through `coll` -- ShardedPrefill::nccl(comm) for NCCL over NVLink -- and every
// rank ends with the identical decision (decision() as for Prefill) and its rows' scan.
class ShardedPrefill : public Prefill {
 public:
  ShardedPrefill(const HistogramSpec& spec, const SchedulerPolicy* policy,
                 const ChunkBounds& bounds, const CalibrationRef& cal, const cl_shard& shard,
                 const cl_collectives& coll)
      : Prefill(spec, policy, bounds, cal), shard_(shard), coll_(coll) {}

  void run(const Mamba1Args& local_args, cudaStream_t stream = nullptr) {
    b200::check(cl_prefill_sharded_f32(b200::Runtime::get().ctx(), &local_args, &shard_, &spec_,
                                       &rule_, &coll_, d_counts_, d_range_, d_decision_, stream));
    stream_ = stream;
  }

  // Hooks over an NCCL communicator (ncclComm_t; NCCL 2.27 in this image).
  static cl_collectives nccl(void* nccl_comm) {
    cl_collectives c{};
    b200::check(cl_collectives_nccl(nccl_comm, &c));
    return c;
  }

  // The shard of `rank` in a world of `world` ranks: whole batches when world divides the
  // batch (C3, C4), else a contiguous d_inner range of every batch (C1, C2).
  static cl_shard plan(std::uint64_t batch, std::uint64_t dim, int rank, int world) {
    cl_shard s{};
    s.global_batch = batch;
    s.global_dim = dim;
    if (world < 1 || rank < 0 || rank >= world) throw invalid_input("bad rank/world");
    const auto w = static_cast<std::uint64_t>(world), r = static_cast<std::uint64_t>(rank);
    if (batch % w == 0) {
      s.b0 = r * (batch / w);
      s.b1 = s.b0 + batch / w;
      s.d0 = 0;
      s.d1 = dim;
    } else if (dim % w == 0) {
      s.b0 = 0;
      s.b1 = batch;
      s.d0 = r * (dim / w);
      s.d1 = s.d0 + dim / w;
    } else {
      throw invalid_input("neither batch nor d_inner divisible by world size");
    }
    return s;
  }

 private:
  cl_shard shard_;
  cl_collectives coll_;
};

}  // namespace chunklab
