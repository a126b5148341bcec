// sharded.cu -- the multi-GPU prefill entry point of the C-ABI:
// cl_prefill_sharded_f32 runs one rank's share of a row-sharded layer call and places
// the two collectives of the protocol exactly where they belong, through caller-supplied
// stream-ordered hooks (cl_collectives); cl_collectives_nccl fills those hooks with
// ncclAllReduce on an NCCL communicator (libnccl.so.2, loaded on first use, so the
// library itself runs without NCCL installed).
//
//   prefill_init(range, counts)
//   minmax over every local segment, stride sampling by GLOBAL flat index
//   -> allreduce MAX(range, 4 doubles)         {-lo, hi, nonfinite, 0}
//   histogram over every local segment (global offsets)
//   -> allreduce SUM(counts, K uint64)
//   decide (every rank: identical inputs, identical device decision -- no broadcast)
//   scan of the local rows
//
// TokenHistogram policies use the per-position buffers instead: MAX over [2L + 1] doubles,
// SUM over [L][K] uint32.  The reference has no multi-GPU path (request-level DP only,
// PAPER.md:1366-1392); this is the north star's "(4) channel-sharded ... the only
// collective is an NCCL allreduce of the K-bin histogram counts" plus the range
// MAX-allreduce that Dynamic-range bit-exactness needs (DESIGN.md (e)).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>
#include <vector>

#include "cl_internal.h"

namespace cl {
namespace {

struct Segment {
  uint64_t local_offset, global_offset, numel;
};

// The rank's rows as contiguous runs of the global (batch * dim, L) flattening.
int plan_segments(cl_ctx* ctx, const cl_mamba1_args& a, const cl_shard& sh,
                  std::vector<Segment>* out) {
  const uint64_t L = a.seq_len, D = sh.global_dim;
  if (sh.b1 <= sh.b0 || sh.d1 <= sh.d0 || sh.b1 > sh.global_batch || sh.d1 > D)
    return fail(ctx, CL_E_INVALID, "invalid shard");
  if (a.batch != sh.b1 - sh.b0 || a.dim != sh.d1 - sh.d0)
    return fail(ctx, CL_E_INVALID, "shape mismatch");
  out->clear();
  if (sh.d0 == 0 && sh.d1 == D) {  // whole batches: one run
    out->push_back({0, sh.b0 * D * L, a.batch * D * L});
  } else {  // a channel range of each owned batch
    const uint64_t ld = sh.d1 - sh.d0;
    for (uint64_t b = 0; b < a.batch; ++b)
      out->push_back({b * ld * L, ((sh.b0 + b) * D + sh.d0) * L, ld * L});
  }
  return CL_OK;
}

int hook(cl_ctx* ctx, int rc, const char* what) {
  if (rc == CL_OK) return CL_OK;
  const std::string prior = thread_error();
  return fail(ctx, rc == CL_E_INVALID ? CL_E_INVALID : CL_E_CUDA,
              std::string(what) + (prior.empty() ? "" : ": " + prior));
}

// ---- NCCL binding (dlopen'ed) ----
using AllReduceFn = ncclResult_t (*)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
                                     ncclComm_t, cudaStream_t);
using ErrorStringFn = const char* (*)(ncclResult_t);
AllReduceFn g_allreduce = nullptr;
ErrorStringFn g_errstr = nullptr;

bool load_nccl() {
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    g_allreduce = reinterpret_cast<AllReduceFn>(dlsym(h, "ncclAllReduce"));
    g_errstr = reinterpret_cast<ErrorStringFn>(dlsym(h, "ncclGetErrorString"));
  });
  return g_allreduce != nullptr;
}

int nccl_call(ncclResult_t r) {
  if (r == ncclSuccess) return CL_OK;
  return fail(nullptr, CL_E_CUDA,
              std::string("ncclAllReduce: ") + (g_errstr ? g_errstr(r) : "error"));
}

int nccl_max_f64(double* d, size_t n, void* stream, void* comm) {
  return nccl_call(g_allreduce(d, d, n, ncclFloat64, ncclMax, static_cast<ncclComm_t>(comm),
                               static_cast<cudaStream_t>(stream)));
}
int nccl_sum_u64(uint64_t* d, size_t n, void* stream, void* comm) {
  return nccl_call(g_allreduce(d, d, n, ncclUint64, ncclSum, static_cast<ncclComm_t>(comm),
                               static_cast<cudaStream_t>(stream)));
}
int nccl_sum_u32(uint32_t* d, size_t n, void* stream, void* comm) {
  return nccl_call(g_allreduce(d, d, n, ncclUint32, ncclSum, static_cast<ncclComm_t>(comm),
                               static_cast<cudaStream_t>(stream)));
}

}  // namespace
}  // namespace cl

using namespace cl;

extern "C" {

int cl_collectives_nccl(void* nccl_comm, cl_collectives* out) {
  if (!nccl_comm || !out) return fail(nullptr, CL_E_INVALID, "null argument");
  if (!load_nccl()) return fail(nullptr, CL_E_CUDA, "libnccl.so.2 not found");
  out->allreduce_max_f64 = nccl_max_f64;
  out->allreduce_sum_u64 = nccl_sum_u64;
  out->allreduce_sum_u32 = nccl_sum_u32;
  out->user = nccl_comm;
  return CL_OK;
}

int cl_prefill_sharded_f32(cl_ctx* ctx, const cl_mamba1_args* args, const cl_shard* shard,
                           const cl_hist_spec* spec, const cl_rule_spec* rule,
                           const cl_collectives* coll, uint64_t* d_counts, double* d_range,
                           cl_decision* d_decision, void* stream) {
  if (!ctx || !args || !shard || !d_counts || !d_range || !d_decision)
    return fail(ctx, CL_E_INVALID, "null argument");
  if (!coll || !coll->allreduce_max_f64 || !coll->allreduce_sum_u64)
    return fail(ctx, CL_E_INVALID, "sharded prefill needs allreduce hooks");
  int rc = cl_validate_hist_spec(ctx, spec);
  if (!rc) rc = cl_validate_rule(ctx, rule);
  if (rc) return rc;
  std::vector<Segment> segs;
  if ((rc = plan_segments(ctx, *args, *shard, &segs))) return rc;
  const uint64_t L = args->seq_len;
  const uint64_t n_global = shard->global_batch * shard->global_dim * L;
  if (n_global == 0) return fail(ctx, CL_E_INVALID, "no samples");
  const float* u = args->u;
  const int kind = rule->kind == CL_POL_GUARDED ? rule->inner_kind : rule->kind;
  if (kind == CL_POL_TOKEN_HIST) {
    // token_entropy (entropy.hpp:180-210) over channels = all global rows; every rank
    // holds all L positions of its rows.  Per-position buffers in the stream workspace.
    if (!coll->allreduce_sum_u32)
      return fail(ctx, CL_E_INVALID, "token policy needs the uint32 SUM hook");
    cl_workspace* w = workspace(ctx, static_cast<cudaStream_t>(stream));
    if (!w) return CL_E_CUDA;
    const int k = spec->bin_count;
    if (k > 4096) return fail(ctx, CL_E_INVALID, "token entropy supports bin_count <= 4096");
    if ((rc = grow_scratch(ctx, w, &w->d_token_range, &w->token_range_bytes,
                           (2 * L + 1) * sizeof(double), "cudaMalloc(token range)")) ||
        (rc = grow_scratch(ctx, w, &w->d_token_counts, &w->token_counts_bytes,
                           L * size_t(k) * sizeof(uint32_t), "cudaMalloc(token counts)")))
      return rc;
    if ((rc = cl_token_range_init(ctx, w->d_token_range, L, stream))) return rc;
    for (const Segment& s : segs)
      if ((rc = cl_token_minmax_f32(ctx, u + s.local_offset, s.numel / L, L, s.global_offset / L,
                                    spec->sample_stride, w->d_token_range, stream)))
        return rc;
    if ((rc = hook(ctx, coll->allreduce_max_f64(w->d_token_range, 2 * L + 1, stream, coll->user),
                   "allreduce_max_f64(token range)")))
      return rc;
    cudaError_t e = cudaMemsetAsync(w->d_token_counts, 0, L * size_t(k) * sizeof(uint32_t),
                                    static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMemsetAsync(token counts)");
    for (const Segment& s : segs)
      if ((rc = cl_token_histogram_f32(ctx, u + s.local_offset, s.numel / L, L,
                                       s.global_offset / L, spec, w->d_token_range,
                                       w->d_token_counts, stream)))
        return rc;
    if ((rc = hook(ctx, coll->allreduce_sum_u32(w->d_token_counts, L * size_t(k), stream,
                                                coll->user),
                   "allreduce_sum_u32(token counts)")))
      return rc;
    const uint64_t channels = shard->global_batch * shard->global_dim;
    const uint64_t per_pos = (channels + spec->sample_stride - 1) / spec->sample_stride;
    if ((rc = cl_token_entropy_counts(ctx, w->d_token_counts, w->d_token_range, L, per_pos, spec,
                                      d_range, stream)) ||
        (rc = cl_decide_token(ctx, d_range, spec, rule, L, d_decision, stream)))
      return rc;
    return cl_selective_scan_f32(ctx, args, d_decision, 0, CL_SCAN_AUTO, stream);
  }
  if ((rc = cl_prefill_init_prepare_f32(ctx, d_range, d_counts, spec->bin_count, args, stream)))
    return rc;
  const bool gather = spec->sample_stride >= CL_GATHER_MIN_STRIDE;
  if (gather) {
    // as cl_prefill_f32: min/max gathers every segment's samples (consecutively; the
    // counts do not depend on their order) and the histogram reads only those
    cl_workspace* w = workspace(ctx, static_cast<cudaStream_t>(stream));
    if (!w) return CL_E_CUDA;
    uint64_t m = 0;
    for (const Segment& s : segs) m += cl_samples_in(s.global_offset, s.numel, spec->sample_stride);
    if ((rc = grow_scratch(ctx, w, &w->d_samples, &w->samples_bytes, (m ? m : 1) * sizeof(float),
                           "cudaMalloc(gathered samples)")))
      return rc;
    uint64_t at = 0;
    for (const Segment& s : segs) {
      if ((rc = cl_minmax_gather_f32(ctx, u + s.local_offset, s.numel, s.global_offset,
                                     spec->sample_stride, d_range, w->d_samples + at, stream)))
        return rc;
      at += cl_samples_in(s.global_offset, s.numel, spec->sample_stride);
    }
    if ((rc = hook(ctx, coll->allreduce_max_f64(d_range, 4, stream, coll->user),
                   "allreduce_max_f64(range)")))
      return rc;
    cl_hist_spec s1 = *spec;
    s1.sample_stride = 1;
    if (m && (rc = cl_histogram_f32(ctx, w->d_samples, m, 0, &s1, d_range, d_counts, stream)))
      return rc;
  } else {
    for (const Segment& s : segs)
      if ((rc = cl_minmax_f32(ctx, u + s.local_offset, s.numel, s.global_offset,
                              spec->sample_stride, d_range, stream)))
        return rc;
    if ((rc = hook(ctx, coll->allreduce_max_f64(d_range, 4, stream, coll->user),
                   "allreduce_max_f64(range)")))
      return rc;
    for (const Segment& s : segs)
      if ((rc = cl_histogram_f32(ctx, u + s.local_offset, s.numel, s.global_offset, spec, d_range,
                                 d_counts, stream)))
        return rc;
  }
  if ((rc = hook(ctx,
                 coll->allreduce_sum_u64(d_counts, size_t(spec->bin_count), stream, coll->user),
                 "allreduce_sum_u64(counts)")))
    return rc;
  const uint64_t n_samples = (n_global + spec->sample_stride - 1) / spec->sample_stride;
  if ((rc = cl_decide(ctx, d_counts, d_range, spec, n_samples, rule, L, d_decision, stream)))
    return rc;
  return cl_selective_scan_f32(ctx, args, d_decision, 0, CL_SCAN_AUTO, stream);
}

}  // extern "C"
