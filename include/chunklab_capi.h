/*
 * chunklab_capi.h -- C-ABI of the B200-native COREY hot path (libchunklab_b200.so).
 *
 * The reference boundary is the header-only C++ API in
 * /root/reference/proj/include/chunklab (namespace chunklab).  This C-ABI is
 * what that API compiles down to in this repo: include/chunklab/*.hpp are
 * drop-in replacements for the reference headers implemented on top of the
 * entry points below, and every compute entry point runs on the GPU
 * (sm_100a kernels in paper_2604_10597_b200/csrc/).  There is no CPU path.
 *
 * Conventions
 *   - Every function returns int status: CL_OK (0) or a CL_E_* code; the
 *     message is available from cl_last_error() on the calling thread
 *     (errno-style) and, for CL_E_INVALID, is byte-identical to the reference's
 *     chunklab::invalid_input what().
 *   - "d_" pointers are device pointers, "h_" pointers are host pointers.
 *     Buffers are caller-owned; scratch belongs to the context.
 *   - Threads and streams (the reference's functions are pure and reentrant,
 *     SPEC.md:86): a context may be shared by any number of host threads.  Its
 *     device scratch (scan work tickets and carries, the B/C transpose, the
 *     fused histogram's arrival ticket, token-entropy buffers) is kept per
 *     stream, so launch sequences on different streams never share scratch;
 *     work captured into CUDA graphs on a stream uses a second workspace of that
 *     stream (so graph replays and eager launches never share scratch either); the
 *     host path (*_host) is serialised on the context.
 *   - Device-path functions (cl_minmax_f32 ... cl_selective_scan_f32) are
 *     asynchronous on the given cudaStream_t (passed as void*) and never
 *     synchronise with the host.  Errors only the device can see
 *     (non-finite input, negative signal) are written into the device-side
 *     cl_decision.status word and surface at cl_decision_check().
 *   - Host-path functions (suffix _host) take host buffers, synchronise, and
 *     are the building blocks of the drop-in C++ headers.
 *   - Multi-GPU: the caller runs the stages on each rank and
 *     performs two collectives between them: MAX-allreduce of the 4-double
 *     range buffer after cl_minmax_*, SUM-allreduce of the uint64 counts
 *     after cl_histogram_*.  Every rank then derives the identical decision.
 */
#ifndef CHUNKLAB_CAPI_H
#define CHUNKLAB_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CL_ABI_VERSION 1

enum cl_status {
  CL_OK = 0,
  CL_E_INVALID = 1, /* chunklab::invalid_input (message verbatim)            */
  CL_E_CUDA = 2,    /* CUDA runtime / launch failure                          */
  CL_E_DEVICE = 3,  /* device-detected error surfaced by cl_decision_check()  */
  CL_E_NOMEM = 4
};

/* Device-side error codes carried in cl_decision.status (0 = ok). */
enum cl_device_error {
  CL_DEV_OK = 0,
  CL_DEV_NON_FINITE = 1, /* "non-finite input"    entropy.hpp:42 / :110        */
  CL_DEV_NO_SAMPLES = 2, /* "no samples"          entropy.hpp:115              */
  CL_DEV_SIGNAL = 3      /* "signal must be >= 0" chunk.hpp:72 (constant input) */
};

typedef struct cl_ctx cl_ctx;

/* ------------------------------------------------------------------------ */
/* Context                                                                   */
/* ------------------------------------------------------------------------ */
int cl_ctx_create(int device, cl_ctx** out);
int cl_ctx_destroy(cl_ctx* ctx);
/* Message of the calling thread's last failed call (ctx may be NULL). */
const char* cl_last_error(const cl_ctx* ctx);
int cl_abi_version(void);
/* Number of kernel launches this context has issued (bench evidence). */
uint64_t cl_launch_count(const cl_ctx* ctx);

/* ------------------------------------------------------------------------ */
/* Specs (POD mirrors of the reference structs)                              */
/* ------------------------------------------------------------------------ */
enum { CL_RANGE_DYNAMIC = 0, CL_RANGE_FIXED = 1 };

/* HistogramSpec, entropy.hpp:47-54 (defaults K=256, eps=1e-8, Dynamic, stride 1). */
typedef struct {
  int bin_count;
  double epsilon;
  int range_mode;
  double fixed_lo, fixed_hi;
  uint64_t sample_stride;
} cl_hist_spec;

/* Policy kinds (chunk.hpp:101-142, the on-device subset). */
enum {
  CL_POL_STATIC = 0,
  CL_POL_MIDPOINT = 1,
  CL_POL_FULL_HIST = 2,
  CL_POL_SAMPLED_HIST = 3,
  CL_POL_LEARNED_TABLE = 4,
  CL_POL_GUARDED = 5,
  CL_POL_RULE = 6, /* bare select_chunk (chunk.hpp:68-89), no bucket snap */
  CL_POL_TOKEN_HIST = 7 /* TokenHistogramPolicy (chunk.hpp:311-315): rule on token_entropy */
};

/* Source tags (ChunkDecision::source_policy, chunk.hpp:265-368):
 * 0 "static", 1 "no_entropy_midpoint", 2 "full_histogram", 3 "sampled_histogram",
 * 4 "learned_table", 6 "rule"; 16+k "guarded[<k>]"; 32 "guarded[fallback]". */
enum { CL_SRC_GUARDED = 16, CL_SRC_GUARDED_FALLBACK = 32 };

/* ChunkBounds (chunk.hpp:29-32) + CalibrationRef (chunk.hpp:42-59) + SchedulerPolicy. */
typedef struct {
  int kind;
  int static_chunk;          /* StaticPolicy::chunk */
  int inner_kind;            /* GuardedPolicy::inner (non-guarded kind) */
  int inner_static_chunk;
  int safe_chunk;            /* GuardedPolicy::safe_chunk (512) */
  int min_delta_buckets;     /* GuardedPolicy::min_delta_buckets (2) */
  uint64_t threshold_tokens; /* LearnedTablePolicy (50, 128, 512) */
  int short_chunk, long_chunk;
  int n_buckets;             /* SchedulerPolicy::bucket_set, <= 16 */
  int buckets[16];
  int c_min, c_max;          /* ChunkBounds */
  double h_ref_nats;         /* CalibrationRef::h_ref_nats (log K or legacy) */
} cl_rule_spec;

/* Decision record written by the device (ChunkDecision + EntropyEstimate + Histogram scalars). */
typedef struct {
  int32_t status;        /* cl_device_error */
  int32_t chunk;         /* ChunkDecision::chunk */
  int32_t source;        /* source tag */
  int32_t bin_count;
  double r;              /* ChunkDecision::r */
  double signal_nats;    /* ChunkDecision::signal_nats */
  double raw_nats;       /* EntropyEstimate::raw_nats */
  double normalized;     /* EntropyEstimate::normalized */
  double lo, hi;         /* Histogram::lo/hi */
  uint64_t sample_count; /* Histogram::sample_count */
  double margin;         /* |log2(target) - (e - 0.5)|: knife-edge diagnostic */
} cl_decision;

/* ------------------------------------------------------------------------ */
/* Device path (async, stream-ordered; the prefill hot path)                 */
/* ------------------------------------------------------------------------ */
/* Stage 1 (entropy.hpp:108-114): strided min/max over the samples whose GLOBAL
 * flat index (global_offset + i) is a multiple of stride, and a finite check
 * over EVERY element (entropy.hpp:42).  d_range (4 doubles, MAX-allreducible):
 * {-lo, hi, nonfinite(0/1), 0}.  Initialise with cl_range_init. */
int cl_range_init(cl_ctx* ctx, double* d_range, void* stream);
int cl_minmax_f32(cl_ctx* ctx, const float* d_values, uint64_t n, uint64_t global_offset,
                  uint64_t stride, double* d_range, void* stream);
int cl_minmax_f64(cl_ctx* ctx, const double* d_values, uint64_t n, uint64_t global_offset,
                  uint64_t stride, double* d_range, void* stream);
/* cl_minmax_f32 that also writes every sampled value, in index order, to d_samples:
 * d_samples[j] = d_values[i] for the j-th i whose global index (global_offset + i) is a
 * multiple of stride (capacity: cl_samples_in(global_offset, n, stride) floats).  A
 * strided histogram of d_samples with stride 1 counts exactly what the strided
 * histogram of d_values counts, reading n / stride values instead of n; cl_prefill_f32
 * takes this path for stride >= 4. */
#define CL_GATHER_MIN_STRIDE 4
int cl_minmax_gather_f32(cl_ctx* ctx, const float* d_values, uint64_t n,
                         uint64_t global_offset, uint64_t stride, double* d_range,
                         float* d_samples, void* stream);
/* Number of global indices in [global_offset, global_offset + n) that are multiples of
 * stride (0 for stride 0). */
uint64_t cl_samples_in(uint64_t global_offset, uint64_t n, uint64_t stride);

/* Producer fusion (no reference counterpart -- the paper's u comes
 * out of mamba_ssm's causal_conv1d_fn):
 *   u[b,d,t] = act(bias[d] + sum_{k<width} weight[d,k] * x[b,d,t-width+1+k])
 * with x zero before t = 0, act = SiLU (silu != 0) or identity; x, u (batch, dim,
 * seq_len) fp32, weight (dim, width), bias (dim) or NULL, width in [1, 4].  When
 * d_range is not NULL the kernel also performs cl_minmax_f32 over the u it writes
 * (same global_offset / stride semantics, same d_range protocol), so the separate
 * min/max pass -- one full read of u -- disappears from the prefill. */
int cl_conv1d_f32(cl_ctx* ctx, const float* d_x, const float* d_weight, const float* d_bias,
                  float* d_u, uint64_t batch, uint64_t dim, uint64_t seq_len, int width,
                  int silu, uint64_t global_offset, uint64_t stride, double* d_range,
                  void* stream);

/* Stage 2 (entropy.hpp:116-126): accumulate K uint64 counts of the strided
 * samples, binned exactly as detail::bin_index (entropy.hpp:87-94) over the
 * (global) range in d_range, or the spec's fixed range.  d_counts must be
 * zeroed first (cl_counts_zero) when starting a new histogram. */
int cl_counts_zero(cl_ctx* ctx, uint64_t* d_counts, int bin_count, void* stream);
/* cl_range_init + cl_counts_zero as one launch (the first node of a prefill). */
int cl_prefill_init(cl_ctx* ctx, double* d_range, uint64_t* d_counts, int bin_count, void* stream);
int cl_histogram_f32(cl_ctx* ctx, const float* d_values, uint64_t n, uint64_t global_offset,
                     const cl_hist_spec* spec, const double* d_range, uint64_t* d_counts,
                     void* stream);
int cl_histogram_f64(cl_ctx* ctx, const double* d_values, uint64_t n, uint64_t global_offset,
                     const cl_hist_spec* spec, const double* d_range, uint64_t* d_counts,
                     void* stream);

/* Stage 3 (entropy.hpp:149-164 + chunk.hpp:68-89/256-368): masses, entropy,
 * rule, bucket snap, guarded / learned-table policy -> d_decision.
 * n_samples_total = number of samples over all ranks (ceil(N_global/stride)).
 * seq_len feeds the learned-table policy. */
int cl_decide(cl_ctx* ctx, const uint64_t* d_counts, const double* d_range,
              const cl_hist_spec* spec, uint64_t n_samples_total, const cl_rule_spec* rule,
              uint64_t seq_len, cl_decision* d_decision, void* stream);

/* Stages 2+3 in one launch for a single-GPU call (no collective between them):
 * cl_histogram_f32 over all n values (global_offset 0) followed by cl_decide with
 * n_samples_total = ceil(n / stride), same results bit for bit.  Where the
 * register-fed histogram applies (K <= 256, Dynamic range, stride 1, n >= 4096) its
 * last CTA writes the decision; otherwise the two kernels run back to back.
 * d_range from cl_range_init + cl_minmax_f32 of this call; d_counts zeroed as for
 * cl_histogram_f32.  The CTAs' arrival ticket lives in the stream's workspace.  Replaces the compute_histogram -> estimate_entropy ->
 * select_chunk sequence of entropy.hpp:101-174 / chunk.hpp:68-89. */
int cl_histogram_decide_f32(cl_ctx* ctx, const float* d_values, uint64_t n,
                            const cl_hist_spec* spec, const double* d_range, uint64_t* d_counts,
                            const cl_rule_spec* rule, uint64_t seq_len, cl_decision* d_decision,
                            void* stream);

/* The entropy stages of a single-GPU prefill (range init, min/max, histogram + decision;
 * results identical to cl_prefill_init + cl_minmax_f32 + cl_histogram_decide_f32) in LEAN
 * kernels: one CTA per SM of 4 warps, <= 64 registers per thread and ~66 KB of shared
 * memory, fed by cp.async.bulk rings -- small enough to run on the same SMs as another
 * call's scan.  For pipelined serving: call i+1's entropy on one stream while call i's
 * MUFU-bound scan runs on another (the scan leaves about half of HBM idle).  Configurations
 * other than Dynamic range, stride 1, K <= 256 use the regular kernels. */
int cl_entropy_lean_f32(cl_ctx* ctx, const float* d_values, uint64_t n, const cl_hist_spec* spec,
                        const cl_rule_spec* rule, uint64_t seq_len, uint64_t* d_counts,
                        double* d_range, cl_decision* d_decision, void* stream);

/* Stage 4: fused Mamba-1 selective scan (fp32), chunk read from d_decision.
 * Layouts (mamba_ssm selective_scan_fn): u, delta, z, out: (batch, dim, L)
 * row-major; A: (dim, N); B, C: (batch, N, L); D, delta_bias: (dim) or NULL;
 * z NULL -> no gate; h0 NULL -> zeros; h_last (batch, dim, N) or NULL.
 * N must be 16 on the TMA fast path, <= 64 in general. */
typedef struct {
  const float* u;
  const float* delta;
  const float* A;
  const float* B;
  const float* C;
  const float* D;
  const float* z;
  const float* delta_bias;
  const float* h0;
  float* out;
  float* h_last;
  uint64_t batch, dim, seq_len, d_state;
  int delta_softplus;
} cl_mamba1_args;

/* Scan variants.  CL_SCAN_AUTO picks by shape: the chained-carry kernels for shapes with
 * enough 16-row tiles to fill the GPU, the L-parallel kernel (scan_lookback.cu) for few
 * rows.  Every chained variant (CL_SCAN_ROWSEQ_TMA, CL_SCAN_GENERIC, CL_SCAN_CHAINED,
 * CL_SCAN_CONFIG_BASE + i = row i of scan_mamba1.cu's kCfgs) gives the same bits for every
 * chunk.  The L-parallel kernel splits L by the shape, never by the chunk, so its bits are
 * also chunk-independent; against the chained kernels it agrees to rounding (<= 1e-6
 * normwise: the segment carry-in is a fold of segment aggregates).  CL_SCAN_LOOKBACK
 * forces it, CL_SCAN_LOOKBACK_BASE + i forces its table row i. */
enum {
  CL_SCAN_AUTO = 0,
  CL_SCAN_ROWSEQ_TMA = 1,
  CL_SCAN_GENERIC = 2,
  CL_SCAN_LOOKBACK = 3,
  CL_SCAN_CHAINED = 4,
  CL_SCAN_CONFIG_BASE = 16,
  CL_SCAN_LOOKBACK_BASE = 64
};
int cl_selective_scan_f32(cl_ctx* ctx, const cl_mamba1_args* args, const cl_decision* d_decision,
                          int fixed_chunk /* used when d_decision == NULL */, int variant,
                          void* stream);

/* cl_prefill_init plus the scan's B / C re-layout for `scan_args` in the same launch: the
 * next cl_selective_scan_f32 on this stream with the same B, C, batch and seq_len reuses it
 * instead of launching its own transpose (B and C must not change in between). */
int cl_prefill_init_prepare_f32(cl_ctx* ctx, double* d_range, uint64_t* d_counts, int bin_count,
                                const cl_mamba1_args* scan_args, void* stream);

/* Which kernel cl_selective_scan_f32 runs for these arguments and variant (host-only
 * query, no launch): kernel kind, its table row, TMA box (timesteps), consumer warps per
 * CTA, ring stages, and for the L-parallel kernel its shape-tied split (n_seg segments of
 * seg_len timesteps; -1 for the chained kernels, whose segment is the decided chunk). */
enum { CL_KERNEL_GENERIC = 0, CL_KERNEL_CHAINED = 1, CL_KERNEL_ROWSEQ = 2, CL_KERNEL_LOOKBACK = 3 };
typedef struct {
  int kernel, config, box, warps, stages, n_seg, seg_len;
} cl_scan_plan;
int cl_scan_plan_f32(cl_ctx* ctx, const cl_mamba1_args* args, int variant, cl_scan_plan* out);

/* Single-GPU convenience: range_init -> minmax -> histogram -> decide -> scan,
 * all on one stream, no host sync.  d_counts: K uint64 scratch; d_range: 4 doubles. */
int cl_prefill_f32(cl_ctx* ctx, const cl_mamba1_args* args, const cl_hist_spec* spec,
                   const cl_rule_spec* rule, uint64_t* d_counts, double* d_range,
                   cl_decision* d_decision, void* stream);

/* ------------------------------------------------------------------------ */
/* Multi-GPU: one rank's share of a row-sharded layer call      */
/* ------------------------------------------------------------------------ */
/* The rank owns batches [b0, b1) x channels [d0, d1) of the global (global_batch,
 * global_dim, L) tensors: whole batches (d0 = 0, d1 = global_dim; C3/C4 plans) or a
 * channel range of every batch (b0 = 0, b1 = global_batch; C1/C2 plans, B and C
 * replicated).  args describe the LOCAL tensors ((b1-b0), (d1-d0), L). */
typedef struct {
  uint64_t global_batch, global_dim;
  uint64_t b0, b1, d0, d1;
} cl_shard;

/* Stream-ordered in-place allreduce hooks (device buffers, enqueued on `stream`; return
 * CL_OK or a CL_E_* code).  cl_collectives_nccl binds them to ncclAllReduce; any other
 * transport (MPI, a host-staged test harness) fills them itself. */
typedef struct {
  int (*allreduce_max_f64)(double* d_buf, size_t count, void* stream, void* user);
  int (*allreduce_sum_u64)(uint64_t* d_buf, size_t count, void* stream, void* user);
  int (*allreduce_sum_u32)(uint32_t* d_buf, size_t count, void* stream, void* user);
  void* user;
} cl_collectives;

/* Hooks calling ncclAllReduce on the communicator (an ncclComm_t passed as void*);
 * libnccl.so.2 is loaded on first use. */
int cl_collectives_nccl(void* nccl_comm, cl_collectives* out);

/* One rank's prefill: prefill_init -> min/max of every local run (stride sampling by
 * GLOBAL flat index) -> allreduce MAX(d_range, 4) -> histogram -> allreduce SUM(d_counts,
 * K) -> device decision (identical on every rank) -> scan of the local rows.
 * TokenHistogram policies: MAX over the [2L+1] per-position range, SUM over the [L][K]
 * uint32 counts (stream workspace), then the token decision.  Counts, range and the
 * decision equal the single-GPU call's bit for bit. */
int cl_prefill_sharded_f32(cl_ctx* ctx, const cl_mamba1_args* local_args, const cl_shard* shard,
                           const cl_hist_spec* spec, const cl_rule_spec* rule,
                           const cl_collectives* coll, uint64_t* d_counts, double* d_range,
                           cl_decision* d_decision, void* stream);

/* The prefill with its producer fused ("deeper
 * kernel fusion of the entropy estimator"): u = act(causal_conv1d(x)) is produced into
 * args->u (a caller buffer, (batch, dim, L)) and the entropy estimate rides on it:
 *   Dynamic range: conv with the min/max epilogue -> histogram + decision -> scan
 *                  (u is read once for the histogram instead of twice);
 *   Fixed range:   conv with the HISTOGRAM epilogue (bin edges are known before u exists)
 *                  -> decision -> scan (u is never re-read for the entropy);
 *   TokenHistogram policies: conv -> token entropy -> decision -> scan.
 * Results (u, counts, decision, scan output) equal cl_conv1d_f32 + cl_prefill_f32 bit for
 * bit. */
typedef struct {
  const float* x;      /* (batch, dim, L) conv input */
  const float* weight; /* (dim, width) */
  const float* bias;   /* (dim) or NULL */
  int width;           /* 1..4 */
  int silu;            /* activation: SiLU (1) or identity (0) */
} cl_conv_args;
int cl_prefill_from_conv_f32(cl_ctx* ctx, const cl_conv_args* conv, const cl_mamba1_args* args,
                             const cl_hist_spec* spec, const cl_rule_spec* rule,
                             uint64_t* d_counts, double* d_range, cl_decision* d_decision,
                             void* stream);

/* Sync point: copy the decision to the host and convert a device error into
 * CL_E_DEVICE with the reference's message. */
int cl_decision_check(cl_ctx* ctx, const cl_decision* d_decision, cl_decision* h_out,
                      void* stream);

/* fp64 reference-mode recurrence on device (scan.hpp:77-136), bit-identical
 * to chunklab::scan_sequential / scan_chunked: h = a*h + b*x; out += c*h;
 * y = out + d*x, no FMA contraction, state order s = 0..N-1.
 * a: d*N (constant) or L*d*N [t][c][s]; b, c: N or L*N [t][s]; d: channels;
 * x: [c][t].  h0 NULL -> zeros.  chunk 0 -> sequential. */
typedef struct {
  uint64_t channels, state_dim, seq_len;
  const double *a, *b, *c, *d, *x;
  uint64_t a_len, b_len, c_len, d_len, x_len;
} cl_scan_params_f64;
int cl_scan_f64(cl_ctx* ctx, const cl_scan_params_f64* d_params, const double* d_h0,
                uint64_t chunk, double* d_y, double* d_h, void* stream);

/* Decode step: one token per (b, d) row through the Mamba-1
 * recurrence, state updated in place -- mamba_ssm selective_state_update(state, x, dt,
 * A, B, C, D, z, dt_bias, dt_softplus).  state (batch, dim, d_state); x, dt, z, out
 * (batch, dim); A (dim, d_state); B, C (batch, d_state); D, dt_bias (dim) or NULL.
 * Same elementwise math and (d_state 16) the same C.h order as cl_selective_scan_f32,
 * so a prefill over L tokens followed by k decode steps equals a prefill over L + k
 * tokens bit for bit. */
typedef struct {
  float* state;
  const float* x;
  const float* dt;
  const float* A;
  const float* B;
  const float* C;
  const float* D;       /* may be NULL */
  const float* z;       /* may be NULL */
  const float* dt_bias; /* may be NULL */
  float* out;
  uint64_t batch, dim, d_state;
  int dt_softplus;
} cl_state_update_args;
int cl_selective_state_update_f32(cl_ctx* ctx, const cl_state_update_args* args, void* stream);

/* token_entropy (entropy.hpp:180-210) of a (channels, length) tensor, length contiguous
 * (Mamba u (B, D, L) is channels = B*D): one histogram per position t over its channel
 * slice (slice index c sampled iff c % stride == 0; the slice's Dynamic range or the
 * Fixed range), raw entropies averaged over positions in order.  bin_count <= 4096.
 *
 * One call: d_out (4 doubles) = {raw_nats, normalized, sample_count, nonfinite (0/1,
 * any element)}; scratch belongs to the context. */
int cl_token_entropy_f32(cl_ctx* ctx, const float* d_values, uint64_t channels, uint64_t length,
                         const cl_hist_spec* spec, double* d_out, void* stream);
/* The same as stages, for row-sharded tensors (channel_offset = global index of this
 * rank's first channel; every rank holds all L positions):
 *   cl_token_range_init(d_trange)         d_trange: 2*length + 1 doubles
 *   cl_token_minmax_f32(...)              -> ncclAllReduce(d_trange, 2L+1, ncclDouble, MAX)
 *   zero d_counts (length * bin_count u32)
 *   cl_token_histogram_f32(...)           -> ncclAllReduce(d_counts, L*K, ncclUint32, SUM)
 *   cl_token_entropy_counts(..., samples_per_position = ceil(total_channels / stride)) */
int cl_token_range_init(cl_ctx* ctx, double* d_trange, uint64_t length, void* stream);
int cl_token_minmax_f32(cl_ctx* ctx, const float* d_values, uint64_t channels, uint64_t length,
                        uint64_t channel_offset, uint64_t stride, double* d_trange,
                        void* stream);
int cl_token_histogram_f32(cl_ctx* ctx, const float* d_values, uint64_t channels, uint64_t length,
                           uint64_t channel_offset, const cl_hist_spec* spec,
                           const double* d_trange, uint32_t* d_counts, void* stream);
int cl_token_entropy_counts(cl_ctx* ctx, const uint32_t* d_counts, const double* d_trange,
                            uint64_t length, uint64_t samples_per_position,
                            const cl_hist_spec* spec, double* d_out, void* stream);
/* Device decision from cl_token_entropy_f32's output for rule kind CL_POL_TOKEN_HIST or
 * CL_POL_GUARDED with inner CL_POL_TOKEN_HIST (and any entropy-free kind).  Deferred
 * errors (non-finite input, negative signal) as for cl_decide. */
int cl_decide_token(cl_ctx* ctx, const double* d_token, const cl_hist_spec* spec,
                    const cl_rule_spec* rule, uint64_t seq_len, cl_decision* d_out, void* stream);

/* ------------------------------------------------------------------------ */
/* Host path (synchronous; used by include/chunklab/*.hpp)                    */
/* ------------------------------------------------------------------------ */
/* validate_spec (entropy.hpp:56-62), validate_bounds (chunk.hpp:34-40). */
int cl_validate_hist_spec(cl_ctx* ctx, const cl_hist_spec* spec);
int cl_validate_rule(cl_ctx* ctx, const cl_rule_spec* rule);

/* all_finite over every value (validate_tensor, entropy.hpp:42), on the GPU. */
int cl_all_finite_host(cl_ctx* ctx, const double* h_values, uint64_t n, int* h_all_finite);
/* compute_histogram(span, spec) (entropy.hpp:101-138) on the GPU.  Like the reference's
 * span overload, only the sampled values (index % stride == 0) are checked for
 * finiteness; the tensor overload adds cl_all_finite_host first. */
int cl_compute_histogram_host(cl_ctx* ctx, const double* h_values, uint64_t n,
                              const cl_hist_spec* spec, uint64_t* h_counts, double* h_masses,
                              double* h_lo, double* h_hi, uint64_t* h_sample_count);
/* token_entropy(tensor, spec) (entropy.hpp:180-210) on the GPU, host fp64 values. */
int cl_token_entropy_host(cl_ctx* ctx, const double* h_values, uint64_t channels,
                          uint64_t length, const cl_hist_spec* spec, double* h_raw,
                          double* h_normalized, uint64_t* h_sample_count);
/* estimate_entropy(hist, eps) (entropy.hpp:149-164) on the GPU. */
int cl_estimate_entropy_host(cl_ctx* ctx, const double* h_masses, int bin_count, double epsilon,
                             double* h_raw, double* h_normalized);

/* Scheduler::decide for pre-computed host features (chunk.hpp:256-368), on the GPU.
 * has_* flags mirror std::optional presence (chunk.hpp:185-193). */
typedef struct {
  int has_full_entropy;
  double full_entropy_nats;
  int has_sampled_entropy;
  double sampled_entropy_nats;
  int has_seq_len;
  uint64_t seq_len;
  int has_token_entropy; /* ScheduleFeatures::token_entropy (chunk.hpp:188) */
  double token_entropy_nats;
} cl_features;
int cl_schedule_host(cl_ctx* ctx, const cl_rule_spec* rule, const cl_features* features,
                     cl_decision* h_out);

/* scan_sequential / scan_chunked (scan.hpp:113-136) on the GPU (fp64, bit-exact). */
int cl_scan_f64_host(cl_ctx* ctx, const cl_scan_params_f64* h_params, const double* h_h0,
                     uint64_t chunk, double* h_y, double* h_h);

#ifdef __cplusplus
}
#endif
#endif /* CHUNKLAB_CAPI_H */
